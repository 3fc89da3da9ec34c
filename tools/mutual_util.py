"""Lane utilisation of the mutual P2P layout (p2p_mutual.cu) on a bench config: useful
body-body pairs / pairs the warps evaluate (A in chunks of 64*NP targets, B in chunks of 32),
against the one-sided big-leaf layout's.

    python tools/mutual_util.py [config] [NP]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1405_7487_b200.fmm import FMM


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "sph"
    c = synth.CONFIGS[name]
    pos, _ = synth.generate(c["kind"], c["n"], c["seed"], np.float32)
    f = FMM(c["n"], c["P"], c["theta"], c["ncrit"], c["prec"])
    f.build(torch.from_numpy(pos).cuda())
    torch.cuda.synchronize()
    bc = f.cells()["body_count"].astype(np.int64)
    _, p2p = f.lists()
    a, b = p2p[:, 0].astype(np.int64), p2p[:, 1].astype(np.int64)
    m = b > a
    useful = (bc[a[m]] * bc[b[m]]).sum()
    for NP in (2, 4, 5, 6, 8):
        ch = 64 * NP
        cap = (np.ceil(bc[a[m]] / ch) * ch) * (np.ceil(bc[b[m]] / 32) * 32)
        print(f"{name} NP={NP}: chunk {ch}, utilisation {useful / cap.sum():.3f}")
    lv = bc[f.cells()["child_count"] == 0]
    print("leaf sizes: mean", lv.mean(), "percentiles 10/50/90", np.percentile(lv, [10, 50, 90]))
    f.close()


if __name__ == "__main__":
    main()
