"""P2P work per leaf class (tiny <= 16 bodies: warp per leaf; mid; big >= 128: 4 pairs per
thread) for a bench config: leaves, body-body interactions and the share of each class.

    python tools/p2p_classes.py [config]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1405_7487_b200.fmm import FMM


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    c = synth.CONFIGS[name]
    pos, q = synth.generate(c["kind"], c["n"], c["seed"], np.float32)
    f = FMM(c["n"], c["P"], c["theta"], c["ncrit"], c["prec"])
    P = torch.from_numpy(pos).cuda()
    f.build(P)
    torch.cuda.synchronize()
    cells = f.cells()
    _, p2p = f.lists()
    bc = cells["body_count"].astype(np.int64)
    leaf = cells["child_count"] == 0
    per_t = np.bincount(p2p[:, 0], weights=bc[p2p[:, 1]], minlength=len(bc)).astype(np.int64)
    inter = per_t * bc
    cls = np.where(bc <= 16, 0, np.where(bc >= 128, 2, 1))
    tot = inter[leaf].sum()
    print(f"{name}: leaves {leaf.sum()}, interactions {tot:.4e}")
    for k, nm in enumerate(["tiny <=16", "mid", "big >=128"]):
        m = leaf & (cls == k)
        if m.sum() == 0:
            continue
        print(f"  {nm:10s} leaves {m.sum():8d}  mean bodies {bc[m].mean():6.1f}  mean sources/leaf {per_t[m].mean():8.1f}"
              f"  interactions {inter[m].sum():.4e} ({100 * inter[m].sum() / tot:5.1f}%)")
    h = np.bincount(bc[leaf], minlength=65)[:65]
    print("  leaf body-count histogram (0..64):", h.tolist())
    f.close()


if __name__ == "__main__":
    main()
