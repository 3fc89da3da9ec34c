"""Build the tree + lists of a bench config twice and bracket the second build with
cudaProfilerStart/Stop, for `ncu --profile-from-start off` captures of the traversal kernels.

    ncu --profile-from-start off -k regex:k_tct_level ... python tools/prof_build.py c3
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1405_7487_b200.fmm import FMM


def main():
    c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
    pos, _ = synth.generate(c["kind"], c["n"], c["seed"], np.float32)
    f = FMM(c["n"], c["P"], c["theta"], c["ncrit"], c["prec"])
    P = torch.from_numpy(pos).cuda()
    f.build(P)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    f.build(P)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f.counts())
    f.close()


if __name__ == "__main__":
    main()
