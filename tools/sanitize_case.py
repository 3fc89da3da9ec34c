#!/usr/bin/env python
"""Small c2-shaped cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the default fp32 path (TMA P2P, mirror M2L, target-ordered traversal, onesweep sort) on a
uniform cube and on an adaptive Plummer cloud (every P2P leaf class), plus the fp64 path.

  compute-sanitizer --tool racecheck python tools/sanitize_case.py [small]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1405_7487_b200 import FMM  # noqa: E402

small = len(sys.argv) > 1 and sys.argv[1] == "small"
cases = [("cube", 1 << (13 if small else 15), 10, 0.4, 64, "f32"),
         ("plummer", 6000 if small else 20000, 10, 0.4, 64, "f32"),
         ("plummer", 3000, 6, 0.4, 16, "f64")]
for kind, n, P, theta, ncrit, prec in cases:
    dt = np.float32 if prec == "f32" else np.float64
    pos, q = synth.generate(kind, n, 7, dt)
    f = FMM(n, P, theta, ncrit, prec)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    for _ in range(2):                     # first build and the size-learning rebuild
        phi, grad = f.solve(tp, tq)
    torch.cuda.synchronize()
    print(kind, n, prec, f.counts(), float(phi.abs().max()), flush=True)
    f.close()
print("sanitize_case done")
