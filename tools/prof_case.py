#!/usr/bin/env python
"""Small profiling driver: `reps` fmm_solve calls of one BASELINE config (default c2) -- the
command ncu wraps (ncu --set full -k regex:<kernel> -s <skip> -c <n> python tools/prof_case.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1405_7487_b200 import FMM, build  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
build.build()
pos, q = synth.generate(cfg["kind"], cfg["n"], cfg["seed"], np.float32 if cfg["prec"] == "f32" else np.float64)
f = FMM(cfg["n"], cfg["P"], cfg["theta"], cfg["ncrit"], cfg["prec"])
tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
for _ in range(reps):
    phi, grad = f.solve(tp, tq)
torch.cuda.synchronize()
print("prof_case done", cfg["n"], float(phi.abs().max()))
