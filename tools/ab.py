#!/usr/bin/env python
"""A/B timing of library switches: for each ENV=value setting (comma-separated groups separated by
spaces), a fresh context runs `reps` fmm_solve calls of one BASELINE config after warm-up; prints
the step time and the per-phase CUDA-event times (ms).

  python tools/ab.py c2 10 "FMM_P2P_TMA=0" "FMM_P2P_TMA=1" ...
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1405_7487_b200 import FMM, build  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2])
build.build()
pos, q = synth.generate(cfg["kind"], cfg["n"], cfg["seed"], np.float32 if cfg["prec"] == "f32" else np.float64)
tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ref = None
for setting in sys.argv[3:]:
    env = dict(kv.split("=") for kv in setting.split(",") if kv)
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    f = FMM(cfg["n"], cfg["P"], cfg["theta"], cfg["ncrit"], cfg["prec"])
    for _ in range(3):
        phi, grad = f.solve(tp, tq)
    torch.cuda.synchronize()
    f.set_timing(True)
    f.phase_times(reset=True)
    ms = 0.0
    s = torch.cuda.current_stream()
    for i in range(reps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        phi, grad = f.solve(tp, tq)
        b.record(s)
        b.synchronize()
        ms += a.elapsed_time(b)
    ph = f.phase_times(reset=True)
    out = phi.double().cpu().numpy()
    if ref is None:
        ref = out
    rel = float(np.linalg.norm(out - ref) / np.linalg.norm(ref))
    for k, v in old.items():   # the setting stays in the environment while its context runs
        if v is None:
            del os.environ[k]
        else:
            os.environ[k] = v
    print(json.dumps({"setting": setting, "ms_step": round(ms / reps, 4),
                      "phases": {k: round(v / reps, 4) for k, v in ph.items() if v > 0},
                      "phi_rel_vs_first": rel}), flush=True)
    f.close()
