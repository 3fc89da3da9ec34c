"""Quick timing probe (not the bench): per-phase CUDA-event times of one config."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_1405_7487_b200 import FMM

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dt = np.float32 if cfg["prec"] == "f32" else np.float64
pos, q = synth.generate(cfg["kind"], cfg["n"], cfg["seed"], dt)
tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
f = FMM(cfg["n"], cfg["P"], cfg["theta"], cfg["ncrit"], cfg["prec"])
for it in range(3):
    f.set_timing(True)
    torch.cuda.synchronize(); t0 = time.time()
    phi, grad = f.solve(tp, tq)
    torch.cuda.synchronize(); t1 = time.time()
    print(it, f"wall {1e3*(t1-t0):.1f} ms", json.dumps({k: round(v, 3) for k, v in f.phase_times().items()}))
print(f.counts())
