"""Per-phase times of one single-GPU FMM on a cube of N particles (fp32, P=10, theta=0.4, ncrit=64)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1405_7487_b200 import FMM
n = int(sys.argv[1])
pos, q = synth.generate("cube", n, 2, np.float32)
tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
f = FMM(n, 10, 0.4, 64, "f32")
for it in range(3):
    f.set_timing(True)
    torch.cuda.synchronize(); t0 = time.time()
    f.solve(tp, tq)
    torch.cuda.synchronize(); t1 = time.time()
    print(it, f"wall {1e3*(t1-t0):.1f} ms", json.dumps({k: round(v, 2) for k, v in f.phase_times().items()}))
print(f.counts())
