import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth
from paper_1405_7487_b200 import FMM
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4133
pos, q = synth.generate("cube", n, 100 + n, np.float32)
f = FMM(n, 4, 0.5, 32, "f32")
phi, grad = f.solve(torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda())
torch.cuda.synchronize()
print("ok", f.counts(), float(phi.abs().max()))
