"""One P2P evaluation at small leaves (2^22 cube, ncrit 32: mean leaf 8) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1405_7487_b200 import FMM
n = 1 << 22
pos, q = synth.generate("cube", n, 4, np.float32)
tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
f = FMM(n, 4, 0.4, int(sys.argv[1]) if len(sys.argv) > 1 else 32, "f32")
f.solve(tp, tq)
torch.cuda.synchronize()
print(f.counts())
