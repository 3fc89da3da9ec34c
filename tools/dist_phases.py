"""Host-timed phases of one DistFMM step (LoopbackComm on one GPU, K virtual ranks)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_1405_7487_b200.dist import DistFMM, LoopbackComm

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 1 << 20
from bench import weak_offset
pos, q = synth.generate("cube", n * K, 2, np.float32)
if len(sys.argv) > 2 and sys.argv[2] == "weak":
    for r in range(K):
        pos[r * n:(r + 1) * n] += weak_offset(r).astype(np.float32)
P_in = [torch.from_numpy(pos[r * n:(r + 1) * n]).cuda() for r in range(K)]
Q_in = [torch.from_numpy(q[r * n:(r + 1) * n]).cuda() for r in range(K)]
D = DistFMM(LoopbackComm(K), n * K, 10, 0.4, 64, "f32")
gb = [r * n for r in range(K)]
for it in range(3):
    t = {}
    torch.cuda.synchronize(); t0 = time.perf_counter()
    lpos, lq, lgid, back, packed, cnt = D.partition(P_in, Q_in, gb, D.weights)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    if len(sys.argv) > 3 and sys.argv[3] == "split":   # the two-exchange flow (build, then evaluate)
        D.build(lpos)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        res = D.evaluate(lpos, lq)
    else:                                              # solve's flow: one exchange, upward overlapped
        res = D.build_evaluate(lpos, lq)
        torch.cuda.synchronize(); t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    wts = [f.work(D.c_m2l, D.alpha)[0] for f in D.fmm]
    torch.cuda.synchronize(); t4 = time.perf_counter()
    out, D.weights = D.gather_back(res, wts, back, packed, cnt, gb, [n] * K)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"K={K} it={it} partition {1e3*(t1-t0):.2f} build {1e3*(t2-t1):.2f} evaluate {1e3*(t3-t2):.2f} "
          f"work {1e3*(t4-t3):.2f} gather {1e3*(t5-t4):.2f} total {1e3*(t5-t0):.2f} ms", D.stats)
for i, f in enumerate(D.fmm):
    c = f.counts()
    print(i, c, "remote:", [f.let_remote(k, with_orig=False)[1:3] for k in range(len(D._peers[i]))])
