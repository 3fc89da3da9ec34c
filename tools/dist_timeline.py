#!/usr/bin/env python
"""Per-rank CUDA-event timeline of the distributed step (fmm_dist_timeline): K ranks of an
in-process group on ONE GPU (host threads; the ranks share the GPU, so absolute times are not a
multi-GPU measurement -- the ORDER and overlap of the spans is what this shows: the LET structure
rounds posted before the local traversal, the LET data after the upward pass, the staying
particles' sort beside the particle exchange).  Also one rank through NCCL (--nccl), the path
bench.py --dist takes.

  python tools/dist_timeline.py [K] [N per rank] [steps]  > profiles/r02_dist_timeline.jsonl
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from bench import weak_offset  # noqa: E402
from paper_1405_7487_b200.dist import DistFMM, LocalGroup, run_ranks  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
P_in, Q_in = [], []
for r in range(K):                       # weak scaling at constant density (bench.py's layout)
    p, q = synth.generate("cube", n, 4, np.float32, start=r * n, n_total=n * K)
    P_in.append(torch.from_numpy((p + weak_offset(r)).astype(np.float32)).cuda())
    Q_in.append(torch.from_numpy(q).cuda())
G = LocalGroup(K)
D = [DistFMM(2 * n, 10, 0.4, 64, "f32", 0, K, r, group=G) for r in range(K)]
streams = [torch.cuda.Stream() for _ in range(K)]
for f in D:
    f.set_timing(True)
for s in range(steps):
    run_ranks(lambda r: D[r].solve(P_in[r], Q_in[r], r * n, reuse_weights=True, stream=streams[r]), K)
    torch.cuda.synchronize()
for r, f in enumerate(D):
    tl = f.timeline()
    st = f.stats()
    print(json.dumps({"rank": r, "K": K, "n_per_rank": n, "step": steps - 1, "timeline_ms": tl,
                      "let_struct_bytes": st["let_struct_bytes"], "let_data_bytes": st["let_data_bytes"],
                      "part_bytes": st["part_bytes"], "n_local": st["n_local"], "npeers": st["npeers"],
                      "note": "K ranks share one GPU (in-process group); spans are CUDA events on the "
                              "stream each ran on, ms after the step began"}), flush=True)
for f in D:
    f.close()
G.close()
