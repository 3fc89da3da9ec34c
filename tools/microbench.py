"""Kernel microbenchmarks of BASELINE.json configs[4] on the real pipeline (one JSON line each).

  P2P: uniform cube, 2^24 targets = sources, ncrit in {32, 64, 128, 256}, the traversal's own P2P
       list at theta = 0.4, fp32 -- k_p2p_cta interactions/s and its FP32 roofline fraction.
  M2L: uniform cube, 2^21 particles, fp32, theta = 0.4, P in {4, 6, 8, 10} (the register kernel;
       the configs[4] uniform level-7 grid with the classic 189-entry list is stood in for by the
       adaptive traversal's own list on a uniform cube, ~700 pairs per cell) -- k_m2l_fast pairs/s.

Kernel times are the CUDA events libfmm records around each kernel on its stream, averaged over
`--reps` evaluations after warm-up.  python tools/microbench.py [--only p2p|m2l] [--reps R]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from bench import FP32_LANES_PER_SM, P2P_FLOPS, P2P_INSTR, m2l_flops_per_pair, peaks  # noqa: E402
from paper_1405_7487_b200 import FMM, build  # noqa: E402


def run(n, P, ncrit, reps, seed=4):
    pos, q = synth.generate("cube", n, seed, np.float32)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    f = FMM(n, P, 0.4, ncrit, "f32")
    f.build(tp)
    phi = torch.empty(n, device="cuda"); grad = torch.empty((n, 3), device="cuda")
    f.evaluate(tp, tq, phi, grad)
    torch.cuda.synchronize()
    f.set_timing(True)
    f.phase_times(reset=True)
    for _ in range(reps):
        f.evaluate(tp, tq, phi, grad)
    torch.cuda.synchronize()
    ph = f.phase_times(reset=True)
    c = f.counts()
    f.close()
    return c, ph["m2l_kernel"] / reps, ph["p2p_kernel"] / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["p2p", "m2l"])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    build.build()
    pk = peaks()
    lanes = 148 * FP32_LANES_PER_SM * pk["sm_max_mhz"] * 1e6          # FP32 lane-ops / s
    if a.only in (None, "p2p"):
        for ncrit in (32, 64, 128, 256):
            c, _, ms = run(1 << 24, 4, ncrit, a.reps)
            ips = c["p2p_interactions"] / (ms * 1e-3)
            print(json.dumps({"micro": "p2p", "kernel": "k_p2p_cta", "N": 1 << 24, "ncrit": ncrit,
                              "mean_leaf": c["n"] / c["nleaf"], "interactions": c["p2p_interactions"],
                              "ms": round(ms, 4), "interactions_per_s": ips,
                              "tflops": ips * P2P_FLOPS / 1e12, "frac_fp32_flops": ips * P2P_FLOPS / (2 * lanes),
                              "frac_fp32_issue": ips * P2P_INSTR / lanes}), flush=True)
    if a.only in (None, "m2l"):
        for P in (4, 6, 8, 10):
            c, ms, _ = run(1 << 21, P, 64, a.reps)
            w = m2l_flops_per_pair(P)
            pps = c["n_m2l"] / (ms * 1e-3)
            print(json.dumps({"micro": "m2l", "kernel": "k_m2l_fast", "N": 1 << 21, "P": P, "pairs": c["n_m2l"],
                              "pairs_per_cell": c["n_m2l"] / c["ncell"], "ms": round(ms, 4), "pairs_per_s": pps,
                              "flops_per_pair": w["flops"], "tflops": pps * w["flops"] / 1e12,
                              "frac_fp32_flops": pps * w["flops"] / (2 * lanes)}), flush=True)


if __name__ == "__main__":
    main()
