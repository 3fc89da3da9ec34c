"""Kernel microbenchmarks of BASELINE.json configs[4] (one JSON line each).

  P2P: uniform cube, 2^24 targets = sources, ncrit in {32, 64, 128, 256}, the traversal's own P2P
       list at theta = 0.4, fp32 -- the P2P kernels' interactions/s and FP32 roofline fractions.
  M2L: the uniform level-7 octree exactly as configs[4] states it: 2^21 cells
       at geometric centres of the unit cube, the classic interaction list (children of the
       parent's neighbours that are not adjacent: <= 189 sources per cell, 383,233,032 pairs with
       an open boundary), multipoles random with |M_beta| ~ w^|beta| / beta! in cell-width units
       (w = 1/128), fp32 arithmetic, P in {4, 8, 12, 16} -- fed to the product M2L kernels through
       fmm_debug_m2l (the register kernel k_m2l_mir<P>; at P = 12 and 16 its D and L tables exceed the
       register file and spill to local memory).  Checked on sampled targets against per-pair oracle.m2l sums (R14).

Kernel times are the CUDA events libfmm records around each kernel on its stream, averaged over
`--reps` launches after a warm-up.  python tools/microbench.py [--only p2p|m2l] [--reps R] [--P 4,8]
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

LEVEL = 7
G = 1 << LEVEL


def run_p2p(n, ncrit, reps, seed=4):
    pos, q = synth.generate("cube", n, seed, np.float32)
    tp, tq = torch.from_numpy(pos).cuda(), torch.from_numpy(q).cuda()
    f = FMM(n, 4, 0.4, ncrit, "f32")
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
    return c, ph["p2p_kernel"] / reps


def multi_indices(P):
    """R11 order: degree n, then alpha_x descending, then alpha_y descending."""
    out = []
    for n in range(P):
        for a in range(n, -1, -1):
            for b in range(n - a, -1, -1):
                out.append((a, b, n - a - b))
    return np.array(out, dtype=np.int64)


def morton7(x, y, z):
    k = torch.zeros_like(x)
    for l in range(LEVEL):
        k |= ((x >> l) & 1) << (3 * l) | ((y >> l) & 1) << (3 * l + 1) | ((z >> l) & 1) << (3 * l + 2)
    return k


def uniform_grid():
    """Level-7 cells in Morton (key) order: centres, and the classic list as sorted (target, source)."""
    ids = torch.arange(G ** 3, device="cuda", dtype=torch.int64)
    xyz = torch.zeros((G ** 3, 3), dtype=torch.int64, device="cuda")
    for l in range(LEVEL):
        for a in range(3):
            xyz[:, a] |= ((ids >> (3 * l + a)) & 1) << l
    centre = (xyz.double() + 0.5) / G
    # candidate offsets: children of the parent's neighbours -> per axis [-2 - p, 3 - p] for parity p
    r = torch.arange(-3, 4, device="cuda")
    off = torch.stack(torch.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)          # 343
    par = xyz & 1
    lo, hi = -2 - par, 3 - par                                                              # [n, 3]
    srcs = []
    CH = 1 << 18
    for s in range(0, G ** 3, CH):
        t = xyz[s:s + CH]
        o = off[None, :, :]
        ok = ((o >= lo[s:s + CH, None, :]) & (o <= hi[s:s + CH, None, :])).all(-1)
        ok &= (o.abs().max(-1).values > 1)                                                  # not adjacent
        sc = t[:, None, :] + o
        ok &= ((sc >= 0) & (sc < G)).all(-1)
        key = morton7(sc[..., 0].clamp(0, G - 1), sc[..., 1].clamp(0, G - 1), sc[..., 2].clamp(0, G - 1))
        key = torch.where(ok, key, torch.full_like(key, 1 << 40))
        srcs.append(torch.sort(key, dim=1).values[:, :189])
    src = torch.cat(srcs)                                                                   # [n, 189]
    valid = src < (1 << 40)
    tgt = ids[:, None].expand_as(src)
    pairs = torch.stack([tgt[valid], src[valid]], 1).to(torch.int32).contiguous()
    return centre, pairs


def run_m2l_uniform(P, reps, seed=5, check=16):
    centre, pairs = uniform_grid()
    nc = G ** 3
    ex = multi_indices(P)
    deg = ex.sum(1)
    import math
    fact = np.array([math.factorial(int(e[0])) * math.factorial(int(e[1])) * math.factorial(int(e[2])) for e in ex],
                    dtype=np.float64)
    w = 1.0 / G
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    M = torch.rand((nc, len(ex)), generator=gen, dtype=torch.float64, device="cuda") * 2 - 1
    M *= torch.from_numpy(w ** deg / fact).cuda()[None, :]
    level = torch.full((nc,), LEVEL, dtype=torch.int32, device="cuda")
    f = FMM(1, P, 0.4, 64, "f32")
    L = f.debug_m2l(centre, level, M, 0.5, pairs)      # warm-up (and the operand table)
    torch.cuda.synchronize()
    f.set_timing(True)
    f.phase_times(reset=True)
    for _ in range(reps):
        L = f.debug_m2l(centre, level, M, 0.5, pairs)
    torch.cuda.synchronize()
    ms = f.phase_times(reset=True)["m2l_kernel"] / reps
    f.close()
    # check sampled targets against the oracle's R14 (per-pair sums of oracle.m2l)
    err = None
    if check:
        import oracle
        rng = np.random.default_rng(seed)
        tg = rng.choice(nc, check, replace=False)
        tcol = pairs[:, 0].contiguous()
        cen = centre.cpu().numpy()
        errs = []
        for t in tg:
            a = int(torch.searchsorted(tcol, torch.tensor([t], dtype=torch.int32, device="cuda")).item())
            b = int(torch.searchsorted(tcol, torch.tensor([t], dtype=torch.int32, device="cuda"), right=True).item())
            rows = pairs[a:b, 1].long()
            Mh = M[rows].cpu().numpy()
            rows = rows.cpu().numpy()
            ref = np.zeros(len(ex))
            for j, src in enumerate(rows):
                oracle.m2l(P, Mh[j], cen[t] - cen[src], ref)
            Lt = L[t].cpu().numpy()
            for n in range(P):
                k = deg == n
                errs.append(np.abs(Lt[k] - ref[k]).max() / max(np.abs(ref[k]).max(), 1e-300))
        err = float(max(errs))
    return int(pairs.shape[0]), ms, err


def dense_instr(P):
    """SURVEY §8(d) I(P) = C(P+5, 6) FMA + R(P) recurrence ops of the dense R14 form."""
    from math import comb
    R = {4: 119, 8: 897, 10: 1732, 12: 2971, 16: 6981}.get(P)
    return comb(P + 5, 6) + (R or 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", choices=["p2p", "m2l"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--P", default="4,8,12,16")
    a = ap.parse_args()
    build.build()
    pk = peaks()
    lanes = 148 * FP32_LANES_PER_SM * pk["sm_max_mhz"] * 1e6          # FP32 lane-ops / s
    if a.only in (None, "p2p"):
        for ncrit in (32, 64, 128, 256):
            c, ms = run_p2p(1 << 24, ncrit, a.reps)
            ips = c["p2p_interactions"] / (ms * 1e-3)
            print(json.dumps({"micro": "p2p", "kernel": "k_p2p_cta/k_p2p_tma", "N": 1 << 24, "ncrit": ncrit,
                              "mean_leaf": c["n"] / c["nleaf"], "interactions": c["p2p_interactions"],
                              "ms": round(ms, 4), "interactions_per_s": ips,
                              "tflops": ips * P2P_FLOPS / 1e12, "frac_fp32_flops": ips * P2P_FLOPS / (2 * lanes),
                              "frac_fp32_issue": ips * P2P_INSTR / lanes}), flush=True)
    if a.only in (None, "m2l"):
        for P in [int(x) for x in a.P.split(",")]:
            npairs, ms, err = run_m2l_uniform(P, a.reps)
            h = m2l_flops_per_pair(P)
            pps = npairs / (ms * 1e-3)
            kern = f"k_m2l_mir<{P}>" if P in (4, 6, 8, 10, 12, 16) else "k_m2l_generic<float> (scaled)"
            print(json.dumps({"micro": "m2l", "grid": "uniform level 7, 2^21 cells, classic list", "kernel": kern,
                              "P": P, "pairs": npairs, "pairs_per_cell": npairs / G ** 3, "ms": round(ms, 4),
                              "pairs_per_s": pps, "harmonic_flops_per_pair": h["flops"],
                              "tflops_harmonic": pps * h["flops"] / 1e12,
                              "frac_fp32_flops_harmonic": pps * h["flops"] / (2 * lanes),
                              "dense_instr_per_pair": dense_instr(P),
                              "frac_fp32_issue_dense": pps * dense_instr(P) / lanes,
                              "max_rel_err_vs_oracle_by_degree": err}), flush=True)


if __name__ == "__main__":
    main()
