#!/usr/bin/env python
"""Tensor-core M2L experiment on BASELINE configs[4]'s uniform level-7 grid (tools/m2l_tc.cu): the
classic-list M2L as degree-block GEMMs with shared per-displacement operators, in FP32 (CUDA
cores), TF32 and BF16x9-emulated FP32 (tensor cores), checked on sampled targets against per-pair
oracle.m2l sums (R14).  One JSON line per (P, precision).

  python tools/m2l_tc.py [--P 4,8,12,16] [--reps 3]
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

SRC = os.path.join(ROOT, "tools", "m2l_tc.cu")
LIB = os.path.join(ROOT, "tools", "libm2ltc.so")
G = 128


def build():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-std=c++17", "-shared", "-Xcompiler", "-fPIC", SRC, "-o", LIB,
                               "-L/usr/local/cuda/lib64", "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-lcublas"])
    L = C.CDLL(LIB)
    L.m2ltc_setup.argtypes = [C.c_int, C.c_uint64]
    L.m2ltc_run.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_float)]
    L.m2ltc_rows.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    return L


def morton(x, y, z):
    k = 0
    for l in range(7):
        k |= ((x >> l) & 1) << (3 * l) | ((y >> l) & 1) << (3 * l + 1) | ((z >> l) & 1) << (3 * l + 2)
    return k


def sources(x, y, z):
    out = []
    p = (x & 1, y & 1, z & 1)
    for vz in range(-2 - p[2], 4 - p[2]):
        for vy in range(-2 - p[1], 4 - p[1]):
            for vx in range(-2 - p[0], 4 - p[0]):
                if max(abs(vx), abs(vy), abs(vz)) <= 1:
                    continue
                s = (x + vx, y + vy, z + vz)
                if all(0 <= c < G for c in s):
                    out.append(s)
    return out


def check(L, P, nt=12, seed=3):
    import oracle
    nco = P * (P + 1) * (P + 2) // 6
    deg = np.array([n for n in range(P) for _ in range((n + 1) * (n + 2) // 2)])
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(nt):
        x, y, z = (int(v) for v in rng.integers(0, G, 3))
        srcs = sources(x, y, z)
        ids = np.array([morton(*s) for s in srcs], dtype=np.int64)
        Ms = np.zeros((len(ids), nco))
        assert L.m2ltc_rows(0, len(ids), ids.ctypes.data, Ms.ctypes.data) == 0
        tid = np.array([morton(x, y, z)], dtype=np.int64)
        Lt = np.zeros(nco)
        assert L.m2ltc_rows(1, 1, tid.ctypes.data, Lt.ctypes.data) == 0
        ct = (np.array([x, y, z]) + 0.5) / G
        ref = np.zeros(nco)
        for s, M in zip(srcs, Ms):
            oracle.m2l(P, M, ct - (np.array(s) + 0.5) / G, ref)
        for n in range(P):
            k = deg == n
            worst = max(worst, float(np.abs(Lt[k] - ref[k]).max() / np.abs(ref[k]).max()))
    return worst


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", default="4,8,12,16")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="0,1,2")
    a = ap.parse_args()
    L = build()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        pk = json.load(f)
    fp32_tf = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
    names = {0: "FP32 (cuBLAS SIMT)", 1: "TF32 tensor cores", 2: "FP32 emulated BF16x9 tensor cores"}
    from math import comb
    for P in [int(x) for x in a.P.split(",")]:
        rc = L.m2ltc_setup(P, 12345)
        if rc != 0:
            print(json.dumps({"micro": "m2l_tc", "P": P, "setup_error": rc}), flush=True)
            continue
        npairs = 383233032
        for mode in [int(x) for x in a.modes.split(",")]:
            ms = C.c_float()
            rc = L.m2ltc_run(mode, a.reps, C.byref(ms))
            if rc != 0:
                print(json.dumps({"micro": "m2l_tc", "P": P, "precision": names[mode], "error": rc}), flush=True)
                continue
            err = check(L, P)
            grouped = bool(L.m2ltc_grouped())
            fl = 2 * comb(P + 5, 6)                      # dense degree-block contraction, FMA = 2
            pps = npairs / (ms.value * 1e-3)
            print(json.dumps({"micro": "m2l_tc", "grid": "uniform level 7, 2^21 cells, classic list", "P": P,
                              "precision": names[mode], "pairs": npairs, "ms": round(ms.value, 3),
                              "pairs_per_s": pps, "gemm_flops_per_pair": fl,
                              "tflops_dense": pps * fl / 1e12, "frac_fp32_cuda_core_peak": pps * fl / 1e12 / fp32_tf,
                              "max_rel_err_vs_oracle_by_degree": err,
                              "calls": "one grouped GEMM call per displacement" if grouped else
                                       "one cuBLAS GEMM per (class, displacement, degree)"}), flush=True)


if __name__ == "__main__":
    main()
