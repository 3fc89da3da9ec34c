"""Algorithmic work counts of the two hot kernels (bench roofline, Eq. (1) cost ratio)."""
from __future__ import annotations

# 18 FP32 flops (FFMA = 2) + 1 MUFU rsqrt per interaction:
# 3 sub, |r|^2 (1 mul + 2 fma = 5), q/r (1 mul), phi add (1), 1/r^2 and q/r^3 (2 mul), grad (3 fma = 6)
P2P_FLOPS = 18
P2P_INSTR = 13      # FP32-pipe lane-ops per interaction (SASS, -ftz)


def t2n(P):
    return P * (P + 1) // 2


def m2l_flops_per_pair(P: int) -> dict:
    """Algorithmic FP work of one M2L pair in the harmonic form the kernel evaluates
    (m2l_fast.cu; FMA = 2 flops).  Returns flops and lane-instruction counts."""
    fma = 0
    # contraction: S0.D0 -> L0, S0.D1 -> L1, S1.D1 -> L0, N.D0 -> L1
    for m in range(P):                 # S0 element of degree m (m+1 of them)
        fma += (m + 1) * (t2n(P - m) + t2n(P - 1 - m))
    for m in range(P - 1):             # S1
        fma += (m + 1) * t2n(P - 1 - m)
    for m in range(2, P):              # N
        fma += (m + 1) * t2n(P - m)
    # recurrence: per D entry ~ (terms) multiply-adds; count exactly as the kernel forms it
    rec_instr = 0
    for n in range(1, P):
        for z in range(n + 1):         # D0 entries of degree n
            y = n - z
            t1 = (y > 0) + (z > 0)
            t2 = (y > 1) + (z > 1)
            rec_instr += t1 + t2 + (2 if n > 1 else 1)
        for z in range(n):             # D1 entries of degree n
            y = n - 1 - z
            t1 = 1 + (y > 0) + (z > 0)
            t2 = (y > 1) + (z > 1)
            rec_instr += t1 + t2 + (2 if n > 1 else 1)
    rec_instr += 2 * (P - 1) + 3 * P + 6   # m*u tables, per-degree A/B, r2, rcp, rsqrt
    return {"fma": fma, "rec_instr": rec_instr, "instr": fma + rec_instr, "flops": 2 * fma + 2 * rec_instr}



def m2l_cost_ratio(P: int) -> float:
    """Cost of one M2L pair in P2P interactions (FP32 lane-op model), the c_m2l of fmm_work."""
    return m2l_flops_per_pair(P)["instr"] / P2P_INSTR
