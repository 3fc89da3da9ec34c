"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds ONLY random-number generation and the particle distributions the
paper names (§III-A "Cube", "Sphere", "Plummer"; Table I).
It contains none of the FMM's arithmetic, so both sides may import it.

Generator: SplitMix64, counter based.  Particle i draws the four
64-bit words at counters 4i, 4i+1, 4i+2, 4i+3; a double in [0,1) is (h >> 11) * 2^-53.
fp32 inputs are the fp64 draws rounded to nearest (numpy astype).

Distributions:
  cube     x,y,z = u0,u1,u2 in [0,1)^3, q = 2*u3 - 1 in [-1,1)   (BASELINE.json configs[0,1,3,4])
  plummer  scale radius a=1, radius truncated at 100 by exact inverse transform
           r = a / sqrt(u^(-2/3) - 1), u = u0 * m(100), m(r) = r^3/(r^2+1)^(3/2);
           isotropic direction cos(t) = 2*u1-1, phi = 2*pi*u2; q = 1/N  (configs[2]; Q18)
  sphere   unit sphere surface, same direction rule, q = 2*u3 - 1   (Table I case 2)
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

KINDS = ("cube", "plummer", "sphere")


def splitmix64(seed: int, counters: np.ndarray) -> np.ndarray:
    """SplitMix64 output for the given counters: mix(seed + (c+1)*GOLDEN)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (counters.astype(np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, counters: np.ndarray) -> np.ndarray:
    """Doubles in [0,1) from 53 random bits."""
    return (splitmix64(seed, counters) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _draws(n: int, seed: int, start: int = 0) -> np.ndarray:
    c = np.arange(4 * start, 4 * (start + n), dtype=np.uint64)
    return uniform01(seed, c).reshape(n, 4)


def generate(kind: str, n: int, seed: int, dtype=np.float64, start: int = 0, n_total: int = None):
    """Return (pos[n,3], q[n]) as C-contiguous arrays of `dtype` (float64 or float32).

    Particles start .. start+n-1 of an n_total-particle set (default: the whole set of n),
    so that ranks of a multi-GPU run can each draw their own slice of one global set."""
    if kind not in KINDS:
        raise ValueError(f"unknown distribution {kind!r}; expected one of {KINDS}")
    if n < 0 or start < 0:
        raise ValueError("n and start must be >= 0")
    n_total = n if n_total is None else n_total
    u = _draws(n, seed, start)
    if kind == "cube":
        pos = u[:, :3].copy()
        q = 2.0 * u[:, 3] - 1.0
    else:
        cth = 2.0 * u[:, 1] - 1.0
        sth = np.sqrt(np.maximum(0.0, 1.0 - cth * cth))
        ph = 2.0 * np.pi * u[:, 2]
        if kind == "sphere":
            r = np.ones(n)
            q = 2.0 * u[:, 3] - 1.0
        else:
            rmax = 100.0
            mmax = rmax ** 3 / (rmax ** 2 + 1.0) ** 1.5
            m = u[:, 0] * mmax
            with np.errstate(divide="ignore"):
                r = np.where(m > 0.0, 1.0 / np.sqrt(np.maximum(m, 1e-300) ** (-2.0 / 3.0) - 1.0), 0.0)
            q = np.full(n, 1.0 / max(n_total, 1))
        pos = np.stack([r * sth * np.cos(ph), r * sth * np.sin(ph), r * cth], axis=1)
    pos = np.ascontiguousarray(pos.astype(dtype))
    q = np.ascontiguousarray(q.astype(dtype))
    return pos, q


def sample_targets(n: int, k: int, seed: int) -> np.ndarray:
    """k distinct indices in [0,n) by partial Fisher-Yates with SplitMix64 stream `seed+1000` (Q20).

    Returned in ascending order (int64)."""
    k = min(k, n)
    perm = {}
    out = np.empty(k, dtype=np.int64)
    r = splitmix64(seed + 1000, np.arange(k, dtype=np.uint64))
    for i in range(k):
        j = i + int(r[i] % np.uint64(n - i))
        vi = perm.get(i, i)
        vj = perm.get(j, j)
        perm[i], perm[j] = vj, vi
        out[i] = vj
    out.sort()
    return out


# Workload recipes of BASELINE.json configs (seeds per Q19).
CONFIGS = {
    "c1": dict(kind="cube", n=4096, P=4, theta=0.5, ncrit=32, prec="f64", seed=1),
    "c2": dict(kind="cube", n=1 << 20, P=10, theta=0.4, ncrit=64, prec="f32", seed=2),
    "c3": dict(kind="plummer", n=10_000_000, P=10, theta=0.4, ncrit=64, prec="f32", seed=3),
    # configs[3] on one GPU: the strong-scaling problem (N = 2^26, Q24) and the weak-scaling
    # per-GPU size (2^24); same parameters as c2
    "c4s": dict(kind="cube", n=1 << 26, P=10, theta=0.4, ncrit=64, prec="f32", seed=4),
    "c4w": dict(kind="cube", n=1 << 24, P=10, theta=0.4, ncrit=64, prec="f32", seed=4),
    # Table I case 2: sphere surface, P=10, theta=0.4, ncrit=512
    "sph": dict(kind="sphere", n=1 << 22, P=10, theta=0.4, ncrit=512, prec="f32", seed=5),
    # configs[4] P2P microbench leaf sizes at a smaller N (ncrit 32: mean leaf 8), for A/B runs
    "c5n32": dict(kind="cube", n=1 << 22, P=4, theta=0.4, ncrit=32, prec="f32", seed=4),
}
