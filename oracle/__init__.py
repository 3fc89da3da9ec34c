"""ctypes wrapper of the plain C fp64 oracle (oracle/fmm_oracle.c).

TEST INFRASTRUCTURE ONLY: importable by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
Parity status of every function: pinned by tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fmm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-ffp-contract=off: expressions evaluated as written)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "fmm_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        i64, i32, dbl, p = C.c_int64, C.c_int, C.c_double, C.c_void_p
        sig = {
            "ofmm_ncoef": (i32, [i32]),
            "ofmm_multi_index": (None, [i32, i32, p]),
            "ofmm_root_cube": (None, [i64, p, p, p, p]),
            "ofmm_keys": (None, [i64, p, p]),
            "ofmm_p2m": (None, [i32, i64, p, p, p, p]),
            "ofmm_m2m": (None, [i32, p, p, p]),
            "ofmm_deriv": (None, [i32, p, p]),
            "ofmm_m2l": (None, [i32, p, p, p]),
            "ofmm_l2l": (None, [i32, p, p, p]),
            "ofmm_l2p": (None, [i32, p, p, i64, p, p, p]),
            "ofmm_p2p": (None, [i64, p, i64, p, p, p, p]),
            "ofmm_direct": (None, [i64, p, p, p, i64, p, p]),
            "ofmm_create": (p, [i64, p, p, i32, dbl, i32]),
            "ofmm_create_in": (p, [i64, p, p, i32, dbl, i32, p]),
            "ofmm_destroy": (None, [p]),
            "ofmm_traverse": (i32, [p]),
            "ofmm_evaluate": (i32, [p, p, i64, p, p]),
            "ofmm_counts": (None, [p, p]),
            "ofmm_sorted": (None, [p, p, p]),
            "ofmm_cells": (None, [p] * 12),
            "ofmm_lists": (None, [p, p, p]),
            "ofmm_expansions": (None, [p, p, p]),
            "ofmm_traverse_pair": (p, [p, p]),
            "ofmm_pairlists_get": (None, [p, p, p, p]),
            "ofmm_pairlists_free": (None, [p]),
            "ofmm_evaluate_multi": (i32, [p, p, i32, p, p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data


def ncoef(P: int) -> int:
    return lib().ofmm_ncoef(P)


def multi_indices(P: int) -> np.ndarray:
    out = np.zeros((ncoef(P), 3), dtype=np.int32)
    e = np.zeros(3, dtype=np.int32)
    for k in range(out.shape[0]):
        lib().ofmm_multi_index(P, k, _ptr(e))
        out[k] = e
    return out


def root_cube(pos):
    pos = _d(pos)
    o = np.zeros(3); s = np.zeros(1); h = np.zeros(1)
    lib().ofmm_root_cube(pos.shape[0], _ptr(pos), _ptr(o), _ptr(s), _ptr(h))
    return o, float(s[0]), float(h[0])


def keys(pos):
    pos = _d(pos)
    k = np.zeros(pos.shape[0], dtype=np.uint64)
    lib().ofmm_keys(pos.shape[0], _ptr(pos), _ptr(k))
    return k


def p2m(P, pos, q, c, M=None):
    pos, q, c = _d(pos), _d(q), _d(c)
    M = np.zeros(ncoef(P)) if M is None else M
    lib().ofmm_p2m(P, pos.shape[0], _ptr(pos), _ptr(q), _ptr(c), _ptr(M))
    return M


def m2m(P, Mc, shift, Mp=None):
    Mc, shift = _d(Mc), _d(shift)
    Mp = np.zeros(ncoef(P)) if Mp is None else Mp
    lib().ofmm_m2m(P, _ptr(Mc), _ptr(shift), _ptr(Mp))
    return Mp


def deriv(P, d):
    d = _d(d)
    D = np.zeros(ncoef(P))
    lib().ofmm_deriv(P, _ptr(d), _ptr(D))
    return D


def m2l(P, M, d, L=None):
    M, d = _d(M), _d(d)
    L = np.zeros(ncoef(P)) if L is None else L
    lib().ofmm_m2l(P, _ptr(M), _ptr(d), _ptr(L))
    return L


def l2l(P, Lp, shift, Lc=None):
    Lp, shift = _d(Lp), _d(shift)
    Lc = np.zeros(ncoef(P)) if Lc is None else Lc
    lib().ofmm_l2l(P, _ptr(Lp), _ptr(shift), _ptr(Lc))
    return Lc


def l2p(P, L, c, pos):
    L, c, pos = _d(L), _d(c), _d(pos)
    n = pos.shape[0]
    phi = np.zeros(n); grad = np.zeros((n, 3))
    lib().ofmm_l2p(P, _ptr(L), _ptr(c), n, _ptr(pos), _ptr(phi), _ptr(grad))
    return phi, grad


def p2p(tpos, spos, sq):
    tpos, spos, sq = _d(tpos), _d(spos), _d(sq)
    phi = np.zeros(tpos.shape[0]); grad = np.zeros((tpos.shape[0], 3))
    lib().ofmm_p2p(tpos.shape[0], _ptr(tpos), spos.shape[0], _ptr(spos), _ptr(sq), _ptr(phi), _ptr(grad))
    return phi, grad


def direct(pos, q, targets=None):
    """O(N^2) direct sum (R1), all particles or the given original indices."""
    pos, q = _d(pos), _d(q)
    n = pos.shape[0]
    t = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    nt = n if t is None else t.shape[0]
    phi = np.zeros(nt); grad = np.zeros((nt, 3))
    lib().ofmm_direct(n, _ptr(pos), _ptr(q), _ptr(t), nt, _ptr(phi), _ptr(grad))
    return phi, grad


class FMM:
    """The whole method on one set of particles: create (R2-R7), traverse (R8-R10), evaluate (R12-R18)."""

    def __init__(self, pos, q, P: int, theta: float, ncrit: int, bounds=None):
        """bounds (lo xyz, hi xyz): the box the R2 root cube is taken from (default: the
        particles' own min/max)."""
        self.pos, self.q = _d(pos).reshape(-1, 3), _d(q).reshape(-1)
        self.n, self.P = self.pos.shape[0], P
        self._bounds = None if bounds is None else _d(bounds).reshape(6)
        self._h = lib().ofmm_create_in(self.n, _ptr(self.pos), _ptr(self.q), P, float(theta), ncrit,
                                       None if self._bounds is None else _ptr(self._bounds))
        if not self._h:
            raise ValueError("oracle rejected arguments")
        self._traversed = False

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ofmm_destroy(h)
            self._h = None

    def traverse(self):
        if lib().ofmm_traverse(self._h) != 0:
            raise RuntimeError("oracle traversal produced duplicate pairs")
        self._traversed = True
        return self

    def evaluate(self, targets=None):
        if not self._traversed:
            self.traverse()
        t = None if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
        nt = self.n if t is None else t.shape[0]
        phi = np.zeros(nt); grad = np.zeros((nt, 3))
        rc = lib().ofmm_evaluate(self._h, _ptr(t), nt, _ptr(phi), _ptr(grad))
        if rc != 0:
            raise RuntimeError(f"oracle evaluate failed ({rc})")
        return phi, grad

    def counts(self) -> dict:
        c = np.zeros(6, dtype=np.int64)
        lib().ofmm_counts(self._h, _ptr(c))
        return dict(zip(["ncell", "nleaf", "depth", "n_m2l", "n_p2p", "p2p_interactions"], map(int, c)))

    def sorted(self):
        k = np.zeros(self.n, dtype=np.uint64); p = np.zeros(self.n, dtype=np.uint32)
        lib().ofmm_sorted(self._h, _ptr(k), _ptr(p))
        return k, p

    def cells(self) -> dict:
        nc = self.counts()["ncell"]
        out = dict(level=np.zeros(nc, np.int32), key=np.zeros(nc, np.uint64),
                   body_begin=np.zeros(nc, np.uint32), body_count=np.zeros(nc, np.uint32),
                   child_begin=np.zeros(nc, np.uint32), child_count=np.zeros(nc, np.uint32),
                   parent=np.zeros(nc, np.int32), bmin=np.zeros((nc, 3)), bmax=np.zeros((nc, 3)),
                   center=np.zeros((nc, 3)), radius=np.zeros(nc))
        order = ["level", "key", "body_begin", "body_count", "child_begin", "child_count", "parent",
                 "bmin", "bmax", "center", "radius"]
        lib().ofmm_cells(self._h, *[_ptr(out[k]) for k in order])
        return out

    def lists(self):
        c = self.counts()
        m2l = np.zeros((c["n_m2l"], 2), dtype=np.uint32)
        p2p = np.zeros((c["n_p2p"], 2), dtype=np.uint32)
        lib().ofmm_lists(self._h, _ptr(m2l), _ptr(p2p))
        return m2l, p2p

    def expansions(self):
        nc = self.counts()["ncell"]
        M = np.zeros((nc, ncoef(self.P))); L = np.zeros((nc, ncoef(self.P)))
        lib().ofmm_expansions(self._h, _ptr(M), _ptr(L))
        return M, L


def traverse_pair(T: "FMM", S: "FMM"):
    """Per-partition mode: canonical (target in T, source in S) M2L and P2P lists."""
    h = lib().ofmm_traverse_pair(T._h, S._h)
    c = np.zeros(2, dtype=np.int64)
    lib().ofmm_pairlists_get(h, _ptr(c), None, None)
    m2l = np.zeros((c[0], 2), dtype=np.uint32); p2p = np.zeros((c[1], 2), dtype=np.uint32)
    lib().ofmm_pairlists_get(h, _ptr(c), _ptr(m2l), _ptr(p2p))
    lib().ofmm_pairlists_free(h)
    return m2l, p2p


def evaluate_multi(T: "FMM", sources):
    """phi/grad of T's particles (T's input order) with sources T and every tree in `sources`."""
    if not T._traversed:
        T.traverse()
    arr = (C.c_void_p * max(len(sources), 1))(*[s._h for s in sources])
    phi = np.zeros(T.n); grad = np.zeros((T.n, 3))
    rc = lib().ofmm_evaluate_multi(T._h, arr, len(sources), _ptr(phi), _ptr(grad))
    if rc != 0:
        raise RuntimeError(f"oracle evaluate_multi failed ({rc})")
    return phi, grad


def rel_l2(a, b) -> float:
    """Q21: ||a - b||_2 / ||b||_2 (b = the reference)."""
    a = np.asarray(a, dtype=np.float64).ravel(); b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a - b))
