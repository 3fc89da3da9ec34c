"""Multi-GPU FMM: thin ctypes binding of libfmm's distributed driver.

The library owns the whole distributed step (csrc/dist.cu, include/fmm.h "multi-GPU driver"):
the communicator (NCCL from a 128-byte unique id, or an in-process group of K ranks on host
threads), the Morton-range / ORB partition arithmetic, the Eq. (1) weights and alpha search,
the particle and LET exchanges and their overlap with the traversal.  This module only
marshals arguments:

* `DistFMM`       -- one rank's context (fmm_create_dist) with `solve()` (fmm_dist_solve) and the
                     introspection of the single-GPU `FMM` (its local tree, lists, LET regions);
* `LocalGroup`    -- fmm_group: K ranks of one process (one host thread per rank) -- several GPUs
                     of a process, or K ranks on one GPU in the parity tests (no kernel waits for
                     another rank's kernel: the host threads meet at barriers);
* `nccl_unique_id`-- fmm_dist_unique_id (rank 0 makes it; the caller broadcasts the 128 bytes
                     with its process group, e.g. torch.distributed.broadcast_object_list);
* `partition_splitters`, `orb_plan`, `AlphaTuner` -- the driver's host rules (fmm_splitters,
                     fmm_orb_plan, fmm_alpha_tuner_*), callable without a device (CPU tests).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from .fmm import FMM, FMMError, FMM_ERR_ARG, F32, F64, HIST_FN, ORB_HIST_FN, ORB_SPLIT_FN, _np_ptr, lib

PART = {"morton": 0, "orb": 1}
HIST_BITS = 16


class DistStats(C.Structure):
    _fields_ = [("bounds", C.c_double * 6), ("alpha", C.c_double), ("c_m2l", C.c_double), ("n_local", C.c_int64),
                ("npeers", C.c_int32), ("tuner_probes", C.c_int32), ("let_struct_bytes", C.c_int64),
                ("let_data_bytes", C.c_int64), ("part_bytes", C.c_int64), ("work_local", C.c_double),
                ("work_remote", C.c_double), ("tuner_converged", C.c_int32), ("pad", C.c_int32),
                ("tuner_best", C.c_double)]



def _check(st, what):
    if st != 0:
        raise FMMError(st, what)


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for fmm_create_dist."""
    buf = C.create_string_buffer(128)
    _check(lib().fmm_dist_unique_id(buf), "fmm_dist_unique_id")
    return buf.raw


class LocalGroup:
    """fmm_group: K ranks inside this process (create K DistFMM with group=this, run their solve()
    on K threads, e.g. with run_ranks)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        _check(lib().fmm_group_create(int(nranks), C.byref(h)), "fmm_group_create")
        self._h, self.nranks = h, nranks

    def close(self):
        if getattr(self, "_h", None):
            if lib().fmm_group_destroy(self._h) == 0:
                self._h = None

    def __del__(self):
        self.close()


def run_ranks(fn, nranks: int):
    """fn(rank) on one host thread per rank (libfmm calls release the GIL); re-raises the first error."""
    out, errs = [None] * nranks, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:   # noqa: BLE001 -- propagated below
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return out


class DistFMM(FMM):
    """One rank of the distributed FMM (fmm_create_dist).  Exactly one of unique_id (NCCL) /
    group (LocalGroup).  solve(pos, q, gid_base) -> (phi, grad) for this rank's particles."""

    def __init__(self, n_local_max: int, P: int, theta: float, ncrit: int, prec: str = "f32", device: int = 0,
                 nranks: int = 1, rank: int = 0, unique_id: bytes = None, group: LocalGroup = None,
                 partitioner: str = "morton"):
        if (unique_id is None) == (group is None):
            raise FMMError(FMM_ERR_ARG, "give exactly one of unique_id (NCCL) or group (LocalGroup)")
        if partitioner not in PART:
            raise FMMError(FMM_ERR_ARG, "partitioner must be 'morton' or 'orb'")
        self.prec = {"f32": F32, "f64": F64}[prec]
        self.P, self.theta, self.ncrit, self.device = P, theta, ncrit, device
        self.nranks, self.rank, self.partitioner = nranks, rank, partitioner
        self._group = group          # keeps the group alive while this context exists
        uid = None if unique_id is None else C.create_string_buffer(bytes(unique_id), 128)
        h = C.c_void_p()
        st = lib().fmm_create_dist(int(n_local_max), int(P), float(theta), int(ncrit), self.prec, int(device),
                                   int(nranks), int(rank), uid, None if group is None else group._h,
                                   PART[partitioner], C.byref(h))
        if st != 0:
            raise FMMError(st, "fmm_create_dist")
        self._h = h
        self._pos = None

    def solve(self, pos, q, gid_base: int = 0, reuse_weights: bool = False, phi=None, grad=None, stream=None):
        import torch
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        self._check_tensor(q, (n,), "q")
        phi = torch.empty(n, dtype=self.dtype, device=pos.device) if phi is None else phi
        grad = torch.empty((n, 3), dtype=self.dtype, device=pos.device) if grad is None else grad
        self._check_tensor(phi, (n,), "phi")
        self._check_tensor(grad, (n, 3), "grad")
        self._check(lib().fmm_dist_solve(self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()), n,
                                         int(gid_base), int(bool(reuse_weights)), C.c_void_p(phi.data_ptr()),
                                         C.c_void_p(grad.data_ptr()), C.c_void_p(self._stream(stream))),
                    "fmm_dist_solve")
        self._pos = None
        self.n = self.stats()["n_local"]      # the local tree's particle count (FMM.work, introspection)
        return phi, grad

    def set_weights(self, w=None):
        n = 0 if w is None else w.shape[0]
        self._check(lib().fmm_set_weights(self._h, None if w is None else C.c_void_p(w.data_ptr()), n),
                    "fmm_set_weights")

    def set_alpha(self, alpha: float, c_m2l: float = 0.0):
        self._check(lib().fmm_dist_set_alpha(self._h, float(alpha), float(c_m2l)), "fmm_dist_set_alpha")

    def tune_alpha(self, lo: float = 1.0 / 16, hi: float = 16.0, tol: float = 0.1):
        self._check(lib().fmm_dist_tune_alpha(self._h, float(lo), float(hi), float(tol)), "fmm_dist_tune_alpha")

    def stats(self) -> dict:
        s = DistStats()
        self._check(lib().fmm_dist_get_stats(self._h, C.byref(s)), "fmm_dist_get_stats")
        d = {k: getattr(s, k) for k, _ in DistStats._fields_ if k != "pad"}
        d["bounds"] = np.array(list(s.bounds))
        return d

    @property
    def alpha(self) -> float:
        return self.stats()["alpha"]

    def local(self):
        """(global ids of this rank's particles in local order, peers in LET graft order)."""
        nl = self.stats()["n_local"]
        gid = np.zeros(nl, np.int64)
        peers = np.zeros(self.nranks, np.int32)
        self._check(lib().fmm_dist_local(self._h, _np_ptr(gid), _np_ptr(peers)), "fmm_dist_local")
        return gid, [int(p) for p in peers if p >= 0]

    def weights(self, n: int) -> np.ndarray:
        w = np.zeros(n, np.float32)
        self._check(lib().fmm_dist_weights(self._h, _np_ptr(w)), "fmm_dist_weights")
        return w

    def orb_boxes(self) -> np.ndarray:
        b = np.zeros((self.nranks, 6), np.int32)
        self._check(lib().fmm_dist_orb_boxes(self._h, _np_ptr(b)), "fmm_dist_orb_boxes")
        return b

    def timeline(self) -> dict:
        ms = np.zeros((32, 2))
        k = C.c_int()
        self._check(lib().fmm_dist_timeline(self._h, _np_ptr(ms), 32, C.byref(k)), "fmm_dist_timeline")
        return {lib().fmm_dist_timeline_name(i).decode(): (float(ms[i, 0]), float(ms[i, 1])) for i in range(k.value)}


# ------------------------------------------------------------------ host rules (no device)
def partition_splitters(hist_fn, nranks: int, bits: int = HIST_BITS, tol: float = 1.0 / 512) -> np.ndarray:
    """fmm_splitters with a Python histogram: hist_fn(prefixes, prefix_bits, bits) -> [len, 2^bits]
    GLOBAL weights.  Returns the K-1 splitter keys (uint64)."""
    def cb(_user, pre, npre, pbits, b, out):
        try:
            h = np.asarray(hist_fn([int(pre[i]) for i in range(npre)], pbits, b), dtype=np.float64)
            C.memmove(out, h.ctypes.data, h.size * 8)
            return 0
        except Exception:   # noqa: BLE001 -- reported as a failed call
            return 1
    spl = np.zeros(max(nranks - 1, 1), np.uint64)
    _check(lib().fmm_splitters(int(nranks), int(bits), float(tol), HIST_FN(cb), None, _np_ptr(spl)), "fmm_splitters")
    return spl[:nranks - 1]


def orb_plan(hist_fn, split_fn, nranks: int, bits: int = HIST_BITS) -> dict:
    """fmm_orb_plan with Python callbacks: hist_fn(axis[K], prefix[K], prefix_bits, bits) -> [K, 2^bits]
    global weights; split_fn(axis, cut, right).  Returns {rank: {"lo": [3], "hi": [3]}}."""
    K = nranks

    def hcb(_u, axis, prefix, pbits, b, out):
        try:
            h = np.asarray(hist_fn(np.ctypeslib.as_array(axis, (K,)).copy(), np.ctypeslib.as_array(prefix, (K,)).copy(),
                                   pbits, b), dtype=np.float64)
            C.memmove(out, h.ctypes.data, h.size * 8)
            return 0
        except Exception:   # noqa: BLE001
            return 1

    def scb(_u, axis, cut, right):
        try:
            split_fn(np.ctypeslib.as_array(axis, (K,)).copy(), np.ctypeslib.as_array(cut, (K,)).copy(),
                     np.ctypeslib.as_array(right, (K,)).copy())
            return 0
        except Exception:   # noqa: BLE001
            return 1
    boxes = np.zeros((K, 6), np.int32)
    _check(lib().fmm_orb_plan(int(K), int(bits), ORB_HIST_FN(hcb), ORB_SPLIT_FN(scb), None, _np_ptr(boxes)),
           "fmm_orb_plan")
    return {r: {"lo": [int(x) for x in boxes[r, :3]], "hi": [int(x) for x in boxes[r, 3:]]} for r in range(K)}


class AlphaTuner:
    """fmm_alpha_tuner_*: golden-section search of Eq. (1)'s alpha over time steps."""

    def __init__(self, lo: float = 1.0 / 16, hi: float = 16.0, tol: float = 0.1):
        if not (0 < lo < hi):
            raise ValueError("need 0 < lo < hi")
        h = C.c_void_p()
        _check(lib().fmm_alpha_tuner_create(float(lo), float(hi), float(tol), C.byref(h)), "fmm_alpha_tuner_create")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib().fmm_alpha_tuner_destroy(self._h)
            self._h = None

    def next_alpha(self) -> float:
        return float(lib().fmm_alpha_tuner_next(self._h))

    def report(self, runtime: float) -> None:
        _check(lib().fmm_alpha_tuner_report(self._h, float(runtime)), "fmm_alpha_tuner_report")

    def _state(self):
        conv, best, nh = C.c_int(), C.c_double(), C.c_int()
        _check(lib().fmm_alpha_tuner_state(self._h, C.byref(conv), C.byref(best), C.byref(nh), None, 0),
               "fmm_alpha_tuner_state")
        hist = np.zeros((max(nh.value, 1), 2))
        _check(lib().fmm_alpha_tuner_state(self._h, None, None, None, _np_ptr(hist), nh.value), "fmm_alpha_tuner_state")
        return bool(conv.value), best.value, [tuple(x) for x in hist[:nh.value]]

    @property
    def converged(self) -> bool:
        return self._state()[0]

    @property
    def best(self) -> float:
        return self._state()[1]

    @property
    def history(self):
        return self._state()[2]
