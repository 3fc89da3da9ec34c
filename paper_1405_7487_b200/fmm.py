"""Thin ctypes binding of libfmm.so (include/fmm.h).  Argument marshalling only: every
step of the FMM runs in the library's CUDA kernels.  There is no CPU fallback: if the
library or a CUDA device is missing, construction raises.

PyTorch supplies device memory and the current CUDA stream; numpy is used only for the
host-side introspection buffers and fmm_solve_host.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfmm.so")

FMM_OK, FMM_ERR_ARG, FMM_ERR_STATE, FMM_ERR_NONFINITE, FMM_ERR_OOM, FMM_ERR_CUDA, FMM_ERR_NCCL = range(7)
STATUS = {0: "FMM_OK", 1: "FMM_ERR_ARG", 2: "FMM_ERR_STATE", 3: "FMM_ERR_NONFINITE", 4: "FMM_ERR_OOM",
          5: "FMM_ERR_CUDA", 6: "FMM_ERR_NCCL"}
F32, F64 = 0, 1

# every symbol include/fmm.h declares: (restype, argtypes)
_p, _i, _i64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double
# host-logic callbacks of the distributed driver (fmm_hist_fn, fmm_orb_hist_fn, fmm_orb_split_fn)
HIST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double))
ORB_HIST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_uint32), C.c_int, C.c_int,
                          C.POINTER(C.c_double))
ORB_SPLIT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_uint32), C.POINTER(C.c_int32))
SYMBOLS = {
    "fmm_version": (_i, []),
    "fmm_create": (_i, [_i64, _i, _d, _i, _i, _i, C.POINTER(_p)]),
    "fmm_destroy": (_i, [_p]),
    "fmm_last_error": (C.c_char_p, [_p]),
    "fmm_build": (_i, [_p, _p, _i64, _p]),
    "fmm_evaluate": (_i, [_p, _p, _p, _p, _p, _p]),
    "fmm_solve": (_i, [_p, _p, _p, _i64, _p, _p, _p]),
    "fmm_solve_host": (_i, [_p, _p, _p, _i64, _p, _p, _p]),
    "fmm_get_counts": (_i, [_p, _p]),
    "fmm_copy_sorted": (_i, [_p, _p, _p]),
    "fmm_copy_cells": (_i, [_p] * 12),
    "fmm_copy_lists": (_i, [_p, _p, _p]),
    "fmm_copy_expansions": (_i, [_p, _p, _p]),
    "fmm_set_timing": (_i, [_p, _i]),
    "fmm_phase_times": (_i, [_p, _p, _i, _p, _i]),
    "fmm_phase_name": (C.c_char_p, [_i]),
    "fmm_launch_count": (_i64, [_p, _i]),
    "fmm_build_tree": (_i, [_p, _p, _i64, _p]),
    "fmm_set_root_bounds": (_i, [_p, _p]),
    "fmm_dtt": (_i, [_p, _i, _p]),
    "fmm_lists": (_i, [_p, _p]),
    "fmm_upward": (_i, [_p, _p, _p, _p]),
    "fmm_interact": (_i, [_p, _p, _p, _p]),
    "fmm_bounds": (_i, [_p, _p, _i64, _p, _p]),
    "fmm_part_keys": (_i, [_p, _p, _i64, _p, _p, _p]),
    "fmm_part_histogram": (_i, [_p, _p, _p, _i64, C.c_uint64, _i, _i, _p, _p]),
    "fmm_part_pack": (_i, [_p, _p, _p, _p, _i64, _p, _i, _i64, _p, _p, _p, _p, _p]),
    "fmm_let_cover": (_i, [_p, _p, _p, _p]),
    "fmm_let_plan": (_i, [_p, _i, _p, _i, _p, _p, _p]),
    "fmm_let_pack_struct": (_i, [_p, _i, _p, _p]),
    "fmm_let_pack_data": (_i, [_p, _i, _p, _p]),
    "fmm_let_graft": (_i, [_p, _i, _p, _p, _p]),
    "fmm_let_unpack": (_i, [_p, _i, _i, _p, _p, _p]),
    "fmm_let_remote": (_i, [_p, _i, _p, _p, _p, _p]),
    "fmm_work": (_i, [_p, _d, C.c_float, _p, _p, _p]),
    "fmm_orb_histogram": (_i, [_p, _p, _p, _p, _i64, _i, _p, _p, _i, _i, _p, _p]),
    "fmm_orb_split": (_i, [_p, _p, _p, _i64, _i, _p, _p, _p, _p]),
    "fmm_part_pack_dest": (_i, [_p, _p, _p, _p, _i64, _i, _i64, _p, _p, _p, _p, _p]),
    "fmm_debug_p2p": (_i, [_p, _p, _p, _i64, _p, _p, _p]),
    "fmm_debug_m2l": (_i, [_p, _p, _p, _i64, _p, _p]),
    "fmm_debug_check": (_i, [_p, _p]),
    "fmm_group_create": (_i, [_i, _p]),
    "fmm_group_destroy": (_i, [_p]),
    "fmm_dist_unique_id": (_i, [_p]),
    "fmm_create_dist": (_i, [_i64, _i, _d, _i, _i, _i, _i, _i, _p, _p, _i, _p]),
    "fmm_set_weights": (_i, [_p, _p, _i64]),
    "fmm_dist_set_alpha": (_i, [_p, _d, _d]),
    "fmm_dist_tune_alpha": (_i, [_p, _d, _d, _d]),
    "fmm_dist_solve": (_i, [_p, _p, _p, _i64, _i64, _i, _p, _p, _p]),
    "fmm_dist_get_stats": (_i, [_p, _p]),
    "fmm_dist_local": (_i, [_p, _p, _p]),
    "fmm_dist_weights": (_i, [_p, _p]),
    "fmm_dist_orb_boxes": (_i, [_p, _p]),
    "fmm_dist_timeline": (_i, [_p, _p, _i, _p]),
    "fmm_dist_timeline_name": (C.c_char_p, [_i]),
    "fmm_splitters": (_i, [_i, _i, _d, HIST_FN, _p, _p]),
    "fmm_orb_plan": (_i, [_i, _i, ORB_HIST_FN, ORB_SPLIT_FN, _p, _p]),
    "fmm_alpha_tuner_create": (_i, [_d, _d, _d, _p]),
    "fmm_alpha_tuner_next": (_d, [_p]),
    "fmm_alpha_tuner_report": (_i, [_p, _d]),
    "fmm_alpha_tuner_state": (_i, [_p, _p, _p, _p, _p, _i]),
    "fmm_alpha_tuner_destroy": (_i, [_p]),
}
LET_MAX_COVER = 73

_lib = None


class FMMError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libfmm.so (build it first with paper_1405_7487_b200.build.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FMMError(FMM_ERR_CUDA, f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SYMBOLS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class _Counts(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n", "ncell", "nleaf", "depth", "n_m2l", "n_p2p", "p2p_interactions")]


class _TreeView(C.Structure):
    """fmm_tree_view (include/fmm.h): device pointers of a caller-supplied tree."""
    _fields_ = [("n", C.c_int64), ("ncell", C.c_int64), ("pos", C.c_void_p), ("q", C.c_void_p),
                ("body_begin", C.c_void_p), ("body_count", C.c_void_p), ("child_count", C.c_void_p),
                ("center", C.c_void_p), ("level", C.c_void_p), ("M", C.c_void_p), ("root_half_width", C.c_double)]


def _tp(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _np_ptr(a):
    return None if a is None else a.ctypes.data


class FMM:
    """One FMM context: fmm_create(N, P, theta, ncrit) -> build(pos) -> evaluate(pos, q)."""

    def __init__(self, n_max: int, P: int, theta: float, ncrit: int, prec: str = "f32", device: int = 0):
        self.prec = {"f32": F32, "f64": F64}[prec]
        self.P, self.theta, self.ncrit, self.device = P, theta, ncrit, device
        h = C.c_void_p()
        st = lib().fmm_create(int(n_max), int(P), float(theta), int(ncrit), self.prec, int(device), C.byref(h))
        if st != FMM_OK:
            raise FMMError(st, "fmm_create")
        self._h = h
        self._pos = None

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().fmm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _check(self, st, what):
        if st != FMM_OK:
            msg = lib().fmm_last_error(self._h)
            raise FMMError(st, f"{what}: {msg.decode() if msg else ''}")

    @property
    def dtype(self):
        import torch
        return torch.float32 if self.prec == F32 else torch.float64

    def _stream(self, stream):
        """cudaStream_t of `stream`, default: the current stream of the CONTEXT's device."""
        import torch
        return (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream

    def _check_tensor(self, t, shape, name):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise FMMError(FMM_ERR_ARG, f"{name} must be a CUDA tensor")
        if t.dtype != self.dtype:
            raise FMMError(FMM_ERR_ARG, f"{name} dtype {t.dtype} != context precision {self.dtype}")
        if not t.is_contiguous() or tuple(t.shape) != tuple(shape):
            raise FMMError(FMM_ERR_ARG, f"{name} must be contiguous with shape {shape}")

    # -- the path ----------------------------------------------------------
    def build(self, pos, stream=None):
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        self._check(lib().fmm_build(self._h, C.c_void_p(pos.data_ptr()), n, C.c_void_p(self._stream(stream))),
                    "fmm_build")
        self._pos = pos
        self.n = n
        return self

    def evaluate(self, pos, q, phi=None, grad=None, stream=None):
        import torch
        n = pos.shape[0]
        self._check_tensor(q, (n,), "q")
        if phi is None:
            phi = torch.empty(n, dtype=self.dtype, device=pos.device)
        if grad is None:
            grad = torch.empty((n, 3), dtype=self.dtype, device=pos.device)
        self._check_tensor(phi, (n,), "phi")
        self._check_tensor(grad, (n, 3), "grad")
        self._check(lib().fmm_evaluate(self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()),
                                       C.c_void_p(phi.data_ptr()), C.c_void_p(grad.data_ptr()),
                                       C.c_void_p(self._stream(stream))), "fmm_evaluate")
        return phi, grad

    def solve(self, pos, q, phi=None, grad=None, stream=None):
        """fmm_solve: build + evaluate in one call (the library overlaps independent passes)."""
        import torch
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        self._check_tensor(q, (n,), "q")
        if phi is None:
            phi = torch.empty(n, dtype=self.dtype, device=pos.device)
        if grad is None:
            grad = torch.empty((n, 3), dtype=self.dtype, device=pos.device)
        self._check_tensor(phi, (n,), "phi")
        self._check_tensor(grad, (n, 3), "grad")
        self._check(lib().fmm_solve(self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()), n,
                                    C.c_void_p(phi.data_ptr()), C.c_void_p(grad.data_ptr()),
                                    C.c_void_p(self._stream(stream))), "fmm_solve")
        self._pos = pos
        self.n = n
        return phi, grad

    def solve_host(self, pos: np.ndarray, q: np.ndarray, phi: np.ndarray = None, grad: np.ndarray = None,
                   stream=None):
        """fmm_solve_host: host arrays in, host arrays out (copies inside the library)."""
        dt = np.float32 if self.prec == F32 else np.float64
        pos = np.ascontiguousarray(pos, dtype=dt)
        q = np.ascontiguousarray(q, dtype=dt)
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise FMMError(FMM_ERR_ARG, f"pos must have shape (n, 3), got {pos.shape}")
        n = pos.shape[0]
        if q.shape != (n,):
            raise FMMError(FMM_ERR_ARG, f"q must have shape ({n},), got {q.shape}")
        phi = np.empty(n, dt) if phi is None else phi
        grad = np.empty((n, 3), dt) if grad is None else grad
        for a, shape, name in ((phi, (n,), "phi"), (grad, (n, 3), "grad")):
            # the library writes n*es / 3n*es bytes straight into these buffers
            if not isinstance(a, np.ndarray) or a.dtype != dt or a.shape != shape:
                raise FMMError(FMM_ERR_ARG, f"{name} must be a numpy {np.dtype(dt).name} array of shape {shape}")
            if not a.flags.c_contiguous or not a.flags.writeable:
                raise FMMError(FMM_ERR_ARG, f"{name} must be C-contiguous and writeable")
        s = None if stream is None else C.c_void_p(stream.cuda_stream)
        self._check(lib().fmm_solve_host(self._h, _np_ptr(pos), _np_ptr(q), n, _np_ptr(phi), _np_ptr(grad), s),
                    "fmm_solve_host")
        self._pos = None
        return phi, grad

    # -- the path in halves (multi-GPU: LET grafted between tree and traversal) --
    def build_tree(self, pos, stream=None):
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        self._check(lib().fmm_build_tree(self._h, C.c_void_p(pos.data_ptr()), n, C.c_void_p(self._stream(stream))),
                    "fmm_build_tree")
        self._pos = pos
        self.n = n
        return self

    def set_root_bounds(self, bounds=None):
        """R2 root cube of later builds from these bounds (lo xyz, hi xyz); None: own bounds."""
        self._root_bounds = None if bounds is None else np.ascontiguousarray(bounds, dtype=np.float64).reshape(6)
        self._check(lib().fmm_set_root_bounds(self._h, _np_ptr(self._root_bounds)), "fmm_set_root_bounds")

    def dtt(self, remote: bool = False, stream=None):
        self._check(lib().fmm_dtt(self._h, int(remote), C.c_void_p(self._stream(stream))), "fmm_dtt")

    def make_lists(self, stream=None):
        self._check(lib().fmm_lists(self._h, C.c_void_p(self._stream(stream))), "fmm_lists")

    def upward(self, pos, q, stream=None):
        n = pos.shape[0]
        self._check_tensor(q, (n,), "q")
        self._check(lib().fmm_upward(self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()),
                                     C.c_void_p(self._stream(stream))), "fmm_upward")

    def interact(self, phi, grad, stream=None):
        n = phi.shape[0]
        self._check_tensor(phi, (n,), "phi")
        self._check_tensor(grad, (n, 3), "grad")
        self._check(lib().fmm_interact(self._h, C.c_void_p(phi.data_ptr()), C.c_void_p(grad.data_ptr()),
                                       C.c_void_p(self._stream(stream))), "fmm_interact")
        return phi, grad

    # -- multi-GPU: partition (part.cu) --------------------------------------
    def bounds(self, pos, stream=None) -> np.ndarray:
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        out = np.zeros(6)
        self._check(lib().fmm_bounds(self._h, C.c_void_p(pos.data_ptr()), n, _np_ptr(out),
                                     C.c_void_p(self._stream(stream))), "fmm_bounds")
        return out

    def part_keys(self, pos, bounds: np.ndarray, stream=None):
        """Morton keys under the root cube of the global bounds (int64 tensor holding u64 bits)."""
        import torch
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        b = np.ascontiguousarray(bounds, dtype=np.float64)
        keys = torch.empty(n, dtype=torch.int64, device=pos.device)
        self._check(lib().fmm_part_keys(self._h, C.c_void_p(pos.data_ptr()), n, _np_ptr(b), C.c_void_p(keys.data_ptr()),
                                        C.c_void_p(self._stream(stream))), "fmm_part_keys")
        return keys

    def part_histogram(self, keys, w=None, bits: int = 16, prefix: int = 0, prefix_bits: int = 0, out=None,
                       stream=None):
        import torch
        hist = torch.empty(1 << bits, dtype=torch.float64, device=keys.device) if out is None else out
        wp = None if w is None else C.c_void_p(w.data_ptr())
        self._check(lib().fmm_part_histogram(self._h, C.c_void_p(keys.data_ptr()), wp, keys.shape[0], int(prefix),
                                             int(prefix_bits), bits, C.c_void_p(hist.data_ptr()),
                                             C.c_void_p(self._stream(stream))), "fmm_part_histogram")
        return hist

    def part_pack(self, pos, q, keys, splitters: np.ndarray, nranks: int, gid_base: int, stream=None):
        import torch
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        self._check_tensor(q, (n,), "q")
        spl = np.ascontiguousarray(splitters, dtype=np.uint64)
        opos = torch.empty_like(pos); oq = torch.empty_like(q)
        gid = torch.empty(n, dtype=torch.int64, device=pos.device)
        counts = np.zeros(nranks, np.int64)
        self._check(lib().fmm_part_pack(self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()),
                                        C.c_void_p(keys.data_ptr()), n, _np_ptr(spl), int(nranks), int(gid_base),
                                        C.c_void_p(opos.data_ptr()), C.c_void_p(oq.data_ptr()),
                                        C.c_void_p(gid.data_ptr()), _np_ptr(counts), C.c_void_p(self._stream(stream))),
                    "fmm_part_pack")
        return opos, oq, gid, counts

    def orb_histogram(self, keys, group, axis, prefix, prefix_bits, bits, w=None, stream=None):
        import torch
        ng = len(axis)
        ax = np.ascontiguousarray(axis, dtype=np.int32); pre = np.ascontiguousarray(prefix, dtype=np.uint32)
        hist = torch.empty((ng, 1 << bits), dtype=torch.float64, device=keys.device)
        wp = None if w is None else C.c_void_p(w.data_ptr())
        self._check(lib().fmm_orb_histogram(self._h, C.c_void_p(keys.data_ptr()), wp, C.c_void_p(group.data_ptr()),
                                            keys.shape[0], ng, _np_ptr(ax), _np_ptr(pre), int(prefix_bits), int(bits),
                                            C.c_void_p(hist.data_ptr()), C.c_void_p(self._stream(stream))),
                    "fmm_orb_histogram")
        return hist

    def orb_split(self, keys, group, axis, cut, right, stream=None):
        ax = np.ascontiguousarray(axis, dtype=np.int32); ct = np.ascontiguousarray(cut, dtype=np.uint32)
        rt = np.ascontiguousarray(right, dtype=np.int32)
        self._check(lib().fmm_orb_split(self._h, C.c_void_p(keys.data_ptr()), C.c_void_p(group.data_ptr()),
                                        keys.shape[0], len(ax), _np_ptr(ax), _np_ptr(ct), _np_ptr(rt),
                                        C.c_void_p(self._stream(stream))), "fmm_orb_split")

    def part_pack_dest(self, pos, q, dest, nranks: int, gid_base: int, stream=None):
        import torch
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        self._check_tensor(q, (n,), "q")
        opos = torch.empty_like(pos); oq = torch.empty_like(q)
        gid = torch.empty(n, dtype=torch.int64, device=pos.device)
        counts = np.zeros(nranks, np.int64)
        self._check(lib().fmm_part_pack_dest(self._h, C.c_void_p(pos.data_ptr()), C.c_void_p(q.data_ptr()),
                                             C.c_void_p(dest.data_ptr()), n, int(nranks), int(gid_base),
                                             C.c_void_p(opos.data_ptr()), C.c_void_p(oq.data_ptr()),
                                             C.c_void_p(gid.data_ptr()), _np_ptr(counts),
                                             C.c_void_p(self._stream(stream))), "fmm_part_pack_dest")
        return opos, oq, gid, counts

    # -- multi-GPU: local essential tree (let.cu) -------------------------------
    def let_cover(self, stream=None) -> np.ndarray:
        cov = np.zeros((LET_MAX_COVER, 8)); k = C.c_int()
        self._check(lib().fmm_let_cover(self._h, _np_ptr(cov), C.byref(k), C.c_void_p(self._stream(stream))),
                    "fmm_let_cover")
        return cov[:k.value].copy()

    def let_plan(self, peer: int, cover: np.ndarray, stream=None):
        cov = np.ascontiguousarray(cover, dtype=np.float64).reshape(-1, 8)
        sb, db = C.c_int64(), C.c_int64()
        self._check(lib().fmm_let_plan(self._h, int(peer), _np_ptr(cov) if len(cov) else None, len(cov),
                                       C.byref(sb), C.byref(db), C.c_void_p(self._stream(stream))), "fmm_let_plan")
        return int(sb.value), int(db.value)

    def let_pack_struct(self, peer: int, dst, stream=None):
        self._check(lib().fmm_let_pack_struct(self._h, int(peer), C.c_void_p(dst.data_ptr()),
                                              C.c_void_p(self._stream(stream))), "fmm_let_pack_struct")

    def let_pack_data(self, peer: int, dst, stream=None):
        self._check(lib().fmm_let_pack_data(self._h, int(peer), C.c_void_p(dst.data_ptr()),
                                            C.c_void_p(self._stream(stream))), "fmm_let_pack_data")

    @staticmethod
    def _buf_arrays(bufs):
        ptrs = (C.c_void_p * max(len(bufs), 1))(*[b.data_ptr() for b in bufs])
        sizes = (C.c_int64 * max(len(bufs), 1))(*[b.numel() * b.element_size() for b in bufs])
        return ptrs, sizes

    def let_graft(self, bufs, stream=None):
        ptrs, sizes = self._buf_arrays(bufs)
        self._check(lib().fmm_let_graft(self._h, len(bufs), ptrs, sizes, C.c_void_p(self._stream(stream))),
                    "fmm_let_graft")

    def let_unpack(self, bufs, first: int = 0, stream=None):
        ptrs, sizes = self._buf_arrays(bufs)
        self._check(lib().fmm_let_unpack(self._h, int(first), len(bufs), ptrs, sizes,
                                         C.c_void_p(self._stream(stream))), "fmm_let_unpack")

    def let_remote(self, k: int, with_orig: bool = True):
        base, nc, nb = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(lib().fmm_let_remote(self._h, int(k), C.byref(base), C.byref(nc), C.byref(nb), None),
                    "fmm_let_remote")
        orig = None
        if with_orig:
            orig = np.zeros(nc.value, np.uint32)
            self._check(lib().fmm_let_remote(self._h, int(k), None, None, None, _np_ptr(orig)), "fmm_let_remote")
        return int(base.value), int(nc.value), int(nb.value), orig

    def work(self, c_m2l: float, alpha: float = 1.0, out=None, stream=None):
        """Eq. (1) weights of the last build (caller order) and the sums of l and r."""
        import torch
        w = torch.empty(self.n, dtype=torch.float32, device=torch.device("cuda", self.device)) if out is None else out
        lr = np.zeros(2)
        self._check(lib().fmm_work(self._h, float(c_m2l), float(alpha), C.c_void_p(w.data_ptr()), _np_ptr(lr),
                                   C.c_void_p(self._stream(stream))), "fmm_work")
        return w, lr

    # -- debug stage entry points (caller-supplied tree and lists) ------------
    def _pairs(self, pairs):
        import torch
        if pairs.dtype not in (torch.int32, torch.uint32) or not pairs.is_cuda or not pairs.is_contiguous() \
                or pairs.dim() != 2 or pairs.shape[1] != 2:
            raise FMMError(FMM_ERR_ARG, "pairs must be a contiguous CUDA (n, 2) int32/uint32 tensor")
        return pairs

    def debug_p2p(self, pos, q, body_begin, body_count, child_count, pairs, stream=None):
        """fmm_debug_p2p: near field (R17) of the given P2P cell pairs on the given sorted bodies
        and cells; phi [n], grad [n][3] in the bodies' order."""
        import torch
        n = pos.shape[0]
        self._check_tensor(pos, (n, 3), "pos")
        self._check_tensor(q, (n,), "q")
        pairs = self._pairs(pairs)
        v = _TreeView(n=n, ncell=body_begin.shape[0], pos=pos.data_ptr(), q=q.data_ptr(),
                      body_begin=body_begin.data_ptr(), body_count=body_count.data_ptr(),
                      child_count=child_count.data_ptr(), root_half_width=0.0)
        phi = torch.empty(n, dtype=self.dtype, device=pos.device)
        grad = torch.empty((n, 3), dtype=self.dtype, device=pos.device)
        self._check(lib().fmm_debug_p2p(self._h, C.byref(v), _tp(pairs), pairs.shape[0], _tp(phi), _tp(grad),
                                        C.c_void_p(self._stream(stream))), "fmm_debug_p2p")
        self._pos = None
        return phi, grad

    def debug_m2l(self, center, level, M, root_half_width, pairs, stream=None):
        """fmm_debug_m2l: L [ncell][ncoef] (fp64) = R14 summed over the given M2L cell pairs."""
        import torch
        nc = center.shape[0]
        pairs = self._pairs(pairs)
        L = torch.empty_like(M)
        v = _TreeView(n=0, ncell=nc, center=center.data_ptr(), level=level.data_ptr(), M=M.data_ptr(),
                      root_half_width=float(root_half_width))
        self._check(lib().fmm_debug_m2l(self._h, C.byref(v), _tp(pairs), pairs.shape[0], _tp(L),
                                        C.c_void_p(self._stream(stream))), "fmm_debug_m2l")
        self._pos = None
        return L

    def debug_check(self) -> int:
        """fmm_debug_check: number of guarded buffers written past their end (FMM_GUARD=1)."""
        nb = C.c_int64()
        st = lib().fmm_debug_check(self._h, C.byref(nb))
        if st not in (FMM_OK, FMM_ERR_STATE):
            self._check(st, "fmm_debug_check")
        return int(nb.value)

    # -- introspection -----------------------------------------------------
    def counts(self) -> dict:
        c = _Counts()
        self._check(lib().fmm_get_counts(self._h, C.byref(c)), "fmm_get_counts")
        return {k: int(getattr(c, k)) for k, _ in _Counts._fields_}

    def sorted(self):
        n = self.counts()["n"]
        k = np.zeros(n, np.uint64); p = np.zeros(n, np.uint32)
        self._check(lib().fmm_copy_sorted(self._h, _np_ptr(k), _np_ptr(p)), "fmm_copy_sorted")
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
        self._check(lib().fmm_copy_cells(self._h, *[_np_ptr(out[k]) for k in order]), "fmm_copy_cells")
        return out

    def lists(self):
        c = self.counts()
        m2l = np.zeros((c["n_m2l"], 2), np.uint32); p2p = np.zeros((c["n_p2p"], 2), np.uint32)
        self._check(lib().fmm_copy_lists(self._h, _np_ptr(m2l), _np_ptr(p2p)), "fmm_copy_lists")
        return m2l, p2p

    def expansions(self):
        c = self.counts()
        nco = self.P * (self.P + 1) * (self.P + 2) // 6
        M = np.zeros((c["ncell"], nco)); L = np.zeros((c["ncell"], nco))
        self._check(lib().fmm_copy_expansions(self._h, _np_ptr(M), _np_ptr(L)), "fmm_copy_expansions")
        return M, L

    # -- timing ------------------------------------------------------------
    def set_timing(self, on: bool = True):
        self._check(lib().fmm_set_timing(self._h, int(on)), "fmm_set_timing")

    def phase_times(self, reset: bool = True) -> dict:
        ms = np.zeros(32); n = C.c_int()
        self._check(lib().fmm_phase_times(self._h, _np_ptr(ms), 32, C.byref(n), int(reset)), "fmm_phase_times")
        return {lib().fmm_phase_name(i).decode(): float(ms[i]) for i in range(n.value)}

    def launch_count(self, reset: bool = True) -> int:
        return int(lib().fmm_launch_count(self._h, int(reset)))
