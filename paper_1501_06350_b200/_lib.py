"""ctypes binding of libdit.so (include/dit.h) -- argument marshalling only.

Every function keeps the C name and order of arguments; arrays may be numpy
arrays (host memory) or torch tensors (host or CUDA).  No computation happens
here: each call goes straight to the CUDA engine, and importing this module
fails loudly if the engine library is missing.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdit.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libdit.so not found at {LIB_PATH}: build the CUDA engine first "
        "(python paper_1501_06350_b200/build.py or __graft_entry__.build()). "
        "There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

DI_OK, DI_ERR_INVALID, DI_ERR_CUDA, DI_ERR_OOM, DI_ERR_EDGE_NOT_FOUND, DI_ERR_STATE = range(6)
DI_MEM_HOST, DI_MEM_DEVICE = 0, 1
DI_W_NONE, DI_W_F32, DI_W_F64 = 0, 1, 2
DI_DANGLING_DROP, DI_DANGLING_COMPLETE = 0, 1
DI_VARIANT_AUTO, DI_VARIANT_PUSH, DI_VARIANT_PULL, DI_VARIANT_TILED = 0, 1, 2, 3
DI_TILE_NODES = 512   # include/dit.h
DI_TILE_WAVES = 3     # include/dit.h (shards too: cross-rank pushes wait a sweep, R16)

EXPORTS = ["di_solve_opts_default", "di_graph_create", "di_graph_destroy", "di_graph_info", "di_solve",
           "di_resume", "di_update_edges", "di_get_state", "di_set_state", "di_last_error",
           "di_kernel_launches", "di_profile_enable", "di_profile_get", "di_sweep_history", "di_plan_stats",
           "di_release_memory"]


class di_profile(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("select_ms", "push_ms", "pull_ms", "reduce_ms", "select_bytes",
                                               "push_bytes", "pull_bytes", "reduce_bytes")] + \
               [(k, ctypes.c_int64) for k in ("select_launches", "push_launches", "pull_launches",
                                              "reduce_launches", "sweeps")] + \
               [("tile_ms", ctypes.c_double), ("tile_bytes", ctypes.c_double), ("tile_launches", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class di_solve_opts(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("variant", ctypes.c_int32), ("dangling", ctypes.c_int32),
                ("max_sweeps", ctypes.c_int64), ("pull_frac", ctypes.c_double), ("local_rounds", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class di_result(ctypes.Structure):
    _fields_ = [("residual_l1", ctypes.c_double), ("bound", ctypes.c_double), ("leak", ctypes.c_double),
                ("norm_factor", ctypes.c_double), ("sweeps", ctypes.c_int64), ("diffused_nodes", ctypes.c_int64),
                ("diffused_edges", ctypes.c_int64), ("push_sweeps", ctypes.c_int64),
                ("pull_sweeps", ctypes.c_int64), ("converged", ctypes.c_int32), ("reserved", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_lib.di_solve_opts_default.argtypes = [ctypes.POINTER(di_solve_opts)]
_lib.di_solve_opts_default.restype = None
_lib.di_graph_create.argtypes = [_I64, _I64, _P, _P, _P, _I32, _I32, _I32, _P, ctypes.POINTER(_P)]
_lib.di_graph_destroy.argtypes = [_P]
_lib.di_graph_info.argtypes = [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I32)]
_lib.di_solve.argtypes = [_P, _D, _P, _I32, _D, ctypes.POINTER(di_solve_opts), _P, _I32, ctypes.POINTER(di_result)]
_lib.di_resume.argtypes = [_P, _D, ctypes.POINTER(di_solve_opts), _P, _I32, ctypes.POINTER(di_result)]
_lib.di_update_edges.argtypes = [_P, _I64, _P, _P, _P, _I32, _I64, _P, _P, _I32]
_lib.di_get_state.argtypes = [_P, _P, _P, _I32, ctypes.POINTER(_D), ctypes.POINTER(_D)]
_lib.di_set_state.argtypes = [_P, _D, _P, _P, _I32, _D]
_lib.di_profile_enable.argtypes = [_P, _I32]
_lib.di_profile_get.argtypes = [_P, ctypes.POINTER(di_profile)]
_lib.di_sweep_history.argtypes = [_P, _I64, _P, _P, _P, _P, ctypes.POINTER(_I64)]
_lib.di_plan_stats.argtypes = [_P, _P, ctypes.c_int32]
_lib.di_release_memory.argtypes = [_I32]
_lib.di_last_error.restype = ctypes.c_char_p
_lib.di_kernel_launches.restype = _I64
for _name in EXPORTS:
    if _name not in ("di_solve_opts_default", "di_last_error", "di_kernel_launches"):
        getattr(_lib, _name).restype = ctypes.c_int


class DIError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != DI_OK:
        raise DIError(rc, di_last_error())


def _ptr_mem(a, dtype=None):
    """(pointer, mem kind, keep-alive) for a numpy array / torch tensor / None."""
    if a is None:
        return None, DI_MEM_HOST, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if not a.is_contiguous():
                a = a.contiguous()
            return a.data_ptr(), (DI_MEM_DEVICE if a.is_cuda else DI_MEM_HOST), a
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(a, dtype=dtype) if dtype is not None else np.ascontiguousarray(a)
    return arr.ctypes.data, DI_MEM_HOST, arr


def _wdtype(w):
    if w is None:
        return DI_W_NONE
    dt = str(getattr(w, "dtype", ""))
    if "float32" in dt:
        return DI_W_F32
    if "float64" in dt:
        return DI_W_F64
    raise TypeError(f"weights must be float32 or float64, got {dt}")


def _stream_ptr(stream):
    if stream is None:
        return None
    return getattr(stream, "cuda_stream", stream)


# ------------------------------------------------------------------ C names
def di_solve_opts_default():
    o = di_solve_opts()
    _lib.di_solve_opts_default(ctypes.byref(o))
    return o


def di_last_error():
    return _lib.di_last_error().decode()


def di_kernel_launches():
    return int(_lib.di_kernel_launches())


def di_release_memory(device=0):
    """Return the engine's cached device memory (pool, sort scratch) to the driver."""
    _check(_lib.di_release_memory(device))


def di_graph_create(n, row_ptr, col, weights=None, device=0, stream=None):
    """CSR by source (row_ptr int64[n+1], col int32[m], optional weights) -> handle."""
    m = int(row_ptr[-1]) if len(row_ptr) else 0
    rp, mem, k1 = _ptr_mem(row_ptr, np.int64)
    cp, mem2, k2 = _ptr_mem(col, np.int32)
    wp, mem3, k3 = _ptr_mem(weights)
    if len({mem, mem2} | ({mem3} if weights is not None else set())) != 1:
        raise ValueError("row_ptr, col and weights must all be host or all be device")
    h = _P()
    _check(_lib.di_graph_create(n, m, rp, cp, wp, _wdtype(weights), mem, device, _stream_ptr(stream),
                                ctypes.byref(h)))
    return h


def di_graph_destroy(h):
    _check(_lib.di_graph_destroy(h))


def di_graph_info(h):
    n, m, w = _I64(), _I64(), _I32()
    _check(_lib.di_graph_info(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(w)))
    return n.value, m.value, w.value


def _opts(theta=1.0, variant=DI_VARIANT_AUTO, dangling=DI_DANGLING_DROP, max_sweeps=0, pull_frac=0.25,
          local_rounds=4):
    o = di_solve_opts_default()
    o.theta, o.variant, o.dangling, o.max_sweeps, o.pull_frac = theta, variant, dangling, max_sweeps, pull_frac
    o.local_rounds = local_rounds
    return o


def di_solve(h, d, Z=None, tol=1e-12, H_out=None, **opts):
    """Cold solve; H_out (numpy / torch, host or device) receives H; returns di_result."""
    zp, zmem, kz = _ptr_mem(Z, np.float64)
    hp, hmem, kh = _ptr_mem(H_out)
    res = di_result()
    o = _opts(**opts)
    _check(_lib.di_solve(h, d, zp, zmem, tol, ctypes.byref(o), hp, hmem, ctypes.byref(res)))
    return res


def di_resume(h, tol=1e-12, H_out=None, **opts):
    hp, hmem, kh = _ptr_mem(H_out)
    res = di_result()
    o = _opts(**opts)
    _check(_lib.di_resume(h, tol, ctypes.byref(o), hp, hmem, ctypes.byref(res)))
    return res


def di_update_edges(h, add_src=None, add_dst=None, add_w=None, rem_src=None, rem_dst=None):
    na = 0 if add_src is None else len(add_src)
    nr = 0 if rem_src is None else len(rem_src)
    asp, m1, k1 = _ptr_mem(add_src, np.int32) if na else (None, None, None)
    adp, m2, k2 = _ptr_mem(add_dst, np.int32) if na else (None, None, None)
    awp, m3, k3 = _ptr_mem(add_w) if (na and add_w is not None) else (None, None, None)
    rsp, m4, k4 = _ptr_mem(rem_src, np.int32) if nr else (None, None, None)
    rdp, m5, k5 = _ptr_mem(rem_dst, np.int32) if nr else (None, None, None)
    mems = {m for m in (m1, m2, m3, m4, m5) if m is not None}
    if len(mems) > 1:
        raise ValueError("all update arrays must be host or all device")
    mem = mems.pop() if mems else DI_MEM_HOST
    wd = _wdtype(add_w) if awp is not None else DI_W_NONE
    _check(_lib.di_update_edges(h, na, asp, adp, awp, wd, nr, rsp, rdp, mem))


def di_get_state(h, F=None, H=None):
    """Copy F and H into the given arrays (numpy or torch); returns (d, leak)."""
    fp, fm, kf = _ptr_mem(F)
    hp, hm, kh = _ptr_mem(H)
    if F is not None and H is not None and fm != hm:
        raise ValueError("F and H must live in the same memory")
    d, lk = _D(), _D()
    _check(_lib.di_get_state(h, fp, hp, fm if F is not None else hm, ctypes.byref(d), ctypes.byref(lk)))
    return d.value, lk.value


def di_set_state(h, d, F, H, leak=0.0):
    fp, fm, kf = _ptr_mem(F, np.float64)
    hp, hm, kh = _ptr_mem(H, np.float64)
    if fm != hm:
        raise ValueError("F and H must live in the same memory")
    _check(_lib.di_set_state(h, d, fp, hp, fm, leak))


def di_profile_enable(h, on=True):
    _check(_lib.di_profile_enable(h, 1 if on else 0))


def di_profile_get(h):
    p = di_profile()
    _check(_lib.di_profile_get(h, ctypes.byref(p)))
    return p.as_dict()


def di_sweep_history(h, cap=1 << 16):
    """Per-sweep (nodes, edges, entries, variant) arrays of the last solve call."""
    nodes = np.zeros(cap, np.int64)
    edges = np.zeros(cap, np.int64)
    ent = np.zeros(cap, np.int64)
    var = np.zeros(cap, np.int32)
    cnt = _I64()
    _check(_lib.di_sweep_history(h, cap, nodes.ctypes.data, edges.ctypes.data, ent.ctypes.data,
                                 var.ctypes.data, ctypes.byref(cnt)))
    k = cnt.value
    return nodes[:k], edges[:k], ent[:k], var[:k]


PLAN_STATS = ("tiles", "local_edges", "ell_slots", "light_edges", "heavy_edges", "heavy_targets", "heavy_segments",
              "heavy_runs", "heavy_chunks", "stripes")


def di_plan_stats(h):
    """Sizes of the tiled plan (include/dit.h di_plan_stats) as a dict."""
    v = np.zeros(len(PLAN_STATS), np.int64)
    _check(_lib.di_plan_stats(h, v.ctypes.data, len(PLAN_STATS)))
    return {k: int(x) for k, x in zip(PLAN_STATS, v)}


# ------------------------------------------------------------------ shards (multi-GPU)
EXPORTS += ["di_shard_create", "di_shard_info", "di_shard_ghost_ids", "di_shard_set_recv", "di_shard_begin",
            "di_shard_control", "di_shard_sweep", "di_shard_apply", "di_shard_reduce", "di_shard_poll",
            "di_shard_finish", "di_shard_flush", "di_shard_flush_apply", "di_shard_heavy_local"]
_lib.di_shard_create.argtypes = [_I64, _I64, _I64, _I64, _P, _P, _P, _I32, _I32, _I32, _P, ctypes.POINTER(_P)]
_lib.di_shard_info.argtypes = [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64)]
_lib.di_shard_ghost_ids.argtypes = [_P, _P, _I32]
_lib.di_shard_set_recv.argtypes = [_P, _I64, _P, _I32, _P, _I32]
_lib.di_shard_begin.argtypes = [_P, _D, _P, _I32, _D, ctypes.POINTER(di_solve_opts), _P]
_lib.di_shard_control.argtypes = [_P, _P, _I32]
_lib.di_shard_sweep.argtypes = [_P, _P]
_lib.di_shard_apply.argtypes = [_P, _P]
_lib.di_shard_heavy_local.argtypes = [_P]
_lib.di_shard_flush.argtypes = [_P, _P]
_lib.di_shard_flush_apply.argtypes = [_P, _P]
_lib.di_shard_reduce.argtypes = [_P]
_lib.di_shard_poll.argtypes = [_P, ctypes.POINTER(_I32)]
_lib.di_shard_finish.argtypes = [_P, _D, ctypes.POINTER(di_solve_opts), _P, _I32, ctypes.POINTER(di_result)]
for _name in EXPORTS[-12:]:
    getattr(_lib, _name).restype = ctypes.c_int


def di_shard_create(n_global, lo, hi, row_ptr, col, weights=None, device=0, stream=None):
    m = int(row_ptr[-1]) if len(row_ptr) else 0
    rp, mem, k1 = _ptr_mem(row_ptr, np.int64)
    cp, mem2, k2 = _ptr_mem(col, np.int32)
    wp, mem3, k3 = _ptr_mem(weights)
    if len({mem, mem2} | ({mem3} if weights is not None else set())) != 1:
        raise ValueError("row_ptr, col and weights must all be host or all be device")
    h = _P()
    _check(_lib.di_shard_create(n_global, lo, hi, m, rp, cp, wp, _wdtype(weights), mem, device,
                                _stream_ptr(stream), ctypes.byref(h)))
    return h


def di_shard_info(h):
    a, b, c = _I64(), _I64(), _I64()
    _check(_lib.di_shard_info(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def di_shard_ghost_ids(h, out):
    p, mem, k = _ptr_mem(out)
    _check(_lib.di_shard_ghost_ids(h, p, mem))
    return out


def di_shard_set_recv(h, local_idx, seg_counts):
    p, mem, k = _ptr_mem(local_idx, np.int32)
    seg = np.ascontiguousarray(seg_counts, dtype=np.int64)
    _check(_lib.di_shard_set_recv(h, int(seg.sum()), p, len(seg), seg.ctypes.data, mem))


def di_shard_begin(h, d, Z=None, tol=1e-12, stats=None, **opts):
    zp, zmem, kz = _ptr_mem(Z, np.float64)
    sp, smem, ks = _ptr_mem(stats)
    o = _opts(**opts)
    _check(_lib.di_shard_begin(h, d, zp, zmem, tol, ctypes.byref(o), sp))


def di_shard_control(h, gathered, nranks):
    _check(_lib.di_shard_control(h, _ptr_mem(gathered)[0], int(nranks)))


def di_shard_sweep(h, ghost_out):
    _check(_lib.di_shard_sweep(h, _ptr_mem(ghost_out)[0]))


def di_shard_heavy_local(h):
    _check(_lib.di_shard_heavy_local(h))


def di_shard_apply(h, recv):
    _check(_lib.di_shard_apply(h, _ptr_mem(recv)[0]))


def di_shard_flush(h, ghost_out):
    _check(_lib.di_shard_flush(h, _ptr_mem(ghost_out)[0]))


def di_shard_flush_apply(h, recv):
    _check(_lib.di_shard_flush_apply(h, _ptr_mem(recv)[0]))


def di_shard_reduce(h):
    _check(_lib.di_shard_reduce(h))


def di_shard_poll(h):
    d = _I32()
    _check(_lib.di_shard_poll(h, ctypes.byref(d)))
    return bool(d.value)


def di_shard_finish(h, tol=1e-12, H_out=None, **opts):
    hp, hmem, kh = _ptr_mem(H_out)
    res = di_result()
    o = _opts(**opts)
    _check(_lib.di_shard_finish(h, tol, ctypes.byref(o), hp, hmem, ctypes.byref(res)))
    return res
