"""Seeded synthetic workloads (BASELINE.json configs) -- shared input generator.

This module holds none of the D-Iteration arithmetic: it emits graph
structure (CSR by source: row_ptr int64[n+1], col int32[m]), optional raw
edge weights (float32, values exactly representable), and edge deltas for the
dynamic-update config.  Both the CUDA path (tests, bench, smoke) and the CPU
oracle consume its output.  The generator is counter-based (synth/gen.c), so
node ranges can be generated independently per rank.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsynth.so")

DEG_UNIFORM, DEG_GEOMETRIC, DEG_POWERLAW = 0, 1, 2
TGT_UNIFORM, TGT_HOSTZIPF = 0, 1


class _Params(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n", ctypes.c_int64), ("deg_kind", ctypes.c_int),
                ("deg_a", ctypes.c_double), ("deg_b", ctypes.c_double), ("deg_cap", ctypes.c_int64),
                ("p_dangling", ctypes.c_double), ("tgt_kind", ctypes.c_int), ("block", ctypes.c_int64),
                ("p_local", ctypes.c_double), ("zipf_s", ctypes.c_double)]


@dataclass(frozen=True)
class GraphSpec:
    name: str
    n: int
    deg_kind: int
    deg_a: float
    deg_b: float = 1.0
    deg_cap: int = 1 << 40
    p_dangling: float = 0.0
    tgt_kind: int = TGT_HOSTZIPF
    block: int = 100
    p_local: float = 0.8
    weighted: bool = False
    seed: int = 0
    d: float = 0.85
    tol: float = 1e-12

    def scaled(self, n, **kw):
        return replace(self, n=n, **kw)


# BASELINE.json "configs", in order.  The power-law x_min = 3.75 is calibrated
# so that n = 50M gives ~1B edges (mean out-degree ~20, as config 2 states).
CONFIGS = {
    0: GraphSpec("tiny-uniform-1k", 1000, DEG_UNIFORM, 10, p_dangling=0.05,
                 tgt_kind=TGT_UNIFORM, seed=0, tol=1e-12),
    1: GraphSpec("web-1M-10M", 1_000_000, DEG_GEOMETRIC, 10, deg_cap=1000, p_dangling=0.15,
                 seed=1, tol=1e-10),
    2: GraphSpec("web-50M-1B-weighted", 50_000_000, DEG_POWERLAW, 2.1, deg_b=3.75, deg_cap=5000,
                 p_dangling=0.12, weighted=True, seed=2, tol=1e-9),
    3: GraphSpec("web-400M-8B-sharded", 400_000_000, DEG_POWERLAW, 2.1, deg_b=3.75, deg_cap=5000,
                 p_dangling=0.12, weighted=True, seed=3, tol=1e-9),
    # "dynamic update on the config-2 graph": configs[2]'s graph, 1% of its edges rewired
    4: GraphSpec("web-50M-1B-weighted-dynamic", 50_000_000, DEG_POWERLAW, 2.1, deg_b=3.75, deg_cap=5000,
                 p_dangling=0.12, weighted=True, seed=2, tol=1e-9),
}

_lib = None


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _clib():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        lib.synth_degrees.argtypes = [ctypes.POINTER(_Params), ctypes.c_int64, ctypes.c_int64, P]
        lib.synth_edges.argtypes = [ctypes.POINTER(_Params), ctypes.c_int64, ctypes.c_int64, P, P, P]
        lib.synth_targets.argtypes = [ctypes.POINTER(_Params), ctypes.c_int64, P, P, ctypes.c_uint64, P]
        lib.synth_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _params(spec: GraphSpec):
    return _Params(spec.seed, spec.n, spec.deg_kind, float(spec.deg_a), float(spec.deg_b),
                   int(min(spec.deg_cap, 1 << 62)), spec.p_dangling, spec.tgt_kind, spec.block,
                   spec.p_local, 1.0)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Graph:
    n: int
    row_ptr: np.ndarray       # int64[hi-lo+1], offsets from 0
    col: np.ndarray           # int32[m], global target ids
    w: np.ndarray | None      # float32[m] raw weights or None
    lo: int = 0
    hi: int = 0

    @property
    def m(self):
        return int(self.row_ptr[-1])


def generate(spec: GraphSpec, lo=0, hi=None, pinned_alloc=None) -> Graph:
    """Rows [lo, hi) of the graph described by ``spec`` (whole graph by default).

    ``pinned_alloc(shape, dtype)`` may supply (pinned) numpy buffers for col/w."""
    hi = spec.n if hi is None else hi
    lib = _clib()
    prm = _params(spec)
    deg = np.empty(hi - lo, dtype=np.int64)
    lib.synth_degrees(ctypes.byref(prm), lo, hi, _ptr(deg))
    row_ptr = np.zeros(hi - lo + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    m = int(row_ptr[-1])
    alloc = pinned_alloc or (lambda shape, dt: np.empty(shape, dtype=dt))
    col = alloc((m,), np.int32)
    w = alloc((m,), np.float32) if spec.weighted else None
    lib.synth_edges(ctypes.byref(prm), lo, hi, _ptr(row_ptr), _ptr(col),
                    _ptr(w) if w is not None else None)
    return Graph(n=spec.n, row_ptr=row_ptr, col=col, w=w, lo=lo, hi=hi)


def uniform_Z(n):
    """Z uniform ("often set to the uniform distribution", §2.1)."""
    return np.full(n, 1.0 / n, dtype=np.float64)


def rewire(spec: GraphSpec, g: Graph, fraction=0.01, seed=7):
    """Config 4's edge delta: ``fraction`` of m edges rewired, half removals
    (distinct existing (s,t) pairs, every parallel copy removed) and half
    insertions (uniform source, target drawn with the same locality/Zipf rule).
    Returns dict(add_src, add_dst, add_w, rem_src, rem_dst) as numpy arrays."""
    rng = np.random.default_rng(seed)
    m = g.m
    k = max(1, int(m * fraction) // 2)
    src_of = np.repeat(np.arange(g.lo, g.hi, dtype=np.int64), np.diff(g.row_ptr))
    pick = rng.choice(m, size=min(k, m), replace=False)
    pairs = np.unique(np.stack([src_of[pick], g.col[pick].astype(np.int64)], 1), axis=0)
    add_src = rng.integers(0, spec.n, size=k, dtype=np.int64)
    add_k = np.arange(k, dtype=np.int64)
    add_dst = np.empty(k, dtype=np.int32)
    _clib().synth_targets(ctypes.byref(_params(spec)), k, _ptr(add_src), _ptr(add_k), seed,
                          _ptr(add_dst))
    add_w = None
    if spec.weighted:
        j = rng.integers(0, 1 << 22, size=k)
        add_w = (0.5 + 3.0 * j / 8388608.0).astype(np.float32)
    return dict(add_src=add_src.astype(np.int32), add_dst=add_dst, add_w=add_w,
                rem_src=pairs[:, 0].astype(np.int32), rem_dst=pairs[:, 1].astype(np.int32))


def num_threads():
    return int(_clib().synth_num_threads())
