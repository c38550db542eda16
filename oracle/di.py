"""Oracle: D-Iteration (§3) -- TEST INFRASTRUCTURE ONLY.

Pure-Python pieces follow the paper's equations literally and are meant for
small cases; the loops that must run on up to ~10^7 edges are the C functions
of ``oracle/c/di_oracle.c`` reached through ctypes (``seq_run``,
``sweep_run``, ``power_iteration``).

Notation (§3.1): fluid F, history H, damping d, default distribution
Z, F_0 = (1-d) Z, H_0 = 0; leak l_k (§3.3) = fluid consumed at dangling nodes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "c", "di_oracle.c")
_CLIB = os.path.join(_HERE, "c", "libdi_oracle.so")


# --------------------------------------------------------------------------
# state + single elementary diffusion (pure Python, small cases)
# --------------------------------------------------------------------------
@dataclass
class DiState:
    F: np.ndarray
    H: np.ndarray
    d: float
    leak: float = 0.0
    k: int = 0
    F0: np.ndarray = field(default=None)


def di_init(n, d, Z=None):
    """Eq. (7): F_0 = (1-d) Z; H_0 = 0 (uniform Z when None)."""
    Z = np.full(n, 1.0 / n) if Z is None else np.asarray(Z, dtype=np.float64)
    F = (1.0 - d) * Z
    return DiState(F=F.copy(), H=np.zeros(n), d=d, F0=F.copy())


def di_step(state, col_ptr, row_idx, pval, i):
    """One diffusion of node i, Eqs. (8) and (10), in the paper's order:
    H_k = H_{k-1} + F_{k-1}(i) e_i ;  F_k = F_{k-1} + d F_{k-1}(i) P e_i - F_{k-1}(i) e_i.
    Dangling i: the fluid leaves, l += F_{k-1}(i) (§3.3)."""
    f = state.F[i]
    state.H[i] += f
    state.F[i] -= f
    b, e = int(col_ptr[i]), int(col_ptr[i + 1])
    if b == e:
        state.leak += f
    for k in range(b, e):
        state.F[row_idx[k]] += state.d * f * pval[k]
    state.k += 1
    return state


def residual_l1(F):
    """|F|_1 (signed fluid after a Theorem 4 restart: magnitudes)."""
    return float(np.abs(F).sum())


def bound_uncompleted(F, d):
    """Eq. (11): |x - H_k| <= |F_k| / (1-d)."""
    return residual_l1(F) / (1.0 - d)


def bound_completed(F, d, leak):
    """§3.3 final display: |x - (1-d)/(1-d-d l_k) H_k| = |F_k| / (1-d-d l_k)."""
    return residual_l1(F) / (1.0 - d - d * leak)


def normalized_history(H, d, leak):
    """§3.3: "H_k needs to be renormalized (multiplication) by (1-d)/(1-d-d l_k)"."""
    return (1.0 - d) / (1.0 - d - d * leak) * np.asarray(H)


def update_fluid(F, H, d, P_old_apply, P_new_apply):
    """Theorem 4: F'_0 = F_{k0} + d (P' - P) H_{k0}; H'_0 = H_{k0}.

    P_*_apply(v) returns the product P v (dense matmul or ``spmv`` below)."""
    return np.asarray(F) + d * (P_new_apply(H) - P_old_apply(H))


def spmv(n, col_ptr, row_idx, pval):
    """v -> P v for P given by columns (Eq. (1)); used by tests and update_fluid."""
    col_ptr = np.asarray(col_ptr, dtype=np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(col_ptr))
    rows = np.asarray(row_idx, dtype=np.int64)

    def apply(v):
        return np.bincount(rows, weights=pval * np.asarray(v)[src], minlength=n)

    return apply


# --------------------------------------------------------------------------
# C loops (ctypes).  Build on first use with gcc; build() in __graft_entry__
# compiles it ahead of time as well.
# --------------------------------------------------------------------------
_lib = None


def build_clib(force=False):
    if force or not os.path.exists(_CLIB) or os.path.getmtime(_CLIB) < os.path.getmtime(_CSRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-Wall", "-o", _CLIB, _CSRC, "-lm"])
    return _CLIB


def _clib():
    global _lib
    if _lib is None:
        build_clib()
        lib = ctypes.CDLL(_CLIB)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        lib.orc_seq_run.argtypes = [I64, P, P, P, D, ctypes.c_int, D, I64, P, P, P, P, P]
        lib.orc_seq_run.restype = I64
        lib.orc_sweep_run.argtypes = [I64, P, P, P, D, D, D, I64, P, P, P, P, P, P]
        lib.orc_sweep_run.restype = I64
        lib.orc_power_iteration.argtypes = [I64, P, P, P, D, P, D, I64, P, P]
        lib.orc_tiled_sweep_run.argtypes = [I64, P, P, P, D, I64, ctypes.c_int, ctypes.c_int, D, I64, P, P, P, P, P,
                                            P, P, I64]
        lib.orc_tiled_sweep_run.restype = I64
        lib.orc_power_iteration.restype = I64
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _cols(col_ptr, row_idx, pval):
    return (np.ascontiguousarray(col_ptr, dtype=np.int64),
            np.ascontiguousarray(row_idx, dtype=np.int32),
            np.ascontiguousarray(pval, dtype=np.float64))


@dataclass
class RunResult:
    F: np.ndarray
    H: np.ndarray
    leak: float
    steps: int            # diffusions (seq) or sweeps (sweep)
    edges: int            # diffused edges (sum of out-degrees of diffused nodes)
    nodes: int = 0        # diffused nodes (sweep)
    residual: float = 0.0
    cursor: int = 0


def seq_run(n, col_ptr, row_idx, pval, d, F, H, sched="argmax", tol=1e-12,
            max_steps=10**10, leak=0.0, cursor=0):
    """Sequential DI (§3.4 DI-cyc / DI-argmax) from state (F, H); copies inputs."""
    cp, ri, pv = _cols(col_ptr, row_idx, pval)
    F = np.array(F, dtype=np.float64, copy=True)
    H = np.array(H, dtype=np.float64, copy=True)
    lk = np.array([leak], dtype=np.float64)
    ed = np.zeros(1, dtype=np.int64)
    cur = np.array([cursor], dtype=np.int64)
    k = _clib().orc_seq_run(n, _p(cp), _p(ri), _p(pv), d, {"cyc": 0, "argmax": 1}[sched],
                            tol, max_steps, _p(F), _p(H), _p(lk), _p(ed), _p(cur))
    return RunResult(F=F, H=H, leak=float(lk[0]), steps=int(k), edges=int(ed[0]),
                     residual=residual_l1(F), cursor=int(cur[0]))


def sweep_run(n, col_ptr, row_idx, pval, d, F, H, theta=1.0, tol=1e-12,
              max_sweeps=1_000_000, leak=0.0):
    """Data-parallel frontier sweeps (reading R1) from (F, H)."""
    cp, ri, pv = _cols(col_ptr, row_idx, pval)
    F = np.array(F, dtype=np.float64, copy=True)
    H = np.array(H, dtype=np.float64, copy=True)
    lk = np.array([leak], dtype=np.float64)
    ed = np.zeros(1, dtype=np.int64)
    nd = np.zeros(1, dtype=np.int64)
    res = np.zeros(1, dtype=np.float64)
    s = _clib().orc_sweep_run(n, _p(cp), _p(ri), _p(pv), d, theta, tol, max_sweeps,
                              _p(F), _p(H), _p(lk), _p(ed), _p(nd), _p(res))
    return RunResult(F=F, H=H, leak=float(lk[0]), steps=int(s), edges=int(ed[0]),
                     nodes=int(nd[0]), residual=float(res[0]))


def tiled_sweep_run(n, col_ptr, row_idx, pval, d, F, H, tile=1024, rounds=4, tol=1e-12,
                    max_sweeps=1_000_000, leak=0.0, waves=1, bounds=None):
    """Tile-local sweeps (readings R12, R15) from (F, H); tiles run in
    `waves` waves (tile index mod waves), a wave's remote pushes reaching later
    waves of the same sweep.  `bounds` (partition starts + n, R16): pushes
    between partitions reach their target after the sweep."""
    cp, ri, pv = _cols(col_ptr, row_idx, pval)
    F = np.array(F, dtype=np.float64, copy=True)
    H = np.array(H, dtype=np.float64, copy=True)
    lk = np.array([leak], dtype=np.float64)
    ed = np.zeros(1, dtype=np.int64)
    nd = np.zeros(1, dtype=np.int64)
    res = np.zeros(1, dtype=np.float64)
    bd = np.ascontiguousarray(bounds if bounds is not None else [0, n], dtype=np.int64)
    s = _clib().orc_tiled_sweep_run(n, _p(cp), _p(ri), _p(pv), d, tile, rounds, waves, tol, max_sweeps,
                                    _p(F), _p(H), _p(lk), _p(ed), _p(nd), _p(res), _p(bd), len(bd))
    return RunResult(F=F, H=H, leak=float(lk[0]), steps=int(s), edges=int(ed[0]),
                     nodes=int(nd[0]), residual=float(res[0]))


def power_iteration(n, col_ptr, row_idx, pval, d, Z, eps=1e-13, max_iter=100000, x0=None):
    """Eq. (5) x_{k+1} = d P x_k + (1-d) Z from x_0 = Z (or x0)."""
    cp, ri, pv = _cols(col_ptr, row_idx, pval)
    Z = np.ascontiguousarray(Z, dtype=np.float64)
    x = np.array(Z if x0 is None else x0, dtype=np.float64, copy=True)
    delta = np.zeros(1, dtype=np.float64)
    it = _clib().orc_power_iteration(n, _p(cp), _p(ri), _p(pv), d, _p(Z), eps, max_iter,
                                     _p(x), _p(delta))
    return x, int(it), float(delta[0])


def di_solve(n, row_ptr, col, w, d, Z=None, tol=1e-12, theta=1.0, method="sweep"):
    """Cold DI solve from Eq. (7) on a CSR graph: returns RunResult.

    method 'sweep' = DESIGN.md reading R1 (what the GPU path computes);
    'argmax' / 'cyc' = the paper's sequential schedulers (§3.4)."""
    from .graph import column_entries
    cp, ri, pv = column_entries(n, row_ptr, col, w)
    st = di_init(n, d, Z)
    if method == "sweep":
        return sweep_run(n, cp, ri, pv, d, st.F, st.H, theta=theta, tol=tol)
    return seq_run(n, cp, ri, pv, d, st.F, st.H, sched=method, tol=tol)
