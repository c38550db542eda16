"""B200-native D-Iteration (arxiv 1501.06350) PageRank engine.

The engine is libdit.so (hand-written CUDA for sm_100a) behind the C ABI in
include/dit.h; ``_lib`` is its thin ctypes binding with the same names, and
``DIGraph`` below is a convenience owner of a graph handle (marshalling only).
"""
from __future__ import annotations

from . import _lib
from ._lib import (DI_DANGLING_COMPLETE, DI_DANGLING_DROP, DI_MEM_DEVICE, DI_MEM_HOST,  # noqa: F401
                   DI_VARIANT_AUTO, DI_VARIANT_PULL, DI_VARIANT_PUSH, DI_W_F32, DI_W_F64, DI_W_NONE,
                   DIError, di_get_state, di_graph_create, di_graph_destroy, di_graph_info,
                   di_kernel_launches, di_last_error, di_resume, di_set_state, di_solve, di_update_edges)

VARIANTS = {"auto": DI_VARIANT_AUTO, "push": DI_VARIANT_PUSH, "pull": DI_VARIANT_PULL, "tiled": _lib.DI_VARIANT_TILED}
DANGLING = {"drop": DI_DANGLING_DROP, "complete": DI_DANGLING_COMPLETE}


class DIGraph:
    """Owner of one engine graph handle (CSR by source, optional weights)."""

    def __init__(self, n, row_ptr, col, weights=None, device=0, stream=None):
        self.n = int(n)
        self.device = device
        self.handle = di_graph_create(self.n, row_ptr, col, weights, device=device, stream=stream)

    @property
    def m(self):
        return di_graph_info(self.handle)[1]

    @property
    def weight_storage(self):
        return di_graph_info(self.handle)[2]

    def _out(self, out):
        import torch
        if out is None:
            out = torch.empty(self.n, dtype=torch.float64, device=f"cuda:{self.device}")
        return out

    def solve(self, d=0.85, Z=None, tol=1e-12, out=None, theta=1.0, variant="auto", dangling="drop",
              max_sweeps=0, pull_frac=0.25, local_rounds=4):
        out = self._out(out)
        res = di_solve(self.handle, d, Z, tol, out, theta=theta, variant=VARIANTS[variant],
                       dangling=DANGLING[dangling], max_sweeps=max_sweeps, pull_frac=pull_frac,
                       local_rounds=local_rounds)
        return out, res.as_dict()

    def resume(self, tol=1e-12, out=None, theta=1.0, variant="auto", dangling="drop", max_sweeps=0,
               pull_frac=0.25, local_rounds=4):
        out = self._out(out)
        res = di_resume(self.handle, tol, out, theta=theta, variant=VARIANTS[variant],
                        dangling=DANGLING[dangling], max_sweeps=max_sweeps, pull_frac=pull_frac,
                        local_rounds=local_rounds)
        return out, res.as_dict()

    def update_edges(self, add_src=None, add_dst=None, add_w=None, rem_src=None, rem_dst=None):
        di_update_edges(self.handle, add_src, add_dst, add_w, rem_src, rem_dst)

    def state(self):
        import torch
        F = torch.empty(self.n, dtype=torch.float64, device=f"cuda:{self.device}")
        H = torch.empty_like(F)
        d, leak = di_get_state(self.handle, F, H)
        return F, H, d, leak

    def set_state(self, d, F, H, leak=0.0):
        di_set_state(self.handle, d, F, H, leak)

    def close(self):
        if self.handle:
            di_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
