"""Oracle: the diffusion matrix P (§2.1, Eq. (1)) -- TEST INFRASTRUCTURE ONLY.

    P_{i,j} = w_{j,i} / sum_{(j,k) in E} w_{j,k}   if (j,i) in E, else 0.

The graph arrives as a CSR edge list by source j (row_ptr[j]..row_ptr[j+1]-1
hold the out-edges j -> col[e] with raw weight w[e], default 1).  Column j of
P is then exactly the out-edge list of j with each weight divided by the row's
weight sum.  Parallel edges are kept as separate entries; since they add
inside every product with P, that is the same as merging w_{j,i} by summation
(reading R3).
"""
from __future__ import annotations

import numpy as np


def column_entries(n, row_ptr, col, w=None):
    """Columns of P per Eq. (1), source-major.

    Returns (col_ptr int64[n+1], row_idx int32[m], pval float64[m]) with
    pval[e] = w[e] / sum of w over e's source row.  Dangling sources have an
    empty column ("column i summing to 0 if i is a dangling node", §2.1).
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int32)
    m = int(row_ptr[-1]) if len(row_ptr) else 0
    if w is None:
        w = np.ones(m, dtype=np.float64)
    else:
        w = np.asarray(w, dtype=np.float64)
    deg = np.diff(row_ptr)
    src = np.repeat(np.arange(n, dtype=np.int64), deg)
    wsum = np.bincount(src, weights=w, minlength=n).astype(np.float64)
    pval = w / wsum[src] if m else np.zeros(0, dtype=np.float64)
    return row_ptr.copy(), col.copy(), pval


def dangling_mask(n, row_ptr):
    """True for nodes with no outgoing edge (§2.1 "dangling node")."""
    return np.diff(np.asarray(row_ptr, dtype=np.int64)) == 0


def dense_P(n, col_ptr, row_idx, pval):
    """Dense n x n P for small n (Eq. (1)); parallel entries summed."""
    P = np.zeros((n, n), dtype=np.float64)
    deg = np.diff(col_ptr)
    src = np.repeat(np.arange(n), deg)
    np.add.at(P, (np.asarray(row_idx, dtype=np.int64), src), pval)
    return P


def apply_delta(n, row_ptr, col, w, add_src, add_dst, add_w, rem_src, rem_dst):
    """Edge-level graph update (§3.5 "consider a new matrix P'").

    Removal (s, t) deletes every CSR entry s -> t (the merged edge (s,t) of
    Eq. (1)); an absent edge raises KeyError.  Each addition (s, t, w) appends
    one entry to row s.  Returns (row_ptr', col', w', changed_sources), w' is
    None if both w and add_w are None.
    """
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    m = int(row_ptr[-1])
    weighted = w is not None or add_w is not None
    wv = np.ones(m) if w is None else np.asarray(w, dtype=np.float64)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr))
    keep = np.ones(m, dtype=bool)
    rem_src = np.asarray(rem_src, dtype=np.int64)
    rem_dst = np.asarray(rem_dst, dtype=np.int64)
    if len(rem_src):
        key = src * n + col
        rkey = rem_src * n + rem_dst
        hit = np.isin(key, rkey)
        found = np.isin(rkey, key[hit])
        if not found.all():
            k = int(np.flatnonzero(~found)[0])
            raise KeyError(f"removal of absent edge ({rem_src[k]}, {rem_dst[k]})")
        keep &= ~hit
    add_src = np.asarray(add_src, dtype=np.int64)
    add_dst = np.asarray(add_dst, dtype=np.int64)
    aw = np.ones(len(add_src)) if add_w is None else np.asarray(add_w, dtype=np.float64)
    all_src = np.concatenate([src[keep], add_src])
    all_dst = np.concatenate([col[keep], add_dst])
    all_w = np.concatenate([wv[keep], aw])
    order = np.argsort(all_src, kind="stable")     # keeps old entries before new ones
    new_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(all_src, minlength=n), out=new_ptr[1:])
    changed = np.unique(np.concatenate([add_src, rem_src])).astype(np.int64)
    return (new_ptr, all_dst[order].astype(np.int32),
            all_w[order] if weighted else None, changed)
