"""Oracle: dense direct solve of the PageRank equation -- TEST INFRASTRUCTURE ONLY.

PAPER.md §2.1, Eq. (3) x = dPx + (1-d)Z, closed form Eq. (4):

    x = (1-d) (I - dP)^{-1} Z

computed with LAPACK's LU solve (numpy.linalg.solve) on the dense matrix; the
"completed" variant first pads every null column of P with Z (§2.1 "one usually
pads the null columns of P with 1/n (dangling nodes completion)", generalised
to Z per §3.3 "if the completion follows the distribution Z").
"""
from __future__ import annotations

import numpy as np

MAX_DENSE_N = 5000


def complete(P, Z):
    """P with every all-zero column replaced by Z (§2.1 dangling completion)."""
    P = np.array(P, dtype=np.float64, copy=True)
    null = P.sum(axis=0) == 0.0
    P[:, null] = np.asarray(Z, dtype=np.float64)[:, None]
    return P


def dense_solve(P, d, Z, completed=False):
    """x solving (I - dP) x = (1-d) Z  (Eq. (4))."""
    P = np.asarray(P, dtype=np.float64)
    n = P.shape[0]
    if n > MAX_DENSE_N:
        raise ValueError(f"dense oracle refuses n={n} > {MAX_DENSE_N}")
    Z = np.asarray(Z, dtype=np.float64)
    if completed:
        P = complete(P, Z)
    return np.linalg.solve(np.eye(n) - d * P, (1.0 - d) * Z)
