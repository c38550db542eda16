"""CPU oracle for the D-Iteration hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct float64 implementation of what the paper
(Hong, Huynh, Mathieu, "D-Iteration: diffusion approach for solving PageRank",
arxiv 1501.06350; /root/reference/PAPER.md) computes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything under
``oracle/``.  The product path (``paper_1501_06350_b200``) never imports it,
shares no code, header, table or constant with it, and fails loudly when its
CUDA extension is missing.

Modules
-------
graph   Eq. (1): the diffusion matrix P from a weighted edge list (CSR by
        source), dense P for small n, dangling set, edge deltas (§3.5).
dense   Eq. (4): x = (1-d)(I-dP)^{-1} Z by dense elimination (uncompleted and
        Z-completed P, §2.1 / §3.3).
di      §3.1-§3.5: one elementary diffusion (Eqs. (8), (10)), the residual
        bound (Eq. (11), §3.3), the implicit-completion normalisation (§3.3),
        the Theorem 4 corrective fluid, and ctypes wrappers over the C loops
        in ``oracle/c/di_oracle.c`` (sequential DI-cyc / DI-argmax, the
        data-parallel sweep of DESIGN.md reading R1, Power Iteration Eq. (5)).

Parity status (pins live in tests/test_oracle_*.py, all ``-m "not gpu"``):
every function above is pinned against values the paper or mathematics fix
(closed forms, Eq. (12), Theorems 1-4, brute force / dense solve on tiny
graphs).  No function is "parity unpinned".
"""
