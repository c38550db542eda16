"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Every test here runs without a GPU.  Each pin names the passage it follows.
A plausible mistake in the oracle (dropped damping, wrong sign in Eq. (8),
transposed P, missing leak, wrong normalisation, wrong update sign) fails at
least one of them.
"""
import numpy as np
import pytest

import synth
from oracle import dense, di, graph
from tests._golden import csr_from_edges, load

D = 0.85


def small_graph(n, seed, dangling=0.1, deg=4, weighted=False):
    spec = synth.CONFIGS[0].scaled(n, seed=seed, p_dangling=dangling, deg_a=2 * deg - 1,
                                   weighted=weighted)
    return synth.generate(spec)


def cols_of(g):
    return graph.column_entries(g.n, g.row_ptr, g.col, g.w)


# ----------------------------------------------------------------- Eq. (1)
def test_eq1_weighted_halving_and_parallel_merge():
    # "0 1 2.0 / 0 2 2.0": column 0 of P = [(1, .5), (2, .5)], nodes 1, 2 dangling
    rp, c, w = csr_from_edges(3, [(0, 1), (0, 2)], [2.0, 2.0])
    cp, ri, pv = graph.column_entries(3, rp, c, w)
    assert list(ri) == [1, 2] and np.allclose(pv, [0.5, 0.5], rtol=0, atol=0)
    assert list(graph.dangling_mask(3, rp)) == [False, True, True]
    # parallel edges "0 1 ; 0 1 3.0" merge: P_{1,0} = 1 (weights 1 + 3 summed)
    rp, c, w = csr_from_edges(2, [(0, 1), (0, 1)], [1.0, 3.0])
    P = graph.dense_P(2, *graph.column_entries(2, rp, c, w))
    assert P[1, 0] == 1.0 and P.sum() == 1.0


@pytest.mark.parametrize("weighted", [False, True])
def test_eq1_columns_stochastic_or_null(weighted):
    # §2.1: "column i summing to 1 if node i has an outgoing edge, 0 if dangling"
    g = small_graph(150, 3, weighted=weighted)
    P = graph.dense_P(g.n, *cols_of(g))
    s = P.sum(axis=0)
    dang = graph.dangling_mask(g.n, g.row_ptr)
    assert np.all(np.abs(s[~dang] - 1.0) < 1e-12) and np.all(s[dang] == 0.0)
    # P_{i,j} is w_{j,i}/sum_k w_{j,k}: entry (target, source), not transposed
    j = int(np.flatnonzero(~dang)[0])
    b, e = g.row_ptr[j], g.row_ptr[j + 1]
    ww = np.ones(e - b) if g.w is None else g.w[b:e].astype(np.float64)
    for t, wt in zip(g.col[b:e], ww):
        assert P[t, j] >= wt / ww.sum() - 1e-15


# ----------------------------------------------------------------- Eq. (4)
def test_dense_solve_golden_chain_and_cycle():
    ch = load("chain3.txt")
    rp, c, _ = csr_from_edges(3, ch["edges"])
    P = graph.dense_P(3, *graph.column_entries(3, rp, c))
    x = dense.dense_solve(P, ch["d"], np.full(3, 1 / 3))
    assert np.allclose(x, ch["x"], rtol=0, atol=1e-15)
    cy = load("cycle2.txt")
    rp, c, _ = csr_from_edges(2, cy["edges"])
    P = graph.dense_P(2, *graph.column_entries(2, rp, c))
    assert np.allclose(dense.dense_solve(P, 0.3, [0.5, 0.5]), cy["x"], atol=1e-15)
    # single dangling node: P = 0 forces x = (1-d) Z; completed P = (1) gives x = 1
    assert dense.dense_solve(np.zeros((1, 1)), D, [1.0])[0] == pytest.approx(0.15, abs=1e-15)
    assert dense.dense_solve(np.zeros((1, 1)), D, [1.0], completed=True)[0] == pytest.approx(1.0, abs=1e-14)


def test_dense_solve_equals_neumann_series():
    # Eq. (4) via (I - dP)^{-1} = sum_k d^k P^k (P substochastic, d < 1)
    g = small_graph(60, 1)
    P = graph.dense_P(g.n, *cols_of(g))
    Z = synth.uniform_Z(g.n)
    x = dense.dense_solve(P, D, Z)
    acc, term = np.zeros(g.n), (1 - D) * Z
    for _ in range(400):
        acc += term
        term = D * (P @ term)
    assert np.abs(acc - x).sum() < 1e-13


def test_completed_solve_is_distribution():
    g = small_graph(80, 2, dangling=0.2)
    P = graph.dense_P(g.n, *cols_of(g))
    xc = dense.dense_solve(P, D, synth.uniform_Z(g.n), completed=True)
    assert abs(xc.sum() - 1.0) < 1e-12 and xc.min() > 0


# ----------------------------------------------------------------- Eq. (5)
def test_power_iteration_matches_dense_and_contracts():
    g = small_graph(120, 4)
    cp, ri, pv = cols_of(g)
    P = graph.dense_P(g.n, cp, ri, pv)
    Z = synth.uniform_Z(g.n)
    x = dense.dense_solve(P, D, Z)
    xk = Z.copy()
    err = np.abs(xk - x).sum()
    for _ in range(30):   # §2.2 "the error decays by a factor at least d"
        xk, _, _ = di.power_iteration(g.n, cp, ri, pv, D, Z, eps=0, max_iter=1, x0=xk)
        e2 = np.abs(xk - x).sum()
        assert e2 <= D * err + 1e-15
        err = e2
    xp, it, delta = di.power_iteration(g.n, cp, ri, pv, D, Z, eps=1e-14)
    assert np.abs(xp - x).sum() < 1e-12


# ------------------------------------------------------- Eqs. (7), (8), (10)
def test_di_step_spec_examples():
    # 0 -> {1, 2} equal weights, F = (0.2, 0, 0.1), diffuse 0:
    rp, c, _ = csr_from_edges(3, [(0, 1), (0, 2)])
    cp, ri, pv = graph.column_entries(3, rp, c)
    st = di.DiState(F=np.array([0.2, 0.0, 0.1]), H=np.zeros(3), d=D)
    di.di_step(st, cp, ri, pv, 0)
    assert st.H[0] == 0.2 and np.allclose(st.F, [0.0, 0.085, 0.185], rtol=0, atol=1e-17)
    # single dangling node: the fluid leaves and is counted in l (§3.3)
    st = di.DiState(F=np.array([0.15]), H=np.zeros(1), d=D)
    di.di_step(st, np.array([0, 0]), np.zeros(0, np.int32), np.zeros(0), 0)
    assert st.H[0] == 0.15 and st.F[0] == 0.0 and st.leak == 0.15
    # self-loop 0 -> 0: d F P_{0,0} remains at 0 (Eq. (8), "up to loops")
    st = di.DiState(F=np.array([0.15]), H=np.zeros(1), d=D)
    di.di_step(st, np.array([0, 1]), np.array([0], np.int32), np.array([1.0]), 0)
    assert st.H[0] == 0.15 and st.F[0] == pytest.approx(0.1275, abs=1e-17)


def test_di_cyc_chain_one_round_exact():
    ch = load("chain3.txt")
    rp, c, _ = csr_from_edges(3, ch["edges"])
    cp, ri, pv = graph.column_entries(3, rp, c)
    st = di.di_init(3, ch["d"])
    for i in range(3):
        di.di_step(st, cp, ri, pv, i)
    assert np.all(st.F == 0) and np.allclose(st.H, ch["x"], rtol=0, atol=1e-16)
    assert st.leak == pytest.approx(ch["leak"], abs=1e-16)
    # §3.3: normalised history is the completed solution (a distribution)
    xn = di.normalized_history(st.H, ch["d"], st.leak)
    P = graph.dense_P(3, cp, ri, pv)
    assert np.allclose(xn, dense.dense_solve(P, ch["d"], np.full(3, 1 / 3), completed=True), atol=1e-14)
    assert xn.sum() == pytest.approx(1.0, abs=1e-14)


def test_di_cyc_cycle2_round1_and_bound_equality():
    cy = load("cycle2.txt")
    rp, c, _ = csr_from_edges(2, cy["edges"])
    cp, ri, pv = graph.column_entries(2, rp, c)
    st = di.di_init(2, cy["d"], [0.5, 0.5])
    di.di_step(st, cp, ri, pv, 0)
    di.di_step(st, cp, ri, pv, 1)
    assert np.allclose(st.H, cy["H_round1"], atol=1e-17) and np.allclose(st.F, cy["F_round1"], atol=1e-17)
    err = np.abs(cy["x"] - st.H).sum()
    assert err == pytest.approx(di.bound_uncompleted(st.F, cy["d"]), abs=1e-15) == pytest.approx(0.78625)


def test_theorem2_ccw_cycle_round1():
    cc = load("ccw_cycle10.txt")
    n = cc["n"]
    rp, c, _ = csr_from_edges(n, [(i, (i - 1) % n) for i in range(n)])
    cp, ri, pv = graph.column_entries(n, rp, c)
    st = di.di_init(n, cc["d"])
    r = di.seq_run(n, cp, ri, pv, cc["d"], st.F, st.H, sched="cyc", tol=0, max_steps=n)
    assert np.allclose(r.F, cc["F_round1"], rtol=0, atol=1e-17)
    x = np.full(n, 1 / n)
    assert np.abs(x - r.H).sum() <= cc["d"] ** 1 + 1e-15


# ---------------------------------------------------------- C loop == Eq. (8)
@pytest.mark.parametrize("sched", ["cyc", "argmax"])
def test_c_seq_run_bitwise_equals_python_steps(sched):
    g = small_graph(40, 5, weighted=True)
    cp, ri, pv = cols_of(g)
    st = di.di_init(g.n, D)
    r = di.seq_run(g.n, cp, ri, pv, D, st.F, st.H, sched=sched, tol=0, max_steps=300)
    # replay with the pure-Python Eq. (8)/(10) step and the same scheduler rule
    cur = 0
    for _ in range(300):
        if sched == "cyc":
            i, cur = cur, (cur + 1) % g.n
        else:
            a = np.abs(st.F)
            avg = min(a.sum() / g.n, a.max())
            while True:
                i, cur = cur, (cur + 1) % g.n
                if abs(st.F[i]) >= avg and st.F[i] != 0:
                    break
        di.di_step(st, cp, ri, pv, i)
    assert np.array_equal(r.H, st.H) and np.array_equal(r.F, st.F) and r.leak == st.leak


# ---------------------------------------- Eq. (12), Theorems 1-3 on a corpus
def _corpus():
    for n in (10, 50, 200):
        for s in range(3):
            yield n, s


@pytest.mark.parametrize("n,seed", list(_corpus()))
def test_conservation_identity_and_theorem1_every_step(n, seed):
    g = small_graph(n, seed)
    cp, ri, pv = cols_of(g)
    P = graph.dense_P(n, cp, ri, pv)
    Z = synth.uniform_Z(n)
    x = dense.dense_solve(P, D, Z)
    for sched in ("cyc", "argmax"):
        st = di.di_init(n, D, Z)
        F, H, lk, cur = st.F, st.H, 0.0, 0
        for _ in range(5 * n):
            r = di.seq_run(n, cp, ri, pv, D, F, H, sched=sched, tol=0, max_steps=1, leak=lk, cursor=cur)
            F, H, lk, cur = r.F, r.H, r.leak, r.cursor
            # Eq. (12): H_k + F_k = F_0 + d P H_k
            assert np.abs(H + F - st.F0 - D * (P @ H)).max() <= 1e-15
            # Eq. (11): |x - H_k| <= |F_k| / (1-d)
            assert np.abs(x - H).sum() <= di.bound_uncompleted(F, D) + 1e-14
            # leak l_k equals the history of the dangling nodes (R5)
            assert lk == pytest.approx(H[graph.dangling_mask(n, g.row_ptr)].sum(), abs=1e-15)


@pytest.mark.parametrize("n,seed", [(10, 0), (50, 1), (200, 2)])
def test_theorem2_and_theorem3_bounds_dangling_free(n, seed):
    g = small_graph(n, seed, dangling=0.0)
    cp, ri, pv = cols_of(g)
    P = graph.dense_P(n, cp, ri, pv)
    Z = synth.uniform_Z(n)
    x = dense.dense_solve(P, D, Z)
    st = di.di_init(n, D, Z)
    F, H, cur = st.F, st.H, 0
    for k in range(1, 8 * n + 1):       # Theorem 2: |x - H_k| <= d^floor(k/n)
        r = di.seq_run(n, cp, ri, pv, D, F, H, sched="cyc", tol=0, max_steps=1, cursor=cur)
        F, H, cur = r.F, r.H, r.cursor
        assert np.abs(x - H).sum() <= D ** (k // n) + 1e-14
    F, H, cur = st.F, st.H, 0
    for k in range(1, 8 * n + 1):       # Theorem 3: |x - H_k| <= (1 - (1-d)/n)^k
        r = di.seq_run(n, cp, ri, pv, D, F, H, sched="argmax", tol=0, max_steps=1, cursor=cur)
        F, H, cur = r.F, r.H, r.cursor
        assert np.abs(x - H).sum() <= (1 - (1 - D) / n) ** k + 1e-14


@pytest.mark.parametrize("n,seed", list(_corpus()))
def test_all_schedulers_converge_to_dense(n, seed):
    g = small_graph(n, seed)
    cp, ri, pv = cols_of(g)
    P = graph.dense_P(n, cp, ri, pv)
    Z = synth.uniform_Z(n)
    x = dense.dense_solve(P, D, Z)
    xc = dense.dense_solve(P, D, Z, completed=True)
    for method in ("cyc", "argmax", "sweep"):
        r = di.di_solve(n, g.row_ptr, g.col, g.w, D, Z, tol=1e-13, method=method)
        assert np.abs(r.H - x).sum() <= 1e-12
        # §3.3 implicit completion: normalised H -> completed solution, sums to 1
        xn = di.normalized_history(r.H, D, r.leak)
        assert np.abs(xn - xc).sum() <= di.bound_completed(r.F, D, r.leak) + 1e-12
        assert abs(xn.sum() - 1.0) <= 1e-11


# ----------------------------------------------- the data-parallel sweep (R1)
def test_sweep_theta0_equals_power_iteration_partial_sums():
    # theta = 0 diffuses every node holding fluid, so H after k sweeps is
    # sum_{t<k} (dP)^t F_0 -- the Eq. (5) iterate started from x_0 = 0.
    g = small_graph(100, 7, weighted=True)
    cp, ri, pv = cols_of(g)
    Z = synth.uniform_Z(g.n)
    st = di.di_init(g.n, D, Z)
    for k in (1, 2, 5, 13):
        r = di.sweep_run(g.n, cp, ri, pv, D, st.F, st.H, theta=0.0, tol=0, max_sweeps=k)
        xk, _, _ = di.power_iteration(g.n, cp, ri, pv, D, Z, eps=0, max_iter=k, x0=np.zeros(g.n))
        assert r.steps == k and np.abs(r.H - xk).sum() < 1e-15


def test_sweep_conservation_each_sweep_and_nonempty_frontier():
    g = small_graph(200, 8)
    cp, ri, pv = cols_of(g)
    P = graph.dense_P(g.n, cp, ri, pv)
    st = di.di_init(g.n, D)
    F, H, lk = st.F, st.H, 0.0
    prev = di.residual_l1(F)
    for _ in range(60):
        r = di.sweep_run(g.n, cp, ri, pv, D, F, H, theta=1.0, tol=0, max_sweeps=1, leak=lk)
        F, H, lk = r.F, r.H, r.leak
        assert r.nodes >= 1 and r.steps == 1
        assert np.abs(H + F - st.F0 - D * (P @ H)).max() <= 1e-15
        cur = di.residual_l1(F)
        assert cur < prev          # |F|_1 strictly decreasing while fluid remains
        prev = cur


def test_sweep_uniform_start_selects_all_nodes():
    # F_0 = (1-d)Z uniform: every node equals the average fluid, so the first
    # theta = 1 sweep (DI-argmax's "greater or equal to the average") takes all.
    g = small_graph(300, 9)
    cp, ri, pv = cols_of(g)
    st = di.di_init(g.n, D)
    r = di.sweep_run(g.n, cp, ri, pv, D, st.F, st.H, theta=1.0, tol=0, max_sweeps=1)
    assert r.nodes == g.n and np.allclose(r.H, st.F0, rtol=0, atol=0)


# ----------------------------------------------------------------- Theorem 4
def test_theorem4_golden_update():
    u = load("update3.txt")
    old = graph.column_entries(3, *csr_from_edges(3, [(0, 1)])[:2])
    new = graph.column_entries(3, *csr_from_edges(3, [(0, 2)])[:2])
    F2 = di.update_fluid(u["F"], u["H"], u["d"], di.spmv(3, *old), di.spmv(3, *new))
    assert np.allclose(F2, u["F_new"], rtol=0, atol=1e-16)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_theorem4_restart_reaches_new_fixed_point(seed):
    g = small_graph(150, seed, weighted=True)
    spec = synth.CONFIGS[0].scaled(150, seed=seed, weighted=True, deg_a=7, p_dangling=0.1)
    delta = synth.rewire(spec, g, fraction=0.05, seed=seed)
    Z = synth.uniform_Z(g.n)
    old = cols_of(g)
    r0 = di.sweep_run(g.n, *old, D, (1 - D) * Z, np.zeros(g.n), tol=1e-7)
    rp2, c2, w2, changed = graph.apply_delta(g.n, g.row_ptr, g.col, g.w, delta["add_src"], delta["add_dst"],
                                             delta["add_w"], delta["rem_src"], delta["rem_dst"])
    new = graph.column_entries(g.n, rp2, c2, w2)
    F2 = di.update_fluid(r0.F, r0.H, D, di.spmv(g.n, *old), di.spmv(g.n, *new))
    # only the changed columns contribute to d (P' - P) H
    untouched = np.setdiff1d(np.arange(g.n), changed)
    Hm = r0.H.copy()
    Hm[untouched] = 0.0
    F2b = di.update_fluid(r0.F, Hm, D, di.spmv(g.n, *old), di.spmv(g.n, *new))
    assert np.abs(F2 - F2b).max() < 1e-16
    assert (F2 < 0).any() or len(delta["rem_src"]) == 0
    r1 = di.sweep_run(g.n, *new, D, F2, r0.H, tol=1e-13)
    x_new = dense.dense_solve(graph.dense_P(g.n, *new), D, Z)
    assert np.abs(r1.H - x_new).sum() <= 1e-12
    # Eq. (12) re-based at the update: (H - H_k0) + F = F'_0 + dP'(H - H_k0)
    Pn = graph.dense_P(g.n, *new)
    dH = r1.H - r0.H
    assert np.abs(dH + r1.F - F2 - D * (Pn @ dH)).max() < 1e-14


def test_apply_delta_rejects_absent_edge_and_roundtrips():
    rp, c, _ = csr_from_edges(3, [(0, 1), (1, 2)])
    with pytest.raises(KeyError):
        graph.apply_delta(3, rp, c, None, [], [], None, [0], [2])
    rp2, c2, _, ch = graph.apply_delta(3, rp, c, None, [0], [2], None, [0], [1])
    assert list(rp2) == [0, 1, 2, 2] and list(c2) == [2, 2] and list(ch) == [0]
    rp3, c3, _, _ = graph.apply_delta(3, rp2, c2, None, [0], [1], None, [0], [2])
    assert list(rp3) == list(rp) and list(c3) == list(c)


# ------------------------------------------------- tile-local sweeps (R12)
def test_tiled_sweep_chain_exact_in_one_sweep():
    # 3-chain inside one tile, 3 local rounds: D = (0.05, 0.05+0.0425, 0.05+0.0425+0.036125)
    ch = load("chain3.txt")
    rp, c, _ = csr_from_edges(3, ch["edges"])
    cp, ri, pv = graph.column_entries(3, rp, c)
    st = di.di_init(3, ch["d"])
    r = di.tiled_sweep_run(3, cp, ri, pv, ch["d"], st.F, st.H, tile=4, rounds=3, tol=0, max_sweeps=1)
    assert np.allclose(r.H, ch["x"], rtol=0, atol=1e-17) and np.all(r.F == 0)
    assert r.leak == pytest.approx(ch["leak"], abs=1e-17)


def test_tiled_one_round_equals_theta0_sweep():
    g = small_graph(300, 12, weighted=True)
    cp, ri, pv = cols_of(g)
    st = di.di_init(g.n, D)
    for k in (1, 3, 8):
        a = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=32, rounds=1, tol=0, max_sweeps=k)
        b = di.sweep_run(g.n, cp, ri, pv, D, st.F, st.H, theta=0.0, tol=0, max_sweeps=k)
        assert np.allclose(a.H, b.H, rtol=1e-14, atol=0) and np.allclose(a.F, b.F, rtol=1e-13, atol=1e-20)
        assert a.edges == b.edges and a.nodes == b.nodes


def test_tiled_waves_absorb_in_the_same_sweep():
    # R15: tile 0 -> tile 1 push (edge 0 -> 4, tile = 4): with two waves tile 1
    # takes it in during the sweep that produced it, with one wave a sweep later
    n, d = 8, 0.85
    rp, c, _ = csr_from_edges(n, [(0, 4)])
    cp, ri, pv = graph.column_entries(n, rp, c)
    f0 = (1 - d) / n
    st = di.di_init(n, d)
    r2 = di.tiled_sweep_run(n, cp, ri, pv, d, st.F, st.H, tile=4, rounds=1, tol=0, max_sweeps=1, waves=2)
    assert r2.H[0] == f0 and r2.H[4] == pytest.approx(f0 * (1 + d), rel=1e-15) and np.all(r2.F == 0)
    assert r2.leak == pytest.approx(n * f0 + d * f0 - f0, rel=1e-15)      # all but node 0 dangling
    r1 = di.tiled_sweep_run(n, cp, ri, pv, d, st.F, st.H, tile=4, rounds=1, tol=0, max_sweeps=1, waves=1)
    assert r1.H[4] == f0 and r1.F[4] == pytest.approx(d * f0, rel=1e-15)
    # one wave per tile from node 4's side: the push goes back to the earlier wave
    rp, c, _ = csr_from_edges(n, [(4, 0)])
    cp, ri, pv = graph.column_entries(n, rp, c)
    r = di.tiled_sweep_run(n, cp, ri, pv, d, st.F, st.H, tile=4, rounds=1, tol=0, max_sweeps=1, waves=2)
    assert r.H[0] == f0 and r.F[0] == pytest.approx(d * f0, rel=1e-15)


def test_tiled_partitions_defer_cross_pushes():
    # R16: the same tile-0 -> tile-1 push with the tiles in different partitions
    # reaches node 4 only after the sweep, even with two waves
    n, d = 8, 0.85
    rp, c, _ = csr_from_edges(n, [(0, 4)])
    cp, ri, pv = graph.column_entries(n, rp, c)
    f0 = (1 - d) / n
    st = di.di_init(n, d)
    r = di.tiled_sweep_run(n, cp, ri, pv, d, st.F, st.H, tile=4, rounds=1, tol=0, max_sweeps=1, waves=2,
                           bounds=[0, 4, 8])
    assert r.H[4] == f0 and r.F[4] == pytest.approx(d * f0, rel=1e-15) and r.F.sum() == r.F[4]
    # partition bound inside a tile: the local push 1 -> 2 (same tile) is still local
    rp, c, _ = csr_from_edges(n, [(1, 2)])
    cp, ri, pv = graph.column_entries(n, rp, c)
    r = di.tiled_sweep_run(n, cp, ri, pv, d, st.F, st.H, tile=4, rounds=2, tol=0, max_sweeps=1, waves=2,
                           bounds=[0, 2, 8])
    assert r.H[2] == pytest.approx(f0 * (1 + d), rel=1e-15) and np.all(r.F == 0)


@pytest.mark.parametrize("waves", [1, 2, 3])
def test_tiled_partition_limits(waves):
    g = small_graph(320, 21, weighted=True)
    cp, ri, pv = cols_of(g)
    st = di.di_init(g.n, D)
    T = 16
    for k in (1, 4):
        base = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=T, rounds=2, tol=0, max_sweeps=k, waves=waves)
        # one partition: the unpartitioned schedule, bit for bit
        one = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=T, rounds=2, tol=0, max_sweeps=k, waves=waves,
                                 bounds=[0, g.n])
        assert np.array_equal(one.H, base.H) and np.array_equal(one.F, base.F)
        # a partition per tile: every remote push waits for the sweep's end, so the
        # waves no longer matter -- the one-wave schedule (up to summation order)
        per = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=T, rounds=2, tol=0, max_sweeps=k, waves=waves,
                                 bounds=list(range(0, g.n, T)) + [g.n])
        w1 = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=T, rounds=2, tol=0, max_sweeps=k, waves=1)
        assert np.allclose(per.H, w1.H, rtol=1e-13, atol=0) and np.allclose(per.F, w1.F, rtol=1e-12, atol=1e-20)
        assert per.edges == w1.edges


@pytest.mark.parametrize("tile,rounds,waves,bounds", [(16, 2, 1, None), (64, 5, 1, None), (1024, 3, 1, None),
                                                      (16, 2, 2, None), (32, 3, 3, None), (16, 1, 5, None),
                                                      (16, 2, 2, (0, 64, 130, 200)), (32, 3, 3, (0, 96, 200))])
def test_tiled_conservation_and_convergence(tile, rounds, waves, bounds):
    g = small_graph(200, 13)
    cp, ri, pv = cols_of(g)
    P = graph.dense_P(g.n, cp, ri, pv)
    st = di.di_init(g.n, D)
    F, H, lk = st.F, st.H, 0.0
    for _ in range(6):
        r = di.tiled_sweep_run(g.n, cp, ri, pv, D, F, H, tile=tile, rounds=rounds, tol=0, max_sweeps=1, leak=lk,
                               waves=waves, bounds=bounds)
        F, H, lk = r.F, r.H, r.leak
        assert np.abs(H + F - st.F0 - D * (P @ H)).max() <= 1e-15           # Eq. (12)
        assert lk == pytest.approx(H[graph.dangling_mask(g.n, g.row_ptr)].sum(), abs=1e-15)
    x = dense.dense_solve(P, D, synth.uniform_Z(g.n))
    r = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=tile, rounds=rounds, tol=1e-13, waves=waves, bounds=bounds)
    assert np.abs(r.H - x).sum() <= 1e-12
    # more local rounds never need more sweeps than one round
    r1 = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=tile, rounds=1, tol=1e-13, waves=waves, bounds=bounds)
    assert r.steps <= r1.steps


# ----------------------------------------------- §3.3 completed bound, pinned
def test_bound_completed_hand_value():
    # PAPER §3.3 final display |x - (1-d)/(1-d-d l) H| = |F|/(1-d-d l) with
    # |F|_1 = 0.1, l = 0.05, d = 0.85: 0.1 / (0.15 - 0.0425) = 0.1 / 0.1075
    assert di.bound_completed(np.array([0.04, -0.06]), 0.85, 0.05) == pytest.approx(0.9302325581395349, rel=1e-15)
    # no leak: factor 1
    assert di.normalized_history(np.array([1.0]), 0.85, 0.0)[0] == 1.0
    # single dangling node after one step: H = 0.15, l = 0.15 -> factor 0.15 / 0.0225 = 20/3,
    # normalised H = 1 = the completed solution (P completed = (1): x = 0.85 x + 0.15)
    assert di.normalized_history(np.array([0.15]), 0.85, 0.15)[0] == pytest.approx(1.0, rel=1e-15)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bound_completed_is_the_exact_distance(seed):
    # §3.3: "the exact L1 distance between x and the normalized H is equal to
    # |F_k| / (1-d-d l_k)": against the dense completed solve (a wrong denominator
    # or normalisation factor breaks the equality), at several intermediate steps
    rng = np.random.default_rng(seed)
    n = 40
    deg = rng.integers(0, 4, size=n)
    deg[rng.random(n) < 0.2] = 0
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = rng.integers(0, n, size=rp[-1]).astype(np.int32)
    cp, ri, pv = graph.column_entries(n, rp, col, None)
    xc = dense.dense_solve(graph.dense_P(n, cp, ri, pv), D, synth.uniform_Z(n), completed=True)
    st = di.di_init(n, D)
    for k in (1, 5, 17, 60):
        r = di.seq_run(n, cp, ri, pv, D, st.F, st.H, sched="cyc", tol=0, max_steps=k)
        dist = np.abs(xc - di.normalized_history(r.H, D, r.leak)).sum()
        assert dist == pytest.approx(di.bound_completed(r.F, D, r.leak), rel=1e-12)
        assert r.leak > 0 or k < 3
