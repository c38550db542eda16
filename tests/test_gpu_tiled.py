"""GPU parity of the tile-local schedule (DI_VARIANT_TILED, R12)
against the oracle's step-by-step tiled sweep and the converged solution."""
import numpy as np
import pytest
import torch

import synth
from oracle import dense, di, graph

pytestmark = pytest.mark.gpu
D = 0.85


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1501_06350_b200 as eng
    return eng


@pytest.mark.parametrize("weighted,rounds", [(False, 1), (True, 3), (True, 6)])
def test_tiled_sweeps_elementwise(eng, weighted, rounds):
    # ragged: n not a multiple of the DI_TILE_NODES tile
    spec = synth.CONFIGS[1].scaled(10_007, seed=6, weighted=weighted)
    g = synth.generate(spec)
    cp, ri, pv = graph.column_entries(g.n, g.row_ptr, g.col, g.w)
    st = di.di_init(g.n, D)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    for k in (1, 2, 5):
        _, res = G.solve(d=D, tol=0.0, variant="tiled", local_rounds=rounds, max_sweeps=k)
        F, H, _, leak = G.state()
        r = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=eng._lib.DI_TILE_NODES, rounds=rounds, tol=0, max_sweeps=k,
                                 waves=eng._lib.DI_TILE_WAVES)
        assert res["sweeps"] == k
        assert np.allclose(H.cpu().numpy(), r.H, rtol=1e-13, atol=1e-20)
        assert np.allclose(F.cpu().numpy(), r.F, rtol=1e-11, atol=1e-20)
        assert leak == pytest.approx(r.leak, rel=1e-12, abs=1e-20)
        assert res["diffused_edges"] == r.edges and res["diffused_nodes"] == r.nodes


@pytest.mark.parametrize("rounds", [2, 4, 8])
def test_tiled_converges_to_oracle(eng, rounds):
    spec = synth.CONFIGS[1].scaled(100_000, seed=7, weighted=True)
    g = synth.generate(spec)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    H, res = G.solve(d=D, tol=1e-12, variant="tiled", local_rounds=rounds)
    ref = di.di_solve(g.n, g.row_ptr, g.col, g.w, D, tol=1e-12)
    assert res["converged"]
    assert np.abs(H.cpu().numpy() - ref.H).sum() <= 1e-9
    # deterministic: a second solve is bitwise identical
    H2, _ = G.solve(d=D, tol=1e-12, variant="tiled", local_rounds=rounds)
    assert torch.equal(H, H2)


def test_tiled_dense_hubs_and_completion(eng):
    rng = np.random.default_rng(3)
    n = 3000
    deg = rng.integers(0, 8, size=n)
    deg[5] = 2500
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = rng.integers(0, n, size=rp[-1]).astype(np.int32)
    col[rng.random(rp[-1]) < 0.2] = 1030          # remote hub
    col[rng.random(rp[-1]) < 0.1] = 3             # local hub (tile 0)
    P = graph.dense_P(n, *graph.column_entries(n, rp, col, None))
    x = dense.dense_solve(P, D, synth.uniform_Z(n))
    xc = dense.dense_solve(P, D, synth.uniform_Z(n), completed=True)
    G = eng.DIGraph(n, rp, col)
    H, _ = G.solve(d=D, tol=1e-13, variant="tiled", local_rounds=5)
    assert np.abs(H.cpu().numpy() - x).sum() <= 1e-9
    Hc, _ = G.solve(d=D, tol=1e-13, variant="tiled", local_rounds=5, dangling="complete")
    assert np.abs(Hc.cpu().numpy() - xc).sum() <= 1e-9


def test_tiled_after_update(eng):
    spec = synth.CONFIGS[4].scaled(20_000, seed=2, weighted=False)
    g = synth.generate(spec)
    delta = synth.rewire(spec, g, fraction=0.01, seed=5)
    G = eng.DIGraph(g.n, g.row_ptr, g.col)
    G.solve(d=D, tol=1e-12, variant="tiled")
    G.update_edges(**delta)
    H, r = G.resume(tol=1e-12, variant="tiled")
    rp2, c2, w2, _ = graph.apply_delta(g.n, g.row_ptr, g.col, None, delta["add_src"], delta["add_dst"], None,
                                       delta["rem_src"], delta["rem_dst"])
    cold = di.di_solve(g.n, rp2, c2, None, D, tol=1e-12)
    assert np.abs(H.cpu().numpy() - cold.H).sum() <= 1e-9


def _delta_entries(G):
    """delta in-edges the kept tile plan carries (dit_delta.cu debug symbol)"""
    import ctypes
    from paper_1501_06350_b200 import _lib
    f = _lib._lib.di_debug_delta_entries
    f.restype, f.argtypes = ctypes.c_longlong, [ctypes.c_void_p]
    return int(f(G.handle))


@pytest.mark.parametrize("weighted", [False, True])
def test_tiled_update_keeps_plan_two_updates(eng, weighted):
    # DESIGN.md R18: the tile plan stays across Theorem 4 updates, corrected by
    # delta in-edges (+w added, -w per removed CSR entry); two updates in a row,
    # the second removing edges the first added, against cold oracle solves
    spec = synth.CONFIGS[4].scaled(60_000, seed=21, weighted=weighted)
    g = synth.generate(spec)
    d1 = synth.rewire(spec, g, fraction=0.01, seed=6)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    G.solve(d=D, tol=1e-12, variant="tiled")
    m0 = G.m
    G.update_edges(**d1)
    rp1, c1, w1, _ = graph.apply_delta(g.n, g.row_ptr, g.col, g.w, d1["add_src"], d1["add_dst"], d1["add_w"],
                                       d1["rem_src"], d1["rem_dst"])
    n_removed = m0 + len(d1["add_src"]) - len(c1)            # CSR entries (parallel copies) removed
    # edges inside a tile patch the plan's slots; the rest stay delta entries
    assert 0 < _delta_entries(G) < len(d1["add_src"]) + n_removed
    H1, r1 = G.resume(tol=1e-12, variant="tiled")
    cold1 = di.di_solve(g.n, rp1, c1, w1, D, tol=1e-12)
    assert r1["converged"]
    assert np.abs(H1.cpu().numpy() - cold1.H).sum() <= 1e-9
    # second update: remove 200 distinct edges the first one added, add new ones
    pairs = np.unique(np.stack([d1["add_src"], d1["add_dst"]], 1), axis=0)[:200]
    rng = np.random.default_rng(3)
    k = 500
    a_src = rng.integers(0, g.n, size=k).astype(np.int32)
    a_dst = rng.integers(0, g.n, size=k).astype(np.int32)
    a_w = (0.5 + rng.random(k)).astype(np.float32) if weighted else None
    G.update_edges(add_src=a_src, add_dst=a_dst, add_w=a_w, rem_src=pairs[:, 0].astype(np.int32),
                   rem_dst=pairs[:, 1].astype(np.int32))
    rp2, c2, w2, _ = graph.apply_delta(g.n, rp1, c1, w1, a_src, a_dst, a_w, pairs[:, 0], pairs[:, 1])
    assert G.m == len(c2)
    H2, r2 = G.resume(tol=1e-12, variant="tiled")
    cold2 = di.di_solve(g.n, rp2, c2, w2, D, tol=1e-12)
    assert r2["converged"]
    assert np.abs(H2.cpu().numpy() - cold2.H).sum() <= 1e-9
    # a fresh plan of the final graph (no delta) reaches the same solution
    G2 = eng.DIGraph(g.n, rp2, c2, w2)
    H3, _ = G2.solve(d=D, tol=1e-12, variant="tiled")
    assert _delta_entries(G2) == 0
    assert np.abs(H3.cpu().numpy() - cold2.H).sum() <= 1e-9



def test_tiled_update_keeps_plan_f64_weights(eng):
    # float64 weights that are not floats (stored as f64, k_patch_ell's double
    # slots); the update's weights too; against the cold oracle solve
    spec = synth.CONFIGS[4].scaled(40_000, seed=23, weighted=True)
    g = synth.generate(spec)
    rng = np.random.default_rng(5)
    w64 = g.w.astype(np.float64) + rng.random(len(g.w)) * 1e-9
    d1 = synth.rewire(spec, g, fraction=0.01, seed=8)
    a_w = d1["add_w"].astype(np.float64) + 1e-10
    G = eng.DIGraph(g.n, g.row_ptr, g.col, w64)
    G.solve(d=D, tol=1e-12, variant="tiled")
    G.update_edges(add_src=d1["add_src"], add_dst=d1["add_dst"], add_w=a_w, rem_src=d1["rem_src"],
                   rem_dst=d1["rem_dst"])
    assert _delta_entries(G) > 0
    H, r = G.resume(tol=1e-12, variant="tiled")
    rp2, c2, w2, _ = graph.apply_delta(g.n, g.row_ptr, g.col, w64, d1["add_src"], d1["add_dst"], a_w,
                                       d1["rem_src"], d1["rem_dst"])
    cold = di.di_solve(g.n, rp2, c2, w2, D, tol=1e-12)
    assert r["converged"]
    assert np.abs(H.cpu().numpy() - cold.H).sum() <= 1e-9
    # a cold solve on the same handle: the kept plan with its delta entries
    H2, r2 = G.solve(d=D, tol=1e-12, variant="tiled")
    assert r2["converged"]
    assert np.abs(H2.cpu().numpy() - cold.H).sum() <= 1e-9


def test_tiled_update_dangling_transitions(eng):
    # nodes losing every out-edge (their fluid leaks from then on, §3.3) and
    # dangling nodes gaining their first ones, through the kept plan; drop and
    # 1/n completion against the dense solve of the new graph
    rng = np.random.default_rng(8)
    n = 2000
    deg = rng.integers(0, 7, size=n)
    deg[rng.random(n) < 0.1] = 0
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = rng.integers(0, n, size=rp[-1]).astype(np.int32)
    local = rng.random(rp[-1]) < 0.6                       # many edges inside the 512-node tiles
    src = np.repeat(np.arange(n), deg)
    col[local] = ((src[local] // 512) * 512 + rng.integers(0, 512, size=local.sum())) % n
    G = eng.DIGraph(n, rp, col)
    G.solve(d=D, tol=1e-13, variant="tiled")
    lose = [i for i in range(n) if deg[i] > 0][:40]       # every out-edge removed
    rem = sorted({(i, int(t)) for i in lose for t in col[rp[i]:rp[i + 1]]})
    gain = [i for i in range(n) if deg[i] == 0][:40]
    # the first ten gain only a self-loop (all their fluid stays: pushed inside the rounds, R18)
    add = [(i, i) for i in gain[:10]] + [(i, int(rng.integers(0, n))) for i in gain[10:] for _ in range(3)]
    a = np.array(add, np.int32)
    r_ = np.array(rem, np.int32)
    G.update_edges(add_src=a[:, 0], add_dst=a[:, 1], rem_src=r_[:, 0], rem_dst=r_[:, 1])
    assert _delta_entries(G) > 0
    rp2, c2, _, _ = graph.apply_delta(n, rp, col, None, a[:, 0], a[:, 1], None, r_[:, 0], r_[:, 1])
    P = graph.dense_P(n, *graph.column_entries(n, rp2, c2, None))
    x = dense.dense_solve(P, D, synth.uniform_Z(n))
    H, r = G.resume(tol=1e-13, variant="tiled")
    assert r["converged"]
    assert np.abs(H.cpu().numpy() - x).sum() <= 1e-9
    xc = dense.dense_solve(P, D, synth.uniform_Z(n), completed=True)
    Hc, _ = G.resume(tol=1e-13, variant="tiled", dangling="complete")
    assert np.abs(Hc.cpu().numpy() - xc).sum() <= 1e-9

def _stress_graph(wdtype):
    """Every tile-kernel path at once: a tile whose local edges overflow shared
    memory (unstaged rounds), a remote hub spanning several heavy chunks, a tile
    whose light remote records overflow (all of its targets heavy), dangling
    nodes, parallel edges and self-loops."""
    rng = np.random.default_rng(11)
    n = 5000
    rows = []
    for i in range(n):
        k = int(rng.integers(0, 6))
        rows.append(list(rng.integers(0, n, size=k)))
    rows[7] = list(rng.integers(0, 512, size=30000))        # tile 0: ~30K local edges
    for i in range(600, 3600):                               # hub 4321: ~9000 remote in-edges
        rows[i] += [4321] * 3
    for t in range(1536, 2048):                              # tile 3: 512 targets x 8 remote in-edges
        for q in range(8):
            rows[int(rng.integers(2048, n))].append(t)
    rows[9] += [9, 9, 10, 10]                                # self-loop, parallel edges
    for i in range(0, n, 17):
        rows[i] = []                                         # dangling
    rp = np.zeros(n + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=rp[1:])
    col = np.concatenate([np.asarray(r, np.int64) for r in rows]).astype(np.int32)
    w = None
    if wdtype is not None:
        w = (0.5 + rng.integers(0, 1 << 20, size=len(col)) / float(1 << 19)).astype(wdtype)
        if wdtype == np.float64:
            w += 1e-9 * rng.random(len(col))                 # not representable in float32
    return n, rp, col, w


@pytest.mark.parametrize("wdtype", [None, np.float32, np.float64])
def test_tiled_stress_paths_elementwise(eng, wdtype):
    n, rp, col, w = _stress_graph(wdtype)
    cp, ri, pv = graph.column_entries(n, rp, col, w)
    st = di.di_init(n, D)
    G = eng.DIGraph(n, rp, col, w)
    for k in (1, 2, 6):
        _, res = G.solve(d=D, tol=0.0, variant="tiled", local_rounds=3, max_sweeps=k)
        F, H, _, leak = G.state()
        r = di.tiled_sweep_run(n, cp, ri, pv, D, st.F, st.H, tile=eng._lib.DI_TILE_NODES, rounds=3, tol=0,
                               max_sweeps=k, waves=eng._lib.DI_TILE_WAVES)
        assert res["sweeps"] == k
        assert np.allclose(H.cpu().numpy(), r.H, rtol=1e-12, atol=1e-20)
        assert np.allclose(F.cpu().numpy(), r.F, rtol=1e-10, atol=1e-18)
        assert leak == pytest.approx(r.leak, rel=1e-12, abs=1e-20)
        assert res["diffused_edges"] == r.edges and res["diffused_nodes"] == r.nodes
        assert res["residual_l1"] == pytest.approx(np.abs(r.F).sum(), rel=1e-12)
    H, res = G.solve(d=D, tol=1e-13, variant="tiled", local_rounds=4)
    ref = di.di_solve(n, rp, col, w, D, tol=1e-13)
    assert res["converged"] and np.abs(H.cpu().numpy() - ref.H).sum() <= 1e-9
    # a resume after convergence is a no-op; a second solve is bitwise identical
    H2, _ = G.solve(d=D, tol=1e-13, variant="tiled", local_rounds=4)
    assert torch.equal(H, H2)


def test_tiled_resume_chunks_match_one_call(eng):
    # sweeps split over several calls (flush between calls) = one call
    spec = synth.CONFIGS[1].scaled(30_011, seed=9, weighted=True)
    g = synth.generate(spec)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    H1, r1 = G.solve(d=D, tol=0.0, variant="tiled", max_sweeps=9)
    F1, _, _, _ = G.state()
    G2 = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    G2.solve(d=D, tol=0.0, variant="tiled", max_sweeps=4)
    H2, r2 = G2.resume(tol=0.0, variant="tiled", max_sweeps=5)
    F2, _, _, _ = G2.state()
    assert r2["sweeps"] == 5
    assert np.allclose(H1.cpu().numpy(), H2.cpu().numpy(), rtol=1e-14, atol=0)
    assert np.allclose(F1.cpu().numpy(), F2.cpu().numpy(), rtol=1e-12, atol=1e-22)
