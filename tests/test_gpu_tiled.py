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
