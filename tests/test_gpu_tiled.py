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
    # ragged: n not a multiple of the 1024-node tile
    spec = synth.CONFIGS[1].scaled(10_007, seed=6, weighted=weighted)
    g = synth.generate(spec)
    cp, ri, pv = graph.column_entries(g.n, g.row_ptr, g.col, g.w)
    st = di.di_init(g.n, D)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    for k in (1, 2, 5):
        _, res = G.solve(d=D, tol=0.0, variant="tiled", local_rounds=rounds, max_sweeps=k)
        F, H, _, leak = G.state()
        r = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=1024, rounds=rounds, tol=0, max_sweeps=k)
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
    spec = synth.CONFIGS[4].scaled(20_000, seed=2)
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
