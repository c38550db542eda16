"""GPU parity tests: the CUDA engine (through the C ABI) against the CPU oracle.

North-star bar (BASELINE.json): ||H_gpu - H_oracle||_1 <= 1e-9 at tol = 1e-12
(float64 fluid) and the top-1000 ranking identical (ties within the two
solutions' error bounds may swap: both orders are correct, R9).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import dense, di, graph
from tests._golden import csr_from_edges, load

pytestmark = pytest.mark.gpu
D = 0.85
L1_BAR = 1e-9


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1501_06350_b200 as eng
    return eng


def oracle_solve(g, tol=1e-12, theta=1.0, method="sweep", Z=None):
    return di.di_solve(g.n, g.row_ptr, g.col, g.w, D, Z=Z, tol=tol, theta=theta, method=method)


_AUTO = object()


def gpu_solve(eng, g, tol=1e-12, weights=_AUTO, **kw):
    w = g.w if weights is _AUTO else weights
    G = eng.DIGraph(g.n, g.row_ptr, g.col, w)
    H, res = G.solve(d=D, tol=tol, **kw)
    return G, H.cpu().numpy(), res


def assert_topk(h_gpu, h_ref, k, eps):
    k = min(k, len(h_ref))
    ia = np.argsort(-h_gpu, kind="stable")[:k]
    ib = np.argsort(-h_ref, kind="stable")[:k]
    for p in np.flatnonzero(ia != ib):
        assert abs(h_ref[ia[p]] - h_ref[ib[p]]) <= eps, f"rank {p}: {ia[p]} vs {ib[p]}"


# ----------------------------------------------------------------- config 0
@pytest.mark.parametrize("variant", ["push", "pull", "auto"])
def test_config0_parity(eng, variant):
    spec = synth.CONFIGS[0]
    g = synth.generate(spec)
    G, H, res = gpu_solve(eng, g, variant=variant)
    assert res["converged"] and res["residual_l1"] <= 1e-12
    for method in ("sweep", "argmax"):
        r = oracle_solve(g, method=method)
        assert np.abs(H - r.H).sum() <= L1_BAR
    r = oracle_solve(g)
    assert_topk(H, r.H, 1000, 2 * (res["bound"] + r.residual / (1 - D)))
    # same frontier rule => about the same sweep count (threshold ties may differ)
    assert abs(res["sweeps"] - r.steps) <= max(2, r.steps // 20)


def test_theta0_sweeps_elementwise(eng):
    # theta = 0 diffuses every node holding fluid: no threshold ties, so each
    # GPU sweep must equal the oracle sweep up to float64 summation order
    spec = synth.CONFIGS[0].scaled(3001, seed=5, weighted=True)
    g = synth.generate(spec)
    cp, ri, pv = graph.column_entries(g.n, g.row_ptr, g.col, g.w)
    st = di.di_init(g.n, D)
    for variant in ("push", "pull"):
        G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
        for k in (1, 2, 7):
            _, res = G.solve(d=D, tol=0.0, theta=0.0, variant=variant, max_sweeps=k)
            F, H, d, leak = G.state()
            r = di.sweep_run(g.n, cp, ri, pv, D, st.F, st.H, theta=0.0, tol=0, max_sweeps=k)
            assert res["sweeps"] == k
            assert np.allclose(H.cpu().numpy(), r.H, rtol=1e-13, atol=1e-18)
            assert np.allclose(F.cpu().numpy(), r.F, rtol=1e-12, atol=1e-18)
            assert leak == pytest.approx(r.leak, rel=1e-12, abs=1e-18)
            assert res["diffused_edges"] == r.edges and res["diffused_nodes"] == r.nodes


def test_conservation_identity_on_gpu_state(eng):
    spec = synth.CONFIGS[0].scaled(500, seed=3, p_dangling=0.2)
    g = synth.generate(spec)
    P = graph.dense_P(g.n, *graph.column_entries(g.n, g.row_ptr, g.col, g.w))
    F0 = np.full(g.n, (1 - D) / g.n)
    G = eng.DIGraph(g.n, g.row_ptr, g.col)
    for k in (1, 3, 10, 40):
        G.solve(d=D, tol=0.0, max_sweeps=k, variant="push")
        F, H, _, leak = G.state()
        F, H = F.cpu().numpy(), H.cpu().numpy()
        assert np.abs(H + F - F0 - D * (P @ H)).max() < 1e-15          # Eq. (12)
        assert leak == pytest.approx(H[graph.dangling_mask(g.n, g.row_ptr)].sum(), rel=1e-12)


def test_pull_is_bitwise_deterministic(eng):
    g = synth.generate(synth.CONFIGS[1].scaled(20000, seed=4, weighted=True))
    outs = []
    for _ in range(2):
        G, H, res = gpu_solve(eng, g, variant="pull", tol=1e-12)
        outs.append(H)
    assert np.array_equal(outs[0], outs[1])


# ----------------------------------------------------------------- weights
def test_weight_storage_and_parity(eng):
    g = synth.generate(synth.CONFIGS[0].scaled(2000, seed=11, weighted=True))
    r = oracle_solve(g)
    # float32 weights, float64 weights exactly representable as float -> f32 storage
    for w in (g.w, g.w.astype(np.float64)):
        G, H, res = gpu_solve(eng, g, weights=w)
        assert G.weight_storage == eng.DI_W_F32
        assert np.abs(H - r.H).sum() <= L1_BAR
    # float64 weights that are not floats keep f64 storage
    w64 = g.w.astype(np.float64) * (1.0 + 1e-12)
    r64 = di.di_solve(g.n, g.row_ptr, g.col, w64, D, tol=1e-12)
    G, H, res = gpu_solve(eng, g, weights=w64, variant="push")
    assert G.weight_storage == eng.DI_W_F64
    assert np.abs(H - r64.H).sum() <= L1_BAR


# ----------------------------------------------------------------- edge cases
@pytest.mark.parametrize("variant", ["auto", "tiled"])
def test_edge_cases_small_graphs(eng, variant):
    kw = dict(variant=variant)
    # single dangling node: x = (1-d) Z; completed: 1
    G = eng.DIGraph(1, np.array([0, 0]), np.zeros(0, np.int32))
    H, res = G.solve(d=D, tol=0.0, **kw)
    assert H.item() == pytest.approx(0.15, abs=1e-16) and res["leak"] == pytest.approx(0.15)
    H, res = G.solve(d=D, tol=0.0, dangling="complete", **kw)
    assert H.item() == pytest.approx(1.0, abs=1e-14)
    # golden 3-chain and 2-cycle
    ch = load("chain3.txt")
    rp, c, _ = csr_from_edges(3, ch["edges"])
    H, res = eng.DIGraph(3, rp, c).solve(d=ch["d"], tol=0.0, **kw)
    assert np.allclose(H.cpu().numpy(), ch["x"], atol=1e-16)
    cy = load("cycle2.txt")
    rp, c, _ = csr_from_edges(2, cy["edges"])
    H, res = eng.DIGraph(2, rp, c).solve(d=cy["d"], Z=np.array([0.5, 0.5]), tol=1e-15, **kw)
    assert np.allclose(H.cpu().numpy(), cy["x"], atol=1e-14)
    # self-loop only: x = (1-d)/(1-d) Z = 1 on one node
    H, res = eng.DIGraph(1, np.array([0, 1]), np.array([0], np.int32)).solve(d=D, tol=1e-15, **kw)
    assert H.item() == pytest.approx(1.0, abs=1e-13)
    # empty graph n = 0, and nodes without any edge
    G0 = eng.DIGraph(0, np.array([0]), np.zeros(0, np.int32))
    H, res = G0.solve(d=D, tol=1e-12, **kw)
    assert H.numel() == 0 and res["sweeps"] == 0
    Ge = eng.DIGraph(700, np.zeros(701, np.int64), np.zeros(0, np.int32))
    H, res = Ge.solve(d=D, tol=0.0, **kw)
    assert np.allclose(H.cpu().numpy(), 0.15 / 700, rtol=1e-15) and res["converged"]
    # a ring longer than a tile: all pushes remote at the tile seams, exact x = 1/n
    n = 1100
    rp = np.arange(n + 1, dtype=np.int64)
    c = ((np.arange(n) + 1) % n).astype(np.int32)
    H, res = eng.DIGraph(n, rp, c).solve(d=D, tol=1e-14, **kw)
    assert np.abs(H.cpu().numpy() - 1.0 / n).sum() <= 1e-12


@pytest.mark.parametrize("variant", ["push", "pull", "tiled"])
def test_heavy_rows_hubs_and_ragged_sizes(eng, variant):
    # out-degrees far above the 512-edge split, a hub with in-degree far above
    # the 256-edge pull piece, n not a multiple of 32 / 256
    rng = np.random.default_rng(0)
    n = 4099
    deg = rng.integers(0, 6, size=n)
    deg[[0, 17, 4098]] = [2000, 1537, 513]
    deg[rng.choice(n, 40, replace=False)] = 0
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = rng.integers(0, n, size=rp[-1]).astype(np.int32)
    col[rng.random(rp[-1]) < 0.3] = 7       # hub 7
    w = rng.uniform(0.5, 2.0, size=rp[-1])
    g = synth.Graph(n=n, row_ptr=rp, col=col, w=w)
    P = graph.dense_P(n, *graph.column_entries(n, rp, col, w))
    x = dense.dense_solve(P, D, synth.uniform_Z(n))
    G, H, res = gpu_solve(eng, g, variant=variant)
    assert np.abs(H - x).sum() <= L1_BAR
    xc = dense.dense_solve(P, D, synth.uniform_Z(n), completed=True)
    _, Hc, resc = gpu_solve(eng, g, variant=variant, dangling="complete")
    assert np.abs(Hc - xc).sum() <= L1_BAR and abs(Hc.sum() - 1) < 1e-9


def test_nonuniform_Z(eng):
    g = synth.generate(synth.CONFIGS[0].scaled(800, seed=2))
    Z = np.random.default_rng(1).random(g.n)
    Z /= Z.sum()
    r = oracle_solve(g, Z=Z)
    G = eng.DIGraph(g.n, g.row_ptr, g.col)
    H, res = G.solve(d=D, Z=Z, tol=1e-12)
    assert np.abs(H.cpu().numpy() - r.H).sum() <= L1_BAR
    H2, _ = G.solve(d=D, Z=torch.tensor(Z, device="cuda"), tol=1e-12)
    assert np.abs(H2.cpu().numpy() - r.H).sum() <= L1_BAR


def test_invalid_inputs(eng):
    with pytest.raises(eng.DIError) as e:
        eng.DIGraph(3, np.array([0, 1, 2, 3]), np.array([0, 1, 5], np.int32))
    assert e.value.code == 1
    with pytest.raises(eng.DIError):
        eng.DIGraph(2, np.array([0, 2, 1]), np.array([0, 1], np.int32))
    with pytest.raises(eng.DIError):
        eng.DIGraph(2, np.array([0, 1, 2]), np.array([1, 0], np.int32), np.array([1.0, -1.0]))
    G = eng.DIGraph(2, np.array([0, 1, 2]), np.array([1, 0], np.int32))
    with pytest.raises(eng.DIError):
        G.solve(d=1.0)
    with pytest.raises(eng.DIError):
        G.solve(d=0.85, theta=2.0)
    with pytest.raises(eng.DIError) as e:
        G.resume()
    assert e.value.code == 5
    with pytest.raises(eng.DIError) as e:
        G.update_edges(rem_src=np.array([0], np.int32), rem_dst=np.array([0], np.int32))
    assert e.value.code == 4


# ----------------------------------------------------------------- Theorem 4
def test_update_golden_fluid(eng):
    u = load("update3.txt")
    G = eng.DIGraph(3, np.array([0, 1, 1, 1]), np.array([1], np.int32))
    G.set_state(u["d"], u["F"], u["H"])
    G.update_edges(add_src=np.array([0], np.int32), add_dst=np.array([2], np.int32),
                   rem_src=np.array([0], np.int32), rem_dst=np.array([1], np.int32))
    F, H, d, leak = G.state()
    assert np.allclose(F.cpu().numpy(), u["F_new"], atol=1e-16)
    assert np.array_equal(H.cpu().numpy(), u["H"])


@pytest.mark.parametrize("weighted", [False, True])
def test_dynamic_update_matches_cold_solve(eng, weighted):
    spec = synth.CONFIGS[4].scaled(30000, seed=9, weighted=weighted)
    g = synth.generate(spec)
    delta = synth.rewire(spec, g, fraction=0.01, seed=3)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    _, r0 = G.solve(d=D, tol=1e-12)
    G.update_edges(**delta)
    H, r1 = G.resume(tol=1e-12)
    rp2, c2, w2, _ = graph.apply_delta(g.n, g.row_ptr, g.col, g.w, delta["add_src"], delta["add_dst"],
                                       delta["add_w"], delta["rem_src"], delta["rem_dst"])
    cold = di.di_solve(g.n, rp2, c2, w2, D, tol=1e-12)
    assert np.abs(H.cpu().numpy() - cold.H).sum() <= L1_BAR
    assert G.m == len(c2)
    # the warm restart diffuses fewer edges than a cold solve (§3.5 "quickly absorbed")
    G2 = eng.DIGraph(g.n, rp2, c2, w2)
    _, rc = G2.solve(d=D, tol=1e-12)
    assert r1["diffused_edges"] < rc["diffused_edges"]


# ----------------------------------------------------------------- full sizes
def test_config1_full_size(eng):
    spec = synth.CONFIGS[1]
    g = synth.generate(spec)
    r = oracle_solve(g, tol=1e-12)
    for variant, rounds in (("push", 4), ("auto", 4), ("tiled", 3), ("tiled", 4)):
        G, H, res = gpu_solve(eng, g, tol=1e-12, variant=variant, local_rounds=rounds)
        assert res["converged"]
        assert np.abs(H - r.H).sum() <= L1_BAR
        assert_topk(H, r.H, 1000, 2 * (res["bound"] + r.residual / (1 - D)))


def _rewired(spec, seed):
    g = synth.generate(spec)
    delta = synth.rewire(spec, g, fraction=0.01, seed=seed)
    rp2, c2, w2, _ = graph.apply_delta(g.n, g.row_ptr, g.col, g.w, delta["add_src"], delta["add_dst"],
                                       delta["add_w"], delta["rem_src"], delta["rem_dst"])
    return g, delta, rp2, c2, w2


def test_config4_scaled_update_vs_cold_oracle(eng):
    # BASELINE configs[4] (1% of the config-2 graph rewired, warm restart by
    # Theorem 4) at a size the cold oracle solve of the modified graph finishes in seconds
    spec = synth.CONFIGS[4].scaled(400_000, seed=14)
    g, delta, rp2, c2, w2 = _rewired(spec, 4)
    cold = di.di_solve(g.n, rp2, c2, w2, D, tol=1e-12)
    for variant in ("auto", "tiled"):
        G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
        G.solve(d=D, tol=spec.tol, variant=variant)
        G.update_edges(**delta)
        H, r = G.resume(tol=1e-12, variant=variant)
        assert r["converged"]
        assert np.abs(H.cpu().numpy() - cold.H).sum() <= L1_BAR
        assert_topk(H.cpu().numpy(), cold.H, 1000, 2 * (r["bound"] + cold.residual / (1 - D)))


_CFG2 = []


def _config2_graph():
    if not _CFG2:
        _CFG2.append(synth.generate(synth.CONFIGS[2]))
    return _CFG2[0]


def _sampled_identity(g, H, F, d, rng, k=2000):
    """Eq. (12) on sampled nodes i: H_i + F_i - F0_i - d sum_j P_ij H_j, with
    the in-edges of i found by a scan of the CSR (oracle arithmetic, float64)."""
    n = g.n
    sample = np.unique(rng.choice(n, size=k, replace=False))
    deg = np.diff(g.row_ptr)
    wsum = np.ones(n) * deg if g.w is None else np.bincount(
        np.repeat(np.arange(n), deg), weights=g.w.astype(np.float64), minlength=n)
    hit = np.flatnonzero(np.isin(g.col, sample))
    src = np.searchsorted(g.row_ptr, hit, side="right") - 1
    wv = np.ones(len(hit)) if g.w is None else g.w[hit].astype(np.float64)
    contrib = d * H[src] * wv / wsum[src]
    acc = np.zeros(n)
    np.add.at(acc, g.col[hit], contrib)
    F0 = (1 - d) / n
    resid = H[sample] + F[sample] - F0 - acc[sample]
    return np.abs(resid).max()


@pytest.mark.parametrize("variant", ["auto"])
def test_config2_full_size_sampled(eng, variant):
    # configs[2] through the push / pull engine (the tiled schedule at full size is
    # tests/test_gpu_fullsize.py, against the oracle)
    spec = synth.CONFIGS[2]
    g = _config2_graph()
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    H, res = G.solve(d=D, tol=spec.tol, variant=variant, local_rounds=4)
    assert res["converged"] and res["residual_l1"] <= spec.tol
    F, H2, d, leak = G.state()
    H2 = H2.cpu().numpy()
    F = F.cpu().numpy()
    assert np.abs(F).sum() == pytest.approx(res["residual_l1"], rel=1e-9)
    assert _sampled_identity(g, H2, F, D, np.random.default_rng(0)) < 1e-15
    # Theorem 1 through Eq. (12): sum H = (|F0| - |F| - l)/(1-d) for nonnegative F
    assert H2.sum() == pytest.approx((1 - D - F.sum() - D * leak) / (1 - D), abs=1e-9)


def test_release_memory_then_rebuild(eng):
    # the cached pool / sort scratch go back to the driver; a later graph builds and
    # solves as before (configs[1] at full size, tiled)
    from paper_1501_06350_b200 import _lib
    spec = synth.CONFIGS[1]
    g = synth.generate(spec)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    H1, r1 = G.solve(d=D, tol=spec.tol, variant="tiled")
    H1 = H1.cpu().numpy()
    G.close()
    _lib.di_release_memory(0)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    H2, r2 = G.solve(d=D, tol=spec.tol, variant="tiled")
    assert np.array_equal(H1, H2.cpu().numpy()) and r1["sweeps"] == r2["sweeps"]
    G.close()


@pytest.mark.parametrize("variant", ["pull", "tiled"])
def test_completed_bound_and_norm_factor_exact(eng, variant):
    # PAPER §3.3 (final display): with dangling completion the engine returns the
    # normalised history (1-d)/(1-d-d l) H_k, and |x_completed - that|_1 is EXACTLY
    # the returned bound |F_k|/(1-d-d l_k) (pinned on the oracle in test_oracle.py);
    # a wrong leak, factor or denominator on the device breaks the equality
    rng = np.random.default_rng(17)
    n = 900
    deg = rng.integers(0, 6, size=n)
    deg[rng.random(n) < 0.15] = 0
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(deg, out=rp[1:])
    col = rng.integers(0, n, size=rp[-1]).astype(np.int32)
    cp, ri, pv = graph.column_entries(n, rp, col, None)
    xc = dense.dense_solve(graph.dense_P(n, cp, ri, pv), D, synth.uniform_Z(n), completed=True)
    G = eng.DIGraph(n, rp, col)
    for k in (1, 3, 8):
        H, res = G.solve(d=D, tol=0.0, variant=variant, theta=0.0, max_sweeps=k, dangling="complete")
        F, Hraw, _, leak = G.state()
        assert res["leak"] == pytest.approx(leak, rel=1e-15) and leak > 0
        assert res["norm_factor"] == pytest.approx((1 - D) / (1 - D - D * leak), rel=1e-14)
        assert np.allclose(H.cpu().numpy(), res["norm_factor"] * Hraw.cpu().numpy(), rtol=1e-15, atol=0)
        assert res["bound"] == pytest.approx(np.abs(F.cpu().numpy()).sum() / (1 - D - D * leak), rel=1e-13)
        assert np.abs(xc - H.cpu().numpy()).sum() == pytest.approx(res["bound"], rel=1e-9)
