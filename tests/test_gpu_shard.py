"""GPU tests of the sharded path (libdit di_shard_* through paper_1501_06350_b200/dist.py).

Only one GPU is available, so R ranks are emulated in one process: R shard
handles on cuda:0 driven in lock step by the same dist.solve() protocol, with
the all-to-all / all-reduce done by device copies (LockstepCollectives below,
test infrastructure).  No kernel ever waits on another rank.  A world_size=1
NCCL run checks the torch.distributed collectives themselves.
"""
import socket

import numpy as np
import pytest
import torch

import synth
from oracle import di, graph

pytestmark = pytest.mark.gpu
D = 0.85


class LockstepCollectives:
    """All ranks in one process: collectives as device copies (same stream)."""

    def plan(self, shards, bounds):
        world = len(shards)
        per_send = []
        for s in shards:
            ids = s.ghost_ids.cpu().numpy().astype(np.int64)
            owner = np.searchsorted(np.asarray(bounds), ids, side="right") - 1
            s.send_counts = np.bincount(owner, minlength=world).astype(np.int64).tolist()
            per_send.append((ids, owner))
        self.soff = [np.concatenate([[0], np.cumsum(s.send_counts)]) for s in shards]
        for r, s in enumerate(shards):
            idx = [per_send[q][0][per_send[q][1] == r] - s.lo for q in range(world)]
            s.set_recv(torch.tensor(np.concatenate(idx).astype(np.int32), device=s.dev),
                       [len(x) for x in idx])
        self.roff = [np.concatenate([[0], np.cumsum(s.recv_counts)]) for s in shards]

    def allreduce_stats(self, shards):
        allst = torch.cat([s.stats for s in shards])        # the all-gather, rank order
        for s in shards:
            s.gathered.copy_(allst)

    def alltoall(self, shards):
        for r, s in enumerate(shards):
            for q, sq in enumerate(shards):
                c = sq.send_counts[r]
                if c:
                    a, b = int(self.roff[r][q]), int(self.soff[q][r])
                    s.recv[a:a + c].copy_(sq.send[b:b + c])


def _shards(spec, world):
    from paper_1501_06350_b200.dist import CudaShard, node_ranges
    bounds = node_ranges(spec.n, world)
    out = []
    for r in range(world):
        g = synth.generate(spec, bounds[r], bounds[r + 1])
        out.append(CudaShard(spec.n, bounds[r], bounds[r + 1], g.row_ptr, g.col, g.w,
                             stream=torch.cuda.current_stream()))
    return out, bounds


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1501_06350_b200  # noqa: F401
    return True


@pytest.mark.parametrize("world,variant", [(2, 0), (4, 1), (3, 2), (2, 3), (3, 3)])
def test_lockstep_shards_match_oracle(gpu, world, variant):
    from paper_1501_06350_b200 import dist
    spec = synth.CONFIGS[1].scaled(200_000, seed=8, weighted=True)
    shards, bounds = _shards(spec, world)
    coll = LockstepCollectives()
    coll.plan(shards, bounds)
    Hs, res = dist.solve(shards, coll, d=D, tol=1e-12, variant=variant)
    H = torch.cat(Hs).cpu().numpy()
    g = synth.generate(spec)
    ref = di.di_solve(g.n, g.row_ptr, g.col, g.w, D, tol=1e-12)
    assert np.abs(H - ref.H).sum() <= 1e-9
    assert len({r["sweeps"] for r in res}) == 1 and all(r["residual_l1"] <= 1e-12 for r in res)
    assert sum(s.n_ghost for s in shards) > 0
    for s in shards:
        s.close()


@pytest.mark.parametrize("world,variant", [(2, 2), (3, 3)])
def test_lockstep_shards_completion_uses_global_leak(gpu, world, variant):
    # PAPER §3.3 on shards: every rank's completion factor (1-d)/(1-d-d l) and
    # bound |F|/(1-d-d l) take the leak l of the WHOLE graph (all-gathered with
    # the residual), so the concatenated H is the completed solution
    from paper_1501_06350_b200 import DANGLING, dist
    spec = synth.CONFIGS[1].scaled(60_000, seed=18, weighted=True)
    shards, bounds = _shards(spec, world)
    coll = LockstepCollectives()
    coll.plan(shards, bounds)
    Hs, res = dist.solve(shards, coll, d=D, tol=1e-12, variant=variant, dangling=DANGLING["complete"])
    H = torch.cat(Hs).cpu().numpy()
    g = synth.generate(spec)
    ref = di.di_solve(g.n, g.row_ptr, g.col, g.w, D, tol=1e-12)
    xc = di.normalized_history(ref.H, D, ref.leak)
    assert abs(H.sum() - 1.0) <= 1e-9
    assert np.abs(H - xc).sum() <= 1e-9
    assert len({r["leak"] for r in res}) == 1 and res[0]["leak"] == pytest.approx(ref.leak, rel=1e-9)
    assert len({r["norm_factor"] for r in res}) == 1
    assert all(r["bound"] == pytest.approx(r["residual_l1"] / (1 - D - D * r["leak"]), rel=1e-15) for r in res)
    for s in shards:
        s.close()


def test_lockstep_theta0_sweeps_elementwise(gpu):
    from paper_1501_06350_b200 import dist
    spec = synth.CONFIGS[0].scaled(5000, seed=4, weighted=True)
    shards, bounds = _shards(spec, 2)
    coll = LockstepCollectives()
    coll.plan(shards, bounds)
    Hs, res = dist.solve(shards, coll, d=D, tol=0.0, theta=0.0, max_sweeps=5)
    g = synth.generate(spec)
    cp, ri, pv = graph.column_entries(g.n, g.row_ptr, g.col, g.w)
    st = di.di_init(g.n, D)
    r = di.sweep_run(g.n, cp, ri, pv, D, st.F, st.H, theta=0.0, tol=0, max_sweeps=5)
    assert all(x["sweeps"] == 5 for x in res)
    assert np.allclose(torch.cat(Hs).cpu().numpy(), r.H, rtol=1e-13, atol=1e-18)


@pytest.mark.parametrize("weighted,world", [(False, 2), (True, 2), (True, 3)])
def test_lockstep_tiled_sweeps_elementwise(gpu, weighted, world):
    # shard bounds on multiples of W tiles: the sharded tiled schedule is exactly
    # the oracle's tiled sweep with the shards as partitions (cross-shard pushes
    # land after the sweep, R12/R13/R15/R16)
    from paper_1501_06350_b200 import _lib, dist
    T, W = _lib.DI_TILE_NODES, _lib.DI_TILE_WAVES
    spec = synth.CONFIGS[1].scaled(world * 4 * W * T, seed=12, weighted=weighted)
    shards, bounds = _shards(spec, world)
    assert all(b % (W * T) == 0 for b in bounds)
    coll = LockstepCollectives()
    coll.plan(shards, bounds)
    g = synth.generate(spec)
    cp, ri, pv = graph.column_entries(g.n, g.row_ptr, g.col, g.w)
    st = di.di_init(g.n, D)
    for k in (1, 3):
        Hs, res = dist.solve(shards, coll, d=D, tol=0.0, variant=3, local_rounds=3, max_sweeps=k)
        r = di.tiled_sweep_run(g.n, cp, ri, pv, D, st.F, st.H, tile=T, rounds=3, tol=0, max_sweeps=k, waves=W,
                               bounds=list(bounds))
        assert all(x["sweeps"] == k for x in res)
        assert np.allclose(torch.cat(Hs).cpu().numpy(), r.H, rtol=1e-12, atol=1e-20)
        assert sum(x["diffused_edges"] for x in res) == r.edges
    for s in shards:
        s.close()


def test_nccl_world1(gpu):
    import torch.distributed as tdist

    from paper_1501_06350_b200 import dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    tdist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                             device_id=torch.device("cuda", 0))
    try:
        spec = synth.CONFIGS[0].scaled(4000, seed=3)
        shards, bounds = _shards(spec, 1)
        coll = dist.TorchCollectives()
        coll.plan(shards, bounds)
        g = synth.generate(spec)
        ref = di.di_solve(g.n, g.row_ptr, g.col, g.w, D, tol=1e-12)
        for variant in (0, 3):
            Hs, res = dist.solve(shards, coll, d=D, tol=1e-12, variant=variant)
            assert np.abs(Hs[0].cpu().numpy() - ref.H).sum() <= 1e-9
        shards[0].close()
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_lockstep_tiled_full_size_sampled(gpu, world):
    # BASELINE configs[2] at full size (50M nodes, ~1B weighted edges) split over
    # `world` lock-step shards, in the sharded bench's schedule (tiled, 4 local rounds, DI_TILE_WAVES waves
    # per rank): converged to tol, and Eq. (12) H + F = F0 + d P H on sampled nodes
    # (the oracle's float64 arithmetic over the global CSR)
    from paper_1501_06350_b200 import _lib, dist
    from tests.test_gpu import _config2_graph, _sampled_identity
    spec = synth.CONFIGS[2]
    g = _config2_graph()
    bounds = dist.node_ranges(g.n, world)
    shards = [dist.CudaShard(g.n, lo, hi, g.row_ptr[lo:hi + 1] - g.row_ptr[lo],
                             g.col[g.row_ptr[lo]:g.row_ptr[hi]], g.w[g.row_ptr[lo]:g.row_ptr[hi]],
                             stream=torch.cuda.current_stream())
              for lo, hi in zip(bounds[:-1], bounds[1:])]
    coll = LockstepCollectives()
    coll.plan(shards, bounds)
    Hs, res = dist.solve(shards, coll, d=D, tol=spec.tol, variant=3, local_rounds=4)
    assert all(r["converged"] for r in res)
    F = torch.empty(g.n, dtype=torch.float64, device="cuda")
    H = torch.empty_like(F)
    for s, lo, hi in zip(shards, bounds[:-1], bounds[1:]):
        _lib.di_get_state(s.h, F[lo:hi], H[lo:hi])
    F, H = F.cpu().numpy(), H.cpu().numpy()
    assert np.abs(F).sum() <= spec.tol
    assert np.array_equal(torch.cat(Hs).cpu().numpy(), H)
    assert _sampled_identity(g, H, F, D, np.random.default_rng(2)) < 1e-15
    for s in shards:
        s.close()
