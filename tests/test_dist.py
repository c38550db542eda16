"""Multi-rank host logic of the sharded solver (paper_1501_06350_b200/dist.py),
world_size 2 and 3 over gloo on CPU, each rank running the CPU stand-in of a
libdit shard (tests/_cpu_shard.py).  Checks the partition, the ghost exchange
plan, the all-to-all / all-reduce protocol and the stop test against the
single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import di, graph

D = 0.85


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, tol, theta, max_sweeps, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1501_06350_b200 import build
        build.build()
        from paper_1501_06350_b200 import dist as pdist
        from tests._cpu_shard import CpuShard
        bounds = pdist.node_ranges(spec.n, world)
        lo, hi = bounds[rank], bounds[rank + 1]
        g = synth.generate(spec, lo, hi)
        sh = CpuShard(spec.n, lo, hi, g.row_ptr, g.col, g.w)
        coll = pdist.TorchCollectives()
        coll.plan([sh], bounds)
        H, res = pdist.solve([sh], coll, d=D, tol=tol, theta=theta, max_sweeps=max_sweeps)
        np.save(os.path.join(out_dir, f"H{rank}.npy"), H[0].numpy())
        np.save(os.path.join(out_dir, f"meta{rank}.npy"),
                np.array([res[0]["sweeps"], res[0]["residual_l1"], sh.n_ghost, g.m]))
    finally:
        dist.destroy_process_group()


def _run(world, spec, tol, theta=1.0, max_sweeps=0, tmp_path=None):
    mp.spawn(_worker, args=(world, _free_port(), spec, tol, theta, max_sweeps, str(tmp_path)), nprocs=world,
             join=True)
    H = np.concatenate([np.load(tmp_path / f"H{r}.npy") for r in range(world)])
    meta = [np.load(tmp_path / f"meta{r}.npy") for r in range(world)]
    return H, meta


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solve_matches_oracle(world, tmp_path):
    spec = synth.CONFIGS[1].scaled(20000, seed=5, weighted=True)
    H, meta = _run(world, spec, 1e-12, tmp_path=tmp_path)
    g = synth.generate(spec)
    ref = di.di_solve(g.n, g.row_ptr, g.col, g.w, D, tol=1e-12)
    assert np.abs(H - ref.H).sum() <= 1e-9
    assert all(m[1] <= 1e-12 for m in meta)
    assert len({int(m[0]) for m in meta}) == 1          # every rank stopped at the same sweep
    assert sum(int(m[3]) for m in meta) == g.m
    assert all(int(m[2]) > 0 for m in meta)              # cross-partition edges exist


def test_sharded_sweeps_equal_global_sweeps(tmp_path):
    # theta = 0 (no threshold ties): k sharded sweeps == k global oracle sweeps
    spec = synth.CONFIGS[0].scaled(3000, seed=2)
    H, meta = _run(2, spec, 0.0, theta=0.0, max_sweeps=6, tmp_path=tmp_path)
    g = synth.generate(spec)
    cp, ri, pv = graph.column_entries(g.n, g.row_ptr, g.col, g.w)
    st = di.di_init(g.n, D)
    r = di.sweep_run(g.n, cp, ri, pv, D, st.F, st.H, theta=0.0, tol=0, max_sweeps=6)
    assert all(int(m[0]) == 6 for m in meta)
    assert np.allclose(H, r.H, rtol=1e-13, atol=1e-18)


def test_node_ranges_partition():
    from paper_1501_06350_b200.dist import node_ranges
    for n, w in [(10, 3), (400_000_000, 8), (7, 7), (5, 8)]:
        b = node_ranges(n, w)
        assert b[0] == 0 and b[-1] == n and all(b[i] <= b[i + 1] for i in range(w))
        assert max(b[i + 1] - b[i] for i in range(w)) - min(b[i + 1] - b[i] for i in range(w)) <= 1


def test_bench_spec_weak_scaling_and_config3():
    # bench.py --gpus N: 8 ranks run BASELINE configs[3] itself (400M nodes, 50M per
    # rank); 2 / 4 ranks the same generator on N x 50M nodes (weak-scaling slices)
    from paper_1501_06350_b200.dist import bench_spec, node_ranges
    s8, name8 = bench_spec(8, 2)
    assert s8 == synth.CONFIGS[3] and "configs[3]" in name8 and "8 GPUs" in name8
    b = node_ranges(s8.n, 8)
    assert all(b[r + 1] - b[r] == 50_000_000 for r in range(8))
    for w in (2, 4):
        s, name = bench_spec(w, 2)
        assert s.n == w * 50_000_000 and s.seed == synth.CONFIGS[3].seed and s.deg_cap == 5000
        assert "weak-scaling slice" in name
    s1, _ = bench_spec(2, 2, scale_n=1000)
    assert s1.n == 2000


def test_bench_relaunch_without_enough_gpus():
    # without torchrun, bench.py --gpus N re-executes itself under torch.distributed.run;
    # with fewer visible GPUs than N it says so on one JSON line and exits non-zero
    import json
    import subprocess
    import sys
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode == 1
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert "error" in line and line["n_gpus"] == 2
