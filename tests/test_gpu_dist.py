"""Real libdit shards in separate processes (world 2, gloo, host-staged
collectives, every rank on cuda:0): the dist.solve protocol of the multi-GPU
bench with CudaShard instead of the CPU stand-in, against the oracle.  No kernel
ever waits on another rank: the exchanges are host-side collectives."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth
from oracle import di

pytestmark = pytest.mark.gpu
D = 0.85


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spec, variant, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1501_06350_b200 import dist as pdist
        bounds = pdist.node_ranges(spec.n, world)
        lo, hi = bounds[rank], bounds[rank + 1]
        g = synth.generate(spec, lo, hi)
        sh = pdist.CudaShard(spec.n, lo, hi, g.row_ptr, g.col, g.w, device=0, stream=torch.cuda.current_stream())
        coll = pdist.TorchCollectives(stage_host=True)
        coll.plan([sh], bounds)
        H, res = pdist.solve([sh], coll, d=D, tol=1e-12, variant=variant)
        np.save(os.path.join(out_dir, f"H{rank}.npy"), H[0].cpu().numpy())
        np.save(os.path.join(out_dir, f"meta{rank}.npy"),
                np.array([res[0]["sweeps"], res[0]["residual_l1"], sh.n_ghost]))
        sh.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", [1, 3])   # push, tiled
def test_two_process_cuda_shards_match_oracle(variant, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    spec = synth.CONFIGS[1].scaled(40_000, seed=19, weighted=True)
    mp.spawn(_worker, args=(world, _free_port(), spec, variant, str(tmp_path)), nprocs=world, join=True)
    H = np.concatenate([np.load(tmp_path / f"H{r}.npy") for r in range(world)])
    meta = [np.load(tmp_path / f"meta{r}.npy") for r in range(world)]
    g = synth.generate(spec)
    ref = di.di_solve(g.n, g.row_ptr, g.col, g.w, D, tol=1e-12)
    assert np.abs(H - ref.H).sum() <= 1e-9
    assert len({int(m[0]) for m in meta}) == 1                 # the ranks stopped at the same sweep
    assert all(m[1] <= 1e-12 for m in meta) and all(int(m[2]) > 0 for m in meta)
