"""One rank of the sharded configs[3] workload on a single B200.

    python scripts/config3_rank.py [--world 8] [--rank 0] [--sweeps 12]

Generates rank `rank`'s slice of bench_spec(world) (configs[3] itself at
world 8: 400M nodes, ~8B weighted edges, int64 row offsets; 50M nodes per
rank), builds its libdit shard and tiled plan, and reports: edges, ghost slots
(= values sent per sweep), the destination-rank split of the exchange, device
memory after the build, and the device time of `sweeps` tiled sweeps run in
isolation (the ghost sums go to the send buffer and are dropped, nothing is
received: the per-rank compute of a sweep, not a solve).  One JSON line.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1501_06350_b200 import _lib  # noqa: E402
from paper_1501_06350_b200.dist import CudaShard, bench_spec, node_ranges  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--sweeps", type=int, default=12)
    a = ap.parse_args()
    spec, name = bench_spec(a.world, 3)
    bounds = node_ranges(spec.n, a.world)
    lo, hi = bounds[a.rank], bounds[a.rank + 1]
    t0 = time.perf_counter()
    g = synth.generate(spec, lo, hi)
    gen_s = time.perf_counter() - t0
    torch.cuda.set_device(0)
    free0, total = torch.cuda.mem_get_info()
    stream = torch.cuda.current_stream()
    sh = CudaShard(spec.n, lo, hi, g.row_ptr, g.col, g.w, device=0, stream=stream)
    ids = sh.ghost_ids.cpu().numpy().astype(np.int64)
    owner = np.searchsorted(np.asarray(bounds), ids, side="right") - 1
    send_counts = np.bincount(owner, minlength=a.world)
    # isolated rank: nothing received (empty segments), own stats only
    sh.set_recv(torch.zeros(1, dtype=torch.int32, device=sh.dev), [0])
    sh.send_counts = send_counts.tolist()
    opts = dict(variant=_lib.DI_VARIANT_TILED, local_rounds=4, max_sweeps=a.sweeps)
    sh.begin(spec.d, 0.0, **opts)
    sh.gathered.copy_(sh.stats)
    sh.control()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(stream)
    for _ in range(a.sweeps):
        sh.sweep()
        sh.apply()
        sh.reduce()
        sh.gathered.copy_(sh.stats)
        sh.control()
    ev[1].record(stream)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    free2, _ = torch.cuda.mem_get_info()
    plan = _lib.di_plan_stats(sh.h)
    out = {"workload": name, "world": a.world, "rank": a.rank, "n_global": spec.n, "n_local": hi - lo,
           "m_local": int(g.m), "row_ptr_dtype": str(g.row_ptr.dtype), "generate_s": round(gen_s, 1),
           "ghost_slots": int(sh.n_ghost), "send_bytes_per_sweep": int(sh.n_ghost) * 8,
           "send_counts_by_rank": send_counts.tolist(),
           "cross_partition_edge_share": float(np.mean((g.col < lo) | (g.col >= hi))),
           "device_mem_used_after_shard_gb": round((free0 - free1) / 1e9, 2),
           "device_mem_used_after_plan_gb": round((free0 - free2) / 1e9, 2),
           "device_mem_total_gb": round(total / 1e9, 1),
           "isolated_sweeps": a.sweeps, "ms_per_isolated_sweep": ms / a.sweeps, "tiled_plan": plan}
    print(json.dumps(out), flush=True)
    sh.close()


if __name__ == "__main__":
    main()
