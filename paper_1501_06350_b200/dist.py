"""Multi-GPU D-Iteration: one process per GPU, contiguous node ranges.

Rank r owns nodes [lo_r, hi_r) = [r n / R, (r+1) n / R) and their out-edges.
Every sweep of every rank runs in libdit (di_shard_sweep: frontier select +
diffusion, fluid for other ranks accumulating in ghost slots); between sweeps
the ranks exchange ghost fluid with one NCCL all-to-all over NVLink and
all-reduce the residual (sum) and the max fluid (max) that set the next
frontier threshold and the stop test.  This module only sequences those calls
(argument marshalling and collectives); it does no arithmetic of the method.

The protocol is written against a `collectives` object so that the same code
drives torch.distributed (NCCL on GPUs, gloo in the CPU tests) and, in the
tests, several shards of one process on one GPU run in lock step.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib


def node_ranges(n, world):
    """Contiguous, balanced node ranges: bounds[r] .. bounds[r+1]."""
    return [n * r // world for r in range(world + 1)]


class CudaShard:
    """One rank's libdit shard handle plus its device exchange buffers."""

    def __init__(self, n_global, lo, hi, row_ptr, col, weights=None, device=0, stream=None):
        self.n_global, self.lo, self.hi = int(n_global), int(lo), int(hi)
        self.dev = torch.device("cuda", device)
        self.h = _lib.di_shard_create(n_global, lo, hi, row_ptr, col, weights, device=device, stream=stream)
        self.n_local, self.n_ghost, _ = _lib.di_shard_info(self.h)
        self.ghost_ids = torch.empty(self.n_ghost, dtype=torch.int32, device=self.dev)
        if self.n_ghost:
            _lib.di_shard_ghost_ids(self.h, self.ghost_ids)
        self.send = torch.zeros(max(self.n_ghost, 1), dtype=torch.float64, device=self.dev)
        self.stats = torch.zeros(4, dtype=torch.float64, device=self.dev)
        self.gathered = torch.zeros(4, dtype=torch.float64, device=self.dev)   # [world][4], sized by the plan
        self.world = 1
        self.recv = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.send_counts = None
        self.recv_counts = None

    # --- exchange plan
    def set_recv(self, local_idx, seg_counts):
        self.world = len(seg_counts)
        self.gathered = torch.zeros(4 * self.world, dtype=torch.float64, device=self.dev)
        _lib.di_shard_set_recv(self.h, local_idx, seg_counts)
        self.recv = torch.zeros(max(int(sum(seg_counts)), 1), dtype=torch.float64, device=self.dev)
        self.recv_counts = [int(c) for c in seg_counts]

    # --- protocol steps (asynchronous on the shard's stream)
    def begin(self, d, tol, **opts):
        _lib.di_shard_begin(self.h, d, None, tol, self.stats, **opts)

    def control(self):
        _lib.di_shard_control(self.h, self.gathered, self.world)

    def global_residual(self):
        """sum over ranks of |F|_1 from the last gathered stats (host read, for chunk sizing)"""
        return float(self.gathered.view(self.world, 4)[:, 0].sum().item())

    def sweep(self):
        _lib.di_shard_sweep(self.h, self.send)

    def heavy_local(self):
        _lib.di_shard_heavy_local(self.h)

    def apply(self):
        _lib.di_shard_apply(self.h, self.recv)

    def reduce(self):
        _lib.di_shard_reduce(self.h)

    def flush(self):
        _lib.di_shard_flush(self.h, self.send)

    def flush_apply(self):
        _lib.di_shard_flush_apply(self.h, self.recv)

    def poll(self):
        return _lib.di_shard_poll(self.h)

    def finish(self, tol, out=None, **opts):
        if out is None:
            out = torch.empty(self.n_local, dtype=torch.float64, device=self.dev)
        res = _lib.di_shard_finish(self.h, tol, out, **opts)
        return out, res.as_dict()

    def close(self):
        if self.h:
            _lib.di_graph_destroy(self.h)
            self.h = None


class TorchCollectives:
    """torch.distributed collectives for a single local shard (NCCL or gloo).

    stage_host=True moves every buffer through host memory around the
    collective (gloo with CUDA shards: the tests run real libdit shards of
    several processes on one GPU that way; no kernel waits on another rank)."""

    def __init__(self, group=None, stage_host=False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.stage = stage_host

    def _c(self, t):
        return t.cpu() if self.stage else t

    def plan(self, shards, bounds):
        (s,) = shards
        ids = s.ghost_ids.cpu().numpy().astype(np.int64)
        owner = np.searchsorted(np.asarray(bounds), ids, side="right") - 1
        send_counts = np.bincount(owner, minlength=self.world).astype(np.int64)
        dev = s.send.device
        cdev = torch.device("cpu") if self.stage else dev
        sc = torch.tensor(send_counts, dtype=torch.int64, device=cdev)
        rc = torch.empty_like(sc)
        self.dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = rc.cpu().numpy()
        recv_ids = torch.empty(int(recv_counts.sum()), dtype=torch.int32, device=cdev)
        self.dist.all_to_all_single(recv_ids, s.ghost_ids.to(cdev), output_split_sizes=recv_counts.tolist(),
                                    input_split_sizes=send_counts.tolist(), group=self.group)
        recv_ids = recv_ids.to(dev)
        s.send_counts = send_counts.tolist()
        s.set_recv((recv_ids - s.lo).to(torch.int32), recv_counts.tolist())

    def allreduce_stats(self, shards):
        # one collective per sweep: every rank's {|F|_1, max|F|, leak, edges}, reduced on
        # the device in rank order by di_shard_control (deterministic, identical on all ranks)
        (s,) = shards
        if self.stage:
            out = torch.empty(s.gathered.shape, dtype=s.gathered.dtype)
            self.dist.all_gather_into_tensor(out, s.stats.cpu(), group=self.group)
            s.gathered.copy_(out)
        else:
            self.dist.all_gather_into_tensor(s.gathered, s.stats, group=self.group)

    def alltoall(self, shards):
        (s,) = shards
        if self.world == 1:
            return
        if self.stage:
            out = torch.empty(sum(s.recv_counts), dtype=s.recv.dtype)
            self.dist.all_to_all_single(out, s.send[:sum(s.send_counts)].cpu(), output_split_sizes=s.recv_counts,
                                        input_split_sizes=s.send_counts, group=self.group)
            s.recv[:sum(s.recv_counts)].copy_(out)
            return
        self.dist.all_to_all_single(s.recv[:sum(s.recv_counts)], s.send[:sum(s.send_counts)],
                                    output_split_sizes=s.recv_counts, input_split_sizes=s.send_counts,
                                    group=self.group)

    def alltoall_start(self, shards):
        """Start the ghost exchange; its wait is alltoall_finish.  NCCL: asynchronous,
        so the rank's own wave-0 heavy gather (enqueued after this call) runs while the
        exchange moves over NVLink; the wait orders the stream before di_shard_apply."""
        (s,) = shards
        if self.world == 1 or self.stage:
            self.alltoall(shards)
            return None
        return self.dist.all_to_all_single(s.recv[:sum(s.recv_counts)], s.send[:sum(s.send_counts)],
                                           output_split_sizes=s.recv_counts, input_split_sizes=s.send_counts,
                                           group=self.group, async_op=True)

    def alltoall_finish(self, work):
        if work is not None:
            work.wait()

    def allreduce_sum(self, values, device):
        t = torch.tensor(values, dtype=torch.float64, device="cpu" if self.stage else device)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().tolist()

    def allreduce_max(self, values, device):
        t = torch.tensor(values, dtype=torch.float64, device="cpu" if self.stage else device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t.cpu().tolist()


def solve(shards, coll, d=0.85, tol=1e-12, max_chunk=64, **opts):
    """Cold sharded solve; returns (list of local H tensors, list of local result dicts).

    Per sweep: sweep (ghost sums) -> all-to-all(ghost fluid), overlapped with
    heavy_local (the rank's own wave-0 heavy gather) -> apply -> reduce -> all-gather
    of the ranks' {|F|_1, max |F|, leak} -> control (reduced on the device).  The host polls `done` once per chunk.
    The tiled schedule (variant 3) leaves the last sweep's remote pushes
    pending (R13): once done, they are exchanged and applied like a
    sweep (flush -> all-to-all -> flush_apply -> all-reduce -> control), and
    the sweeps go on if the exact residual is still above tol."""
    start = getattr(coll, "alltoall_start", None) or (lambda sh: coll.alltoall(sh))
    finish = getattr(coll, "alltoall_finish", None) or (lambda w: None)
    for s in shards:
        s.begin(d, tol, **opts)
    coll.allreduce_stats(shards)
    for s in shards:
        s.control()
    chunk = 2
    r_prev, s_prev, swept = None, 0, 0
    while True:
        swept += chunk
        for _ in range(chunk):
            for s in shards:
                s.sweep()
            # the exchange overlaps each rank's own wave-0 heavy gather (tiled)
            work = start(shards)
            for s in shards:
                s.heavy_local()
            finish(work)
            for s in shards:
                s.apply()
                s.reduce()
            coll.allreduce_stats(shards)
            for s in shards:
                s.control()
        done = [s.poll() for s in shards]
        if all(done) and opts.get("variant") == _lib.DI_VARIANT_TILED:
            for s in shards:
                s.flush()
            coll.alltoall(shards)
            for s in shards:
                s.flush_apply()
            coll.allreduce_stats(shards)
            for s in shards:
                s.control()
            done = [s.poll() for s in shards]
        if all(done):
            break
        if any(done):
            raise RuntimeError("ranks disagree on convergence")
        # next chunk from the decay of the global residual (identical on every rank,
        # so the ranks stay in lock step): the sweeps still needed to reach tol
        r = shards[0].global_residual()
        nxt = min(chunk * 2, max_chunk)
        if r_prev is not None and 0.0 < r < r_prev and tol > 0.0:
            rate = (r / r_prev) ** (1.0 / (swept - s_prev))
            need = math.log(tol / r) / math.log(rate)
            if math.isfinite(need):
                nxt = int(min(max_chunk, max(1, math.ceil(need - 1e-3))))
        r_prev, s_prev, chunk = r, swept, nxt
    outs = [s.finish(tol, **opts) for s in shards]
    return [o[0] for o in outs], [o[1] for o in outs]


# ------------------------------------------------------------------ bench (torchrun)
def bench_spec(world, config, scale_n=None):
    """The sharded bench's workload: BASELINE configs[3] (400M nodes, ~8B weighted
    edges, int64 row offsets) over 8 GPUs; at 2 / 4 GPUs the same generator on
    world x 50M nodes (weak-scaling slices: 50M nodes, ~1B edges per GPU, the
    shape of one configs[3] rank).  Returns (spec, workload name)."""
    import synth
    base = synth.CONFIGS[3] if config in (2, 3) else synth.CONFIGS[config]
    per = scale_n or synth.CONFIGS[2].n
    if config in (2, 3) and scale_n is None and world * per == base.n:
        return base, f"{base.name} (BASELINE configs[3]) over {world} GPUs"
    spec = base.scaled(per * world)
    return spec, f"{base.name} generator, {world} x {per} nodes (weak-scaling slice of configs[3])"


def bench_sharded(args, metric, tools):
    """bench.py --gpus N under torchrun (bench.py re-executes itself under
    torch.distributed.run when started without it): weak scaling, each rank owns
    a contiguous 50M-node range with its ~1B out-edges (bench_spec).  `tools`
    carries bench.py's clock sampler, roofline arithmetic, pinned allocator and
    CPU-oracle timer (measurement plumbing only)."""
    import json
    import os

    import torch.distributed as dist

    import synth
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec, workload = bench_spec(world, args.config, args.scale_n)
    tol = args.tol if args.tol is not None else spec.tol
    bounds = node_ranges(spec.n, world)
    lo, hi = bounds[rank], bounds[rank + 1]
    g = synth.generate(spec, lo, hi)
    stream = torch.cuda.current_stream()
    sh = CudaShard(spec.n, lo, hi, g.row_ptr, g.col, g.w, device=local, stream=stream)
    coll = TorchCollectives()
    coll.plan([sh], bounds)
    variant = args.variant
    kw = dict(theta=args.theta, variant={"auto": 0, "push": 1, "pull": 2, "tiled": 3}[variant],
              local_rounds=args.rounds)
    for _ in range(args.warmup):
        solve([sh], coll, d=spec.d, tol=tol, **kw)
    torch.cuda.synchronize()
    dist.barrier()
    _lib.di_profile_enable(sh.h, True)
    prof_tot = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = _lib.di_kernel_launches()
    with tools["clock"](local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        res = []
        for _ in range(args.steps):
            _, r = solve([sh], coll, d=spec.d, tol=tol, **kw)
            res.append(r[0])
            for k, v in _lib.di_profile_get(sh.h).items():
                prof_tot[k] = prof_tot.get(k, 0) + v
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    _lib.di_profile_enable(sh.h, False)
    ms = e0.elapsed_time(e1)
    launches = _lib.di_kernel_launches() - l0
    ms_max = coll.allreduce_max([ms], stream.device)[0]
    edges = coll.allreduce_sum([float(sum(r["diffused_edges"] for r in res))], stream.device)[0]
    cross = coll.allreduce_sum([float(sh.n_ghost), float(g.m)], stream.device)
    plan = _lib.di_plan_stats(sh.h) if variant == "tiled" else None
    sh.close()                                 # the e2e shards below reuse its pooled memory
    torch.cuda.synchronize()
    # e2e: every rank builds its shard from pinned host buffers, solves and reads H back
    e2e = None
    if args.e2e_steps > 0:
        pin = tools["pinned"]
        rp = pin((len(g.row_ptr),), np.int64)
        rp[:] = g.row_ptr
        cl = pin((len(g.col),), np.int32)
        cl[:] = g.col
        wv = None
        if g.w is not None:
            wv = pin((len(g.w),), np.float32)
            wv[:] = g.w
        Hh = torch.from_numpy(pin((hi - lo,), np.float64))
        e_ms, e_edges = 0.0, 0.0
        for it in range(args.e2e_steps + 1):   # the first (untimed) step warms the memory pool
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            dist.barrier()
            a.record(stream)
            s2 = CudaShard(spec.n, lo, hi, rp, cl, wv, device=local, stream=stream)
            coll.plan([s2], bounds)
            Hd, r2 = solve([s2], coll, d=spec.d, tol=tol, **kw)
            Hh.copy_(Hd[0], non_blocking=True)
            b.record(stream)
            torch.cuda.synchronize()
            ms2 = coll.allreduce_max([a.elapsed_time(b)], stream.device)[0]
            ed2 = coll.allreduce_sum([float(r2[0]["diffused_edges"])], stream.device)[0]
            s2.close()
            if it == 0:
                continue
            e_ms += ms2
            e_edges += ed2
        h2d = coll.allreduce_sum([float(rp.nbytes + cl.nbytes + (wv.nbytes if wv is not None else 0))],
                                 stream.device)[0]
        e2e = {"value": e_edges / (e_ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(spec.n * 8), "ms_per_step": e_ms / args.e2e_steps}
    dist.barrier()
    if rank == 0:
        cpu = None if args.no_cpu else tools["cpu_baseline"](args)
        line = {"metric": metric, "value": edges / (ms_max / 1e3), "unit": "edges/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "time_to_tol_s": ms_max / args.steps / 1e3, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload, "n": spec.n, "m": int(cross[1]), "tol": tol, "theta": args.theta,
                           "variant": variant, "local_rounds": args.rounds, "ghost_slots_total": int(cross[0]),
                           "exchange_bytes_per_sweep": int(cross[0]) * 8,
                           "sweeps_per_solve": res[-1]["sweeps"], "rank0_plan": plan,
                           "l2": "inputs larger than L2 (F 8n B, CSR ~8m B >> 126 MB); no flush",
                           "parallelism": f"node-range partition x{world}, NCCL all-to-all + all-gather"},
                "roofline": tools["roofline"](prof_tot, spec.name, variant), "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0
