#!/usr/bin/env python
"""Benchmark: D-Iteration solves on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one cold solve to |F|_1 <= tol (every sweep of the hot path: frontier
select, diffusion push/pull, residual reduction) on the synthetic graph of
BASELINE.json configs[C] (default 2: n = 50M, ~1B weighted edges, tol 1e-9),
already resident in HBM.  value = diffused edges / s; time_to_tol_s = seconds
per solve.  e2e = the same metric through the C ABI from pinned HOST buffers
(graph upload + build + solve + H download inside the timed region).
`--impl reference` times the CPU oracle (oracle/, the reference arm of this
tier) on the same workload, a bounded number of sweeps per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "diffused edges/s & time to |F|_1<=tol, fraction of HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=2)
    p.add_argument("--variant", default="tiled", choices=["auto", "push", "pull", "tiled"])
    p.add_argument("--rounds", type=int, default=4, help="local rounds per sweep (variant tiled)")
    p.add_argument("--theta", type=float, default=1.0)
    p.add_argument("--tol", type=float, default=None)
    p.add_argument("--e2e-steps", type=int, default=4)
    p.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    p.add_argument("--scale-n", type=int, default=None, help="override n (debug only)")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, nm in enumerate(names):
                    if r[5 + k].strip().lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def spec_for(args):
    spec = synth.CONFIGS[args.config]
    if args.scale_n:
        spec = spec.scaled(args.scale_n)
    return spec


def workload_name(spec, cfg):
    return f"{spec.name} (BASELINE configs[{cfg}])"


# ------------------------------------------------------------------ CPU oracle
TILE_NODES = 512   # include/dit.h DI_TILE_NODES (the oracle takes the tile as a parameter)
TILE_WAVES = 3     # include/dit.h DI_TILE_WAVES


def oracle_run(args, spec, cols, n, sweeps):
    """The CPU oracle (oracle/, test infrastructure) timed as it stands: `sweeps`
    sweeps of the same schedule as the GPU arm (tiled: orc_tiled_sweep_run with
    the same tile and rounds; else the theta frontier sweep) from the cold start
    F_0 = (1-d)Z, single-threaded C.  Returns (diffused edges, seconds)."""
    from oracle import di as odi
    cp, ri, pv = cols
    F = np.full(n, (1 - spec.d) / n)
    H = np.zeros(n)
    t0 = time.perf_counter()
    if args.variant == "tiled":
        r = odi.tiled_sweep_run(n, cp, ri, pv, spec.d, F, H, tile=TILE_NODES, rounds=args.rounds, tol=0.0,
                                max_sweeps=sweeps, waves=TILE_WAVES)
    else:
        r = odi.sweep_run(n, cp, ri, pv, spec.d, F, H, theta=args.theta, tol=0.0, max_sweeps=sweeps)
    return r.edges, time.perf_counter() - t0


def oracle_cols(g):
    from oracle import graph as ograph
    return ograph.column_entries(g.n, g.row_ptr, g.col, g.w)


def oracle_desc(args, sweeps):
    sched = (f"tiled sweep (tile {TILE_NODES}, {args.rounds} rounds, {TILE_WAVES} waves)" if args.variant == "tiled"
             else f"theta={args.theta} frontier sweep")
    return f"first {sweeps} {sched} sweep(s) of the cold solve on the full graph, single-threaded C oracle"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    spec = spec_for(args)
    g = synth.generate(spec)
    cols = oracle_cols(g)
    sweeps = 1 if g.m > 50_000_000 else 5
    times, edges = [], []
    for it in range(args.warmup + args.steps):
        e, dt = oracle_run(args, spec, cols, g.n, sweeps)
        if it >= args.warmup:
            times.append(dt)
            edges.append(e)
    tot = sum(times)
    value = sum(edges) / tot
    sample = oracle_desc(args, sweeps) + f" per step; n={g.n} m={g.m}"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_name(spec, args.config), "n": g.n, "m": g.m,
                                            "variant": args.variant, "local_rounds": args.rounds,
                                            "theta": args.theta},
            "cpu_baseline": {"value": value, "unit": "edges/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def pinned_alloc(shape, dtype):
    import torch
    tdt = {np.int32: torch.int32, np.float32: torch.float32, np.int64: torch.int64,
           np.float64: torch.float64}[dtype]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()


def load_traffic(workload, kernel):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            tr = json.load(fh)
        return tr.get(workload, {}).get(kernel)
    except Exception:
        return None


KERNEL_NAMES = {"tiled": {"pull": "k_heavy_chunks+k_heavy_fold", "tile": "k_tile"}}


def roofline_from(prof_tot, workload, variant):
    """Roofline of the dominant kernel class (largest summed CUDA-event time):
    algorithmic bytes / event time, against the measured peak."""
    peak, peak_kind = load_peaks()
    kinds = ["select", "push", "pull", "reduce", "tile"]
    dom = max(kinds, key=lambda k: prof_tot.get(f"{k}_ms", 0.0))
    dom_ms = prof_tot[f"{dom}_ms"]
    dom_launch = max(1, prof_tot[f"{dom}_launches"])
    achieved = prof_tot[f"{dom}_bytes"] / (dom_ms / 1e3) / 1e9
    tot_ms = max(1e-9, sum(prof_tot.get(f"{q}_ms", 0.0) for q in kinds))
    names = KERNEL_NAMES.get(variant, {})
    share = {names.get(k, f"k_{k}"): prof_tot.get(f"{k}_ms", 0.0) / tot_ms for k in kinds}
    name = names.get(dom, f"k_{dom}")
    return {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "peak_source": peak_kind,
            "traffic": load_traffic(workload, name), "algorithmic_bytes_per_launch": prof_tot[f"{dom}_bytes"] / dom_launch,
            "avg_launch_ms": dom_ms / dom_launch, "share_of_step": share,
            "sweep_bytes_per_s_all_kernels": sum(prof_tot.get(f"{k}_bytes", 0) for k in kinds) / (tot_ms / 1e3) / 1e9}


def cpu_baseline(args, gpu_edges_per_solve=None, g=None):
    """The CPU oracle (oracle/, test infrastructure) timed as it stands on this
    host: a bounded sample of the bench workload (configs[args.config] at its
    single-GPU size), the same schedule as the GPU arm, one core."""
    spec = spec_for(args)
    if g is None:
        g = synth.generate(spec)
    sw = 1 if g.m > 50_000_000 else 5
    ce, cdt = oracle_run(args, spec, oracle_cols(g), g.n, sw)
    out = {"value": ce / cdt, "unit": "edges/s", "cores": 1, "kind": "oracle",
           "sample": oracle_desc(args, sw) + f" ({ce} diffused edges, {cdt:.1f} s)"}
    if gpu_edges_per_solve:
        # the oracle runs the GPU's schedule: a solve diffuses the same edges at its measured rate
        out["time_to_tol_s"] = gpu_edges_per_solve / out["value"]
        out["time_to_tol_kind"] = "estimate: the GPU solve's diffused edges / the oracle's measured edges/s"
    return out


def relaunch_distributed(args):
    """`bench.py --gpus N` started without torchrun: re-execute under
    torch.distributed.run, one rank per GPU (RANK / LOCAL_RANK / WORLD_SIZE from
    the launcher, rendezvous on 127.0.0.1); rank 0's JSON line passes through."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but {have} visible CUDA device(s)",
                          "n_gpus": args.gpus}), flush=True)
        return 1
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the communicator's rank count shows in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_update(args):
    """--config 4: BASELINE configs[4], the dynamic update.  A step = di_update_edges
    (1% of the configs[2] graph rewired: Theorem 4 corrective fluid + CSR rebuild on
    the device) + the warm di_resume to tol, on a graph solved to tol beforehand
    (untimed).  Beside it, the cold alternative: plan build (transpose + tile
    plan) + cold solve of the modified graph (its CSR made by the same
    di_update_edges on a fresh handle, untimed)."""
    import torch
    import paper_1501_06350_b200 as eng
    from paper_1501_06350_b200 import _lib
    torch.cuda.set_device(0)
    spec = synth.CONFIGS[4]
    tol = args.tol if args.tol is not None else spec.tol
    g = synth.generate(spec)
    delta = synth.rewire(spec, g, fraction=0.01, seed=4)
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    rp, cl, wv = t(g.row_ptr), t(g.col), t(g.w)
    dd = {k: (t(v) if v is not None else None) for k, v in delta.items()}
    kw = dict(d=spec.d, tol=tol, variant=args.variant, local_rounds=args.rounds)
    stream = torch.cuda.current_stream()
    out = torch.empty(g.n, dtype=torch.float64, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    upd_ms, res_ms, cold_ms, edges, sweeps, cold_sweeps, prof_tot = [], [], [], 0, [], [], {}
    with ClockSampler(0) as clk:
        for it in range(args.warmup + args.steps):
            G = eng.DIGraph(g.n, rp, cl, wv, stream=stream)
            G.solve(out=out, **kw)
            torch.cuda.synchronize()
            a, b, c = ev(), ev(), ev()
            a.record(stream)
            G.update_edges(**dd)
            b.record(stream)
            if it >= args.warmup:
                _lib.di_profile_enable(G.handle, True)
            _, r = G.resume(out=out, tol=tol, variant=args.variant, local_rounds=args.rounds)
            c.record(stream)
            torch.cuda.synchronize()
            assert r["converged"], r
            if it >= args.warmup:
                for k, v in _lib.di_profile_get(G.handle).items():
                    prof_tot[k] = prof_tot.get(k, 0) + v
                upd_ms.append(a.elapsed_time(b))
                res_ms.append(b.elapsed_time(c))
                edges += r["diffused_edges"]
                sweeps.append(r["sweeps"])
            G.close()
            # the cold alternative: plan build + cold solve of the modified graph from F_0
            G2 = eng.DIGraph(g.n, rp, cl, wv, stream=stream)
            G2.update_edges(**dd)
            a, b = ev(), ev()
            torch.cuda.synchronize()
            a.record(stream)
            _, rc = G2.solve(out=out, **kw)
            b.record(stream)
            torch.cuda.synchronize()
            G2.close()
            if it >= args.warmup:
                cold_ms.append(a.elapsed_time(b))
                cold_sweeps.append(rc["sweeps"])
    total = sum(upd_ms) + sum(res_ms)
    line = {"metric": METRIC, "value": edges / (total / 1e3), "unit": "edges/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total / args.steps, "time_to_tol_s": total / args.steps / 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{spec.name} (BASELINE configs[4]): update 1% of the edges + warm resume",
                       "n": g.n, "m": g.m, "edges_added": int(len(delta["add_src"])),
                       "edge_pairs_removed": int(len(delta["rem_src"])), "tol": tol, "variant": args.variant,
                       "local_rounds": args.rounds, "update_ms": statistics.mean(upd_ms),
                       "resume_ms": statistics.mean(res_ms), "resume_sweeps": sweeps[-1],
                       "cold_build_and_solve_ms": statistics.mean(cold_ms), "cold_sweeps": cold_sweeps[-1],
                       "l2": "inputs larger than L2; no flush"},
            "roofline": roofline_from(prof_tot, spec.name, args.variant) if prof_tot else None,
            "cpu_baseline": None, "e2e": None, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_1501_06350_b200 as eng
    from paper_1501_06350_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.config == 4:
        return run_update(args)
    if args.gpus > 1 and world == 0:
        return relaunch_distributed(args)
    if world > 1 or args.gpus > 1:
        from paper_1501_06350_b200 import dist
        return dist.bench_sharded(args, METRIC, {"clock": ClockSampler, "roofline": roofline_from,
                                                 "pinned": pinned_alloc, "cpu_baseline": cpu_baseline})
    torch.cuda.set_device(0)
    spec = spec_for(args)
    tol = args.tol if args.tol is not None else spec.tol
    t0 = time.perf_counter()
    g = synth.generate(spec, pinned_alloc=pinned_alloc)
    gen_s = time.perf_counter() - t0
    row_ptr = pinned_alloc((g.n + 1,), np.int64)
    row_ptr[:] = g.row_ptr
    stream = torch.cuda.current_stream()
    G = eng.DIGraph(g.n, row_ptr, g.col, g.w, stream=stream)
    kw = dict(d=spec.d, tol=tol, theta=args.theta, variant=args.variant, local_rounds=args.rounds)
    out = torch.empty(g.n, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        G.solve(out=out, **kw)
    torch.cuda.synchronize()
    _lib.di_profile_enable(G.handle, True)
    prof_tot = {}
    edges_tot = 0
    sweeps = []
    l0 = eng.di_kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        results = []
        for _ in range(args.steps):
            _, res = G.solve(out=out, **kw)
            results.append(res)
            p = _lib.di_profile_get(G.handle)
            for k, v in p.items():
                prof_tot[k] = prof_tot.get(k, 0) + v
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = eng.di_kernel_launches() - l0
    _lib.di_profile_enable(G.handle, False)
    total_ms = ev0.elapsed_time(ev1)
    for r in results:
        edges_tot += r["diffused_edges"]
        sweeps.append(r["sweeps"])
    value = edges_tot / (total_ms / 1e3)
    res = results[-1]
    assert res["converged"], res
    roofline = roofline_from(prof_tot, spec.name, args.variant)
    tiled_plan = _lib.di_plan_stats(G.handle) if args.variant == "tiled" else None
    G.close()                                      # the e2e graphs below reuse its pooled memory
    torch.cuda.synchronize()
    # e2e through the C ABI with host buffers
    e2e = None
    if args.e2e_steps > 0:
        Hh = pinned_alloc((g.n,), np.float64)
        h2d = row_ptr.nbytes + g.col.nbytes + (g.w.nbytes if g.w is not None else 0)
        e_edges, e_ms = 0, 0.0
        for it in range(args.e2e_steps + 1):       # the first (untimed) step warms the memory pool
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            h = _lib.di_graph_create(g.n, row_ptr, g.col, g.w, device=0, stream=stream)
            r = _lib.di_solve(h, spec.d, None, tol, Hh, theta=args.theta,
                              variant=eng.VARIANTS[args.variant], local_rounds=args.rounds)
            b.record(stream)
            torch.cuda.synchronize()
            _lib.di_graph_destroy(h)
            print(f"[bench] e2e step {it}: {a.elapsed_time(b):.1f} ms" + (" (untimed)" if it == 0 else ""),
                  file=sys.stderr, flush=True)
            if it == 0:
                continue
            e_ms += a.elapsed_time(b)
            e_edges += r.diffused_edges
        e2e = {"value": e_edges / (e_ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(Hh.nbytes), "ms_per_step": e_ms / args.e2e_steps}
    # CPU oracle baseline (bounded sample)
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline(args, results[-1]["diffused_edges"], g)
    clocks = clk.summary()
    line = {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "time_to_tol_s": total_ms / args.steps / 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(spec, args.config), "n": g.n, "m": g.m, "d": spec.d, "tol": tol,
                       "theta": args.theta, "variant": args.variant, "local_rounds": args.rounds,
                       "weighted": spec.weighted,
                       "sweeps_per_solve": sweeps[-1], "diffused_edges_per_solve": results[-1]["diffused_edges"],
                       "push_sweeps": res["push_sweeps"], "pull_sweeps": res["pull_sweeps"],
                       "l2": "inputs larger than L2 (F 8n B, CSR ~8m B >> 126 MB); no flush",
                       "generate_s": round(gen_s, 2),
                       "tiled_plan": tiled_plan},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks}
    print(json.dumps(line), flush=True)
    G.close()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
