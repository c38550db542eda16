"""Experiment: configs[2] with host blocks of 100 (BASELINE) vs 128 ids (tiles of 512 hold whole
blocks): how much of the tiled solve's time comes from blocks cut by tile boundaries."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1501_06350_b200 as eng
from paper_1501_06350_b200 import _lib
for block in (100, 128):
    spec = synth.CONFIGS[2].scaled(synth.CONFIGS[2].n, block=block)
    g = synth.generate(spec)
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    out = torch.empty(g.n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        G.solve(d=spec.d, tol=spec.tol, variant="tiled", out=out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    _, r = G.solve(d=spec.d, tol=spec.tol, variant="tiled", out=out)
    b.record(); torch.cuda.synchronize()
    st = _lib.di_plan_stats(G.handle)
    print(f"block {block}: {a.elapsed_time(b):.1f} ms, {r['sweeps']} sweeps, local {st['local_edges']:.3e} light {st['light_edges']:.3e} heavy {st['heavy_edges']:.3e}", flush=True)
    G.close()
    del g
