"""Debug: wall time of a tiled solve vs the summed CUDA-event time of its sweep kernels (configs[2])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1501_06350_b200 as eng
from paper_1501_06350_b200 import _lib
spec = synth.CONFIGS[2]
g = synth.generate(spec)
G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
out = torch.empty(g.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    G.solve(d=spec.d, tol=spec.tol, variant="tiled", out=out)
_lib.di_profile_enable(G.handle, True)
for it in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    _, r = G.solve(d=spec.d, tol=spec.tol, variant="tiled", out=out)
    b.record(); torch.cuda.synchronize()
    p = _lib.di_profile_get(G.handle)
    k = p.get("tile_ms", 0) + p.get("pull_ms", 0)
    print(f"solve {a.elapsed_time(b):.2f} ms, sweep kernels {k:.2f} ms (tile {p.get('tile_ms',0):.2f}, heavy {p.get('pull_ms',0):.2f}), sweeps {r['sweeps']}", flush=True)
