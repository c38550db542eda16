"""Debug: how concentrated is the residual |F| over tiles after k tiled sweeps (configs[2])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_1501_06350_b200 as eng
spec = synth.CONFIGS[2]
g = synth.generate(spec)
G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
for k in (3, 8, 14, 18):
    G.solve(d=spec.d, tol=spec.tol, variant="tiled", local_rounds=4, max_sweeps=k)
    F, H, d, leak = G.state()
    f = F.abs().cpu().numpy()
    t = np.add.reduceat(f, np.arange(0, g.n, 512))
    s = np.sort(t)[::-1]
    c = np.cumsum(s) / s.sum()
    print(f"sweeps {k}: |F|_1 {f.sum():.3e}; tiles for 50/90/99% of it: " +
          " ".join(f"{np.searchsorted(c, q) / len(t):.3f}" for q in (0.5, 0.9, 0.99)), flush=True)
