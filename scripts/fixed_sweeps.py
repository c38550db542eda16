"""Debug: device time per sweep of the tiled kernels over a FIXED number of sweeps
(tol 0), for kernel ablations whose arithmetic no longer converges.

    python scripts/fixed_sweeps.py [sweeps]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1501_06350_b200 as eng
from paper_1501_06350_b200 import _lib
sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
spec = synth.CONFIGS[2]
g = synth.generate(spec)
dev = torch.device("cuda", 0)
G = eng.DIGraph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
G.solve(d=spec.d, tol=0.0, variant="tiled", local_rounds=4, max_sweeps=2)
_lib.di_profile_enable(G.handle, True)
for it in range(3):
    G.solve(d=spec.d, tol=0.0, variant="tiled", local_rounds=4, max_sweeps=sweeps)
    p = _lib.di_profile_get(G.handle)
    print(f"k_tile {p['tile_ms'] / p['sweeps']:.3f} ms/sweep, heavy {p['pull_ms'] / p['sweeps']:.3f} ms/sweep", flush=True)
G.close()
