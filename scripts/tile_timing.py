"""Debug: per-phase cycle breakdown of k_tile on configs[2] (DIT_TILE_TIMING=1)."""
import ctypes, os, sys, time
os.environ["DIT_TILE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1501_06350_b200 as eng
from paper_1501_06350_b200 import _lib
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
spec = synth.CONFIGS[2]
g = synth.generate(spec)
G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
H, r = G.solve(d=spec.d, tol=spec.tol, variant="tiled", local_rounds=rounds, max_sweeps=int(os.environ.get("MAX_SWEEPS", "0")))
out = (ctypes.c_double * 5)()
_lib._lib.di_debug_tile_timing(out)
v = list(out)
tot = sum(v[:4])
print("rounds", rounds, "sweeps", r["sweeps"], "iterations", v[4])
for k, name in enumerate(["wait bundle", "remote inflow", "local rounds", "state out"]):
    print(f"{name:14s} {v[k]/v[4]:10.0f} cycles/tile  {100*v[k]/tot:5.1f}%")
