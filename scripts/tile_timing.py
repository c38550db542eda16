"""Debug: per-phase cycle breakdown of k_tile on configs[2] (DIT_TILE_TIMING=1).

    python scripts/tile_timing.py [rounds]

Counters are summed over CTAs (one per SM) and divided by the tiles each group
processed: round warps {wait prepared rows, wait edge bundle, local rounds,
state out}, prep warps {node loads + wait records, gathers + sums, wait for
the round warps}.
"""
import ctypes, os, sys
os.environ["DIT_TILE_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1501_06350_b200 as eng
from paper_1501_06350_b200 import _lib
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = int(os.environ.get("CONFIG", "2"))
spec = synth.CONFIGS[cfg]
g = synth.generate(spec)
G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
H, r = G.solve(d=spec.d, tol=spec.tol, variant="tiled", local_rounds=rounds,
               max_sweeps=int(os.environ.get("MAX_SWEEPS", "0")))
out = (ctypes.c_double * 48)()
_lib._lib.di_debug_tile_timing(out)
v = list(out)
it = max(v[7], 1.0)
print("rounds", rounds, "sweeps", r["sweeps"], "tile iterations", v[7])
names = ["RW wait prepared rows", "RW wait edge bundle", "RW local rounds", "RW state out",
         "PW node loads + wait recs", "PW gathers + sums", "PW wait round warps"]
for k, name in enumerate(names):
    print(f"{name:28s} {v[k]/it:10.0f} cycles/tile")
print(f"{'RW local sums (per warp)':28s} {v[8]/it/16:10.0f} cycles/tile")
print(f"{'RW wait after sums (per warp)':28s} {v[9]/it/16:10.0f} cycles/tile")
print(f"{'RW node sums (per warp)':28s} {v[14]/it/16:10.0f} cycles/tile")
print(f"{'RW gq write + barrier (per warp)':28s} {v[15]/it/16:10.0f} cycles/tile")
print(f"rounds of fully staged tiles {v[10]/max(v[11],1):10.0f} cycles/tile over {v[11]:.0f} tiles")
print(f"rounds of partly staged tiles {v[12]/max(v[13],1):9.0f} cycles/tile over {v[13]:.0f} tiles")
for k, name in ((35, "PW gathers (thread 0)"), (36, "PW wait other prep warps"), (32, "RW state out: barrier"), (33, "RW state out: issue"), (34, "RW state out: stores")):
    print(f"{name:28s} {v[k]/it:10.0f} cycles/tile")
print("per round warp: local-sum cycles/tile")
for w in range(16):
    print(f"  warp {w:2d} {v[16+w]/it:8.0f}")
