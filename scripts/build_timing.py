"""Debug: phase times of graph create + tiled plan build + solve on configs[2] (DIT_BUILD_TIMING=1)."""
import os, sys, time
os.environ["DIT_BUILD_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1501_06350_b200 as eng
spec = synth.CONFIGS[2]
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
g = synth.generate(spec)
rp, col, w = pin(g.row_ptr), pin(g.col), pin(g.w)
for it in range(2):
    t0 = time.perf_counter()
    G = eng.DIGraph(g.n, rp, col, w)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    H, r = G.solve(d=spec.d, tol=spec.tol, variant="tiled")
    torch.cuda.synchronize(); t2 = time.perf_counter()
    Hh = H.cpu(); t3 = time.perf_counter()
    G.close(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):.0f} ms, build+solve {1e3*(t2-t1):.0f} ms, D2H {1e3*(t3-t2):.0f} ms, destroy {1e3*(t4-t3):.0f} ms", flush=True)
