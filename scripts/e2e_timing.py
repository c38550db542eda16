"""Debug: the bench's e2e step (C ABI, pinned host buffers) with build phase marks."""
import os, sys, time
os.environ["DIT_BUILD_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1501_06350_b200 as eng
from paper_1501_06350_b200 import _lib
spec = synth.CONFIGS[2]
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
g = synth.generate(spec)
rp, col, w = pin(g.row_ptr), pin(g.col), pin(g.w)
Hh = pin(np.empty(g.n))
stream = torch.cuda.current_stream()
for it in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = _lib.di_graph_create(g.n, rp, col, w, device=0, stream=stream)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = _lib.di_solve(h, spec.d, None, spec.tol, Hh, variant=eng.VARIANTS["tiled"], local_rounds=4)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    _lib.di_graph_destroy(h)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):.0f} ms, solve(+build+D2H) {1e3*(t2-t1):.0f} ms, destroy {1e3*(t3-t2):.0f} ms", flush=True)
