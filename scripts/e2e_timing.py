"""Debug: the bench's e2e step (C ABI, pinned host buffers): host time of create /
solve / destroy per step, with DIT_E2E_MARKS=1 the build's host-side phase
times (no extra synchronisation: time from the create's start to each mark)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1501_06350_b200 as eng
from paper_1501_06350_b200 import _lib
spec = synth.CONFIGS[2]
g = synth.generate(spec, pinned_alloc=lambda shape, dt: torch.empty(shape, dtype={np.int32: torch.int32, np.float32: torch.float32, np.int64: torch.int64, np.float64: torch.float64}[dt], pin_memory=True).numpy())
rp = torch.from_numpy(g.row_ptr).pin_memory().numpy()
Hh = torch.empty(g.n, dtype=torch.float64, pin_memory=True).numpy()
stream = torch.cuda.current_stream()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for it in range(steps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = _lib.di_graph_create(g.n, rp, g.col, g.w, device=0, stream=stream)
    t1 = time.perf_counter()
    r = _lib.di_solve(h, spec.d, None, spec.tol, Hh, variant=eng.VARIANTS["tiled"], local_rounds=4)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    _lib.di_graph_destroy(h)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms, destroy {1e3*(t3-t2):.1f} ms", flush=True)
