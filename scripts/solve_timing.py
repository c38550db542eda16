"""Debug: time fixed-sweep tiled solves on configs[2] (env knobs select diagnostic paths)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1501_06350_b200 as eng
spec = synth.CONFIGS[2]
g = synth.generate(spec)
G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
sw = int(os.environ.get("MAX_SWEEPS", "21"))
for it in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    H, r = G.solve(d=spec.d, tol=spec.tol, variant="tiled", local_rounds=int(os.environ.get("ROUNDS", "4")), max_sweeps=sw)
    b.record(); torch.cuda.synchronize()
    if it: print(os.environ.get("TAG", ""), "sweeps", r["sweeps"], "ms", round(a.elapsed_time(b), 2))
