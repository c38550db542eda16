"""configs[4]: time of di_update_edges + warm resume vs a cold solve of the modified graph (tiled)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1501_06350_b200 as eng
from oracle import graph
spec = synth.CONFIGS[4]
g = synth.generate(spec)
delta = synth.rewire(spec, g, fraction=0.01, seed=4)
G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
G.solve(d=spec.d, tol=spec.tol, variant="tiled")
ev = lambda: torch.cuda.Event(enable_timing=True)
a, b, c = ev(), ev(), ev()
torch.cuda.synchronize(); a.record()
G.update_edges(**delta)
b.record()
H, r = G.resume(tol=spec.tol, variant="tiled")
c.record(); torch.cuda.synchronize()
print(f"update {a.elapsed_time(b):.1f} ms, resume {b.elapsed_time(c):.1f} ms ({r['sweeps']} sweeps, {r['diffused_edges']:.3e} edges)")
# the resume again on the already updated graph state (plan built): sweeps only
F, Hs, d, leak = G.state()
rp2, c2, w2, _ = graph.apply_delta(g.n, g.row_ptr, g.col, g.w, delta["add_src"], delta["add_dst"], delta["add_w"],
                                   delta["rem_src"], delta["rem_dst"])
G2 = eng.DIGraph(g.n, rp2, c2, w2)
t0 = ev(); t1 = ev()
G2.solve(d=spec.d, tol=spec.tol, variant="tiled")
torch.cuda.synchronize(); t0.record()
_, rc = G2.solve(d=spec.d, tol=spec.tol, variant="tiled")
t1.record(); torch.cuda.synchronize()
print(f"cold solve of the modified graph (plan built): {t0.elapsed_time(t1):.1f} ms ({rc['sweeps']} sweeps, {rc['diffused_edges']:.3e} edges)")
