"""Debug: where the fluid sits after k warm sweeps with the kept plan (R18)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1501_06350_b200 as eng
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
spec = synth.CONFIGS[4].scaled(n, seed=14)
g = synth.generate(spec)
delta = synth.rewire(spec, g, fraction=0.01, seed=4)
deg = np.diff(g.row_ptr)
a_s, a_d = delta["add_src"].astype(np.int64), delta["add_dst"].astype(np.int64)
m = deg[a_s] == 0
sub = dict(add_src=delta["add_src"][m], add_dst=delta["add_dst"][m], add_w=delta["add_w"][m])
for mode in ("delta", "rebuild"):
    if mode == "rebuild": os.environ["DIT_NO_DELTA"] = "1"
    G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
    G.solve(d=spec.d, tol=spec.tol, variant="tiled")
    G.update_edges(**sub)
    for k in (6, 12, 20):
        _, r = G.resume(tol=0.0, variant="tiled", max_sweeps=k)
        F, H, _, _ = G.state()
        F = F.cpu().numpy()
        top = np.argsort(-np.abs(F))[:8]
        print(mode, "after", k, "|F|1 %.3e" % np.abs(F).sum(), "top share %.3f" % (np.abs(F[top]).sum() / np.abs(F).sum()))
        for i in top[:5]:
            outs = [int(t) for t, s in zip(a_d[m], a_s[m]) if s == i]
            ins = int(((a_d[m] == i)).sum())
            print("   node", i, "F %.3e" % F[i], "plan deg", deg[i], "added out", outs[:4], "added in", ins, "tile", i // 512)
        G.close()
        G = eng.DIGraph(g.n, g.row_ptr, g.col, g.w)
        G.solve(d=spec.d, tol=spec.tol, variant="tiled")
        G.update_edges(**sub)
