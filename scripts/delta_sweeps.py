"""Debug: configs[4]-style update + warm tiled resume with the kept plan (delta
in-edges, R18) against DIT_NO_DELTA (plan rebuilt from the new CSR):
update ms, resume ms, sweeps.   python scripts/delta_sweeps.py [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1501_06350_b200 as eng
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
spec = synth.CONFIGS[4] if n >= synth.CONFIGS[4].n else synth.CONFIGS[4].scaled(n, seed=14)
g = synth.generate(spec)
delta = synth.rewire(spec, g, fraction=0.01, seed=4)
dev = torch.device("cuda", 0)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
rp, cl, wv = t(g.row_ptr), t(g.col), t(g.w) if g.w is not None else None
dd = {k: (t(v) if v is not None else None) for k, v in delta.items()}
adds = {k: (v if k.startswith("add") else None) for k, v in dd.items()}
rems = {k: (v if k.startswith("rem") else None) for k, v in dd.items()}
deg = np.diff(g.row_ptr)
def sub(mask):
    return dict(add_src=t(delta["add_src"][mask]), add_dst=t(delta["add_dst"][mask]),
                add_w=t(delta["add_w"][mask]) if delta["add_w"] is not None else None, rem_src=None, rem_dst=None)
a_s, a_d = delta["add_src"].astype(np.int64), delta["add_dst"].astype(np.int64)
cases = [("delta-adds", adds), ("rebuild-adds", adds)]
if len(sys.argv) > 2 and sys.argv[2] == "deltaonly":
    cases = [("delta", dd)]
elif len(sys.argv) > 2 and sys.argv[2] == "full":
    cases = [("delta", dd), ("rebuild", dd)]
elif len(sys.argv) > 2:
    cases = [("delta-adds-nondangling", sub(deg[a_s] > 0)), ("delta-adds-dangling", sub(deg[a_s] == 0)),
             ("delta-adds-sametile", sub(a_s // 512 == a_d // 512)), ("delta-adds-othertile", sub(a_s // 512 != a_d // 512)),
             ("rebuild-adds-othertile", sub(a_s // 512 != a_d // 512))]
for mode, upd in cases:
    dd_ = upd
    if mode.startswith("rebuild"): os.environ["DIT_NO_DELTA"] = "1"
    else: os.environ.pop("DIT_NO_DELTA", None)
    G = eng.DIGraph(g.n, rp, cl, wv)
    _, r0 = G.solve(d=spec.d, tol=spec.tol, variant="tiled")
    torch.cuda.synchronize(); a = time.perf_counter()
    G.update_edges(**dd_)
    torch.cuda.synchronize(); b = time.perf_counter()
    _, r = G.resume(tol=spec.tol, variant="tiled")
    torch.cuda.synchronize(); c = time.perf_counter()
    print(mode, "cold sweeps", r0["sweeps"], "update ms %.1f" % ((b - a) * 1e3), "resume ms %.1f" % ((c - b) * 1e3),
          "sweeps", r["sweeps"], "bound %.3g" % r["bound"], flush=True)
    G.close()
