"""Debug: the tiled plan build's phase times on configs[2] (DIT_BUILD_TIMING=1,
stream-synchronised marks), plan built from a device-resident CSR."""
import os, sys
os.environ["DIT_BUILD_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1501_06350_b200 as eng
spec = synth.CONFIGS[int(os.environ.get("CONFIG", "2"))]
g = synth.generate(spec)
dev = torch.device("cuda", 0)
for it in range(2):
    G = eng.DIGraph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
    print(f"--- build {it}", flush=True)
    G.solve(d=spec.d, tol=spec.tol, variant="tiled", max_sweeps=1)
    G.close()
