"""One line from a bench.py JSON output: label, ms per solve, sweeps, dominant kernel ms per sweep, frac, shares."""
import json, sys
label, path = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(label, round(d["ms_per_step"], 2), d["config"]["sweeps_per_solve"], round(r["avg_launch_ms"], 3),
          round(r["frac"], 3), {k: round(v, 3) for k, v in r["share_of_step"].items() if v}, flush=True)
except Exception as e:
    print(label, "no result:", e, flush=True)
