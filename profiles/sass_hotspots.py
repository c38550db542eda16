"""SASS hotspots of an ncu --set full capture (needs --import-source on).

    ncu -i REP --page source --csv --print-source sass > src.csv
    python profiles/sass_hotspots.py src.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
ia, isrc, iss, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
data = []
for r in rows[2:]:
    try:
        s = int(r[iss])
    except (ValueError, IndexError):
        continue
    data.append((s, r))
tot = sum(s for s, _ in data)
agg = {}
for s, r in data:
    for i in sc:
        try:
            agg[h[i]] = agg.get(h[i], 0) + int(r[i])
        except ValueError:
            pass
print(f"# total samples {tot}; stall totals: " + ", ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for idx, (s, r) in enumerate(data):
    r.append(idx)
for s, r in sorted(data, key=lambda x: -x[0])[:top]:
    st = sorted(((int(r[i]) if r[i].isdigit() else 0, h[i][6:]) for i in sc), reverse=True)[:2]
    print(f"{100*s/tot:5.1f}% {r[-1]:5d} {r[iex]:>10s}  {r[isrc].strip()[:60]:60s} " + " ".join(f"{n}={v}" for v, n in st))
