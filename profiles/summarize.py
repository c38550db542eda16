"""Summarise ncu outputs brought back under gpurun_out/ into profiles/ text files.

    python profiles/summarize.py launches <launches.csv>      # per-kernel share of the run
    python profiles/summarize.py full <report.ncu-rep>        # key metrics + top stalls per kernel
"""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    S = sum(tot.values())
    print(f"# ncu launch list {path}: gpu__time_duration.sum per kernel (cold-cache, serialised)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:40s} launches={cnt[k]:5d} total={v / 1e6:10.3f} ms share={v / S:6.1%} avg={v / cnt[k] / 1e3:10.1f} us")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full {path}")
    for r in rows[2:]:
        print("kernel:", r[hdr.index("Kernel Name")])
        for k in KEYS:
            if k in hdr:
                print(f"  {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
        st = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    st.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("  top stall samples:", ", ".join(f"{n}={int(v)}" for v, n in st[:6]))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
