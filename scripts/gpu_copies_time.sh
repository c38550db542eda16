#!/bin/bash
# total device time of the plan's copy-matching kernels (ncu launch list) per variant: VARIANTS="a|b"
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
IFS='|' read -ra VS <<< "${VARIANTS:-}"
for V in "${VS[@]}"; do
  DIT_NVCC_FLAGS="$V" python paper_1501_06350_b200/build.py --force > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ell_copies|k_plan_ell|k_plan_place" --csv python scripts/build_timing.py 2>/dev/null > gpurun_out/ct.csv
  python - "$V" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open("gpurun_out/ct.csv")) if len(r) > 10]
h = rows[0]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
t = collections.defaultdict(float)
for r in rows[1:]:
    try: t[r[ik].split("(")[0].split("<")[0].replace("void ", "")] += float(r[iv].replace(",", ""))
    except ValueError: pass
print(sys.argv[1], {k: round(v / 2e6, 2) for k, v in t.items()}, "ms per build")
PY
done
