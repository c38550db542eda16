#!/bin/bash
# A/B of compile-flag variants of libdit on one box: FLAGS="|-DX=1|-DY=2" (empty = default build)
mkdir -p gpurun_out
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
IFS='|' read -ra VS <<< "${FLAGS:-}"
for rep in 1 2; do
for V in "${VS[@]}"; do
  DIT_NVCC_FLAGS="$V" python paper_1501_06350_b200/build.py --force > gpurun_out/build_flags.log 2>&1 || { echo "build failed: $V"; continue; }
  timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab_flags.jsonl 2>/dev/null
  python scripts/bench_brief.py "[$V]#$rep" gpurun_out/ab_flags.jsonl
done
done
python paper_1501_06350_b200/build.py --force > /dev/null 2>&1
