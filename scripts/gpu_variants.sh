#!/bin/bash
# build variants of libdit (compile-time flags) and time the bench on each: VARIANTS="flagsA|flagsB" ROUNDS="2 4"
mkdir -p gpurun_out
IFS='|' read -ra VS <<< "${VARIANTS:-}"
for V in "${VS[@]}"; do
  DIT_NVCC_FLAGS="$V" python paper_1501_06350_b200/build.py --force > gpurun_out/build_v.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v.log; continue; }
  python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
  for R in ${ROUNDS:-4}; do
    timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 0 --rounds $R 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$V] R=$R', round(d['ms_per_step'],2), d['config']['sweeps_per_solve'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['roofline']['share_of_step'].items() if v})"
  done
done
