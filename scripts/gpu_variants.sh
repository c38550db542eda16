#!/bin/bash
# build variants of libdit (compile-time flags) and time the bench on each: VARIANTS="flagsA|flagsB" ROUNDS="2 4"
mkdir -p gpurun_out
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
IFS='|' read -ra VS <<< "${VARIANTS:-}"
i=0
for V in "${VS[@]}"; do
  i=$((i+1))
  DIT_NVCC_FLAGS="$V" python paper_1501_06350_b200/build.py --force > gpurun_out/build_v$i.log 2>&1 || { echo "build failed: $V"; tail -5 gpurun_out/build_v$i.log; continue; }
  for R in ${ROUNDS:-4}; do
    timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 0 --rounds $R > gpurun_out/var_$i_$R.json 2> gpurun_out/var_$i_$R.err
    python scripts/bench_brief.py "[$V] R=$R" gpurun_out/var_$i_$R.json
  done
done
