#!/bin/bash
# per variant (compile flags): k_tile phase cycles (tile_timing.py) and the shared-memory
# load wavefronts / bank conflicts of one k_tile launch (ncu); VARIANTS="flagsA|flagsB"
mkdir -p gpurun_out
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
IFS='|' read -ra VS <<< "${VARIANTS:-}"
M=l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_shared_ld.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg
i=0
for V in "${VS[@]}"; do
  i=$((i+1))
  DIT_NVCC_FLAGS="$V" python paper_1501_06350_b200/build.py --force > gpurun_out/build_b$i.log 2>&1 || { echo "build failed: $V"; continue; }
  echo "== [$V]"
  timeout 300 python scripts/tile_timing.py 4 2>&1 | head -12
  timeout 600 ncu --metrics $M --clock-control none -k k_tile -s 10 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 2>&1 | grep -E "^\s+(l1tex|smsp|gpu__|sm__)" 
done
