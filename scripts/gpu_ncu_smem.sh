#!/bin/bash
# shared-memory wavefronts / bank conflicts of one k_tile launch, with and without the bank-aware slot order
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --steps 1 --warmup 2 --no-cpu --e2e-steps 0"
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed
$B > gpurun_out/plain_smem.log 2>&1 && ncu --metrics $M --clock-control none -k k_tile -s 10 -c 1 $B 2>&1 | grep -E "k_tile|l1tex|smsp|gpu__" 
DIT_NO_BANK_ORDER=1 $B > gpurun_out/plain_smem2.log 2>&1 && DIT_NO_BANK_ORDER=1 ncu --metrics $M --clock-control none -k k_tile -s 10 -c 1 $B 2>&1 | grep -E "k_tile|l1tex|smsp|gpu__"
