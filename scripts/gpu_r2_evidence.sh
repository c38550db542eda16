#!/bin/bash
# round 2 evidence: default bench line, reference arm, configs[4] mode, configs[3] ranks, launch list, ncu full captures
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/r2_bench_default.jsonl 2> gpurun_out/r2_bench_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference.jsonl 2> gpurun_out/r2_bench_reference.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 > gpurun_out/r2_bench_config4.jsonl 2> gpurun_out/r2_bench_config4.err
for w in 8 4 2; do timeout 600 python scripts/config3_rank.py --world $w --rank 0 >> gpurun_out/r2_config3_rank0.jsonl 2>> gpurun_out/r2_config3.err; done
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain_ev.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2_launches.csv $B > gpurun_out/ncu_l.log 2>&1
$B > gpurun_out/plain_ev2.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_tile -s 10 -c 2 -o gpurun_out/r2_final_k_tile_full $B > gpurun_out/ncu_t.log 2>&1
$B > gpurun_out/plain_ev3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_heavy -s 60 -c 9 -o gpurun_out/r2_final_k_heavy_full $B > gpurun_out/ncu_h.log 2>&1
ls -la gpurun_out | tail -30
