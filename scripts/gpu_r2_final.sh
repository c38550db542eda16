#!/bin/bash
# round 2 final evidence for the current kernels: GPU suite, default bench line, reference arm,
# configs[4] mode, launch list, ncu full captures of one sweep (3 k_tile waves, 3x2 heavy launches)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python __graft_entry__.py > gpurun_out/r2f_smoke.txt 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2f_gpu_tests.txt 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/r2f_bench_default.jsonl 2> gpurun_out/r2f_bench_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2f_bench_reference.jsonl 2> gpurun_out/r2f_bench_reference.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 > gpurun_out/r2f_bench_config4.jsonl 2> gpurun_out/r2f_bench_config4.err
DIT_BUILD_TIMING=1 timeout 600 python scripts/delta_sweeps.py 50000000 full > gpurun_out/r2f_delta_phases.txt 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain_ev.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r2f_launches.csv $B > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k k_tile -s 15 -c 3 -o gpurun_out/r2f_k_tile_full $B > gpurun_out/ncu_t.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_heavy -s 60 -c 6 -o gpurun_out/r2f_k_heavy_full $B > gpurun_out/ncu_h.log 2>&1
ls -la gpurun_out | tail -30
