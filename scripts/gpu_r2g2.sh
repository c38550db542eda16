#!/bin/bash
# k_tile ncu capture (one sweep), tile timing, update tests and configs[4] of the current build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_tiled.py tests/test_gpu.py -k "update or golden" 2>&1 | tail -2
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 > gpurun_out/r2f_bench_config4.jsonl 2> gpurun_out/r2f_bench_config4.err
python -c "import json; d=json.loads(open('gpurun_out/r2f_bench_config4.jsonl').read().strip().splitlines()[-1]); c=d['config']; print({k:c[k] for k in ('update_ms','resume_ms','resume_sweeps','cold_build_and_solve_ms')}, d['ms_per_step'])"
DIT_BUILD_TIMING=1 timeout 600 python scripts/delta_sweeps.py 50000000 full > gpurun_out/r2f_delta_phases.txt 2>&1
timeout 300 python scripts/tile_timing.py 4 > gpurun_out/r2f_tile_timing.txt 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain_ev.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_tile -s 15 -c 3 -o gpurun_out/r2f_k_tile_full $B > gpurun_out/ncu_t.log 2>&1; echo ncu=$?
