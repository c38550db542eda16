#!/bin/bash
# round 2: heavy-path rewrite check + microbench + configs[3] rank 0 + configs[4] bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_fullsize.py -k "not full_size" -x -q 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q -k "not full_size" 2>&1 | tail -2
for R in 3 4; do timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 0 --rounds $R 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($R, round(d['ms_per_step'],2), d['config']['sweeps_per_solve'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['roofline']['share_of_step'].items() if v})"; done
timeout 120 ./scripts/mb_rounds
timeout 600 python scripts/config3_rank.py --world 8 --rank 0 > gpurun_out/r2_config3_rank0_w8.json 2> gpurun_out/r2_config3.err; tail -c 1500 gpurun_out/r2_config3_rank0_w8.json; tail -3 gpurun_out/r2_config3.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 > gpurun_out/r2_bench_config4.json 2> gpurun_out/r2_bench_config4.err; tail -c 1500 gpurun_out/r2_bench_config4.json; tail -3 gpurun_out/r2_bench_config4.err
