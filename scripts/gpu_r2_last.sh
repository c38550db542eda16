#!/bin/bash
# last evidence of round 2 on the final tree: smoke, GPU suite, default bench line, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python __graft_entry__.py > gpurun_out/r2z_smoke.txt 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2z_gpu_tests.txt 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/r2z_bench_default.jsonl 2> gpurun_out/r2z_bench_default.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2z_bench_reference.jsonl 2> gpurun_out/r2z_bench_reference.err; echo ref=$?
