#!/bin/bash
# TMEM microbenchmark, k_tile phase timing, bench of the current build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 120 ./scripts/mb_tmem > gpurun_out/mb_tmem.txt 2>&1; echo mb=$?
cat gpurun_out/mb_tmem.txt
timeout 600 python scripts/tile_timing.py 4 > gpurun_out/tile_timing.txt 2>&1; echo tt=$?

cat gpurun_out/tile_timing.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/bench_g.jsonl 2>/dev/null
python scripts/bench_brief.py hoist_hsum gpurun_out/bench_g.jsonl
