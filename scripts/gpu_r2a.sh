#!/bin/bash
# round 2: new warp-specialised k_tile -- tiled parity tests, tile timing, bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1 || { tail gpurun_out/r2a_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tiled.py -x -q 2>&1 | tail -15
timeout 300 python scripts/tile_timing.py 4 2>&1 | tail -12
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/r2a_bench.log 2>&1; tail -c 3000 gpurun_out/r2a_bench.log
