#!/bin/bash
# ncu --set full of one k_tile launch (default bench schedule); usage: gpu_ncu_tile.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_tile -s 10 -c 1 -o gpurun_out/${TAG}_k_tile_full $B > gpurun_out/ncu_tile_$TAG.log 2>&1; echo t=$?
