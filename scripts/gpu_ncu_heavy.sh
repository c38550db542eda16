#!/bin/bash
# ncu --set full of k_heavy_chunks launches (default bench schedule); usage: gpu_ncu_heavy.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain_h_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_heavy -s 60 -c 4 -o gpurun_out/${TAG}_k_heavy_full $B > gpurun_out/ncu_heavy_$TAG.log 2>&1; echo h=$?
