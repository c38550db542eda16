#!/bin/bash
# ncu launch list (device time per launch, cold-cache, serialised) of the default bench: usage gpu_launches.sh TAG [extra bench args]
TAG=${1:-r2}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 $*"
$B > gpurun_out/plain_l_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_l_$TAG.log 2>&1; echo rc=$?
python profiles/summarize.py launches gpurun_out/launches_$TAG.csv | head -20
