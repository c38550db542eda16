#!/bin/bash
# A/B of configs[4] (bench.py --config 4) on one box: VARIANTS="c4base cur"
mkdir -p gpurun_out
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
C=paper_1501_06350_b200/csrc
mkdir -p /tmp/cur && cp $C/*.cu $C/*.cuh /tmp/cur/
for rep in 1 2; do
for V in ${VARIANTS:-c4base cur}; do
  cp /tmp/cur/* $C/
  [ "$V" != cur ] && cp variants/$V/* $C/
  python paper_1501_06350_b200/build.py > gpurun_out/build_$V.log 2>&1 || { echo "build failed $V"; continue; }
  timeout 900 python bench.py --config 4 --steps ${STEPS:-3} --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); c=d['config']; print('$V#$rep', {k:round(c[k],1) for k in ('update_ms','resume_ms','resume_sweeps','cold_build_and_solve_ms')}, round(d['ms_per_step'],1))"
done
done
cp /tmp/cur/* $C/
python paper_1501_06350_b200/build.py > /dev/null 2>&1
