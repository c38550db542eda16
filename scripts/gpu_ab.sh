#!/bin/bash
# A/B on one box: variants/<name>/ holds replacement csrc files; "cur" = the working tree.
# usage: VARIANTS="base cur" STEPS=5 bash scripts/gpu_ab.sh [extra]
mkdir -p gpurun_out
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
C=paper_1501_06350_b200/csrc
mkdir -p /tmp/cur && cp $C/*.cu $C/*.cuh /tmp/cur/
for rep in 1 2; do
for V in ${VARIANTS:-base cur}; do
  cp /tmp/cur/* $C/
  [ "$V" != cur ] && cp variants/$V/* $C/
  python paper_1501_06350_b200/build.py > gpurun_out/build_$V.log 2>&1 || { echo "build failed $V"; tail -5 gpurun_out/build_$V.log; continue; }
  timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu --e2e-steps 0 > gpurun_out/ab_$V.jsonl 2>/dev/null
  python scripts/bench_brief.py "$V#$rep" gpurun_out/ab_$V.jsonl
done
done
cp /tmp/cur/* $C/
python paper_1501_06350_b200/build.py > /dev/null 2>&1
