#!/bin/bash
# heavy variants: tiled / shard GPU tests on the working tree, then the same-box A/B (variants/<name>/)
mkdir -p gpurun_out
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
python paper_1501_06350_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_shard.py -x -q -m gpu > gpurun_out/heavy_tests.txt 2>&1; tail -3 gpurun_out/heavy_tests.txt
VARIANTS="${VARIANTS:-base cur}" STEPS=5 bash scripts/gpu_ab.sh
