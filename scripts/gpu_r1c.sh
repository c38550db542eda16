set -x
timeout 600 python -m pytest tests/test_gpu_tiled.py -x -q > gpurun_out/pytest_tiled.log 2>&1; echo tiled=$?
tail -30 gpurun_out/pytest_tiled.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for v in "--variant tiled --rounds 4" "--variant tiled --rounds 8" "--variant tiled --rounds 2"; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 $v >> gpurun_out/bench_tiled2.log 2>&1; echo bench=$?
done
tail -3 gpurun_out/bench_tiled2.log
