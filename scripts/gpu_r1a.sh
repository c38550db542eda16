set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for v in "--variant auto --theta 1" "--variant pull --theta 0" "--variant tiled --rounds 4" "--variant tiled --rounds 8" "--variant tiled --rounds 2"; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 $v >> gpurun_out/bench_variants.log 2>&1; echo bench=$?
done
