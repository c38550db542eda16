set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_default.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log | head -c 400
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_default.csv $B > gpurun_out/ncu_launch.log 2>&1; echo l=$?
