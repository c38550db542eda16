timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_shard.py -q -x 2>&1 | tail -1
B="python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1"
$B > gpurun_out/b_e2e.log 2>&1; tail -1 gpurun_out/b_e2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', d['e2e'])"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_e2e.csv $B > gpurun_out/ncu_launch.log 2>&1; echo l=$?
