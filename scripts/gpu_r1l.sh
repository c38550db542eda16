timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_tiled.py -x -q > gpurun_out/pytest_shard.log 2>&1; echo shard=$?; tail -25 gpurun_out/pytest_shard.log
