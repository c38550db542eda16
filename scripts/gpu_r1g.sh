B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --variant tiled --rounds 4"
timeout 600 python -m pytest tests/test_gpu_tiled.py -x -q > gpurun_out/pytest_tiled.log 2>&1; echo tiled=$?; tail -2 gpurun_out/pytest_tiled.log
python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 --variant tiled --rounds 4 > gpurun_out/b7.log 2>&1
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_heavy_s|k_tile$" -s 60 -c 10 -o gpurun_out/v3_full $B > gpurun_out/ncu_v3.log 2>&1; echo t=$?
