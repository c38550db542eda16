B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --variant tiled --rounds 4"
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_tile -s 10 -c 1 -o gpurun_out/v4_tile $B > gpurun_out/ncu_v4.log 2>&1; echo t=$?
