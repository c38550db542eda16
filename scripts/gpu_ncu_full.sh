# ncu --set full captures of the default schedule's top kernels (one k_tile wave launch, four k_heavy_s launches)
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_tile -s 10 -c 1 -o gpurun_out/r1_k_tile_full $B > gpurun_out/ncu_tile.log 2>&1; echo t=$?
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_heavy_s -s 40 -c 4 -o gpurun_out/r1_k_heavy_full $B > gpurun_out/ncu_heavy.log 2>&1; echo h=$?
