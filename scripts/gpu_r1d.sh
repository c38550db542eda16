B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --variant tiled --rounds 4"
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_tile<|k_heavy" -s 30 -c 3 -o gpurun_out/tile2_full $B > gpurun_out/ncu_tile2.log 2>&1; echo t=$?
