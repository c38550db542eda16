# the default bench line, its ncu launch list, and one --set full capture of the top kernels
python bench.py > gpurun_out/bench_r1_default.log 2>&1; echo bench=$?
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r1_default.csv $B > gpurun_out/ncu_launch.log 2>&1; echo l=$?
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_tile -s 10 -c 1 -o gpurun_out/r1_k_tile_full $B > gpurun_out/ncu_tile.log 2>&1; echo t=$?
$B > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_heavy_s -s 40 -c 4 -o gpurun_out/r1_k_heavy_full $B > gpurun_out/ncu_heavy.log 2>&1; echo h=$?
