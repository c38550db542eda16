set -x
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0 --variant tiled --rounds 4"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_tiled.csv $B > gpurun_out/ncu_launch.log 2>&1; echo l=$?
ncu --set full --clock-control none --import-source on -k regex:k_tile_local -s 3 -c 1 -o gpurun_out/tile_full $B > gpurun_out/ncu_tile.log 2>&1; echo t=$?
ncu --set full --clock-control none --import-source on -k regex:k_pull -s 3 -c 1 -o gpurun_out/rpull_full $B > gpurun_out/ncu_rpull.log 2>&1; echo p=$?
