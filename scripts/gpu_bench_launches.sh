# the default bench line and its ncu launch list (no --set full captures)
python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r1_default.csv $B > gpurun_out/ncu_launch.log 2>&1; echo l=$?
