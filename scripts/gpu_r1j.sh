timeout 600 python -m pytest tests/test_gpu_tiled.py -x -q > gpurun_out/pytest_tiled.log 2>&1; echo tiled=$?; tail -1 gpurun_out/pytest_tiled.log
rm -f gpurun_out/bench_j.log
for r in 4 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 0 --variant tiled --rounds $r >> gpurun_out/bench_j.log 2>&1; echo bench=$?
done
python - <<'PY'
import json
for l in open('gpurun_out/bench_j.log'):
    if l.startswith('{'):
        d=json.loads(l); c=d['config']; r=d['roofline']
        print(c['local_rounds'],'sweeps',c['sweeps_per_solve'],'ms %.1f'%d['ms_per_step'],'dom',r['kernel'],'frac %.3f'%r['frac'],'avg_ms %.3f'%r['avg_launch_ms'], {k:round(v,3) for k,v in r['share_of_step'].items()})
PY
