python -m pytest tests/test_gpu_tiled.py -q -x 2>&1 | tail -1
timeout 300 python scripts/tile_timing.py 3 2>&1 | tail -5
timeout 300 python bench.py --steps 3 --no-cpu --e2e-steps 0 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('1024-block', d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
DIT_NO_EDGE_STAGING=1 timeout 300 python bench.py --steps 3 --no-cpu --e2e-steps 0 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('1024-block unstaged', d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
