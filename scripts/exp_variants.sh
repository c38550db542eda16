#!/bin/bash
# usage: scripts/exp_variants.sh name1 name2 ...: per variant lib, tiled GPU tests + k_tile phases + bench
cp paper_1501_06350_b200/libdit.so /tmp/libdit_orig.so
for v in "$@"; do
  cp variants/libdit_$v.so paper_1501_06350_b200/libdit.so
  echo "== $v"
  [ -n "$EXP_TESTS" ] && timeout 600 python -m pytest tests/test_gpu_tiled.py -q -x 2>&1 | tail -1
  [ -n "$EXP_TIMING" ] && timeout 300 python scripts/tile_timing.py 4 2>&1 | tail -5
  timeout 300 python bench.py --steps 3 --no-cpu --e2e-steps 0 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', 'ms', round(d['ms_per_step'],2), 'sweeps', d['config']['sweeps_per_solve'], 'tile_ms', round(r['avg_launch_ms'],3), 'frac', round(r['frac'],3), 'share', {k: round(v,3) for k,v in r['share_of_step'].items() if v}, 'light', d['config']['tiled_plan']['light_edges'], 'heavy', d['config']['tiled_plan']['heavy_edges'])"
done
cp /tmp/libdit_orig.so paper_1501_06350_b200/libdit.so
