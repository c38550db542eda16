#!/bin/bash
# round 2: tiled parity + tile timing + rounds sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_tiled.py -x -q 2>&1 | tail -5
timeout 300 python scripts/tile_timing.py 4 2>&1 | tail -14
for R in ${ROUNDS:-2 3 4}; do timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 0 --rounds $R 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($R, round(d['ms_per_step'],2), d['config']['sweeps_per_solve'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['roofline']['share_of_step'].items() if v})"; done
