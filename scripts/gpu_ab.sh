#!/bin/bash
# A/B: the bench in variants/old (an older commit's tree, built here) vs the current tree
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for d in variants/old .; do
  (cd $d && timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 0 --rounds 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', round(d['ms_per_step'],2), d['config']['sweeps_per_solve'], round(d['roofline']['avg_launch_ms'],3), round(d['roofline']['frac'],3), {k: round(v,3) for k,v in d['roofline']['share_of_step'].items() if v})")
done
