#!/bin/bash
# runtime variants of the default build: ENVS="|DIT_TILE_WAVES_RT=4|..." (empty = default); ARGS per variant via "env;args"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
IFS='|' read -ra VS <<< "${ENVS:-}"
for rep in 1 2; do
for V in "${VS[@]}"; do
  E="${V%%;*}"; A=""; [[ "$V" == *";"* ]] && A="${V#*;}"
  env $E timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 0 $A > gpurun_out/ab_env.jsonl 2>/dev/null
  python scripts/bench_brief.py "[$V]#$rep" gpurun_out/ab_env.jsonl
done
done
