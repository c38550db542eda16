#!/bin/bash
# round 2: k_tile phase timing (+ diagnostic variants)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python scripts/tile_timing.py 4 2>&1 | tail -14
echo "--- DIT_TILE_DIAG=1 (unstaged local sums skipped)"
DIT_TILE_DIAG=1 MAX_SWEEPS=21 timeout 300 python scripts/tile_timing.py 4 2>&1 | tail -14
