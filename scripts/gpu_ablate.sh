#!/bin/bash
# k_tile ablations (compile flags; results are wrong by design): device ms per sweep over fixed sweeps
python -c "from oracle import di; di.build_clib(); import synth; synth.build()" > /dev/null 2>&1
IFS='|' read -ra VS <<< "${VARIANTS:-}"
for V in "${VS[@]}"; do
  DIT_NVCC_FLAGS="$V" python paper_1501_06350_b200/build.py --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  echo "[$V] $(timeout 300 python scripts/fixed_sweeps.py 8 2>&1 | tail -1)"
done
