# k_tile phase timing at a given local_rounds with fixed 21 sweeps (diagnostic builds)
cp paper_1501_06350_b200/libdit.so /tmp/libdit_orig.so
R=$1; shift
for v in "$@"; do
  cp variants/libdit_$v.so paper_1501_06350_b200/libdit.so
  echo "== $v R=$R"; MAX_SWEEPS=21 timeout 300 python scripts/tile_timing.py $R 2>&1 | tail -5
  MAX_SWEEPS=21 TAG=$v timeout 300 python scripts/solve_timing.py 2>&1 | tail -1
done
cp /tmp/libdit_orig.so paper_1501_06350_b200/libdit.so
