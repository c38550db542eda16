# k_tile phase timing of diagnostic builds (wrong results: fixed 21 sweeps)
cp paper_1501_06350_b200/libdit.so /tmp/libdit_orig.so
for v in "$@"; do
  cp variants/libdit_$v.so paper_1501_06350_b200/libdit.so
  echo "== $v"; MAX_SWEEPS=21 timeout 300 python scripts/tile_timing.py 4 2>&1 | tail -5
done
cp /tmp/libdit_orig.so paper_1501_06350_b200/libdit.so
