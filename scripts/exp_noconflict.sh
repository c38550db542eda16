mkdir -p /tmp/bx; cp -r paper_1501_06350_b200 include /tmp/bx/
(cd /tmp/bx && sed -i 's/^FLAGS = \[/FLAGS = ["-DDIT_EXPERIMENT_NOCONFLICT", /' paper_1501_06350_b200/build.py && python paper_1501_06350_b200/build.py --force > /dev/null 2>&1)
cp /tmp/bx/paper_1501_06350_b200/libdit.so paper_1501_06350_b200/libdit.so
MAX_SWEEPS=31 timeout 300 python scripts/tile_timing.py 3 2>&1 | tail -5
