d=/tmp/lean1; mkdir -p $d; cp -r paper_1501_06350_b200 include $d/
(cd $d && sed -i 's/^FLAGS = \[/FLAGS = ["-DDIT_LEAN_BUNDLE=1", "-DDIT_LIGHT_CAP=1024", /' paper_1501_06350_b200/build.py && python paper_1501_06350_b200/build.py --force > /dev/null 2>&1)
cp $d/paper_1501_06350_b200/libdit.so paper_1501_06350_b200/libdit.so
python -m pytest tests/test_gpu_tiled.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout 300 python bench.py --steps 3 --no-cpu --e2e-steps 0 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lean1', d['ms_per_step'], d['config']['sweeps_per_solve'], d['roofline']['avg_launch_ms'])"
MAX_SWEEPS=21 timeout 300 python scripts/tile_timing.py 4 | tail -4
