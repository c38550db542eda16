for th in 4 8 16; do
  mkdir -p /tmp/b$th; cp -r paper_1501_06350_b200 /tmp/b$th/; cp -r include /tmp/b$th/
  (cd /tmp/b$th && sed -i "s/^FLAGS = \[/FLAGS = [\"-DDIT_HEAVY_TH=$th\", /" paper_1501_06350_b200/build.py && python paper_1501_06350_b200/build.py --force > /dev/null 2>&1)
  cp /tmp/b$th/paper_1501_06350_b200/libdit.so paper_1501_06350_b200/libdit.so
  python bench.py --steps 3 --no-cpu --e2e-steps 0 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('th', $th, d['ms_per_step'], d['config']['sweeps_per_solve'], d['config']['tiled_plan']['light_edges'], d['config']['tiled_plan']['heavy_edges'], {k:round(v,3) for k,v in d['roofline']['share_of_step'].items() if v})"
done
