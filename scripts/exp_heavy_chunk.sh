for c in 24 16 96; do
  mkdir -p /tmp/hc$c; cp -r paper_1501_06350_b200 include /tmp/hc$c/
  (cd /tmp/hc$c && sed -i "s/^FLAGS = \[/FLAGS = [\"-DDIT_STRIPE_MB=$c\", /" paper_1501_06350_b200/build.py && python paper_1501_06350_b200/build.py --force > /dev/null 2>&1)
  cp /tmp/hc$c/paper_1501_06350_b200/libdit.so paper_1501_06350_b200/libdit.so
  timeout 300 python bench.py --steps 3 --no-cpu --e2e-steps 0 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($c, d['ms_per_step'], d['config']['sweeps_per_solve'], d['roofline']['share_of_step']['k_heavy_s'])"
done
