# k_tile carveout / L1 hit rate / duration for a variants/libdit_<v>.so
cp paper_1501_06350_b200/libdit.so /tmp/libdit_orig.so
for v in "$@"; do
  cp variants/libdit_$v.so paper_1501_06350_b200/libdit.so
  B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
  echo "== $v"; $B > /dev/null 2>&1 && ncu --metrics launch__shared_mem_config_size,l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct,gpu__time_duration.sum --clock-control none -k k_tile -s 10 -c 1 $B 2>&1 | grep -E "config_size|hit_rate|duration"
done
cp /tmp/libdit_orig.so paper_1501_06350_b200/libdit.so
