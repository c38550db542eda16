# usage: scripts/ncu_variant.sh <variant>: one k_tile launch under ncu --set full with variants/libdit_<variant>.so
v=$1
cp paper_1501_06350_b200/libdit.so /tmp/libdit_orig.so
cp variants/libdit_$v.so paper_1501_06350_b200/libdit.so
B="python bench.py --steps 1 --warmup 3 --no-cpu --e2e-steps 0"
$B > gpurun_out/plain_$v.log 2>&1 && ncu --set full --clock-control none --import-source on -k k_tile -s 10 -c 1 -o gpurun_out/var_${v}_tile $B > gpurun_out/ncu_var_$v.log 2>&1; echo t=$?
cp /tmp/libdit_orig.so paper_1501_06350_b200/libdit.so
