#!/bin/bash
# Build a libdit.so variant with extra nvcc defines into variants/libdit_<name>.so
# (experiments only; the product build is paper_1501_06350_b200/build.py).
# usage: scripts/build_variant.sh <name> -DKNOB=V ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
python "$root/paper_1501_06350_b200/build.py" > /dev/null
obj=$root/paper_1501_06350_b200/build
mkdir -p "$root/variants" /tmp/dit_var_$name
objs=""
for o in $obj/*.o; do
  b=$(basename $o .o)
  if [ "$b" = dit_tile ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I"$root/include" "$@" -c "$root/paper_1501_06350_b200/csrc/dit_tile.cu" -o /tmp/dit_var_$name/dit_tile.o
    objs="$objs /tmp/dit_var_$name/dit_tile.o"
  else
    objs="$objs $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/variants/libdit_$name.so" $objs -lcudart_static -lrt -ldl -lpthread
echo "$root/variants/libdit_$name.so"
