#!/bin/bash
# usage: gpurun_var.sh tag v1 v2 ...  (variants built by tools/build_variants.sh)
tag=$1; shift; mkdir -p gpurun_out; out=gpurun_out/var_$tag.log; : > $out
for v in "$@"; do
  export KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/$v/libkbgrid.so
  timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 1 | sed "s/^/$v pytest: /" >> $out
  timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 >> $out 2>&1
done
cat $out
