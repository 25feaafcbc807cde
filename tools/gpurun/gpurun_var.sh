#!/bin/bash
# usage: [CONFIGS="cubic56_200Ry super448_200Ry"] gpurun_var.sh tag v1 v2 ...  (variants built by tools/build_variants.sh)
tag=$1; shift; mkdir -p gpurun_out; out=gpurun_out/var_$tag.log; : > $out
for v in "$@"; do
  export KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/$v/libkbgrid.so
  timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 1 | sed "s/^/$v pytest: /" >> $out
  for c in ${CONFIGS:-cubic56_200Ry}; do
    timeout 300 python tools/kernel_times.py --config $c --schedules 3 --fallback 0 2>&1 | sed "s/^/$v /" >> $out
  done
done
cat $out
