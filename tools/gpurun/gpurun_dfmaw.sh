#!/bin/bash
# experiment: H accumulate with k consumer warps running tasks on the DFMA pipe (KBG_EXPERIMENTS build)
for k in 0 2 4 6 8; do
  echo "dfma_warps=$k $(KBG_DFMA_WARPS=$k KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/exp/libkbgrid.so timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 --kernels h_accumulate | grep -o '"median_ms": [0-9.]*\|"rel_diff_vs_first": [-0-9.e]*' | tr '\n' ' ')"
done
echo "product $(timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 --kernels h_accumulate | grep -o '"median_ms": [0-9.]*')"
