#!/bin/bash
# deterministic-H cost split (KBG_EXPERIMENTS build): scatter bits 4 = no lo RED, 8 = no hi RED, 2 = no scatter
L=KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/exp/libkbgrid.so
for r in 1 2; do
for det in 0 1; do for sc in 0 4 8 12 2; do
  echo "det=$det scatter=$sc $(env $L timeout 120 python tools/kernel_times.py --schedules 3 --fallback 0 --det $det --scatter $sc --kernels h_accumulate | grep -o '"median_ms": [0-9.]*')"
done; done; done
echo "product det=0 $(timeout 120 python tools/kernel_times.py --schedules 3 --fallback 0 --det 0 --kernels h_accumulate | grep -o '"median_ms": [0-9.]*')"
echo "product det=1 $(timeout 120 python tools/kernel_times.py --schedules 3 --fallback 0 --det 1 --kernels h_accumulate | grep -o '"median_ms": [0-9.]*')"
