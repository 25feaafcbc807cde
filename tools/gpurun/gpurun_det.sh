#!/bin/bash
# deterministic-H cost: legacy FP64 atomics vs two-limb exact scatter, plus the GPU tests
tag=${1:-det}; mkdir -p gpurun_out; out=gpurun_out/det_$tag.log; : > $out
kt="python tools/kernel_times.py --schedules 3 --fallback 0"
for d in 0 1 0 1; do timeout 120 $kt --det $d >> $out 2>&1; done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
grep -o '"det": [01], "kernel": "[a-z_]*".*"median_ms": [0-9.]*' $out | sed 's/"plan".*"median/median/' ; tail -15 gpurun_out/pytest_gpu_$tag.log
