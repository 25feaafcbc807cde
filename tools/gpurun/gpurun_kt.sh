#!/bin/bash
# quick: GPU tests + kernel times (FP64 atomics and deterministic) on the 56-atom cell
tag=${1:-kt}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 > gpurun_out/kernel_times_$tag.log 2>&1
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 --det 1 --kernels h_accumulate >> gpurun_out/kernel_times_$tag.log 2>&1
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 --config super448_200Ry >> gpurun_out/kernel_times_$tag.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$tag.log; python3 -c "
import json
for l in open('gpurun_out/kernel_times_$tag.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['det'], d['kernel'], d['median_ms'])"
