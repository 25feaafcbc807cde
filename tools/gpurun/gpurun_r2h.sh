#!/bin/bash
# GPU tests, the 1-GPU bench line and the kernel times inside a pass, on one box
tag=${1:-r2h}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 --kernels density,h_accumulate,pass > gpurun_out/kernel_times_$tag.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$tag.log
python3 -c "
import json
d=json.loads(open('gpurun_out/bench_$tag.json').read().strip().splitlines()[-1])
print(d['value'], d['segments_ms'], d['roofline']['kernel'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
grep -o '"kernel": "[a-z_]*".*"median_ms": [0-9.]*\|"pass_order".*' gpurun_out/kernel_times_$tag.log | sed 's/"plan".*"median/median/'
