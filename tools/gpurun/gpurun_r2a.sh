#!/bin/bash
# round-2 iteration: GPU tests, kernel times, a short bench (both arms)
tag=${1:-r2a}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python tools/kernel_times.py > gpurun_out/kernel_times_$tag.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
tail -n 5 gpurun_out/pytest_gpu_$tag.log; cat gpurun_out/kernel_times_$tag.log; cut -c1-1500 gpurun_out/bench_$tag.json
