#!/bin/bash
# usage: gpurun_iter.sh [tag] [ncu]
tag=${1:-it}; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python tools/kernel_times.py > gpurun_out/kernel_times_$tag.log 2>&1
if [ "$2" == "ncu" ]; then
timeout 300 python bench.py --profile --no-e2e > gpurun_out/plain_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_density|k_hamiltonian|k_persist" -c 2 -o gpurun_out/prof_$tag python bench.py --profile --no-e2e > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$tag.log
fi
tail -n 2 gpurun_out/pytest_gpu_$tag.log; cat gpurun_out/kernel_times_$tag.log
