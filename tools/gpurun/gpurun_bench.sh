#!/bin/bash
# usage: gpurun_bench.sh tag
tag=${1:-r01}; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$tag.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$tag.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$tag.log
timeout 300 python bench.py --profile --no-e2e > gpurun_out/plain_$tag.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --profile --no-e2e > gpurun_out/ncu_launch_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_persist|k_dm_repack|k_mirror" -c 5 -o gpurun_out/prof_$tag python bench.py --profile --no-e2e > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$tag.log
tail -n 2 gpurun_out/bench_$tag.log gpurun_out/bench_ref_$tag.log gpurun_out/ncu_full_$tag.log
