#!/bin/bash
n=${1:-2}; tag=${2:-r01}; mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/bench_n${n}_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n${n}_$tag.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 10 --warmup 3 --config super448_200Ry > gpurun_out/bench448_n${n}_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/bench448_n${n}_$tag.log
timeout 300 python bench.py --steps 10 --warmup 3 --config super448_200Ry --no-cpu-baseline > gpurun_out/bench448_n1_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/bench448_n1_$tag.log
grep -h '"value"' gpurun_out/bench_n${n}_$tag.log gpurun_out/bench448_n${n}_$tag.log gpurun_out/bench448_n1_$tag.log | cut -c1-400; tail -n 3 gpurun_out/bench_n${n}_$tag.log
