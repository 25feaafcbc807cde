#!/bin/bash
# 2-GPU checks: the multi-GPU pytest (p2p reduction vs oracle, bitwise vs 1 GPU), bench --gpus N self-launch
tag=${1:-n2}; n=${2:-2}; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -v -p no:cacheprovider > gpurun_out/pytest_gpu_n${n}_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_n${n}_$tag.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 tools/p2p_check.py super448_200Ry > gpurun_out/p2p448_n${n}_$tag.log 2>&1
timeout 600 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/bench_n${n}_$tag.json 2> gpurun_out/bench_n${n}_$tag.err
timeout 600 python bench.py --gpus $n --steps 10 --warmup 3 --config super448_200Ry --no-cpu-baseline > gpurun_out/bench448_n${n}_$tag.json 2>> gpurun_out/bench_n${n}_$tag.err
tail -5 gpurun_out/pytest_gpu_n${n}_$tag.log; grep "^{" gpurun_out/p2p448_n${n}_$tag.log | cut -c1-900; cut -c1-700 gpurun_out/bench_n${n}_$tag.json; cut -c1-600 gpurun_out/bench448_n${n}_$tag.json; tail -3 gpurun_out/bench_n${n}_$tag.err
