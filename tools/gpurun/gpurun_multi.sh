#!/bin/bash
# usage: gpurun_multi.sh N tag [configs]  -- strong scaling of the given configs on N GPUs (+ 1-GPU reference lines)
n=${1:-2}; tag=${2:-r01}; cfgs=${3:-"cubic56_200Ry super448_200Ry super1512_200Ry"}; mkdir -p gpurun_out
port=29511
for c in $cfgs; do
  port=$((port + 1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port \
    bench.py --gpus $n --steps 10 --warmup 3 --config $c > gpurun_out/multi_${c}_n${n}_$tag.log 2>&1
  echo "rc=$?" >> gpurun_out/multi_${c}_n${n}_$tag.log
  grep -h '"value"' gpurun_out/multi_${c}_n${n}_$tag.log | cut -c1-600
  tail -n 2 gpurun_out/multi_${c}_n${n}_$tag.log
done
