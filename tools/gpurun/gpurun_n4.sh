#!/bin/bash
# 4-GPU strong scaling through bench.py's self-launch (56 / 448 / 1512 atoms) + the p2p check at 448 atoms
tag=${1:-n4}; n=${2:-4}; mkdir -p gpurun_out
for c in cubic56_200Ry super448_200Ry super1512_200Ry; do
  timeout 900 python bench.py --gpus $n --steps 10 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/bench_${c}_n${n}_$tag.json 2>> gpurun_out/bench_n${n}_$tag.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29543 tools/p2p_check.py super448_200Ry > gpurun_out/p2p448_n${n}_$tag.log 2>&1
for c in cubic56_200Ry super448_200Ry super1512_200Ry; do cut -c1-200 gpurun_out/bench_${c}_n${n}_$tag.json; done
grep "^{" gpurun_out/p2p448_n${n}_$tag.log | cut -c1-400; tail -3 gpurun_out/bench_n${n}_$tag.err
