#!/bin/bash
# kbg_grid_pass phase timelines (KBG_PHASE_TIMING) at N = 1 and N = $2 for config $1
c=${1:-cubic56_200Ry}; n=${2:-2}
KBG_PHASE_TIMING=1 python tools/e2e_probe.py $c > gpurun_out/phase_${c}_n1.log 2>&1
KBG_PHASE_TIMING=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29544 tools/e2e_probe.py $c > gpurun_out/phase_${c}_n$n.log 2>&1
for f in gpurun_out/phase_${c}_n1.log gpurun_out/phase_${c}_n$n.log; do grep "^{" $f | cut -c1-230; grep phases $f | sed -n '8p;9p'; done
