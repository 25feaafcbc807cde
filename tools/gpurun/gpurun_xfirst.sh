#!/bin/bash
# e2e A/B: exchange after (default) / before (KBG_XCHG_FIRST) the density pass, N = $2, config $1
c=${1:-super448_200Ry}; n=${2:-4}
for r in 1 2; do for x in 0 1; do
  KBG_XCHG_FIRST=$x KBG_PHASE_TIMING=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29544 tools/e2e_probe.py $c > gpurun_out/xf_${c}_n${n}_$x.log 2>&1
  echo "xfirst=$x"; grep "^{" gpurun_out/xf_${c}_n${n}_$x.log | head -1 | cut -c1-230; grep phases gpurun_out/xf_${c}_n${n}_$x.log | sed -n '8p'
done; done
