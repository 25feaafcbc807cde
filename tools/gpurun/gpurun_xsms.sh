#!/bin/bash
# exchange next to the density pass (--xsms / KBG_OPT_EXCHANGE_SMS): bench at N = 2, 4 and the p2p check
out=gpurun_out/xsms_${1:-a}.jsonl; : > $out
for c in cubic56_200Ry super448_200Ry; do for n in 2 4; do for x in 0 4 8 16; do
  timeout 600 python bench.py --gpus $n --steps 10 --warmup 3 --config $c --no-cpu-baseline --xsms $x 2>/dev/null | grep '"metric"' | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'config': d['config']['workload'], 'n': d['n_gpus'], 'xsms': $x, 'value': d['value'], 'e2e': d['e2e']['value'], 'seg': d['segments_ms']}))" >> $out
done; done; done
cat $out
P2P_XSMS=8 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29545 tools/p2p_check.py super448_200Ry 2>&1 | grep "^{" | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('exchange_sms','ok','same_bits_all_ranks','bitwise_equal_single_gpu','grid_pass_h_vs_p2p','dm_asymmetry_detected_ranks')})"
