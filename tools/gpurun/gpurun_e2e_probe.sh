#!/bin/bash
# e2e variants (zero-copy in/out, shard IO, pinned) at N=1 and N=2
python tools/e2e_probe.py ${1:-cubic56_200Ry} | grep "^{" | cut -c1-260
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 tools/e2e_probe.py ${1:-cubic56_200Ry} 2>&1 | grep "^{" | cut -c1-260
