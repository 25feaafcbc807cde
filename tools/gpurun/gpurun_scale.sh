#!/bin/bash
# strong scaling on one box: bench.py at N = 1, 2, 4 (self-launching) for 56 / 448 / 1512 atoms,
# the p2p check at 448 atoms, and the 2-rank GPU test
tag=${1:-sc}; mkdir -p gpurun_out; out=gpurun_out/scale_$tag.jsonl; : > $out
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_multi_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_multi_$tag.log
for c in cubic56_200Ry super448_200Ry super1512_200Ry; do
  for n in 1 2 4; do
    timeout 900 python bench.py --gpus $n --steps 10 --warmup 3 --config $c --no-cpu-baseline 2>> gpurun_out/scale_$tag.err | grep '"metric"' >> $out
  done
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543 tools/p2p_check.py super448_200Ry > gpurun_out/p2p448_n4_$tag.log 2>&1
tail -2 gpurun_out/pytest_multi_$tag.log
python3 - "$out" <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1])]
base = {}
for d in rows:
    c, n = d["config"]["workload"], d["n_gpus"]
    if n == 1: base[c] = (d["value"], d["e2e"]["value"])
    b = base.get(c, (None, None))
    eff = lambda x, y: round(x / (n * y), 3) if x and y else None
    print(c, n, d["value"], d["e2e"]["value"], "eff_dev", eff(b[0], d["value"]), "eff_e2e", eff(b[1], d["e2e"]["value"]), d["segments_ms"])
PY
grep "^{" gpurun_out/p2p448_n4_$tag.log | cut -c1-300
