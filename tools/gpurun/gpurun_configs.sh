#!/bin/bash
# Configs 4 and 5 on one GPU: the 1512-atom 3x3x3 supercell and the 56-atom cutoff sweep.
# usage: gpurun_configs.sh tag
tag=${1:-r06}; mkdir -p gpurun_out
out=gpurun_out/configs_$tag.jsonl; : > $out
for c in sweep56_100Ry sweep56_150Ry cubic56_200Ry sweep56_250Ry sweep56_300Ry sweep56_350Ry sweep56_400Ry super448_200Ry super1512_200Ry; do
  timeout 600 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline > gpurun_out/cfg_${c}_$tag.log 2>&1
  echo "$c rc=$?" >> gpurun_out/cfg_${c}_$tag.log
  grep '"metric"' gpurun_out/cfg_${c}_$tag.log >> $out
done
python -c "
import json
for l in open('$out'):
    d = json.loads(l); c = d['config']; r = d.get('run', c)
    print(c['workload'], c['grid'], d['value'], 'ms', r['achieved_pass_tflops'], 'TF', d['segments_ms'], d['roofline']['frac'], d['e2e'] and d['e2e']['value'])
"
