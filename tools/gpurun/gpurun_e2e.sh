mkdir -p gpurun_out; out=gpurun_out/e2e_$1.log; : > $out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 2 >> $out
for v in "" "KBG_NO_ZERO_COPY_OUT=1" "KBG_NO_ZERO_COPY=1 KBG_NO_ZERO_COPY_OUT=1"; do
  for c in cubic56_200Ry super448_200Ry; do
    env $v timeout 300 python bench.py --steps 20 --warmup 5 --config $c --no-cpu-baseline 2>&1 | grep '"metric"' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], d['value'], d['segments_ms'], 'e2e', d['e2e']['value'])" >> $out
  done
done
cat $out
