#!/bin/bash
# A/B of library variants (tools/build_variants.sh) on one box: kernel times, 3 alternating rounds
# usage: [CONFIG=..] [KERNELS=density,h_accumulate,pass] gpurun_ab.sh tag variant...
tag=$1; shift; mkdir -p gpurun_out; out=gpurun_out/ab_$tag.log; : > $out
for r in 1 2 3; do
  for v in "$@"; do
    KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/$v/libkbgrid.so timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 ${CONFIG:+--config $CONFIG} ${KERNELS:+--kernels $KERNELS} 2>&1 | sed "s/^/$v /" >> $out
  done
done
python3 - "$out" <<'PY'
import json,sys,collections
d=collections.defaultdict(list)
for l in open(sys.argv[1]):
    v,_,j=l.partition(' ')
    if j.startswith('{'):
        r=json.loads(j)
        if 'kernel' in r: d[(v,r['kernel'])].append(r['median_ms'])
        else:
            for k,x in r.items():
                if k.endswith('_median_ms'): d[(v,'pass '+'>'.join(r['pass_order'])+' '+k[:-10])].append(x)
for k,x in sorted(d.items()): print(k, x, min(x))
PY
