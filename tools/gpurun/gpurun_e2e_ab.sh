#!/bin/bash
# e2e (host-pointer grid pass) A/B of library variants, alternating, 3 rounds
for r in 1 2 3; do for v in "$@"; do
  KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/$v/libkbgrid.so timeout 300 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['segments_ms'], 'e2e', d['e2e']['value'])"
done; done
