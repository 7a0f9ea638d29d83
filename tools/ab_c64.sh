#!/bin/bash
# complex64 A/B of library builds / knobs (config 5 c64 bench stages + config 3 c64 apply):
#   tools/ab_c64.sh "name:ENV=VAL ..." ...   (INFT_LIB=exp/lib_x.so selects a build)
for v in "$@"; do
  n=${v%%:*}; e=${v#*:}
  env $e python bench.py --prec c64 --no-cpu-baseline --no-e2e --no-configs --steps 10 --warmup 3 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$n', round(d['ms_per_step'],4), {k:round(v['ms_per_launch'],4) for k,v in d['stages'].items()})
except Exception as ex:
    print('$n FAILED', ex)"
  env $e PYTHONPATH=. python tools/cfg_apply_time.py 3 c64 2>&1 | tail -1
done
