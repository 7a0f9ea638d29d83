#!/bin/bash
# A/B timing of library builds / knobs on one B200 (through gpurun from the repo root):
#   tools/ab.sh "name:ENV=VAL ENV2=VAL" ...   (INFT_LIB=exp/lib_x.so selects a build)
# prints per-stage ms per launch of the default bench workload for each variant
for v in "$@"; do
  n=${v%%:*}; e=${v#*:}
  env $e python bench.py --no-cpu-baseline --no-e2e --no-configs --steps 10 --warmup 3 > gpurun_out/ab_$n.log 2>&1
  tail -1 gpurun_out/ab_$n.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
    print('$n', round(d['ms_per_step'],4), {k:round(v['ms_per_launch'],4) for k,v in d['stages'].items()})
except Exception as ex:
    print('$n', 'FAILED', ex)
"
done
