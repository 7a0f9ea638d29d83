#!/bin/bash
# Per-config kernel launch lists (ncu gpu__time_duration, cold/serialised) for configs 1-5 and
# the complex64 variant of config 5, plus the tools/all_configs.py table -> gpurun_out/
set -e
export PYTHONPATH=.
python tools/all_configs.py > gpurun_out/allcfg_r01.txt 2>&1
for a in "1 c128" "2 c128" "3 c128" "4 c128" "5 c64"; do
  set -- $a
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_cfg$1_$2.csv \
      python tools/cfg_apply_time.py $1 $2 > /dev/null 2>&1
done
echo done
