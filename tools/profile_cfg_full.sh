#!/bin/bash
# ncu --set full captures of the config-3 (1-D Chebyshev, split heavy segments) and config-4
# (2-D polar) apply kernels, one launch each, summarised ON the box (raw metrics + executed
# instruction / stall mix) so only text comes back -> gpurun_out/
TAG=${1:-r02}
export PYTHONPATH=.
for c in ${CFGS:-3 4}; do
  if [ $c = 3 ]; then K="k_spread|k_gather|k_pass|ring::"; else K="k_spread_line|k_line_fix|k_gather_2d|k_transpose_f|k_trunc_deconv|k_deconv_pad"; fi
  ncu --set full --import-source on --clock-control none -k regex:"$K" -c 8 \
      -o /tmp/cfg${c}_full -f python tools/cfg_apply_time.py $c c128 > gpurun_out/ncu_cfg${c}_${TAG}.log 2>&1
  python tools/ncu_summary.py raw /tmp/cfg${c}_full.ncu-rep > gpurun_out/cfg${c}_ncu_${TAG}.txt 2>&1
  ncu -i /tmp/cfg${c}_full.ncu-rep --page source --csv --print-source sass > /tmp/cfg${c}_sass.csv 2>/dev/null
  python tools/sass_mix.py /tmp/cfg${c}_sass.csv > gpurun_out/cfg${c}_sassmix_${TAG}.txt 2>&1
  ncu -i /tmp/cfg${c}_full.ncu-rep --page details > gpurun_out/cfg${c}_details_${TAG}.txt 2>&1
done
for a in ${TIMES-"3 c128" "4 c128" "5 c64"}; do
  set -- $a
  python tools/cfg_apply_time.py $1 $2 >> gpurun_out/cfg_times_${TAG}.txt 2>&1
done
echo done
