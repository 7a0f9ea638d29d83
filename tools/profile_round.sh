#!/bin/bash
# Round profile on one B200 (run through gpurun from the repo root):
#   1. the default bench line (no profiler), 2. the ncu launch list of a short bench run,
#   3. one `ncu --set full` capture of the six apply kernels of one step.
# Outputs land in gpurun_out/ (scratch); summarise into profiles/ with tools/ncu_summary.py.
set -e
TAG=${1:-r02}
python bench.py > gpurun_out/bench_${TAG}.log 2>&1
tail -1 gpurun_out/bench_${TAG}.log > gpurun_out/bench_${TAG}.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/ncu_launch_${TAG}.log 2>&1
# skip the setup kernels: capture the first six launches of the apply kernels
ncu --set full --import-source on --clock-control none \
    -k regex:"k_pass_|k_spread|k_gather|ring::" -c 6 -o gpurun_out/full_${TAG} -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/ncu_full_${TAG}.log 2>&1
echo done
