#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
#   1. the bench line (no profiler),
#   2. the launch list of the same command (gpu__time_duration per launch),
#   3. one full ncu capture of the timed bench launch (k_memetic) at N=64 and
#      N=119 (tools/prof_kernel.sh), exported as raw / details / source CSV.
# Each ncu pass follows a plain run of the same command that exited 0.
set -e
mkdir -p gpurun_out
TAG=${TAG:-final}
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
tail -1 gpurun_out/bench_$TAG.log > gpurun_out/bench_${TAG}_line.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 10 --warmup 3 \
    > gpurun_out/ncu_launches_$TAG.log 2>&1
NS_LIST="64 119" TAG=$TAG bash tools/prof_kernel.sh
echo profile_round done
