#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
#   1. the bench line (no profiler),
#   2. the launch list of the same command (gpu__time_duration per launch),
#   3. one full ncu capture of the bench kernel (k_memetic, N=64), exported
#      as CSV (raw metrics, per-SASS source page); the .ncu-rep stays on the box.
# Each ncu pass follows a plain run of the same command that exited 0.
set -e
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.log 2>&1
tail -1 gpurun_out/bench_final.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_final.csv python bench.py --steps 10 --warmup 3 \
    > gpurun_out/ncu_launches.log 2>&1
python bench.py --quick --steps 1 --warmup 1 --epoch-ms 20 > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_memetic -s 1 -c 1 \
    -o /tmp/prof_final python bench.py --quick --steps 1 --warmup 1 --epoch-ms 20 \
    > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/prof_final.ncu-rep --page raw --csv > gpurun_out/prof_final_raw.csv
ncu -i /tmp/prof_final.ncu-rep --page details --csv > gpurun_out/prof_final_details.csv
ncu -i /tmp/prof_final.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_final_sass.csv
echo profile_round done
