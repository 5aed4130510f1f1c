#!/bin/bash
# One ncu --set full capture of k_memetic per N (after a plain run of the
# same command exits 0), exported as raw + details + per-SASS source CSV.
# usage (under gpurun): NS_LIST="64 119" TAG=r02 bash tools/prof_kernel.sh
set -e
mkdir -p gpurun_out
for n in ${NS_LIST:-64 119}; do
  python bench.py --quick --steps 1 --warmup 1 --epoch-ms 50 --n $n > gpurun_out/plain_$n.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_memetic -s 1 -c 1 \
      -o /tmp/prof_${TAG:-x}_n$n python bench.py --quick --steps 1 --warmup 1 --epoch-ms 50 --n $n \
      > gpurun_out/ncu_full_$n.log 2>&1
  ncu -i /tmp/prof_${TAG:-x}_n$n.ncu-rep --page raw --csv > gpurun_out/prof_${TAG:-x}_n${n}_raw.csv
  ncu -i /tmp/prof_${TAG:-x}_n$n.ncu-rep --page details --csv > gpurun_out/prof_${TAG:-x}_n${n}_details.csv
  ncu -i /tmp/prof_${TAG:-x}_n$n.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${TAG:-x}_n${n}_sass.csv
done
echo prof_kernel done
