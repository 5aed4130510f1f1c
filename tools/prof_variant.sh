#!/bin/bash
# ncu --set full of k_memetic for library variants (LABS_LIB_PATH), one N.
# usage: N=119 TAG=r02 bash tools/prof_variant.sh v1 v2 ...
set -e
mkdir -p gpurun_out
for v in "$@"; do
  lib=$PWD/paper_2504_00987_b200/lib/variants/liblabs_b200_$v.so
  LABS_LIB_PATH=$lib python bench.py --quick --steps 1 --warmup 1 --epoch-ms 50 --n ${N:-119} > /dev/null 2>&1
  LABS_LIB_PATH=$lib ncu --set full --clock-control none --import-source on -k regex:k_memetic -s 1 -c 1 \
      -o /tmp/pv_$v python bench.py --quick --steps 1 --warmup 1 --epoch-ms 50 --n ${N:-119} > /dev/null 2>&1
  ncu -i /tmp/pv_$v.ncu-rep --page raw --csv > gpurun_out/pv_${TAG:-x}_${v}_n${N:-119}_raw.csv
  ncu -i /tmp/pv_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/pv_${TAG:-x}_${v}_n${N:-119}_sass.csv
done
echo prof_variant done
