#!/bin/bash
# A/B a set of library variants on one box: parity subset + bench at N=64/119.
# usage: bash tools/ab.sh pre unroll hn4 ...   (paper_2504_00987_b200/lib/variants/liblabs_b200_<v>.so)
for v in "$@"; do
  lib=$PWD/paper_2504_00987_b200/lib/variants/liblabs_b200_$v.so
  LABS_LIB_PATH=$lib timeout 600 python -m pytest -q -x -m gpu tests/test_parity_gpu.py \
      -k "tabu_walks or memetic or flip_trace or scan" 2>&1 | tail -1 | sed "s/^/$v parity: /"
done
for rep in 1 2; do
  for v in "$@"; do
    for n in 64 119; do
      LABS_LIB_PATH=$PWD/paper_2504_00987_b200/lib/variants/liblabs_b200_$v.so \
        python bench.py --quick --steps 10 --warmup 3 --n $n 2>&1 | tail -1 | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', $n, '%.4e' % d['value'])"
    done
  done
done
