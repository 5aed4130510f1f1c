#!/bin/bash
# A/B library variants on one box: bench at N=64 and N=119 (interleaved,
# REPS rounds), optional parity subset per variant (PARITY=1).
# usage: bash tools/ab.sh base ten ...  (paper_2504_00987_b200/lib/variants/liblabs_b200_<v>.so)
mkdir -p gpurun_out
if [ "${PARITY:-0}" = 1 ]; then
for v in "$@"; do
  lib=$PWD/paper_2504_00987_b200/lib/variants/liblabs_b200_$v.so
  LABS_LIB_PATH=$lib timeout 900 python -m pytest -q -x -m gpu tests/test_parity_gpu.py tests/test_solver_gpu.py \
      2>&1 | tail -1 | sed "s/^/$v parity: /"
done
fi
for rep in $(seq ${REPS:-2}); do
  for v in "$@"; do
    for n in ${NS:-64 119}; do
      LABS_LIB_PATH=$PWD/paper_2504_00987_b200/lib/variants/liblabs_b200_$v.so \
        timeout 300 python bench.py --quick --steps 10 --warmup 3 --n $n ${BENCH_ARGS:-} > gpurun_out/ab_$v_$n.log 2>&1
      tail -1 gpurun_out/ab_$v_$n.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', $n, d['config']['replicas_per_gpu'], '%.4e' % d['value'])" || tail -3 gpurun_out/ab_$v_$n.log
    done
  done
done
