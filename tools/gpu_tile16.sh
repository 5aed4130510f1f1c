#!/bin/bash
# T=16 tiles (two replicas per warp) vs T=32 with the current step, N=64/32.
for n in 64 32; do for t in 32 16; do
  LABS_TILE=$t timeout 300 python bench.py --quick --steps 10 --warmup 3 --n $n > gpurun_out/t_${n}_$t.log 2>&1
  tail -1 gpurun_out/t_${n}_$t.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('n=$n T=$t', d['config']['replicas_per_gpu'], '%.4e' % d['value'])" || tail -3 gpurun_out/t_${n}_$t.log
done; done
LABS_TILE=16 timeout 900 python -m pytest -q -x -m gpu tests/test_parity_gpu.py tests/test_solver_gpu.py 2>&1 | tail -1
