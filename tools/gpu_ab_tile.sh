# A/B of the memetic kernel tile width (LABS_TILE) and RNG mode; optional
# parity pass first (PARITY=1).
mkdir -p gpurun_out
if [ "${PARITY:-0}" = 1 ]; then
LABS_TILE=16 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t16_tests.log 2>&1; tail -1 gpurun_out/t16_tests.log
LABS_TILE=32 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t32_tests.log 2>&1; tail -1 gpurun_out/t32_tests.log
fi
for n in ${NS:-64}; do for t in ${TILES:-16 32}; do for r in ${RNGS:-mt19937_64 philox}; do
LABS_TILE=$t timeout 120 python bench.py --quick --steps 10 --warmup 3 --rng $r --n $n > gpurun_out/b_${n}_${t}_$r.log 2>&1
tail -1 gpurun_out/b_${n}_${t}_$r.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('n=$n T=$t', '$r', d['config']['replicas_per_gpu'], '%.4e' % d['value'], '%.4e' % d['e2e']['value'])" || tail -5 gpurun_out/b_${n}_${t}_$r.log
done; done; done
