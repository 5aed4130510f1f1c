# ncu full capture of k_memetic for each tile width; exports CSV summaries
# (raw metrics + per-SASS source page) and drops the large .ncu-rep.
mkdir -p gpurun_out
for t in ${TILES:-16 32}; do
LABS_TILE=$t timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_memetic -s 1 -c 1 \
  -o /tmp/prof_t$t python bench.py --quick --steps 1 --warmup 1 --epoch-ms 20 ${BENCH_ARGS} > gpurun_out/ncu_t$t.log 2>&1
tail -1 gpurun_out/ncu_t$t.log
ncu -i /tmp/prof_t$t.ncu-rep --page raw --csv > gpurun_out/prof_t${t}_raw.csv 2>&1
ncu -i /tmp/prof_t$t.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_t${t}_sass.csv 2>&1
ncu -i /tmp/prof_t$t.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_t${t}_cuda.csv 2>&1
ls -la gpurun_out/prof_t${t}_*.csv
done
