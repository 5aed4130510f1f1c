#!/bin/bash
# Round-2 evidence run (one gpurun call): bench line, TTS scaling fit on the
# proven/literature optima 41..66, and the N=107 product-kernel sweep.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02.log 2>&1
tail -1 gpurun_out/bench_r02.log > gpurun_out/bench_r02_line.json
timeout 1200 python -m paper_2504_00987_b200.tts --n 41-66 --reps 12 \
    --targets paper_2504_00987_b200/data/optima_literature.txt --time-limit 60 \
    --fit 48-66 --seed 500000 --out gpurun_out/tts_fit_41_66.jsonl > gpurun_out/tts_fit.log 2>&1
tail -1 gpurun_out/tts_fit.log
timeout 1500 bash tools/sweep_n107.sh
echo evidence done
