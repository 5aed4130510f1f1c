#!/bin/bash
# Round-2: TTS scaling fit with 40 disjoint samples per n (44..66), then the
# island-exchange study with the reference replacement policy: no exchange
# vs sparse migration (top-4 every 30 s) at equal wall time (150 s) on the
# long instances (previous best-known targets).
mkdir -p gpurun_out
timeout 1500 python -m paper_2504_00987_b200.tts --n 44-66 --reps 40 \
    --targets paper_2504_00987_b200/data/optima_literature.txt --time-limit 60 \
    --fit 52-66 --seed 9000000 --out gpurun_out/tts_fit40_44_66.jsonl > gpurun_out/tts_fit40.log 2>&1
tail -1 gpurun_out/tts_fit40.log | cut -c1-400
for every in 0 30; do
  timeout 900 python tools/islands_tts.py --n 98,99,104,107 --limit 150 --every $every --epoch 1.0 \
      --k 4 --replacement random --seed 11 --out gpurun_out/islands_r02_every$every.jsonl \
      > gpurun_out/islands_r02_every$every.log 2>&1
  tail -4 gpurun_out/islands_r02_every$every.log
done
echo tts_islands done
