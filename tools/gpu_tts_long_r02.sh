#!/bin/bash
# configs[2]: time to the previous best-known energy (targets_long.txt column
# 2) on one B200, 600 s limit per instance, one replica set (resident
# capacity) per instance, seed block disjoint from round 1.
mkdir -p gpurun_out
count=$(echo "${NS:-98,99,104,107,110,112}" | tr ',' '\n' | wc -l)
timeout $(( ${LIMIT:-600} * count + 300 )) python -m paper_2504_00987_b200.tts --n ${NS:-98,99,104,107,110,112} --reps 1 \
    --targets paper_2504_00987_b200/data/targets_long.txt --target-column 2 \
    --time-limit ${LIMIT:-600} --seed ${SEED:-77000000} --out gpurun_out/tts_long_r02_${TAG:-a}.jsonl \
    > gpurun_out/tts_long_r02_${TAG:-a}.log 2>&1
tail -3 gpurun_out/tts_long_r02_${TAG:-a}.log | cut -c1-600
