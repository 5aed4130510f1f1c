#!/bin/bash
# Record attempt: time to the paper's new best energy (targets_long.txt
# column 1) for one instance, one replica set, long limit.
mkdir -p gpurun_out
count=$(echo "${NS:-98}" | tr ',' '\n' | wc -l)   # one replica set per instance, run in turn
timeout $(( ${LIMIT:-3300} * count + 300 )) python -m paper_2504_00987_b200.tts --n ${NS:-98} --reps 1 \
    --targets paper_2504_00987_b200/data/targets_long.txt --target-column 1 \
    --time-limit ${LIMIT:-3300} --seed ${SEED:-81000000} --out gpurun_out/tts_record_r02_${TAG:-a}.jsonl \
    > gpurun_out/tts_record_r02_${TAG:-a}.log 2>&1
tail -2 gpurun_out/tts_record_r02_${TAG:-a}.log | cut -c1-400
