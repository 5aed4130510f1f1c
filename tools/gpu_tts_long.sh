# configs[2]: time to the previous best-known energy for every long instance
# of the paper's table (one replica set of resident capacity per n).
mkdir -p gpurun_out
python -m paper_2504_00987_b200.tts --n ${TTS_N:-92,98,99,104,106,107,108,109,110,112,113,114,116,118,119,120} \
  --reps ${TTS_REPS:-1} --targets paper_2504_00987_b200/data/targets_long.txt --target-column 2 \
  --time-limit ${TTS_LIMIT:-180} --seed ${TTS_SEED:-11} --out gpurun_out/tts_long_oldE.jsonl > gpurun_out/tts_long.log 2>&1
tail -3 gpurun_out/tts_long.log
