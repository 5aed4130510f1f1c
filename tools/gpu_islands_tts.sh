# Elite exchange vs none (both with worst-member replacement) on the long
# instances the plain 180 s sweep missed.
mkdir -p gpurun_out
python tools/islands_tts.py --n ${ISL_N:-98,99,104,107} --limit ${ISL_LIMIT:-180} --every 1 --epoch 1.0 \
  --out gpurun_out/islands_tts.jsonl > gpurun_out/islands_tts.log 2>&1
python tools/islands_tts.py --n ${ISL_N:-98,99,104,107} --limit ${ISL_LIMIT:-180} --every 0 --epoch 1.0 \
  --out gpurun_out/islands_tts.jsonl >> gpurun_out/islands_tts.log 2>&1
tail -8 gpurun_out/islands_tts.log
