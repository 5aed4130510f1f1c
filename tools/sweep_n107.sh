#!/bin/bash
# configs[3]: N=107 replica-count sweep of the product kernel k_memetic, with
# one ncu launch per point (pipe utilisation, shared wavefronts and bank
# conflicts, achieved occupancy, DRAM bytes, issue activity).
# usage (under gpurun): bash tools/sweep_n107.sh
mkdir -p gpurun_out
W="128,256,512,1024,2048,3552,4096,8192,16384"
python -m paper_2504_00987_b200.sweep --kernel memetic --n 107 --walkers $W --reps 3 \
    --epoch-ms 50 > gpurun_out/sweep_n107.jsonl 2>&1
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
sm__warps_active.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,\
l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,\
l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,\
dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,\
sm__throughput.avg.pct_of_peak_sustained_elapsed
for w in ${W//,/ }; do
  ncu --metrics $M --clock-control none -k regex:k_memetic -s 1 -c 1 --csv \
      python -m paper_2504_00987_b200.sweep --kernel memetic --n 107 --walkers $w --reps 1 \
      --epoch-ms 20 > gpurun_out/sweep_n107_ncu_$w.csv 2> gpurun_out/sweep_n107_ncu_$w.err
done
echo sweep done
