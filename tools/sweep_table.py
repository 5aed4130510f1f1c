"""configs[3] table: N=107 replica sweep of k_memetic (throughput from the
plain run, counters from one ncu launch per point).
usage: python tools/sweep_table.py profiles/r02_sweep_n107 > profiles/r02_sweep_n107.md"""
import csv
import json
import sys

pre = sys.argv[1]
rows = [json.loads(l) for l in open(pre + ".jsonl") if l.startswith("{") and "replicas" in l]
print("| replicas | waves | flip-evals/s | issue active | warps active | ALU pipe | FMA pipe | "
      "LSU pipe | shared wavefronts / flip-eval | bank-conflicted | DRAM bytes / flip-eval |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    W = r["replicas"]
    m = {}
    for line in csv.reader(l for l in open(f"{pre}_ncu_{W}.csv") if l.startswith('"')):
        if len(line) > 14 and line[12] != "Metric Name":
            m[line[12]] = float(line[14].replace(",", ""))
    # the ncu launch is its own run: flip-evals from its JSON line
    js = [json.loads(l) for l in open(f"{pre}_ncu_{W}.csv") if l.startswith("{")]
    evals = js[0]["tabu_iterations"] * 107 if js else None
    wf = m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    bc = m.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    dram = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    print(f"| {W} | {r['waves']} | {r['flip_evals_per_s']:.3e} | "
          f"{m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} % | "
          f"{m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} % | "
          f"{m.get('sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 0):.1f} % | "
          f"{m.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 0):.1f} % | "
          f"{m.get('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 0):.1f} % | "
          f"{wf / evals:.2f} | {bc / wf:.1%} | {dram / evals:.4f} |")
