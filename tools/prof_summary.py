"""Summarise an ncu export pair (raw CSV + per-SASS source CSV) of k_memetic:
issue/occupancy/stall mix, per-step instruction counts and the hottest
instructions. usage: python tools/prof_summary.py gpurun_out/prof_t16"""
import collections
import csv
import sys

pre = sys.argv[1]
rows = list(csv.reader(open(pre + "_raw.csv")))
d = dict(zip(rows[0], rows[2]))
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]
for k in keys:
    print(k, d.get(k))
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
      and v.replace(".", "", 1).isdigit()}
tot = sum(st.values())
print("stalls", [(k, round(v / tot, 3)) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]])
rows = list(csv.reader(open(pre + "_sass.csv")))
hdr, data = rows[1], rows[2:]
iE, iS, iW = (hdr.index("Instructions Executed"), hdr.index("Source"),
              hdr.index("Warp Stall Sampling (All Samples)"))
cnt = [int(r[iE] or 0) for r in data]
tot = sum(cnt)
c = collections.Counter(cnt)
print("kernel instrs", len(data), "executed", tot)
print("top count classes", [(v, k, round(v * k / tot, 3)) for v, k in
                            sorted(c.items(), key=lambda kv: -kv[0] * kv[1])[:8]])
