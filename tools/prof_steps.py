"""Dynamic instructions per tabu step of k_memetic from an ncu source page
(per-SASS 'Instructions Executed'): steps = executions of CREDUX.MIN (one
argmin per step); the step loop = the address range [first, last] of the
hottest CREDUX-containing loop, found as every instruction whose execution
count is >= half the CREDUX count and lies between the loop's bounds.
usage: python tools/prof_steps.py gpurun_out/prof_TAG_nN_sass.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1] if "Address" not in rows[0] else rows[0]
data = rows[2:] if hdr is rows[1] else rows[1:]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
ins = [(int(r[iA], 16) if r[iA].startswith("0x") else int(r[iA]), r[iS], int(r[iE] or 0))
       for r in data if r[iA]]
total = sum(c for _, _, c in ins)
cred = [(a, c) for a, src, c in ins if "CREDUX" in src and c > 0]
steps = sum(c for _, c in cred)
print(f"executed warp-instructions {total}, tabu steps (CREDUX executions) {steps}, "
      f"all instructions per step {total / steps:.1f}")
hot = max(cred, key=lambda x: x[1])
lo = min(a for a, _ in cred if _ > hot[1] // 4)
hi = max(a for a, _ in cred if _ > hot[1] // 4)
# extend the range to the loop: instructions executed at least steps/4 times
# around the hot CREDUXes
idx = {a: i for i, (a, _, _) in enumerate(ins)}
i0, i1 = idx[lo], idx[hi]
thr = min(c for a, c in cred if c > hot[1] // 4) // 2
while i0 > 0 and ins[i0 - 1][2] >= thr:
    i0 -= 1
while i1 + 1 < len(ins) and ins[i1 + 1][2] >= thr:
    i1 += 1
loop = ins[i0:i1 + 1]
lt = sum(c for _, _, c in loop)
print(f"step loop {loop[0][0]:x}-{loop[-1][0]:x}: {len(loop)} static, {lt / steps:.1f} "
      f"executed per step ({lt / total:.1%} of all)")
ops = {}
for _, src, c in loop:
    op = src.split()[1] if src.startswith("@") else src.split()[0]
    op = op.split(".")[0]
    ops[op] = ops.get(op, 0) + c
print("per step:", ", ".join(f"{k} {v / steps:.1f}" for k, v in
                             sorted(ops.items(), key=lambda kv: -kv[1])[:16]))
