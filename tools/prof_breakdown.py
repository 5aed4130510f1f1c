"""Per-tabu-step instruction breakdown of k_memetic from an ncu source page:
all executed warp-instructions / CREDUX executions, split into the main
body's step loop (the hottest blocks) and the rest, and the out-of-line
subroutines (CALL targets) with their call counts.
usage: python tools/prof_breakdown.py gpurun_out/prof_TAG_nN_sass.csv"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
ins = [(int(r[iA], 16), r[iS].strip(), int(r[iE] or 0)) for r in data if r[iA]]
steps = sum(c for _, s, c in ins if "CREDUX" in s)
tot = sum(c for _, _, c in ins)
calls = {}
for a, s, c in ins:
    m = re.search(r"CALL\.REL\.NOINC\s+0x([0-9a-f]+)", s)
    if m:
        t = int(m.group(1), 16)
        calls[t] = calls.get(t, 0) + c
ents = sorted(calls)
first_sub = ents[0] if ents else None
main = [(a, s, c) for a, s, c in ins if first_sub is None or a < first_sub]
# step loop: instructions executed at least steps/4 times (the two unrolled
# bodies each run ~steps/2 times) in the main body
loop = [(a, s, c) for a, s, c in main if c >= steps // 4]
rest = [(a, s, c) for a, s, c in main if c < steps // 4]
print(f"all: {tot / steps:.1f} warp-instructions per tabu step ({steps} steps)")
print(f"  step loop: {sum(c for *_, c in loop) / steps:.1f} ({len(loop)} static)")
print(f"  rest of the main body: {sum(c for *_, c in rest) / steps:.1f}")
base = ins[0][0]
for t in ents:
    nxt = [e for e in ents if e > t]
    hi = nxt[0] if nxt else 1 << 62
    n = sum(c for a, _, c in ins if t <= a < hi)
    print(f"  sub +{t - base:x}: {calls[t]} calls, {n / steps:.2f} per step")
