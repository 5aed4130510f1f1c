"""Attribute ncu per-SASS instruction counts to source lines.

usage: python tools/sass_lines.py <nvdisasm -gi dump of one function> <ncu sass csv> [file-filter]

Each SASS offset carries its inline chain from nvdisasm's line info; executed
warp-instructions are summed per innermost line and per outermost line that
matches the filter (default labs_memetic.cuh)."""
import collections
import csv
import re
import sys

dump, sass_csv = sys.argv[1], sys.argv[2]
filt = sys.argv[3] if len(sys.argv) > 3 else "labs_memetic.cuh"
loc_re = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
ins_re = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);")
chain = []
pending = []
off2chain = {}
for line in open(dump):
    m = loc_re.search(line)
    if m:
        pending.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    m = ins_re.search(line)
    if m:
        if pending:
            chain = pending
            pending = []
        off2chain[int(m.group(1), 16)] = (chain, m.group(2).strip())
rows = list(csv.reader(open(sass_csv)))
hdr, data = rows[1], rows[2:]
iE, iA = hdr.index("Instructions Executed"), hdr.index("Address")
base = int(data[0][iA], 16)
inner = collections.Counter()
outer = collections.Counter()
tot = 0
for r in data:
    off = int(r[iA], 16) - base
    c = int(r[iE] or 0)
    tot += c
    ch, _ = off2chain.get(off, ([("?", 0)], ""))
    inner[f"{ch[0][0]}:{ch[0][1]}"] += c
    outs = [f"{f}:{l}" for f, l in ch if filt in f]
    outer[outs[-1] if outs else "other"] += c
print("total", tot)
print("-- by outermost", filt, "line")
for k, v in outer.most_common(40):
    print(f"{v / tot:7.3%} {k}")
print("-- by innermost line")
for k, v in inner.most_common(40):
    print(f"{v / tot:7.3%} {k}")
