"""Static per-step instruction count of k_memetic's unrolled tabu step bodies
(SASS between consecutive CREDUX.MIN of one policy instantiation).
usage: cuobjdump -sass -fun <k_memetic mangled> lib.o > f.sass; python tools/sass_steps.py f.sass"""
import re
import sys

lines = [l for l in open(sys.argv[1]) if re.search(r"/\*[0-9a-f]+\*/\s+\S", l)]
ins = []
for l in lines:
    m = re.search(r"/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
idx = [i for i, (_, t) in enumerate(ins) if "CREDUX" in t]
for a, b in zip(idx[0::2], idx[1::2]):
    body = ins[a:b]
    ops = [t.split()[0] if not t.startswith("@") else t.split()[1] for _, t in body]
    vote = any("VOTE" in o for o in ops)
    setp = sum(o.startswith("ISETP") for o in ops)
    print(f"{ins[a][0]:x}: {len(body)} instrs, vote={vote}, ISETP={setp}, LDS={sum(o.startswith('LDS') for o in ops)}, STS={sum(o.startswith('STS') for o in ops)}")
if len(sys.argv) > 2:
    a, b = idx[int(sys.argv[2]) * 2], idx[int(sys.argv[2]) * 2 + 1]
    for off, t in ins[a:b]:
        print(f"{off:6x}  {t}")
