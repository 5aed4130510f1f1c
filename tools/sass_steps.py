"""Static size of k_memetic's tabu step loop(s): for each CREDUX.MIN (the
step's argmin), the innermost backward branch around it delimits the step
body; prints its instruction count and op mix.
usage: cuobjdump -sass -fun <k_memetic mangled> lib.o > f.sass;
python tools/sass_steps.py f.sass [index-to-print]"""
import re
import sys

ins = []
for l in open(sys.argv[1]):
    m = re.search(r"/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for c, (ca, t) in enumerate(ins):
    if "CREDUX" not in t:
        continue
    best = None
    for k in range(c, len(ins)):
        m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)", ins[k][1])
        if m and "BRA.DIV" not in ins[k][1]:
            tgt = int(m.group(1), 16)
            if tgt <= ca and tgt in addr:
                best = (addr[tgt], k)
                break
    if best and best not in loops:
        loops.append(best)
for n, (a, b) in enumerate(loops):
    body = ins[a:b + 1]
    ops = [t.split()[1] if t.startswith("@") else t.split()[0] for _, t in body]
    print(f"[{n}] {ins[a][0]:x}-{ins[b][0]:x}: {len(body)} instrs, "
          f"LDS={sum(o.startswith('LDS') for o in ops)}, STS={sum(o.startswith('STS') for o in ops)}, "
          f"VOTE={sum('VOTE' in o for o in ops)}, CALL={sum(o.startswith('CALL') for o in ops)}")
if len(sys.argv) > 2:
    a, b = loops[int(sys.argv[2])]
    for off, t in ins[a:b + 1]:
        print(f"{off:6x}  {t}")
