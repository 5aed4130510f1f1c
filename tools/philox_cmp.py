import json, os, subprocess, sys
code = r'''
import json, sys
from paper_2504_00987_b200 import capi
ctx = capi.Context(0)
out = []
for n in (24, 64, 119):
    p = capi.memetic_params(target_energy=0, max_iterations=5, rng_kind=capi.RNG_PHILOX)
    best, per = ctx.run_replicas(n, 16, 3, p)
    out.append([(r["best"].tolist(), r["best_energy"], r["iterations"]) for r in per])
print(json.dumps(out))
'''
res = []
for lib in ("paper_2504_00987_b200/lib/variants/liblabs_b200_prev_philox.so", "paper_2504_00987_b200/lib/liblabs_b200.so"):
    env = dict(os.environ, LABS_LIB_PATH=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    res.append(json.loads(r.stdout.strip().splitlines()[-1]))
print("philox stream identical:", res[0] == res[1])
