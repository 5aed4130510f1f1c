"""One-off equivalence check: the Philox stream served from the shared-block
buffer equals the earlier per-draw implementation (same draw definition).
Usage: python tools/philox_cmp.py OLD_LIB NEW_LIB"""
import ctypes as C
import json
import os
import subprocess
import sys

CODE = r'''
import ctypes as C, json, sys
sys.path.insert(0, ".")
from paper_2504_00987_b200 import capi as k
L = C.CDLL(sys.argv[1])
L.labs_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
L.labs_run_replicas.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.POINTER(k.MemeticParams),
                                C.POINTER(k.RunResult), C.POINTER(k.RunResult), C.c_void_p, C.c_int64, C.c_void_p]
h = C.c_void_p(); assert L.labs_ctx_create(0, C.byref(h)) == 0
out = []
for n in (24, 64, 119):
    p = k.memetic_params(target_energy=0, max_iterations=5, rng_kind=k.RNG_PHILOX)
    best = k.RunResult(); per = (k.RunResult * 16)()
    assert L.labs_run_replicas(h, n, 16, 3, C.byref(p), C.byref(best), per, None, 0, None) == 0
    out.append([(list(r.best), r.best_energy, r.iterations) for r in per])
print(json.dumps(out))
'''
res = []
for lib in sys.argv[1:3]:
    r = subprocess.run([sys.executable, "-c", CODE, os.path.abspath(lib)], capture_output=True,
                       text=True)
    if r.returncode:
        sys.exit(f"{lib}: {r.stderr[-2000:]}")
    res.append(json.loads(r.stdout.splitlines()[-1]))
print("philox stream identical:", res[0] == res[1])
