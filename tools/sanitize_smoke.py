"""Small end-to-end workload for compute-sanitizer (racecheck / memcheck /
synccheck, one tool per run): every kernel family on tiny inputs.

    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_00987_b200 import capi  # noqa: E402
from paper_2504_00987_b200.sequence import random_words  # noqa: E402


def main():
    ctx = capi.Context(0)
    rs = np.random.default_rng(1)
    for n in (5, 33, 64, 100, 200):
        w = random_words(n, 4, rs)
        ctx.build_state(n, w)
        ctx.flip_trace(n, w, rs.integers(0, n, size=(4, 5)))
        ctx.scan(n, w, rs.integers(0, 2, size=(4, n)), capi.rng_states(range(4)))
        ctx.tabu_walks(n, w, capi.rng_states(range(4)), trace=True)
    ctx.memetic(24, 3, capi.memetic_params(max_iterations=3))
    ctx.run_replicas(40, 8, 1, capi.memetic_params(max_iterations=2))
    p = capi.memetic_params(max_iterations=2, rng_kind=capi.RNG_PHILOX,
                            crossover=capi.CROSSOVER_ONE_POINT, replacement=capi.REPLACE_WORST)
    ctx.run_replicas(70, 8, 1, p)
    ctx.exhaustive_optimum(18)
    ctx.local_optima(12)
    ctx.synchronize()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
