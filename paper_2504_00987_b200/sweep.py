"""Walker-count / occupancy sweep (BASELINE configs[3]) of the product kernel
K4 (`--kernel memetic`, default) or of the bare tabu kernel K3.

K4 (labs_solver_run): W memetic replicas (reference MemeticParams, target
unreachable), one warp each; above the resident capacity the grid stays
capacity-sized and each warp serves its replicas in waves. A launch gives
every replica `--epoch-ms` of device time; flip-evaluations/s = tabu
iterations x n / launch time (CUDA events, best of --reps launches).

K3 (`labs_tabu_walks_device`): W independent walkers, one warp each, each
running `--walks` tabu_search walks back to back (walk k+1 starts from walk
k's best), reference TabuParams, starting sequences i.i.d. Bernoulli(1/2).
Reports tabu flip-evaluations/s per W (CUDA events on the library stream,
best of --reps) so the residency knee (148 SMs x resident warps/SM) shows.

    python -m paper_2504_00987_b200.sweep --n 107 --walkers 128,256,...,16384
"""
from __future__ import annotations

import argparse
import json
import sys


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=107)
    ap.add_argument("--walkers", default="128,256,512,1024,2048,4096,8192,16384")
    ap.add_argument("--walks", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--rng", choices=["mt19937_64", "philox"], default="mt19937_64")
    ap.add_argument("--kernel", choices=["memetic", "tabu"], default="memetic")
    ap.add_argument("--epoch-ms", type=float, default=50.0)
    args = ap.parse_args(argv)
    if args.kernel == "memetic":
        return sweep_memetic(args)

    import numpy as np
    import torch
    from paper_2504_00987_b200 import capi
    from paper_2504_00987_b200.sequence import random_words

    ctx = capi.Context(0)
    ext = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
    n = args.n
    kind = capi.RNG_PHILOX if args.rng == "philox" else capi.RNG_MT19937_64
    rows = []
    for W in [int(x) for x in args.walkers.split(",")]:
        words = random_words(n, W, np.random.default_rng(42 + W))
        d_start = torch.from_numpy(words.view(np.int64)).cuda()
        d_best = torch.zeros_like(d_start)
        d_e = torch.zeros(W, dtype=torch.int64, device="cuda")
        d_it = torch.zeros(1, dtype=torch.int64, device="cuda")
        d_rng = None
        if kind == capi.RNG_MT19937_64:
            d_rng = torch.zeros(W * capi.C.sizeof(capi.RngState), dtype=torch.uint8,
                                device="cuda")
            ctx.rng_seed_device(W, 42, d_rng.data_ptr())
        torch.cuda.synchronize()
        ctx.synchronize()
        best = None
        for rep in range(args.reps + 1):  # first rep warms up
            d_it.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(ext):
                e0.record(ext)
            ctx.tabu_walks_device(n, W, args.walks, d_start.data_ptr(), d_best.data_ptr(),
                                  d_e.data_ptr(), rng_kind=kind,
                                  d_rng=d_rng.data_ptr() if d_rng is not None else 0,
                                  seed=7, ctr_base=rep << 40, d_iterations=d_it.data_ptr())
            with torch.cuda.stream(ext):
                e1.record(ext)
            ctx.synchronize()
            ms = e0.elapsed_time(e1)
            rate = float(d_it.item()) * n / (ms / 1e3)
            if rep and (best is None or rate > best[0]):
                best = (rate, ms, int(d_it.item()))
        row = {"n": n, "walkers": W, "flip_evals_per_s": best[0], "ms": best[1],
               "tabu_iterations": best[2], "rng": args.rng}
        rows.append(row)
        print(json.dumps(row), flush=True)
    cap = capi.Solver.capacity(ctx, n, kind)
    print(json.dumps({"resident_warps": cap, "sm_count": ctx.sm_count}), flush=True)
    return 0


def sweep_memetic(args):
    import torch
    from paper_2504_00987_b200 import capi

    ctx = capi.Context(0)
    ext = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
    n = args.n
    kind = capi.RNG_PHILOX if args.rng == "philox" else capi.RNG_MT19937_64
    cap = capi.Solver.capacity(ctx, n, kind)
    for W in [int(x) for x in args.walkers.split(",")]:
        sv = capi.Solver(ctx, n, W, base_seed=42, params=capi.memetic_params(
            target_energy=0, rng_kind=kind))
        sv.run(epoch_seconds=args.epoch_ms / 1e3, race=False)  # init + warm-up
        best = None
        for _ in range(args.reps):
            t_before, _ = sv.counters()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(ext):
                e0.record(ext)
            sv.run(epoch_seconds=args.epoch_ms / 1e3, race=False)
            with torch.cuda.stream(ext):
                e1.record(ext)
            ctx.synchronize()
            ms = e0.elapsed_time(e1)
            t_after, _ = sv.counters()
            rate = (t_after - t_before) * n / (ms / 1e3)
            if best is None or rate > best[0]:
                best = (rate, ms, t_after - t_before)
        sv.close()
        row = {"kernel": "k_memetic", "n": n, "replicas": W, "resident_capacity": cap,
               "waves": -(-W // cap), "flip_evals_per_s": best[0], "launch_ms": best[1],
               "tabu_iterations": best[2], "epoch_ms": args.epoch_ms, "rng": args.rng}
        print(json.dumps(row), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
