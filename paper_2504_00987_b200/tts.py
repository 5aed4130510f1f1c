"""Time-to-target harness and scaling fit on the B200 solver.

Python face of proj/src/fit.cpp:15-182 (the C++ drop-in is
include/labsolve/fit.hpp): for each n and repetition, a fresh replica set
(disjoint seed block base + run_index * replicas, fit.cpp:30-31) races to the
target; wall time from solver creation to the first replica at the target
(or censored at the time limit); medians over uncensored samples; OLS of
log(median) vs n with Student-t 95% intervals, reported as runtime ~ a * b^n
(the paper's form). Samples are JSON lines in the
reference's format (fit.cpp:120-133).

    python -m paper_2504_00987_b200.tts --n 24-40 --reps 5 \
        --targets paper_2504_00987_b200/data/optima.txt --out tts.jsonl
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))


# ----------------------------------------------------------------- stats --
def quantile(values, q):
    if not values:
        raise ValueError("quantile of empty sample")
    if not 0.0 <= q <= 1.0:
        raise ValueError("quantile level")
    v = sorted(values)
    pos = q * (len(v) - 1)
    i = int(math.floor(pos))
    if i + 1 >= len(v):
        return v[-1]
    return v[i] + (pos - i) * (v[i + 1] - v[i])


def median_runtime_by_n(samples):
    by = {}
    for s in samples:
        if s["reachedTarget"]:
            by.setdefault(s["n"], []).append(s["runtime"])
    return {n: quantile(r, 0.5) for n, r in sorted(by.items())}


def _betacf(a, b, x):
    tiny = 1e-300
    c, d = 1.0, 1.0 - (a + b) * x / (a + 1.0)
    d = 1.0 / (d if abs(d) > tiny else tiny)
    h = d
    for m in range(1, 401):
        m2 = 2 * m
        for num in (m * (b - m) * x / ((a + m2 - 1) * (a + m2)),
                    -(a + m) * (a + b + m) * x / ((a + m2) * (a + m2 + 1))):
            d = 1.0 + num * d
            c = 1.0 + num / c
            d = 1.0 / (d if abs(d) > tiny else tiny)
            c = c if abs(c) > tiny else tiny
            h *= d * c
        if abs(d * c - 1.0) < 1e-15:
            break
    return h


def _incbeta(a, b, x):
    if x <= 0:
        return 0.0
    if x >= 1:
        return 1.0
    front = math.exp(math.lgamma(a + b) - math.lgamma(a) - math.lgamma(b) +
                     a * math.log(x) + b * math.log1p(-x))
    if x < (a + 1) / (a + b + 2):
        return front * _betacf(a, b, x) / a
    return 1.0 - front * _betacf(b, a, 1 - x) / b


def student_t_quantile(dof, p):
    """Same algorithm as csrc/host/fit.cpp (replaces Boost.Math)."""
    def cdf(t):
        tail = 0.5 * _incbeta(0.5 * dof, 0.5, dof / (dof + t * t))
        return 1.0 - tail if t >= 0 else tail
    lo, hi = -1.0, 1.0
    while cdf(lo) > p:
        lo *= 2
    while cdf(hi) < p:
        hi *= 2
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if cdf(mid) < p:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def fit_exponential(samples, n_min, n_max):
    """fit_exponential (fit.cpp:64-118)."""
    med = {n: m for n, m in median_runtime_by_n(samples).items() if n_min <= n <= n_max}
    if len(med) < 3:
        raise ValueError("fit needs at least three uncensored medians")
    xs = list(med)
    ys = [math.log(med[n]) for n in xs]
    m = len(xs)
    xm, ym = sum(xs) / m, sum(ys) / m
    sxx = sum((x - xm) ** 2 for x in xs)
    sxy = sum((x - xm) * (y - ym) for x, y in zip(xs, ys))
    slope = sxy / sxx
    icpt = ym - slope * xm
    rss = sum((y - icpt - slope * x) ** 2 for x, y in zip(xs, ys))
    dof = m - 2
    s2 = rss / dof
    se_b = math.sqrt(s2 / sxx)
    se_a = math.sqrt(s2 * (1.0 / m + xm * xm / sxx))
    t = student_t_quantile(dof, 0.975)
    return {"a": math.exp(icpt), "b": math.exp(slope),
            "a_ci": [math.exp(icpt - t * se_a), math.exp(icpt + t * se_a)],
            "b_ci": [math.exp(slope - t * se_b), math.exp(slope + t * se_b)],
            "n_min_fit": n_min, "n_max_fit": n_max, "points_used": m}


def read_targets(path, column=1):
    """n -> target energy from whitespace columns (n, E, ...); `column`
    picks which energy column (targets_long.txt: 1 = the paper's record,
    2 = the previous literature best)."""
    t = {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                cols = line.split()
                t[int(cols[0])] = int(cols[column])
    return t


# ------------------------------------------------------------------- run --
def run_tts(ctx, n_values, targets, reps=5, replicas=0, base_seed=7, time_limit=60.0,
            rng_kind=None, log=None):
    """run_tts (fit.cpp:15-41) on the device solver. replicas=0: resident
    capacity. Returns reference-format sample dicts."""
    from paper_2504_00987_b200 import capi
    rng_kind = capi.RNG_MT19937_64 if rng_kind is None else rng_kind
    out, run = [], 0
    for n in n_values:
        if n not in targets:
            raise ValueError(f"no target energy for n = {n}")
        R = replicas or capi.Solver.capacity(ctx, n, rng_kind)
        for _ in range(reps):
            seed = base_seed + run * R
            run += 1
            params = capi.memetic_params(target_energy=targets[n], max_seconds=time_limit,
                                         rng_kind=rng_kind)
            t0 = time.perf_counter()
            sv = capi.Solver(ctx, n, R, base_seed=seed, params=params)
            sv.run(race=True)
            st = sv.status()
            dt = time.perf_counter() - t0
            from paper_2504_00987_b200.sequence import encode_hex
            win = sv.results()[st["best_replica"]]
            sv.close()
            rec = {"n": n, "targetE": targets[n], "runtime": dt,
                   "reachedTarget": st["best_energy"] <= targets[n], "seed": seed,
                   "replicas": R, "bestE": st["best_energy"],
                   "bestSeq": encode_hex(win["best"], n), "bestReplica": st["best_replica"]}
            out.append(rec)
            if log:
                log(rec)
    return out


def run_tts_islands(ctx, n_values, targets, reps, replicas, base_seed, time_limit,
                    rng_kind=None, log=None, epoch_seconds=1.0):
    """run_tts over every rank of the process group (one GPU per rank; the
    island model of configs[4] without migration): sample s uses the global
    seed block base + s * R * world, rank g owns global replicas g*R + r
    (seeds base + id, proj/src/parallel.cpp:38). A target reached on any
    rank stops every rank from the device (IPC peer stop flags); runtime =
    max over ranks of creation -> stop."""
    import torch
    import torch.distributed as dist
    from paper_2504_00987_b200 import capi
    from paper_2504_00987_b200.islands import Islands
    from paper_2504_00987_b200.sequence import encode_hex
    rng_kind = capi.RNG_MT19937_64 if rng_kind is None else rng_kind
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", ctx.device)
    out, run = [], 0
    for n in n_values:
        R = replicas or capi.Solver.capacity(ctx, n, rng_kind)
        for _ in range(reps):
            seed = base_seed + run * R * world
            run += 1
            params = capi.memetic_params(target_energy=targets[n], max_seconds=time_limit + 5,
                                         rng_kind=rng_kind)
            dist.barrier()
            t0 = time.perf_counter()
            sv = capi.Solver(ctx, n, R, base_seed=seed, replica_offset=rank * R, params=params)
            isl = Islands(sv, n, k_elites=1, device=dev)
            rep = isl.run(targets[n], epoch_seconds=epoch_seconds, max_seconds=time_limit)
            dt = time.perf_counter() - t0
            t = torch.tensor([dt], dtype=torch.float64,
                             device=dev if dist.get_backend() == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e, r = rep.best_energy, rep.best_replica
            seq = ""
            if r // R == rank:
                seq = encode_hex(sv.results()[r - rank * R]["best"], n)
            seqs = [None] * world
            dist.all_gather_object(seqs, seq)
            isl.close()
            sv.close()
            rec = {"n": n, "targetE": targets[n], "runtime": float(t.item()),
                   "reachedTarget": e <= targets[n], "seed": seed, "replicas": R * world,
                   "gpus": world, "bestE": e, "bestSeq": next(x for x in seqs if x) if any(seqs)
                   else "", "bestReplica": r}
            out.append(rec)
            if log and rank == 0:
                log(rec)
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--n", "--lengths", dest="n", default="24-40", help="range a-b or comma list")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--targets", default=os.path.join(HERE, "data", "optima.txt"))
    ap.add_argument("--replicas", type=int, default=0)
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--time-limit", type=float, default=60.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--fit", default=None, help="n_min-n_max window")
    ap.add_argument("--target-column", type=int, default=1,
                    help="energy column of --targets (targets_long.txt: 2 = previous best)")
    ap.add_argument("--gpus", type=int, default=1,
                    help="island model over this many GPUs (one rank each; re-executes "
                         "under torch.distributed.run when not already under it)")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        import socket
        import torch
        if torch.cuda.device_count() < args.gpus:
            sys.stderr.write(f"tts: --gpus {args.gpus} needs {args.gpus} CUDA devices; "
                             f"{torch.cuda.device_count()} visible\n")
            return 2
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={port}", "-m", "paper_2504_00987_b200.tts"] + \
            ["--lengths" if a == "--n" else a for a in (argv if argv is not None else sys.argv[1:])]
        os.execv(sys.executable, cmd)
    if "-" in args.n:
        a, b = map(int, args.n.split("-"))
        ns = list(range(a, b + 1))
    else:
        ns = [int(x) for x in args.n.split(",")]
    from paper_2504_00987_b200 import capi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = capi.Context(local)
    targets = read_targets(args.targets, args.target_column)
    fh = open(args.out, "a") if args.out and rank == 0 else None

    def log(rec):
        line = json.dumps(rec, sort_keys=True)
        print(line, flush=True)
        if fh:
            fh.write(line + "\n")
            fh.flush()

    if world > 1:
        samples = run_tts_islands(ctx, ns, targets, args.reps, args.replicas, args.seed,
                                  args.time_limit, log=log)
        if rank != 0:
            return 0
    else:
        samples = run_tts(ctx, ns, targets, args.reps, args.replicas, args.seed,
                          args.time_limit, log=log)
    med = median_runtime_by_n(samples)
    quart = {}
    for n in sorted({s["n"] for s in samples}):
        t = [s["runtime"] for s in samples if s["n"] == n and s["reachedTarget"]]
        quart[n] = {"q1": quantile(t, 0.25), "median": quantile(t, 0.5),
                    "q3": quantile(t, 0.75), "uncensored": len(t)} if t else {"uncensored": 0}
    summary = {"medians": med, "quartiles": quart,
               "censored": sum(not s["reachedTarget"] for s in samples)}
    if args.fit:
        lo, hi = map(int, args.fit.split("-"))
        summary["fit"] = fit_exponential(samples, lo, hi)
    print(json.dumps({"summary": summary}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
