#!/usr/bin/env python3
"""bench.py — tabu flip-evaluations/s of the B200 memetic tabu search (LABS).

Workload (BASELINE.json configs[1]): LABS N=64 on one B200, one warp per
replica/walker, replicas = device resident capacity, reference MemeticParams
(K=100, p_comb=0.9, p_mutate=1/N, tenure 0.10/0.12), target unreachable so
every replica keeps searching. A "step" is one labs_solver_run launch: every
replica advances its memetic_tabu loop for `--epoch-ms` of device time
(population, RNG and best stay resident in HBM between steps). One
flip-evaluation = the dE of one candidate flip in one tabu iteration (N per
iteration).

  value   flip-evals/s, device-resident, CUDA events on the solver stream,
          L2 flushed (256 MiB write) between timed steps, max over ranks.
  e2e     same metric through the reference-facing C-ABI call
          labs_run_replicas (host buffers in and out, allocation, seeding,
          population init and result copy-back inside the timed region).
  cpu_baseline   the reference's own tabu_search (oracle/_ref, unmodified
          sources) on every host core for --cpu-seconds.
  tts     time to the best-known energy (N=64 -> 208) on this GPU: >= 10
          samples from disjoint seed blocks base + run * R (fit.cpp:30-31),
          median / Q1 / Q3 / censored count, the winning sequence per sample;
          cpu_tts: the reference's own run_replicas (oracle/_ref) on every
          host core racing to the same target, censored at a stated limit.

--impl reference runs the reference's multithreaded CPU tabu_search on the
host cores with the same metric (rank 0 only under torchrun).
Multi-GPU: `--gpus N` (N > 1) re-executes itself under torch.distributed.run
with N ranks (one per GPU) unless it already runs under torchrun; each rank
runs its own replica set (global replica ids rank*R + r, seeds base + id);
weak scaling, no data-path collective. The island model (elite allgather) is
exercised by --islands.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time


ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

OPS_PER_FLIP_EVAL = 13  # int32 ops per candidate per tabu iteration
TARGETS = {32: 64, 64: 208}  # Packebusch & Mertens 2016 optima
PAPER_A100_FIT = (8.23e-8, 1.313)  # TTS(N) = a * b^N s


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", "--length", dest="n", type=int, default=64)
    ap.add_argument("--epoch-ms", type=float, default=100.0)
    ap.add_argument("--rng", choices=["mt19937_64", "philox"], default="mt19937_64")
    ap.add_argument("--replicas", type=int, default=0, help="0 = resident capacity")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--tts-samples", type=int, default=12,
                    help="disjoint-seed TTS samples at N=64 (0 = skip)")
    ap.add_argument("--tts-limit", type=float, default=20.0)
    ap.add_argument("--cpu-tts-seconds", type=float, default=20.0,
                    help="censoring limit of the reference CPU run_replicas TTS")
    ap.add_argument("--islands", type=int, default=0,
                    help="elite exchange every this many steps (0 = off)")
    ap.add_argument("--quick", action="store_true", help="skip cpu baseline and TTS")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def maybe_spawn(args):
    """`--gpus N` outside torchrun: re-exec under torch.distributed.run with
    N ranks, after checking that N devices are visible (fail loudly)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices; "
                             f"{have} visible\n")
            sys.exit(2)
    # torchrun's own parser would take "--n" for an abbreviation of one of its
    # options: pass the sequence length as --length
    fwd = ["--length" if a == "--n" else ("--length=" + a[4:] if a.startswith("--n=") else a)
           for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + fwd
    sys.stderr.write("bench.py: launching " + " ".join(cmd[1:6]) + "\n")
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def admissible_fraction(n: int, walks: int = 200) -> float:
    """Mean fraction of the N candidates that are admissible (not tabu) per
    tabu iteration — the share the reference actually scores
    (tabu.cpp:43-44) — from oracle walks of random starts."""
    from oracle.pyoracle import Oracle
    o = Oracle()
    adm, tot = 0, 0
    for w in range(walks):
        start = o.random_sequence(n, o.rng(7000 + w))
        out = o.tabu(n, start, o.rng(9000 + w), trace=True)
        expiry = [0] * n
        for (t, pos, _e, tenure, _fb) in out["steps"]:
            adm += sum(1 for j in range(n) if expiry[j] < t)
            tot += n
            expiry[pos] = t + tenure
    return adm / tot


def cpu_reference_throughput(n: int, seconds: float):
    """The reference's tabu_search on every host core (or the oracle port)."""
    from oracle.pyoracle import Oracle, Reference, reference_available
    threads = os.cpu_count() or 1
    if reference_available():
        it, walks, el = Reference().tabu_throughput(n, threads, seconds)
        kind = "reference"
    else:
        it, walks, el = Oracle().tabu_throughput(n, threads, seconds)
        kind = "port"
    return {"value": it * n / el, "unit": "flip-evals/s", "cores": threads, "kind": kind,
            "cpu_model": cpu_model(),
            "sample": f"{walks} tabu_search walks from Sequence::random({n}), "
                      f"{threads} threads x {seconds:.0f} s, TabuParams{{0.10,0.12}}"}


def cpu_reference_tts(n: int, target: int, seconds: float, base_seed: int = 50_000):
    """The reference's own run_replicas (oracle/_ref, threaded, replicas =
    host cores) racing to `target`, censored at `seconds` (run_tts,
    fit.cpp:15-41)."""
    from oracle.pyoracle import Reference, reference_available
    threads = os.cpu_count() or 1
    if not reference_available():
        return {"unavailable": "oracle/_ref not built"}
    t0 = time.perf_counter()
    best, _ = Reference().run_replicas(n, threads, base_seed, threaded=True,
                                       target_energy=target, max_seconds=seconds)
    dt = time.perf_counter() - t0
    reached = best["best_energy"] <= target
    return {"n": n, "target": target, "replicas": threads, "cores": threads,
            "cpu_model": cpu_model(), "limit_s": seconds, "runtime_s": dt,
            "reachedTarget": reached, "censored": not reached,
            "bestE": best["best_energy"], "seed": base_seed, "kind": "reference"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    per_step = max(1.0, min(5.0, 60.0 / max(args.steps + args.warmup, 1)))
    for _ in range(args.warmup):
        cpu_reference_throughput(args.n, min(per_step, 1.0))
    vals = []
    total_evals, total_t = 0.0, 0.0
    for _ in range(args.steps):
        r = cpu_reference_throughput(args.n, per_step)
        vals.append(r)
        total_evals += r["value"] * per_step
        total_t += per_step
    v = total_evals / total_t
    line = {"metric": "tabu flip-evals/sec", "value": v, "unit": "flip-evals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"LABS N={args.n} tabu_search throughput, reference CPU",
                       "n": args.n},
            "impl": "reference",
            "cpu_baseline": {**vals[-1], "value": v},
            "e2e": {"value": v, "unit": "flip-evals/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    maybe_spawn(args)
    world, rank, local = dist_setup()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        sys.stderr.write(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}\n")
        sys.exit(2)
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    from paper_2504_00987_b200 import capi

    # LABS_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0 with gloo
    # collectives, to exercise the multi-rank code path on a one-GPU box; the
    # ranks' kernels never wait on one another, and the number is not a
    # scaling measurement.
    one_dev = os.environ.get("LABS_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    if torch.cuda.device_count() <= local:
        sys.stderr.write(f"bench.py: rank {rank} needs cuda:{local}; "
                         f"{torch.cuda.device_count()} device(s) visible\n")
        sys.exit(2)
    torch.cuda.set_device(local)
    cdev = "cpu" if one_dev else f"cuda:{local}"  # collective tensors
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        sys.stderr.write(f"bench.py: rank {rank}/{world} on cuda:{local}, communicator "
                         f"up (backend {dist.get_backend()})\n")
    ctx = capi.Context(local)
    ext = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    n = args.n
    rng_kind = capi.RNG_PHILOX if args.rng == "philox" else capi.RNG_MT19937_64
    cap = capi.Solver.capacity(ctx, n, rng_kind)
    R = args.replicas or cap
    params = capi.memetic_params(target_energy=0, rng_kind=rng_kind)
    solver = capi.Solver(ctx, n, R, base_seed=1000, replica_offset=rank * R, params=params)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{local}")
    epoch_s = args.epoch_ms / 1e3

    # islands: k elites per GPU, all_gathered over NCCL between steps
    isl = None
    if args.islands:
        from paper_2504_00987_b200.islands import Islands
        isl = Islands(solver, n, k_elites=16, device=torch.device("cuda", local))

    for _ in range(args.warmup):
        solver.run(epoch_seconds=epoch_s, race=False)
    ctx.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_before, m_before = solver.counters()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.synchronize()
    launches = 0
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            with torch.cuda.stream(ext):
                flush.fill_(k)  # evict L2 between timed steps (not timed)
                starts[k].record(ext)
            solver.run(epoch_seconds=epoch_s, race=False)
            launches += 1
            with torch.cuda.stream(ext):
                ends[k].record(ext)
            if isl is not None and (k + 1) % args.islands == 0:
                isl.exchange(rotation=k)
        ctx.synchronize()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_after, m_after = solver.counters()
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    evals_local = float(t_after - t_before) * n
    if world > 1:
        tt = torch.tensor([evals_local, dev_ms], dtype=torch.float64, device=cdev)
        ev = tt[:1].clone()
        dist.all_reduce(ev, op=dist.ReduceOp.SUM)
        mx = tt[1:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        evals_total, time_ms = float(ev.item()), float(mx.item())
    else:
        evals_total, time_ms = evals_local, dev_ms
    value = evals_total / (time_ms / 1e3)
    per_gpu = value / world

    # Roofline: (N-1) lag-term MACs per flip-evaluation over
    # the measured IMAD rate of this device. The kernel's O(1)-per-candidate
    # update does far fewer operations than the reference's O(N) scoring, so
    # frac > 1 is possible; executed_* keys give the work actually issued.
    imad_peak = ctx.imad_peak_gops()
    int_peak = ctx.int_peak_gops()
    lag_gmacs = per_gpu * (n - 1) / 1e9
    exec_gops = per_gpu * OPS_PER_FLIP_EVAL / 1e9
    traffic, issue, prof_src = None, None, None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            # DRAM bytes of one k_memetic launch: replica state in and out
            # (MT states, populations), nearly independent of the launch
            # length (16.4 MB at 20 ms, 16.8 MB at 50 ms, N=64)
            traffic = pj.get(f"k_memetic_n{n}_dram_bytes")
            issue = pj.get(f"k_memetic_n{n}_issue_slots_busy")
            prof_src = pj.get("source")
        except Exception:
            traffic = None

    # e2e through the reference-facing C-ABI call with host buffers: a solve
    # with a wall budget (`labs solve --time-limit`), so every replica works
    # until the budget and none idles at the end of the call.
    e2e_budget = 0.5
    e2e_params = capi.memetic_params(target_energy=0, max_seconds=e2e_budget,
                                     rng_kind=rng_kind)
    ctx.run_replicas(n, R, 7, capi.memetic_params(target_energy=0, max_iterations=2,
                                                  rng_kind=rng_kind))  # warm
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    best, per = ctx.run_replicas(n, R, 1000 + rank * R, e2e_params)
    e2e_t = time.perf_counter() - t0
    e2e_evals = sum(p["tabu_iterations"] for p in per) * n
    e2e_value = e2e_evals / e2e_t
    if world > 1:
        t = torch.tensor([e2e_evals, e2e_t], dtype=torch.float64, device=cdev)
        a = t[:1].clone()
        dist.all_reduce(a)
        b = t[1:].clone()
        dist.all_reduce(b, op=dist.ReduceOp.MAX)
        e2e_value = float(a.item()) / float(b.item())
    d2h = R * capi.C.sizeof(capi.RunResult) + R * 4 * 3
    h2d = capi.C.sizeof(capi.MemeticParams)

    line = {
        "metric": "tabu flip-evals/sec", "value": value, "unit": "flip-evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": time_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": f"LABS N={n} memetic tabu search, {R} replicas/GPU "
                               f"(one warp each), K=100, {args.rng} RNG, "
                               f"{args.epoch_ms:.0f} ms device epochs",
                   "n": n, "replicas_per_gpu": R, "population": 100,
                   "rng": args.rng, "epoch_ms": args.epoch_ms,
                   "l2": "flushed (256 MiB write) between timed steps",
                   "islands": args.islands},
        "per_gpu": per_gpu,
        "memetic_iterations": m_after - m_before,
        "gpu_launches": launches,
        "roofline": {"bound": "int32", "achieved": lag_gmacs, "peak": imad_peak,
                     "unit": "Gop/s", "frac": lag_gmacs / imad_peak, "traffic": traffic,
                     "traffic_source": (f"from_ncu ({prof_src}): dram__bytes_read + write of one "
                                        "k_memetic launch (per-launch replica state traffic; "
                                        "not measured inside this run)")
                     if traffic is not None else None,
                     "work_per_flip_eval": f"{n - 1} lag-term MACs (N-1, SURVEY.md §8d)",
                     "peak_source": "IMAD-only probe labs_bench_imad_peak, measured on "
                                    "this device in this run",
                     "frac_vs_all_int_pipes": lag_gmacs / int_peak,
                     "int_peak_all_pipes": int_peak,
                     "executed_ops_per_flip_eval": OPS_PER_FLIP_EVAL,
                     "executed_ops_frac": exec_gops / int_peak,
                     "issue_slots_busy_ncu": issue},
        "e2e": {"value": e2e_value, "unit": "flip-evals/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "call": f"labs_run_replicas(n={n}, replicas={R}, max_seconds={e2e_budget})"},
        "clocks": clocks.summary(),
    }
    solver.close()

    if rank == 0 and world == 1 and not args.quick:
        try:
            cb = cpu_reference_throughput(n, args.cpu_seconds)
            frac = admissible_fraction(n)
            cb["admissible_fraction"] = frac
            cb["value_admissible_only"] = cb["value"] * frac
            line["cpu_baseline"] = cb
        except Exception as e:  # the checker library was not built on this host
            line["cpu_baseline"] = {"unavailable": f"{type(e).__name__}: {e}"}
        if n in TARGETS and args.tts_samples > 0:
            line["tts"] = time_to_target(ctx, n, TARGETS[n], R, rng_kind, args)
            try:
                line["tts"]["cpu_tts"] = cpu_reference_tts(n, TARGETS[n], args.cpu_tts_seconds)
            except Exception as e:
                line["tts"]["cpu_tts"] = {"unavailable": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def time_to_target(ctx, n, target, R, rng_kind, args):
    """run_tts (fit.cpp:15-41) at one n: `--tts-samples` fresh replica sets
    from disjoint seed blocks base + run * R, wall time from solver creation
    to the first replica at the target (censored at --tts-limit)."""
    from paper_2504_00987_b200.tts import quantile, run_tts
    recs = run_tts(ctx, [n], {n: target}, reps=args.tts_samples, replicas=R,
                   base_seed=100_000, time_limit=args.tts_limit, rng_kind=rng_kind)
    times = [r["runtime"] for r in recs if r["reachedTarget"]]
    a, b = PAPER_A100_FIT
    return {"n": n, "target": target, "samples": len(recs),
            "censored": sum(not r["reachedTarget"] for r in recs),
            "limit_s": args.tts_limit, "replicas": R,
            "seed_blocks": "base 100000 + run * replicas (disjoint; fit.cpp:30-31)",
            "median_s": quantile(times, 0.5) if times else None,
            "q1_s": quantile(times, 0.25) if times else None,
            "q3_s": quantile(times, 0.75) if times else None,
            "samples_detail": [{k: r[k] for k in ("seed", "runtime", "reachedTarget", "bestE",
                                                  "bestSeq", "bestReplica")} for r in recs],
            "paper_a100_fit_s": a * b ** n}


if __name__ == "__main__":
    main()
