"""`labs solve` wire format on the B200.

Same options, result line and exit codes as the reference CLI's solve
subcommand (proj/tools/labs_cli.cpp:28-61, 161-305): replicas race to the
target through labs_run_replicas; one JSON object (keys sorted, compact, as
nlohmann::json dumps it) on stdout, appended to --out when given. Exit 0 on
success, 2 on invalid arguments (std::invalid_argument / out_of_range), 1 on
any other failure.

    python -m paper_2504_00987_b200.solve --n 20 --target 26 --replicas 2 --seed 42
"""
from __future__ import annotations

import argparse
import json
import sys


def result_json(n, r):
    from paper_2504_00987_b200.sequence import encode_hex
    return {"n": n, "bestSeq": encode_hex(r["best"], n), "bestE": r["best_energy"],
            "mf": r["merit"], "iterations": r["iterations"], "wallTime": r["wall_seconds"],
            "seed": r["seed"], "replicaId": r["replica_id"],
            "reachedTarget": r["reached_target"]}


def main(argv=None):
    ap = argparse.ArgumentParser(prog="labs solve")
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--target", type=int, default=0)
    ap.add_argument("--replicas", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--scan-workers", type=int, default=1)
    ap.add_argument("--time-limit", type=float, default=None)
    ap.add_argument("--max-iterations", type=int, default=None)
    ap.add_argument("--out", default="")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    from paper_2504_00987_b200 import capi
    try:
        if args.scan_workers < 1:
            raise ValueError("scan workers must be >= 1")
        ctx = capi.Context(0)
        params = capi.memetic_params(target_energy=args.target, max_seconds=args.time_limit,
                                     max_iterations=args.max_iterations)
        best, _ = ctx.run_replicas(args.n, args.replicas, args.seed, params)
    except (ValueError, IndexError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - CLI maps everything else to 1
        print(f"error: {e}", file=sys.stderr)
        return 1
    line = json.dumps(result_json(args.n, best), sort_keys=True, separators=(",", ":"))
    print(line)
    if args.out:
        with open(args.out, "a") as f:
            f.write(line + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
