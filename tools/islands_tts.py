"""Time to target with the island model's elite exchange on one GPU (the
exchange is replica-to-replica through k_export/k_import_elites; with more
GPUs the same driver all_gathers elites over NCCL). Compare with
`python -m paper_2504_00987_b200.tts` (no exchange) on the same instances.

usage: python tools/islands_tts.py --n 98,99,104,107 --limit 180 --every 30 --epoch 1.0 \
           --k 4 --replacement random      (--every 0: no exchange)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2504_00987_b200 import capi  # noqa: E402
from paper_2504_00987_b200.islands import Islands  # noqa: E402
from paper_2504_00987_b200.tts import read_targets  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="98,99,104,107")
    ap.add_argument("--limit", type=float, default=180.0)
    ap.add_argument("--every", type=int, default=1, help="exchange every this many epochs")
    ap.add_argument("--epoch", type=float, default=1.0, help="epoch seconds")
    ap.add_argument("--k", type=int, default=16, help="elites per exchange")
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--replacement", choices=["random", "worst"], default="random",
                    help="population replacement: the reference's uniform victim "
                         "(memetic.cpp:100-102) or elite-preserving worst member")
    ap.add_argument("--targets", default=os.path.join(ROOT, "paper_2504_00987_b200", "data",
                                                      "targets_long.txt"))
    ap.add_argument("--target-column", type=int, default=2)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    ctx = capi.Context(0)
    targets = read_targets(a.targets, a.target_column)
    fh = open(a.out, "a") if a.out else None
    for n in [int(x) for x in a.n.split(",")]:
        R = capi.Solver.capacity(ctx, n, capi.RNG_MT19937_64)
        params = capi.memetic_params(target_energy=targets[n], max_seconds=a.limit + 5,
                                     replacement=capi.REPLACE_WORST if a.replacement == "worst"
                                     else capi.REPLACE_RANDOM)
        t0 = time.perf_counter()
        sv = capi.Solver(ctx, n, R, base_seed=a.seed, params=params)
        isl = Islands(sv, n, k_elites=a.k, device=torch.device("cuda", 0))
        rep = isl.run(targets[n], epoch_seconds=a.epoch, exchange_every=a.every,
                      max_seconds=a.limit)
        dt = time.perf_counter() - t0
        rec = {"n": n, "targetE": targets[n], "bestE": rep.best_energy,
               "reachedTarget": rep.reached, "runtime": dt, "replicas": R,
               "exchange_every_epochs": a.every, "epoch_s": a.epoch, "k_elites": a.k,
               "replacement": a.replacement, "seed": a.seed, "epochs": rep.epochs,
               "exchanges": rep.exchanges}
        sv.close()
        line = json.dumps(rec, sort_keys=True)
        print(line, flush=True)
        if fh:
            fh.write(line + "\n")
            fh.flush()


if __name__ == "__main__":
    main()
