"""Generate tests/golden/*.json from the UNMODIFIED reference.

Runs only in the build container, where /root/reference exists and
oracle/Makefile has compiled the reference sources into
oracle/_ref/libref_labsolve.so. The GPU box never runs this; it reads the
committed JSON. Re-run with:

    make -C oracle && python tests/golden/make_golden.py

Every vector below is produced by the reference's own code path
(labsolve::Rng, CorrelationState, scan_neighborhood, tabu_search,
memetic_tabu, run_replicas) through oracle/ref_capi.cpp.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference, double_bits  # noqa: E402
from paper_2504_00987_b200.sequence import decode_hex, encode_hex  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
REF_DATA = "/root/reference/proj/data"


def words_list(w):
    return [int(x) for x in np.asarray(w, dtype=np.uint64).reshape(-1)]


def main():
    ref = Reference()
    rs = np.random.default_rng(20261018)

    # 1. RNG draw streams (rng.hpp:10-28 over libstdc++ 13).
    rng_cases = []
    for seed in (0, 1, 42, 1000, 2**63 + 12345, 2**64 - 1):
        kinds = rs.integers(0, 3, size=400).tolist()
        lo = rs.integers(-50, 50, size=400).tolist()
        span = [int(x) for x in rs.choice([1, 2, 3, 7, 100, 2**40, 2**62 + 1], size=400)]
        hi = [l + s - 1 for l, s in zip(lo, span)]
        out = ref.rng_draws(seed, kinds, lo, hi)
        rng_cases.append({"seed": seed, "kinds": kinds, "lo": lo, "hi": hi,
                          "out": [int(x) for x in out]})

    # 2. Known-answer tests (test_correlation.cpp:31-78, test_sequence.cpp).
    kats = {
        "all_plus_5": {"n": 5, "C": [4, 3, 2, 1], "E": 30},
        "all_plus_4_neighbors": {"n": 4, "E": 14, "neighbors": [2, 2, 2, 2]},
        "n92": {"n": 92, "hex": "EE01C0E77667DD34DAE94B5", "E": 490},
    }
    table = []
    with open(os.path.join(REF_DATA, "published_sequences.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            n, hx, e, mf, d = line.split()
            w = decode_hex(hx, int(n))
            assert ref.energy(int(n), w) == int(e), (n, hx)
            table.append({"n": int(n), "hex": hx, "E": int(e), "mf": float(mf), "d": int(d)})
    targets = {}
    with open(os.path.join(REF_DATA, "targets_published.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                n, e = line.split()
                targets[int(n)] = int(e)
    small = {}
    with open(os.path.join(REF_DATA, "targets_small.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                n, e = line.split()[:2]
                small[int(n)] = int(e)

    # 3. CorrelationState probes: C_k, E, every neighbor energy.
    probes = []
    ns = [2, 3, 4, 5, 8, 13, 31, 32, 33, 63, 64, 65, 92, 100, 107, 119, 120, 127, 128,
          129, 160, 187, 200, 255, 256]
    for i, n in enumerate(ns):
        for rep in range(2):
            w = ref.random_sequences(n, 37 + 100 * i + rep, 1)[0]
            corr, e, nb = ref.probe(n, w)
            probes.append({"n": n, "words": words_list(w), "C": [int(x) for x in corr],
                           "E": e, "neighbors": [int(x) for x in nb]})
    for row in table:
        w = decode_hex(row["hex"], row["n"])
        corr, e, nb = ref.probe(row["n"], w)
        probes.append({"n": row["n"], "words": words_list(w), "C": [int(x) for x in corr],
                       "E": e, "neighbors": [int(x) for x in nb]})

    # 4. scan_neighborhood with explicit masks and draw seeds.
    scans = []
    for i in range(120):
        n = int(rs.choice([2, 3, 4, 6, 8, 17, 32, 40, 64, 65, 100, 119, 128, 200, 256]))
        w = ref.random_sequences(n, 5000 + i, 1)[0]
        mode = i % 4
        if mode == 0:
            adm = np.ones(n, dtype=np.uint8)
        elif mode == 1:
            adm = (rs.random(n) < 0.7).astype(np.uint8)
        elif mode == 2:
            adm = (rs.random(n) < 0.1).astype(np.uint8)
        else:
            adm = np.zeros(n, dtype=np.uint8)
        seed = int(rs.integers(0, 2**63))
        r = ref.scan(n, w, adm, seed)
        scans.append({"n": n, "words": words_list(w), "admissible": adm.tolist(),
                      "draw_seed": seed, **r})
    # all-plus(4): a four-way tie (test_correlation.cpp:176-191)
    for seed in range(8):
        w = np.zeros(1, dtype=np.uint64)
        r = ref.scan(4, w, np.ones(4, dtype=np.uint8), seed)
        scans.append({"n": 4, "words": [0], "admissible": [1, 1, 1, 1], "draw_seed": seed, **r})

    # 5. tabu_search trajectories (tabu.cpp:17-56), full traces.
    walks = []
    cases = [(n, 42, 7) for n in (32, 64, 119)]  # survey G2a-c
    for i, n in enumerate([2, 3, 5, 8, 13, 20, 24, 31, 32, 33, 48, 63, 64, 65, 92, 99, 107,
                           119, 120, 128, 129, 150, 187, 200, 255, 256]):
        cases.append((n, 900 + i, 7000 + i))
    for n, sseed, wseed in cases:
        start = ref.random_sequences(n, sseed, 1)[0]
        r = ref.tabu(n, start, wseed)
        walks.append({"n": n, "start": words_list(start), "seed": wseed, "min_factor": 0.10,
                      "max_factor": 0.12, "best": words_list(r["best"]), "energy": r["energy"],
                      "max_iter": r["max_iter"], "min_tabu": r["min_tabu"],
                      "max_tabu": r["max_tabu"], "steps": r["steps"],
                      "post_draw": r["post_draw"]})
    # fallback-heavy walks (test_tabu.cpp:103-114: factors 0.9/0.99)
    for i, n in enumerate([4, 6, 9, 33]):
        start = ref.random_sequences(n, 77 + i, 1)[0]
        r = ref.tabu(n, start, 101 + i, fmin=0.9, fmax=0.99)
        walks.append({"n": n, "start": words_list(start), "seed": 101 + i, "min_factor": 0.9,
                      "max_factor": 0.99, "best": words_list(r["best"]), "energy": r["energy"],
                      "max_iter": r["max_iter"], "min_tabu": r["min_tabu"],
                      "max_tabu": r["max_tabu"], "steps": r["steps"],
                      "post_draw": r["post_draw"]})

    # 6. memetic_tabu (memetic.cpp:44-117).
    memetic = []
    mcases = [dict(n=20, seed=43, target_energy=26)]  # README.md:114-117 (G1)
    # configs[0] (BASELINE.json): N=32, K=100, run to the optimum E=64 —
    # survey G4, 793 iterations, best 64C75280
    mcases.append(dict(n=32, seed=1032, target_energy=64))
    for n in (32, 64, 107, 119):  # survey G3
        mcases.append(dict(n=n, seed=1000 + n, target_energy=0, max_iterations=20))
    for n in (13, 20):  # test_memetic.cpp:106-120
        mcases.append(dict(n=n, seed=1000 + n, target_energy=small[n]))
    mcases.append(dict(n=24, seed=5, target_energy=0, max_iterations=30, population_size=7,
                       p_comb=0.5))
    mcases.append(dict(n=40, seed=9, target_energy=0, max_iterations=15, p_mutate=0.2,
                       min_tabu_factor=0.2, max_tabu_factor=0.5))
    mcases.append(dict(n=150, seed=3, target_energy=0, max_iterations=4, population_size=12))
    # edge cases: tiny n, K = 2, p_comb in {0, 1}, p_mutate = 1, zero tenure,
    # fallback-heavy tenure, aspiration-free long walks
    mcases.append(dict(n=2, seed=1, target_energy=0, max_iterations=5, population_size=2))
    mcases.append(dict(n=3, seed=2, target_energy=0, max_iterations=8, population_size=3))
    mcases.append(dict(n=17, seed=3, target_energy=0, max_iterations=10, p_comb=0.0))
    mcases.append(dict(n=17, seed=4, target_energy=0, max_iterations=10, p_comb=1.0,
                       p_mutate=1.0))
    mcases.append(dict(n=33, seed=5, target_energy=0, max_iterations=6, min_tabu_factor=0.0,
                       max_tabu_factor=0.0))
    mcases.append(dict(n=33, seed=6, target_energy=0, max_iterations=6, min_tabu_factor=0.9,
                       max_tabu_factor=0.99))
    mcases.append(dict(n=65, seed=7, target_energy=0, max_iterations=5, population_size=2,
                       p_comb=0.5, p_mutate=0.05))
    mcases.append(dict(n=256, seed=4, target_energy=0, max_iterations=2, population_size=5))
    for c in mcases:
        c = dict(c)
        n, seed = c.pop("n"), c.pop("seed")
        r = ref.memetic(n, seed, child_cap=100000, **c)
        memetic.append({"n": n, "seed": seed, "params": c, "best": r["best"],
                        "best_energy": r["best_energy"], "iterations": r["iterations"],
                        "reached_target": r["reached_target"],
                        "child_energies": r["child_energies"]})

    # 7. run_replicas, sequential mode (parallel.cpp:22-61; test_parallel.cpp).
    replicas = []
    for n, R, base, its in ((18, 1, 777, 20), (24, 2, 99, 10), (20, 3, 555, 12),
                            (64, 4, 1, 3)):
        best, per = ref.run_replicas(n, R, base, threaded=False, target_energy=0,
                                     max_iterations=its)
        replicas.append({"n": n, "replicas": R, "base_seed": base, "max_iterations": its,
                         "best": best, "per_replica": per})
    # configs[0] through run_replicas: one replica, seed 1032, target 64 (G4)
    best, per = ref.run_replicas(32, 1, 1032, threaded=False, target_energy=64)
    replicas.append({"n": 32, "replicas": 1, "base_seed": 1032, "max_iterations": None,
                     "target_energy": 64, "best": best, "per_replica": per})

    # 8. Exhaustive ground truth (oracle.cpp:70-151): optimal E + canonical
    # witnesses for n = 3..24, strict local-optima census for n = 3..20.
    exhaustive = []
    for n in range(3, 25):
        e, w = ref.brute_force(n)
        exhaustive.append({"n": n, "E": e, "witnesses": [encode_hex(x, n) for x in w]})
    local_optima = {n: ref.local_optima(n) for n in range(3, 21)}

    # 9. Skew deviation d(S) (skew.cpp:110-187): the Table II rows and random
    # short sequences, plain and with edits, with and without budgets.
    skew = []
    for row in table:
        w = decode_hex(row["hex"], row["n"])
        skew.append({"n": row["n"], "words": words_list(w), "budget": 0, "edits": False,
                     **ref.deviation(row["n"], w)})
    for i in range(24):
        n = int(rs.integers(3, 40))
        w = ref.random_sequences(n, 9000 + i, 1)[0]
        for edits in (False, True):
            for budget in (0, int(rs.integers(1, 60))):
                skew.append({"n": n, "words": words_list(w), "budget": budget, "edits": edits,
                             **ref.deviation(n, w, budget, edits)})

    fixtures = {"rng": rng_cases, "skew": skew, "exhaustive": exhaustive, "local_optima": local_optima, "kats": kats, "table": table, "targets": targets,
                "targets_small": small, "probes": probes, "scans": scans, "walks": walks,
                "memetic": memetic, "replicas": replicas}
    for item in replicas:
        for rr in [item["best"]] + item["per_replica"]:
            rr["best"] = [int(x) for x in rr["best"]]
            rr.pop("wall_seconds", None)
    for item in memetic:
        item["best"] = [int(x) for x in item["best"]]
    with open(os.path.join(OUT, "table2.txt"), "w") as f:
        f.write("# Table II rows (proj/data/published_sequences.txt): n hex E MF d\n")
        for row in table:
            f.write(f'{row["n"]} {row["hex"]} {row["E"]} {row["mf"]} {row["d"]}\n')
    path = os.path.join(OUT, "reference_vectors.json")
    with open(path, "w") as f:
        json.dump(fixtures, f, separators=(",", ":"))
    print(f"wrote {path} ({os.path.getsize(path) // 1024} KiB)")
    _ = double_bits


if __name__ == "__main__":
    main()
