"""GPU parity tests: the sm_100a kernels, called through the C ABI
(include/labs_b200.h via paper_2504_00987_b200/capi.py), against the golden
vectors produced by the unmodified reference and against the oracle.

Bar: bit-exact for every integer — C_k, E, every neighbor energy, the chosen
move, the tie set, the tabu update, the RNG consumption, whole trajectories."""
import ctypes as C

import numpy as np
import pytest

from oracle.pyoracle import LoRng
from paper_2504_00987_b200 import capi
from paper_2504_00987_b200.sequence import decode_hex, random_words

pytestmark = pytest.mark.gpu


def lo_from_state(st) -> LoRng:
    r = LoRng()
    C.memmove(C.byref(r), C.byref(st), 312 * 8 + 4)
    return r


def test_build_state_matches_reference_probes(ctx, golden):
    by_n = {}
    for p in golden["probes"]:
        by_n.setdefault(p["n"], []).append(p)
    for n, ps in by_n.items():
        corr, e, nb = ctx.build_state(n, [p["words"] for p in ps])
        for i, p in enumerate(ps):
            assert e[i] == p["E"], n
            assert corr[i].tolist() == p["C"], n
            assert nb[i].tolist() == p["neighbors"], n


def test_kats(ctx, golden):
    corr, e, nb = ctx.build_state(5, [[0]])
    assert e[0] == 30 and corr[0].tolist() == [4, 3, 2, 1]
    corr, e, nb = ctx.build_state(4, [[0]])
    assert e[0] == 14 and nb[0].tolist() == [2, 2, 2, 2]
    assert ctx.energies(92, [decode_hex("EE01C0E77667DD34DAE94B5", 92)])[0] == 490
    for row in golden["table"]:
        assert ctx.energies(row["n"], [decode_hex(row["hex"], row["n"])])[0] == row["E"]


@pytest.mark.parametrize("n", [2, 3, 5, 31, 32, 33, 64, 65, 92, 107, 119, 120, 128, 129,
                               187, 255, 256])
def test_flip_trace_matches_oracle(ctx, oracle, n):
    """Incremental commit (apply_flip, correlation_state.cpp:73-98) after every
    flip of random traces: energy and all n neighbor energies."""
    rs = np.random.default_rng(n)
    count, flips = 6, 60
    words = random_words(n, count, rs)
    pos = rs.integers(0, n, size=(count, flips)).astype(np.int32)
    e, nb = ctx.flip_trace(n, words, pos)
    for c in range(count):
        st = oracle.state(n, words[c])
        for f in range(flips):
            oracle.lib.lo_apply_flip(C.byref(st), int(pos[c, f]))
            assert e[c, f] == st.E
            want = [oracle.lib.lo_neighbor_energy(C.byref(st), j) for j in range(n)]
            assert nb[c, f].tolist() == want, (c, f)


def test_scan_matches_reference(ctx, oracle, golden):
    by_n = {}
    for s in golden["scans"]:
        by_n.setdefault(s["n"], []).append(s)
    for n, ss in by_n.items():
        rngs = capi.rng_states([s["draw_seed"] for s in ss])
        r = ctx.scan(n, [s["words"] for s in ss], [s["admissible"] for s in ss], rngs)
        for i, s in enumerate(ss):
            assert (int(r["position"][i]), int(r["energy"][i]), bool(r["fallback"][i])) == (
                s["position"], s["energy"], s["fallback"]), (n, i)
            lo = oracle.rng(s["draw_seed"])
            o = oracle.scan(n, s["words"], s["admissible"], lo)
            assert int(r["ntie"][i]) == len(o["ties"])
            mask = [int(x) for x in r["tie_mask"][i]]
            got = [j for j in range(n) if (mask[j >> 6] >> (j & 63)) & 1]
            assert got == o["ties"]
            # RNG consumption identical: same engine state afterwards
            assert list(rngs[i].mt) == list(lo.mt) and rngs[i].idx == lo.idx


def test_scan_without_fallback_raises(ctx):
    rngs = capi.rng_states([1])
    with pytest.raises(RuntimeError):
        ctx.scan(6, [[0]], [[0] * 6], rngs, allow_fallback=False)


def test_tabu_walks_match_reference_trajectories(ctx, oracle, golden):
    by_key = {}
    for wk in golden["walks"]:
        by_key.setdefault((wk["n"], wk["min_factor"], wk["max_factor"]), []).append(wk)
    for (n, fmin, fmax), wks in by_key.items():
        rngs = capi.rng_states([wk["seed"] for wk in wks])
        out = ctx.tabu_walks(n, [wk["start"] for wk in wks], rngs,
                             capi.tabu_params(fmin, fmax), trace=True)
        for i, wk in enumerate(wks):
            assert out["steps"][i] == [tuple(s) for s in wk["steps"]], n
            assert out["energy"][i] == wk["energy"]
            assert out["best"][i].tolist() == wk["best"]
            assert (out["max_iter"][i], out["min_tabu"][i], out["max_tabu"][i]) == (
                wk["max_iter"], wk["min_tabu"], wk["max_tabu"])
            lo = lo_from_state(rngs[i])
            assert oracle.lib.lo_rng_bits64(lo) == wk["post_draw"]


@pytest.mark.parametrize("n", [32, 64, 107, 119, 120, 200])
def test_tabu_walks_batch_matches_oracle(ctx, oracle, n):
    """A batch of independent walks (one warp each) equals the oracle walk by walk."""
    rs = np.random.default_rng(1000 + n)
    count = 40
    words = random_words(n, count, rs)
    seeds = [int(x) for x in rs.integers(0, 2**63, size=count)]
    rngs = capi.rng_states(seeds)
    out = ctx.tabu_walks(n, words, rngs)
    for c in range(count):
        lo = oracle.rng(seeds[c])
        o = oracle.tabu(n, words[c], lo, trace=False)
        assert out["energy"][c] == o["energy"]
        assert out["best"][c].tolist() == o["best"].tolist()
        assert list(rngs[c].mt) == list(lo.mt) and rngs[c].idx == lo.idx


def test_tie_rule_lowest_and_aspiration_invariants(ctx, oracle):
    """Policy switches (north_star): deterministic lowest-index tie-break and
    aspiration. Checked by replaying each step against the oracle state."""
    n = 48
    rs = np.random.default_rng(5)
    words = random_words(n, 8, rs)
    for asp in (False, True):
        rngs = capi.rng_states(range(8))
        out = ctx.tabu_walks(n, words, rngs,
                             capi.tabu_params(tie_rule=capi.TIE_LOWEST, aspiration=asp),
                             trace=True)
        for c in range(8):
            st = oracle.state(n, words[c])
            expiry = [0] * n
            best = st.E
            for (t, pos, e, ten, fb) in out["steps"][c]:
                nb = [oracle.lib.lo_neighbor_energy(C.byref(st), j) for j in range(n)]
                adm = [expiry[j] < t or (asp and nb[j] < best) for j in range(n)]
                if any(adm):
                    m = min(nb[j] for j in range(n) if adm[j])
                    assert not fb and pos == min(j for j in range(n) if adm[j] and nb[j] == m)
                else:
                    assert fb
                oracle.lib.lo_apply_flip(C.byref(st), pos)
                assert st.E == e
                expiry[pos] = t + ten
                best = min(best, e)
            assert out["energy"][c] == best


def test_memetic_matches_reference(ctx, golden):
    for m in golden["memetic"]:
        p = dict(m["params"])
        tabu_kw = {k: p.pop(k) for k in ("min_tabu_factor", "max_tabu_factor") if k in p}
        params = capi.memetic_params(**p, **tabu_kw)
        d = ctx.memetic(m["n"], m["seed"], params, trace_cap=len(m["child_energies"]) + 1)
        assert d["best_energy"] == m["best_energy"], m["n"]
        assert d["iterations"] == m["iterations"]
        assert d["best"].tolist() == m["best"]
        assert d["reached_target"] == m["reached_target"]
        assert [t[2] for t in d["trace"]] == m["child_energies"]
        assert not any(t[1] for t in d["trace"])


def test_readme_trajectory(ctx):
    """README.md:114-117: replica seed 43, n=20, target 26 -> E=26 after 98
    iterations, best C9EF5."""
    from paper_2504_00987_b200.sequence import encode_hex
    d = ctx.memetic(20, 43, capi.memetic_params(target_energy=26))
    assert (d["best_energy"], d["iterations"], encode_hex(d["best"], 20)) == (26, 98, "C9EF5")
    assert d["reached_target"]


def test_configs0_run_to_optimum(ctx, golden):
    """BASELINE configs[0]: N=32, one population (K=100), fixed seed, run to
    the known optimum E=64 — survey fingerprint G4 from the compiled
    reference: reached after 793 iterations with best 64C75280. Checked
    through labs_memetic (every child energy) and labs_run_replicas."""
    from paper_2504_00987_b200.sequence import encode_hex
    g = [m for m in golden["memetic"] if m["n"] == 32 and m["seed"] == 1032][0]
    assert (g["best_energy"], g["iterations"], g["reached_target"]) == (64, 793, True)
    d = ctx.memetic(32, 1032, capi.memetic_params(target_energy=64), trace_cap=1000)
    assert (d["best_energy"], d["iterations"], encode_hex(d["best"], 32)) == (64, 793, "64C75280")
    assert [t[2] for t in d["trace"]] == g["child_energies"]
    best, per = ctx.run_replicas(32, 1, 1032, capi.memetic_params(target_energy=64))
    assert (best["best_energy"], best["iterations"], encode_hex(best["best"], 32)) == \
        (64, 793, "64C75280")
    assert best["reached_target"] and best["seed"] == 1032


@pytest.mark.parametrize("n", [64, 119])
def test_bench_scale_replicas_match_oracle(ctx, oracle, n):
    """The bench configuration itself: R = resident capacity (k_memetic<2,32,MT>
    at N=64, NS=4 at N=119), run in time-sliced epochs like bench.py (20 us
    slices: about one memetic iteration per launch);
    33 replicas spread over the whole grid (so over every SM's warps)
    replay the oracle's memetic_tabu(n, base + r) exactly: best, energy,
    iterations and every child energy."""
    iters = 4
    R = capi.Solver.capacity(ctx, n, capi.RNG_MT19937_64)
    assert R >= 148 * 4
    p = capi.memetic_params(target_energy=0, max_iterations=iters)
    sv = capi.Solver(ctx, n, R, base_seed=31337, params=p, trace_cap=iters + 1)
    launches = 0
    while True:
        sv.run(epoch_seconds=2e-5, race=False)
        launches += 1
        if sv.status()["running"] == 0:
            break
    assert launches >= 3  # the time slices really cut every replica's run
    res = sv.results()
    picks = sorted(set([k * (R - 1) // 32 for k in range(33)]))
    for r in picks:
        want = oracle.memetic(n, 31337 + r, child_cap=iters, target_energy=0,
                              max_iterations=iters)
        got = res[r]
        assert got["seed"] == 31337 + r
        assert (got["best_energy"], got["iterations"]) == (want["best_energy"], want["iterations"])
        assert got["best"].tolist() == want["best"]
        assert [t[2] for t in got["trace"]] == want["child_energies"]
    sv.close()


def test_run_replicas_matches_reference(ctx, golden):
    for c in golden["replicas"]:
        best, per = ctx.run_replicas(c["n"], c["replicas"], c["base_seed"],
                                     capi.memetic_params(target_energy=c.get("target_energy", 0),
                                                         max_iterations=c["max_iterations"]))
        for a, b in zip(per, c["per_replica"]):
            assert a["best"].tolist() == b["best"]
            for k in ("best_energy", "iterations", "seed", "replica_id", "reached_target"):
                assert a[k] == b[k], k
        assert best["best_energy"] == c["best"]["best_energy"]


def test_replicas_race_to_target(ctx, golden):
    """test_parallel.cpp:94-117: replicas race; stop seen only at the last record."""
    target = golden["targets_small"]["16"]
    best, per = ctx.run_replicas(16, 6, 20000, capi.memetic_params(target_energy=target,
                                                                   max_seconds=60.0),
                                 trace_cap=100000)
    assert best["reached_target"] and best["best_energy"] == target
    assert best["seed"] == 20000 + best["replica_id"]
    for r in per:
        tr = r["trace"]
        assert not any(t[1] for t in tr[:-1])


@pytest.mark.parametrize("n", [13, 20, 24])
def test_reaches_proven_optima(ctx, golden, n):
    """acceptance.cpp:162-191 (criterion C5), both RNG modes."""
    target = golden["targets_small"][str(n)]
    for kind in (capi.RNG_MT19937_64, capi.RNG_PHILOX):
        d = ctx.memetic(n, 1000 + n, capi.memetic_params(target_energy=target,
                                                         max_seconds=60.0, rng_kind=kind))
        assert d["reached_target"] and d["best_energy"] == target


def test_device_walks_philox_are_consistent(ctx, oracle):
    """Throughput path (device pointers, Philox): every returned best is a
    real sequence with the reported energy, never worse than its start."""
    import torch
    n, count = 64, 512
    rs = np.random.default_rng(3)
    words = random_words(n, count, rs)
    d_start = torch.from_numpy(words.view(np.int64)).cuda()
    d_best = torch.zeros_like(d_start)
    d_e = torch.zeros(count, dtype=torch.int64, device="cuda")
    d_it = torch.zeros(1, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    ctx.tabu_walks_device(n, count, 3, d_start.data_ptr(), d_best.data_ptr(), d_e.data_ptr(),
                          rng_kind=capi.RNG_PHILOX, seed=99, d_iterations=d_it.data_ptr())
    ctx.synchronize()
    best = d_best.cpu().numpy().view(np.uint64)
    e = d_e.cpu().numpy()
    start_e = ctx.energies(n, words)
    for c in range(0, count, 37):
        assert oracle.energy(n, best[c]) == e[c]
    assert (e <= start_e).all()
    its = int(d_it.item())
    assert count * 3 * (n // 2) <= its <= count * 3 * (n + n // 2)


def test_validation_errors(ctx):
    with pytest.raises(ValueError):
        ctx.build_state(1, [[0]])
    with pytest.raises(ValueError):
        ctx.build_state(capi.LABS_MAX_N + 1, [[0] * 5])
    with pytest.raises(ValueError):
        ctx.tabu_walks(8, [[0]], capi.rng_states([1]), capi.tabu_params(0.5, 1.0))
    with pytest.raises(ValueError):
        ctx.tabu_walks(8, [[0]], capi.rng_states([1]), capi.tabu_params(-0.1, 0.12))
    with pytest.raises(IndexError):
        ctx.flip_trace(8, [[0]], [[8]])
    with pytest.raises(ValueError):
        ctx.run_replicas(12, 3, 1, capi.memetic_params(population_size=1))
    with pytest.raises(ValueError):
        ctx.build_state(3, [[0b1000]])  # nonzero padding bit


def test_readme_solve_example(ctx):
    """README.md:110-117: `labs solve --n 20 --target 26 --replicas 2 --seed 42`
    -> replica 1 (seed 43) wins with E=26 after 98 iterations, best C9EF5."""
    from paper_2504_00987_b200.sequence import encode_hex
    best, per = ctx.run_replicas(20, 2, 42, capi.memetic_params(target_energy=26,
                                                                max_seconds=30.0))
    assert best["reached_target"] and best["best_energy"] == 26
    r1 = per[1]
    assert r1["reached_target"] and r1["iterations"] == 98
    assert encode_hex(r1["best"], 20) == "C9EF5"


def _canonical_hex(words, n):
    """canonical() (sequence.cpp:162-169): lexicographic minimum (position 0
    most significant = hex string order) over the four symmetries."""
    from paper_2504_00987_b200.sequence import encode_hex, from_spins, spins
    s = spins(words, n)
    cands = [s, -s, s[::-1], -s[::-1]]
    return min(encode_hex(from_spins(c), n) for c in cands)


def test_exhaustive_matches_reference(ctx, golden):
    """brute_force_optimum (oracle.cpp:70-110) for n = 3..24: optimal energy
    and the canonical witness set, exactly."""
    for case in golden["exhaustive"]:
        n = case["n"]
        e, raw = ctx.exhaustive_optimum(n)
        assert e == case["E"], n
        assert sorted({_canonical_hex([w], n) for w in raw}) == case["witnesses"], n


def test_exhaustive_proven_optima_and_beyond(ctx, golden):
    """targets_small.txt (proven optima, n = 2..30) and the literature optimum
    E(32) = 64 (Packebusch & Mertens 2016), beyond the reference's n <= 30."""
    for n_str, e_want in golden["targets_small"].items():
        e, _ = ctx.exhaustive_optimum(int(n_str), cap=4096)
        assert e == e_want, n_str
    e, _ = ctx.exhaustive_optimum(32, cap=4096)
    assert e == 64


def test_local_optima_census_matches_reference(ctx, golden):
    for n_str, want in golden["local_optima"].items():
        assert ctx.local_optima(int(n_str)) == want, n_str


def test_solve_cli_wire_format(tmp_path):
    """README.md:110-117: `labs solve --n 20 --target 26 --replicas 2 --seed 42`."""
    import json
    import subprocess
    import sys
    out = tmp_path / "solve.jsonl"
    r = subprocess.run([sys.executable, "-m", "paper_2504_00987_b200.solve", "--n", "20",
                        "--target", "26", "--replicas", "2", "--seed", "42", "--time-limit",
                        "30", "--out", str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    assert list(d) == sorted(d)
    assert d["bestE"] == 26 and d["reachedTarget"] and d["n"] == 20
    assert d["seed"] == 42 + d["replicaId"]
    assert json.loads(out.read_text().splitlines()[0]) == d
    bad = subprocess.run([sys.executable, "-m", "paper_2504_00987_b200.solve", "--n", "1"],
                         capture_output=True, text=True, timeout=120)
    assert bad.returncode == 2


@pytest.mark.parametrize("n,lo,hi,iters", [(60, 0.10, 0.90, 6), (200, 0.0, 0.95, 2),
                                           (33, 0.0, 0.0, 8), (256, 0.5, 0.99, 3),
                                           (119, 0.10, 0.12, 40), (64, 0.10, 0.12, 60)])
def test_memetic_wide_tenure_windows(ctx, oracle, n, lo, hi, iters):
    """Tenure windows far from the default 0.10/0.12 (wide ones exercise the
    range-specialized Lemire reduction with large ranges; a one-value window
    still consumes one draw per step; max_t > 254 is served without the
    tenure table), and long default runs that cross many table windows and
    MT twists. Whole memetic runs must replay the oracle draw for draw."""
    kw = dict(min_tabu_factor=lo, max_tabu_factor=hi)
    want = oracle.memetic(n, 4242, child_cap=iters, max_iterations=iters, **kw)
    d = ctx.memetic(n, 4242, capi.memetic_params(max_iterations=iters, **kw), trace_cap=iters + 1)
    assert d["best_energy"] == want["best_energy"]
    assert d["best"].tolist() == want["best"]
    assert d["iterations"] == want["iterations"]
    assert [t[2] for t in d["trace"]] == want["child_energies"]


@pytest.mark.parametrize("n", [2, 13, 64, 92, 119, 256])
def test_evaluator_matches_build_state(ctx, oracle, n):
    """labs_eval (the persistent evaluator behind CorrelationState) equals the
    batch build and the oracle for consecutive flips of one sequence; a
    commit costs one round trip (reported, not asserted)."""
    import time
    from paper_2504_00987_b200.sequence import random_words
    rs = np.random.default_rng(n)
    w = random_words(n, 1, rs)[0].copy()
    ev = capi.Evaluator(ctx, n)
    t0 = time.perf_counter()
    flips = 40
    for f in range(flips):
        corr, e, nb = ev(w)
        c2, e2, nb2 = ctx.build_state(n, w)
        assert e == int(e2[0]) == oracle.energy(n, w)
        assert corr.tolist() == c2[0].tolist() and nb.tolist() == nb2[0].tolist()
        j = int(rs.integers(0, n))
        w[j // 64] ^= np.uint64(1) << np.uint64(j % 64)
    dt = (time.perf_counter() - t0) / flips
    print(f"n={n}: {dt * 1e6:.1f} us per evaluate+build pair")
    ev.close()
