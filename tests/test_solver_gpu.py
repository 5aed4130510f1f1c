"""Device solver API (labs_solver_*): epoch invariance, production policies,
island export/import semantics. Complements the reference-parity tests."""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from paper_2504_00987_b200 import capi

pytestmark = pytest.mark.gpu


def _results(sv):
    return [(r["best"].tolist(), r["best_energy"], r["iterations"]) for r in sv.results()]


def test_epochs_do_not_change_trajectories(ctx):
    """Cutting a run into epochs (the island model's exchange points) leaves
    every replica's trajectory bit-identical to one uninterrupted run."""
    n, R, iters = 48, 64, 12
    p = capi.memetic_params(target_energy=0, max_iterations=iters)
    one = capi.Solver(ctx, n, R, base_seed=5, params=p)
    one.run(race=False)
    cut = capi.Solver(ctx, n, R, base_seed=5, params=p)
    for _ in range(iters):
        cut.run(epoch_iterations=1, race=False)
    assert cut.status()["running"] == 0
    assert _results(one) == _results(cut)
    w1, e1 = one.population()
    w2, e2 = cut.population()
    assert (w1 == w2).all() and (e1 == e2).all()


def test_solver_matches_run_replicas_and_oracle(ctx):
    n, R, iters = 30, 5, 6
    p = capi.memetic_params(target_energy=0, max_iterations=iters)
    sv = capi.Solver(ctx, n, R, base_seed=100, params=p, replica_offset=3)
    sv.run(race=False)
    o = Oracle()
    for r in sv.results():
        # global id = offset + r, seed = base + id (parallel.cpp:38)
        want = o.memetic(n, 100 + r["replica_id"], max_iterations=iters)
        assert r["seed"] == 100 + r["replica_id"]
        assert r["best_energy"] == want["best_energy"] and r["best"].tolist() == want["best"]


def test_population_energies_are_consistent(ctx, oracle):
    n, R = 40, 8
    sv = capi.Solver(ctx, n, R, base_seed=1, params=capi.memetic_params(max_iterations=5))
    sv.run(race=False)
    w, e = sv.population()
    for r in range(R):
        for k in range(0, 100, 17):
            assert oracle.energy(n, w[r, k]) == e[r, k]


@pytest.mark.parametrize("kind", [capi.RNG_PHILOX, capi.RNG_MT19937_64])
@pytest.mark.parametrize("cross,repl", [(capi.CROSSOVER_ONE_POINT, capi.REPLACE_WORST),
                                        (capi.CROSSOVER_UNIFORM, capi.REPLACE_WORST),
                                        (capi.CROSSOVER_ONE_POINT, capi.REPLACE_RANDOM)])
def test_production_policies(ctx, oracle, kind, cross, repl):
    """One-point crossover, elite replacement, Philox: reproducible per seed,
    energies consistent, elite replacement never raises the population max."""
    n, R = 36, 16
    p = capi.memetic_params(target_energy=0, max_iterations=6, rng_kind=kind, crossover=cross,
                            replacement=repl, tie_rule=capi.TIE_LOWEST)
    a = capi.Solver(ctx, n, R, base_seed=9, params=p)
    a.run(epoch_iterations=1, race=False)
    w0, e0 = a.population()
    a.run(race=False)
    b = capi.Solver(ctx, n, R, base_seed=9, params=p)
    b.run(race=False)
    assert _results(a) == _results(b)
    w, e = a.population()
    for r in range(0, R, 5):
        for k in range(0, 100, 23):
            assert oracle.energy(n, w[r, k]) == e[r, k]
    if repl == capi.REPLACE_WORST:
        assert (e.max(axis=1) <= e0.max(axis=1)).all()
    for r in a.results():
        assert oracle.energy(n, r["best"]) == r["best_energy"]


def test_island_export_import(ctx):
    import torch
    n, R, k = 40, 32, 4
    sv = capi.Solver(ctx, n, R, base_seed=11, params=capi.memetic_params(max_iterations=3))
    sv.run(epoch_iterations=2, race=False)
    nw = 1
    d_w = torch.zeros(k * nw, dtype=torch.int64, device="cuda")
    d_e = torch.zeros(k, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    sv.export_elites(k, d_w.data_ptr(), d_e.data_ptr())
    sv.sync()
    res = sv.results()
    bestE = sorted(r["best_energy"] for r in res)
    got = d_e.cpu().tolist()
    assert got == bestE[:k]
    words = d_w.cpu().numpy().view(np.uint64)
    byE = {}
    for r in res:
        byE.setdefault(r["best_energy"], []).append(r["best"][0])
    for i in range(k):
        assert words[i] in byE[got[i]]
    # import an elite better than every member: each replica's worst slot takes it
    _, e_before = sv.population()
    elite_e = int(e_before.min()) - 1  # synthetic key, strictly better than all
    d_w2 = torch.tensor([int(words[0].astype(np.int64))], dtype=torch.int64, device="cuda")
    d_e2 = torch.tensor([elite_e], dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    sv.import_elites(1, d_w2.data_ptr(), d_e2.data_ptr(), rotation=0)
    sv.sync()
    w_after, e_after = sv.population()
    for r in range(R):
        if res[r]["iterations"] >= 3:
            continue  # finished replicas do not import
        worst = int(np.argmax(e_before[r]))
        assert e_after[r, worst] == elite_e
        assert w_after[r, worst, 0] == words[0]


def test_checkpoint_resume_is_exact(ctx):
    """Save after some epochs, resume in a fresh solver: the continued run is
    bit-identical to an uninterrupted one (SURVEY §5 checkpoint/resume)."""
    n, R = 52, 40
    for kind in (capi.RNG_MT19937_64, capi.RNG_PHILOX):
        p = capi.memetic_params(target_energy=0, max_iterations=10, rng_kind=kind)
        ref = capi.Solver(ctx, n, R, base_seed=77, params=p, trace_cap=16)
        ref.run(race=False)
        a = capi.Solver(ctx, n, R, base_seed=77, params=p, trace_cap=16)
        a.run(epoch_iterations=4, race=False)
        blob = a.save()
        a.close()
        b = capi.Solver(ctx, n, R, base_seed=77, params=p, trace_cap=16)
        b.load(blob)
        b.run(race=False)
        ra, rb = ref.results(), b.results()
        assert [(r["best"].tolist(), r["best_energy"], r["iterations"], r["trace"]) for r in ra] \
            == [(r["best"].tolist(), r["best_energy"], r["iterations"], r["trace"]) for r in rb]
        bad = capi.Solver(ctx, n + 1, R, base_seed=77, params=p, trace_cap=16)
        with pytest.raises(ValueError):
            bad.load(blob)
        # every trajectory-shaping setting is part of the checkpoint header
        for kw in ({"base_seed": 78}, {"replica_offset": 5},
                   {"params": capi.memetic_params(target_energy=3, max_iterations=10,
                                                  rng_kind=kind)},
                   {"params": capi.memetic_params(target_energy=0, max_iterations=10,
                                                  rng_kind=kind, p_comb=0.5)},
                   {"params": capi.memetic_params(target_energy=0, max_iterations=10,
                                                  rng_kind=kind, max_tabu_factor=0.2)},
                   {"params": capi.memetic_params(target_energy=0, max_iterations=11,
                                                  rng_kind=kind)}):
            args = {"base_seed": 77, "params": p, "trace_cap": 16, **kw}
            other = capi.Solver(ctx, n, R, **args)
            with pytest.raises(ValueError):
                other.load(blob)


def test_checkpoint_keeps_wall_times(ctx):
    """Finished replicas keep their wall time across save/load, and running
    ones continue their max_seconds budget (t0 was restamped)."""
    import time
    n, R = 40, 8
    p = capi.memetic_params(target_energy=0, max_iterations=3)
    a = capi.Solver(ctx, n, R, base_seed=9, params=p)
    a.run(race=False)
    before = [r["wall_seconds"] for r in a.results()]
    blob = a.save()
    time.sleep(0.3)
    b = capi.Solver(ctx, n, R, base_seed=9, params=p)
    b.load(blob)
    after = [r["wall_seconds"] for r in b.results()]
    assert all(x > 0 for x in before)
    assert after == pytest.approx(before, abs=2e-3)


def test_islands_driver_single_rank(ctx):
    """islands.Islands on one GPU (world 1): epochs, elite exchange through
    device buffers, stop on target."""
    import torch
    from paper_2504_00987_b200.islands import Islands
    n, R = 40, 64
    target = 108  # proven optimum (paper_2504_00987_b200/data/optima.txt)
    sv = capi.Solver(ctx, n, R, base_seed=3, params=capi.memetic_params(
        target_energy=target, max_seconds=120.0))
    isl = Islands(sv, n, k_elites=4, device=torch.device("cuda", 0))
    rep = isl.run(target=target, epoch_seconds=0.05, exchange_every=1, max_seconds=120.0)
    assert rep.reached and rep.best_energy == target
    assert rep.exchanges == rep.epochs and rep.epochs >= 1
    best = sv.results()[rep.best_replica]
    assert best["best_energy"] == target


def test_more_replicas_than_resident_warps(ctx, oracle):
    """Replicas beyond the resident capacity run in later waves of the same
    persistent grid; each is still the reference trajectory of its seed."""
    n = 20
    cap = capi.Solver.capacity(ctx, n)
    R = cap + 37
    p = capi.memetic_params(target_energy=0, max_iterations=2)
    best, per = ctx.run_replicas(n, R, 500, p)
    for r in (0, 1, cap - 1, cap, R - 1):
        want = oracle.memetic(n, 500 + r, max_iterations=2)
        assert per[r]["best"].tolist() == want["best"]
        assert per[r]["best_energy"] == want["best_energy"]
    assert best["best_energy"] == min(x["best_energy"] for x in per)


@pytest.mark.parametrize("kind", [capi.RNG_PHILOX, capi.RNG_MT19937_64])
@pytest.mark.parametrize("n,asp,tie", [(30, 0, capi.TIE_REFERENCE), (64, 1, capi.TIE_LOWEST),
                                       (50, 0, capi.TIE_REFERENCE)])
def test_tile_widths_agree(ctx, monkeypatch, kind, n, asp, tie):
    """K4 with two replicas per warp (16-lane tiles) and with one per warp
    runs every replica through the same trajectory: both RNG streams are
    defined per draw, independent of the tile width. Odd replica counts leave
    a half-idle warp at the end of the grid."""
    p = capi.memetic_params(target_energy=0, max_iterations=4, rng_kind=kind,
                            tie_rule=tie, aspiration=bool(asp))
    out = {}
    for tile in ("32", "16"):
        monkeypatch.setenv("LABS_TILE", tile)
        sv = capi.Solver(ctx, n, 37, base_seed=11, params=p)
        sv.run(race=False)
        out[tile] = (_results(sv), sv.population()[1].tolist())
        sv.close()
    assert out["16"] == out["32"]


def test_run_replicas_multi_matches_single_gpu(ctx, oracle):
    """labs_run_replicas_multi over two contexts of one device: contiguous
    replica blocks (4 + 3), seeds base + r, every replica equal to the oracle
    and to the single-GPU run; winner = strictly lowest energy."""
    n, R, base = 36, 7, 321
    p = capi.memetic_params(target_energy=0, max_iterations=5)
    ctx2 = capi.Context(0)
    best, per = capi.run_replicas_multi([ctx, ctx2], n, R, base, p, trace_cap=8)
    b1, per1 = ctx.run_replicas(n, R, base, p, trace_cap=8)
    _, ref = oracle.run_replicas(n, R, base, target_energy=0, max_iterations=5)
    for r in range(R):
        assert per[r]["replica_id"] == r and per[r]["seed"] == base + r
        for k in ("best_energy", "iterations", "seed"):
            assert per[r][k] == per1[r][k] == ref[r][k]
        assert per[r]["best"].tolist() == per1[r]["best"].tolist() == ref[r]["best"]
        assert per[r]["trace"] == per1[r]["trace"]
    assert best["best_energy"] == min(x["best_energy"] for x in per)
    one, _ = capi.run_replicas_multi([ctx], n, R, base, p)
    # Ties go to the first publisher, which is completion order on the device
    # (as in the reference's threaded run), so two runs may pick different
    # members of the tie.
    ties = {r for r in range(R) if per[r]["best_energy"] == best["best_energy"]}
    assert one["best_energy"] == b1["best_energy"] == best["best_energy"]
    assert {one["replica_id"], b1["replica_id"], best["replica_id"]} <= ties
    with pytest.raises(ValueError):
        capi.run_replicas_multi([], n, R, base, p)
    ctx2.close()


def test_run_replicas_multi_cross_island_stop(ctx):
    """A target reached on island 1 stops island 0 through the peer flag:
    n=37, target 86, seed 2011 needs 18138 iterations and seed 2012 489
    (oracle), one replica per island."""
    ctx2 = capi.Context(0)
    p = capi.memetic_params(target_energy=86, max_seconds=120.0)
    best, per = capi.run_replicas_multi([ctx, ctx2], 37, 2, 2011, p)
    assert best["reached_target"] and best["replica_id"] == 1 and best["iterations"] == 489
    assert not per[0]["reached_target"] and per[0]["iterations"] < 18138
    ctx2.close()
