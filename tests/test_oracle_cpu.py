"""CPU tests: pin the oracle (oracle/labs_oracle.c) against the reference's
golden vectors, and prove the O(n)-per-step update identities the CUDA walker
uses (labs_walker.cuh header) on random flip traces."""
import numpy as np
import pytest

from oracle.pyoracle import Reference, double_bits, reference_available
from paper_2504_00987_b200.sequence import decode_hex, encode_hex, energy_naive, spins


def test_rng_streams_match_reference(golden, oracle):
    """Rng::bits64 / uniform_int / uniform01 (rng.hpp:10-28) bit for bit."""
    for case in golden["rng"]:
        r = oracle.rng(case["seed"])
        for k, lo, hi, want in zip(case["kinds"], case["lo"], case["hi"], case["out"]):
            if k == 0:
                got = oracle.lib.lo_rng_bits64(r)
            elif k == 1:
                got = oracle.lib.lo_rng_uniform_int(r, lo, hi) & (2**64 - 1)
            else:
                got = double_bits(oracle.lib.lo_rng_uniform01(r))
            assert got == want


def test_kats(golden, oracle):
    k = golden["kats"]
    corr, e, nb = oracle.probe(5, np.zeros(1, dtype=np.uint64))
    assert e == k["all_plus_5"]["E"] and corr.tolist() == k["all_plus_5"]["C"]
    corr, e, nb = oracle.probe(4, np.zeros(1, dtype=np.uint64))
    assert e == 14 and nb.tolist() == [2, 2, 2, 2]
    w = decode_hex(k["n92"]["hex"], 92)
    assert oracle.energy(92, w) == 490


def test_hex_codec_and_table(golden, oracle):
    for row in golden["table"]:
        w = decode_hex(row["hex"], row["n"])
        assert encode_hex(w, row["n"]) == row["hex"]
        assert oracle.energy(row["n"], w) == row["E"]
        assert energy_naive(w, row["n"]) == row["E"]
    # "8" -> spin(0) = -1 (test_sequence.cpp:50-57): bit 1 is spin -1.
    assert spins(decode_hex("8", 4), 4).tolist() == [-1, 1, 1, 1]
    with pytest.raises(ValueError):
        decode_hex("F", 3)  # nonzero padding bit
    with pytest.raises(ValueError):
        decode_hex("G", 4)


def test_state_probes(golden, oracle):
    for p in golden["probes"]:
        corr, e, nb = oracle.probe(p["n"], p["words"])
        assert e == p["E"]
        assert corr.tolist() == p["C"]
        assert nb.tolist() == p["neighbors"]


def test_scans(golden, oracle):
    for s in golden["scans"]:
        r = oracle.scan(s["n"], s["words"], s["admissible"], oracle.rng(s["draw_seed"]))
        assert (r["position"], r["energy"], r["fallback"]) == (s["position"], s["energy"],
                                                               s["fallback"])


def test_tabu_walks(golden, oracle):
    for wk in golden["walks"]:
        r = oracle.rng(wk["seed"])
        out = oracle.tabu(wk["n"], wk["start"], r, wk["min_factor"], wk["max_factor"])
        assert out["steps"] == [tuple(s) for s in wk["steps"]]
        assert out["energy"] == wk["energy"]
        assert out["best"].tolist() == wk["best"]
        assert (out["max_iter"], out["min_tabu"], out["max_tabu"]) == (
            wk["max_iter"], wk["min_tabu"], wk["max_tabu"])
        assert oracle.lib.lo_rng_bits64(r) == wk["post_draw"]


def test_memetic(golden, oracle):
    for m in golden["memetic"]:
        d = oracle.memetic(m["n"], m["seed"], child_cap=len(m["child_energies"]), **m["params"])
        assert d["best_energy"] == m["best_energy"]
        assert d["iterations"] == m["iterations"]
        assert d["best"] == m["best"]
        assert d["reached_target"] == m["reached_target"]
        assert d["child_energies"] == m["child_energies"]
    # README.md:114-117 — the one published trajectory pin.
    d = oracle.memetic(20, 43, target_energy=26)
    assert (d["best_energy"], d["iterations"], encode_hex(d["best"], 20)) == (26, 98, "C9EF5")


def test_run_replicas_sequential(golden, oracle):
    for c in golden["replicas"]:
        its = c["max_iterations"]
        best, per = oracle.run_replicas(c["n"], c["replicas"], c["base_seed"],
                                        target_energy=c.get("target_energy", 0),
                                        max_iterations=-1 if its is None else its)
        for a, b in zip(per, c["per_replica"]):
            for k in ("best", "best_energy", "iterations", "seed", "replica_id",
                      "reached_target"):
                assert a[k] == b[k], k
        assert best["best_energy"] == c["best"]["best_energy"]
        assert best["replica_id"] == c["best"]["replica_id"]


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference():
    """Random cases beyond the fixtures, against the compiled reference."""
    from oracle.pyoracle import Oracle
    o, ref = Oracle(), Reference()
    rs = np.random.default_rng(7)
    for i in range(40):
        n = int(rs.integers(2, 200))
        start = ref.random_sequences(n, 10_000 + i, 1)[0]
        a = ref.tabu(n, start, 20_000 + i)
        b = o.tabu(n, start, o.rng(20_000 + i))
        assert a["steps"] == b["steps"] and a["energy"] == b["energy"]


def _vectors(s):
    n = len(s)
    C = np.array([np.dot(s[:n - k], s[k:]) if k else n for k in range(n)])
    Q = np.array([sum(s[i] * s[m - i] for i in range(n) if 0 <= m - i < n)
                  for m in range(2 * n - 1)])
    h = np.array([sum(C[abs(i - j)] * s[i] for i in range(n) if i != j) for j in range(n)])
    return C, Q, h


def test_incremental_identities(oracle):
    """The walker's O(n) update (labs_walker.cuh) against the oracle's
    neighbor_energy after every flip of random traces."""
    rs = np.random.default_rng(11)
    for trial in range(60):
        n = int(rs.integers(2, 48))
        s = rs.choice([-1, 1], size=n)
        C, Q, h = _vectors(s)
        E = int(sum(int(c) ** 2 for c in C[1:]))
        for step in range(25):
            dE = 4 * (n - 2 + Q[2 * np.arange(n)] - s * h)
            words = np.zeros((n + 63) // 64, dtype=np.uint64)
            for i in range(n):
                if s[i] < 0:
                    words[i >> 6] |= np.uint64(1 << (i & 63))
            corr, e, nb = oracle.probe(n, words)
            assert e == E and (nb - E).tolist() == dE.tolist()
            p = int(rs.integers(0, n))
            sg = int(s[p])
            sv = lambda i: int(s[i]) if 0 <= i < n else 0  # noqa: E731
            nC = C.copy()
            for k in range(1, n):
                nC[k] = C[k] - 2 * sg * (sv(p - k) + sv(p + k))
            nQ = Q.copy()
            for j in range(n):
                if j != p:
                    nQ[p + j] = Q[p + j] - 4 * sg * s[j]
            nh = h.copy()
            for j in range(n):
                if j != p:
                    nh[j] = h[j] - 4 * sg * C[abs(j - p)] + 4 * sv(2 * p - j) \
                        - 2 * sg * Q[p + j] + 8 * s[j]
                else:
                    nh[j] = h[j] - 2 * sg * (n - 2 + Q[2 * p])
            E += int(dE[p])
            s = s.copy()
            s[p] = -s[p]
            C, Q, h = nC, nQ, nh
            C2, Q2, h2 = _vectors(s)
            assert (C[1:] == C2[1:]).all() and (Q == Q2).all() and (h == h2).all()
