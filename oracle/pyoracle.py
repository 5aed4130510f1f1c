"""ctypes bindings for the parity oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, both built by oracle/Makefile:

* ``Oracle``   — oracle/build/liblabs_oracle.so, the C restatement of the
  reference algorithm (labs_oracle.c; every function cites its
  /root/reference/proj file:line).
* ``Reference`` — oracle/_ref/libref_labsolve.so, the unmodified reference
  sources plus the probe harness ref_capi.cpp. Optional: present only when the
  reference tree was available at build time (it ships to the GPU box as a
  prebuilt .so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liblabs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_labsolve.so")

LO_MAXN = 1024
LO_MAXW = LO_MAXN // 64

u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)


def nwords(n: int) -> int:
    return (n + 63) // 64


def _p(arr, ty):
    return arr.ctypes.data_as(ty)


class LoRng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int)]


class LoState(C.Structure):
    _fields_ = [("n", C.c_int), ("w", C.c_uint64 * LO_MAXW),
                ("C", C.c_int32 * LO_MAXN), ("E", C.c_int64)]


class LoScanResult(C.Structure):
    _fields_ = [("position", C.c_int), ("energy", C.c_int64), ("fallback", C.c_int)]


class LoTabuStep(C.Structure):
    _fields_ = [("iteration", C.c_int), ("position", C.c_int), ("energy", C.c_int64),
                ("tenure", C.c_int), ("fallback", C.c_int)]


class LoTabuInfo(C.Structure):
    _fields_ = [("max_iter", C.c_int), ("min_tabu", C.c_int), ("max_tabu", C.c_int)]


class LoMemeticParams(C.Structure):
    _fields_ = [("population_size", C.c_int), ("p_comb", C.c_double),
                ("p_mutate", C.c_double), ("target_energy", C.c_int64),
                ("max_seconds", C.c_double), ("max_iterations", C.c_int64),
                ("min_tabu_factor", C.c_double), ("max_tabu_factor", C.c_double)]


class LoRunResult(C.Structure):
    _fields_ = [("best", C.c_uint64 * LO_MAXW), ("best_energy", C.c_int64),
                ("iterations", C.c_int64), ("wall_seconds", C.c_double),
                ("seed", C.c_uint64), ("replica_id", C.c_int),
                ("reached_target", C.c_int)]


class RefResult(C.Structure):
    _fields_ = [("best", C.c_uint64 * 16), ("best_energy", C.c_int64),
                ("iterations", C.c_int64), ("wall_seconds", C.c_double),
                ("seed", C.c_uint64), ("replica_id", C.c_int32),
                ("reached_target", C.c_int32)]


def _result_dict(r, n):
    return {"best": [int(r.best[i]) for i in range(nwords(n))],
            "best_energy": int(r.best_energy), "iterations": int(r.iterations),
            "wall_seconds": float(r.wall_seconds), "seed": int(r.seed),
            "replica_id": int(r.replica_id), "reached_target": bool(r.reached_target)}


class Oracle:
    """The C restatement (labs_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle not built: {path} (run make -C oracle)")
        L = self.lib = C.CDLL(path)
        L.lo_rng_seed.argtypes = [C.POINTER(LoRng), C.c_uint64]
        L.lo_rng_bits64.argtypes = [C.POINTER(LoRng)]
        L.lo_rng_bits64.restype = C.c_uint64
        L.lo_rng_uniform_int.argtypes = [C.POINTER(LoRng), C.c_int64, C.c_int64]
        L.lo_rng_uniform_int.restype = C.c_int64
        L.lo_rng_uniform01.argtypes = [C.POINTER(LoRng)]
        L.lo_rng_uniform01.restype = C.c_double
        L.lo_seq_random.argtypes = [C.c_int, C.POINTER(LoRng), u64p]
        L.lo_energy.argtypes = [C.c_int, u64p]
        L.lo_energy.restype = C.c_int64
        L.lo_state_build.argtypes = [C.POINTER(LoState), C.c_int, u64p]
        L.lo_neighbor_energy.argtypes = [C.POINTER(LoState), C.c_int]
        L.lo_neighbor_energy.restype = C.c_int64
        L.lo_apply_flip.argtypes = [C.POINTER(LoState), C.c_int]
        L.lo_scan.argtypes = [C.POINTER(LoState), u8p, C.POINTER(LoRng), C.c_int,
                              C.POINTER(LoScanResult), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lo_scan.restype = C.c_int
        L.lo_tabu_search.argtypes = [C.c_int, u64p, C.c_double, C.c_double,
                                     C.POINTER(LoRng), u64p, i64p, C.POINTER(LoTabuInfo),
                                     C.POINTER(LoTabuStep)]
        L.lo_tabu_search.restype = C.c_int
        L.lo_memetic_defaults.argtypes = [C.POINTER(LoMemeticParams)]
        L.lo_memetic_tabu.argtypes = [C.c_int, C.POINTER(LoMemeticParams), C.c_uint64,
                                      C.POINTER(C.c_int), C.c_int, C.POINTER(LoRunResult),
                                      i64p, C.c_int64]
        L.lo_memetic_tabu.restype = C.c_int
        L.lo_run_replicas_sequential.argtypes = [C.c_int, C.c_int, C.c_uint64,
                                                 C.POINTER(LoMemeticParams),
                                                 C.POINTER(LoRunResult), C.POINTER(LoRunResult)]
        L.lo_run_replicas_sequential.restype = C.c_int
        L.lo_tabu_throughput.argtypes = [C.c_int, C.c_int, C.c_double, i64p,
                                         C.POINTER(C.c_double)]
        L.lo_tabu_throughput.restype = C.c_int64

    # -- rng --------------------------------------------------------------
    def rng(self, seed: int) -> LoRng:
        r = LoRng()
        self.lib.lo_rng_seed(C.byref(r), C.c_uint64(seed))
        return r

    def random_sequence(self, n: int, rng: LoRng) -> np.ndarray:
        w = np.zeros(nwords(n), dtype=np.uint64)
        self.lib.lo_seq_random(n, C.byref(rng), _p(w, u64p))
        return w

    def energy(self, n: int, words) -> int:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        return int(self.lib.lo_energy(n, _p(w, u64p)))

    def state(self, n: int, words) -> LoState:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        st = LoState()
        self.lib.lo_state_build(C.byref(st), n, _p(w, u64p))
        return st

    def probe(self, n: int, words):
        """(C[1..n-1], E, neighbor energies[n]) — correlation_state.cpp:9-71."""
        st = self.state(n, words)
        corr = np.array([st.C[k] for k in range(n - 1)], dtype=np.int64)
        nb = np.array([self.lib.lo_neighbor_energy(C.byref(st), j) for j in range(n)],
                      dtype=np.int64)
        return corr, int(st.E), nb

    def scan(self, n, words, admissible, rng: LoRng, allow_fallback=True):
        st = self.state(n, words)
        adm = np.ascontiguousarray(admissible, dtype=np.uint8)
        out = LoScanResult()
        ntie = C.c_int(0)
        ties = (C.c_int * n)()
        rc = self.lib.lo_scan(C.byref(st), _p(adm, u8p), C.byref(rng),
                              1 if allow_fallback else 0, C.byref(out), C.byref(ntie), ties)
        if rc != 0:
            raise RuntimeError("no admissible position in neighborhood scan")
        return {"position": out.position, "energy": int(out.energy),
                "fallback": bool(out.fallback), "ties": [ties[i] for i in range(ntie.value)]}

    def tabu(self, n, start, rng: LoRng, fmin=0.10, fmax=0.12, trace=True):
        w = np.ascontiguousarray(start, dtype=np.uint64)
        best = np.zeros(nwords(n), dtype=np.uint64)
        be = C.c_int64(0)
        info = LoTabuInfo()
        steps = (LoTabuStep * (3 * n // 2 + 2))() if trace else None
        rc = self.lib.lo_tabu_search(n, _p(w, u64p), fmin, fmax, C.byref(rng), _p(best, u64p),
                                     C.byref(be), C.byref(info), steps)
        if rc != 0:
            raise ValueError("tabu tenure factors need 0 <= min <= max < 1, n >= 2")
        out = {"best": best, "energy": int(be.value), "max_iter": info.max_iter,
               "min_tabu": info.min_tabu, "max_tabu": info.max_tabu}
        if trace:
            out["steps"] = [(s.iteration, s.position, int(s.energy), s.tenure, bool(s.fallback))
                            for s in steps[:info.max_iter]]
        return out

    def params(self, **kw) -> LoMemeticParams:
        p = LoMemeticParams()
        self.lib.lo_memetic_defaults(C.byref(p))
        for k, v in kw.items():
            setattr(p, k, v)
        return p

    def memetic(self, n, seed, child_cap=None, **kw):
        p = self.params(**kw)
        out = LoRunResult()
        ce = np.zeros(max(child_cap or 0, 1), dtype=np.int64)
        rc = self.lib.lo_memetic_tabu(n, C.byref(p), C.c_uint64(seed), None, 0, C.byref(out),
                                      _p(ce, i64p), child_cap or 0)
        if rc != 0:
            raise ValueError("invalid memetic parameters")
        d = _result_dict(out, n)
        if child_cap is not None:
            d["child_energies"] = ce[:min(child_cap, d["iterations"])].tolist()
        return d

    def run_replicas(self, n, replicas, base_seed, **kw):
        p = self.params(**kw)
        out = LoRunResult()
        per = (LoRunResult * replicas)()
        rc = self.lib.lo_run_replicas_sequential(n, replicas, C.c_uint64(base_seed), C.byref(p),
                                                 C.byref(out), per)
        if rc != 0:
            raise ValueError("invalid run parameters")
        return _result_dict(out, n), [_result_dict(per[i], n) for i in range(replicas)]

    def tabu_throughput(self, n, threads, seconds):
        walks = C.c_int64(0)
        el = C.c_double(0)
        it = self.lib.lo_tabu_throughput(n, threads, seconds, C.byref(walks), C.byref(el))
        return int(it), int(walks.value), float(el.value)


class Reference:
    """The unmodified reference library (oracle/_ref), via ref_capi.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference build absent: {path}")
        L = self.lib = C.CDLL(path)
        L.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.POINTER(C.c_int), i64p, i64p, u64p]
        L.ref_random_sequences.argtypes = [C.c_int, C.c_uint64, C.c_int, u64p]
        L.ref_energy.argtypes = [C.c_int, u64p]
        L.ref_energy.restype = C.c_int64
        L.ref_state_probe.argtypes = [C.c_int, u64p, i64p, i64p, i64p]
        L.ref_scan.argtypes = [C.c_int, u64p, u8p, C.c_uint64, C.c_int, C.c_int,
                               C.POINTER(C.c_int), i64p, C.POINTER(C.c_int)]
        L.ref_scan.restype = C.c_int
        L.ref_tabu.argtypes = [C.c_int, u64p, C.c_double, C.c_double, C.c_uint64, C.c_int,
                               u64p, i64p, C.POINTER(C.c_int), i64p, C.c_int, u64p]
        L.ref_tabu.restype = C.c_int
        L.ref_memetic.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int64,
                                  C.c_double, C.c_int64, C.c_double, C.c_double, C.c_uint64,
                                  C.POINTER(RefResult), i64p, C.c_int64]
        L.ref_memetic.restype = C.c_int
        L.ref_run_replicas.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_double,
                                       C.c_double, C.c_int64, C.c_double, C.c_int64,
                                       C.c_double, C.c_double, C.c_int,
                                       C.POINTER(RefResult), C.POINTER(RefResult)]
        L.ref_run_replicas.restype = C.c_int
        L.ref_tabu_throughput.argtypes = [C.c_int, C.c_int, C.c_double, i64p,
                                          C.POINTER(C.c_double)]
        L.ref_tabu_throughput.restype = C.c_int64
        L.ref_brute_force.argtypes = [C.c_int, C.c_int, i64p, u64p, C.c_int]
        L.ref_brute_force.restype = C.c_int
        L.ref_local_optima.argtypes = [C.c_int, C.c_int]
        L.ref_local_optima.restype = C.c_int64
        L.ref_deviation.argtypes = [C.c_int, u64p, C.c_uint64, C.c_int, i64p]
        L.ref_deviation.restype = C.c_int

    def deviation(self, n, words, budget=0, edits=False):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        out = np.zeros(3, dtype=np.int64)
        if self.lib.ref_deviation(n, _p(w, u64p), C.c_uint64(budget), 1 if edits else 0,
                                  _p(out, i64p)) != 0:
            raise ValueError("deviation failed")
        return {"value": int(out[0]), "budget_exceeded": bool(out[1]),
                "evaluations": int(out[2])}

    def brute_force(self, n, workers=8, cap=4096):
        e = C.c_int64(0)
        w = np.zeros(cap * nwords(n), dtype=np.uint64)
        c = self.lib.ref_brute_force(n, workers, C.byref(e), _p(w, u64p), cap)
        if c < 0:
            raise ValueError("brute force failed")
        return int(e.value), w[:c * nwords(n)].reshape(c, nwords(n))

    def local_optima(self, n, workers=8):
        return int(self.lib.ref_local_optima(n, workers))

    def rng_draws(self, seed, kinds, lo=None, hi=None):
        k = np.ascontiguousarray(kinds, dtype=np.int32)
        lo = np.ascontiguousarray(lo if lo is not None else np.zeros(len(k)), dtype=np.int64)
        hi = np.ascontiguousarray(hi if hi is not None else np.zeros(len(k)), dtype=np.int64)
        out = np.zeros(len(k), dtype=np.uint64)
        self.lib.ref_rng_draws(C.c_uint64(seed), len(k), k.ctypes.data_as(C.POINTER(C.c_int)),
                               _p(lo, i64p), _p(hi, i64p), _p(out, u64p))
        return out

    def random_sequences(self, n, seed, count):
        w = np.zeros(count * nwords(n), dtype=np.uint64)
        self.lib.ref_random_sequences(n, C.c_uint64(seed), count, _p(w, u64p))
        return w.reshape(count, nwords(n))

    def energy(self, n, words):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        return int(self.lib.ref_energy(n, _p(w, u64p)))

    def probe(self, n, words):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        corr = np.zeros(max(n - 1, 1), dtype=np.int64)
        e = C.c_int64(0)
        nb = np.zeros(n, dtype=np.int64)
        self.lib.ref_state_probe(n, _p(w, u64p), _p(corr, i64p), C.byref(e), _p(nb, i64p))
        return corr[:n - 1], int(e.value), nb

    def scan(self, n, words, admissible, draw_seed, workers=1, allow_fallback=True):
        w = np.ascontiguousarray(words, dtype=np.uint64)
        adm = np.ascontiguousarray(admissible, dtype=np.uint8)
        pos, fb = C.c_int(0), C.c_int(0)
        e = C.c_int64(0)
        rc = self.lib.ref_scan(n, _p(w, u64p), _p(adm, u8p), C.c_uint64(draw_seed), workers,
                               1 if allow_fallback else 0, C.byref(pos), C.byref(e), C.byref(fb))
        if rc != 0:
            raise RuntimeError("no admissible position in neighborhood scan")
        return {"position": pos.value, "energy": int(e.value), "fallback": bool(fb.value)}

    def tabu(self, n, start, seed, fmin=0.10, fmax=0.12, workers=1):
        w = np.ascontiguousarray(start, dtype=np.uint64)
        best = np.zeros(nwords(n), dtype=np.uint64)
        be = C.c_int64(0)
        info = (C.c_int * 3)()
        cap = 3 * n // 2 + 2
        steps = np.zeros(5 * cap, dtype=np.int64)
        post = C.c_uint64(0)
        m = self.lib.ref_tabu(n, _p(w, u64p), fmin, fmax, C.c_uint64(seed), workers,
                              _p(best, u64p), C.byref(be), info, _p(steps, i64p), cap,
                              C.byref(post))
        if m < 0:
            raise ValueError("invalid tabu arguments")
        st = steps[:5 * m].reshape(m, 5)
        return {"best": best, "energy": int(be.value), "max_iter": info[0], "min_tabu": info[1],
                "max_tabu": info[2],
                "steps": [(int(a), int(b), int(c), int(d), bool(e)) for a, b, c, d, e in st],
                "post_draw": int(post.value)}

    def memetic(self, n, seed, population_size=100, p_comb=0.9, p_mutate=-1.0,
                target_energy=0, max_seconds=-1.0, max_iterations=-1,
                min_tabu_factor=0.10, max_tabu_factor=0.12, child_cap=0):
        out = RefResult()
        ce = np.zeros(max(child_cap, 1), dtype=np.int64)
        rc = self.lib.ref_memetic(n, population_size, p_comb, p_mutate, target_energy,
                                  max_seconds, max_iterations, min_tabu_factor, max_tabu_factor,
                                  C.c_uint64(seed), C.byref(out), _p(ce, i64p), child_cap)
        if rc != 0:
            raise ValueError("invalid memetic parameters")
        d = _result_dict(out, n)
        if child_cap:
            d["child_energies"] = ce[:min(child_cap, d["iterations"])].tolist()
        return d

    def run_replicas(self, n, replicas, base_seed, threaded=False, population_size=100,
                     p_comb=0.9, p_mutate=-1.0, target_energy=0, max_seconds=-1.0,
                     max_iterations=-1, min_tabu_factor=0.10, max_tabu_factor=0.12):
        out = RefResult()
        per = (RefResult * replicas)()
        rc = self.lib.ref_run_replicas(n, replicas, C.c_uint64(base_seed), population_size,
                                       p_comb, p_mutate, target_energy, max_seconds,
                                       max_iterations, min_tabu_factor, max_tabu_factor,
                                       1 if threaded else 0, C.byref(out), per)
        if rc != 0:
            raise ValueError("invalid run parameters")
        return _result_dict(out, n), [_result_dict(per[i], n) for i in range(replicas)]

    def tabu_throughput(self, n, threads, seconds):
        walks = C.c_int64(0)
        el = C.c_double(0)
        it = self.lib.ref_tabu_throughput(n, threads, seconds, C.byref(walks), C.byref(el))
        return int(it), int(walks.value), float(el.value)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def double_bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]
