"""ctypes mirror of the C ABI in include/labs_b200.h.

This is the Python face of the B200 path (tests and bench.py call through it;
the C++ drop-in in include/labsolve/ calls the same entry points). Every call
goes to lib/liblabs_b200.so — there is no CPU fallback: if the library or a
CUDA device is missing, construction raises.

Reference interface mirrored (names, argument meaning, error classes):
/root/reference/proj/include/labsolve/{correlation_state,tabu,memetic,
parallel}.hpp. Errors map back to the reference's exception classes:
LABS_ERR_INVALID_ARGUMENT -> ValueError (std::invalid_argument),
LABS_ERR_OUT_OF_RANGE -> IndexError (std::out_of_range),
LABS_ERR_RUNTIME -> RuntimeError (std::runtime_error),
LABS_ERR_CUDA -> LabsCudaError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LABS_LIB_PATH") or os.path.join(HERE, "lib", "liblabs_b200.so")

LABS_OK = 0
LABS_ERR_INVALID_ARGUMENT = 1
LABS_ERR_OUT_OF_RANGE = 2
LABS_ERR_RUNTIME = 3
LABS_ERR_CUDA = 4
LABS_MAX_N = 256
LABS_MAX_WORDS = 4
LABS_MAX_PEERS = 15
LABS_IPC_HANDLE_BYTES = 64
RNG_MT19937_64 = 0
RNG_PHILOX = 1
TIE_REFERENCE = 0
TIE_LOWEST = 1

# Every symbol include/labs_b200.h declares (checked by tests/test_capi_cpu.py).
EXPORTS = [
    "labs_last_error", "labs_ctx_create", "labs_ctx_destroy", "labs_ctx_stream",
    "labs_ctx_sm_count", "labs_ctx_synchronize", "labs_max_n", "labs_rng_seed",
    "labs_build_state", "labs_flip_trace", "labs_scan", "labs_tabu_walks",
    "labs_tabu_walks_device", "labs_rng_seed_device", "labs_memetic",
    "labs_run_replicas", "labs_solver_create", "labs_solver_destroy", "labs_solver_capacity",
    "labs_solver_run", "labs_solver_request_stop", "labs_solver_status", "labs_solver_counters",
    "labs_solver_results", "labs_solver_export_elites", "labs_solver_import_elites",
    "labs_bench_int_peak", "labs_exhaustive_optimum", "labs_local_optima",
    "labs_solver_population", "labs_solver_state_size", "labs_solver_save", "labs_solver_load",
    "labs_solver_stop_flag", "labs_solver_set_peer_stops", "labs_ipc_export", "labs_ipc_open",
    "labs_ipc_close", "labs_run_replicas_multi", "labs_bench_imad_peak",
    "labs_eval_create", "labs_eval_destroy", "labs_eval_run", "labs_skew_deviation",
]
CROSSOVER_UNIFORM = 0
CROSSOVER_ONE_POINT = 1
REPLACE_RANDOM = 0
REPLACE_WORST = 1


class LabsCudaError(RuntimeError):
    pass


class RngState(C.Structure):
    """labs_rng_state: mt19937_64 engine (312 words + next index)."""
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int32), ("pad_", C.c_int32)]


class TabuParams(C.Structure):
    _fields_ = [("min_tabu_factor", C.c_double), ("max_tabu_factor", C.c_double),
                ("tie_rule", C.c_int32), ("aspiration", C.c_int32)]


class TabuStep(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("position", C.c_int32), ("energy", C.c_int64),
                ("tenure", C.c_int32), ("fallback", C.c_int32)]


class MemeticParams(C.Structure):
    _fields_ = [("population_size", C.c_int32), ("rng_kind", C.c_int32),
                ("p_comb", C.c_double), ("p_mutate", C.c_double),
                ("target_energy", C.c_int64), ("max_seconds", C.c_double),
                ("max_iterations", C.c_int64), ("tabu", TabuParams),
                ("crossover", C.c_int32), ("replacement", C.c_int32)]


class RunResult(C.Structure):
    _fields_ = [("best", C.c_uint64 * LABS_MAX_WORDS), ("best_energy", C.c_int64),
                ("merit", C.c_double), ("iterations", C.c_int64),
                ("wall_seconds", C.c_double), ("seed", C.c_uint64),
                ("replica_id", C.c_int32), ("reached_target", C.c_int32),
                ("tabu_iterations", C.c_int64)]


class MemeticRecord(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("stop_seen", C.c_int32), ("pad_", C.c_int32),
                ("child_energy", C.c_int64)]


def tabu_params(min_tabu_factor=0.10, max_tabu_factor=0.12, tie_rule=TIE_REFERENCE,
                aspiration=False) -> TabuParams:
    """TabuParams defaults (proj/include/labsolve/tabu.hpp:11-14)."""
    return TabuParams(min_tabu_factor, max_tabu_factor, tie_rule, 1 if aspiration else 0)


def memetic_params(population_size=100, p_comb=0.9, p_mutate=None, target_energy=0,
                   max_seconds=None, max_iterations=None, rng_kind=RNG_MT19937_64,
                   crossover=CROSSOVER_UNIFORM, replacement=REPLACE_RANDOM,
                   **tabu_kw) -> MemeticParams:
    """MemeticParams defaults (proj/include/labsolve/memetic.hpp:15-24); the
    reference policies are the defaults of every switch."""
    return MemeticParams(population_size, rng_kind, p_comb,
                         -1.0 if p_mutate is None else float(p_mutate), int(target_energy),
                         -1.0 if max_seconds is None else float(max_seconds),
                         -1 if max_iterations is None else int(max_iterations),
                         tabu_params(**tabu_kw), crossover, replacement)


u64p = C.POINTER(C.c_uint64)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)


def _ptr(a, ty):
    return a.ctypes.data_as(ty)


def nwords(n: int) -> int:
    return (n + 63) // 64


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load lib/liblabs_b200.so; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: build it with __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(path)
    L.labs_last_error.restype = C.c_char_p
    L.labs_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
    L.labs_ctx_destroy.argtypes = [C.c_void_p]
    L.labs_ctx_stream.argtypes = [C.c_void_p]
    L.labs_ctx_stream.restype = C.c_void_p
    L.labs_ctx_sm_count.argtypes = [C.c_void_p]
    L.labs_ctx_synchronize.argtypes = [C.c_void_p]
    L.labs_rng_seed.argtypes = [C.c_uint64, C.POINTER(RngState)]
    L.labs_rng_seed.restype = None
    L.labs_build_state.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, i32p, i64p, i64p]
    L.labs_flip_trace.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, C.c_int, i32p, i64p,
                                  i64p]
    L.labs_scan.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, u8p, C.POINTER(RngState),
                            C.c_int, C.c_int, i32p, i64p, i32p, i32p, u64p]
    L.labs_tabu_walks.argtypes = [C.c_void_p, C.c_int, C.c_int, u64p, C.POINTER(TabuParams),
                                  C.POINTER(RngState), u64p, i64p, i32p, C.POINTER(TabuStep)]
    L.labs_tabu_walks_device.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                         C.POINTER(TabuParams), C.c_int, C.c_void_p,
                                         C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
    L.labs_rng_seed_device.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_void_p]
    L.labs_memetic.argtypes = [C.c_void_p, C.c_int, C.POINTER(MemeticParams), C.c_uint64,
                               i32p, C.c_int, C.POINTER(RunResult), C.POINTER(MemeticRecord),
                               C.c_int64, i64p]
    L.labs_run_replicas.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64,
                                    C.POINTER(MemeticParams), C.POINTER(RunResult),
                                    C.POINTER(RunResult), C.POINTER(MemeticRecord), C.c_int64,
                                    i64p]
    L.labs_solver_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_uint64, C.c_int64,
                                     C.POINTER(MemeticParams), C.c_int64,
                                     C.POINTER(C.c_void_p)]
    L.labs_solver_destroy.argtypes = [C.c_void_p]
    L.labs_solver_capacity.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.labs_solver_run.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_int]
    L.labs_solver_request_stop.argtypes = [C.c_void_p]
    L.labs_solver_status.argtypes = [C.c_void_p, i32p, i64p, i32p]
    L.labs_solver_counters.argtypes = [C.c_void_p, u64p, i64p]
    L.labs_solver_results.argtypes = [C.c_void_p, C.POINTER(RunResult),
                                      C.POINTER(MemeticRecord), i64p, i32p]
    L.labs_solver_export_elites.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.labs_solver_import_elites.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_int]
    L.labs_bench_int_peak.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    L.labs_bench_imad_peak.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
    L.labs_eval_create.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
    L.labs_eval_destroy.argtypes = [C.c_void_p]
    L.labs_eval_run.argtypes = [C.c_void_p, u64p, i32p, i64p, i64p]
    L.labs_skew_deviation.argtypes = [C.c_void_p, C.c_int, u64p, C.c_int, C.c_uint64, i32p,
                                      i32p, u64p]
    L.labs_exhaustive_optimum.argtypes = [C.c_void_p, C.c_int, i64p, u64p, C.c_int64, i64p]
    L.labs_local_optima.argtypes = [C.c_void_p, C.c_int, i64p]
    L.labs_solver_population.argtypes = [C.c_void_p, u64p, i32p]
    L.labs_solver_state_size.argtypes = [C.c_void_p]
    L.labs_solver_state_size.restype = C.c_int64
    L.labs_solver_save.argtypes = [C.c_void_p, C.c_void_p]
    L.labs_solver_load.argtypes = [C.c_void_p, C.c_void_p]
    L.labs_solver_stop_flag.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.labs_solver_set_peer_stops.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
    L.labs_ipc_export.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    L.labs_ipc_open.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
    L.labs_ipc_close.argtypes = [C.c_void_p, C.c_void_p]
    L.labs_run_replicas_multi.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int,
                                          C.c_uint64, C.POINTER(MemeticParams),
                                          C.POINTER(RunResult), C.POINTER(RunResult),
                                          C.POINTER(MemeticRecord), C.c_int64, i64p]
    _lib = L
    return L


def _check(rc: int):
    if rc == LABS_OK:
        return
    msg = _lib.labs_last_error().decode()
    if rc == LABS_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == LABS_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if rc == LABS_ERR_RUNTIME:
        raise RuntimeError(msg)
    raise LabsCudaError(msg)


def rng_state(seed: int) -> RngState:
    """Engine state of Rng(seed) (proj/include/labsolve/rng.hpp:13)."""
    L = load_library()
    st = RngState()
    L.labs_rng_seed(C.c_uint64(seed), C.byref(st))
    return st


def rng_states(seeds) -> "C.Array":
    arr = (RngState * len(seeds))()
    L = load_library()
    for i, s in enumerate(seeds):
        L.labs_rng_seed(C.c_uint64(int(s)), C.byref(arr[i]))
    return arr


def _words(words, n, count=None):
    w = np.ascontiguousarray(words, dtype=np.uint64)
    if w.ndim == 1:
        w = w.reshape(1, -1)
    if w.shape[1] != nwords(n):
        raise ValueError(f"expected {nwords(n)} words per sequence for n={n}")
    return w


def _result(r: RunResult, n: int) -> dict:
    return {"best": np.array([r.best[i] for i in range(nwords(n))], dtype=np.uint64),
            "best_energy": int(r.best_energy), "merit": float(r.merit),
            "iterations": int(r.iterations), "wall_seconds": float(r.wall_seconds),
            "seed": int(r.seed), "replica_id": int(r.replica_id),
            "reached_target": bool(r.reached_target), "tabu_iterations": int(r.tabu_iterations)}


class Context:
    """One CUDA device + stream (labs_ctx)."""

    def __init__(self, device: int = 0):
        self.L = load_library()
        h = C.c_void_p()
        _check(self.L.labs_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.labs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.L.labs_ctx_stream(self.h) or 0)

    @property
    def sm_count(self) -> int:
        return int(self.L.labs_ctx_sm_count(self.h))

    def synchronize(self):
        _check(self.L.labs_ctx_synchronize(self.h))

    # -- CUDA IPC (multi-process island stop flags) -------------------------
    def ipc_export(self, d_ptr: int) -> bytes:
        h = (C.c_ubyte * LABS_IPC_HANDLE_BYTES)()
        _check(self.L.labs_ipc_export(self.h, C.c_void_p(d_ptr), h))
        return bytes(h)

    def ipc_open(self, handle: bytes) -> int:
        h = (C.c_ubyte * LABS_IPC_HANDLE_BYTES).from_buffer_copy(handle)
        p = C.c_void_p()
        _check(self.L.labs_ipc_open(self.h, h, C.byref(p)))
        return int(p.value)

    def ipc_close(self, d_ptr: int):
        _check(self.L.labs_ipc_close(self.h, C.c_void_p(d_ptr)))

    # -- K5 ---------------------------------------------------------------
    def exhaustive_optimum(self, n: int, cap: int = 1 << 16):
        """(optimal E, raw optimal sequences with s_0 = +1) by full enumeration."""
        e, cnt = C.c_int64(0), C.c_int64(0)
        w = np.zeros(max(cap, 1), dtype=np.uint64)
        _check(self.L.labs_exhaustive_optimum(self.h, n, C.byref(e), _ptr(w, u64p), cap,
                                              C.byref(cnt)))
        if cnt.value > cap:
            raise RuntimeError("optimal witness set exceeded the tracking cap")
        return int(e.value), w[:cnt.value].copy()

    def local_optima(self, n: int) -> int:
        c = C.c_int64(0)
        _check(self.L.labs_local_optima(self.h, n, C.byref(c)))
        return int(c.value)

    def int_peak_gops(self) -> float:
        """Measured INT32 lane-instruction rate, both integer pipes."""
        g = C.c_double(0)
        _check(self.L.labs_bench_int_peak(self.h, C.byref(g)))
        return float(g.value)

    def imad_peak_gops(self) -> float:
        """Measured IMAD-only rate (the §8(d) lag-term roofline denominator)."""
        g = C.c_double(0)
        _check(self.L.labs_bench_imad_peak(self.h, C.byref(g)))
        return float(g.value)

    # -- K6 ---------------------------------------------------------------
    def skew_deviation(self, n: int, words, with_edits: bool = False, budget: int = 0):
        """(value, budget_exceeded, evaluations) of deviation[_with_edits]."""
        w = _words(words, n)
        v, ex, ev = C.c_int32(0), C.c_int32(0), C.c_uint64(0)
        _check(self.L.labs_skew_deviation(self.h, n, _ptr(w, u64p), 1 if with_edits else 0,
                                          C.c_uint64(budget), C.byref(v), C.byref(ex),
                                          C.byref(ev)))
        return int(v.value), bool(ex.value), int(ev.value)

    # -- K1 ---------------------------------------------------------------
    def build_state(self, n: int, words, neighbors: bool = True):
        """CorrelationState for a batch: (C[count, n-1], E[count], nbr[count, n])."""
        w = _words(words, n)
        cnt = w.shape[0]
        corr = np.zeros((cnt, max(n - 1, 1)), dtype=np.int32)
        e = np.zeros(cnt, dtype=np.int64)
        nb = np.zeros((cnt, n), dtype=np.int64) if neighbors else None
        _check(self.L.labs_build_state(self.h, n, cnt, _ptr(w, u64p), _ptr(corr, i32p),
                                       _ptr(e, i64p), _ptr(nb, i64p) if neighbors else None))
        return corr[:, :n - 1], e, nb

    def energies(self, n: int, words) -> np.ndarray:
        return self.build_state(n, words, neighbors=False)[1]

    def flip_trace(self, n: int, words, positions, neighbors: bool = True):
        w = _words(words, n)
        cnt = w.shape[0]
        p = np.ascontiguousarray(positions, dtype=np.int32).reshape(cnt, -1)
        flips = p.shape[1]
        e = np.zeros((cnt, flips), dtype=np.int64)
        nb = np.zeros((cnt, flips, n), dtype=np.int64) if neighbors else None
        _check(self.L.labs_flip_trace(self.h, n, cnt, _ptr(w, u64p), flips, _ptr(p, i32p),
                                      _ptr(e, i64p), _ptr(nb, i64p) if neighbors else None))
        return e, nb

    # -- K2 ---------------------------------------------------------------
    def scan(self, n: int, words, admissible, rngs, allow_fallback=True,
             tie_rule=TIE_REFERENCE):
        """scan_neighborhood for a batch; `rngs` (RngState array) advance in place."""
        w = _words(words, n)
        cnt = w.shape[0]
        adm = np.ascontiguousarray(admissible, dtype=np.uint8).reshape(cnt, n)
        pos = np.zeros(cnt, dtype=np.int32)
        e = np.zeros(cnt, dtype=np.int64)
        fb = np.zeros(cnt, dtype=np.int32)
        nt = np.zeros(cnt, dtype=np.int32)
        tm = np.zeros((cnt, LABS_MAX_WORDS), dtype=np.uint64)
        rc = self.L.labs_scan(self.h, n, cnt, _ptr(w, u64p), _ptr(adm, u8p), rngs,
                              1 if allow_fallback else 0, tie_rule, _ptr(pos, i32p),
                              _ptr(e, i64p), _ptr(fb, i32p), _ptr(nt, i32p), _ptr(tm, u64p))
        _check(rc)
        return {"position": pos, "energy": e, "fallback": fb.astype(bool), "ntie": nt,
                "tie_mask": tm}

    # -- K3 ---------------------------------------------------------------
    def tabu_walks(self, n: int, starts, rngs, params: TabuParams | None = None,
                   trace: bool = False):
        """tabu_search for a batch of walks in reference-RNG mode."""
        params = params or tabu_params()
        w = _words(starts, n)
        cnt = w.shape[0]
        best = np.zeros_like(w)
        be = np.zeros(cnt, dtype=np.int64)
        info = np.zeros((cnt, 3), dtype=np.int32)
        stride = n + n // 2 + 1
        steps = (TabuStep * (cnt * stride))() if trace else None
        _check(self.L.labs_tabu_walks(self.h, n, cnt, _ptr(w, u64p), C.byref(params), rngs,
                                      _ptr(best, u64p), _ptr(be, i64p), _ptr(info, i32p),
                                      steps))
        out = {"best": best, "energy": be, "max_iter": info[:, 0].copy(),
               "min_tabu": info[:, 1].copy(), "max_tabu": info[:, 2].copy()}
        if trace:
            out["steps"] = [[(steps[c * stride + t].iteration, steps[c * stride + t].position,
                              int(steps[c * stride + t].energy), steps[c * stride + t].tenure,
                              bool(steps[c * stride + t].fallback))
                             for t in range(int(info[c, 0]))] for c in range(cnt)]
        return out

    def tabu_walks_device(self, n, count, walks_per_walker, d_start, d_best, d_best_energy,
                          params=None, rng_kind=RNG_PHILOX, d_rng=0, seed=0, ctr_base=0,
                          d_iterations=0):
        """Asynchronous throughput form on device pointers (ints)."""
        params = params or tabu_params()
        _check(self.L.labs_tabu_walks_device(self.h, n, count, walks_per_walker,
                                             C.c_void_p(d_start), C.byref(params), rng_kind,
                                             C.c_void_p(d_rng or None), C.c_uint64(seed),
                                             C.c_uint64(ctr_base), C.c_void_p(d_best),
                                             C.c_void_p(d_best_energy),
                                             C.c_void_p(d_iterations or None)))

    def rng_seed_device(self, count, base_seed, d_rng):
        _check(self.L.labs_rng_seed_device(self.h, count, C.c_uint64(base_seed),
                                           C.c_void_p(d_rng)))

    # -- K4 ---------------------------------------------------------------
    def memetic(self, n: int, seed: int, params: MemeticParams | None = None,
                replica_id: int = 0, trace_cap: int = 0, stop=None):
        params = params or memetic_params()
        out = RunResult()
        tr = (MemeticRecord * max(trace_cap, 1))() if trace_cap else None
        tl = C.c_int64(0)
        stop_ptr = None
        if stop is not None:
            stop_ptr = _ptr(stop, i32p)
        _check(self.L.labs_memetic(self.h, n, C.byref(params), C.c_uint64(seed), stop_ptr,
                                   replica_id, C.byref(out), tr, trace_cap,
                                   C.byref(tl) if trace_cap else None))
        d = _result(out, n)
        if trace_cap:
            d["trace"] = [(int(tr[i].iteration), bool(tr[i].stop_seen), int(tr[i].child_energy))
                          for i in range(min(tl.value, trace_cap))]
        return d

    def run_replicas(self, n: int, replicas: int, base_seed: int,
                     params: MemeticParams | None = None, trace_cap: int = 0):
        params = params or memetic_params()
        out = RunResult()
        per = (RunResult * replicas)()
        tr = (MemeticRecord * (replicas * max(trace_cap, 1)))() if trace_cap else None
        tl = np.zeros(replicas, dtype=np.int64)
        _check(self.L.labs_run_replicas(self.h, n, replicas, C.c_uint64(base_seed),
                                        C.byref(params), C.byref(out), per, tr, trace_cap,
                                        _ptr(tl, i64p) if trace_cap else None))
        res = _result(out, n)
        reps = [_result(per[i], n) for i in range(replicas)]
        if trace_cap:
            for r in range(replicas):
                reps[r]["trace"] = [(int(tr[r * trace_cap + i].iteration),
                                     bool(tr[r * trace_cap + i].stop_seen),
                                     int(tr[r * trace_cap + i].child_energy))
                                    for i in range(min(int(tl[r]), trace_cap))]
        return res, reps


def run_replicas_multi(ctxs, n: int, replicas: int, base_seed: int,
                       params: MemeticParams | None = None, trace_cap: int = 0):
    """labs_run_replicas_multi: one host thread, len(ctxs) GPUs (contexts may
    share a device), contiguous replica blocks, device-side cross-GPU stop."""
    params = params or memetic_params()
    L = load_library()
    arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
    out = RunResult()
    per = (RunResult * replicas)()
    tr = (MemeticRecord * (replicas * max(trace_cap, 1)))() if trace_cap else None
    tl = np.zeros(replicas, dtype=np.int64)
    _check(L.labs_run_replicas_multi(arr, len(ctxs), n, replicas, C.c_uint64(base_seed),
                                     C.byref(params), C.byref(out), per, tr, trace_cap,
                                     _ptr(tl, i64p) if trace_cap else None))
    res = _result(out, n)
    reps = [_result(per[i], n) for i in range(replicas)]
    if trace_cap:
        for r in range(replicas):
            reps[r]["trace"] = [(int(tr[r * trace_cap + i].iteration),
                                 bool(tr[r * trace_cap + i].stop_seen),
                                 int(tr[r * trace_cap + i].child_energy))
                                for i in range(min(int(tl[r]), trace_cap))]
    return res, reps


class Evaluator:
    """labs_eval: persistent single-sequence evaluator (C_k, E, neighbors)."""

    def __init__(self, ctx: Context, n: int):
        self.L, self.n = ctx.L, n
        h = C.c_void_p()
        _check(self.L.labs_eval_create(ctx.h, n, C.byref(h)))
        self.h = h

    def __call__(self, words):
        w = _words(words, self.n)
        corr = np.zeros(max(self.n - 1, 1), dtype=np.int32)
        e = C.c_int64(0)
        nb = np.zeros(self.n, dtype=np.int64)
        _check(self.L.labs_eval_run(self.h, _ptr(w, u64p), _ptr(corr, i32p), C.byref(e),
                                    _ptr(nb, i64p)))
        return corr[:self.n - 1], int(e.value), nb

    def close(self):
        if getattr(self, "h", None):
            self.L.labs_eval_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """Device-resident replica set (labs_solver_*): epochs, counters, island
    exchange. Replica r has global id replica_offset + r and seed
    base_seed + replica_offset + r."""

    def __init__(self, ctx: Context, n: int, replicas: int, base_seed: int,
                 params: MemeticParams | None = None, replica_offset: int = 0,
                 trace_cap: int = 0):
        self.ctx, self.L = ctx, ctx.L
        self.n, self.replicas, self.trace_cap = n, replicas, trace_cap
        self.params = params or memetic_params()
        h = C.c_void_p()
        _check(self.L.labs_solver_create(ctx.h, n, replicas, C.c_uint64(base_seed),
                                         replica_offset, C.byref(self.params), trace_cap,
                                         C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.labs_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def capacity(ctx: Context, n: int, rng_kind: int = RNG_MT19937_64) -> int:
        return int(ctx.L.labs_solver_capacity(ctx.h, n, rng_kind))

    def run(self, epoch_iterations: int = -1, epoch_seconds: float = -1.0, race: bool = True):
        _check(self.L.labs_solver_run(self.h, epoch_iterations, epoch_seconds, 1 if race else 0))

    def request_stop(self):
        _check(self.L.labs_solver_request_stop(self.h))

    def sync(self):
        self.ctx.synchronize()

    def status(self):
        run, be, br = C.c_int32(0), C.c_int64(0), C.c_int32(0)
        _check(self.L.labs_solver_status(self.h, C.byref(run), C.byref(be), C.byref(br)))
        return {"running": run.value, "best_energy": be.value, "best_replica": br.value}

    def counters(self):
        t, m = C.c_uint64(0), C.c_int64(0)
        _check(self.L.labs_solver_counters(self.h, C.byref(t), C.byref(m)))
        return int(t.value), int(m.value)

    def results(self):
        per = (RunResult * self.replicas)()
        order = np.zeros(self.replicas, dtype=np.int32)
        tr = (MemeticRecord * (self.replicas * self.trace_cap))() if self.trace_cap else None
        tl = np.zeros(self.replicas, dtype=np.int64)
        _check(self.L.labs_solver_results(self.h, per, tr, _ptr(tl, i64p) if self.trace_cap
                                          else None, _ptr(order, i32p)))
        reps = [_result(per[i], self.n) for i in range(self.replicas)]
        for i, r in enumerate(reps):
            r["publish_order"] = int(order[i])
            if self.trace_cap:
                r["trace"] = [(int(tr[i * self.trace_cap + j].iteration),
                               bool(tr[i * self.trace_cap + j].stop_seen),
                               int(tr[i * self.trace_cap + j].child_energy))
                              for j in range(min(int(tl[i]), self.trace_cap))]
        return reps

    def population(self):
        """(words[R, K, W], energies[R, K]) copied out of HBM."""
        K = self.params.population_size
        w = np.zeros((self.replicas, K, nwords(self.n)), dtype=np.uint64)
        e = np.zeros((self.replicas, K), dtype=np.int32)
        _check(self.L.labs_solver_population(self.h, _ptr(w, u64p), _ptr(e, i32p)))
        return w, e

    def save(self) -> bytes:
        """Checkpoint of every replica's complete state (labs_solver_save)."""
        size = int(self.L.labs_solver_state_size(self.h))
        buf = (C.c_ubyte * size)()
        _check(self.L.labs_solver_save(self.h, buf))
        return bytes(buf)

    def load(self, blob: bytes):
        """Resume from a checkpoint made by a solver with the same setup."""
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(self.L.labs_solver_load(self.h, buf))

    @property
    def stop_flag(self) -> int:
        """Device address of this solver's stop flag (IPC-exportable)."""
        p = C.c_void_p()
        _check(self.L.labs_solver_stop_flag(self.h, C.byref(p)))
        return int(p.value)

    def set_peer_stops(self, d_flags):
        """Flags (device pointers valid in this process) a replica reaching
        the target raises together with its own."""
        arr = (C.c_void_p * max(len(d_flags), 1))(*[C.c_void_p(int(f)) for f in d_flags])
        _check(self.L.labs_solver_set_peer_stops(self.h, len(d_flags), arr))

    def export_elites(self, k: int, d_words: int, d_energies: int):
        _check(self.L.labs_solver_export_elites(self.h, k, C.c_void_p(d_words),
                                                C.c_void_p(d_energies)))

    def import_elites(self, count: int, d_words: int, d_energies: int, rotation: int = 0):
        _check(self.L.labs_solver_import_elites(self.h, count, C.c_void_p(d_words),
                                                C.c_void_p(d_energies), rotation))
