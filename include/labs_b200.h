/*
 * labs_b200.h — C ABI of the B200-native LABS memetic-tabu-search hot path.
 *
 * The drop-in boundary for the reference's solver path
 * (/root/reference/proj/include/labsolve/{sequence,rng,correlation_state,
 * tabu,memetic,parallel}.hpp). Plain C: POD structs, plain pointers and
 * sizes, int status codes, no C++ or torch types. The C++ drop-in headers in
 * include/labsolve/ (namespace labsolve, signature-compatible with the
 * reference) are implemented on top of these entry points, and so is the
 * Python ctypes mirror in paper_2504_00987_b200/capi.py.
 *
 * Conventions shared with the reference:
 *  - a sequence of length n is ceil(n/64) little-endian uint64 words; position
 *    i is bit i%64 of word i/64; bit 0 = spin +1, bit 1 = spin -1; padding
 *    bits are zero (proj/include/labsolve/sequence.hpp:11-14);
 *  - energies are E = sum_{k=1}^{n-1} C_k^2 (proj/src/sequence.cpp:138-147);
 *  - random streams: labs_rng_state is the mt19937_64 engine state behind
 *    labsolve::Rng (proj/include/labsolve/rng.hpp:10-28); in
 *    LABS_RNG_MT19937_64 mode every kernel consumes draws in the reference
 *    order with libstdc++ 13's distribution algorithms, so trajectories are
 *    bit-identical to the reference's.
 *
 * Errors mirror the reference's exception classes (proj/include/labsolve/
 * *.hpp): LABS_ERR_INVALID_ARGUMENT <-> std::invalid_argument,
 * LABS_ERR_OUT_OF_RANGE <-> std::out_of_range, LABS_ERR_RUNTIME <->
 * std::runtime_error; LABS_ERR_CUDA reports a device failure. The message of
 * the last failure on the calling thread is labs_last_error().
 *
 * Host-pointer entry points copy inputs to the device, run, copy results back
 * and synchronize the context stream. *_device entry points take device
 * pointers and are asynchronous on labs_ctx_stream().
 */
#ifndef LABS_B200_H
#define LABS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LABS_OK 0
#define LABS_ERR_INVALID_ARGUMENT 1
#define LABS_ERR_OUT_OF_RANGE 2
#define LABS_ERR_RUNTIME 3
#define LABS_ERR_CUDA 4

#define LABS_MAX_N 256 /* device walkers hold n <= 256 (8 slots x 32 lanes) */
#define LABS_MAX_WORDS 4
#define LABS_MAX_PEERS 15 /* other islands' stop flags a solver can raise */
#define LABS_IPC_HANDLE_BYTES 64 /* cudaIpcMemHandle_t */

#define LABS_RNG_MT19937_64 0 /* reference-RNG mode (bit-exact trajectories) */
#define LABS_RNG_PHILOX 1     /* production mode: counter-based Philox4x32-10 */

#define LABS_TIE_REFERENCE 0 /* uniform draw among ties (reference) */
#define LABS_TIE_LOWEST 1    /* deterministic: lowest position, no draw */

#define LABS_CROSSOVER_UNIFORM 0   /* one bits64() mask per word (reference) */
#define LABS_CROSSOVER_ONE_POINT 1 /* cut = uniform_int(1, n-1) */

#define LABS_REPLACE_RANDOM 0 /* victim = uniform_int(0, K-1) (reference) */
#define LABS_REPLACE_WORST 1  /* elite-preserving: child replaces the worst
                                 member only if strictly better */

typedef struct labs_ctx labs_ctx;

/* mt19937_64 engine state: 312 words + next-output index (312 = fresh). */
typedef struct {
  uint64_t mt[312];
  int32_t idx;
  int32_t pad_;
} labs_rng_state;

/* TabuParams (proj/include/labsolve/tabu.hpp:11-14) + policy switches. */
typedef struct {
  double min_tabu_factor; /* default 0.10 */
  double max_tabu_factor; /* default 0.12 */
  int32_t tie_rule;       /* LABS_TIE_*; reference: LABS_TIE_REFERENCE */
  int32_t aspiration;     /* 0 (reference) or 1 */
} labs_tabu_params;

/* TabuStep (proj/include/labsolve/tabu.hpp:16-22). */
typedef struct {
  int32_t iteration;
  int32_t position;
  int64_t energy;
  int32_t tenure;
  int32_t fallback;
} labs_tabu_step;

/* MemeticParams (proj/include/labsolve/memetic.hpp:15-24). Optional fields
 * use sentinels: p_mutate <= 0 -> 1/n, max_seconds < 0 -> unlimited,
 * max_iterations < 0 -> unlimited. */
typedef struct {
  int32_t population_size; /* K, default 100 */
  int32_t rng_kind;        /* LABS_RNG_*, default MT19937_64 */
  double p_comb;           /* default 0.9 */
  double p_mutate;
  int64_t target_energy;
  double max_seconds;
  int64_t max_iterations;
  labs_tabu_params tabu;
  int32_t crossover;   /* LABS_CROSSOVER_*; reference: UNIFORM */
  int32_t replacement; /* LABS_REPLACE_*; reference: RANDOM */
} labs_memetic_params;

/* RunResult (proj/include/labsolve/memetic.hpp:26-35). */
typedef struct {
  uint64_t best[LABS_MAX_WORDS];
  int64_t best_energy;
  double merit;
  int64_t iterations;
  double wall_seconds;
  uint64_t seed;
  int32_t replica_id;
  int32_t reached_target;
  int64_t tabu_iterations; /* extension: tabu iterations this replica ran */
} labs_run_result;

/* MemeticIterRecord (proj/include/labsolve/memetic.hpp:37-41). */
typedef struct {
  int64_t iteration;
  int32_t stop_seen;
  int32_t pad_;
  int64_t child_energy;
} labs_memetic_record;

/* ---------------------------------------------------------------- context */
const char* labs_last_error(void);
int labs_ctx_create(int device, labs_ctx** out);
int labs_ctx_destroy(labs_ctx* ctx);
void* labs_ctx_stream(labs_ctx* ctx); /* cudaStream_t */
int labs_ctx_sm_count(labs_ctx* ctx);
int labs_ctx_synchronize(labs_ctx* ctx);
int labs_max_n(void);
/* Host-side engine seeding, identical to Rng(seed) (rng.hpp:13). */
void labs_rng_seed(uint64_t seed, labs_rng_state* out);

/* ------------------------------------------------ K1: state / energies --- */
/* Replaces the CorrelationState constructor + correlation(k) + energy() +
 * neighbor_energy(j) (correlation_state.hpp:17-36; .cpp:9-71) for a batch of
 * `count` sequences, and energy() (sequence.hpp:57) for population init.
 * corr_out: count x (n-1) C_k, k = 1..n-1 (may be NULL); energy_out: count;
 * neighbor_out: count x n energies after flipping j (may be NULL). */
int labs_build_state(labs_ctx* ctx, int n, int count, const uint64_t* words,
                     int32_t* corr_out, int64_t* energy_out,
                     int64_t* neighbor_out);

/* Persistent single-sequence evaluator behind the C++ CorrelationState
 * (correlation_state.hpp:17-36; .cpp:9-98): device and pinned host buffers
 * are allocated once, so each evaluation (construction or apply_flip) is one
 * H2D, one launch, one D2H and a synchronization. Outputs as
 * labs_build_state with count = 1 (corr_out / neighbor_out may be NULL).
 * For long flip sequences use labs_flip_trace (one launch for all flips). */
typedef struct labs_eval labs_eval;
int labs_eval_create(labs_ctx* ctx, int n, labs_eval** out);
int labs_eval_destroy(labs_eval* e);
int labs_eval_run(labs_eval* e, const uint64_t* words, int32_t* corr_out,
                  int64_t* energy_out, int64_t* neighbor_out);

/* Replaces a sequence of CorrelationState::apply_flip calls
 * (correlation_state.cpp:73-98): for each sequence, commit `flips` positions
 * (count x flips, row-major) in order; after flip f report the energy
 * (count x flips) and, when neighbor_out != NULL, every neighbor energy
 * (count x flips x n). Positions must be in [0, n) (else OUT_OF_RANGE). */
int labs_flip_trace(labs_ctx* ctx, int n, int count, const uint64_t* words,
                    int flips, const int32_t* positions, int64_t* energy_out,
                    int64_t* neighbor_out);

/* ------------------------------------------------------ K2: one scan ---- */
/* Replaces scan_neighborhood(state, admissible, rng, workers, allow_fallback)
 * (correlation_state.hpp:56-62; .cpp:100-166) for `count` independent
 * (sequence, admissible mask, rng) triples. admissible: count x n bytes.
 * rng: count engine states, advanced in place exactly as the reference
 * advances its Rng. Outputs per item: position, energy, fallback flag, size
 * of the tie set and the tie set as a bitmask (count x LABS_MAX_WORDS words,
 * may be NULL). If nothing is admissible and allow_fallback == 0 the item's
 * position is -1 and the call returns LABS_ERR_RUNTIME after writing all
 * items (the reference throws std::runtime_error). */
int labs_scan(labs_ctx* ctx, int n, int count, const uint64_t* words,
              const uint8_t* admissible, labs_rng_state* rng,
              int allow_fallback, int tie_rule, int32_t* position,
              int64_t* energy, int32_t* fallback, int32_t* ntie,
              uint64_t* tie_mask);

/* ------------------------------------------------- K3: tabu walks ------- */
/* Replaces tabu_search(seq, params, rng, scan_workers, trace)
 * (tabu.hpp:37-41; tabu.cpp:17-56) for `count` independent walks in
 * reference-RNG mode. start/best_out: count x ceil(n/64) words;
 * best_energy: count; info (may be NULL): count x {max_iter, min_tabu,
 * max_tabu}; steps (may be NULL): count x (n + n/2 + 1) records, walk c's
 * step t at steps[c * (n + n/2 + 1) + t - 1]. rng is advanced in place. */
int labs_tabu_walks(labs_ctx* ctx, int n, int count, const uint64_t* start,
                    const labs_tabu_params* params, labs_rng_state* rng,
                    uint64_t* best_out, int64_t* best_energy, int32_t* info,
                    labs_tabu_step* steps);

/* Throughput form (device pointers, asynchronous). Each of `count` walkers
 * runs `walks_per_walker` tabu walks back to back, each from the previous
 * walk's best (walk 1 from d_start). rng_kind MT: d_rng holds count device
 * engine states (see labs_rng_seed_device); PHILOX: seed keys the stream,
 * walker c uses stream c and counter base ctr_base. d_iterations (may be
 * NULL) accumulates the tabu iterations executed (flip-evals = n x that). */
int labs_tabu_walks_device(labs_ctx* ctx, int n, int count,
                           int walks_per_walker, const uint64_t* d_start,
                           const labs_tabu_params* params, int rng_kind,
                           labs_rng_state* d_rng, uint64_t seed,
                           uint64_t ctr_base, uint64_t* d_best,
                           int64_t* d_best_energy,
                           unsigned long long* d_iterations);

/* Seed `count` device engine states: state c = Rng(base_seed + c). */
int labs_rng_seed_device(labs_ctx* ctx, int count, uint64_t base_seed,
                         labs_rng_state* d_rng);

/* --------------------------------------------- K4: memetic replicas ----- */
/* Replaces memetic_tabu(n, params, seed, stop, trace, replica_id)
 * (memetic.hpp:61-65; memetic.cpp:44-117). stop: optional host flag polled
 * once per memetic iteration (pass pinned/mapped memory or NULL). trace (may
 * be NULL): up to trace_cap records are stored; *trace_len receives the
 * number of records the run produced, which exceeds trace_cap when the
 * trace was truncated (never silently: compare the two). */
int labs_memetic(labs_ctx* ctx, int n, const labs_memetic_params* params,
                 uint64_t seed, const volatile int32_t* stop, int replica_id,
                 labs_run_result* out, labs_memetic_record* trace,
                 int64_t trace_cap, int64_t* trace_len);

/* Replaces run_replicas(cfg, report) (parallel.hpp:47-51; parallel.cpp:22-61):
 * `replicas` replicas, replica r seeded base_seed + r, racing to the target
 * with a device-resident stop flag; result = strictly-lowest energy, first
 * publisher keeps a tie. per_replica (may be NULL): replicas results.
 * traces (may be NULL): replicas x trace_cap records, trace_len: replicas
 * (records produced per replica; > trace_cap means truncated, as for
 * labs_memetic). */
int labs_run_replicas(labs_ctx* ctx, int n, int replicas, uint64_t base_seed,
                      const labs_memetic_params* params, labs_run_result* out,
                      labs_run_result* per_replica,
                      labs_memetic_record* traces, int64_t trace_cap,
                      int64_t* trace_len);

/* run_replicas over several GPUs of one node from one host thread (the
 * multi-GPU form SURVEY.md §8b proposes; configs[4]'s island model without
 * migration). The global replicas [0, replicas) are cut into ngpu
 * contiguous blocks (sizes differ by at most one, larger blocks first);
 * block g runs on ctxs[g], replica r keeps seed base_seed + r
 * (parallel.cpp:38), so every replica's trajectory is the one it has on one
 * GPU or in the reference until a stop fires. Stop: when every pair of
 * devices has peer access, each GPU's stop flag is raised by the winning
 * replica directly over NVLink (P2P stores, no host in the loop);
 * otherwise the host forwards it between 10 ms epochs. Result: strictly
 * lowest energy; ties go to the earlier publisher (one global publish
 * counter when the devices have native P2P atomics, else (order, block)).
 * ctxs may repeat a device (two islands sharing one GPU). per_replica,
 * traces and trace_len are indexed by global replica as in
 * labs_run_replicas. */
int labs_run_replicas_multi(labs_ctx* const* ctxs, int ngpu, int n, int replicas,
                            uint64_t base_seed, const labs_memetic_params* params,
                            labs_run_result* out, labs_run_result* per_replica,
                            labs_memetic_record* traces, int64_t trace_cap,
                            int64_t* trace_len);

/* ------------------------------------------- solver (epoch-driven K4) ---- */
/* Device-resident replica set for long runs, throughput measurement and the
 * island model: population, energies, best and RNG state of every replica
 * stay in HBM between labs_solver_run calls, so cutting a run into epochs
 * never changes a replica's trajectory. Replica r (global id
 * replica_offset + r) is seeded base_seed + replica_offset + r.
 * trace_cap > 0 keeps up to trace_cap memetic records per replica. */
typedef struct labs_solver labs_solver;

int labs_solver_create(labs_ctx* ctx, int n, int replicas, uint64_t base_seed,
                       int64_t replica_offset,
                       const labs_memetic_params* params, int64_t trace_cap,
                       labs_solver** out);
int labs_solver_destroy(labs_solver* s);
/* Replicas resident at once for (n, rng_kind) on this device. */
int labs_solver_capacity(labs_ctx* ctx, int n, int rng_kind);
/* One launch (asynchronous on the context stream). Each replica stops at
 * its reference exit conditions, or after epoch_iterations more memetic
 * iterations (< 0: no limit), or when epoch_seconds have elapsed since the
 * replica resumed (< 0: no limit; checked between memetic iterations).
 * race != 0: a replica reaching the target raises the stop flag. */
int labs_solver_run(labs_solver* s, int64_t epoch_iterations,
                    double epoch_seconds, int race);
/* Set the device stop flag (replicas see it at their next loop check). */
int labs_solver_request_stop(labs_solver* s);
/* Synchronizing queries. */
int labs_solver_status(labs_solver* s, int32_t* running, int64_t* best_energy,
                       int32_t* best_replica);
int labs_solver_counters(labs_solver* s, uint64_t* tabu_iterations,
                         int64_t* memetic_iterations);
/* Per-replica RunResults (replicas entries), optional traces
 * (replicas x trace_cap) with lengths, optional publish order. */
int labs_solver_results(labs_solver* s, labs_run_result* per_replica,
                        labs_memetic_record* traces, int64_t* trace_len,
                        int32_t* publish_order);
/* Island model (device pointers, asynchronous). export: the k best replica
 * bests (k x ceil(n/64) words, k energies), best first. import: replica r
 * offers elite (r + rotation) % count to its population, replacing its worst
 * member if the elite is strictly better. */
int labs_solver_export_elites(labs_solver* s, int k, uint64_t* d_words,
                              int64_t* d_energies);
int labs_solver_import_elites(labs_solver* s, int count,
                              const uint64_t* d_words,
                              const int64_t* d_energies, int rotation);
/* Cross-island stop (the device-resident stop flag of SURVEY.md §8e).
 * stop_flag: device address of this solver's int32 stop flag (a plain
 * cudaMalloc allocation, so labs_ipc_export can share it with other
 * processes). set_peer_stops: up to LABS_MAX_PEERS flags, valid in this
 * process (another device's flag with peer access enabled, or one opened by
 * labs_ipc_open), that a replica reaching the target raises together with
 * its own (proj/src/parallel.cpp:40 request_stop, across GPUs over NVLink);
 * count = 0 clears them. */
int labs_solver_stop_flag(labs_solver* s, int32_t** d_flag);
int labs_solver_set_peer_stops(labs_solver* s, int count, int32_t* const* d_flags);
/* CUDA IPC for the multi-process island model: export a device allocation
 * made by this library (e.g. a stop flag) as LABS_IPC_HANDLE_BYTES opaque
 * bytes; open a handle exported by another process (on ctx's device, peer
 * access enabled lazily); close what was opened. */
int labs_ipc_export(labs_ctx* ctx, const void* d_ptr, void* handle);
int labs_ipc_open(labs_ctx* ctx, const void* handle, void** d_ptr);
int labs_ipc_close(labs_ctx* ctx, void* d_ptr);
/* Copy every population out (host buffers, synchronizing): words
 * replicas x K x ceil(n/64), energies replicas x K. For inspection and
 * checkpointing between epochs. */
int labs_solver_population(labs_solver* s, uint64_t* words, int32_t* energies);
/* Checkpoint / resume for long runs: the complete replica state (populations,
 * energies, bests, counters, RNG states, traces) as one host blob.
 * state_size returns the byte count; load requires a solver created with the
 * same n, replicas, base_seed, replica_offset, trace_cap and every field of
 * params (checked; LABS_ERR_INVALID_ARGUMENT otherwise). A resumed run
 * continues every replica's trajectory exactly; each replica's elapsed time
 * is saved, so max_seconds budgets and reported wall times continue from
 * the checkpoint. */
int64_t labs_solver_state_size(labs_solver* s);
int labs_solver_save(labs_solver* s, void* blob);
int labs_solver_load(labs_solver* s, const void* blob);

/* ------------------------------------- K5: exhaustive ground truth ------ */
/* Replaces brute_force_optimum / enumerate_local_optima
 * (proj/include/labsolve/oracle.hpp:18-24; oracle.cpp:23-151) on the device:
 * a Gray-code walk over the 2^(n-1) sequences with s_0 = +1, n <= 64 (the
 * reference stops at 30 / 24). exhaustive_optimum returns the optimal energy
 * and every optimal sequence of that half (raw, not canonicalized; up to cap,
 * *count = how many exist). local_optima counts strict local optima of the
 * whole space (x2 for the complement half, as the reference does). */
int labs_exhaustive_optimum(labs_ctx* ctx, int n, int64_t* optimal_energy,
                            uint64_t* witnesses, int64_t cap, int64_t* count);
int labs_local_optima(labs_ctx* ctx, int n, int64_t* count);

/* ------------------------------------------ K6: skew-symmetry deviation - */
/* Replaces deviation / deviation_with_edits (proj/include/labsolve/
 * skew.hpp:21-40; skew.cpp:110-187) on the device: every pair-count
 * evaluation of the reference's loop order runs in its own thread, and the
 * reference's early exit (right after the first zero) and budget charging
 * are recovered exactly, so value, budget_exceeded and evaluations equal
 * the reference's. budget = 0: unlimited. 3 <= n <= LABS_MAX_N. */
int labs_skew_deviation(labs_ctx* ctx, int n, const uint64_t* words, int with_edits,
                        uint64_t budget, int32_t* value, int32_t* budget_exceeded,
                        uint64_t* evaluations);

/* ------------------------------------------------------- diagnostics --- */
/* Measured INT32 lane-instruction rate of this device (IMAD on the FMA pipe
 * alongside IADD3/LOP3 on the ALU pipe), in Gop/s: the issue ceiling of
 * every integer instruction the walker executes (both pipes). */
int labs_bench_int_peak(labs_ctx* ctx, double* gops);
/* Measured IMAD-only rate (INT32 multiply-adds on the FMA pipe alone), in
 * Gop/s: the denominator of SURVEY.md §8(d)'s lag-term roofline ((N-1) MACs
 * per flip-evaluation). */
int labs_bench_imad_peak(labs_ctx* ctx, double* gmacs);

#ifdef __cplusplus
}
#endif

#endif /* LABS_B200_H */
