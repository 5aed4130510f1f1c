/*
 * labs_oracle.h — CPU restatement of the reference MTS hot path (TEST
 * INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle: a plain-C restatement of the reference
 * algorithm in /root/reference/proj/src/{sequence,correlation_state,tabu,
 * memetic,parallel}.cpp and of the libstdc++ 13 random-number distributions
 * the reference's Rng (proj/include/labsolve/rng.hpp:10-28) is built on.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it, and only as the checker or as the
 * timed CPU baseline — never as a product path.
 *
 * Parity status: PINNED. The restatement is checked against
 *   - the reference's own golden vectors (README.md:114-117 trajectory,
 *     test_correlation.cpp KATs, data/published_sequences.txt), and
 *   - the unmodified reference compiled from /root/reference into
 *     oracle/_ref/ (oracle/Makefile), via fixtures in tests/golden/ made by
 *     tests/golden/make_golden.py.
 *
 * Conventions (proj/include/labsolve/sequence.hpp:11-14): bit i of the
 * packed sequence lives in word i/64 at bit i%64; bit 0 = spin +1, bit 1 =
 * spin -1; padding bits are zero.
 */
#ifndef LABS_ORACLE_H
#define LABS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LO_MAXN 1024
#define LO_MAXW (LO_MAXN / 64)

/* mt19937_64 + libstdc++ 13 distributions (rng.hpp:10-28). */
typedef struct {
  uint64_t mt[312];
  int idx; /* next output position; 312 = twist before next draw */
} lo_rng;

void lo_rng_seed(lo_rng* r, uint64_t seed);
uint64_t lo_rng_bits64(lo_rng* r);
int64_t lo_rng_uniform_int(lo_rng* r, int64_t lo, int64_t hi);
double lo_rng_uniform01(lo_rng* r);

/* Sequence helpers (sequence.cpp). */
int lo_words(int n);
void lo_seq_random(int n, lo_rng* r, uint64_t* words);
int lo_spin(const uint64_t* words, int i);
int64_t lo_autocorrelation(int n, const uint64_t* words, int k);
int64_t lo_energy(int n, const uint64_t* words);

/* CorrelationState (correlation_state.cpp:9-98), kept as C_k + E. */
typedef struct {
  int n;
  uint64_t w[LO_MAXW];
  int32_t C[LO_MAXN]; /* C[k-1] = C_k */
  int64_t E;
} lo_state;

void lo_state_build(lo_state* s, int n, const uint64_t* words);
int64_t lo_neighbor_energy(const lo_state* s, int j);
void lo_apply_flip(lo_state* s, int j);

/* scan_neighborhood (correlation_state.cpp:100-166).
 * admissible[j] != 0 marks admissible positions. Returns 0 on success, -1 if
 * nothing is admissible and !allow_fallback (reference throws
 * std::runtime_error). Optional outputs: ntie/ties (ascending). */
typedef struct {
  int position;
  int64_t energy;
  int fallback;
} lo_scan_result;

int lo_scan(const lo_state* s, const uint8_t* admissible, lo_rng* r,
            int allow_fallback, lo_scan_result* out, int* ntie, int* ties);

/* tabu_search (tabu.cpp:12-56). */
typedef struct {
  int iteration;
  int position;
  int64_t energy;
  int tenure;
  int fallback;
} lo_tabu_step;

typedef struct {
  int max_iter;
  int min_tabu;
  int max_tabu;
} lo_tabu_info;

int lo_sample_max_iter(int n, lo_rng* r);
/* Returns 0, or -1 on invalid arguments (reference: std::invalid_argument).
 * steps may be NULL; otherwise it must hold max_iter <= 3n/2+1 entries. */
int lo_tabu_search(int n, const uint64_t* start, double min_factor,
                   double max_factor, lo_rng* r, uint64_t* best_out,
                   int64_t* best_energy, lo_tabu_info* info,
                   lo_tabu_step* steps);

/* memetic (memetic.cpp:8-117). */
typedef struct {
  int population_size;  /* K */
  double p_comb;
  double p_mutate;      /* <= 0: 1/n */
  int64_t target_energy;
  double max_seconds;   /* < 0: unlimited */
  int64_t max_iterations; /* < 0: unlimited */
  double min_tabu_factor;
  double max_tabu_factor;
} lo_memetic_params;

typedef struct {
  uint64_t best[LO_MAXW];
  int64_t best_energy;
  int64_t iterations;
  double wall_seconds;
  uint64_t seed;
  int replica_id;
  int reached_target;
} lo_run_result;

void lo_memetic_defaults(lo_memetic_params* p);
void lo_select_parents(const int64_t* energies, int k, lo_rng* r, int* p1,
                       int* p2);
void lo_combine(int n, const uint64_t* a, const uint64_t* b, lo_rng* r,
                uint64_t* child);
void lo_mutate(int n, uint64_t* child, double p_mutate, lo_rng* r);
/* stop: optional flag polled at the top of every iteration (memetic.cpp:80).
 * child_energies: optional trace of refined child energies (len >= cap). */
int lo_memetic_tabu(int n, const lo_memetic_params* p, uint64_t seed,
                    const volatile int* stop, int replica_id,
                    lo_run_result* out, int64_t* child_energies,
                    int64_t child_cap);

/* run_replicas (parallel.cpp:22-61), sequential mode (run_threaded=false).
 * per_replica may be NULL. */
int lo_run_replicas_sequential(int n, int replicas, uint64_t base_seed,
                               const lo_memetic_params* p,
                               lo_run_result* out, lo_run_result* per_replica);

/* Throughput harness for the CPU baseline: `threads` independent streams,
 * each running tabu_search from Sequence::random(n) back to back for
 * `seconds`; stream t seeds Rng(42 + t). Returns total tabu iterations. */
int64_t lo_tabu_throughput(int n, int threads, double seconds,
                           int64_t* walks_out, double* elapsed_out);

#ifdef __cplusplus
}
#endif

#endif
