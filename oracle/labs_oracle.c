/*
 * labs_oracle.c — CPU restatement of the reference MTS hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see labs_oracle.h): the checker for the CUDA
 * path and the "port" CPU baseline. Never linked into the product.
 * Each function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.
 */
#define _POSIX_C_SOURCE 200809L
#include "labs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ RNG -- */
/* std::mt19937_64 (the engine behind Rng, rng.hpp:26) — standard MT19937-64
 * parameters; seeding per [rand.eng.mers]. */
#define MT_N 312
#define MT_M 156
#define MT_UM 0xFFFFFFFF80000000ULL
#define MT_LM 0x7FFFFFFFULL
#define MT_A 0xB5026F5AA96619E9ULL

void lo_rng_seed(lo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(lo_rng* r) {
  uint64_t* mt = r->mt;
  int i;
  for (i = 0; i < MT_N - MT_M; ++i) {
    uint64_t x = (mt[i] & MT_UM) | (mt[i + 1] & MT_LM);
    mt[i] = mt[i + MT_M] ^ (x >> 1) ^ ((x & 1) ? MT_A : 0);
  }
  for (; i < MT_N - 1; ++i) {
    uint64_t x = (mt[i] & MT_UM) | (mt[i + 1] & MT_LM);
    mt[i] = mt[i + MT_M - MT_N] ^ (x >> 1) ^ ((x & 1) ? MT_A : 0);
  }
  uint64_t x = (mt[MT_N - 1] & MT_UM) | (mt[0] & MT_LM);
  mt[MT_N - 1] = mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1) ? MT_A : 0);
  r->idx = 0;
}

/* Rng::bits64 (rng.hpp:15) = engine(). */
uint64_t lo_rng_bits64(lo_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* Rng::uniform_int (rng.hpp:17-20): std::uniform_int_distribution<long long>
 * with a 64-bit engine takes libstdc++ 13's downscaling branch, Lemire's
 * nearly-divisionless method over a 128-bit product
 * (/usr/include/c++/13/bits/uniform_int_dist.h:255-281, 306-319). One engine
 * draw at least, even when lo == hi. */
int64_t lo_rng_uniform_int(lo_rng* r, int64_t lo, int64_t hi) {
  uint64_t range = (uint64_t)hi - (uint64_t)lo + 1ULL;
  if (range == 0) /* full 64-bit range: urngrange == urange branch */
    return (int64_t)lo_rng_bits64(r);
  unsigned __int128 prod = (unsigned __int128)lo_rng_bits64(r) * range;
  uint64_t low = (uint64_t)prod;
  if (low < range) {
    uint64_t thr = (0ULL - range) % range;
    while (low < thr) {
      prod = (unsigned __int128)lo_rng_bits64(r) * range;
      low = (uint64_t)prod;
    }
  }
  return (int64_t)((uint64_t)lo + (uint64_t)(prod >> 64));
}

/* Rng::uniform01 (rng.hpp:23-25): uniform_real_distribution<double>(0,1) =
 * generate_canonical<double,53> with one 64-bit draw
 * (/usr/include/c++/13/bits/random.tcc:3346-3381): double(u) / 2^64,
 * clamped below 1 with nextafter. */
double lo_rng_uniform01(lo_rng* r) {
  double d = (double)lo_rng_bits64(r) / 18446744073709551616.0;
  if (d >= 1.0) d = nextafter(1.0, 0.0);
  return d * (1.0 - 0.0) + 0.0;
}

/* ------------------------------------------------------------- Sequence -- */
int lo_words(int n) { return (n + 63) / 64; }

static uint64_t tail_mask(int n) {
  int rem = n % 64;
  return rem == 0 ? ~0ULL : ((1ULL << rem) - 1ULL);
}

/* Sequence::random (sequence.cpp:28-33). */
void lo_seq_random(int n, lo_rng* r, uint64_t* w) {
  int nw = lo_words(n);
  for (int i = 0; i < nw; ++i) w[i] = lo_rng_bits64(r);
  if (nw > 0) w[nw - 1] &= tail_mask(n);
}

/* Sequence::spin (sequence.hpp:27): bit 1 -> -1. */
int lo_spin(const uint64_t* w, int i) {
  return ((w[i >> 6] >> (i & 63)) & 1ULL) ? -1 : 1;
}

/* autocorrelation (sequence.cpp:130-136). */
int64_t lo_autocorrelation(int n, const uint64_t* w, int k) {
  int64_t sum = 0;
  for (int i = 0; i + k < n; ++i) sum += lo_spin(w, i) * lo_spin(w, i + k);
  return sum;
}

/* energy (sequence.cpp:138-147). */
int64_t lo_energy(int n, const uint64_t* w) {
  int64_t e = 0;
  for (int k = 1; k < n; ++k) {
    int64_t c = lo_autocorrelation(n, w, k);
    e += c * c;
  }
  return e;
}

/* ----------------------------------------------------- CorrelationState -- */
/* Constructor (correlation_state.cpp:9-27): C_k and E from the pivot. The
 * reference also stores the packed product table; its entries are
 * s_i*s_{i+k}, which this restatement reads from the pivot directly. */
void lo_state_build(lo_state* s, int n, const uint64_t* w) {
  memset(s, 0, sizeof(*s));
  s->n = n;
  memcpy(s->w, w, sizeof(uint64_t) * (size_t)lo_words(n));
  s->E = 0;
  for (int k = 1; k < n; ++k) {
    int32_t c = (int32_t)lo_autocorrelation(n, w, k);
    s->C[k - 1] = c;
    s->E += (int64_t)c * c;
  }
}

/* neighbor_energy (correlation_state.cpp:50-71): for each lag k the <= 2
 * products containing position j flip sign; d = -2*sum; E += d(2C_k + d). */
int64_t lo_neighbor_energy(const lo_state* s, int j) {
  int n = s->n;
  int64_t e = s->E;
  for (int k = 1; k < n; ++k) {
    int64_t sum = 0;
    if (j - k >= 0) sum += lo_spin(s->w, j - k) * lo_spin(s->w, j);
    if (j + k < n) sum += lo_spin(s->w, j) * lo_spin(s->w, j + k);
    if (sum != 0) {
      int64_t d = -2 * sum;
      e += d * (2 * (int64_t)s->C[k - 1] + d);
    }
  }
  return e;
}

/* apply_flip (correlation_state.cpp:73-98). */
void lo_apply_flip(lo_state* s, int j) {
  int n = s->n;
  int64_t e = s->E;
  for (int k = 1; k < n; ++k) {
    int64_t sum = 0;
    if (j - k >= 0) sum += lo_spin(s->w, j - k) * lo_spin(s->w, j);
    if (j + k < n) sum += lo_spin(s->w, j) * lo_spin(s->w, j + k);
    if (sum != 0) {
      int64_t d = -2 * sum;
      e += d * (2 * (int64_t)s->C[k - 1] + d);
      s->C[k - 1] += (int32_t)d;
    }
  }
  s->E = e;
  s->w[j >> 6] ^= 1ULL << (j & 63);
}

/* scan_neighborhood (correlation_state.cpp:100-166): admissible argmin, tie
 * list in ascending j (the chunked merge at :141-153 yields exactly the
 * single-pass order), fallback uniform_int(0, n-1) when nothing is
 * admissible, otherwise ties[uniform_int(0, |ties|-1)] with no draw for a
 * single tie. */
int lo_scan(const lo_state* s, const uint8_t* admissible, lo_rng* r,
            int allow_fallback, lo_scan_result* out, int* ntie_out,
            int* ties_out) {
  int n = s->n;
  int64_t best = 0;
  int ntie = 0;
  int* ties = (int*)malloc(sizeof(int) * (size_t)n);
  for (int j = 0; j < n; ++j) {
    if (!admissible[j]) continue;
    int64_t e = lo_neighbor_energy(s, j);
    if (ntie == 0 || e < best) {
      best = e;
      ntie = 0;
      ties[ntie++] = j;
    } else if (e == best) {
      ties[ntie++] = j;
    }
  }
  if (ntie_out) *ntie_out = ntie;
  if (ties_out && ntie) memcpy(ties_out, ties, sizeof(int) * (size_t)ntie);
  if (ntie == 0) {
    free(ties);
    if (!allow_fallback) return -1;
    int pos = (int)lo_rng_uniform_int(r, 0, n - 1);
    out->position = pos;
    out->energy = lo_neighbor_energy(s, pos);
    out->fallback = 1;
    return 0;
  }
  int pick = ntie == 1 ? ties[0]
                       : ties[lo_rng_uniform_int(r, 0, (int64_t)ntie - 1)];
  free(ties);
  out->position = pick;
  out->energy = best;
  out->fallback = 0;
  return 0;
}

/* ----------------------------------------------------------------- tabu -- */
/* sample_max_iter (tabu.cpp:12-15). */
int lo_sample_max_iter(int n, lo_rng* r) {
  return (int)lo_rng_uniform_int(r, 0, n) + n / 2;
}

/* tabu_search (tabu.cpp:17-56). */
int lo_tabu_search(int n, const uint64_t* start, double fmin, double fmax,
                   lo_rng* r, uint64_t* best_out, int64_t* best_energy,
                   lo_tabu_info* info, lo_tabu_step* steps) {
  if (n < 2 || n > LO_MAXN) return -1;
  if (fmin < 0 || fmax < fmin || fmax >= 1) return -1;
  int max_iter = lo_sample_max_iter(n, r);
  /* volatile keeps the product and the +1e-9 as two rounded operations,
   * exactly like the reference build (no FMA contraction). */
  volatile double pm = fmin * (double)max_iter;
  volatile double px = fmax * (double)max_iter;
  int min_tabu = (int)floor(pm + 1e-9);
  int max_tabu = (int)floor(px + 1e-9);
  if (info) {
    info->max_iter = max_iter;
    info->min_tabu = min_tabu;
    info->max_tabu = max_tabu;
  }
  lo_state st;
  lo_state_build(&st, n, start);
  int nw = lo_words(n);
  memcpy(best_out, start, sizeof(uint64_t) * (size_t)nw);
  int64_t best_e = st.E;
  int64_t* expiry = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  uint8_t* adm = (uint8_t*)malloc((size_t)n);
  for (int t = 1; t <= max_iter; ++t) {
    for (int j = 0; j < n; ++j) adm[j] = expiry[j] < t;
    lo_scan_result pick;
    lo_scan(&st, adm, r, 1, &pick, NULL, NULL);
    lo_apply_flip(&st, pick.position);
    int tenure = (int)lo_rng_uniform_int(r, min_tabu, max_tabu);
    expiry[pick.position] = t + tenure;
    if (st.E < best_e) {
      best_e = st.E;
      memcpy(best_out, st.w, sizeof(uint64_t) * (size_t)nw);
    }
    if (steps) {
      steps[t - 1].iteration = t;
      steps[t - 1].position = pick.position;
      steps[t - 1].energy = st.E;
      steps[t - 1].tenure = tenure;
      steps[t - 1].fallback = pick.fallback;
    }
  }
  free(expiry);
  free(adm);
  *best_energy = best_e;
  return 0;
}

/* -------------------------------------------------------------- memetic -- */
void lo_memetic_defaults(lo_memetic_params* p) {
  /* MemeticParams defaults (memetic.hpp:15-24), TabuParams (tabu.hpp:11-14) */
  p->population_size = 100;
  p->p_comb = 0.9;
  p->p_mutate = -1.0;
  p->target_energy = 0;
  p->max_seconds = -1.0;
  p->max_iterations = -1;
  p->min_tabu_factor = 0.10;
  p->max_tabu_factor = 0.12;
}

/* select_parents (memetic.cpp:8-22). */
static int tournament(const int64_t* e, int k, lo_rng* r) {
  int a = (int)lo_rng_uniform_int(r, 0, (int64_t)k - 1);
  int b = (int)lo_rng_uniform_int(r, 0, (int64_t)k - 1);
  if (e[a] < e[b]) return a;
  if (e[b] < e[a]) return b;
  return lo_rng_uniform_int(r, 0, 1) == 0 ? a : b;
}

void lo_select_parents(const int64_t* e, int k, lo_rng* r, int* p1, int* p2) {
  *p1 = tournament(e, k, r);
  *p2 = tournament(e, k, r);
}

/* combine (memetic.cpp:24-33): uniform crossover, one mask per word. */
void lo_combine(int n, const uint64_t* a, const uint64_t* b, lo_rng* r,
                uint64_t* child) {
  int nw = lo_words(n);
  for (int w = 0; w < nw; ++w) {
    uint64_t mask = lo_rng_bits64(r);
    child[w] = (a[w] & mask) | (b[w] & ~mask);
  }
  child[nw - 1] &= tail_mask(n);
}

/* mutate (memetic.cpp:35-42). */
void lo_mutate(int n, uint64_t* c, double p_mutate, lo_rng* r) {
  for (int i = 0; i < n; ++i)
    if (lo_rng_uniform01(r) < p_mutate) c[i >> 6] ^= 1ULL << (i & 63);
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* memetic_tabu (memetic.cpp:44-117). */
int lo_memetic_tabu(int n, const lo_memetic_params* p, uint64_t seed,
                    const volatile int* stop, int replica_id,
                    lo_run_result* out, int64_t* child_energies,
                    int64_t child_cap) {
  if (n < 2 || n > LO_MAXN) return -1;
  if (p->population_size < 2) return -1;
  if (p->p_comb < 0.0 || p->p_comb > 1.0) return -1;
  double p_mutate = p->p_mutate > 0.0 ? p->p_mutate : 1.0 / n;
  if (!(p_mutate > 0.0) || p_mutate > 1.0) return -1;
  double t0 = now_seconds();
  lo_rng r;
  lo_rng_seed(&r, seed);
  int k = p->population_size;
  int nw = lo_words(n);
  uint64_t* pop = (uint64_t*)calloc((size_t)k * nw, sizeof(uint64_t));
  int64_t* e = (int64_t*)calloc((size_t)k, sizeof(int64_t));
  for (int i = 0; i < k; ++i) lo_seq_random(n, &r, pop + (size_t)i * nw);
  for (int i = 0; i < k; ++i) e[i] = lo_energy(n, pop + (size_t)i * nw);
  int best_idx = 0;
  for (int i = 1; i < k; ++i)
    if (e[i] < e[best_idx]) best_idx = i;
  uint64_t best[LO_MAXW];
  memcpy(best, pop + (size_t)best_idx * nw, sizeof(uint64_t) * nw);
  int64_t best_e = e[best_idx];
  int64_t it = 0;
  uint64_t child[LO_MAXW], refined[LO_MAXW];
  while (best_e > p->target_energy) {
    if (stop && *stop) break;
    if (p->max_iterations >= 0 && it >= p->max_iterations) break;
    if (p->max_seconds >= 0 && now_seconds() - t0 >= p->max_seconds) break;
    if (lo_rng_uniform01(&r) < p->p_comb) {
      int p1, p2;
      lo_select_parents(e, k, &r, &p1, &p2);
      lo_combine(n, pop + (size_t)p1 * nw, pop + (size_t)p2 * nw, &r, child);
    } else {
      int idx = (int)lo_rng_uniform_int(&r, 0, (int64_t)k - 1);
      memcpy(child, pop + (size_t)idx * nw, sizeof(uint64_t) * nw);
    }
    lo_mutate(n, child, p_mutate, &r);
    int64_t re;
    lo_tabu_search(n, child, p->min_tabu_factor, p->max_tabu_factor, &r,
                   refined, &re, NULL, NULL);
    if (re < best_e) {
      best_e = re;
      memcpy(best, refined, sizeof(uint64_t) * nw);
    }
    int victim = (int)lo_rng_uniform_int(&r, 0, (int64_t)k - 1);
    memcpy(pop + (size_t)victim * nw, refined, sizeof(uint64_t) * nw);
    e[victim] = re;
    if (child_energies && it < child_cap) child_energies[it] = re;
    ++it;
  }
  memset(out, 0, sizeof(*out));
  memcpy(out->best, best, sizeof(uint64_t) * nw);
  out->best_energy = best_e;
  out->iterations = it;
  out->wall_seconds = now_seconds() - t0;
  out->seed = seed;
  out->replica_id = replica_id;
  out->reached_target = best_e <= p->target_energy;
  free(pop);
  free(e);
  return 0;
}

/* run_replicas with run_threaded=false (parallel.cpp:22-61): replica r uses
 * seed base+r; reaching the target raises the stop flag that later replicas
 * see at their first loop check; publish keeps strictly lower energy. */
int lo_run_replicas_sequential(int n, int replicas, uint64_t base_seed,
                               const lo_memetic_params* p, lo_run_result* out,
                               lo_run_result* per_replica) {
  if (n < 2 || replicas < 1) return -1;
  volatile int stop = 0;
  int have = 0;
  for (int rr = 0; rr < replicas; ++rr) {
    lo_run_result res;
    if (lo_memetic_tabu(n, p, base_seed + (uint64_t)rr, &stop, rr, &res, NULL,
                        0) != 0)
      return -1;
    if (res.reached_target) stop = 1;
    if (!have || res.best_energy < out->best_energy) {
      *out = res;
      have = 1;
    }
    if (per_replica) per_replica[rr] = res;
  }
  return 0;
}

/* ------------------------------------------------- throughput baseline -- */
typedef struct {
  int n;
  int t;
  double seconds;
  int64_t iters;
  int64_t walks;
} tp_arg;

static void* tp_worker(void* vp) {
  tp_arg* a = (tp_arg*)vp;
  lo_rng r;
  lo_rng_seed(&r, 42ULL + (uint64_t)a->t);
  uint64_t start[LO_MAXW], best[LO_MAXW];
  int64_t be;
  lo_tabu_info info;
  double t0 = now_seconds();
  while (now_seconds() - t0 < a->seconds) {
    lo_seq_random(a->n, &r, start);
    lo_tabu_search(a->n, start, 0.10, 0.12, &r, best, &be, &info, NULL);
    a->iters += info.max_iter;
    a->walks += 1;
  }
  return NULL;
}

int64_t lo_tabu_throughput(int n, int threads, double seconds,
                           int64_t* walks_out, double* elapsed_out) {
  pthread_t th[512];
  tp_arg args[512];
  if (threads > 512) threads = 512;
  double t0 = now_seconds();
  for (int t = 0; t < threads; ++t) {
    args[t].n = n;
    args[t].t = t;
    args[t].seconds = seconds;
    args[t].iters = 0;
    args[t].walks = 0;
    pthread_create(&th[t], NULL, tp_worker, &args[t]);
  }
  int64_t it = 0, walks = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    it += args[t].iters;
    walks += args[t].walks;
  }
  if (elapsed_out) *elapsed_out = now_seconds() - t0;
  if (walks_out) *walks_out = walks;
  return it;
}
