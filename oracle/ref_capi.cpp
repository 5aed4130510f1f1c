// ref_capi.cpp — extern "C" probe harness around the UNMODIFIED reference
// library (TEST INFRASTRUCTURE ONLY).
//
// oracle/Makefile compiles this file together with the reference's own
// sources where they lie (/root/reference/proj/src/{sequence,
// correlation_state,tabu,memetic,parallel}.cpp) into oracle/_ref/. Nothing in
// the product links it: tests/golden/make_golden.py uses it to generate the
// committed fixtures, tests use it (when built) to pin the C restatement in
// labs_oracle.c, and bench.py --impl reference times the reference's own
// multithreaded tabu_search with it on the host cores.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "labsolve/correlation_state.hpp"
#include "labsolve/memetic.hpp"
#include "labsolve/oracle.hpp"
#include "labsolve/parallel.hpp"
#include "labsolve/rng.hpp"
#include "labsolve/sequence.hpp"
#include "labsolve/skew.hpp"
#include "labsolve/tabu.hpp"

using namespace labsolve;

namespace {

Sequence from_words(int n, const uint64_t* w) {
  Sequence s(n);
  for (int i = 0; i < s.word_count(); ++i) s.set_word(i, w[i]);
  return s;
}

void to_words(const Sequence& s, uint64_t* w) {
  for (int i = 0; i < s.word_count(); ++i) w[i] = s.word(i);
}

struct RefResult {
  uint64_t best[16];
  int64_t best_energy;
  int64_t iterations;
  double wall_seconds;
  uint64_t seed;
  int32_t replica_id;
  int32_t reached_target;
};

void fill(const RunResult& r, RefResult* o) {
  std::memset(o, 0, sizeof(*o));
  to_words(r.best, o->best);
  o->best_energy = r.best_energy;
  o->iterations = r.iterations;
  o->wall_seconds = r.wall_seconds;
  o->seed = r.seed;
  o->replica_id = r.replica_id;
  o->reached_target = r.reached_target ? 1 : 0;
}

MemeticParams make_params(int pop, double p_comb, double p_mutate,
                          int64_t target, double max_seconds,
                          int64_t max_iterations, double fmin, double fmax) {
  MemeticParams p;
  p.population_size = pop;
  p.p_comb = p_comb;
  if (p_mutate > 0) p.p_mutate = p_mutate;
  p.target_energy = target;
  if (max_seconds >= 0) p.max_seconds = max_seconds;
  if (max_iterations >= 0) p.max_iterations = max_iterations;
  p.tabu.min_tabu_factor = fmin;
  p.tabu.max_tabu_factor = fmax;
  return p;
}

}  // namespace

extern "C" {

// kinds[i]: 0 = bits64, 1 = uniform_int(lo[i], hi[i]), 2 = uniform01 (bits
// of the double returned in out[i]).
void ref_rng_draws(uint64_t seed, int count, const int* kinds,
                   const int64_t* lo, const int64_t* hi, uint64_t* out) {
  Rng rng(seed);
  for (int i = 0; i < count; ++i) {
    if (kinds[i] == 0) {
      out[i] = rng.bits64();
    } else if (kinds[i] == 1) {
      out[i] = static_cast<uint64_t>(rng.uniform_int(lo[i], hi[i]));
    } else {
      double d = rng.uniform01();
      std::memcpy(&out[i], &d, sizeof(d));
    }
  }
}

// Sequence::random(n, Rng(seed)) repeated `count` times from one stream.
void ref_random_sequences(int n, uint64_t seed, int count, uint64_t* words) {
  Rng rng(seed);
  int nw = (n + 63) / 64;
  for (int c = 0; c < count; ++c)
    to_words(Sequence::random(n, rng), words + static_cast<size_t>(c) * nw);
}

int64_t ref_energy(int n, const uint64_t* w) { return energy(from_words(n, w)); }

// CorrelationState probe: C_k (k=1..n-1), E and every neighbor energy.
void ref_state_probe(int n, const uint64_t* w, int64_t* corr, int64_t* energy_out,
                     int64_t* neighbors) {
  CorrelationState st(from_words(n, w));
  for (int k = 1; k < n; ++k) corr[k - 1] = st.correlation(k);
  *energy_out = st.energy();
  for (int j = 0; j < n; ++j) neighbors[j] = st.neighbor_energy(j);
}

// scan_neighborhood over an explicit admissible mask with Rng(draw_seed).
// Returns 0, or -1 when it throws (nothing admissible, no fallback).
int ref_scan(int n, const uint64_t* w, const uint8_t* admissible,
             uint64_t draw_seed, int workers, int allow_fallback, int* position,
             int64_t* energy_out, int* fallback) {
  CorrelationState st(from_words(n, w));
  Rng rng(draw_seed);
  try {
    ScanResult r = scan_neighborhood(
        st, [&](int i) { return admissible[i] != 0; }, rng, workers,
        allow_fallback != 0);
    *position = r.position;
    *energy_out = r.energy;
    *fallback = r.fallback ? 1 : 0;
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// tabu_search(start, {fmin,fmax}, Rng(seed), workers, &trace).
// steps: [iteration, position, energy, tenure, fallback] x max_iter int64s.
// post_draw receives one bits64() drawn after the walk (pins RNG consumption).
int ref_tabu(int n, const uint64_t* start, double fmin, double fmax,
             uint64_t seed, int workers, uint64_t* best, int64_t* best_energy,
             int* info, int64_t* steps, int steps_cap, uint64_t* post_draw) {
  Rng rng(seed);
  TabuTrace trace;
  try {
    TabuResult r = tabu_search(from_words(n, start), TabuParams{fmin, fmax}, rng,
                               workers, &trace);
    to_words(r.best, best);
    *best_energy = r.energy;
  } catch (const std::exception&) {
    return -1;
  }
  info[0] = trace.max_iter;
  info[1] = trace.min_tabu;
  info[2] = trace.max_tabu;
  int m = static_cast<int>(trace.steps.size());
  for (int i = 0; i < m && i < steps_cap; ++i) {
    steps[5 * i + 0] = trace.steps[i].iteration;
    steps[5 * i + 1] = trace.steps[i].position;
    steps[5 * i + 2] = trace.steps[i].energy;
    steps[5 * i + 3] = trace.steps[i].tenure;
    steps[5 * i + 4] = trace.steps[i].fallback ? 1 : 0;
  }
  if (post_draw) *post_draw = rng.bits64();
  return m;
}

int ref_memetic(int n, int pop, double p_comb, double p_mutate, int64_t target,
                double max_seconds, int64_t max_iterations, double fmin,
                double fmax, uint64_t seed, RefResult* out,
                int64_t* child_energies, int64_t cap) {
  MemeticParams p = make_params(pop, p_comb, p_mutate, target, max_seconds,
                                max_iterations, fmin, fmax);
  MemeticTrace trace;
  try {
    RunResult r = memetic_tabu(n, p, seed, nullptr, &trace, 0);
    fill(r, out);
  } catch (const std::exception&) {
    return -1;
  }
  int64_t m = static_cast<int64_t>(trace.iters.size());
  for (int64_t i = 0; i < m && i < cap; ++i)
    child_energies[i] = trace.iters[i].child_energy;
  return 0;
}

int ref_run_replicas(int n, int replicas, uint64_t base_seed, int pop,
                     double p_comb, double p_mutate, int64_t target,
                     double max_seconds, int64_t max_iterations, double fmin,
                     double fmax, int threaded, RefResult* out,
                     RefResult* per_replica) {
  ParallelConfig cfg;
  cfg.n = n;
  cfg.replicas = replicas;
  cfg.base_seed = base_seed;
  cfg.memetic = make_params(pop, p_comb, p_mutate, target, max_seconds,
                            max_iterations, fmin, fmax);
  cfg.run_threaded = threaded != 0;
  ReplicaReport report;
  try {
    RunResult r = run_replicas(cfg, &report);
    fill(r, out);
  } catch (const std::exception&) {
    return -1;
  }
  if (per_replica)
    for (int i = 0; i < replicas; ++i) fill(report.results[i], &per_replica[i]);
  return 0;
}

// brute_force_optimum (oracle.cpp:70-110): optimal E and canonical witnesses
// (words, sorted). Returns the witness count or -1.
int ref_brute_force(int n, int workers, int64_t* energy, uint64_t* witnesses, int cap) {
  try {
    BruteForceResult r = brute_force_optimum(n, workers);
    *energy = r.optimal_energy;
    const int nw = (n + 63) / 64;
    int c = 0;
    for (const Sequence& s : r.witnesses) {
      if (c < cap) to_words(s, witnesses + static_cast<size_t>(c) * nw);
      ++c;
    }
    return c;
  } catch (const std::exception&) {
    return -1;
  }
}

int64_t ref_local_optima(int n, int workers) {
  try {
    return enumerate_local_optima(n, workers);
  } catch (const std::exception&) {
    return -1;
  }
}

// deviation / deviation_with_edits (skew.cpp:110-187): out = {value,
// budget_exceeded, evaluations}.
int ref_deviation(int n, const uint64_t* w, uint64_t budget, int edits, int64_t* out) {
  try {
    DeviationResult d = edits ? deviation_with_edits(from_words(n, w), budget)
                              : deviation(from_words(n, w), budget);
    out[0] = d.value;
    out[1] = d.budget_exceeded ? 1 : 0;
    out[2] = static_cast<int64_t>(d.evaluations);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// CPU baseline: `threads` independent streams running the
// reference tabu_search back to back for `seconds`; stream t is seeded
// 42 + t, scan_workers = 1. Returns total tabu iterations (flip-evals / n).
int64_t ref_tabu_throughput(int n, int threads, double seconds,
                            int64_t* walks_out, double* elapsed_out) {
  std::vector<int64_t> iters(threads, 0), walks(threads, 0);
  auto t0 = std::chrono::steady_clock::now();
  auto body = [&](int t) {
    Rng rng(42 + static_cast<uint64_t>(t));
    TabuTrace trace;
    auto start = std::chrono::steady_clock::now();
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() -
                                         start)
               .count() < seconds) {
      Sequence s = Sequence::random(n, rng);
      tabu_search(s, TabuParams{}, rng, 1, &trace);
      iters[t] += trace.max_iter;
      walks[t] += 1;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(body, t);
  for (auto& th : pool) th.join();
  if (elapsed_out)
    *elapsed_out = std::chrono::duration<double>(
                       std::chrono::steady_clock::now() - t0)
                       .count();
  int64_t total = 0, w = 0;
  for (int t = 0; t < threads; ++t) {
    total += iters[t];
    w += walks[t];
  }
  if (walks_out) *walks_out = w;
  return total;
}

}  // extern "C"
