// labs_memetic.cuh — the memetic layer, one warp per replica (K4).
//
// Restates memetic_tabu (proj/src/memetic.cpp:44-117) on device: random
// population, binary tournaments (memetic.cpp:8-22), uniform crossover
// (:24-33), Bernoulli mutation (:35-42), the tabu refinement (labs_walker.cuh)
// and uniform replacement (:100-102), with the reference's draw order and
// loop-check order. Population, energies, best and the RNG state live in
// global memory between launches, so a run can be cut into epochs (the
// island model exchanges elites between epochs) without changing any
// replica's trajectory.
#pragma once
#include <cstdint>

#include "labs_b200.h"
#include "labs_walker.cuh"

namespace labsk {

enum ReplicaStatus : int32_t {
  kRunning = 0,
  kReached = 1,
  kStopped = 2,   // saw the stop flag
  kMaxIter = 3,
  kTimeout = 4,
};

struct MemeticArgs {
  int n, nw, replicas, K;
  double p_comb, p_mutate;
  int64_t target;
  int64_t max_ns;          // < 0: unlimited (max_seconds)
  int64_t max_iterations;  // < 0: unlimited
  int64_t epoch_iters;     // < 0: run to completion in this launch
  int64_t epoch_ns;        // < 0: no per-launch time slice
  int crossover;           // 0 uniform (reference), 1 one-point
  int replacement;         // 0 random victim (reference), 1 worst if better
  TabuCfg tabu;
  int race;                // raise *stop when a replica reaches the target
  uint64_t base_seed;      // Philox key
  int64_t replica_offset;  // global id of local replica 0
  // replica state (global memory)
  uint64_t* pop;           // R x K x nw
  int32_t* popE;           // R x K
  uint64_t* best;          // R x nw
  int32_t* bestE;          // R
  int64_t* iters;          // R
  int32_t* status;         // R
  int32_t* initialized;    // R
  int64_t* t0;             // R, globaltimer at init
  int64_t* t_end;          // R, globaltimer at exit
  int32_t* pub_order;      // R, order in which finished replicas published
  int32_t* pub_counter;    // 1
  labs_rng_state* mt;      // R (MT mode)
  uint64_t* ctr;           // R (Philox mode)
  volatile int32_t* stop;  // device-resident stop flag
  unsigned long long* tabu_iters;  // accumulated tabu iterations (optional)
  int64_t* tabu_per_replica;       // R, tabu iterations per replica
  // optional trace
  int64_t* trace;          // R x cap x 3 {iteration, stop_seen, child_energy}
  int64_t trace_cap;
  int64_t* trace_len;      // R
};

__device__ __forceinline__ int64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return static_cast<int64_t>(t);
}

// E = sum C_k^2 of a sequence given as chunks (uses the walker's bit arrays).
template <int NS>
__device__ __forceinline__ int energy_of(WalkSmem<NS>& s, int n,
                                         const uint32_t (&c)[NS]) {
  const int ln = lane_id();
  s.put_bits(n, c);
  const uint32_t* B32 = s.B32();
  int e2 = 0;
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    const int k = 32 * b + ln;
    if (k >= 1 && k < n) {
      const int len = n - k;
      int acc = 0;
#pragma unroll
      for (int cc = 0; cc < NS; ++cc) {
        const uint32_t a = B32[NS + cc];
        const uint32_t x = window32<NS>(B32, 32 * cc + k);
        acc += __popc((a ^ x) & lowmask(len - 32 * cc));
      }
      const int cv = len - 2 * acc;
      e2 += cv * cv;
    }
  }
  __syncwarp();
  return __reduce_add_sync(kFull, e2);
}

template <int NS>
__device__ __forceinline__ void load_seq(const uint64_t* g, int nw,
                                         uint32_t (&c)[NS]) {
  load_chunks<NS>(g, nw, c);
}

// mutate (memetic.cpp:35-42): draw i decides position i; lane i takes draw i
// of each chunk of <= 32 draws (chunks never straddle an mt19937 twist).
template <int NS, class R>
__device__ __forceinline__ void mutate_chunks(uint32_t (&c)[NS], int n,
                                              double p, R& rng) {
  const int ln = lane_id();
  int done = 0;
  while (done < n) {
    int room = rng.room();
    int chunk = n - done < 32 ? n - done : 32;
    if (room < chunk) chunk = room;
    bool flip = false;
    if (ln < chunk) flip = u01_from_bits(rng.peek_lane(ln)) < p;
    uint32_t m = __ballot_sync(kFull, flip);
    rng.advance(chunk);
    // XOR m into positions [done, done + chunk)
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int o = done - 32 * b;  // chunk start relative to word b
      const uint32_t lo = (o >= 0 && o < 32) ? (m << o) : 0u;
      const uint32_t hi = (o < 0 && o > -32) ? (m >> (-o)) : 0u;
      c[b] ^= lo | hi;
    }
    done += chunk;
  }
}

// First index of the maximum energy (warp-parallel scan over K entries).
__device__ __forceinline__ int worst_member(const int32_t* e, int K) {
  long long best = -1;
  for (int i = lane_id(); i < K; i += 32) {
    const long long key = (static_cast<long long>(e[i]) << 32) | (0x7fffffff - i);
    best = key > best ? key : best;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const long long other = __shfl_xor_sync(kFull, best, o);
    best = other > best ? other : best;
  }
  return 0x7fffffff - static_cast<int>(best & 0xffffffffLL);
}

template <class R>
__device__ __forceinline__ int tournament(const int32_t* e, int K, R& rng) {
  const int a = static_cast<int>(uniform_int(rng, 0, K - 1));
  const int b = static_cast<int>(uniform_int(rng, 0, K - 1));
  const int ea = e[a], eb = e[b];
  if (ea < eb) return a;
  if (eb < ea) return b;
  return uniform_int(rng, 0, 1) == 0 ? a : b;
}

// One replica for as long as this launch allows. Returns with the replica's
// state saved in global memory.
template <int NS, class R>
__device__ void memetic_replica(const MemeticArgs& A, int r, Walker<NS>& w,
                                R& rng) {
  const int ln = lane_id();
  const int n = A.n, nw = A.nw, K = A.K;
  uint64_t* pop = A.pop + static_cast<size_t>(r) * K * nw;
  int32_t* popE = A.popE + static_cast<size_t>(r) * K;
  uint64_t* best = A.best + static_cast<size_t>(r) * nw;

  if (!A.initialized[r]) {
    // Population: K x Sequence::random (sequence.cpp:28-33), then energies.
    for (int i = 0; i < K; ++i) {
      for (int wi = 0; wi < nw; ++wi) {
        uint64_t v = rng.next();
        if (wi == nw - 1 && (n & 63)) v &= (1ULL << (n & 63)) - 1ULL;
        if (ln == 0) pop[static_cast<size_t>(i) * nw + wi] = v;
      }
    }
    __syncwarp();
    __threadfence_block();
    int bi = 0, be = 0;
    for (int i = 0; i < K; ++i) {
      uint32_t c[NS];
      load_seq<NS>(pop + static_cast<size_t>(i) * nw, nw, c);
      const int e = energy_of<NS>(*w.sm, n, c);
      if (ln == 0) popE[i] = e;
      if (i == 0 || e < be) {  // first strict minimum (memetic.cpp:72-74)
        be = e;
        bi = i;
      }
    }
    if (ln == 0) {
      for (int wi = 0; wi < nw; ++wi)
        best[wi] = pop[static_cast<size_t>(bi) * nw + wi];
      A.bestE[r] = be;
      A.iters[r] = 0;
      A.status[r] = kRunning;
      A.initialized[r] = 1;
      A.t0[r] = globaltimer_ns();
      if (A.trace_len) A.trace_len[r] = 0;
    }
    __syncwarp();
  }
  if (A.status[r] != kRunning) return;

  int bestE = A.bestE[r];
  int64_t it = A.iters[r];
  const int64_t t0 = A.t0[r];
  int64_t tlen = A.trace_len ? A.trace_len[r] : 0;
  const int64_t it_start = it;
  const int64_t resume_ns = globaltimer_ns();
  int32_t st = kRunning;
  unsigned long long tabu_steps = 0;
  while (true) {
    // Loop-top checks in reference order (memetic.cpp:79-85).
    if (!(static_cast<int64_t>(bestE) > A.target)) {
      st = kReached;
      break;
    }
    if (*A.stop) {
      if (A.trace && tlen < A.trace_cap && ln == 0) {
        int64_t* rec = A.trace + (static_cast<size_t>(r) * A.trace_cap + tlen) * 3;
        rec[0] = it;
        rec[1] = 1;
        rec[2] = -1;
      }
      ++tlen;
      st = kStopped;
      break;
    }
    if (A.max_iterations >= 0 && it >= A.max_iterations) {
      st = kMaxIter;
      break;
    }
    if (A.max_ns >= 0 && globaltimer_ns() - t0 >= A.max_ns) {
      st = kTimeout;
      break;
    }
    if (A.epoch_iters >= 0 && it - it_start >= A.epoch_iters) break;  // epoch
    if (A.epoch_ns >= 0 && globaltimer_ns() - resume_ns >= A.epoch_ns) break;

    uint32_t child[NS];
    if (uniform01(rng) < A.p_comb) {
      const int p1 = tournament(popE, K, rng);
      const int p2 = tournament(popE, K, rng);
      uint32_t a[NS], b[NS];
      load_seq<NS>(pop + static_cast<size_t>(p1) * nw, nw, a);
      load_seq<NS>(pop + static_cast<size_t>(p2) * nw, nw, b);
      if (A.crossover == 0) {
        // combine (memetic.cpp:24-33): one bits64() mask per 64-bit word.
#pragma unroll
        for (int wi = 0; wi < (NS + 1) / 2; ++wi) {
          const uint64_t mask = rng.next();
          const uint32_t mlo = static_cast<uint32_t>(mask);
          const uint32_t mhi = static_cast<uint32_t>(mask >> 32);
          child[2 * wi] = (a[2 * wi] & mlo) | (b[2 * wi] & ~mlo);
          if (2 * wi + 1 < NS)
            child[2 * wi + 1] = (a[2 * wi + 1] & mhi) | (b[2 * wi + 1] & ~mhi);
        }
      } else {
        // one-point: positions [0, cut) from parent 1, [cut, n) from parent 2.
        const int cut = static_cast<int>(uniform_int(rng, 1, n - 1));
#pragma unroll
        for (int b2 = 0; b2 < NS; ++b2) {
          const uint32_t m1 = lowmask(cut - 32 * b2);
          child[b2] = (a[b2] & m1) | (b[b2] & ~m1);
        }
      }
#pragma unroll
      for (int b2 = 0; b2 < NS; ++b2) child[b2] &= lowmask(n - 32 * b2);
    } else {
      const int idx = static_cast<int>(uniform_int(rng, 0, K - 1));
      load_seq<NS>(pop + static_cast<size_t>(idx) * nw, nw, child);
    }
    mutate_chunks<NS>(child, n, A.p_mutate, rng);
    uint32_t refined[NS];
    int steps = 0;
    const int re =
        tabu_walk<NS>(w, n, child, rng, A.tabu, refined, nullptr, nullptr, &steps);
    tabu_steps += static_cast<unsigned long long>(steps);
    if (re < bestE) {
      bestE = re;
      store_chunks<NS>(best, nw, refined);
    }
    if (A.replacement == 0) {
      // memetic.cpp:100-102: uniform victim, best not protected.
      const int victim = static_cast<int>(uniform_int(rng, 0, K - 1));
      store_chunks<NS>(pop + static_cast<size_t>(victim) * nw, nw, refined);
      if (ln == 0) popE[victim] = re;
    } else {
      // elite-preserving: the child displaces the worst member if better.
      const int victim = worst_member(popE, K);
      if (re < popE[victim]) {
        store_chunks<NS>(pop + static_cast<size_t>(victim) * nw, nw, refined);
        if (ln == 0) popE[victim] = re;
      }
    }
    if (A.trace && tlen < A.trace_cap && ln == 0) {
      int64_t* rec = A.trace + (static_cast<size_t>(r) * A.trace_cap + tlen) * 3;
      rec[0] = it;
      rec[1] = 0;
      rec[2] = re;
    }
    ++tlen;
    ++it;
    __syncwarp();
    if (A.race && !(static_cast<int64_t>(bestE) > A.target) && ln == 0)
      *A.stop = 1;  // parallel.cpp:40 — reaching the target raises the flag
  }
  if (ln == 0) {
    A.bestE[r] = bestE;
    A.iters[r] = it;
    if (A.trace_len) A.trace_len[r] = tlen;
    if (A.tabu_iters) atomicAdd(A.tabu_iters, tabu_steps);
    if (A.tabu_per_replica) A.tabu_per_replica[r] += static_cast<int64_t>(tabu_steps);
    if (st != kRunning) {
      A.status[r] = st;
      A.t_end[r] = globaltimer_ns();
      A.pub_order[r] = atomicAdd(A.pub_counter, 1);
    }
  }
  __syncwarp();
}

}  // namespace labsk
