// labs_memetic.cuh — the memetic layer, one tile (warp or half-warp) per
// replica (K4).
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

#ifndef LABS_UNROLL_T32
#define LABS_UNROLL_T32 1
#endif
#ifndef LABS_UNROLL_MAX_NS
#define LABS_UNROLL_MAX_NS 2
#endif
#ifndef LABS_UNROLL_EXTRA_NS  // one more walker width that is unrolled
#define LABS_UNROLL_EXTRA_NS 4
#endif
#ifndef LABS_UNROLL_T16
#define LABS_UNROLL_T16 0
#endif

namespace labsk {

constexpr int kMaxPeerStops = LABS_MAX_PEERS;

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
  // Stop flags of the other islands (other GPUs over NVLink P2P, or other
  // processes' flags opened through CUDA IPC): a replica reaching the target
  // raises them together with its own, so every GPU sees the stop at its
  // next loop check without a host round trip (parallel.cpp:40's
  // request_stop, across devices).
  int npeers;
  int32_t* const* peer_stop;  // npeers device pointers (global memory)
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

// Tile-uniform reads of values other agents change concurrently (the global
// timer, the stop flag): tile lane 0 reads, the tile agrees, so every lane
// takes the same branch.
#ifndef LABS_BCAST_READS
#define LABS_BCAST_READS 1
#endif
#ifndef LABS_CTL_SYNC
#define LABS_CTL_SYNC 1
#endif
template <int T>
__device__ __forceinline__ int64_t tile_globaltimer_ns() {
  if constexpr (LABS_BCAST_READS) return __shfl_sync(tile_mask<T>(), globaltimer_ns(), 0, T);
  else return globaltimer_ns();
}
template <int T>
__device__ __forceinline__ bool tile_stop_seen(const volatile int32_t* stop) {
  if constexpr (LABS_BCAST_READS) return __shfl_sync(tile_mask<T>(), *stop, 0, T) != 0;
  else return *stop != 0;
}

// Reaching the target raises the stop flag (parallel.cpp:40), and the flags
// of the other islands (peer GPUs over NVLink, or IPC-mapped flags of other
// processes). Out of line: it runs once per run and must not cost the
// tabu loop registers.
static __device__ __noinline__ void raise_stop(volatile int32_t* stop, int32_t* const* peers,
                                        int npeers) {
  *stop = 1;
  for (int p = 0; p < npeers; ++p) *reinterpret_cast<volatile int32_t*>(peers[p]) = 1;
  if (npeers) __threadfence_system();
}

// E = sum C_k^2 of a sequence given as chunks (uses scratch C buffer 1's
// bit windows; only called while the tile has no walk in flight).
template <int NS, int T>
__device__ __forceinline__ int energy_of(WalkSmemL<T * NS>& s, int n,
                                         const uint32_t (&c)[(T * NS) / 32]) {
  constexpr int NC = (T * NS) / 32;
  const int ln = tile_lane<T>();
  s.template put_bits<T>(n, c, 1);
  const uint32_t* B32 = s.B32(1);
  int e2 = 0;
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    const int k = T * b + ln;
    if (k >= 1 && k < n) {
      const int len = n - k;
      int acc = 0;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const uint32_t a = B32[NC + cc];
        const uint32_t x = window32<NC>(B32, 32 * cc + k);
        acc += __popc((a ^ x) & lowmask(len - 32 * cc));
      }
      const int cv = len - 2 * acc;
      e2 += cv * cv;
    }
  }
  tile_sync<T>();
  return tile_sum<T>(e2);
}

// mutate (memetic.cpp:35-42): draw i decides position i; tile lane i takes
// draw i of each chunk of <= T draws (chunks never straddle a refill).
template <int NC, int T, class R>
__device__ __forceinline__ void mutate_chunks(uint32_t (&c)[NC], int n,
                                              double p, R& rng) {
  const int ln = tile_lane<T>();
  int done = 0;
  while (done < n) {
    int room = rng.room();
    int chunk = n - done < T ? n - done : T;
    if (room < chunk) chunk = room;
    bool flip = false;
    if (ln < chunk) flip = u01_from_bits(rng.peek_lane(ln)) < p;
    const uint32_t m = tile_ballot<T>(flip);
    rng.advance(chunk);
    // XOR m into positions [done, done + chunk)
#pragma unroll
    for (int b = 0; b < NC; ++b) {
      const int o = done - 32 * b;  // chunk start relative to word b
      const uint32_t lo = (o >= 0 && o < 32) ? (m << o) : 0u;
      const uint32_t hi = (o < 0 && o > -32) ? (m >> (-o)) : 0u;
      c[b] ^= lo | hi;
    }
    done += chunk;
  }
}

// First index of the maximum energy (tile-parallel scan over K entries).
template <int T = 32>
__device__ __forceinline__ int worst_member(const int32_t* e, int K) {
  long long best = -1;
  for (int i = tile_lane<T>(); i < K; i += T) {
    const long long key = (static_cast<long long>(e[i]) << 32) | (0x7fffffff - i);
    best = key > best ? key : best;
  }
#pragma unroll
  for (int o = T / 2; o; o >>= 1) {
    const long long other = __shfl_xor_sync(tile_mask<T>(), best, o);
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

// Cold per-tile replica bookkeeping, kept in shared memory so that it does
// not occupy registers across the tabu loop. Every lane of the tile reads
// and writes identical values; an update reads its operands, waits at a
// tile barrier, then writes, so no lane can overwrite a value another lane
// has yet to read.
struct TileCtl {
  int64_t it, it_start, t0, tlen, resume_ns;
  unsigned long long tabu_steps;
  int r;          // current replica (global index within this launch)
  int have;       // a replica is bound
  int bestE;
  int ran;        // the tile has run at least one walk (its walker is valid)
};

// The memetic layer (memetic_tabu, proj/src/memetic.cpp:44-117) for every
// replica a tile owns, restated as a per-tile state machine so that the
// tiles of a warp (T < 32: several replicas per warp) run their tabu steps
// in lockstep: each loop iteration first lets the tiles whose walk has ended
// do their memetic bookkeeping (tile-divergent: post-walk replacement,
// loop-top checks in reference order, replica switch, child generation,
// walk start), then all tiles execute one tabu step together (converged, so
// the per-step argmin and barrier serve every tile at once). The draw order
// of each replica is exactly that of memetic_replica in the reference:
// pop init -> [u01 -> (tournaments + masks | copy idx) -> mutate -> maxIter
// -> tabu steps (tie draw?, tenure) -> victim] per iteration.
//
// RB binds a replica's RNG: load(r) before its first draw, save(r) after its
// last draw in this launch.
template <int NS, int T, bool ASP, bool TIE_REF, class R, class RB>
__device__ __forceinline__ void memetic_tiles(const MemeticArgs& A, Walker<NS, T>& w,
                                              R& rng, RB& rb, TileCtl& ctl) {
  constexpr int NC = (T * NS) / 32;
  // Unrolled by two for short walkers (the two bodies keep different
  // register assignments, which saves moves), and at NS = 4 (+0.6% at
  // n = 119); one body at NS = 3 (-1.4% / +1.3% at n = 80 / 96 unrolled) and
  // from NS = 5 on.
  constexpr bool kUnroll =
      T == 32 ? (LABS_UNROLL_T32 && (NS <= LABS_UNROLL_MAX_NS || NS == LABS_UNROLL_EXTRA_NS))
              : LABS_UNROLL_T16;
  const int ln = tile_lane<T>();
  const int n = A.n, nw = A.nw, K = A.K;
  const int G = gridDim.x * (blockDim.x / T);  // tiles in the grid
  constexpr int tie_rule = TIE_REF ? 0 : 1;  // A.tabu.tie_rule, as a constant
  ctl.r = blockIdx.x * (blockDim.x / T) + static_cast<int>(threadIdx.x) / T - G;
  ctl.have = 0;
  ctl.ran = 0;
  // walk state (registers)
  int t = 1, m = 0, wbestE = 0;
  uint32_t wbest[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) wbest[c] = 0u;
  int par = 0;  // warp-uniform C-buffer parity of the next step

  // Finish the walk that just ended (memetic.cpp:94-107).
  auto post_walk = [&]() {
    const int r = ctl.r;
    const unsigned long long steps0 = ctl.tabu_steps;
    const int best0 = ctl.bestE;
    const int64_t tlen0 = ctl.tlen, it0 = ctl.it;
    if constexpr (LABS_CTL_SYNC) tile_sync<T>();
    uint64_t* pop = A.pop + static_cast<size_t>(r) * K * nw;
    int32_t* popE = A.popE + static_cast<size_t>(r) * K;
    ctl.tabu_steps = steps0 + static_cast<unsigned long long>(m);
    const int re = wbestE;
    if (re < best0) {
      ctl.bestE = re;
      store_chunks<NC, T>(A.best + static_cast<size_t>(r) * nw, nw, wbest);
    }
    if (A.replacement == 0) {
      // memetic.cpp:100-102: uniform victim, best not protected.
      const int victim = static_cast<int>(uniform_int(rng, 0, K - 1));
      store_chunks<NC, T>(pop + static_cast<size_t>(victim) * nw, nw, wbest);
      if (ln == 0) popE[victim] = re;
    } else {
      // elite-preserving: the child displaces the worst member if better.
      const int victim = worst_member<T>(popE, K);
      if (re < popE[victim]) {
        store_chunks<NC, T>(pop + static_cast<size_t>(victim) * nw, nw, wbest);
        if (ln == 0) popE[victim] = re;
      }
    }
    if (A.trace && tlen0 < A.trace_cap && ln == 0) {
      int64_t* rec = A.trace + (static_cast<size_t>(r) * A.trace_cap + tlen0) * 3;
      rec[0] = it0;
      rec[1] = 0;
      rec[2] = re;
    }
    ctl.tlen = tlen0 + 1;
    ctl.it = it0 + 1;
    tile_sync<T>();
    if (A.race && !(static_cast<int64_t>(re < best0 ? re : best0) > A.target) && ln == 0)
      raise_stop(A.stop, A.peer_stop, A.npeers);  // parallel.cpp:40
  };

  // Save the replica's state at the end of its part of this launch.
  auto end_replica = [&](int32_t st) {
    const int r = ctl.r;
    if (ln == 0) {
      A.bestE[r] = ctl.bestE;
      A.iters[r] = ctl.it;
      if (A.trace_len) A.trace_len[r] = ctl.tlen;
      if (A.tabu_iters) atomicAdd(A.tabu_iters, ctl.tabu_steps);
      if (A.tabu_per_replica) A.tabu_per_replica[r] += static_cast<int64_t>(ctl.tabu_steps);
      if (st != kRunning) {
        A.status[r] = st;
        A.t_end[r] = globaltimer_ns();
        A.pub_order[r] = atomicAdd(A.pub_counter, 1);
      }
    }
    tile_sync<T>();
    rb.save(r, rng);
    ctl.have = 0;
  };

  // Bind the next replica of this tile, initializing its population on
  // first use (memetic.cpp:64-76). Returns false when the tile has none left.
  auto next_replica = [&]() -> bool {
    while (true) {
      const int r = ctl.r + G;
      if constexpr (LABS_CTL_SYNC) tile_sync<T>();
      if (r >= A.replicas) return false;
      ctl.r = r;
      if (A.initialized[r] && A.status[r] != kRunning) continue;
      rb.load(r, rng);
      uint64_t* pop = A.pop + static_cast<size_t>(r) * K * nw;
      int32_t* popE = A.popE + static_cast<size_t>(r) * K;
      if (!A.initialized[r]) {
        // Population: K x Sequence::random (sequence.cpp:28-33), then energies.
        for (int i = 0; i < K; ++i) {
          for (int wi = 0; wi < nw; ++wi) {
            uint64_t v = rng.next();
            if (wi == nw - 1 && (n & 63)) v &= (1ULL << (n & 63)) - 1ULL;
            if (ln == 0) pop[static_cast<size_t>(i) * nw + wi] = v;
          }
        }
        tile_sync<T>();
        __threadfence_block();
        int bi = 0, be = 0;
        for (int i = 0; i < K; ++i) {
          uint32_t c[NC];
          load_chunks<NC>(pop + static_cast<size_t>(i) * nw, nw, c);
          const int e = energy_of<NS, T>(*w.sm, n, c);
          if (ln == 0) popE[i] = e;
          if (i == 0 || e < be) {  // first strict minimum (memetic.cpp:72-74)
            be = e;
            bi = i;
          }
        }
        if (ln == 0) {
          for (int wi = 0; wi < nw; ++wi)
            A.best[static_cast<size_t>(r) * nw + wi] = pop[static_cast<size_t>(bi) * nw + wi];
          A.bestE[r] = be;
          A.iters[r] = 0;
          A.status[r] = kRunning;
          A.initialized[r] = 1;
          A.t0[r] = globaltimer_ns();  // lane 0 only
          if (A.trace_len) A.trace_len[r] = 0;
        }
        tile_sync<T>();
      }
      ctl.bestE = A.bestE[r];
      ctl.it = A.iters[r];
      ctl.it_start = ctl.it;
      ctl.t0 = A.t0[r];
      ctl.tlen = A.trace_len ? A.trace_len[r] : 0;
      ctl.resume_ns = tile_globaltimer_ns<T>();
      ctl.tabu_steps = 0;
      ctl.have = 1;
      return true;
    }
  };

  // Everything between two walks of this tile. On return either a new walk
  // is set up (t = 1 <= m) or the tile is done (m = INT_MAX: it keeps
  // stepping its last, valid walker without side effects).
  auto control = [&](int cb0) {
    if (ctl.have) post_walk();
    while (true) {
      if (!ctl.have && !next_replica()) {
        if (!ctl.ran) {  // never walked: give it a valid dummy walker
          uint32_t z[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) z[c] = 0u;
          w.init(n, z, cb0);
          ctl.ran = 1;
        }
        m = INT_MAX;
        return;
      }
      // Loop-top checks in reference order (memetic.cpp:79-85).
      const int r = ctl.r;
      int32_t st = -1;
      if (!(static_cast<int64_t>(ctl.bestE) > A.target)) {
        st = kReached;
      } else if (tile_stop_seen<T>(A.stop)) {
        const int64_t tlen0 = ctl.tlen;
        if constexpr (LABS_CTL_SYNC) tile_sync<T>();
        if (A.trace && tlen0 < A.trace_cap && ln == 0) {
          int64_t* rec = A.trace + (static_cast<size_t>(r) * A.trace_cap + tlen0) * 3;
          rec[0] = ctl.it;
          rec[1] = 1;
          rec[2] = -1;
        }
        ctl.tlen = tlen0 + 1;
        st = kStopped;
      } else if (A.max_iterations >= 0 && ctl.it >= A.max_iterations) {
        st = kMaxIter;
      } else if (A.max_ns >= 0 && tile_globaltimer_ns<T>() - ctl.t0 >= A.max_ns) {
        st = kTimeout;
      } else if ((A.epoch_iters >= 0 && ctl.it - ctl.it_start >= A.epoch_iters) ||
                 (A.epoch_ns >= 0 && tile_globaltimer_ns<T>() - ctl.resume_ns >= A.epoch_ns)) {
        st = kRunning;  // epoch over: the replica continues in the next launch
      }
      if (st >= 0) {
        end_replica(st);
        continue;
      }
      const uint64_t* pop = A.pop + static_cast<size_t>(r) * K * nw;
      const int32_t* popE = A.popE + static_cast<size_t>(r) * K;
      uint32_t child[NC];
      if (uniform01(rng) < A.p_comb) {
        const int p1 = tournament(popE, K, rng);
        const int p2 = tournament(popE, K, rng);
        uint32_t a[NC], b[NC];
        load_chunks<NC>(pop + static_cast<size_t>(p1) * nw, nw, a);
        load_chunks<NC>(pop + static_cast<size_t>(p2) * nw, nw, b);
        if (A.crossover == 0) {
          // combine (memetic.cpp:24-33): one bits64() mask per 64-bit word.
#pragma unroll
          for (int wi = 0; wi < (NC + 1) / 2; ++wi) {
            const uint64_t mask = rng.next();
            const uint32_t mlo = static_cast<uint32_t>(mask);
            const uint32_t mhi = static_cast<uint32_t>(mask >> 32);
            child[2 * wi] = (a[2 * wi] & mlo) | (b[2 * wi] & ~mlo);
            if (2 * wi + 1 < NC)
              child[2 * wi + 1] = (a[2 * wi + 1] & mhi) | (b[2 * wi + 1] & ~mhi);
          }
        } else {
          // one-point: positions [0, cut) from parent 1, [cut, n) from parent 2.
          const int cut = static_cast<int>(uniform_int(rng, 1, n - 1));
#pragma unroll
          for (int b2 = 0; b2 < NC; ++b2) {
            const uint32_t m1 = lowmask(cut - 32 * b2);
            child[b2] = (a[b2] & m1) | (b[b2] & ~m1);
          }
        }
#pragma unroll
        for (int b2 = 0; b2 < NC; ++b2) child[b2] &= lowmask(n - 32 * b2);
      } else {
        const int idx = static_cast<int>(uniform_int(rng, 0, K - 1));
        load_chunks<NC>(pop + static_cast<size_t>(idx) * nw, nw, child);
      }
      mutate_chunks<NC, T>(child, n, A.p_mutate, rng);
      // tabu_search entry (tabu.cpp:12-29): maxIter, then the tenure window
      // floor(f * m + 1e-9) with two rounded double operations, no FMA.
      m = static_cast<int>(uniform_int(rng, 0, n)) + n / 2;
      const int min_t = static_cast<int>(
          floor(__dadd_rn(__dmul_rn(A.tabu.min_factor, static_cast<double>(m)), 1e-9)));
      const int max_t = static_cast<int>(
          floor(__dadd_rn(__dmul_rn(A.tabu.max_factor, static_cast<double>(m)), 1e-9)));
      rng.begin_walk(min_t, static_cast<uint32_t>(max_t - min_t + 1), m);
      w.init(n, child, cb0);
      ctl.ran = 1;
      wbestE = w.E;
#pragma unroll
      for (int c = 0; c < NC; ++c) wbest[c] = child[c];
      t = 1;
      return;
    }
  };

  // One tabu iteration of every tile's walk (tabu.cpp:31-53), whole warp.
  auto step = [&](auto cbc) {
    constexpr bool kKeyed = Walker<NS, T>::kKeyed;
    int dE[NS];  // dE_j, or the argmin key 256 dE_j + j when keyed
    bool adm[NS];
    w.raw(dE);
    if (ASP) {
      // aspiration (not in the reference): a tabu move is admissible if it
      // lands strictly below the walk's best (key < 256 thr <=> dE < thr).
      const int thr = (wbestE - w.E) * (kKeyed ? 256 : 1);
#pragma unroll
      for (int b = 0; b < NS; ++b) adm[b] = (w.EX[b] < t) | (dE[b] < thr);
    } else {
#pragma unroll
      for (int b = 0; b < NS; ++b) adm[b] = w.EX[b] < t;
    }
    int pos, dEp, fb, ntie;
    uint32_t msk[NS];
    select_move<NS, T, false, R, kKeyed>(dE, adm, n, tie_rule, rng, pos, dEp, fb, msk, ntie);
    const int tenure = rng.tenure();  // uniform_int(min_t, max_t) (tabu.cpp:49-50)
    w.template apply_cb<decltype(cbc)::value>(pos, dEp, t, tenure);
    if (w.E < wbestE) {
      wbestE = w.E;
      w.chunks(wbest);
    }
    ++t;
  };

  // Has any tile's walk ended? With one tile per warp t and m are
  // warp-uniform, so no vote is needed.
  auto walk_ended = [&]() -> bool {
    if constexpr (T == 32) return t > m;
    else return __any_sync(kFull, t > m);
  };

  // Outer loop: bookkeeping for the tiles whose walk ended. Inner loop (the
  // hot one): steps until some tile's walk ends. Unrolled by two (the C
  // buffers alternate statically) when both step bodies fit the L0
  // instruction cache together; otherwise one body reads the buffer index.
  while (true) {
    if (t > m) control(par);
    if (__all_sync(kFull, m == INT_MAX)) break;
    if constexpr (LABS_SINGLE_C && !kUnroll) {
      // one C buffer: a single step body
      do {
        step(std::integral_constant<int, 0>{});
      } while (!walk_ended());
    } else if constexpr (LABS_SINGLE_C && kUnroll) {
      // one C buffer, unrolled by two: no parity to carry between walks
      while (true) {
        step(std::integral_constant<int, 0>{});
        if (walk_ended()) break;
        step(std::integral_constant<int, 1>{});
        if (walk_ended()) break;
      }
    } else if constexpr (kUnroll) {
      if (par) goto odd;
      while (true) {
        step(std::integral_constant<int, 0>{});
        if (walk_ended()) {
          par = 1;
          break;
        }
      odd:
        step(std::integral_constant<int, 1>{});
        if (walk_ended()) {
          par = 0;
          break;
        }
      }
    } else {
      do {
        step(std::integral_constant<int, -1>{});
      } while (!walk_ended());
    }
  }
}

}  // namespace labsk
