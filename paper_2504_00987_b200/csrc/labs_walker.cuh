// labs_walker.cuh — the warp-resident LABS tabu walker (the hot path).
//
// One warp owns one walker. Candidate flip j lives in lane j % 32, slot
// j / 32 (NS = ceil(n/32) slots per lane, n <= 32*NS). The reference scores
// every candidate with an O(n) pass over the packed product table
// (proj/src/correlation_state.cpp:50-71), O(n^2) per tabu iteration. This
// walker keeps four small integer vectors instead and updates all of them in
// O(1) per element per committed flip, so a tabu iteration costs O(n):
//
//   C_k = sum_i s_i s_{i+k}                       (k = 1..n-1, autocorrelation)
//   Q_m = sum_i s_i s_{m-i}                       (m = 0..2n-2, self-convolution)
//   h_j = sum_{i != j} C_{|i-j|} s_i              (j = 0..n-1, Toeplitz field)
//   dE_j = 4 (n - 2 + Q_{2j} - s_j h_j)           (exact energy change of flip j)
//
// Committing flip p (sigma = old s_p), for j != p:
//   h_j += -4 sigma C_{|j-p|} + 4 s_{2p-j} - 2 sigma Q_{p+j} + 8 s_j
//   Q_{p+j} -= 4 sigma s_j ;   Q_{2j} -= 4 sigma s_{2j-p}
//   C_j  -= 2 sigma (s_{p-j} + s_{p+j})
// and h_p -= 2 sigma (n - 2 + Q_{2p}); E += dE_p. All right-hand sides use the
// pre-flip vectors; s_x = 0 outside [0, n). Everything is exact int32
// arithmetic, so dE_j is bit-identical to the reference's neighbor_energy(j)
// - E (derivation and the randomized proof-by-test: DESIGN.md §3,
// tests/test_oracle_cpu.py::test_incremental_identities).
//
// Layout: h, Q_{2j}, s_j, expiry and C_j stay in registers (one per slot);
// C and Q also live in shared memory for the two lane-varying gathers
// C_{|j-p|} and Q_{p+j}; spins live in a zero-padded int8 shared array so
// s_x for any x in [-L, 2L) is one LDS with the range check folded into the
// padding. The tabu list is the per-slot `ex` register: admissible iff
// ex < t (proj/src/tabu.cpp:43-47).
#pragma once
#include <climits>
#include <cstdint>

#include "labs_rng.cuh"

namespace labsk {

template <int NS>
struct WalkSmem {
  static constexpr int L = 32 * NS;
  int32_t C[L];                // C[k], k in [1, n); C[0] and k >= n hold 0
  int32_t Q[2 * L];            // Q[m], m in [0, 2n-1)
  uint32_t B32[3 * NS + 2];    // bits of s; position x at word (x + L) >> 5
  uint32_t R32[3 * NS + 2];    // bits of reversed s (R_x = s_{n-1-x})
  int8_t S[3 * L];             // spins (+1/-1), S[L + x]; 0 outside [0, n)
};

// Zero the padding once per kernel; positions [0, n) are rewritten per walk.
template <int NS>
__device__ __forceinline__ void smem_clear(WalkSmem<NS>& sm) {
  const int lane = lane_id();
  for (int i = lane; i < 3 * NS + 2; i += 32) {
    sm.B32[i] = 0u;
    sm.R32[i] = 0u;
  }
  for (int i = lane; i < 3 * 32 * NS; i += 32) sm.S[i] = 0;
  __syncwarp();
}

__device__ __forceinline__ uint32_t lowmask(int x) {
  return x <= 0 ? 0u : (x >= 32 ? kFull : ((1u << x) - 1u));
}

// Bits [o, o+32) of a zero-padded packed array (positions [-L, 2L+32)).
template <int NS>
__device__ __forceinline__ uint32_t window32(const uint32_t* A, int o) {
  const int u = o + 32 * NS;
  const int w = u >> 5, r = u & 31;
  return __funnelshift_r(A[w], A[w + 1], r);
}

struct TabuCfg {
  double min_factor;
  double max_factor;
  int tie_rule;     // 0 = reference (uniform draw among ties), 1 = lowest index
  int aspiration;   // 1: a tabu move that beats the walk's best is admissible
};

struct StepRec {      // mirrors labs_tabu_step (include/labs_b200.h)
  int32_t iteration;
  int32_t position;
  int64_t energy;
  int32_t tenure;
  int32_t fallback;
};

template <int NS>
struct Walker {
  static constexpr int L = 32 * NS;
  WalkSmem<NS>* sm;
  int n;
  // per-slot registers (candidate j = 32*b + lane)
  int h[NS], q[NS], sp[NS], ex[NS], ck[NS];
  int E;

  __device__ __forceinline__ int lane() const { return lane_id(); }

  // Build C, Q, h, E from `in` (chunks of 32 positions, padding zero).
  __device__ __forceinline__ void init(int n_, const uint32_t (&in)[NS]) {
    n = n_;
    const int ln = lane();
    WalkSmem<NS>& s = *sm;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = 32 * b + ln;
      const int bit = ((in[b] & lowmask(n - 32 * b)) >> ln) & 1u;
      sp[b] = j < n ? 1 - 2 * bit : 0;
      s.S[L + j] = static_cast<int8_t>(sp[b]);
      ex[b] = 0;
    }
    if (ln == 0) {
#pragma unroll
      for (int b = 0; b < NS; ++b) s.B32[NS + b] = in[b] & lowmask(n - 32 * b);
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int i = 32 * b + ln;
      const bool rb = i < n && s.S[L + n - 1 - i] < 0;
      const uint32_t m = __ballot_sync(kFull, rb);
      if (ln == 0) s.R32[NS + b] = m;
    }
    __syncwarp();
    // C_k = (n-k) - 2 popc(s xor (s >> k)) over the n-k valid pairs.
    int e2 = 0;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int k = 32 * b + ln;
      int c = 0;
      if (k >= 1 && k < n) {
        const int len = n - k;
        int acc = 0;
#pragma unroll
        for (int cc = 0; cc < NS; ++cc) {
          const uint32_t a = s.B32[NS + cc];
          const uint32_t x = window32<NS>(s.B32, 32 * cc + k);
          acc += __popc((a ^ x) & lowmask(len - 32 * cc));
        }
        c = len - 2 * acc;
      }
      ck[b] = c;
      s.C[k] = c;
      e2 += c * c;
    }
    E = __reduce_add_sync(kFull, e2);
    // Q_m = sum_i s_i s_{m-i}: s against reversed s at offset n-1-m.
#pragma unroll 1
    for (int a = 0; a < 2 * NS; ++a) {
      const int m = 32 * a + ln;
      int qv = 0;
      if (m <= 2 * n - 2) {
        const int lo = m - n + 1 > 0 ? m - n + 1 : 0;
        const int hi = m < n - 1 ? m : n - 1;
        int acc = 0;
#pragma unroll
        for (int cc = 0; cc < NS; ++cc) {
          const uint32_t vm =
              lowmask(hi - 32 * cc + 1) & ~lowmask(lo - 32 * cc);
          if (vm) {
            const uint32_t x = window32<NS>(s.R32, n - 1 - m + 32 * cc);
            acc += __popc((s.B32[NS + cc] ^ x) & vm);
          }
        }
        qv = (hi - lo + 1) - 2 * acc;
      }
      s.Q[m] = qv;
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = 32 * b + ln;
      q[b] = s.Q[2 * j];
      h[b] = 0;
    }
    // h_j = sum_k C_k (s_{j+k} + s_{j-k}).
#pragma unroll 2
    for (int k = 1; k < n; ++k) {
      const int c = s.C[k];
#pragma unroll
      for (int b = 0; b < NS; ++b) {
        const int j = 32 * b + ln;
        h[b] += c * (static_cast<int>(s.S[L + j + k]) +
                     static_cast<int>(s.S[L + j - k]));
      }
    }
  }

  // dE_j for every slot.
  __device__ __forceinline__ void delta(int (&dE)[NS]) const {
#pragma unroll
    for (int b = 0; b < NS; ++b) dE[b] = 4 * (n - 2 + q[b] - sp[b] * h[b]);
  }

  // Commit flip `pos` (warp-uniform). Expiry of pos becomes t + tenure.
  // Phase A updates registers slot by slot from pre-flip shared values; the
  // only cross-lane hazards (C[j] and S[pos] read by other lanes) are written
  // in phase B after a warp barrier. Q[pos+j] is read and written by lane j
  // alone, so it is updated in place during phase A.
  __device__ __forceinline__ void apply(int pos, int dEp, int t, int tenure) {
    const int ln = lane();
    WalkSmem<NS>& s = *sm;
    const int sig = s.S[L + pos];
    const int sig2 = 2 * sig, sig4 = 4 * sig;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = 32 * b + ln;
      const int d = j - pos;
      const int cg = s.C[d < 0 ? -d : d];
      const int qg = s.Q[pos + j];
      const int s1 = s.S[L + 2 * pos - j];
      const int s2 = s.S[L + 2 * j - pos];
      const int sm_ = s.S[L + pos - j];
      const int spl = s.S[L + pos + j];
      if (j < n) {
        if (j != pos) {
          h[b] += 4 * s1 + 8 * sp[b] - sig4 * cg - sig2 * qg;
          s.Q[pos + j] = qg - sig4 * sp[b];
          q[b] -= sig4 * s2;
        } else {
          h[b] -= sig2 * (n - 2 + q[b]);
          sp[b] = -sp[b];
          ex[b] = t + tenure;
        }
        if (j >= 1) ck[b] -= sig2 * (sm_ + spl);
      }
    }
    __syncwarp();
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = 32 * b + ln;
      if (j >= 1 && j < n) s.C[j] = ck[b];
      if (j == pos) s.S[L + pos] = static_cast<int8_t>(-sig);
    }
    E += dEp;
    __syncwarp();
  }

  // Current sequence as 32-bit chunks (bit 1 = spin -1), from the spins.
  __device__ __forceinline__ void chunks(uint32_t (&out)[NS]) const {
#pragma unroll
    for (int b = 0; b < NS; ++b) out[b] = __ballot_sync(kFull, sp[b] < 0);
  }
};

// Value of a per-slot quantity at a warp-uniform position (one lane owns it).
template <int NS>
__device__ __forceinline__ int at_position(const int (&v)[NS], int pos) {
  int mine = 0;
#pragma unroll
  for (int b = 0; b < NS; ++b) mine += (32 * b + lane_id() == pos) ? v[b] : 0;
  return __reduce_add_sync(kFull, mine);
}

// Position of the r-th (0-based) candidate, in ascending position order,
// among the lanes/slots whose `hit` flag is set (msk[b] = ballot of hit[b]).
// Rank arithmetic + a warp min keep every array index compile-time.
template <int NS>
__device__ __forceinline__ int nth_hit(const bool (&hit)[NS],
                                       const uint32_t (&msk)[NS], int r) {
  const int ln = lane_id();
  const uint32_t below = (1u << ln) - 1u;
  int base = 0, cand = INT_MAX;
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    const int rank = base + __popc(msk[b] & below);
    if (hit[b] && rank == r) cand = 32 * b + ln;
    base += __popc(msk[b]);
  }
  return __reduce_min_sync(kFull, cand);
}

// Select the move at iteration t: admissible argmin with the tie/fallback
// semantics of scan_neighborhood (proj/src/correlation_state.cpp:141-165).
// adm_ext: optional external admissibility (one bit per slot per lane).
template <int NS, class R>
__device__ __forceinline__ void select_move(const int (&dE)[NS],
                                            const bool (&adm)[NS], int n,
                                            int tie_rule, R& rng, int& pos,
                                            int& dEp, int& fallback,
                                            uint32_t (&msk)[NS], int& ntie) {
  int key[NS];
  int kmin = INT_MAX;
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    key[b] = adm[b] ? dE[b] : INT_MAX;
    kmin = min(kmin, key[b]);
  }
  kmin = __reduce_min_sync(kFull, kmin);
  if (kmin == INT_MAX) {
    pos = static_cast<int>(uniform_int(rng, 0, n - 1));
    dEp = at_position<NS>(dE, pos);
    fallback = 1;
    ntie = 0;
#pragma unroll
    for (int b = 0; b < NS; ++b) msk[b] = 0u;
    return;
  }
  int cnt = 0;
  bool hit[NS];
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    hit[b] = key[b] == kmin;
    msk[b] = __ballot_sync(kFull, hit[b]);
    cnt += __popc(msk[b]);
  }
  int r = 0;
  if (cnt > 1 && tie_rule == 0)
    r = static_cast<int>(uniform_int(rng, 0, static_cast<long long>(cnt) - 1));
  pos = nth_hit<NS>(hit, msk, r);
  dEp = kmin;
  fallback = 0;
  ntie = cnt;
}

// tabu_search (proj/src/tabu.cpp:17-56) for one walker. `in` is the start
// sequence; on return `best` holds the best visited sequence (the start
// counts as visited) and the return value is its energy.
template <int NS, class R>
__device__ __forceinline__ int tabu_walk(Walker<NS>& w, int n,
                                         const uint32_t (&in)[NS], R& rng,
                                         const TabuCfg& cfg,
                                         uint32_t (&best)[NS], int* info,
                                         StepRec* trace, int* steps_out) {
  // sample_max_iter (tabu.cpp:12-15) and the tenure window (tabu.cpp:27-28):
  // floor(f * m + 1e-9) with two rounded double operations, no FMA.
  const int m = static_cast<int>(uniform_int(rng, 0, n)) + n / 2;
  const int min_t = static_cast<int>(
      floor(__dadd_rn(__dmul_rn(cfg.min_factor, static_cast<double>(m)), 1e-9)));
  const int max_t = static_cast<int>(
      floor(__dadd_rn(__dmul_rn(cfg.max_factor, static_cast<double>(m)), 1e-9)));
  if (info && lane_id() == 0) {
    info[0] = m;
    info[1] = min_t;
    info[2] = max_t;
  }
  w.init(n, in);
  int bestE = w.E;
#pragma unroll
  for (int b = 0; b < NS; ++b) best[b] = in[b] & lowmask(n - 32 * b);
  for (int t = 1; t <= m; ++t) {
    int dE[NS];
    bool adm[NS];
    w.delta(dE);
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = 32 * b + lane_id();
      adm[b] = j < n && (w.ex[b] < t || (cfg.aspiration && w.E + dE[b] < bestE));
    }
    int pos, dEp, fb, ntie;
    uint32_t msk[NS];
    select_move<NS>(dE, adm, n, cfg.tie_rule, rng, pos, dEp, fb, msk, ntie);
    const int tenure = static_cast<int>(uniform_int(rng, min_t, max_t));
    w.apply(pos, dEp, t, tenure);
    if (w.E < bestE) {
      bestE = w.E;
      w.chunks(best);
    }
    if (trace && lane_id() == 0) {
      StepRec rec;
      rec.iteration = t;
      rec.position = pos;
      rec.energy = w.E;
      rec.tenure = tenure;
      rec.fallback = fb;
      trace[t - 1] = rec;
    }
  }
  if (steps_out) *steps_out = m;
  return bestE;
}

// u64 words (global layout) <-> 32-bit chunks (register layout).
template <int NS>
__device__ __forceinline__ void load_chunks(const uint64_t* w, int nw,
                                            uint32_t (&c)[NS]) {
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    const int wi = b >> 1;
    const uint64_t v = wi < nw ? w[wi] : 0ULL;
    c[b] = (b & 1) ? static_cast<uint32_t>(v >> 32) : static_cast<uint32_t>(v);
  }
}

template <int NS>
__device__ __forceinline__ void store_chunks(uint64_t* w, int nw,
                                             const uint32_t (&c)[NS]) {
  if (lane_id() == 0) {
#pragma unroll
    for (int wi = 0; wi < (NS + 1) / 2; ++wi) {
      if (wi < nw) {
        const uint64_t lo = c[2 * wi];
        const uint64_t hi = 2 * wi + 1 < NS ? c[2 * wi + 1] : 0u;
        w[wi] = lo | (hi << 32);
      }
    }
  }
}

}  // namespace labsk
