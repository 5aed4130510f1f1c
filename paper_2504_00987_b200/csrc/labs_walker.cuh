// labs_walker.cuh — the warp-resident LABS tabu walker (the hot path).
//
// One tile of T lanes owns one walker (T = 32: a warp; T = 16: half a warp,
// two walkers per warp stepping in lockstep). Candidate flip j lives in tile
// lane j % T, slot j / T (NS slots per lane, n <= L = T*NS). The reference scores
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
// - E (derivation: DESIGN.md §3; randomized proof-by-test:
// tests/test_oracle_cpu.py::test_incremental_identities; device parity:
// tests/test_parity_gpu.py).
//
// Register layout per slot: D = dE_j itself (for L <= 64 the argmin key
// 256 dE_j + j), MS = -s_j, EX = expiry, CK = C_j. With H = 4 h_j and
// HQ = 4 (n - 2 + Q_{2j}), dE_j = HQ + MS H, so a committed flip p changes D
// by
//   j != p:  dHQ + MS dH = -16 sigma s_{2j-p} + MS (16 s_{2p-j} - 8 sigma
//            (2 C_{|j-p|} + Q_{p+j})) - 32          (MS^2 = 1)
//   j == p:  D -> -D                   (flipping p back undoes the move)
// so neither h nor Q_{2j} is kept per slot. The operands are stored
// pre-scaled (WalkScales: spins x16, C and Q x8, all x256 more when keyed)
// so the update multiplies by sigma alone.
// Shared layout per walker: C mirrored as C2[L + d] = C_{|d|} so the gather
// C_{|j-p|} is one LDS at a per-step base + 128 b (one buffer: a step issues
// all its gathers before any store); Q[m]; spins as a zero-padded array
// S[SO + x] (int8; int32 for walkers of L <= 64) so s_x for any x in
// (-L-4, 2L+4) is one LDS with the range check folded into the padding. The
// flipped spin is stored at the start of the next step. The warp is
// converged through the step and its shared-memory accesses execute in
// order, so the step needs no barrier. Invalid positions (j >= n) keep
// EX = INT_MAX (never admissible) and s_j = 0, which makes every update they
// perform a no-op on the entries valid lanes read.
#pragma once
#include <climits>
#include <cstddef>
#include <cstdint>
#include <type_traits>

#include "labs_rng.cuh"

#ifndef LABS_TILE_BFLY
#define LABS_TILE_BFLY 0
#endif
#ifndef LABS_TIE_INLINE
#define LABS_TIE_INLINE 0
#endif

#ifndef LABS_TIE_XOR
#define LABS_TIE_XOR 1
#endif

#ifndef LABS_S4_MAX_L
#define LABS_S4_MAX_L 64
#endif
#ifndef LABS_SINGLE_C
#define LABS_SINGLE_C 1
#endif

namespace labsk {

#ifndef LABS_ADDR_ASM
#define LABS_ADDR_ASM 1
#endif
#ifndef LABS_CHECKED
#define LABS_CHECKED 0
#endif
// Compile-time loop: f(std::integral_constant<int, i>) for i in [0, N).
template <int N, int I = 0, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<N, I + 1>(f);
  }
}

// Shared loads/stores at a 32-bit shared-window address plus an immediate.
template <int OFF>
__device__ __forceinline__ int lds_s32_off(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
  return v;
}
template <int OFF>
__device__ __forceinline__ void sts_s32_off(uint32_t a, int v) {
  asm volatile("st.shared.s32 [%0+%1], %2;" ::"r"(a), "n"(OFF), "r"(v));
}
template <int E, int OFF>
__device__ __forceinline__ int lds_spin(uint32_t a) {
  int v;
  if constexpr (E == 4) asm volatile("ld.shared.s32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
  else asm volatile("ld.shared.s8 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"(OFF));
  return v;
}
template <int E>
__device__ __forceinline__ void sts_spin(uint32_t a, int v) {
  if constexpr (E == 4) asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v));
  else asm volatile("st.shared.s8 [%0], %1;" ::"r"(a), "r"(v));
}

// Scaled walker state: spins are stored as 16 s (shared memory), C and Q as
// 8 C / 8 Q (registers and shared memory), so the flip update multiplies by
// the sign sigma alone (no per-step constant ladder and no x16 shift of
// s_{2p-j}): D += -sigma (16 s_{2j-p}) + MS ((16 s_{2p-j}) - sigma (2 (8 C)
// + 8 Q)) - 32 is the update below with every operand as stored.
//
// For walkers of L <= LABS_S4_MAX_L (int32 spins) the scales grow by 256 so
// that D itself is the argmin key: D = 256 dE_j + j (keyed), spins 4096 s,
// C and Q 2048 C / 2048 Q. The selection then needs no per-slot key build,
// and the flipped slot becomes 2p - D.
template <int L>
struct WalkScales {
  static constexpr bool kKeyed = L <= LABS_S4_MAX_L;  // D carries the key
  static constexpr int kD = kKeyed ? 256 : 1;        // D = kD dE (+ j)
  static constexpr int kSpin = 16 * kD;              // step spins (S4 / S)
  static constexpr int kSpinShift = kKeyed ? 12 : 4;
  static constexpr int kS8 = kKeyed ? 1 : 16;        // the int8 spin array
  static constexpr int kC = 8 * kD;                  // C and Q
  static_assert(kSpin == 2 * kC, "the Q update uses 2 x the stored spin of p");
};

// Orders one step's shared-memory stores before the next step's loads by
// other lanes of the (converged) warp. LABS_STEP_FENCE=0 keeps only the
// compiler barrier: on a converged warp __syncwarp compiles to a NOP behind
// a divergence check, and a warp's shared-memory accesses execute in order.
#ifndef LABS_STEP_FENCE
#define LABS_STEP_FENCE 0
#endif
__device__ __forceinline__ void step_fence() {
  if constexpr (LABS_STEP_FENCE) __syncwarp();
  else asm volatile("" ::: "memory");
}

// redux.sync.min over the full warp. The walker's control flow is warp-
// uniform by construction, so the intrinsic's divergence guard is dead
// weight on the hot path.
__device__ __forceinline__ int warp_min(int v) {
  int r;
  asm volatile("redux.sync.min.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
  return r;
}

__device__ __forceinline__ uint32_t lowmask(int x);

template <int L_>
struct WalkSmemL {
  static constexpr int L = L_;
  static_assert(L % 32 == 0, "walker length must be a multiple of 32 positions");
  static constexpr int NC = L / 32;  // 32-bit chunks of a sequence
  // C mirror, C2[buf][L + d] = C_{|d|} for d in (-L, L). LABS_SINGLE_C: one
  // buffer — a step issues every gather before any store, and the warp's
  // shared accesses execute in order, so the stores never reach a gather of
  // the same step; else two buffers (a step reads one, writes the other).
  static constexpr int kCBuf = LABS_SINGLE_C ? 1 : 2;
  int32_t C2[kCBuf][2 * L];
  int32_t Q[2 * L];            // Q[m], m in [0, 2n-1)
  static constexpr int SO = L + 4;  // spin x lives at S[SO + x] and S4[SO + x]
  int8_t S[3 * L + 8];         // spins (+1/-1); 0 outside [0, n) (4 guard bytes)
  // For L <= LABS_S4_MAX_L the tabu step keeps its spins in an int32 copy
  // instead (its gathers then share scaled index registers with the Q
  // gather: +3% at n = 64, B200); for longer walkers the extra shared memory
  // costs more than it saves (-3% at n = 119), so the step uses S itself.
  static constexpr bool kS4 = L <= LABS_S4_MAX_L;
  int32_t S4[kS4 ? 3 * L + 8 : 1];
  __device__ __forceinline__ auto* spins() {
    if constexpr (kS4) return S4;
    else return S;
  }
  // Packed bit windows for the O(n^2/32) popcount build: B32 holds s
  // (position x at word (x + L) >> 5), R32 the reversed s (R_x = s_{n-1-x}),
  // V32 the validity mask (1 on [0, n)), all zero-padded, so a shifted
  // window of V32 masks exactly the valid pairs of a shifted window of s.
  // With two C buffers they alias the buffer that is idle until the walk's
  // first step; with one they (and the h build's int8 C) use W.
  static constexpr int kBitWords = 3 * NC + 2;
  static_assert(3 * kBitWords <= 2 * L, "bit windows must fit one C buffer");
  static constexpr int kScratchWords =
      LABS_SINGLE_C ? (3 * kBitWords > (L + 4 + 3) / 4 ? 3 * kBitWords : (L + 4 + 3) / 4) : 1;
  uint32_t W[kScratchWords];
  __device__ __forceinline__ uint32_t* scratch(int buf) {
    if constexpr (LABS_SINGLE_C) return W;
    else return reinterpret_cast<uint32_t*>(C2[buf]);
  }
  __device__ __forceinline__ uint32_t* B32(int buf) { return scratch(buf); }
  __device__ __forceinline__ uint32_t* R32(int buf) { return B32(buf) + kBitWords; }
  __device__ __forceinline__ uint32_t* V32(int buf) { return B32(buf) + 2 * kBitWords; }
  // Zero the windows of buffer `buf`, store the payload chunks of s and the
  // validity mask.
  template <int T>
  __device__ __forceinline__ void put_bits(int n, const uint32_t* in, int buf) {
    uint32_t* b = B32(buf);
    for (int i = tile_lane<T>(); i < 3 * kBitWords; i += T) b[i] = 0u;
    tile_sync<T>();
    if (tile_lane<T>() == 0)
      for (int c = 0; c < NC; ++c) {
        b[NC + c] = in[c] & lowmask(n - 32 * c);
        b[2 * kBitWords + NC + c] = lowmask(n - 32 * c);
      }
    tile_sync<T>();
  }
};
template <int NS>
using WalkSmem = WalkSmemL<32 * NS>;

__device__ __forceinline__ uint32_t lowmask(int x) {
  return x <= 0 ? 0u : (x >= 32 ? kFull : ((1u << x) - 1u));
}

// Zero the spin padding once per kernel; positions [0, n) are rewritten per
// walk.
template <int L, int T = 32>
__device__ __forceinline__ void smem_clear(WalkSmemL<L>& sm) {
  for (int i = tile_lane<T>(); i < 3 * L + 8; i += T) {
    sm.S[i] = 0;
    if constexpr (WalkSmemL<L>::kS4) sm.S4[i] = 0;
  }
  tile_sync<T>();
}

// Bits [o, o+32) of a zero-padded packed array of NC payload chunks
// (positions [-32 NC, 64 NC + 32)).
template <int NC>
__device__ __forceinline__ uint32_t window32(const uint32_t* A, int o) {
  const int u = o + 32 * NC;
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

template <int NS, int T = 32>
struct Walker {
  static constexpr int L = T * NS;
  using Smem = WalkSmemL<L>;
  using Sc = WalkScales<L>;
  static constexpr bool kKeyed = Sc::kKeyed;
  static constexpr int NC = Smem::NC;
  static constexpr int SO = Smem::SO;
  Smem* sm;
  int n;
  int D[NS], MS[NS], EX[NS], CK[NS];
  int E;
  int cb;        // C2 buffer holding the current C
  int pend_pos;  // flipped position whose spin store is pending (-1: none)
  int pend_val;
#if LABS_ADDR_ASM
  // Shared-window byte addresses of the step's gathers, lane constants set by
  // init (e = spin element size): aS0 = &spins[SO], aLm = aS0 - e ln,
  // aLp = aS0 + e ln, aL2 = aS0 + 2 e ln; for byte spins also the C mirror
  // and Q bases (for int32 spins those are aLp / aLm plus an immediate).
  // A step then forms each gather address with one IMAD of the flipped
  // position, and every slot offset is an immediate.
  uint32_t aS0, aLm, aLp, aL2, aCp, aCm, aQ;
  uint32_t pend_a;  // address of the pending spin store
#endif

  // Build C, Q, h, E from `in` (chunks of 32 positions, padding zero) with C
  // in buffer cb0 (the other buffer is scratch until the first step).
  // Divergence-safe: only the tile's lanes take part.
  __device__ __forceinline__ void init(int n_, const uint32_t (&in)[NC], int cb0 = 0) {
    n = n_;
    const int ln = tile_lane<T>();
    Smem& s = *sm;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = T * b + ln;
      const int c = (T * b) >> 5;
      const int bit = ((in[c] & lowmask(n - 32 * c)) >> (((T * b) & 31) + ln)) & 1u;
      const int sp = j < n ? 1 - 2 * bit : 0;
      MS[b] = -sp;
      s.S[SO + j] = static_cast<int8_t>(Sc::kS8 * sp);
      if constexpr (Smem::kS4) s.S4[SO + j] = Sc::kSpin * sp;
      EX[b] = j < n ? 0 : INT_MAX;
    }
    const int scratch = cb0 ^ 1;
    if constexpr (LABS_SINGLE_C) cb0 = 0;  // one C buffer; scratch is W
    s.template put_bits<T>(n, in, scratch);
    uint32_t* B32 = s.B32(scratch);
    uint32_t* R32 = s.R32(scratch);
    const uint32_t* V32 = s.V32(scratch);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      uint32_t word = 0;
#pragma unroll
      for (int b = c * 32 / T; b < (c + 1) * 32 / T; ++b) {
        const int i = T * b + ln;
        const bool rb = i < n && s.S[SO + n - 1 - i] < 0;
        word |= tile_ballot<T>(rb) << ((T * b) & 31);
      }
      if (ln == 0) R32[NC + c] = word;
    }
    tile_sync<T>();
    // C_k = (n-k) - 2 popc(s xor (s >> k)) over the n-k valid pairs.
    int e2 = 0;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int k = T * b + ln;
      int c = 0;
      if (k >= 1 && k < n) {
        const int len = n - k;
        int acc = 0;
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const uint32_t a = B32[NC + cc];
          const uint32_t x = window32<NC>(B32, 32 * cc + k);
          acc += __popc((a ^ x) & window32<NC>(V32, 32 * cc + k));  // pairs i + k < n
        }
        c = len - 2 * acc;
      }
      CK[b] = Sc::kC * c;
      s.C2[cb0][L + k] = Sc::kC * c;
      s.C2[cb0][L - k] = Sc::kC * c;
      e2 += c * c;
    }
    E = tile_sum<T>(e2);
    cb = cb0;
    pend_pos = -1;
    pend_val = 0;
#if LABS_ADDR_ASM
    {
      constexpr uint32_t e = sizeof(*s.spins());
      const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(&s));
      aS0 = base + static_cast<uint32_t>(reinterpret_cast<const char*>(s.spins() + SO) -
                                         reinterpret_cast<const char*>(&s));
      aLm = aS0 - e * ln;
      aLp = aS0 + e * ln;
      aL2 = aS0 + 2 * e * ln;
      aCp = base + 4u * (L + ln);
      aCm = base + 4u * (L - ln);
      aQ = base + static_cast<uint32_t>(offsetof(Smem, Q)) + 4u * ln;
      pend_a = aS0 - e;  // padding entry: the first flush rewrites its zero
    }
#endif
    // Q_m = sum_i s_i s_{m-i}: s against reversed s at offset n-1-m.
#pragma unroll 1
    for (int a = 0; a < 2 * NS; ++a) {
      const int m = T * a + ln;
      int qv = 0;
      if (m <= 2 * n - 2) {
        const int lo = m - n + 1 > 0 ? m - n + 1 : 0;
        const int hi = m < n - 1 ? m : n - 1;
        int acc = 0;
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          // s_i against s_{m-i} = R_{n-1-m+i}; the pair is valid where both
          // validity windows are set (i in [lo, hi])
          const int o = n - 1 - m + 32 * cc;
          const uint32_t x = window32<NC>(R32, o);
          acc += __popc((B32[NC + cc] ^ x) & V32[NC + cc] & window32<NC>(V32, o));
        }
        qv = (hi - lo + 1) - 2 * acc;
      }
      s.Q[m] = Sc::kC * qv;
    }
    tile_sync<T>();
    int h[NS], hq[NS];
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = T * b + ln;
      hq[b] = 4 * (n - 2) + s.Q[2 * j] / (Sc::kC / 4);  // 4 (n - 2 + Q_2j)
      h[b] = 0;
    }
    // h_j = sum_k C_k (s_{j+k} + s_{j-k}).
    if constexpr (L <= 128) {
      // |C_k| <= 127: four lags per DP4A. C as int8 in the scratch C buffer
      // (the bit windows are dead by now); spins read as 4-byte windows of
      // S, the backward window byte-reversed.
      int8_t* c8 = reinterpret_cast<int8_t*>(s.scratch(scratch));
      for (int k = ln; k < L + 4; k += T)
        c8[k] = static_cast<int8_t>(k >= 1 && k < n ? s.C2[cb0][L + k] / Sc::kC : 0);
      tile_sync<T>();
      const uint32_t* c8w = reinterpret_cast<const uint32_t*>(c8);
      const uint32_t* s32 = reinterpret_cast<const uint32_t*>(s.S);
#pragma unroll
      for (int b = 0; b < NS; ++b) {
        const int j = T * b + ln;
        const int fa = SO + j;          // byte of s_j (forward window start)
        const int ba = SO + j - 3;      // byte of s_{j-3} (backward window start)
        const uint32_t* fp = s32 + (fa >> 2);
        const uint32_t* bp = s32 + (ba >> 2);
        const int fsh = 8 * (fa & 3), bsh = 8 * (ba & 3);
        int acc = 0;
        for (int m = 0; 4 * m < n; ++m) {
          const int cw = static_cast<int>(c8w[m]);
          const int fw = static_cast<int>(__funnelshift_r(fp[m], fp[m + 1], fsh));
          const uint32_t bw = __funnelshift_r(bp[-m], bp[-m + 1], bsh);
          acc = __dp4a(cw, fw, acc);
          acc = __dp4a(cw, static_cast<int>(__byte_perm(bw, 0u, 0x0123)), acc);
        }
        h[b] = acc / Sc::kS8;  // the spin bytes are scaled
      }
      tile_sync<T>();  // c8 readers done before the scratch buffer is reused
    } else {
#pragma unroll 2
      for (int k = 1; k < n; ++k) {
        const int c = s.C2[cb0][L + k] / Sc::kC;
#pragma unroll
        for (int b = 0; b < NS; ++b) {
          const int j = T * b + ln;
          h[b] += c * (static_cast<int>(s.S[SO + j + k]) + static_cast<int>(s.S[SO + j - k]));
        }
      }
#pragma unroll
      for (int b = 0; b < NS; ++b) h[b] /= Sc::kS8;
    }
    // Positions j >= n (MS = 0) drift by -32 per step; starting them at
    // 2^22 keeps them positive (never admissible, even under aspiration)
    // for > 10^5 steps, far beyond any walk.
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = T * b + ln;
      D[b] = (j < n ? hq[b] + MS[b] * 4 * h[b] : (1 << 22)) * Sc::kD + (Sc::kKeyed ? j : 0);
    }
  }

  // The selection's operand for every slot: the argmin key 256 dE_j + j
  // when keyed, else dE_j.
  __device__ __forceinline__ void raw(int (&d)[NS]) const {
#pragma unroll
    for (int b = 0; b < NS; ++b) d[b] = D[b];
  }

  // dE_j for every slot.
  __device__ __forceinline__ void delta(int (&dE)[NS]) const {
#pragma unroll
    for (int b = 0; b < NS; ++b) dE[b] = Sc::kKeyed ? D[b] >> 8 : D[b];
  }

  // Spin store of the previous flip, performed by every lane before it reads
  // S (each lane then observes its own store).
  // (pend_pos = -1, pend_val = 0 after init rewrites the zero padding byte
  // of position -1, so the store needs no guard.)
  __device__ __forceinline__ void flush_spin() {
    using E = std::remove_pointer_t<decltype(sm->spins())>;
    sm->spins()[SO + pend_pos] = static_cast<E>(pend_val);
  }

  // Commit flip `pos` (tile-uniform); its expiry becomes t + tenure. Reads
  // pre-flip values (C2[cb], Q, S) and writes C2[cb ^ 1] and Q[pos + j] (read
  // and written by lane j alone); one warp barrier orders this step's stores
  // before the next step's loads. Called by the whole warp (converged).
  __device__ __forceinline__ void apply(int pos, int dEp, int t, int tenure) {
    if (cb) apply_cb<1>(pos, dEp, t, tenure);
    else apply_cb<0>(pos, dEp, t, tenure);
  }

  // apply() with the C buffer index known at compile time (the tabu loop is
  // unrolled by two so the buffers alternate statically); CB = -1 reads the
  // index from `cb` (one step body, smaller code).
  template <int CB>
  __device__ __forceinline__ void apply_cb(int pos, int dEp, int t, int tenure) {
#if LABS_ADDR_ASM
    if constexpr (LABS_SINGLE_C || CB >= 0) {
      apply_asm<LABS_SINGLE_C ? 0 : CB>(pos, dEp, t, tenure);
      return;
    }
#else
    static_assert(!LABS_SINGLE_C, "the single C buffer needs the ordered (asm) update");
#endif
    const int ln = tile_lane<T>();
    Smem& s = *sm;
    flush_spin();
    const auto* sp0 = s.spins();  // int32 (short walkers) or int8 spins, x16
    const int sig16 = sp0[SO + pos];
    const int sig = sig16 >> Sc::kSpinShift;  // old s_p (+1 / -1)
    const int nsig = -sig;
    const int c32 = sig16 + sig16;  // 4 kC sigma (kSpin = 2 kC)
    const int cbv = CB >= 0 ? CB : cb;
    const int32_t* cgp = &s.C2[cbv][L + ln - pos];
    int32_t* cw = &s.C2[cbv ^ 1][L];
    int32_t* qp = &s.Q[pos + ln];
    const auto* s1p = &sp0[SO + 2 * pos - ln];
    const auto* s2p = &sp0[SO + 2 * ln - pos];
    const auto* smp = &sp0[SO + pos - ln];
    const auto* spp = &sp0[SO + pos + ln];
    const int exp_new = t + tenure;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = T * b + ln;
      const bool isp = j == pos;
      const int cg = cgp[T * b];    // 8 C_{|j-p|}
      const int qg = qp[T * b];     // 8 Q_{p+j}
      const int s1 = s1p[-T * b];   // 16 s_{2p-j}
      const int s2 = s2p[2 * T * b];  // 16 s_{2j-p}
      const int smv = smp[-T * b];  // 16 s_{p-j}
      const int spv = spp[T * b];   // 16 s_{p+j}
      // j != p: D += -16 sigma s_{2j-p} + MS (16 s_{2p-j} - 8 sigma (2 C_{|j-p|}
      //          + Q_{p+j})) - 32, with the scaled operands:
      const int wv = s1 + nsig * (cg + cg + qg);
      const int dn = D[b] + nsig * s2 + MS[b] * wv - 32 * Sc::kD;
      D[b] = isp ? (Sc::kKeyed ? 2 * pos - D[b] : -D[b]) : dn;  // j == p: dE_p -> -dE_p
      if (!isp) qp[T * b] = qg + c32 * MS[b];  // Q_{p+j} -= 4 sigma s_j
      CK[b] += nsig * (smv + spv);     // C_j -= 2 sigma (s_{p-j} + s_{p+j})
      cw[j] = CK[b];
      cw[-j] = CK[b];
      MS[b] = isp ? -MS[b] : MS[b];
      EX[b] = isp ? exp_new : EX[b];
    }
    cb = cbv ^ 1;
    pend_pos = pos;
    pend_val = -sig16;
    E += dEp;
    step_fence();
  }

#if LABS_ADDR_ASM
  // Per-step operands of apply_asm's slot updates.
  struct StepOps {
    uint32_t a1, a2, a3, a4, a5, a6, aW, aWm;
    int pos, ln, nsig, c32, exp_new;
  };
  // A slot's six gathers (pre-flip values).
  struct SlotIn {
    int cg, qg, s1, s2, smv, spv;
  };
  template <int CB>
  static constexpr int kBufC = LABS_SINGLE_C ? 0 : CB * 8 * L;
  template <int CB>
  static constexpr int kBufW = LABS_SINGLE_C ? 0 : (CB ^ 1) * 8 * L;
  using SpinT = std::remove_pointer_t<decltype(static_cast<Smem*>(nullptr)->spins())>;
  static constexpr int kE = sizeof(SpinT);
  static constexpr bool kS4 = kE == 4;
  static constexpr int kCOff = kS4 ? 4 * L - (int)offsetof(Smem, S4) - 4 * SO : 0;
  static constexpr int kQOff = kS4 ? (int)offsetof(Smem, Q) - (int)offsetof(Smem, S4) - 4 * SO : 0;

#if LABS_CHECKED
  // Checked builds (-DLABS_CHECKED=1; compute-sanitizer is unavailable on
  // this pool): every gather/store address of the step must fall inside its
  // own array, and a spin read outside [0, n) must hit the zero padding.
  __device__ uint32_t smem_base() const {
    return aS0 - static_cast<uint32_t>(reinterpret_cast<const char*>(sm->spins() + SO) -
                                       reinterpret_cast<const char*>(sm));
  }
  __device__ void check_addr(uint32_t a, int bytes, int array, int line) const {
    const uint32_t base = smem_base();
    uint32_t lo, hi;
    if (array == 0) {  // C mirror
      lo = base + static_cast<uint32_t>(offsetof(Smem, C2));
      hi = lo + sizeof(sm->C2);
    } else if (array == 1) {  // Q
      lo = base + static_cast<uint32_t>(offsetof(Smem, Q));
      hi = lo + sizeof(sm->Q);
    } else {  // spins
      lo = base + static_cast<uint32_t>(reinterpret_cast<const char*>(sm->spins()) -
                                        reinterpret_cast<const char*>(sm));
      hi = lo + static_cast<uint32_t>(kE * (3 * L + 8));
    }
    if (a < lo || a + bytes > hi) {
      printf("LABS_CHECKED line %d: lane %d address %u outside array %d [%u, %u)\n", line,
             tile_lane<T>(), a, array, lo, hi);
      __trap();
    }
  }
  __device__ void check_spin(uint32_t a, int v, int line) const {
    check_addr(a, kE, 2, line);
    const int x = static_cast<int>(a - aS0) / kE;  // logical position
    if ((x < 0 || x >= n) && v != 0) {
      printf("LABS_CHECKED line %d: spin read at position %d (n = %d) is %d, not padding\n",
             line, x, n, v);
      __trap();
    }
  }
#endif

  template <int CB, int B>
  __device__ __forceinline__ void slot_load(const StepOps& o, SlotIn (&v)[NS]) {
    constexpr int e = kE;
    v[B].cg = lds_s32_off<kBufC<CB> + kCOff + 4 * T * B>(o.a5);  // kC C_{|j-p|}
    v[B].qg = lds_s32_off<kQOff + 4 * T * B>(o.a6);              // kC Q_{p+j}
    v[B].s1 = lds_spin<e, -e * T * B>(o.a1);                     // kSpin s_{2p-j}
    v[B].s2 = lds_spin<e, 2 * e * T * B>(o.a4);                  // kSpin s_{2j-p}
    v[B].smv = lds_spin<e, -e * T * B>(o.a2);                    // kSpin s_{p-j}
    v[B].spv = lds_spin<e, e * T * B>(o.a3);                     // kSpin s_{p+j}
#if LABS_CHECKED
    check_addr(o.a5 + kBufC<CB> + kCOff + 4 * T * B, 4, 0, __LINE__);
    check_addr(o.a6 + kQOff + 4 * T * B, 4, 1, __LINE__);
    check_spin(o.a1 - e * T * B, v[B].s1, __LINE__);
    check_spin(o.a4 + 2 * e * T * B, v[B].s2, __LINE__);
    check_spin(o.a2 - e * T * B, v[B].smv, __LINE__);
    check_spin(o.a3 + e * T * B, v[B].spv, __LINE__);
#endif
    if constexpr (B + 1 < NS) slot_load<CB, B + 1>(o, v);
  }
  template <int CB, int B>
  __device__ __forceinline__ void slot_store(const StepOps& o, const SlotIn (&v)[NS]) {
    const int j = T * B + o.ln;
    const bool isp = j == o.pos;
    const int wv = v[B].s1 + o.nsig * (v[B].cg + v[B].cg + v[B].qg);
    if constexpr (NS >= 3) {
      // D += delta, or the flip's -D (2p - D keyed) as an increment, so D
      // stays in its register (no select into a temporary and copy back):
      // +3 % at n = 119, -0.3 % at n = 64 (measured), hence NS >= 3 only
      const int delta = MS[B] * wv + (o.nsig * v[B].s2 - 32 * Sc::kD);
      const int flip = Sc::kKeyed ? 2 * o.pos - D[B] - D[B] : -D[B] - D[B];
      D[B] += isp ? flip : delta;
    } else {
      const int dn = D[B] + o.nsig * v[B].s2 + MS[B] * wv - 32 * Sc::kD;
      D[B] = isp ? (Sc::kKeyed ? 2 * o.pos - D[B] : -D[B]) : dn;
    }
#if LABS_CHECKED
    check_addr(o.aW + kBufW<CB> + kCOff + 4 * T * B, 4, 0, __LINE__);
    check_addr(o.aWm + kBufW<CB> + kCOff - 4 * T * B, 4, 0, __LINE__);
#endif
    if (!isp) sts_s32_off<kQOff + 4 * T * B>(o.a6, v[B].qg + o.c32 * MS[B]);
    CK[B] += o.nsig * (v[B].smv + v[B].spv);
    sts_s32_off<kBufW<CB> + kCOff + 4 * T * B>(o.aW, CK[B]);
    sts_s32_off<kBufW<CB> + kCOff - 4 * T * B>(o.aWm, CK[B]);
    MS[B] = isp ? -MS[B] : MS[B];
    EX[B] = isp ? o.exp_new : EX[B];
    if constexpr (B + 1 < NS) slot_store<CB, B + 1>(o, v);
  }

  // apply_cb with explicit shared-window addressing: one IMAD per gather
  // base per step, every slot offset and buffer choice an immediate.
  template <int CB>
  __device__ __forceinline__ void apply_asm(int pos, int dEp, int t, int tenure) {
    constexpr int e = kE;
    sts_spin<e>(pend_a, pend_val);  // the previous flip's spin
    const uint32_t up = static_cast<uint32_t>(pos);
    const uint32_t a_sig = aS0 + e * up;
    const int sig16 = lds_spin<e, 0>(a_sig);
#if LABS_CHECKED
    check_addr(pend_a, e, 2, __LINE__);
    check_addr(a_sig, e, 2, __LINE__);
    if (pos < 0 || pos >= n || sig16 == 0) {
      printf("LABS_CHECKED: flip position %d (n = %d) with spin %d\n", pos, n, sig16);
      __trap();
    }
#endif
    const int sig = sig16 >> Sc::kSpinShift;
    StepOps o;
    o.nsig = -sig;
    o.c32 = sig16 + sig16;  // 4 kC sigma (kSpin = 2 kC)
    o.pos = pos;
    o.ln = tile_lane<T>();
    o.exp_new = t + tenure;
    o.a1 = aLm + 2 * e * up;  // s_{2p-j}
    o.a2 = aLm + e * up;      // s_{p-j}
    o.a3 = aLp + e * up;      // s_{p+j}
    o.a4 = aL2 - e * up;      // s_{2j-p}
    // C_{|j-p|} at C2[CB][L + j - p]; Q_{p+j}; C stores at C2[CB^1][L +- j]
    // (for int32 spins the C and Q bases are the spin lanes + immediates)
    o.a5 = (kS4 ? aLp : aCp) - 4 * up;
    o.a6 = kS4 ? o.a3 : aQ + 4 * up;
    o.aW = kS4 ? aLp : aCp;
    o.aWm = kS4 ? aLm : aCm;
    SlotIn v[NS];
    slot_load<CB, 0>(o, v);   // every gather of the step ...
    slot_store<CB, 0>(o, v);  // ... before any store (one C buffer)
    cb = CB ^ 1;
    pend_pos = pos;
    pend_a = a_sig;
    pend_val = -sig16;
    E += dEp;
    step_fence();
  }
#endif

  // Current sequence as 32-bit chunks (bit 1 = spin -1). Divergence-safe.
  __device__ __forceinline__ void chunks(uint32_t (&out)[NC]) const {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      uint32_t word = 0;
#pragma unroll
      for (int b = c * 32 / T; b < (c + 1) * 32 / T; ++b)
        word |= tile_ballot<T>(MS[b] > 0) << ((T * b) & 31);
      out[c] = word;
    }
  }
};

// Value of a per-slot quantity at a tile-uniform position (one lane owns it).
template <int NS, int T = 32>
__device__ __forceinline__ int at_position(const int (&v)[NS], int pos) {
  int mine = 0;
#pragma unroll
  for (int b = 0; b < NS; ++b) mine += (T * b + tile_lane<T>() == pos) ? v[b] : 0;
  return tile_sum<T>(mine);
}

// Position of the r-th (0-based) candidate, in ascending position order,
// among the lanes/slots whose `hit` flag is set (msk[b] = tile ballot of
// hit[b]). Rank arithmetic + a tile min keep every array index compile-time.
template <int NS, int T = 32>
__device__ __forceinline__ int nth_hit(const bool (&hit)[NS],
                                       const uint32_t (&msk)[NS], int r) {
  const int ln = tile_lane<T>();
  const uint32_t below = (1u << ln) - 1u;
  int base = 0, cand = INT_MAX;
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    const int rank = base + __popc(msk[b] & below);
    if (hit[b] && rank == r) cand = T * b + ln;
    base += __popc(msk[b]);
  }
  return tile_min<T>(cand);
}

// Tile minimum with the whole warp converged (the tabu step): one redux per
// warp for T = 32; for T = 16 two reduxes over masked copies (independent,
// so their latencies overlap); a butterfly otherwise.
template <int T>
__device__ __forceinline__ int tile_min_converged(int v) {
  if constexpr (T == 32) {
    return warp_min(v);
  } else if constexpr (T == 16 && !LABS_TILE_BFLY) {
    const bool hi = lane_id() >= 16;
    const int a = warp_min(hi ? INT_MAX : v);
    const int b = warp_min(hi ? v : INT_MAX);
    return hi ? b : a;
  } else {
#pragma unroll
    for (int o = T / 2; o; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
    return v;
  }
}

// Per-slot values passed by value to the out-of-line selection paths.
template <int NS>
struct SlotVals {
  int v[NS];
};
template <class R>
struct Pick {
  int pos;
  int aux;  // dE of the fallback move, or the tie count
  R rng;
};

// Fallback of scan_neighborhood (correlation_state.cpp:156-160): nothing is
// admissible, so one uniform_int(0, n-1) draw picks the move. Out of line:
// rare, and it keeps the tabu step's code compact.
template <int NS, int T, class R>
__device__ __noinline__ Pick<R> fallback_pick(SlotVals<NS> dE, int n, R rng) {
  const int pos = uniform_below(rng, static_cast<uint32_t>(n));
  return {pos, at_position<NS, T>(dE.v, pos), rng};
}

// Tie among the admissible minima (correlation_state.cpp:161-165):
// ties[uniform_int(0, #ties - 1)] in ascending position order. Out of line
// (taken on a minority of steps).
template <int NS, int T, class R>
__device__ __noinline__ Pick<R> tie_pick(SlotVals<NS> key, int dmin, int pos, R rng) {
  bool hit[NS];
  uint32_t msk[NS];
  int cnt = 0;
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    hit[b] = (key.v[b] >> 8) == dmin;
    msk[b] = tile_ballot<T>(hit[b]);
    cnt += __popc(msk[b]);
  }
  if (cnt > 1) {
    const int r = uniform_below(rng, static_cast<uint32_t>(cnt));
    if (r) pos = nth_hit<NS, T>(hit, msk, r);
  }
  return {pos, cnt, rng};
}

// Select the move at iteration t: admissible argmin with the tie/fallback
// semantics of scan_neighborhood (proj/src/correlation_state.cpp:141-165).
// Keys pack dE * 256 + j, so one tile min yields the minimum and its lowest
// position (|dE| < 2^22 and j < 256 for n <= 256). Whether the minimum is
// tied is decided before any tile-divergent branch (T = 32: a second min
// over the other keys; T < 32: one warp ballot of "same dE, other position",
// i.e. 0 < key ^ kmin < 256); the tie set (ballots) is only built when it is
// tied (or when FULL_TIES asks for it). Must be entered by the whole warp.
template <int NS, int T, bool FULL_TIES, class R, bool KEYED = false>
__device__ __forceinline__ void select_move(const int (&dE)[NS],
                                            const bool (&adm)[NS], int n,
                                            int tie_rule, R& rng, int& pos,
                                            int& dEp, int& fallback,
                                            uint32_t (&msk)[NS], int& ntie) {
  const int ln = tile_lane<T>();
  SlotVals<NS> key;
  int kmin = INT_MAX;
#pragma unroll
  for (int b = 0; b < NS; ++b) {
    key.v[b] = adm[b] ? (KEYED ? dE[b] : dE[b] * 256 + T * b + ln) : INT_MAX;
    kmin = min(kmin, key.v[b]);
  }
  kmin = tile_min_converged<T>(kmin);
  bool tied_other = false;
  if constexpr ((T < 32 || LABS_TIE_XOR) && !FULL_TIES) {
    bool h = false;
#pragma unroll
    for (int b = 0; b < NS; ++b)
      h |= static_cast<uint32_t>((key.v[b] ^ kmin) - 1) < 255u;
    if constexpr (T == 32) tied_other = __any_sync(kFull, h);
    else tied_other = tile_bits<T>(__ballot_sync(kFull, h)) != 0u;
  }
  if (kmin == INT_MAX) {
    SlotVals<NS> d;
#pragma unroll
    for (int b = 0; b < NS; ++b) d.v[b] = KEYED ? dE[b] >> 8 : dE[b];
    if constexpr (LABS_RARE_INLINE) {
      pos = uniform_below(rng, static_cast<uint32_t>(n));
      dEp = at_position<NS, T>(d.v, pos);
    } else {
      const Pick<R> f = fallback_pick<NS, T>(d, n, rng);
      rng = f.rng;
      pos = f.pos;
      dEp = f.aux;
    }
    fallback = 1;
    ntie = 0;
#pragma unroll
    for (int b = 0; b < NS; ++b) msk[b] = 0u;
    return;
  }
  const int dmin = kmin >> 8;
  pos = kmin & 255;
  dEp = dmin;
  fallback = 0;
  ntie = 1;
  if constexpr (FULL_TIES) {
    // every tie reported (labs_scan): the tie set is always built
    bool hit[NS];
    int cnt = 0;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      hit[b] = (key.v[b] >> 8) == dmin;
      msk[b] = tile_ballot<T>(hit[b]);
      cnt += __popc(msk[b]);
    }
    ntie = cnt;
    if (cnt > 1 && tie_rule == 0) {
      const int r = uniform_below(rng, static_cast<uint32_t>(cnt));
      if (r) pos = nth_hit<NS, T>(hit, msk, r);
    }
  } else if (tie_rule == 0) {
    bool tied;
    if constexpr (T < 32 || LABS_TIE_XOR) {
      tied = tied_other;
    } else {
      int k2 = INT_MAX;
#pragma unroll
      for (int b = 0; b < NS; ++b) k2 = min(k2, key.v[b] == kmin ? INT_MAX : key.v[b]);
      k2 = warp_min(k2);
      tied = (k2 >> 8) == dmin;
    }
    if (tied) {
      if constexpr (LABS_TIE_INLINE || LABS_RARE_INLINE) {
        bool hit[NS];
        int cnt = 0;
#pragma unroll
        for (int b = 0; b < NS; ++b) {
          hit[b] = (key.v[b] >> 8) == dmin;
          msk[b] = tile_ballot<T>(hit[b]);
          cnt += __popc(msk[b]);
        }
        ntie = cnt;
        if (cnt > 1) {
          const int r = uniform_below(rng, static_cast<uint32_t>(cnt));
          if (r) pos = nth_hit<NS, T>(hit, msk, r);
        }
      } else {
        const Pick<R> tp = tie_pick<NS, T>(key, dmin, pos, rng);
        rng = tp.rng;
        pos = tp.pos;
        ntie = tp.aux;
      }
    }
  }
}

// tabu_search (proj/src/tabu.cpp:17-56) for one walker. `in` is the start
// sequence; on return `best` holds the best visited sequence (the start
// counts as visited) and the return value is its energy.
template <int NS, bool ASP, bool TRACE, class R>
__device__ __forceinline__ int tabu_walk_impl(Walker<NS>& w, int n,
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
  const int tie_rule = cfg.tie_rule;
  const uint32_t tenure_range = static_cast<uint32_t>(max_t - min_t + 1);
#pragma unroll
  for (int b = 0; b < NS; ++b) best[b] = in[b] & lowmask(n - 32 * b);
  auto step = [&](auto cbc, int t) {
    int dE[NS];
    bool adm[NS];
    w.delta(dE);
    // aspiration (not in the reference): a tabu move is admissible if it
    // lands strictly below the walk's best.
    if (ASP) {
      const int thr = bestE - w.E;
#pragma unroll
      for (int b = 0; b < NS; ++b) adm[b] = (w.EX[b] < t) | (dE[b] < thr);
    } else {
#pragma unroll
      for (int b = 0; b < NS; ++b) adm[b] = w.EX[b] < t;
    }
    int pos, dEp, fb, ntie;
    uint32_t msk[NS];
    select_move<NS, 32, false>(dE, adm, n, tie_rule, rng, pos, dEp, fb, msk, ntie);
    const int tenure = min_t + uniform_below(rng, tenure_range);
    w.template apply_cb<decltype(cbc)::value>(pos, dEp, t, tenure);
    if (w.E < bestE) {
      bestE = w.E;
      w.chunks(best);
    }
    if (TRACE && lane_id() == 0) {
      StepRec rec;
      rec.iteration = t;
      rec.position = pos;
      rec.energy = w.E;
      rec.tenure = tenure;
      rec.fallback = fb;
      trace[t - 1] = rec;
    }
  };
  // Unrolled by two: even steps read C buffer 0, odd steps buffer 1.
  for (int t = 1; t <= m; t += 2) {
    step(std::integral_constant<int, 0>{}, t);
    if (t + 1 > m) break;
    step(std::integral_constant<int, 1>{}, t + 1);
  }
  if (steps_out) *steps_out = m;
  return bestE;
}

template <int NS, class R>
__device__ __forceinline__ int tabu_walk(Walker<NS>& w, int n, const uint32_t (&in)[NS],
                                         R& rng, const TabuCfg& cfg, uint32_t (&best)[NS],
                                         int* info, StepRec* trace, int* steps_out) {
  if (trace) {
    if (cfg.aspiration)
      return tabu_walk_impl<NS, true, true>(w, n, in, rng, cfg, best, info, trace, steps_out);
    return tabu_walk_impl<NS, false, true>(w, n, in, rng, cfg, best, info, trace, steps_out);
  }
  if (cfg.aspiration)
    return tabu_walk_impl<NS, true, false>(w, n, in, rng, cfg, best, info, nullptr, steps_out);
  return tabu_walk_impl<NS, false, false>(w, n, in, rng, cfg, best, info, nullptr, steps_out);
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

template <int NS, int T = 32>
__device__ __forceinline__ void store_chunks(uint64_t* w, int nw,
                                             const uint32_t (&c)[NS]) {
  if (tile_lane<T>() == 0) {
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
