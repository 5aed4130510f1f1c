// labs_kernels.cu — sm_100a kernels K1..K4 and the C ABI (include/labs_b200.h).
//
// Every kernel is warp-per-walker (or warp-per-replica): 4 independent warps
// per 128-thread block, no block-level barriers, each warp with a private
// slice of dynamic shared memory (WalkSmem + optional mt19937_64 state).
// Kernels are templated on NS = ceil(n/32) so the per-slot register arrays
// are fully unrolled; the host dispatches NS in [1, 8] (n <= 256).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "labs_b200.h"
#include "labs_exhaustive.cuh"
#include "labs_memetic.cuh"
#include "labs_walker.cuh"

namespace labsk {

constexpr int kWarps = 4;  // walkers per block

// Occupancy target. The walker is issue-bound (ncu: ~89% issue slots busy),
// so registers matter more than warps: 6 blocks (24 warps) per SM up to
// n = 128 caps registers at 85/thread, which removed the smem-base
// rematerialization of the 64-register build (+7% at n=64, +12% at n=119,
// measured); longer sequences carry twice the per-slot state.
#ifndef LABS_MINB_SMALL
#define LABS_MINB_SMALL 6
#endif
#ifndef LABS_MINB_LARGE
#define LABS_MINB_LARGE 4
#endif
template <int NS>
__host__ __device__ constexpr int min_blocks() {
  return NS <= 4 ? LABS_MINB_SMALL : LABS_MINB_LARGE;
}

// Shared memory of one walker (tile): RNG block, cold replica bookkeeping,
// walker vectors.
template <int L, bool MT>
struct TileSlot {
  uint64_t mt[MT ? kMtN : 1];    // raw mt19937_64 state
  uint64_t out[MT ? kMtN : PhiloxRng::kBlock];  // tempered block / Philox block
  TileCtl ctl;
  WalkSmemL<L> walk;
};

template <int L, bool MT>
__host__ __device__ constexpr size_t tile_slot_bytes() {
  return (sizeof(TileSlot<L, MT>) + 15) & ~size_t(15);
}

// Tile t of the block owns slot t; T = 32 is the warp-per-walker kernels'.
template <int L, bool MT, int T>
__device__ __forceinline__ TileSlot<L, MT>& my_tile_slot() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return *reinterpret_cast<TileSlot<L, MT>*>(smem_raw +
                                             (threadIdx.x / T) * tile_slot_bytes<L, MT>());
}

template <int NS, bool MT>
__host__ __device__ constexpr size_t slot_bytes() {
  return tile_slot_bytes<32 * NS, MT>();
}

template <int NS, bool MT>
__device__ __forceinline__ TileSlot<32 * NS, MT>& my_slot() {
  return my_tile_slot<32 * NS, MT, 32>();
}

__device__ __forceinline__ int global_warp() {
  return blockIdx.x * kWarps + (threadIdx.x >> 5);
}
__device__ __forceinline__ int total_warps() { return gridDim.x * kWarps; }

// Load an engine state into the tile's slot and bind `rng` to it.
template <int T = 32>
__device__ __forceinline__ void mt_load(uint64_t* s, uint64_t* out, const labs_rng_state& g,
                                        MtRngT<T>& rng) {
  for (int i = tile_lane<T>(); i < kMtN; i += T) s[i] = g.mt[i];
  tile_sync<T>();
  mt_temper_all<T>(s, out);
  rng.bind(s, out, g.idx);
}
template <int T = 32>
__device__ __forceinline__ void mt_store(const uint64_t* s, labs_rng_state& g,
                                         int idx) {
  tile_sync<T>();
  for (int i = tile_lane<T>(); i < kMtN; i += T) g.mt[i] = s[i];
  if (tile_lane<T>() == 0) g.idx = idx;
  tile_sync<T>();
}

// ------------------------------------------------------------------ K1 --
template <int NS>
__global__ void __launch_bounds__(32 * kWarps, min_blocks<NS>())
k_build(int n, int count, const uint64_t* __restrict__ words,
        int32_t* __restrict__ corr, int64_t* __restrict__ energy,
        int64_t* __restrict__ nbr) {
  auto& sl = my_slot<NS, false>();
  smem_clear(sl.walk);
  Walker<NS> w;
  w.sm = &sl.walk;
  const int nw = (n + 63) / 64;
  for (int item = global_warp(); item < count; item += total_warps()) {
    uint32_t in[NS];
    load_chunks<NS>(words + static_cast<size_t>(item) * nw, nw, in);
    w.init(n, in);
    int dE[NS];
    w.delta(dE);
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = 32 * b + lane_id();
      if (j < n && nbr) nbr[static_cast<size_t>(item) * n + j] = w.E + dE[b];
      if (j >= 1 && j < n && corr)
        corr[static_cast<size_t>(item) * (n - 1) + j - 1] = w.CK[b];
    }
    if (lane_id() == 0) energy[item] = w.E;
    __syncwarp();
  }
}

// ----------------------------------------------------------------- K2b --
template <int NS>
__global__ void __launch_bounds__(32 * kWarps, min_blocks<NS>())
k_flip_trace(int n, int count, const uint64_t* __restrict__ words, int flips,
             const int32_t* __restrict__ positions, int64_t* __restrict__ energy,
             int64_t* __restrict__ nbr) {
  auto& sl = my_slot<NS, false>();
  smem_clear(sl.walk);
  Walker<NS> w;
  w.sm = &sl.walk;
  const int nw = (n + 63) / 64;
  for (int item = global_warp(); item < count; item += total_warps()) {
    uint32_t in[NS];
    load_chunks<NS>(words + static_cast<size_t>(item) * nw, nw, in);
    w.init(n, in);
    for (int f = 0; f < flips; ++f) {
      const int pos = positions[static_cast<size_t>(item) * flips + f];
      int dE[NS];
      w.delta(dE);
      const int dEp = at_position<NS>(dE, pos);
      w.apply(pos, dEp, f + 1, 0);
      if (lane_id() == 0) energy[static_cast<size_t>(item) * flips + f] = w.E;
      if (nbr) {
        w.delta(dE);
#pragma unroll
        for (int b = 0; b < NS; ++b) {
          const int j = 32 * b + lane_id();
          if (j < n)
            nbr[(static_cast<size_t>(item) * flips + f) * n + j] = w.E + dE[b];
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K2 --
template <int NS>
__global__ void __launch_bounds__(32 * kWarps, min_blocks<NS>())
k_scan(int n, int count, const uint64_t* __restrict__ words,
       const uint8_t* __restrict__ admissible, labs_rng_state* rng_states,
       int allow_fallback, int tie_rule, int32_t* pos_out, int64_t* e_out,
       int32_t* fb_out, int32_t* ntie_out, uint64_t* tie_out) {
  auto& sl = my_slot<NS, true>();
  smem_clear(sl.walk);
  Walker<NS> w;
  w.sm = &sl.walk;
  const int nw = (n + 63) / 64;
  for (int item = global_warp(); item < count; item += total_warps()) {
    MtRng rng;
    mt_load(sl.mt, sl.out, rng_states[item], rng);
    uint32_t in[NS];
    load_chunks<NS>(words + static_cast<size_t>(item) * nw, nw, in);
    w.init(n, in);
    int dE[NS];
    bool adm[NS];
    w.delta(dE);
    bool any = false;
#pragma unroll
    for (int b = 0; b < NS; ++b) {
      const int j = 32 * b + lane_id();
      adm[b] = j < n && admissible[static_cast<size_t>(item) * n + j] != 0;
      any |= adm[b];
    }
    any = __any_sync(kFull, any);
    int pos = -1, dEp = 0, fb = 0, ntie = 0;
    uint32_t msk[NS];
#pragma unroll
    for (int b = 0; b < NS; ++b) msk[b] = 0u;
    if (any || allow_fallback)
      select_move<NS, 32, true>(dE, adm, n, tie_rule, rng, pos, dEp, fb, msk, ntie);
    if (lane_id() == 0) {
      pos_out[item] = pos;
      e_out[item] = pos >= 0 ? static_cast<int64_t>(w.E) + dEp : 0;
      fb_out[item] = fb;
      ntie_out[item] = ntie;
      if (tie_out) {
#pragma unroll
        for (int wi = 0; wi < LABS_MAX_WORDS; ++wi) {
          uint64_t lo = 2 * wi < NS ? msk[2 * wi] : 0u;
          uint64_t hi = 2 * wi + 1 < NS ? msk[2 * wi + 1] : 0u;
          tie_out[static_cast<size_t>(item) * LABS_MAX_WORDS + wi] = lo | (hi << 32);
        }
      }
    }
    mt_store(sl.mt, rng_states[item], rng.idx);
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K3 --
struct WalkArgs {
  int n, count, walks;
  const uint64_t* start;
  TabuCfg cfg;
  labs_rng_state* mt;
  uint64_t seed, ctr_base;
  uint64_t* best;
  int64_t* bestE;
  int32_t* info;
  StepRec* steps;
  int steps_stride;
  unsigned long long* iters;
};

template <int NS, bool MT>
__global__ void __launch_bounds__(32 * kWarps, min_blocks<NS>()) k_tabu(WalkArgs A) {
  auto& sl = my_slot<NS, MT>();
  smem_clear(sl.walk);
  Walker<NS> w;
  w.sm = &sl.walk;
  const int n = A.n, nw = (n + 63) / 64;
  unsigned long long total = 0;
  for (int item = global_warp(); item < A.count; item += total_warps()) {
    uint32_t cur[NS], best[NS];
    load_chunks<NS>(A.start + static_cast<size_t>(item) * nw, nw, cur);
    int bestE = 0;
    if constexpr (MT) {
      MtRng rng;
      mt_load(sl.mt, sl.out, A.mt[item], rng);
      for (int k = 0; k < A.walks; ++k) {
        int steps = 0;
        bestE = tabu_walk<NS>(w, n, cur, rng, A.cfg, best,
                              A.info ? A.info + 3 * static_cast<size_t>(item) : nullptr,
                              A.steps ? A.steps + static_cast<size_t>(item) * A.steps_stride
                                      : nullptr,
                              &steps);
        total += steps;
#pragma unroll
        for (int b = 0; b < NS; ++b) cur[b] = best[b];
      }
      mt_store(sl.mt, A.mt[item], rng.idx);
    } else {
      PhiloxRng rng;
      rng.k0 = static_cast<uint32_t>(A.seed);
      rng.k1 = static_cast<uint32_t>(A.seed >> 32);
      rng.s0 = static_cast<uint32_t>(item);
      rng.s1 = 0x4C414253u;  // "LABS"
      rng.bind(sl.out, A.ctr_base);
      for (int k = 0; k < A.walks; ++k) {
        int steps = 0;
        bestE = tabu_walk<NS>(w, n, cur, rng, A.cfg, best,
                              A.info ? A.info + 3 * static_cast<size_t>(item) : nullptr,
                              A.steps ? A.steps + static_cast<size_t>(item) * A.steps_stride
                                      : nullptr,
                              &steps);
        total += steps;
#pragma unroll
        for (int b = 0; b < NS; ++b) cur[b] = best[b];
      }
    }
    store_chunks<NS>(A.best + static_cast<size_t>(item) * nw, nw, best);
    if (lane_id() == 0) A.bestE[item] = bestE;
    __syncwarp();
  }
  if (A.iters && lane_id() == 0 && total) atomicAdd(A.iters, total);
}

__global__ void k_seed(int count, uint64_t base, labs_rng_state* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  uint64_t x = base + static_cast<uint64_t>(c);
  out[c].mt[0] = x;
  for (int i = 1; i < kMtN; ++i) {
    x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
    out[c].mt[i] = x;
  }
  out[c].idx = kMtN;
  out[c].pad_ = 0;
}

// ------------------------------------------------------------------ K4 --
// Replica RNG binding for memetic_tiles: mt19937_64 state copied between the
// replica's global record and the tile's shared slot, or the Philox stream
// (key = base seed, stream = global replica id) positioned at its counter.
template <int T>
struct MtBind {
  labs_rng_state* g;
  uint64_t* mt;
  uint64_t* out;
  __device__ __forceinline__ void load(int r, MtRngT<T>& rng) { mt_load<T>(mt, out, g[r], rng); }
  __device__ __forceinline__ void save(int r, MtRngT<T>& rng) { mt_store<T>(mt, g[r], rng.idx); }
};
template <int T>
struct PhiloxBind {
  uint64_t* ctr;
  uint64_t* buf;
  int64_t offset;
  __device__ __forceinline__ void load(int r, PhiloxRngT<T>& rng) {
    rng.s0 = static_cast<uint32_t>(offset + r);
    rng.bind(buf, ctr[r]);
  }
  __device__ __forceinline__ void save(int r, PhiloxRngT<T>& rng) {
    if (tile_lane<T>() == 0) ctr[r] = rng.ctr;
    tile_sync<T>();
  }
};

// Replicas per tile of T lanes; T < 32 packs 32/T replicas into each warp
// (labs_memetic.cuh: memetic_tiles).
template <int NS, int T>
__host__ __device__ constexpr int min_blocks_memetic() {
  return T * NS <= 128 ? LABS_MINB_SMALL : LABS_MINB_LARGE;
}

// The two policy switches (aspiration, tie rule) as template parameters, so
// the tabu step carries no runtime policy tests.
template <int NS, int T, class R, class RB>
__device__ __forceinline__ void run_policy(const MemeticArgs& A, Walker<NS, T>& w, R& rng,
                                           RB& rb, TileCtl& ctl) {
  const bool ref_ties = A.tabu.tie_rule == LABS_TIE_REFERENCE;
  if (A.tabu.aspiration) {
    if (ref_ties) memetic_tiles<NS, T, true, true>(A, w, rng, rb, ctl);
    else memetic_tiles<NS, T, true, false>(A, w, rng, rb, ctl);
  } else {
    if (ref_ties) memetic_tiles<NS, T, false, true>(A, w, rng, rb, ctl);
    else memetic_tiles<NS, T, false, false>(A, w, rng, rb, ctl);
  }
}

template <int NS, int T, bool MT>
__global__ void __launch_bounds__(32 * kWarps, (min_blocks_memetic<NS, T>()))
k_memetic(MemeticArgs A) {
  constexpr int L = T * NS;
  auto& sl = my_tile_slot<L, MT, T>();
  smem_clear<L, T>(sl.walk);
  Walker<NS, T> w;
  w.sm = &sl.walk;
  if constexpr (MT) {
    MtRngT<T> rng;
    rng.bind(sl.mt, sl.out, 0);  // valid until a replica is loaded
    MtBind<T> rb{A.mt, sl.mt, sl.out};
    run_policy<NS, T>(A, w, rng, rb, sl.ctl);
  } else {
    PhiloxRngT<T> rng;
    rng.k0 = static_cast<uint32_t>(A.base_seed);
    rng.k1 = static_cast<uint32_t>(A.base_seed >> 32);
    rng.s0 = 0;
    rng.s1 = 0x4D454D45u;  // "MEME"
    rng.bind(sl.out, 0);  // valid until a replica is loaded
    PhiloxBind<T> rb{A.ctr, sl.out, A.replica_offset};
    run_policy<NS, T>(A, w, rng, rb, sl.ctl);
  }
}


// ---------------------------------------------------- island exchange ----
// Top-k replica bests, best first: k rounds of a block-wide argmin over the
// packed key (E << 32 | replica); taken replicas are masked in `taken`.
__global__ void k_export_elites(int replicas, int nw, int k, const int32_t* bestE,
                                const uint64_t* best, int32_t* taken, uint64_t* out_words,
                                int64_t* out_e) {
  __shared__ unsigned long long red[32];
  for (int i = threadIdx.x; i < replicas; i += blockDim.x) taken[i] = 0;
  __syncthreads();
  for (int sel = 0; sel < k; ++sel) {
    unsigned long long key = ~0ULL;
    for (int i = threadIdx.x; i < replicas; i += blockDim.x)
      if (!taken[i]) {
        const unsigned long long v =
            (static_cast<unsigned long long>(static_cast<uint32_t>(bestE[i])) << 32) | i;
        key = v < key ? v : key;
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long x = __shfl_xor_sync(kFull, key, o);
      key = x < key ? x : key;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned long long v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : ~0ULL;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(kFull, v, o);
        v = x < v ? x : v;
      }
      if (threadIdx.x == 0) {
        const int r = static_cast<int>(v & 0xffffffffULL);
        if (v != ~0ULL) {
          taken[r] = 1;
          out_e[sel] = static_cast<int64_t>(v >> 32);
          for (int w = 0; w < nw; ++w) out_words[static_cast<size_t>(sel) * nw + w] =
              best[static_cast<size_t>(r) * nw + w];
        } else {
          out_e[sel] = INT_MAX;
        }
      }
    }
    __syncthreads();
  }
}

// Replica r offers elite (r + rotation) % count: it replaces the worst
// population member when strictly better. One warp per replica.
__global__ void k_import_elites(int replicas, int nw, int K, int count, int rotation,
                                const uint64_t* words, const int64_t* energies,
                                uint64_t* pop, int32_t* popE, const int32_t* status) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= replicas || status[r] != kRunning) return;
  const int e = (r + rotation) % count;
  const int64_t ee = energies[e];
  int32_t* pe = popE + static_cast<size_t>(r) * K;
  const int victim = worst_member(pe, K);
  if (ee < pe[victim]) {
    if (lane_id() < nw)
      pop[(static_cast<size_t>(r) * K + victim) * nw + lane_id()] =
          words[static_cast<size_t>(e) * nw + lane_id()];
    if (lane_id() == 0) pe[victim] = static_cast<int32_t>(ee);
  }
}


// ------------------------------------------------ INT32 issue-rate probe --
// Roofline denominator for the integer-bound walker: 8 independent chains per
// thread, 4 on the FMA pipe (IMAD) and 4 on the ALU pipe (IADD3/LOP3), so
// both integer pipes issue every cycle. One "op" = one lane-instruction.
__global__ void __launch_bounds__(256) k_int_peak(int iters, int seed, int* sink) {
  int a0 = threadIdx.x ^ seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  int b0 = blockIdx.x ^ seed, b1 = b0 + 5, b2 = b0 + 6, b3 = b0 + 7;
  const int m = seed | 1;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = a0 * m + b3;
      a1 = a1 * m + b2;
      a2 = a2 * m + b1;
      a3 = a3 * m + b0;
      b0 = b0 + a1 + u;
      b1 = b1 ^ a2 ^ u;
      b2 = b2 + a3 + 3;
      b3 = b3 ^ a0 ^ 9;
    }
  }
  const int v = a0 ^ a1 ^ a2 ^ a3 ^ b0 ^ b1 ^ b2 ^ b3;
  if (v == 0x7fffffff) sink[0] = v;  // keep the chains alive
}

}  // namespace labsk

// ====================================================================== ABI
using namespace labsk;

struct labs_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define LABS_CUDA(call)                                                    \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess)                                                 \
      return fail(LABS_ERR_CUDA, std::string(#call) + ": " +               \
                                     cudaGetErrorString(e_));              \
  } while (0)

int check_n(int n) {
  if (n < 2) return fail(LABS_ERR_INVALID_ARGUMENT, "length must be >= 2");
  if (n > LABS_MAX_N)
    return fail(LABS_ERR_INVALID_ARGUMENT,
                "length exceeds the device walker limit " +
                    std::to_string(LABS_MAX_N));
  return LABS_OK;
}

int ns_of(int n) { return (n + 31) / 32; }
int nw_of(int n) { return (n + 63) / 64; }

// RAII device buffer on the context stream.
struct DBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  cudaError_t alloc(size_t bytes, cudaStream_t st) {
    s = st;
    if (bytes == 0) bytes = 16;
    return cudaMallocAsync(&p, bytes, st);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

#define LABS_ALLOC(buf, bytes) LABS_CUDA((buf).alloc((bytes), ctx->stream))
#define LABS_H2D(dst, src, bytes) \
  LABS_CUDA(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyHostToDevice, ctx->stream))
#define LABS_D2H(dst, src, bytes) \
  LABS_CUDA(cudaMemcpyAsync((dst), (src), (bytes), cudaMemcpyDeviceToHost, ctx->stream))

template <class Kern>
int grid_for(labs_ctx* ctx, Kern kern, size_t smem, int items, int* grid,
             int per_block = kWarps) {
  int per_sm = 0;
  LABS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kWarps, smem));
  if (per_sm < 1) per_sm = 1;
  const int want = (items + per_block - 1) / per_block;
  *grid = std::max(1, std::min(want, per_sm * ctx->sm_count));
  return LABS_OK;
}

template <class Kern>
int prep(Kern kern, size_t smem) {
  if (smem > 48 * 1024)
    LABS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  return LABS_OK;
}

// NS dispatch: calls f(std::integral_constant<int, NS>) for NS = ceil(n/32).
template <class F>
int dispatch(int n, F&& f) {
  switch (ns_of(n)) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    case 6: return f(std::integral_constant<int, 6>{});
    case 7: return f(std::integral_constant<int, 7>{});
    case 8: return f(std::integral_constant<int, 8>{});
  }
  return fail(LABS_ERR_INVALID_ARGUMENT, "unsupported length");
}

int check_tabu(const labs_tabu_params* p) {
  if (!p) return fail(LABS_ERR_INVALID_ARGUMENT, "null tabu params");
  if (p->min_tabu_factor < 0 || p->max_tabu_factor < p->min_tabu_factor ||
      p->max_tabu_factor >= 1)
    return fail(LABS_ERR_INVALID_ARGUMENT,
                "tabu tenure factors need 0 <= min <= max < 1");
  if (p->tie_rule != LABS_TIE_REFERENCE && p->tie_rule != LABS_TIE_LOWEST)
    return fail(LABS_ERR_INVALID_ARGUMENT, "unknown tie rule");
  return LABS_OK;
}

TabuCfg to_cfg(const labs_tabu_params* p) {
  TabuCfg c;
  c.min_factor = p->min_tabu_factor;
  c.max_factor = p->max_tabu_factor;
  c.tie_rule = p->tie_rule;
  c.aspiration = p->aspiration ? 1 : 0;
  return c;
}

int check_seq_padding(int n, int count, const uint64_t* words) {
  const int nw = nw_of(n);
  const int rem = n & 63;
  if (!rem) return LABS_OK;
  const uint64_t bad = ~((1ULL << rem) - 1ULL);
  for (int c = 0; c < count; ++c)
    if (words[static_cast<size_t>(c) * nw + nw - 1] & bad)
      return fail(LABS_ERR_INVALID_ARGUMENT, "nonzero padding bits in sequence words");
  return LABS_OK;
}

}  // namespace

extern "C" {

const char* labs_last_error(void) { return g_err.c_str(); }

int labs_max_n(void) { return LABS_MAX_N; }

int labs_ctx_create(int device, labs_ctx** out) {
  if (!out) return fail(LABS_ERR_INVALID_ARGUMENT, "null output");
  int ndev = 0;
  LABS_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev)
    return fail(LABS_ERR_INVALID_ARGUMENT, "no such CUDA device");
  LABS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  LABS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(LABS_ERR_CUDA, std::string("built for sm_100a; device is ") + prop.name);
  auto* c = new labs_ctx;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(LABS_ERR_CUDA, cudaGetErrorString(e));
  }
  *out = c;
  return LABS_OK;
}

int labs_ctx_destroy(labs_ctx* ctx) {
  if (!ctx) return LABS_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return LABS_OK;
}

void* labs_ctx_stream(labs_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
int labs_ctx_sm_count(labs_ctx* ctx) { return ctx ? ctx->sm_count : 0; }

int labs_ctx_synchronize(labs_ctx* ctx) {
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  LABS_CUDA(cudaGetLastError());
  return LABS_OK;
}

void labs_rng_seed(uint64_t seed, labs_rng_state* out) {
  uint64_t x = seed;
  out->mt[0] = x;
  for (int i = 1; i < kMtN; ++i) {
    x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
    out->mt[i] = x;
  }
  out->idx = kMtN;
  out->pad_ = 0;
}

int labs_build_state(labs_ctx* ctx, int n, int count, const uint64_t* words,
                     int32_t* corr_out, int64_t* energy_out, int64_t* neighbor_out) {
  if (int rc = check_n(n)) return rc;
  if (!ctx || count < 0 || (count && (!words || !energy_out)))
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (count == 0) return LABS_OK;
  if (int rc = check_seq_padding(n, count, words)) return rc;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int nw = nw_of(n);
  DBuf dw, dc, de, dn;
  LABS_ALLOC(dw, sizeof(uint64_t) * count * nw);
  LABS_ALLOC(dc, sizeof(int32_t) * count * (n - 1));
  LABS_ALLOC(de, sizeof(int64_t) * count);
  if (neighbor_out) LABS_ALLOC(dn, sizeof(int64_t) * count * n);
  LABS_H2D(dw.p, words, sizeof(uint64_t) * count * nw);
  int rc = dispatch(n, [&](auto ns) -> int {
    constexpr int NS = decltype(ns)::value;
    const size_t smem = kWarps * slot_bytes<NS, false>();
    auto kern = k_build<NS>;
    if (int r = prep(kern, smem)) return r;
    int grid = 0;
    if (int r = grid_for(ctx, kern, smem, count, &grid)) return r;
    kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(n, count, dw.as<uint64_t>(),
                                                   dc.as<int32_t>(), de.as<int64_t>(),
                                                   neighbor_out ? dn.as<int64_t>() : nullptr);
    LABS_CUDA(cudaGetLastError());
    return LABS_OK;
  });
  if (rc) return rc;
  if (corr_out) LABS_D2H(corr_out, dc.p, sizeof(int32_t) * count * (n - 1));
  LABS_D2H(energy_out, de.p, sizeof(int64_t) * count);
  if (neighbor_out) LABS_D2H(neighbor_out, dn.p, sizeof(int64_t) * count * n);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

int labs_flip_trace(labs_ctx* ctx, int n, int count, const uint64_t* words, int flips,
                    const int32_t* positions, int64_t* energy_out, int64_t* neighbor_out) {
  if (int rc = check_n(n)) return rc;
  if (!ctx || count < 0 || flips < 0 || (count && flips && (!words || !positions || !energy_out)))
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (count == 0 || flips == 0) return LABS_OK;
  if (int rc = check_seq_padding(n, count, words)) return rc;
  for (size_t i = 0; i < static_cast<size_t>(count) * flips; ++i)
    if (positions[i] < 0 || positions[i] >= n)
      return fail(LABS_ERR_OUT_OF_RANGE, "flip position");
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int nw = nw_of(n);
  DBuf dw, dp, de, dn;
  LABS_ALLOC(dw, sizeof(uint64_t) * count * nw);
  LABS_ALLOC(dp, sizeof(int32_t) * count * flips);
  LABS_ALLOC(de, sizeof(int64_t) * count * flips);
  if (neighbor_out) LABS_ALLOC(dn, sizeof(int64_t) * count * flips * n);
  LABS_H2D(dw.p, words, sizeof(uint64_t) * count * nw);
  LABS_H2D(dp.p, positions, sizeof(int32_t) * count * flips);
  int rc = dispatch(n, [&](auto ns) -> int {
    constexpr int NS = decltype(ns)::value;
    const size_t smem = kWarps * slot_bytes<NS, false>();
    auto kern = k_flip_trace<NS>;
    if (int r = prep(kern, smem)) return r;
    int grid = 0;
    if (int r = grid_for(ctx, kern, smem, count, &grid)) return r;
    kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(
        n, count, dw.as<uint64_t>(), flips, dp.as<int32_t>(), de.as<int64_t>(),
        neighbor_out ? dn.as<int64_t>() : nullptr);
    LABS_CUDA(cudaGetLastError());
    return LABS_OK;
  });
  if (rc) return rc;
  LABS_D2H(energy_out, de.p, sizeof(int64_t) * count * flips);
  if (neighbor_out) LABS_D2H(neighbor_out, dn.p, sizeof(int64_t) * count * flips * n);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

int labs_scan(labs_ctx* ctx, int n, int count, const uint64_t* words,
              const uint8_t* admissible, labs_rng_state* rng, int allow_fallback,
              int tie_rule, int32_t* position, int64_t* energy, int32_t* fallback,
              int32_t* ntie, uint64_t* tie_mask) {
  if (int rc = check_n(n)) return rc;
  if (!ctx || count < 0 ||
      (count && (!words || !admissible || !rng || !position || !energy || !fallback || !ntie)))
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (tie_rule != LABS_TIE_REFERENCE && tie_rule != LABS_TIE_LOWEST)
    return fail(LABS_ERR_INVALID_ARGUMENT, "unknown tie rule");
  if (count == 0) return LABS_OK;
  if (int rc = check_seq_padding(n, count, words)) return rc;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int nw = nw_of(n);
  DBuf dw, da, dr, dpos, de, dfb, dnt, dtm;
  LABS_ALLOC(dw, sizeof(uint64_t) * count * nw);
  LABS_ALLOC(da, static_cast<size_t>(count) * n);
  LABS_ALLOC(dr, sizeof(labs_rng_state) * count);
  LABS_ALLOC(dpos, sizeof(int32_t) * count);
  LABS_ALLOC(de, sizeof(int64_t) * count);
  LABS_ALLOC(dfb, sizeof(int32_t) * count);
  LABS_ALLOC(dnt, sizeof(int32_t) * count);
  LABS_ALLOC(dtm, sizeof(uint64_t) * count * LABS_MAX_WORDS);
  LABS_H2D(dw.p, words, sizeof(uint64_t) * count * nw);
  LABS_H2D(da.p, admissible, static_cast<size_t>(count) * n);
  LABS_H2D(dr.p, rng, sizeof(labs_rng_state) * count);
  int rc = dispatch(n, [&](auto ns) -> int {
    constexpr int NS = decltype(ns)::value;
    const size_t smem = kWarps * slot_bytes<NS, true>();
    auto kern = k_scan<NS>;
    if (int r = prep(kern, smem)) return r;
    int grid = 0;
    if (int r = grid_for(ctx, kern, smem, count, &grid)) return r;
    kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(
        n, count, dw.as<uint64_t>(), da.as<uint8_t>(), dr.as<labs_rng_state>(),
        allow_fallback, tie_rule, dpos.as<int32_t>(), de.as<int64_t>(), dfb.as<int32_t>(),
        dnt.as<int32_t>(), dtm.as<uint64_t>());
    LABS_CUDA(cudaGetLastError());
    return LABS_OK;
  });
  if (rc) return rc;
  LABS_D2H(position, dpos.p, sizeof(int32_t) * count);
  LABS_D2H(energy, de.p, sizeof(int64_t) * count);
  LABS_D2H(fallback, dfb.p, sizeof(int32_t) * count);
  LABS_D2H(ntie, dnt.p, sizeof(int32_t) * count);
  LABS_D2H(rng, dr.p, sizeof(labs_rng_state) * count);
  if (tie_mask) LABS_D2H(tie_mask, dtm.p, sizeof(uint64_t) * count * LABS_MAX_WORDS);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < count; ++i)
    if (position[i] < 0)
      return fail(LABS_ERR_RUNTIME, "no admissible position in neighborhood scan");
  return LABS_OK;
}

static int launch_tabu(labs_ctx* ctx, int n, WalkArgs& A, bool mt) {
  return dispatch(n, [&](auto ns) -> int {
    constexpr int NS = decltype(ns)::value;
    if (mt) {
      const size_t smem = kWarps * slot_bytes<NS, true>();
      auto kern = k_tabu<NS, true>;
      if (int r = prep(kern, smem)) return r;
      int grid = 0;
      if (int r = grid_for(ctx, kern, smem, A.count, &grid)) return r;
      kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(A);
    } else {
      const size_t smem = kWarps * slot_bytes<NS, false>();
      auto kern = k_tabu<NS, false>;
      if (int r = prep(kern, smem)) return r;
      int grid = 0;
      if (int r = grid_for(ctx, kern, smem, A.count, &grid)) return r;
      kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(A);
    }
    LABS_CUDA(cudaGetLastError());
    return LABS_OK;
  });
}

int labs_tabu_walks(labs_ctx* ctx, int n, int count, const uint64_t* start,
                    const labs_tabu_params* params, labs_rng_state* rng, uint64_t* best_out,
                    int64_t* best_energy, int32_t* info, labs_tabu_step* steps) {
  if (int rc = check_n(n)) return rc;
  if (int rc = check_tabu(params)) return rc;
  if (!ctx || count < 0 || (count && (!start || !rng || !best_out || !best_energy)))
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (count == 0) return LABS_OK;
  if (int rc = check_seq_padding(n, count, start)) return rc;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int nw = nw_of(n);
  const int stride = n + n / 2 + 1;
  DBuf ds, dr, db, de, di, dst;
  LABS_ALLOC(ds, sizeof(uint64_t) * count * nw);
  LABS_ALLOC(dr, sizeof(labs_rng_state) * count);
  LABS_ALLOC(db, sizeof(uint64_t) * count * nw);
  LABS_ALLOC(de, sizeof(int64_t) * count);
  if (info) LABS_ALLOC(di, sizeof(int32_t) * 3 * count);
  if (steps) LABS_ALLOC(dst, sizeof(labs_tabu_step) * count * stride);
  LABS_H2D(ds.p, start, sizeof(uint64_t) * count * nw);
  LABS_H2D(dr.p, rng, sizeof(labs_rng_state) * count);
  WalkArgs A{};
  A.n = n;
  A.count = count;
  A.walks = 1;
  A.start = ds.as<uint64_t>();
  A.cfg = to_cfg(params);
  A.mt = dr.as<labs_rng_state>();
  A.best = db.as<uint64_t>();
  A.bestE = de.as<int64_t>();
  A.info = info ? di.as<int32_t>() : nullptr;
  A.steps = steps ? dst.as<StepRec>() : nullptr;
  A.steps_stride = stride;
  A.iters = nullptr;
  if (int rc = launch_tabu(ctx, n, A, true)) return rc;
  LABS_D2H(best_out, db.p, sizeof(uint64_t) * count * nw);
  LABS_D2H(best_energy, de.p, sizeof(int64_t) * count);
  LABS_D2H(rng, dr.p, sizeof(labs_rng_state) * count);
  if (info) LABS_D2H(info, di.p, sizeof(int32_t) * 3 * count);
  if (steps) LABS_D2H(steps, dst.p, sizeof(labs_tabu_step) * count * stride);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

int labs_tabu_walks_device(labs_ctx* ctx, int n, int count, int walks_per_walker,
                           const uint64_t* d_start, const labs_tabu_params* params,
                           int rng_kind, labs_rng_state* d_rng, uint64_t seed,
                           uint64_t ctr_base, uint64_t* d_best, int64_t* d_best_energy,
                           unsigned long long* d_iterations) {
  if (int rc = check_n(n)) return rc;
  if (int rc = check_tabu(params)) return rc;
  if (!ctx || count < 0 || walks_per_walker < 1 || (count && (!d_start || !d_best || !d_best_energy)))
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (rng_kind != LABS_RNG_MT19937_64 && rng_kind != LABS_RNG_PHILOX)
    return fail(LABS_ERR_INVALID_ARGUMENT, "unknown rng kind");
  if (rng_kind == LABS_RNG_MT19937_64 && !d_rng)
    return fail(LABS_ERR_INVALID_ARGUMENT, "mt19937_64 mode needs engine states");
  if (count == 0) return LABS_OK;
  LABS_CUDA(cudaSetDevice(ctx->device));
  WalkArgs A{};
  A.n = n;
  A.count = count;
  A.walks = walks_per_walker;
  A.start = d_start;
  A.cfg = to_cfg(params);
  A.mt = d_rng;
  A.seed = seed;
  A.ctr_base = ctr_base;
  A.best = d_best;
  A.bestE = d_best_energy;
  A.info = nullptr;
  A.steps = nullptr;
  A.iters = d_iterations;
  return launch_tabu(ctx, n, A, rng_kind == LABS_RNG_MT19937_64);
}

int labs_rng_seed_device(labs_ctx* ctx, int count, uint64_t base_seed, labs_rng_state* d_rng) {
  if (!ctx || count < 0 || (count && !d_rng))
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (count == 0) return LABS_OK;
  LABS_CUDA(cudaSetDevice(ctx->device));
  k_seed<<<(count + 127) / 128, 128, 0, ctx->stream>>>(count, base_seed, d_rng);
  LABS_CUDA(cudaGetLastError());
  return LABS_OK;
}

}  // extern "C"


// ------------------------------------------------------- memetic (K4) ----
namespace {

int check_memetic(int n, const labs_memetic_params* p) {
  if (int rc = check_n(n)) return rc;
  if (!p) return fail(LABS_ERR_INVALID_ARGUMENT, "null params");
  if (p->population_size < 2) return fail(LABS_ERR_INVALID_ARGUMENT, "population must be >= 2");
  if (p->p_comb < 0.0 || p->p_comb > 1.0)
    return fail(LABS_ERR_INVALID_ARGUMENT, "p_comb must be in [0, 1]");
  const double pm = p->p_mutate > 0.0 ? p->p_mutate : 1.0 / n;
  if (!(pm > 0.0) || pm > 1.0)
    return fail(LABS_ERR_INVALID_ARGUMENT, "mutation probability must be in (0, 1]");
  if (p->rng_kind != LABS_RNG_MT19937_64 && p->rng_kind != LABS_RNG_PHILOX)
    return fail(LABS_ERR_INVALID_ARGUMENT, "unknown rng kind");
  if (p->crossover != LABS_CROSSOVER_UNIFORM && p->crossover != LABS_CROSSOVER_ONE_POINT)
    return fail(LABS_ERR_INVALID_ARGUMENT, "unknown crossover");
  if (p->replacement != LABS_REPLACE_RANDOM && p->replacement != LABS_REPLACE_WORST)
    return fail(LABS_ERR_INVALID_ARGUMENT, "unknown replacement policy");
  return check_tabu(&p->tabu);
}

// Memetic kernel shape: one replica per warp (T = 32) by default;
// LABS_TILE=16 in the environment packs two replicas of n <= 64 into each
// warp (16-lane tiles, 2 or 4 slots per lane). Measured on B200 at n = 64:
// the 16-lane form issues ~10% fewer instructions per walker-step but loses
// more to bank conflicts between the two tiles' slots and to L0 I-cache
// misses (optimization log), so it is an option, not the default.
bool memetic_tiled(int n) {
  const char* e = std::getenv("LABS_TILE");
  return n <= 64 && e && std::atoi(e) == 16;
}

template <class F>
int dispatch_memetic(int n, F&& f) {
  if (memetic_tiled(n)) {
    if (n <= 32) return f(std::integral_constant<int, 2>{}, std::integral_constant<int, 16>{});
    return f(std::integral_constant<int, 4>{}, std::integral_constant<int, 16>{});
  }
  return dispatch(n, [&](auto ns) -> int { return f(ns, std::integral_constant<int, 32>{}); });
}

template <int NS, int T, bool MT>
constexpr size_t memetic_smem() {
  return (32 / T) * kWarps * tile_slot_bytes<T * NS, MT>();
}

template <int NS, int T, bool MT>
int launch_memetic(labs_ctx* ctx, const MemeticArgs& A) {
  const size_t smem = memetic_smem<NS, T, MT>();
  auto kern = k_memetic<NS, T, MT>;
  if (int r = prep(kern, smem)) return r;
  int grid = 0;
  if (int r = grid_for(ctx, kern, smem, A.replicas, &grid, kWarps * (32 / T))) return r;
  kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(A);
  LABS_CUDA(cudaGetLastError());
  return LABS_OK;
}

}  // namespace

// Device-resident replica set (include/labs_b200.h: labs_solver_*).
struct labs_solver {
  labs_ctx* ctx = nullptr;
  int n = 0, nw = 0, R = 0, K = 0;
  uint64_t base_seed = 0;
  int64_t offset = 0;
  labs_memetic_params p{};
  bool mt = true;
  int64_t trace_cap = 0;
  DBuf pop, popE, best, bestE, iters, status, init, t0, tend, order, counter, rng, ctr, stop,
      tabu_total, tabu_rep, trace, trace_len, taken;
  MemeticArgs A{};
};

extern "C" {

int labs_solver_capacity(labs_ctx* ctx, int n, int rng_kind) {
  if (!ctx || check_n(n)) return 0;
  int out = 0;
  cudaSetDevice(ctx->device);
  dispatch_memetic(n, [&](auto ns, auto tt) -> int {
    constexpr int NS = decltype(ns)::value, T = decltype(tt)::value;
    int per_sm = 0;
    if (rng_kind == LABS_RNG_MT19937_64) {
      if (prep(k_memetic<NS, T, true>, memetic_smem<NS, T, true>())) return LABS_OK;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_memetic<NS, T, true>, 32 * kWarps,
                                                    memetic_smem<NS, T, true>());
    } else {
      if (prep(k_memetic<NS, T, false>, memetic_smem<NS, T, false>())) return LABS_OK;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_memetic<NS, T, false>, 32 * kWarps,
                                                    memetic_smem<NS, T, false>());
    }
    out = per_sm * ctx->sm_count * kWarps * (32 / T);
    return LABS_OK;
  });
  return out;
}

int labs_solver_create(labs_ctx* ctx, int n, int replicas, uint64_t base_seed,
                       int64_t replica_offset, const labs_memetic_params* params,
                       int64_t trace_cap, labs_solver** out) {
  if (!ctx || !out) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (replicas < 1) return fail(LABS_ERR_INVALID_ARGUMENT, "replicas must be >= 1");
  if (int rc = check_memetic(n, params)) return rc;
  if (trace_cap < 0 || replica_offset < 0)
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad trace capacity or replica offset");
  LABS_CUDA(cudaSetDevice(ctx->device));
  auto* s = new labs_solver;
  std::unique_ptr<labs_solver> guard(s);
  s->ctx = ctx;
  s->n = n;
  s->nw = nw_of(n);
  s->R = replicas;
  s->K = params->population_size;
  s->base_seed = base_seed;
  s->offset = replica_offset;
  s->p = *params;
  s->mt = params->rng_kind == LABS_RNG_MT19937_64;
  s->trace_cap = trace_cap;
  const size_t R = replicas, K = s->K, nw = s->nw;
  LABS_ALLOC(s->pop, sizeof(uint64_t) * R * K * nw);
  LABS_ALLOC(s->popE, sizeof(int32_t) * R * K);
  LABS_ALLOC(s->best, sizeof(uint64_t) * R * nw);
  LABS_ALLOC(s->bestE, sizeof(int32_t) * R);
  LABS_ALLOC(s->iters, sizeof(int64_t) * R);
  LABS_ALLOC(s->status, sizeof(int32_t) * R);
  LABS_ALLOC(s->init, sizeof(int32_t) * R);
  LABS_ALLOC(s->t0, sizeof(int64_t) * R);
  LABS_ALLOC(s->tend, sizeof(int64_t) * R);
  LABS_ALLOC(s->order, sizeof(int32_t) * R);
  LABS_ALLOC(s->counter, sizeof(int32_t));
  LABS_ALLOC(s->stop, sizeof(int32_t));
  LABS_ALLOC(s->tabu_total, sizeof(unsigned long long));
  LABS_ALLOC(s->tabu_rep, sizeof(int64_t) * R);
  LABS_ALLOC(s->taken, sizeof(int32_t) * R);
  if (s->mt) LABS_ALLOC(s->rng, sizeof(labs_rng_state) * R);
  else LABS_ALLOC(s->ctr, sizeof(uint64_t) * R);
  if (trace_cap) {
    LABS_ALLOC(s->trace, sizeof(int64_t) * 3 * R * trace_cap);
    LABS_ALLOC(s->trace_len, sizeof(int64_t) * R);
  }
  cudaStream_t st = ctx->stream;
  LABS_CUDA(cudaMemsetAsync(s->init.p, 0, sizeof(int32_t) * R, st));
  LABS_CUDA(cudaMemsetAsync(s->status.p, 0, sizeof(int32_t) * R, st));
  LABS_CUDA(cudaMemsetAsync(s->iters.p, 0, sizeof(int64_t) * R, st));
  LABS_CUDA(cudaMemsetAsync(s->counter.p, 0, sizeof(int32_t), st));
  LABS_CUDA(cudaMemsetAsync(s->stop.p, 0, sizeof(int32_t), st));
  LABS_CUDA(cudaMemsetAsync(s->tabu_total.p, 0, sizeof(unsigned long long), st));
  LABS_CUDA(cudaMemsetAsync(s->tabu_rep.p, 0, sizeof(int64_t) * R, st));
  LABS_CUDA(cudaMemsetAsync(s->order.p, 0xff, sizeof(int32_t) * R, st));
  if (trace_cap) LABS_CUDA(cudaMemsetAsync(s->trace_len.p, 0, sizeof(int64_t) * R, st));
  if (s->mt) {
    k_seed<<<(replicas + 127) / 128, 128, 0, st>>>(
        replicas, base_seed + static_cast<uint64_t>(replica_offset), s->rng.as<labs_rng_state>());
    LABS_CUDA(cudaGetLastError());
  } else {
    LABS_CUDA(cudaMemsetAsync(s->ctr.p, 0, sizeof(uint64_t) * R, st));
  }
  MemeticArgs& A = s->A;
  A.n = n;
  A.nw = s->nw;
  A.replicas = replicas;
  A.K = s->K;
  A.p_comb = params->p_comb;
  A.p_mutate = params->p_mutate > 0.0 ? params->p_mutate : 1.0 / n;
  A.target = params->target_energy;
  A.max_ns = params->max_seconds >= 0 ? static_cast<int64_t>(params->max_seconds * 1e9) : -1;
  A.max_iterations = params->max_iterations;
  A.epoch_iters = -1;
  A.epoch_ns = -1;
  A.crossover = params->crossover;
  A.replacement = params->replacement;
  A.tabu = to_cfg(&params->tabu);
  A.race = 1;
  A.base_seed = base_seed;
  A.replica_offset = replica_offset;
  A.pop = s->pop.as<uint64_t>();
  A.popE = s->popE.as<int32_t>();
  A.best = s->best.as<uint64_t>();
  A.bestE = s->bestE.as<int32_t>();
  A.iters = s->iters.as<int64_t>();
  A.status = s->status.as<int32_t>();
  A.initialized = s->init.as<int32_t>();
  A.t0 = s->t0.as<int64_t>();
  A.t_end = s->tend.as<int64_t>();
  A.pub_order = s->order.as<int32_t>();
  A.pub_counter = s->counter.as<int32_t>();
  A.mt = s->mt ? s->rng.as<labs_rng_state>() : nullptr;
  A.ctr = s->mt ? nullptr : s->ctr.as<uint64_t>();
  A.stop = s->stop.as<int32_t>();
  A.tabu_iters = s->tabu_total.as<unsigned long long>();
  A.tabu_per_replica = s->tabu_rep.as<int64_t>();
  A.trace = trace_cap ? s->trace.as<int64_t>() : nullptr;
  A.trace_cap = trace_cap;
  A.trace_len = trace_cap ? s->trace_len.as<int64_t>() : nullptr;
  *out = guard.release();
  return LABS_OK;
}

int labs_solver_destroy(labs_solver* s) {
  if (!s) return LABS_OK;
  cudaSetDevice(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  delete s;
  return LABS_OK;
}

int labs_solver_run(labs_solver* s, int64_t epoch_iterations, double epoch_seconds, int race) {
  if (!s) return fail(LABS_ERR_INVALID_ARGUMENT, "null solver");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  MemeticArgs A = s->A;
  A.epoch_iters = epoch_iterations;
  A.epoch_ns = epoch_seconds >= 0 ? static_cast<int64_t>(epoch_seconds * 1e9) : -1;
  A.race = race ? 1 : 0;
  return dispatch_memetic(s->n, [&](auto ns, auto tt) -> int {
    constexpr int NS = decltype(ns)::value, T = decltype(tt)::value;
    return s->mt ? launch_memetic<NS, T, true>(ctx, A) : launch_memetic<NS, T, false>(ctx, A);
  });
}

int labs_solver_request_stop(labs_solver* s) {
  if (!s) return fail(LABS_ERR_INVALID_ARGUMENT, "null solver");
  labs_ctx* ctx = s->ctx;
  static const int32_t one = 1;
  LABS_CUDA(cudaSetDevice(ctx->device));
  LABS_H2D(s->stop.p, &one, sizeof(int32_t));
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

int labs_solver_status(labs_solver* s, int32_t* running, int64_t* best_energy,
                       int32_t* best_replica) {
  if (!s) return fail(LABS_ERR_INVALID_ARGUMENT, "null solver");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  std::vector<int32_t> st(s->R), be(s->R), init(s->R);
  LABS_D2H(st.data(), s->status.p, sizeof(int32_t) * s->R);
  LABS_D2H(be.data(), s->bestE.p, sizeof(int32_t) * s->R);
  LABS_D2H(init.data(), s->init.p, sizeof(int32_t) * s->R);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  LABS_CUDA(cudaGetLastError());
  int run = 0, arg = -1;
  for (int r = 0; r < s->R; ++r) {
    run += (!init[r] || st[r] == kRunning) ? 1 : 0;
    if (init[r] && (arg < 0 || be[r] < be[arg])) arg = r;
  }
  if (running) *running = run;
  if (best_energy) *best_energy = arg >= 0 ? be[arg] : -1;
  if (best_replica) *best_replica = arg >= 0 ? static_cast<int32_t>(arg + s->offset) : -1;
  return LABS_OK;
}

int labs_solver_counters(labs_solver* s, uint64_t* tabu_iterations, int64_t* memetic_iterations) {
  if (!s) return fail(LABS_ERR_INVALID_ARGUMENT, "null solver");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  unsigned long long t = 0;
  std::vector<int64_t> it(s->R);
  LABS_D2H(&t, s->tabu_total.p, sizeof(t));
  LABS_D2H(it.data(), s->iters.p, sizeof(int64_t) * s->R);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (tabu_iterations) *tabu_iterations = t;
  if (memetic_iterations) {
    int64_t sum = 0;
    for (int64_t v : it) sum += v;
    *memetic_iterations = sum;
  }
  return LABS_OK;
}

int labs_solver_results(labs_solver* s, labs_run_result* per_replica, labs_memetic_record* traces,
                        int64_t* trace_len, int32_t* publish_order) {
  if (!s || !per_replica) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int R = s->R, nw = s->nw;
  std::vector<uint64_t> best(static_cast<size_t>(R) * nw);
  std::vector<int32_t> bestE(R), order(R), status(R);
  std::vector<int64_t> iters(R), t0(R), tend(R), tabu(R);
  LABS_D2H(best.data(), s->best.p, sizeof(uint64_t) * R * nw);
  LABS_D2H(bestE.data(), s->bestE.p, sizeof(int32_t) * R);
  LABS_D2H(iters.data(), s->iters.p, sizeof(int64_t) * R);
  LABS_D2H(t0.data(), s->t0.p, sizeof(int64_t) * R);
  LABS_D2H(tend.data(), s->tend.p, sizeof(int64_t) * R);
  LABS_D2H(order.data(), s->order.p, sizeof(int32_t) * R);
  LABS_D2H(status.data(), s->status.p, sizeof(int32_t) * R);
  LABS_D2H(tabu.data(), s->tabu_rep.p, sizeof(int64_t) * R);
  std::vector<int64_t> tr, tl;
  if (traces && s->trace_cap) {
    tr.resize(static_cast<size_t>(3) * R * s->trace_cap);
    tl.resize(R);
    LABS_D2H(tr.data(), s->trace.p, sizeof(int64_t) * tr.size());
    LABS_D2H(tl.data(), s->trace_len.p, sizeof(int64_t) * R);
  }
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  LABS_CUDA(cudaGetLastError());
  for (int r = 0; r < R; ++r) {
    labs_run_result& o = per_replica[r];
    std::memset(&o, 0, sizeof(o));
    for (int wi = 0; wi < nw; ++wi) o.best[wi] = best[static_cast<size_t>(r) * nw + wi];
    o.best_energy = bestE[r];
    o.merit = static_cast<double>(s->n) * s->n / (2.0 * static_cast<double>(bestE[r]));
    o.iterations = iters[r];
    o.wall_seconds = status[r] != kRunning ? 1e-9 * static_cast<double>(tend[r] - t0[r]) : 0.0;
    o.seed = s->base_seed + static_cast<uint64_t>(s->offset + r);
    o.replica_id = static_cast<int32_t>(s->offset + r);
    o.reached_target = bestE[r] <= s->p.target_energy;
    o.tabu_iterations = tabu[r];
    if (traces && s->trace_cap) {
      const int64_t len = std::min(tl[r], s->trace_cap);
      if (trace_len) trace_len[r] = len;
      for (int64_t i = 0; i < len; ++i) {
        const int64_t* rec = &tr[(static_cast<size_t>(r) * s->trace_cap + i) * 3];
        labs_memetic_record& d = traces[static_cast<size_t>(r) * s->trace_cap + i];
        d.iteration = rec[0];
        d.stop_seen = static_cast<int32_t>(rec[1]);
        d.pad_ = 0;
        d.child_energy = rec[2];
      }
    }
  }
  if (publish_order) std::memcpy(publish_order, order.data(), sizeof(int32_t) * R);
  return LABS_OK;
}

int labs_solver_export_elites(labs_solver* s, int k, uint64_t* d_words, int64_t* d_energies) {
  if (!s || k < 1 || !d_words || !d_energies)
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (k > s->R) return fail(LABS_ERR_INVALID_ARGUMENT, "k exceeds the replica count");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  k_export_elites<<<1, 1024, 0, ctx->stream>>>(s->R, s->nw, k, s->bestE.as<int32_t>(),
                                                s->best.as<uint64_t>(), s->taken.as<int32_t>(),
                                                d_words, d_energies);
  LABS_CUDA(cudaGetLastError());
  return LABS_OK;
}

int labs_solver_import_elites(labs_solver* s, int count, const uint64_t* d_words,
                              const int64_t* d_energies, int rotation) {
  if (!s || count < 1 || !d_words || !d_energies || rotation < 0)
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int wpb = 8;
  k_import_elites<<<(s->R + wpb - 1) / wpb, 32 * wpb, 0, ctx->stream>>>(
      s->R, s->nw, s->K, count, rotation, d_words, d_energies, s->pop.as<uint64_t>(),
      s->popE.as<int32_t>(), s->status.as<int32_t>());
  LABS_CUDA(cudaGetLastError());
  return LABS_OK;
}

int labs_solver_population(labs_solver* s, uint64_t* words, int32_t* energies) {
  if (!s || !words || !energies) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const size_t R = s->R, K = s->K, nw = s->nw;
  LABS_D2H(words, s->pop.p, sizeof(uint64_t) * R * K * nw);
  LABS_D2H(energies, s->popE.p, sizeof(int32_t) * R * K);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

}  // extern "C"

namespace {

struct BlobHeader {
  uint64_t magic;  // "LABSCKP1"
  int32_t n, R, K, nw, rng_kind, crossover, replacement, pad_;
  int64_t trace_cap;
};
constexpr uint64_t kBlobMagic = 0x31504B4353424C4CULL;

// (device buffer, bytes) in blob order.
std::vector<std::pair<void*, size_t>> state_parts(labs_solver* s) {
  const size_t R = s->R, K = s->K, nw = s->nw;
  std::vector<std::pair<void*, size_t>> v = {
      {s->pop.p, sizeof(uint64_t) * R * K * nw}, {s->popE.p, sizeof(int32_t) * R * K},
      {s->best.p, sizeof(uint64_t) * R * nw},    {s->bestE.p, sizeof(int32_t) * R},
      {s->iters.p, sizeof(int64_t) * R},         {s->status.p, sizeof(int32_t) * R},
      {s->init.p, sizeof(int32_t) * R},          {s->tend.p, sizeof(int64_t) * R},
      {s->order.p, sizeof(int32_t) * R},         {s->counter.p, sizeof(int32_t)},
      {s->stop.p, sizeof(int32_t)},              {s->tabu_total.p, sizeof(unsigned long long)},
      {s->tabu_rep.p, sizeof(int64_t) * R}};
  if (s->mt) v.push_back({s->rng.p, sizeof(labs_rng_state) * R});
  else v.push_back({s->ctr.p, sizeof(uint64_t) * R});
  if (s->trace_cap) {
    v.push_back({s->trace.p, sizeof(int64_t) * 3 * R * s->trace_cap});
    v.push_back({s->trace_len.p, sizeof(int64_t) * R});
  }
  return v;
}

BlobHeader header_of(labs_solver* s) {
  BlobHeader h{};
  h.magic = kBlobMagic;
  h.n = s->n;
  h.R = s->R;
  h.K = s->K;
  h.nw = s->nw;
  h.rng_kind = s->p.rng_kind;
  h.crossover = s->p.crossover;
  h.replacement = s->p.replacement;
  h.trace_cap = s->trace_cap;
  return h;
}

__global__ void k_restamp(int R, int64_t* t0) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) t0[r] = globaltimer_ns();
}

}  // namespace

extern "C" {

int64_t labs_solver_state_size(labs_solver* s) {
  if (!s) return -1;
  int64_t total = sizeof(BlobHeader);
  for (auto& part : state_parts(s)) total += static_cast<int64_t>(part.second);
  return total;
}

int labs_solver_save(labs_solver* s, void* blob) {
  if (!s || !blob) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  unsigned char* out = static_cast<unsigned char*>(blob);
  const BlobHeader h = header_of(s);
  std::memcpy(out, &h, sizeof h);
  size_t off = sizeof h;
  for (auto& part : state_parts(s)) {
    LABS_D2H(out + off, part.first, part.second);
    off += part.second;
  }
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

int labs_solver_load(labs_solver* s, const void* blob) {
  if (!s || !blob) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const unsigned char* in = static_cast<const unsigned char*>(blob);
  BlobHeader h;
  std::memcpy(&h, in, sizeof h);
  const BlobHeader want = header_of(s);
  if (std::memcmp(&h, &want, sizeof h) != 0)
    return fail(LABS_ERR_INVALID_ARGUMENT, "checkpoint does not match this solver");
  size_t off = sizeof h;
  for (auto& part : state_parts(s)) {
    LABS_H2D(part.first, in + off, part.second);
    off += part.second;
  }
  k_restamp<<<(s->R + 127) / 128, 128, 0, ctx->stream>>>(s->R, s->t0.as<int64_t>());
  LABS_CUDA(cudaGetLastError());
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

int labs_memetic(labs_ctx* ctx, int n, const labs_memetic_params* params, uint64_t seed,
                 const volatile int32_t* stop, int replica_id, labs_run_result* out,
                 labs_memetic_record* trace, int64_t trace_cap, int64_t* trace_len) {
  if (int rc = check_memetic(n, params)) return rc;
  if (!ctx || !out) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (trace && (trace_cap < 0 || !trace_len))
    return fail(LABS_ERR_INVALID_ARGUMENT, "trace needs a capacity and a length output");
  labs_solver* s = nullptr;
  if (int rc = labs_solver_create(ctx, n, 1, seed, 0, params, trace ? trace_cap : 0, &s))
    return rc;
  std::unique_ptr<labs_solver, int (*)(labs_solver*)> guard(s, labs_solver_destroy);
  // With a host stop flag, run in epochs and forward the flag in between.
  for (;;) {
    if (stop && *stop)
      if (int rc = labs_solver_request_stop(s)) return rc;
    if (int rc = labs_solver_run(s, stop ? 8 : -1, -1.0, 0)) return rc;
    int32_t running = 0;
    if (int rc = labs_solver_status(s, &running, nullptr, nullptr)) return rc;
    if (!running) break;
  }
  if (int rc = labs_solver_results(s, out, trace, trace_len, nullptr)) return rc;
  out->seed = seed;
  out->replica_id = replica_id;
  return LABS_OK;
}

int labs_run_replicas(labs_ctx* ctx, int n, int replicas, uint64_t base_seed,
                      const labs_memetic_params* params, labs_run_result* out,
                      labs_run_result* per_replica, labs_memetic_record* traces,
                      int64_t trace_cap, int64_t* trace_len) {
  if (n < 2) return fail(LABS_ERR_INVALID_ARGUMENT, "run needs length >= 2");
  if (replicas < 1) return fail(LABS_ERR_INVALID_ARGUMENT, "replicas must be >= 1");
  if (int rc = check_memetic(n, params)) return rc;
  if (!ctx || !out) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (traces && (trace_cap < 0 || !trace_len))
    return fail(LABS_ERR_INVALID_ARGUMENT, "traces need a capacity and length outputs");
  labs_solver* s = nullptr;
  if (int rc = labs_solver_create(ctx, n, replicas, base_seed, 0, params, traces ? trace_cap : 0,
                                  &s))
    return rc;
  std::unique_ptr<labs_solver, int (*)(labs_solver*)> guard(s, labs_solver_destroy);
  if (int rc = labs_solver_run(s, -1, -1.0, 1)) return rc;
  std::vector<labs_run_result> per(replicas);
  std::vector<int32_t> order(replicas);
  if (int rc = labs_solver_results(s, per.data(), traces, trace_len, order.data())) return rc;
  // SharedState::publish (parallel.cpp:10-15): strictly lower energy wins;
  // among equal energies the earliest publisher keeps the slot.
  int win = 0;
  for (int r = 1; r < replicas; ++r) {
    if (per[r].best_energy < per[win].best_energy ||
        (per[r].best_energy == per[win].best_energy && order[r] < order[win]))
      win = r;
  }
  *out = per[win];
  if (per_replica) std::memcpy(per_replica, per.data(), sizeof(labs_run_result) * replicas);
  return LABS_OK;
}

}  // extern "C"

extern "C" int labs_bench_int_peak(labs_ctx* ctx, double* gops) {
  if (!ctx || !gops) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  LABS_CUDA(cudaSetDevice(ctx->device));
  DBuf sink;
  LABS_ALLOC(sink, sizeof(int));
  const int blocks = ctx->sm_count * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  LABS_CUDA(cudaEventCreate(&e0));
  LABS_CUDA(cudaEventCreate(&e1));
  k_int_peak<<<blocks, threads, 0, ctx->stream>>>(64, 3, sink.as<int>());  // warm-up
  float best_ms = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    LABS_CUDA(cudaEventRecord(e0, ctx->stream));
    k_int_peak<<<blocks, threads, 0, ctx->stream>>>(iters, 3 + rep, sink.as<int>());
    LABS_CUDA(cudaEventRecord(e1, ctx->stream));
    LABS_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    LABS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best_ms = std::min(best_ms, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  LABS_CUDA(cudaGetLastError());
  const double ops = static_cast<double>(blocks) * threads * iters * 16.0 * 8.0;
  *gops = ops / (best_ms * 1e-3) / 1e9;
  return LABS_OK;
}

// ------------------------------------------------- exhaustive oracle (K5) --
namespace {

template <class F>
int dispatch_kmax(int n, F&& f) {
  if (n <= 16) return f(std::integral_constant<int, 16>{});
  if (n <= 32) return f(std::integral_constant<int, 32>{});
  if (n <= 48) return f(std::integral_constant<int, 48>{});
  return f(std::integral_constant<int, 64>{});
}

struct ExhaustShape {
  int B;            // Gray-index bits walked per thread
  uint64_t blocks;  // threads
  unsigned grid;
};

ExhaustShape exhaust_shape(int n) {
  const int free_bits = n - 1;
  ExhaustShape sh;
  sh.B = free_bits > 18 ? free_bits - 18 : 0;  // >= 2^18 threads when possible
  sh.blocks = 1ULL << (free_bits - sh.B);
  sh.grid = static_cast<unsigned>((sh.blocks + 127) / 128);
  return sh;
}

}  // namespace

extern "C" int labs_exhaustive_optimum(labs_ctx* ctx, int n, int64_t* optimal_energy,
                                       uint64_t* witnesses, int64_t cap, int64_t* count) {
  if (!ctx || !optimal_energy || !count || cap < 0 || (cap && !witnesses))
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n < 2 || n > 64)
    return fail(LABS_ERR_INVALID_ARGUMENT, "device exhaustive search needs 2 <= n <= 64");
  LABS_CUDA(cudaSetDevice(ctx->device));
  const ExhaustShape sh = exhaust_shape(n);
  DBuf mins, ids, out, cnt;
  LABS_ALLOC(mins, sizeof(int) * sh.blocks);
  LABS_ALLOC(out, sizeof(uint64_t) * std::max<int64_t>(cap, 1));
  LABS_ALLOC(cnt, sizeof(unsigned long long));
  LABS_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
  // pass 1: per-block minima
  int rc = dispatch_kmax(n, [&](auto km) -> int {
    constexpr int KMAX = decltype(km)::value;
    k_exhaust_min<KMAX><<<sh.grid, 128, 0, ctx->stream>>>(n, sh.B, sh.blocks, mins.as<int>());
    LABS_CUDA(cudaGetLastError());
    return LABS_OK;
  });
  if (rc) return rc;
  std::vector<int> h(sh.blocks);
  LABS_D2H(h.data(), mins.p, sizeof(int) * sh.blocks);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  const int e = *std::min_element(h.begin(), h.end());
  std::vector<uint32_t> sel;
  for (uint64_t t = 0; t < sh.blocks; ++t)
    if (h[t] == e) sel.push_back(static_cast<uint32_t>(t));
  // pass 2: witnesses, only in the blocks that hold the optimum
  LABS_ALLOC(ids, sizeof(uint32_t) * sel.size());
  LABS_H2D(ids.p, sel.data(), sizeof(uint32_t) * sel.size());
  rc = dispatch_kmax(n, [&](auto km) -> int {
    constexpr int KMAX = decltype(km)::value;
    const int cntb = static_cast<int>(sel.size());
    k_exhaust_collect<KMAX><<<(cntb + 127) / 128, 128, 0, ctx->stream>>>(
        n, sh.B, ids.as<uint32_t>(), cntb, e, out.as<uint64_t>(),
        static_cast<unsigned long long>(cap), cnt.as<unsigned long long>());
    LABS_CUDA(cudaGetLastError());
    return LABS_OK;
  });
  if (rc) return rc;
  unsigned long long c = 0;
  LABS_D2H(&c, cnt.p, sizeof(c));
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (cap && c) LABS_D2H(witnesses, out.p, sizeof(uint64_t) * std::min<uint64_t>(c, cap));
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  *optimal_energy = e;
  *count = static_cast<int64_t>(c);
  return LABS_OK;
}

extern "C" int labs_local_optima(labs_ctx* ctx, int n, int64_t* count) {
  if (!ctx || !count) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n < 2 || n > 64)
    return fail(LABS_ERR_INVALID_ARGUMENT, "device local-optima census needs 2 <= n <= 64");
  LABS_CUDA(cudaSetDevice(ctx->device));
  DBuf cnt;
  LABS_ALLOC(cnt, sizeof(unsigned long long));
  LABS_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), ctx->stream));
  const ExhaustShape sh = exhaust_shape(n);
  int rc = dispatch_kmax(n, [&](auto km) -> int {
    constexpr int KMAX = decltype(km)::value;
    k_local_optima<KMAX><<<sh.grid, 128, 0, ctx->stream>>>(n, sh.B, sh.blocks,
                                                           cnt.as<unsigned long long>());
    LABS_CUDA(cudaGetLastError());
    return LABS_OK;
  });
  if (rc) return rc;
  unsigned long long c = 0;
  LABS_D2H(&c, cnt.p, sizeof(c));
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  *count = 2 * static_cast<int64_t>(c);  // the complement half mirrors every optimum
  return LABS_OK;
}
