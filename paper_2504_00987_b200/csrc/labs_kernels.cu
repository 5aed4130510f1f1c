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
#include <cstring>
#include <string>
#include <vector>

#include "labs_b200.h"
#include "labs_memetic.cuh"
#include "labs_walker.cuh"

namespace labsk {

constexpr int kWarps = 4;  // walkers per block

// Occupancy target: 8 blocks (32 warps) per SM up to n = 128 caps registers
// at 64/thread; longer sequences carry twice the per-slot state.
template <int NS>
__host__ __device__ constexpr int min_blocks() {
  return NS <= 4 ? 8 : 4;
}

template <int NS, bool MT>
struct WarpSlot {
  WalkSmem<NS> walk;
  uint64_t mt[MT ? kMtN : 1];
};

template <int NS, bool MT>
__host__ __device__ constexpr size_t slot_bytes() {
  return (sizeof(WarpSlot<NS, MT>) + 15) & ~size_t(15);
}

template <int NS, bool MT>
__device__ __forceinline__ WarpSlot<NS, MT>& my_slot() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return *reinterpret_cast<WarpSlot<NS, MT>*>(smem_raw +
                                              (threadIdx.x >> 5) * slot_bytes<NS, MT>());
}

__device__ __forceinline__ int global_warp() {
  return blockIdx.x * kWarps + (threadIdx.x >> 5);
}
__device__ __forceinline__ int total_warps() { return gridDim.x * kWarps; }

__device__ __forceinline__ void mt_load(uint64_t* s, const labs_rng_state& g,
                                        int& idx) {
  for (int i = lane_id(); i < kMtN; i += 32) s[i] = g.mt[i];
  idx = g.idx;
  __syncwarp();
}
__device__ __forceinline__ void mt_store(const uint64_t* s, labs_rng_state& g,
                                         int idx) {
  __syncwarp();
  for (int i = lane_id(); i < kMtN; i += 32) g.mt[i] = s[i];
  if (lane_id() == 0) g.idx = idx;
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
        corr[static_cast<size_t>(item) * (n - 1) + j - 1] = w.ck[b];
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
    rng.mt = sl.mt;
    mt_load(sl.mt, rng_states[item], rng.idx);
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
      select_move<NS>(dE, adm, n, tie_rule, rng, pos, dEp, fb, msk, ntie);
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
      rng.mt = sl.mt;
      mt_load(sl.mt, A.mt[item], rng.idx);
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
      rng.ctr = A.ctr_base;
      rng.cache = (rng.ctr & 1ULL) ? rng.block_half(rng.ctr) : 0ULL;
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
template <int NS, bool MT>
__global__ void __launch_bounds__(32 * kWarps, min_blocks<NS>()) k_memetic(MemeticArgs A) {
  auto& sl = my_slot<NS, MT>();
  smem_clear(sl.walk);
  Walker<NS> w;
  w.sm = &sl.walk;
  for (int r = global_warp(); r < A.replicas; r += total_warps()) {
    if (A.initialized[r] && A.status[r] != kRunning) continue;
    if constexpr (MT) {
      MtRng rng;
      rng.mt = sl.mt;
      mt_load(sl.mt, A.mt[r], rng.idx);
      memetic_replica<NS>(A, r, w, rng);
      mt_store(sl.mt, A.mt[r], rng.idx);
    } else {
      PhiloxRng rng;
      rng.k0 = static_cast<uint32_t>(A.base_seed);
      rng.k1 = static_cast<uint32_t>(A.base_seed >> 32);
      rng.s0 = static_cast<uint32_t>(r);
      rng.s1 = 0x4D454D45u;  // "MEME"
      rng.ctr = A.ctr[r];
      rng.cache = (rng.ctr & 1ULL) ? rng.block_half(rng.ctr) : 0ULL;
      memetic_replica<NS>(A, r, w, rng);
      if (lane_id() == 0) A.ctr[r] = rng.ctr;
    }
    __syncwarp();
  }
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
int grid_for(labs_ctx* ctx, Kern kern, size_t smem, int items, int* grid) {
  int per_sm = 0;
  LABS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kWarps, smem));
  if (per_sm < 1) per_sm = 1;
  const int want = (items + kWarps - 1) / kWarps;
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

struct MemeticRun {
  DBuf pop, popE, best, bestE, iters, status, init, t0, tend, order, counter, mt, ctr, stop,
      tabu_iters, trace, trace_len;
};

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
  return check_tabu(&p->tabu);
}

// Runs `replicas` memetic replicas to completion. host_stop, when given, is
// polled between epochs and forwarded to the device stop flag.
int run_memetic(labs_ctx* ctx, int n, int replicas, uint64_t base_seed,
                const labs_memetic_params* p, const volatile int32_t* host_stop, int race,
                labs_run_result* per_replica, labs_memetic_record* traces, int64_t trace_cap,
                int64_t* trace_len, std::vector<int32_t>* order_out) {
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int nw = nw_of(n), K = p->population_size;
  const bool mt = p->rng_kind == LABS_RNG_MT19937_64;
  MemeticRun b;
  LABS_ALLOC(b.pop, sizeof(uint64_t) * replicas * K * nw);
  LABS_ALLOC(b.popE, sizeof(int32_t) * replicas * K);
  LABS_ALLOC(b.best, sizeof(uint64_t) * replicas * nw);
  LABS_ALLOC(b.bestE, sizeof(int32_t) * replicas);
  LABS_ALLOC(b.iters, sizeof(int64_t) * replicas);
  LABS_ALLOC(b.status, sizeof(int32_t) * replicas);
  LABS_ALLOC(b.init, sizeof(int32_t) * replicas);
  LABS_ALLOC(b.t0, sizeof(int64_t) * replicas);
  LABS_ALLOC(b.tend, sizeof(int64_t) * replicas);
  LABS_ALLOC(b.order, sizeof(int32_t) * replicas);
  LABS_ALLOC(b.counter, sizeof(int32_t));
  LABS_ALLOC(b.stop, sizeof(int32_t));
  if (mt) LABS_ALLOC(b.mt, sizeof(labs_rng_state) * replicas);
  else LABS_ALLOC(b.ctr, sizeof(uint64_t) * replicas);
  if (traces) {
    LABS_ALLOC(b.trace, sizeof(int64_t) * 3 * replicas * std::max<int64_t>(trace_cap, 1));
    LABS_ALLOC(b.trace_len, sizeof(int64_t) * replicas);
  }
  LABS_CUDA(cudaMemsetAsync(b.init.p, 0, sizeof(int32_t) * replicas, ctx->stream));
  LABS_CUDA(cudaMemsetAsync(b.status.p, 0, sizeof(int32_t) * replicas, ctx->stream));
  LABS_CUDA(cudaMemsetAsync(b.counter.p, 0, sizeof(int32_t), ctx->stream));
  LABS_CUDA(cudaMemsetAsync(b.stop.p, 0, sizeof(int32_t), ctx->stream));
  LABS_CUDA(cudaMemsetAsync(b.order.p, 0xff, sizeof(int32_t) * replicas, ctx->stream));
  if (mt) {
    k_seed<<<(replicas + 127) / 128, 128, 0, ctx->stream>>>(replicas, base_seed,
                                                             b.mt.as<labs_rng_state>());
    LABS_CUDA(cudaGetLastError());
  } else {
    LABS_CUDA(cudaMemsetAsync(b.ctr.p, 0, sizeof(uint64_t) * replicas, ctx->stream));
  }
  MemeticArgs A{};
  A.n = n;
  A.nw = nw;
  A.replicas = replicas;
  A.K = K;
  A.p_comb = p->p_comb;
  A.p_mutate = p->p_mutate > 0.0 ? p->p_mutate : 1.0 / n;
  A.target = p->target_energy;
  A.max_ns = p->max_seconds >= 0 ? static_cast<int64_t>(p->max_seconds * 1e9) : -1;
  A.max_iterations = p->max_iterations;
  A.tabu = to_cfg(&p->tabu);
  A.race = race;
  A.base_seed = base_seed;
  A.pop = b.pop.as<uint64_t>();
  A.popE = b.popE.as<int32_t>();
  A.best = b.best.as<uint64_t>();
  A.bestE = b.bestE.as<int32_t>();
  A.iters = b.iters.as<int64_t>();
  A.status = b.status.as<int32_t>();
  A.initialized = b.init.as<int32_t>();
  A.t0 = b.t0.as<int64_t>();
  A.t_end = b.tend.as<int64_t>();
  A.pub_order = b.order.as<int32_t>();
  A.pub_counter = b.counter.as<int32_t>();
  A.mt = mt ? b.mt.as<labs_rng_state>() : nullptr;
  A.ctr = mt ? nullptr : b.ctr.as<uint64_t>();
  A.stop = b.stop.as<int32_t>();
  A.tabu_iters = nullptr;
  A.trace = traces ? b.trace.as<int64_t>() : nullptr;
  A.trace_cap = traces ? trace_cap : 0;
  A.trace_len = traces ? b.trace_len.as<int64_t>() : nullptr;
  // With a host stop flag, run in epochs and forward the flag in between.
  A.epoch_iters = host_stop ? 8 : -1;
  std::vector<int32_t> status(replicas);
  for (;;) {
    if (host_stop && *host_stop) {
      const int32_t one = 1;
      LABS_H2D(b.stop.p, &one, sizeof(int32_t));
    }
    int rc = dispatch(n, [&](auto ns) -> int {
      constexpr int NS = decltype(ns)::value;
      if (mt) {
        const size_t smem = kWarps * slot_bytes<NS, true>();
        auto kern = k_memetic<NS, true>;
        if (int r = prep(kern, smem)) return r;
        int grid = 0;
        if (int r = grid_for(ctx, kern, smem, replicas, &grid)) return r;
        kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(A);
      } else {
        const size_t smem = kWarps * slot_bytes<NS, false>();
        auto kern = k_memetic<NS, false>;
        if (int r = prep(kern, smem)) return r;
        int grid = 0;
        if (int r = grid_for(ctx, kern, smem, replicas, &grid)) return r;
        kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(A);
      }
      LABS_CUDA(cudaGetLastError());
      return LABS_OK;
    });
    if (rc) return rc;
    LABS_D2H(status.data(), b.status.p, sizeof(int32_t) * replicas);
    LABS_CUDA(cudaStreamSynchronize(ctx->stream));
    bool done = true;
    for (int r = 0; r < replicas; ++r) done &= status[r] != kRunning;
    if (done) break;
  }
  std::vector<uint64_t> best(static_cast<size_t>(replicas) * nw);
  std::vector<int32_t> bestE(replicas), order(replicas);
  std::vector<int64_t> iters(replicas), t0(replicas), tend(replicas);
  LABS_D2H(best.data(), b.best.p, sizeof(uint64_t) * replicas * nw);
  LABS_D2H(bestE.data(), b.bestE.p, sizeof(int32_t) * replicas);
  LABS_D2H(iters.data(), b.iters.p, sizeof(int64_t) * replicas);
  LABS_D2H(t0.data(), b.t0.p, sizeof(int64_t) * replicas);
  LABS_D2H(tend.data(), b.tend.p, sizeof(int64_t) * replicas);
  LABS_D2H(order.data(), b.order.p, sizeof(int32_t) * replicas);
  std::vector<int64_t> tr, tl;
  if (traces) {
    tr.resize(static_cast<size_t>(3) * replicas * std::max<int64_t>(trace_cap, 1));
    tl.resize(replicas);
    LABS_D2H(tr.data(), b.trace.p, sizeof(int64_t) * tr.size());
    LABS_D2H(tl.data(), b.trace_len.p, sizeof(int64_t) * replicas);
  }
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int r = 0; r < replicas; ++r) {
    labs_run_result& o = per_replica[r];
    std::memset(&o, 0, sizeof(o));
    for (int wi = 0; wi < nw; ++wi) o.best[wi] = best[static_cast<size_t>(r) * nw + wi];
    o.best_energy = bestE[r];
    o.merit = static_cast<double>(n) * n / (2.0 * static_cast<double>(bestE[r]));
    o.iterations = iters[r];
    o.wall_seconds = 1e-9 * static_cast<double>(tend[r] - t0[r]);
    o.seed = base_seed + static_cast<uint64_t>(r);
    o.replica_id = r;
    o.reached_target = bestE[r] <= p->target_energy;
    if (traces) {
      const int64_t len = std::min(tl[r], trace_cap);
      trace_len[r] = len;
      for (int64_t i = 0; i < len; ++i) {
        const int64_t* rec = &tr[(static_cast<size_t>(r) * trace_cap + i) * 3];
        labs_memetic_record& d = traces[static_cast<size_t>(r) * trace_cap + i];
        d.iteration = rec[0];
        d.stop_seen = static_cast<int32_t>(rec[1]);
        d.pad_ = 0;
        d.child_energy = rec[2];
      }
    }
  }
  if (order_out) *order_out = order;
  return LABS_OK;
}

}  // namespace

extern "C" {

int labs_memetic(labs_ctx* ctx, int n, const labs_memetic_params* params, uint64_t seed,
                 const volatile int32_t* stop, int replica_id, labs_run_result* out,
                 labs_memetic_record* trace, int64_t trace_cap, int64_t* trace_len) {
  if (int rc = check_memetic(n, params)) return rc;
  if (!ctx || !out) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (trace && (trace_cap < 0 || !trace_len))
    return fail(LABS_ERR_INVALID_ARGUMENT, "trace needs a capacity and a length output");
  int64_t tl = 0;
  int rc = run_memetic(ctx, n, 1, seed, params, stop, 0, out, trace, trace_cap,
                       trace ? &tl : nullptr, nullptr);
  if (rc) return rc;
  out->seed = seed;
  out->replica_id = replica_id;
  if (trace_len) *trace_len = tl;
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
  std::vector<labs_run_result> per(replicas);
  std::vector<int32_t> order;
  int rc = run_memetic(ctx, n, replicas, base_seed, params, nullptr, 1, per.data(), traces,
                       trace_cap, trace_len, &order);
  if (rc) return rc;
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
