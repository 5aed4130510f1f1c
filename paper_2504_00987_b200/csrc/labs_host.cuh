// labs_host.cuh — host-side plumbing shared by the C-ABI translation unit
// (labs_kernels.cu) and the per-NS launch units (labs_ns.cu): the context,
// status codes, device buffers, occupancy-sized grids, NS dispatch, and the
// per-NS launcher declarations. The launchers are defined (and their kernels
// instantiated) only in labs_ns.cu, once per NS.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <type_traits>

#include "labs_b200.h"
#include "labs_device.cuh"

struct labs_ctx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
};

namespace labsh {
using namespace labsk;


extern thread_local std::string g_err;

inline int fail(int code, const std::string& msg) {
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

inline int check_n(int n) {
  if (n < 2) return fail(LABS_ERR_INVALID_ARGUMENT, "length must be >= 2");
  if (n > LABS_MAX_N)
    return fail(LABS_ERR_INVALID_ARGUMENT,
                "length exceeds the device walker limit " +
                    std::to_string(LABS_MAX_N));
  return LABS_OK;
}

inline int ns_of(int n) { return (n + 31) / 32; }
inline int nw_of(int n) { return (n + 63) / 64; }

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

inline int check_tabu(const labs_tabu_params* p) {
  if (!p) return fail(LABS_ERR_INVALID_ARGUMENT, "null tabu params");
  if (p->min_tabu_factor < 0 || p->max_tabu_factor < p->min_tabu_factor ||
      p->max_tabu_factor >= 1)
    return fail(LABS_ERR_INVALID_ARGUMENT,
                "tabu tenure factors need 0 <= min <= max < 1");
  if (p->tie_rule != LABS_TIE_REFERENCE && p->tie_rule != LABS_TIE_LOWEST)
    return fail(LABS_ERR_INVALID_ARGUMENT, "unknown tie rule");
  return LABS_OK;
}

inline TabuCfg to_cfg(const labs_tabu_params* p) {
  TabuCfg c;
  c.min_factor = p->min_tabu_factor;
  c.max_factor = p->max_tabu_factor;
  c.tie_rule = p->tie_rule;
  c.aspiration = p->aspiration ? 1 : 0;
  return c;
}

inline int check_seq_padding(int n, int count, const uint64_t* words) {
  const int nw = nw_of(n);
  const int rem = n & 63;
  if (!rem) return LABS_OK;
  const uint64_t bad = ~((1ULL << rem) - 1ULL);
  for (int c = 0; c < count; ++c)
    if (words[static_cast<size_t>(c) * nw + nw - 1] & bad)
      return fail(LABS_ERR_INVALID_ARGUMENT, "nonzero padding bits in sequence words");
  return LABS_OK;
}


// Launchers of the NS-templated kernels (labs_ns.cu). Device pointers in,
// asynchronous on ctx->stream.
template <int NS>
struct NsOps {
  static int build(labs_ctx* ctx, int n, int count, const uint64_t* dw, int32_t* dc,
                   int64_t* de, int64_t* dn);
  static int flip_trace(labs_ctx* ctx, int n, int count, const uint64_t* dw, int flips,
                        const int32_t* dp, int64_t* de, int64_t* dn);
  static int scan(labs_ctx* ctx, int n, int count, const uint64_t* dw, const uint8_t* da,
                  labs_rng_state* dr, int allow_fallback, int tie_rule, int32_t* dpos,
                  int64_t* de, int32_t* dfb, int32_t* dnt, uint64_t* dtm);
  static int tabu(labs_ctx* ctx, WalkArgs& A, bool mt);
};

template <int NS, int T>
struct MemeticOps {
  static int launch(labs_ctx* ctx, const MemeticArgs& A, bool mt);
  static int blocks_per_sm(labs_ctx* ctx, bool mt, int* per_sm);
};

}  // namespace labsh
