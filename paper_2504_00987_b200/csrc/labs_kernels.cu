// labs_kernels.cu — the C ABI (include/labs_b200.h) over the sm_100a
// kernels: argument checks, device buffers, NS dispatch to the per-NS
// launchers (labs_ns.cu), the epoch-driven solver, checkpoints, the
// multi-GPU run and the island kernels. K5 lives in labs_exhaust.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "labs_host.cuh"

namespace labsk {

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

// IMAD-only probe: the INT32 multiply-add rate alone (FMA pipe), the
// denominator SURVEY.md §8(d) names for the lag-term MACs ((N-1) per
// flip-evaluation). 8 independent IMAD chains per thread, register operands.
__global__ void __launch_bounds__(256) k_imad_peak(int iters, int seed, int* sink) {
  int a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = (threadIdx.x + i) ^ seed;
    b[i] = (blockIdx.x + 3 * i) ^ seed;
  }
  const int m = seed | 1;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = a[i] * m + b[i];
    }
  }
  int v = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) v ^= a[i];
  if (v == 0x7fffffff) sink[0] = v;
}

}  // namespace labsk

using namespace labsk;
using namespace labsh;

namespace labsh {
thread_local std::string g_err;
}


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
    return NsOps<decltype(ns)::value>::build(ctx, n, count, dw.as<uint64_t>(), dc.as<int32_t>(),
                                             de.as<int64_t>(),
                                             neighbor_out ? dn.as<int64_t>() : nullptr);
  });
  if (rc) return rc;
  if (corr_out) LABS_D2H(corr_out, dc.p, sizeof(int32_t) * count * (n - 1));
  LABS_D2H(energy_out, de.p, sizeof(int64_t) * count);
  if (neighbor_out) LABS_D2H(neighbor_out, dn.p, sizeof(int64_t) * count * n);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  return LABS_OK;
}

// Persistent evaluator for one sequence (labs_eval_*): the device buffer and
// a pinned host mirror, laid out [words | E | neighbors | C], so one call is
// one H2D, one launch, one D2H and a sync — no allocation per call.
struct labs_eval {
  labs_ctx* ctx = nullptr;
  int n = 0, nw = 0;
  void* d = nullptr;
  unsigned char* h = nullptr;
  size_t bytes = 0, off_e = 0, off_nb = 0, off_c = 0;
  ~labs_eval() {
    if (d) {
      cudaSetDevice(ctx->device);
      cudaFree(d);
    }
    if (h) cudaFreeHost(h);
  }
};

int labs_eval_create(labs_ctx* ctx, int n, labs_eval** out) {
  if (int rc = check_n(n)) return rc;
  if (!ctx || !out) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  LABS_CUDA(cudaSetDevice(ctx->device));
  auto* e = new labs_eval;
  std::unique_ptr<labs_eval> guard(e);
  e->ctx = ctx;
  e->n = n;
  e->nw = nw_of(n);
  e->off_e = sizeof(uint64_t) * e->nw;
  e->off_nb = e->off_e + sizeof(int64_t);
  e->off_c = e->off_nb + sizeof(int64_t) * n;
  e->bytes = e->off_c + sizeof(int32_t) * (n - 1);
  LABS_CUDA(cudaMalloc(&e->d, e->bytes));
  LABS_CUDA(cudaMallocHost(reinterpret_cast<void**>(&e->h), e->bytes));
  *out = guard.release();
  return LABS_OK;
}

int labs_eval_destroy(labs_eval* e) {
  delete e;
  return LABS_OK;
}

int labs_eval_run(labs_eval* e, const uint64_t* words, int32_t* corr_out, int64_t* energy_out,
                  int64_t* neighbor_out) {
  if (!e || !words || !energy_out) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (int rc = check_seq_padding(e->n, 1, words)) return rc;
  labs_ctx* ctx = e->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  std::memcpy(e->h, words, sizeof(uint64_t) * e->nw);
  unsigned char* d = static_cast<unsigned char*>(e->d);
  LABS_H2D(d, e->h, sizeof(uint64_t) * e->nw);
  const int n = e->n;
  int rc = dispatch(n, [&](auto ns) -> int {
    return NsOps<decltype(ns)::value>::build(
        ctx, n, 1, reinterpret_cast<const uint64_t*>(d), reinterpret_cast<int32_t*>(d + e->off_c),
        reinterpret_cast<int64_t*>(d + e->off_e), reinterpret_cast<int64_t*>(d + e->off_nb));
  });
  if (rc) return rc;
  LABS_D2H(e->h + e->off_e, d + e->off_e, e->bytes - e->off_e);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(energy_out, e->h + e->off_e, sizeof(int64_t));
  if (neighbor_out) std::memcpy(neighbor_out, e->h + e->off_nb, sizeof(int64_t) * n);
  if (corr_out) std::memcpy(corr_out, e->h + e->off_c, sizeof(int32_t) * (n - 1));
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
    return NsOps<decltype(ns)::value>::flip_trace(ctx, n, count, dw.as<uint64_t>(), flips,
                                                  dp.as<int32_t>(), de.as<int64_t>(),
                                                  neighbor_out ? dn.as<int64_t>() : nullptr);
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
    return NsOps<decltype(ns)::value>::scan(
        ctx, n, count, dw.as<uint64_t>(), da.as<uint8_t>(), dr.as<labs_rng_state>(),
        allow_fallback, tie_rule, dpos.as<int32_t>(), de.as<int64_t>(), dfb.as<int32_t>(),
        dnt.as<int32_t>(), dtm.as<uint64_t>());
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
  return dispatch(n, [&](auto ns) -> int { return NsOps<decltype(ns)::value>::tabu(ctx, A, mt); });
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
  DBuf pop, popE, best, bestE, iters, status, init, t0, tend, elapsed, order, counter, rng, ctr,
      tabu_total, tabu_rep, trace, trace_len, taken, peers;
  // The stop flag is a plain cudaMalloc allocation (not stream-ordered) so
  // that other processes can map it through CUDA IPC (labs_ipc_export).
  int32_t* stop = nullptr;
  MemeticArgs A{};
  ~labs_solver() {
    if (stop) {
      cudaSetDevice(ctx->device);
      cudaFree(stop);
    }
  }
};

extern "C" {

int labs_solver_capacity(labs_ctx* ctx, int n, int rng_kind) {
  if (!ctx || check_n(n)) return 0;
  int out = 0;
  cudaSetDevice(ctx->device);
  dispatch_memetic(n, [&](auto ns, auto tt) -> int {
    int per_sm = 0;
    if (MemeticOps<decltype(ns)::value, decltype(tt)::value>::blocks_per_sm(
            ctx, rng_kind == LABS_RNG_MT19937_64, &per_sm))
      return LABS_OK;
    out = per_sm * ctx->sm_count * kWarps * (32 / decltype(tt)::value);
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
  LABS_ALLOC(s->elapsed, sizeof(int64_t) * R);
  LABS_ALLOC(s->order, sizeof(int32_t) * R);
  LABS_ALLOC(s->counter, sizeof(int32_t));
  LABS_CUDA(cudaMalloc(&s->stop, sizeof(int32_t)));
  LABS_ALLOC(s->tabu_total, sizeof(unsigned long long));
  LABS_ALLOC(s->tabu_rep, sizeof(int64_t) * R);
  LABS_ALLOC(s->taken, sizeof(int32_t) * R);
  LABS_ALLOC(s->peers, sizeof(int32_t*) * kMaxPeerStops);
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
  LABS_CUDA(cudaMemsetAsync(s->stop, 0, sizeof(int32_t), st));
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
  A.stop = s->stop;
  A.npeers = 0;
  A.peer_stop = s->peers.as<int32_t*>();
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
    return MemeticOps<decltype(ns)::value, decltype(tt)::value>::launch(ctx, A, s->mt);
  });
}

int labs_solver_request_stop(labs_solver* s) {
  if (!s) return fail(LABS_ERR_INVALID_ARGUMENT, "null solver");
  labs_ctx* ctx = s->ctx;
  static const int32_t one = 1;
  LABS_CUDA(cudaSetDevice(ctx->device));
  LABS_H2D(s->stop, &one, sizeof(int32_t));
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
      // trace_len reports every record the replica produced; only the
      // first trace_cap are stored, so a caller can detect truncation.
      const int64_t len = std::min(tl[r], s->trace_cap);
      if (trace_len) trace_len[r] = tl[r];
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
  uint64_t magic;  // "LABSCKP2"
  int32_t n, R, K, nw;
  int64_t trace_cap;
  uint64_t base_seed;
  int64_t replica_offset;
  // every run parameter that shapes a trajectory (labs_memetic_params)
  int32_t population_size, rng_kind;
  double p_comb, p_mutate;
  int64_t target_energy;
  double max_seconds;
  int64_t max_iterations;
  double min_tabu_factor, max_tabu_factor;
  int32_t tie_rule, aspiration, crossover, replacement;
};
constexpr uint64_t kBlobMagic = 0x32504B4353424C4CULL;

// (device buffer, bytes) in blob order. Timers are saved as each replica's
// elapsed run time (s->elapsed, filled by k_elapsed at save), not as raw
// %globaltimer stamps, so budgets and wall times survive a resume.
std::vector<std::pair<void*, size_t>> state_parts(labs_solver* s) {
  const size_t R = s->R, K = s->K, nw = s->nw;
  std::vector<std::pair<void*, size_t>> v = {
      {s->pop.p, sizeof(uint64_t) * R * K * nw}, {s->popE.p, sizeof(int32_t) * R * K},
      {s->best.p, sizeof(uint64_t) * R * nw},    {s->bestE.p, sizeof(int32_t) * R},
      {s->iters.p, sizeof(int64_t) * R},         {s->status.p, sizeof(int32_t) * R},
      {s->init.p, sizeof(int32_t) * R},          {s->elapsed.p, sizeof(int64_t) * R},
      {s->order.p, sizeof(int32_t) * R},         {s->counter.p, sizeof(int32_t)},
      {s->stop, sizeof(int32_t)},                {s->tabu_total.p, sizeof(unsigned long long)},
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
  BlobHeader h;
  std::memset(&h, 0, sizeof h);
  h.magic = kBlobMagic;
  h.n = s->n;
  h.R = s->R;
  h.K = s->K;
  h.nw = s->nw;
  h.trace_cap = s->trace_cap;
  h.base_seed = s->base_seed;
  h.replica_offset = s->offset;
  const labs_memetic_params& p = s->p;
  h.population_size = p.population_size;
  h.rng_kind = p.rng_kind;
  h.p_comb = p.p_comb;
  h.p_mutate = p.p_mutate;
  h.target_energy = p.target_energy;
  h.max_seconds = p.max_seconds;
  h.max_iterations = p.max_iterations;
  h.min_tabu_factor = p.tabu.min_tabu_factor;
  h.max_tabu_factor = p.tabu.max_tabu_factor;
  h.tie_rule = p.tabu.tie_rule;
  h.aspiration = p.tabu.aspiration;
  h.crossover = p.crossover;
  h.replacement = p.replacement;
  return h;
}

// Elapsed run time per replica: finished replicas keep t_end - t0, running
// ones count up to now; never-initialized replicas have none.
__global__ void k_elapsed(int R, const int64_t* t0, const int64_t* tend, const int32_t* status,
                          const int32_t* init, int64_t* elapsed) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  if (!init[r]) {
    elapsed[r] = 0;
    return;
  }
  elapsed[r] = (status[r] != kRunning ? tend[r] : globaltimer_ns()) - t0[r];
}

// Resume: t0 = now - elapsed, and t_end = now for finished replicas, so
// t_end - t0 (their wall time) and the max_seconds budget of running ones
// continue where the checkpoint left them.
__global__ void k_restamp(int R, const int64_t* elapsed, int64_t* t0, int64_t* tend) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int64_t now = globaltimer_ns();
  t0[r] = now - elapsed[r];
  tend[r] = now;
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
  k_elapsed<<<(s->R + 127) / 128, 128, 0, ctx->stream>>>(
      s->R, s->t0.as<int64_t>(), s->tend.as<int64_t>(), s->status.as<int32_t>(),
      s->init.as<int32_t>(), s->elapsed.as<int64_t>());
  LABS_CUDA(cudaGetLastError());
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
    return fail(LABS_ERR_INVALID_ARGUMENT,
                "checkpoint does not match this solver (n, replicas, seeds, offset, trace "
                "capacity and every run parameter must agree)");
  size_t off = sizeof h;
  for (auto& part : state_parts(s)) {
    LABS_H2D(part.first, in + off, part.second);
    off += part.second;
  }
  k_restamp<<<(s->R + 127) / 128, 128, 0, ctx->stream>>>(s->R, s->elapsed.as<int64_t>(),
                                                          s->t0.as<int64_t>(),
                                                          s->tend.as<int64_t>());
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

int labs_solver_stop_flag(labs_solver* s, int32_t** d_flag) {
  if (!s || !d_flag) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  *d_flag = s->stop;
  return LABS_OK;
}

int labs_solver_set_peer_stops(labs_solver* s, int count, int32_t* const* d_flags) {
  if (!s || count < 0 || count > LABS_MAX_PEERS || (count && !d_flags))
    return fail(LABS_ERR_INVALID_ARGUMENT, "peer stop flags: 0..LABS_MAX_PEERS device pointers");
  for (int i = 0; i < count; ++i)
    if (!d_flags[i]) return fail(LABS_ERR_INVALID_ARGUMENT, "null peer stop flag");
  labs_ctx* ctx = s->ctx;
  LABS_CUDA(cudaSetDevice(ctx->device));
  int32_t* h[kMaxPeerStops] = {};
  for (int i = 0; i < count; ++i) h[i] = d_flags[i];
  LABS_H2D(s->peers.p, h, sizeof h);
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  s->A.npeers = count;
  return LABS_OK;
}

int labs_ipc_export(labs_ctx* ctx, const void* d_ptr, void* handle) {
  if (!ctx || !d_ptr || !handle) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == LABS_IPC_HANDLE_BYTES, "IPC handle size");
  LABS_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  LABS_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
  std::memcpy(handle, &h, sizeof h);
  return LABS_OK;
}

int labs_ipc_open(labs_ctx* ctx, const void* handle, void** d_ptr) {
  if (!ctx || !handle || !d_ptr) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  LABS_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  LABS_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return LABS_OK;
}

int labs_ipc_close(labs_ctx* ctx, void* d_ptr) {
  if (!ctx || !d_ptr) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  LABS_CUDA(cudaSetDevice(ctx->device));
  LABS_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return LABS_OK;
}

int labs_run_replicas_multi(labs_ctx* const* ctxs, int ngpu, int n, int replicas,
                            uint64_t base_seed, const labs_memetic_params* params,
                            labs_run_result* out, labs_run_result* per_replica,
                            labs_memetic_record* traces, int64_t trace_cap, int64_t* trace_len) {
  if (n < 2) return fail(LABS_ERR_INVALID_ARGUMENT, "run needs length >= 2");
  if (replicas < 1) return fail(LABS_ERR_INVALID_ARGUMENT, "replicas must be >= 1");
  if (!ctxs || ngpu < 1 || ngpu > LABS_MAX_PEERS + 1)
    return fail(LABS_ERR_INVALID_ARGUMENT, "need 1..LABS_MAX_PEERS+1 contexts");
  for (int g = 0; g < ngpu; ++g)
    if (!ctxs[g]) return fail(LABS_ERR_INVALID_ARGUMENT, "null context");
  if (int rc = check_memetic(n, params)) return rc;
  if (!out) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (traces && (trace_cap < 0 || !trace_len))
    return fail(LABS_ERR_INVALID_ARGUMENT, "traces need a capacity and length outputs");
  // Contiguous blocks; islands with no replica are dropped.
  std::vector<int> dev_of, first, count;
  for (int g = 0, start = 0; g < ngpu; ++g) {
    const int c = replicas / ngpu + (g < replicas % ngpu ? 1 : 0);
    if (c > 0) {
      dev_of.push_back(g);
      first.push_back(start);
      count.push_back(c);
    }
    start += c;
  }
  const int G = static_cast<int>(dev_of.size());
  // Device-side stop needs peer access between every pair of distinct
  // devices; a shared publish counter additionally needs native P2P atomics.
  bool p2p = true, atomics = true;
  for (int a = 0; a < G; ++a)
    for (int b = 0; b < G; ++b) {
      const int da = ctxs[dev_of[a]]->device, db = ctxs[dev_of[b]]->device;
      if (da == db) continue;
      int can = 0, nat = 0;
      LABS_CUDA(cudaDeviceCanAccessPeer(&can, da, db));
      if (can) LABS_CUDA(cudaDeviceGetP2PAttribute(&nat, cudaDevP2PAttrNativeAtomicSupported, da, db));
      if (!can) p2p = false;
      if (!nat) atomics = false;
      if (can) {
        LABS_CUDA(cudaSetDevice(da));
        const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else LABS_CUDA(e);
      }
    }
  atomics = atomics && p2p;
  std::vector<std::unique_ptr<labs_solver, int (*)(labs_solver*)>> sv;
  for (int i = 0; i < G; ++i) {
    labs_solver* s = nullptr;
    if (int rc = labs_solver_create(ctxs[dev_of[i]], n, count[i], base_seed, first[i], params,
                                    traces ? trace_cap : 0, &s))
      return rc;
    sv.emplace_back(s, labs_solver_destroy);
  }
  if (p2p && G > 1) {
    for (int i = 0; i < G; ++i) {
      int32_t* peers[kMaxPeerStops];
      int np = 0;
      for (int j = 0; j < G; ++j)
        if (j != i) peers[np++] = sv[j]->stop;
      if (int rc = labs_solver_set_peer_stops(sv[i].get(), np, peers)) return rc;
      if (atomics) sv[i]->A.pub_counter = sv[0]->counter.as<int32_t>();
    }
    // Every solver's initialization (flag and counter memsets) is complete
    // before any island can raise a peer's flag.
    for (int i = 0; i < G; ++i) LABS_CUDA(cudaStreamSynchronize(sv[i]->ctx->stream));
    for (int i = 0; i < G; ++i)
      if (int rc = labs_solver_run(sv[i].get(), -1, -1.0, 1)) return rc;
    for (int i = 0; i < G; ++i) {
      LABS_CUDA(cudaSetDevice(sv[i]->ctx->device));
      LABS_CUDA(cudaStreamSynchronize(sv[i]->ctx->stream));
    }
  } else if (G > 1) {
    // No peer access: the host forwards the stop between short epochs.
    for (;;) {
      for (int i = 0; i < G; ++i)
        if (int rc = labs_solver_run(sv[i].get(), -1, 0.01, 1)) return rc;
      int running = 0, stop = 0;
      for (int i = 0; i < G; ++i) {
        int32_t run = 0, flag = 0;
        if (int rc = labs_solver_status(sv[i].get(), &run, nullptr, nullptr)) return rc;
        LABS_CUDA(cudaMemcpy(&flag, sv[i]->stop, sizeof flag, cudaMemcpyDeviceToHost));
        running += run;
        stop |= flag;
      }
      if (!running) break;
      if (stop)
        for (int i = 0; i < G; ++i)
          if (int rc = labs_solver_request_stop(sv[i].get())) return rc;
    }
  } else {
    if (int rc = labs_solver_run(sv[0].get(), -1, -1.0, 1)) return rc;
  }
  std::vector<labs_run_result> per(replicas);
  std::vector<int32_t> order(replicas);
  std::vector<int64_t> rank(replicas);
  std::vector<labs_memetic_record> tr;
  std::vector<int64_t> tl;
  for (int i = 0; i < G; ++i) {
    const int c = count[i], f = first[i];
    if (traces) {
      tr.assign(static_cast<size_t>(c) * trace_cap, labs_memetic_record{});
      tl.assign(c, 0);
    }
    if (int rc = labs_solver_results(sv[i].get(), per.data() + f, traces ? tr.data() : nullptr,
                                     traces ? tl.data() : nullptr, order.data() + f))
      return rc;
    for (int r = 0; r < c; ++r)
      rank[f + r] = atomics ? order[f + r]
                            : (static_cast<int64_t>(order[f + r]) << 8) | static_cast<int64_t>(i);
    if (traces) {
      std::memcpy(traces + static_cast<size_t>(f) * trace_cap, tr.data(),
                  sizeof(labs_memetic_record) * tr.size());
      std::memcpy(trace_len + f, tl.data(), sizeof(int64_t) * c);
    }
  }
  int win = 0;
  for (int r = 1; r < replicas; ++r)
    if (per[r].best_energy < per[win].best_energy ||
        (per[r].best_energy == per[win].best_energy && rank[r] < rank[win]))
      win = r;
  *out = per[win];
  if (per_replica) std::memcpy(per_replica, per.data(), sizeof(labs_run_result) * replicas);
  return LABS_OK;
}

}  // extern "C"

namespace {
// Best-of-5 rate of a probe kernel in Gop/s (ops_per_thread_iter lane-ops
// per thread per loop iteration).
template <class Kern>
int probe_rate(labs_ctx* ctx, Kern kern, double ops_per_thread_iter, double* gops) {
  LABS_CUDA(cudaSetDevice(ctx->device));
  DBuf sink;
  LABS_ALLOC(sink, sizeof(int));
  const int blocks = ctx->sm_count * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  LABS_CUDA(cudaEventCreate(&e0));
  LABS_CUDA(cudaEventCreate(&e1));
  kern<<<blocks, threads, 0, ctx->stream>>>(64, 3, sink.as<int>());  // warm-up
  float best_ms = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    LABS_CUDA(cudaEventRecord(e0, ctx->stream));
    kern<<<blocks, threads, 0, ctx->stream>>>(iters, 3 + rep, sink.as<int>());
    LABS_CUDA(cudaEventRecord(e1, ctx->stream));
    LABS_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    LABS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best_ms = std::min(best_ms, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  LABS_CUDA(cudaGetLastError());
  const double ops = static_cast<double>(blocks) * threads * iters * ops_per_thread_iter;
  *gops = ops / (best_ms * 1e-3) / 1e9;
  return LABS_OK;
}
}  // namespace

extern "C" int labs_bench_imad_peak(labs_ctx* ctx, double* gmacs) {
  if (!ctx || !gmacs) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  return probe_rate(ctx, k_imad_peak, 16.0 * 8.0, gmacs);
}

extern "C" int labs_bench_int_peak(labs_ctx* ctx, double* gops) {
  if (!ctx || !gops) return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  return probe_rate(ctx, k_int_peak, 16.0 * 8.0, gops);
}

