// labs_exhaust.cu — K5, the device exhaustive Gray-code oracle
// (labs_exhaustive.cuh) and its C ABI (include/labs_b200.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "labs_exhaustive.cuh"
#include "labs_host.cuh"

using namespace labsk;
using namespace labsh;

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
