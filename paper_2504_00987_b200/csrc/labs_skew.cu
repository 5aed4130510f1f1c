// labs_skew.cu — K6, the skew-symmetry deviation d(S) on the device
// (proj/src/skew.cpp:110-187) and its C ABI.
//
// The reference evaluates violating-pair counts of edited rotations one by
// one, stops right after the first zero and charges a budget before every
// evaluation. Here every evaluation of the reference's order is indexed
// (rotation-major, exactly as its nested loops visit them) and computed by
// its own thread; the sequential semantics are then recovered exactly:
//   want = first zero index + 1 (+1 where the reference's loop has no exit
//          test between two evaluations), or all evaluations
//   P = min(want, budget (if any));  value = min over [0, P); evaluations = P
//   budget_exceeded = budget < want (a charge was attempted past the budget;
//   a zero at index budget-1 ends the loops without another charge).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "labs_host.cuh"

namespace {

enum SkewMode { kDevOdd = 0, kDevEven = 1, kEditOdd = 2, kEditEven = 3 };

// Evaluations per rotation in the reference's loop order.
__host__ __device__ inline uint64_t per_rotation(int mode, int n) {
  const uint64_t g = 2ull * static_cast<uint64_t>(n + 1);  // (gap, spin) pairs
  switch (mode) {
    case kDevOdd: return 1;
    case kDevEven: return static_cast<uint64_t>(n);
    case kEditOdd: return 1 + g * static_cast<uint64_t>(n + 1);
    default: return static_cast<uint64_t>(n) + g;
  }
}

// Violating mirror pairs of the odd logical length `len` read through `at`
// (pair i violates when s[c+i] != (-1)^i s[c-i], c = (len-1)/2).
template <class At>
__device__ __forceinline__ int violations(int len, At at) {
  const int c = (len - 1) / 2;
  int bad = 0;
  for (int i = 1; i <= c; ++i) {
    const int want = (i & 1) ? -at(c - i) : at(c - i);
    bad += at(c + i) != want;
  }
  return bad;
}

// Evaluation `idx`: decode (rotation, edit) and count its violating pairs.
__device__ int skew_eval(const int8_t* s, int n, int mode, uint64_t idx) {
  const uint64_t per = per_rotation(mode, n);
  const int r = static_cast<int>(idx / per);
  uint64_t k = idx % per;
  auto rot = [&](int i) -> int {
    const int x = i + r;
    return s[x < n ? x : x - n];
  };
  if (mode == kDevOdd) return violations(n, rot);
  if (mode == kDevEven || (mode == kEditEven && k < static_cast<uint64_t>(n))) {
    const int skip = static_cast<int>(k);  // rotation with one deletion
    return violations(n - 1, [&](int i) { return rot(i < skip ? i : i + 1); });
  }
  if (mode == kEditOdd) {
    if (k == 0) return violations(n, rot);
    k -= 1;
    const uint64_t inner = 2ull * static_cast<uint64_t>(n + 1);
    const int gap = static_cast<int>(k / inner);
    const uint64_t rem = k % inner;
    const int spin = rem < static_cast<uint64_t>(n + 1) ? 1 : -1;
    const int skip = static_cast<int>(rem % static_cast<uint64_t>(n + 1));
    // insertion before `gap`, then deletion of physical index `skip`
    auto grown = [&](int i) { return i == gap ? spin : rot(i < gap ? i : i - 1); };
    return violations(n, [&](int i) { return grown(i < skip ? i : i + 1); });
  }
  k -= static_cast<uint64_t>(n);  // kEditEven: one insertion
  const int gap = static_cast<int>(k / 2);
  const int spin = (k & 1) ? -1 : 1;
  return violations(n + 1, [&](int i) { return i == gap ? spin : rot(i < gap ? i : i - 1); });
}

__device__ __forceinline__ void load_spins(int8_t* s, const uint64_t* words, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    s[i] = ((words[i >> 6] >> (i & 63)) & 1ull) ? -1 : 1;
  __syncthreads();
}

__global__ void __launch_bounds__(256) k_skew_eval(int n, int mode, const uint64_t* words,
                                                    uint64_t total, uint8_t* out,
                                                    unsigned long long* first_zero) {
  __shared__ int8_t s[LABS_MAX_N + 8];
  load_spins(s, words, n);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  unsigned long long zero = ~0ull;
  for (uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       idx < total; idx += stride) {
    const int v = skew_eval(s, n, mode, idx);
    out[idx] = static_cast<uint8_t>(v);
    if (v == 0 && idx < zero) zero = idx;
  }
  if (zero != ~0ull) atomicMin(first_zero, zero);
}

__global__ void __launch_bounds__(256) k_skew_min(const uint8_t* vals, uint64_t prefix,
                                                   int* min_out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  int m = INT_MAX;
  for (uint64_t idx = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
       idx < prefix; idx += stride)
    m = min(m, static_cast<int>(vals[idx]));
  m = __reduce_min_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && m != INT_MAX) atomicMin(min_out, m);
}

}  // namespace

using namespace labsh;

extern "C" int labs_skew_deviation(labs_ctx* ctx, int n, const uint64_t* words, int with_edits,
                                   uint64_t budget, int32_t* value, int32_t* budget_exceeded,
                                   uint64_t* evaluations) {
  if (!ctx || !words || !value || !budget_exceeded || !evaluations)
    return fail(LABS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n < 3) return fail(LABS_ERR_INVALID_ARGUMENT, "deviation needs length >= 3");
  if (n > LABS_MAX_N)
    return fail(LABS_ERR_INVALID_ARGUMENT, "length exceeds the device limit");
  if (int rc = check_seq_padding(n, 1, words)) return rc;
  LABS_CUDA(cudaSetDevice(ctx->device));
  const int mode = (with_edits ? 2 : 0) + (n % 2 == 0 ? 1 : 0);
  const uint64_t total = per_rotation(mode, n) * static_cast<uint64_t>(n);
  DBuf dw, dv, dz, dm;
  const int nw = nw_of(n);
  LABS_ALLOC(dw, sizeof(uint64_t) * nw);
  LABS_ALLOC(dv, total);
  LABS_ALLOC(dz, sizeof(unsigned long long));
  LABS_ALLOC(dm, sizeof(int));
  LABS_H2D(dw.p, words, sizeof(uint64_t) * nw);
  LABS_CUDA(cudaMemsetAsync(dz.p, 0xff, sizeof(unsigned long long), ctx->stream));
  const int big = INT_MAX;
  LABS_H2D(dm.p, &big, sizeof(int));
  const uint64_t blocks = (total + 255) / 256;
  const unsigned grid = static_cast<unsigned>(
      blocks < static_cast<uint64_t>(ctx->sm_count) * 16 ? blocks : ctx->sm_count * 16);
  k_skew_eval<<<grid, 256, 0, ctx->stream>>>(n, mode, dw.as<uint64_t>(), total,
                                             dv.as<uint8_t>(), dz.as<unsigned long long>());
  LABS_CUDA(cudaGetLastError());
  unsigned long long zero = 0;
  LABS_D2H(&zero, dz.p, sizeof(zero));
  LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  // Evaluations the reference's loops want: up to the first zero, except
  // that its insertion loop of even lengths with edits has no early-exit
  // test between the two spins (skew.cpp:172-179), so a zero at spin +1
  // still charges and evaluates spin -1.
  uint64_t want = total;
  if (zero != ~0ull) {
    want = zero + 1;
    if (mode == kEditEven) {
      const uint64_t k = zero % per_rotation(mode, n);
      if (k >= static_cast<uint64_t>(n) && ((k - n) & 1) == 0) want += 1;
    }
  }
  uint64_t prefix = want;
  if (budget && budget < prefix) prefix = budget;
  int m = INT_MAX;
  if (prefix) {
    k_skew_min<<<grid, 256, 0, ctx->stream>>>(dv.as<uint8_t>(), prefix, dm.as<int>());
    LABS_CUDA(cudaGetLastError());
    LABS_D2H(&m, dm.p, sizeof(int));
    LABS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  *value = prefix ? m : -1;
  *evaluations = prefix;
  *budget_exceeded = (budget && budget < want) ? 1 : 0;  // a charge past the budget
  return LABS_OK;
}
