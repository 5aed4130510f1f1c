// labs_ns.cu — launchers of the NS-templated kernels K1..K4 for one
// NS = ceil(n/32), compiled once per NS (-DLABS_NS=1..8; Makefile) so the
// instantiation sets build in parallel. Declarations: labs_host.cuh.
#include <cuda_runtime.h>

#include "labs_host.cuh"

#ifndef LABS_NS
#error "compile with -DLABS_NS=<1..8>"
#endif

namespace labsh {

namespace {

template <int NS, int T, bool MT>
constexpr size_t memetic_smem() {
  return (32 / T) * kWarps * tile_slot_bytes<T * NS, MT>();
}

template <class Kern, class... Args>
int launch(labs_ctx* ctx, Kern kern, size_t smem, int items, int per_block, Args... args) {
  if (int r = prep(kern, smem)) return r;
  int grid = 0;
  if (int r = grid_for(ctx, kern, smem, items, &grid, per_block)) return r;
  kern<<<grid, 32 * kWarps, smem, ctx->stream>>>(args...);
  LABS_CUDA(cudaGetLastError());
  return LABS_OK;
}

}  // namespace

template <int NS>
int NsOps<NS>::build(labs_ctx* ctx, int n, int count, const uint64_t* dw, int32_t* dc,
                     int64_t* de, int64_t* dn) {
  return launch(ctx, k_build<NS>, kWarps * slot_bytes<NS, false>(), count, kWarps, n, count, dw,
                dc, de, dn);
}

template <int NS>
int NsOps<NS>::flip_trace(labs_ctx* ctx, int n, int count, const uint64_t* dw, int flips,
                          const int32_t* dp, int64_t* de, int64_t* dn) {
  return launch(ctx, k_flip_trace<NS>, kWarps * slot_bytes<NS, false>(), count, kWarps, n, count,
                dw, flips, dp, de, dn);
}

template <int NS>
int NsOps<NS>::scan(labs_ctx* ctx, int n, int count, const uint64_t* dw, const uint8_t* da,
                    labs_rng_state* dr, int allow_fallback, int tie_rule, int32_t* dpos,
                    int64_t* de, int32_t* dfb, int32_t* dnt, uint64_t* dtm) {
  return launch(ctx, k_scan<NS>, kWarps * slot_bytes<NS, true>(), count, kWarps, n, count, dw, da,
                dr, allow_fallback, tie_rule, dpos, de, dfb, dnt, dtm);
}

template <int NS>
int NsOps<NS>::tabu(labs_ctx* ctx, WalkArgs& A, bool mt) {
  if (mt) return launch(ctx, k_tabu<NS, true>, kWarps * slot_bytes<NS, true>(), A.count, kWarps, A);
  return launch(ctx, k_tabu<NS, false>, kWarps * slot_bytes<NS, false>(), A.count, kWarps, A);
}

template <int NS, int T>
int MemeticOps<NS, T>::launch(labs_ctx* ctx, const MemeticArgs& A, bool mt) {
  constexpr int per_block = kWarps * (32 / T);
  if (mt)
    return labsh::launch(ctx, k_memetic<NS, T, true>, memetic_smem<NS, T, true>(), A.replicas,
                         per_block, A);
  return labsh::launch(ctx, k_memetic<NS, T, false>, memetic_smem<NS, T, false>(), A.replicas,
                       per_block, A);
}

template <int NS, int T>
int MemeticOps<NS, T>::blocks_per_sm(labs_ctx* ctx, bool mt, int* per_sm) {
  LABS_CUDA(cudaSetDevice(ctx->device));
  *per_sm = 0;
  if (mt) {
    if (int r = prep(k_memetic<NS, T, true>, memetic_smem<NS, T, true>())) return r;
    LABS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        per_sm, k_memetic<NS, T, true>, 32 * kWarps, memetic_smem<NS, T, true>()));
  } else {
    if (int r = prep(k_memetic<NS, T, false>, memetic_smem<NS, T, false>())) return r;
    LABS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        per_sm, k_memetic<NS, T, false>, 32 * kWarps, memetic_smem<NS, T, false>()));
  }
  return LABS_OK;
}

template struct NsOps<LABS_NS>;
template struct MemeticOps<LABS_NS, 32>;
#if LABS_NS == 2 || LABS_NS == 4
template struct MemeticOps<LABS_NS, 16>;  // LABS_TILE=16: two replicas per warp (n <= 64)
#endif

}  // namespace labsh
