// labs_device.cuh — the sm_100a kernel templates K1..K4 (one warp per
// walker / replica) shared by the per-NS translation units (labs_ns.cu is
// compiled once per NS = ceil(n/32), so the eight instantiation sets build in
// parallel).
//
// Every kernel is warp-per-walker (or warp-per-replica): 4 independent warps
// per 128-thread block, no block-level barriers, each warp with a private
// slice of dynamic shared memory (WalkSmem + optional mt19937_64 state).
// Kernels are templated on NS = ceil(n/32) so the per-slot register arrays
// are fully unrolled; the host dispatches NS in [1, 8] (n <= 256).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "labs_b200.h"
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
#ifndef LABS_MINB_TINY
#define LABS_MINB_TINY 7
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
  uint8_t tenure[MT ? kMtN : PhiloxRng::kBlock];  // tenure table of the block (labs_rng.cuh)
  // {min_t, range, table window (MT), pad} and, for Philox, {k0, k1, s0, s1}
  int32_t tenure_par[MT ? 4 : 8];
  TileCtl ctl;
  WalkSmemL<L> walk;
};
using TileSlotPh64 = TileSlot<64, false>;
static_assert(offsetof(TileSlotPh64, tenure) - offsetof(TileSlotPh64, out) == kPhTabOff &&
                  offsetof(TileSlotPh64, tenure_par) - offsetof(TileSlotPh64, out) == kPhParOff &&
                  offsetof(TileSlotPh64, tenure_par) + 16 - offsetof(TileSlotPh64, out) ==
                      kPhKeyOff,
              "the Philox table, parameters and key must follow the block");
using TileSlotMt64 = TileSlot<64, true>;
static_assert(offsetof(TileSlotMt64, tenure) - offsetof(TileSlotMt64, out) == kTenOff &&
                  offsetof(TileSlotMt64, tenure_par) - offsetof(TileSlotMt64, out) == kTenParOff,
              "the tenure table must follow the tempered block");

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
  if (tile_lane<T>() == 0) {  // tenure window {0, 1} until a walk sets one
    int32_t* par = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(out) + kTenParOff);
    par[0] = 0;
    par[1] = 1;
    par[2] = kTenWinMin;
  }
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
        corr[static_cast<size_t>(item) * (n - 1) + j - 1] = w.CK[b] / Walker<NS>::Sc::kC;
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
      rng.set_key(sl.out, static_cast<uint32_t>(A.seed), static_cast<uint32_t>(A.seed >> 32),
                  0x4C414253u);  // "LABS"
      rng.set_stream(static_cast<uint32_t>(item));
      rng.bind(A.ctr_base);
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
    rng.set_stream(static_cast<uint32_t>(offset + r));
    rng.bind(ctr[r]);
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
  // n <= 64 (one warp per replica): 7 blocks = 28 warps per SM, which the
  // shared memory allows (7.9 KB per replica) and which caps registers at 72.
  return T * NS <= 64 && T == 32 ? LABS_MINB_TINY
                                 : (T * NS <= 128 ? LABS_MINB_SMALL : LABS_MINB_LARGE);
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
    rng.set_key(sl.out, static_cast<uint32_t>(A.base_seed),
                static_cast<uint32_t>(A.base_seed >> 32), 0x4D454D45u);  // "MEME"
    rng.set_stream(0);
    rng.bind(0);  // valid until a replica is loaded
    PhiloxBind<T> rb{A.ctr, sl.out, A.replica_offset};
    run_policy<NS, T>(A, w, rng, rb, sl.ctl);
  }
}


}  // namespace labsk
