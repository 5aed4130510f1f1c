// labs_rng.cuh — tile-uniform random streams for the MTS kernels.
//
// Every walker/replica is one tile of T lanes (T = 32: a whole warp; T = 16:
// half a warp, two replicas per warp). All lanes of a tile execute each draw
// together and obtain the same value (tile-uniform control flow), so no
// shuffles are needed to share a draw; bulk draws (mutation) hand draw i to
// tile lane i. Collective operations use the tile's lane mask, so a tile may
// draw (and refill its block) while the other tile of its warp does not.
//
// Two engines behind one interface:
//  * MtRngT    — reference-RNG mode. std::mt19937_64 with the state in shared
//               memory and libstdc++ 13's distribution algorithms, restated
//               so trajectories replay the reference bit for bit
//               (proj/include/labsolve/rng.hpp:10-28;
//               /usr/include/c++/13/bits/uniform_int_dist.h:255-281;
//               /usr/include/c++/13/bits/random.tcc:3346-3381).
//  * PhiloxRngT — production mode. Counter-based Philox4x32-10 keyed by
//               (seed, stream); draw d is half (d & 1) of block d >> 1. No
//               per-walker state beyond a 64-bit counter.
// Both streams are defined per draw index, independent of T.
#pragma once
#include <cstdint>

// Rare selection / draw paths of the tabu step (tie draw, fallback move,
// tenure outside the table) inline as cold blocks instead of out-of-line
// calls: no call-ABI register shuffling on the hot path, at the price of a
// larger loop body.
#ifndef LABS_RARE_INLINE
#define LABS_RARE_INLINE 0
#endif

namespace labsk {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMtN = 312;
constexpr int kMtM = 156;

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ------------------------------------------------------------- tiles -----
// A tile is T consecutive lanes (T in {8, 16, 32}); tile lane = lane % T.
template <int T>
__device__ __forceinline__ int tile_lane() {
  return T == 32 ? lane_id() : (lane_id() & (T - 1));
}
template <int T>
__device__ __forceinline__ int tile_base() {  // warp lane of tile lane 0
  return T == 32 ? 0 : (lane_id() & ~(T - 1));
}
template <int T>
__device__ __forceinline__ unsigned tile_mask() {
  return T == 32 ? kFull : (((1u << (T & 31)) - 1u) << tile_base<T>());
}
// The tile's bits of a warp-wide ballot, shifted down to bit 0.
template <int T>
__device__ __forceinline__ uint32_t tile_bits(uint32_t bal) {
  return T == 32 ? bal : ((bal >> tile_base<T>()) & ((1u << (T & 31)) - 1u));
}
// Ballot over the tile (divergence-safe: only the tile's lanes take part).
template <int T>
__device__ __forceinline__ uint32_t tile_ballot(bool p) {
  return tile_bits<T>(__ballot_sync(tile_mask<T>(), p));
}
template <int T>
__device__ __forceinline__ void tile_sync() {
  __syncwarp(tile_mask<T>());
}
// Divergence-safe tile reductions.
template <int T>
__device__ __forceinline__ int tile_sum(int v) {
  if constexpr (T == 32) {
    return __reduce_add_sync(kFull, v);
  } else {
#pragma unroll
    for (int o = T / 2; o; o >>= 1) v += __shfl_xor_sync(tile_mask<T>(), v, o);
    return v;
  }
}
template <int T>
__device__ __forceinline__ int tile_min(int v) {
  if constexpr (T == 32) {
    return __reduce_min_sync(kFull, v);
  } else {
#pragma unroll
    for (int o = T / 2; o; o >>= 1) v = min(v, __shfl_xor_sync(tile_mask<T>(), v, o));
    return v;
  }
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t a, uint64_t b, uint64_t c) {
  // a = mt[i], b = mt[i+1], c = mt[i +/- M]
  uint64_t x = (a & 0xFFFFFFFF80000000ULL) | (b & 0x7FFFFFFFULL);
  return c ^ (x >> 1) ^ ((x & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

// libstdc++ generate_canonical<double, 53> with one 64-bit draw.
__device__ __forceinline__ double u01_from_bits(uint64_t x) {
  double d = __dmul_rn(__ull2double_rn(x), 5.421010862427522170e-20);  // 2^-64
  if (d >= 1.0) d = 0.99999999999999988898;  // nextafter(1.0, 0.0)
  return d;
}

// ---------------------------------------------------------------- MtRng --
// State layout matches labs_rng_state (include/labs_b200.h): 312 words plus
// the index of the next output; idx == 312 means "twist before next draw",
// which is what a freshly seeded engine holds. Alongside the raw state the
// warp keeps the tempered outputs of the current block (`out`), produced by
// the twist, so a draw is one shared load.

// Warp-cooperative twist: regenerates mt[0..312) and tempers the new block
// into out[0..312). Reads of "old" words happen before any lane overwrites
// them (syncwarp between the read and write half of each chunk). Out of line
// and pointer-only so the caller's index stays in a register.
__device__ __forceinline__ uint64_t lds_u64(uint32_t saddr) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(saddr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u64(uint32_t saddr, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(saddr), "l"(v) : "memory");
}

__device__ __forceinline__ int32_t lds_s32(uint32_t saddr) {
  int32_t v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_s32(uint32_t saddr, int32_t v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t saddr) {
  uint16_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(saddr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_u8(uint32_t saddr, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(saddr), "h"(static_cast<uint16_t>(v)) : "memory");
}

// ------------------------------------------------------- tenure table --
// The tabu step's tenure draw, uniform_int(min_t, max_t) (tabu.cpp:49-50),
// is the only RNG draw on every step. In reference-RNG mode its Lemire
// reduction is precomputed for every draw of the current tempered block:
// byte i of the table (right after the block) holds min_t + draw_i * range
// >> 64 for the current walk's window, so a step's draw is one byte load
// while the engine index still advances by exactly one (the draw order, and
// so the trajectory, is unchanged). Entries whose reduction might reject
// (p mod 2^64 < range, probability ~2^-32) hold 0xFF and are never served
// from the table: tc_hi (the first such index, or the block end) bounds the
// fast path, and the slow path runs the full uniform_int. The table is
// rebuilt from the current index when a walk starts (new window) and for
// the whole block at every twist; windows with max_t > 254 are not cached.
constexpr uint32_t kTenOff = 8u * kMtN;          // table offset from the block
constexpr uint32_t kTenParOff = 8u * kMtN + kMtN;  // {min_t, range, window} (int32)

// Tenure entries are tabulated in windows (the tail of a block is usually
// not reached by the walk that tabulated it): the window length, set per
// walk from its step count, is the third parameter word.
constexpr int kTenWinMin = 64;

// Build table entries [lo, min(lo + window, kMtN)) from the tempered block;
// returns the first index >= lo that is not served from the table (a
// possibly-rejecting entry, or the window end).
template <int T>
__device__ __forceinline__ int mt_tenure_fill(uint32_t out, int lo) {
  const int min_t = lds_s32(out + kTenParOff);
  const uint32_t r32 = static_cast<uint32_t>(lds_s32(out + kTenParOff + 4));
  if (min_t + static_cast<int>(r32) - 1 > 254) return lo;
  const int win = lds_s32(out + kTenParOff + 8);
  const int hi = lo + win < kMtN ? lo + win : kMtN;
  int first = hi;
#pragma unroll 1
  for (int base = lo; base < hi; base += T) {
    const int i = base + tile_lane<T>();
    bool rej = false;
    if (i < hi) {
      const uint64_t x = lds_u64(out + 8u * static_cast<uint32_t>(i));
      const uint64_t p0 = static_cast<uint64_t>(static_cast<uint32_t>(x)) * r32;
      const uint64_t p1 =
          static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * r32 + (p0 >> 32);
      rej = static_cast<uint32_t>(p1) == 0 && static_cast<uint32_t>(p0) < r32;
      sts_u8(out + kTenOff + i, static_cast<uint32_t>(min_t) + static_cast<uint32_t>(p1 >> 32));
    }
    const uint32_t b = tile_ballot<T>(rej);
    if (b) {
      first = base + __ffs(b) - 1;
      break;
    }
  }
  return first;
}

template <int T>
__device__ __noinline__ int mt_tenure_window(uint32_t out, int lo) {
  return mt_tenure_fill<T>(out, lo);
}

template <int T>
__device__ __noinline__ int mt_tenure_table(uint32_t out, int lo, int min_t, uint32_t range,
                                            int steps) {
  if (tile_lane<T>() == 0) {
    sts_s32(out + kTenParOff, min_t);
    sts_s32(out + kTenParOff + 4, static_cast<int32_t>(range));
    // about one window per walk: its steps plus the expected tie draws
    const int w = (steps + steps / 8 + 8 + 31) & ~31;
    sts_s32(out + kTenParOff + 8, w < kTenWinMin ? kTenWinMin : (w > kMtN ? kMtN : w));
  }
  tile_sync<T>();
  return mt_tenure_fill<T>(out, lo);
}

// Twist, temper the new block, tabulate its first tenure window; returns
// tc_hi. Each lane's reads of a chunk are issued before its stores, and a
// warp's shared-memory accesses execute in order, so no lane overwrites a
// word another lane has yet to read (the tile is converged).
template <int T>
__device__ __noinline__ int mt_twist(uint32_t mt, uint32_t out) {
  const int lane = tile_lane<T>();
  // i in [0, 156): inputs mt[i], mt[i+1], mt[i+156], all old.
#pragma unroll 1
  for (int base = 0; base < kMtN - kMtM; base += T) {
    const uint32_t i = base + lane;
    if (i < kMtN - kMtM) {
      const uint64_t v =
          mt_mix(lds_u64(mt + 8 * i), lds_u64(mt + 8 * (i + 1)), lds_u64(mt + 8 * (i + kMtM)));
      sts_u64(mt + 8 * i, v);
      sts_u64(out + 8 * i, mt_temper(v));
    }
  }
  // i in [156, 311): inputs mt[i], mt[i+1] old, mt[i-156] new.
#pragma unroll 1
  for (int base = kMtN - kMtM; base < kMtN - 1; base += T) {
    const uint32_t i = base + lane;
    if (i < kMtN - 1) {
      const uint64_t v = mt_mix(lds_u64(mt + 8 * i), lds_u64(mt + 8 * (i + 1)),
                                lds_u64(mt + 8 * (i - (kMtN - kMtM))));
      sts_u64(mt + 8 * i, v);
      sts_u64(out + 8 * i, mt_temper(v));
    }
  }
  if (lane == 0) {
    const uint64_t v =
        mt_mix(lds_u64(mt + 8 * (kMtN - 1)), lds_u64(mt), lds_u64(mt + 8 * (kMtM - 1)));
    sts_u64(mt + 8 * (kMtN - 1), v);
    sts_u64(out + 8 * (kMtN - 1), mt_temper(v));
  }
  tile_sync<T>();
  return mt_tenure_fill<T>(out, 0);
}

// Temper the current block without advancing (after loading a state).
template <int T = 32>
__device__ __forceinline__ void mt_temper_all(const uint64_t* mt, uint64_t* out) {
  for (int i = tile_lane<T>(); i < kMtN; i += T) out[i] = mt_temper(mt[i]);
  tile_sync<T>();
}

template <int T>
struct MtRngT;
template <int T>
struct TenurePick;

template <int T>
struct MtRngT {
  uint32_t mt_s;   // shared-window address of the raw engine state
  uint32_t out_s;  // shared-window address of the tempered block (+ tenure table)
  int idx;         // tile-uniform
  int tc_hi;       // draws [idx, tc_hi) have their tenure in the table

  // The tempered block must be followed by the tenure table and its
  // parameters (kTenOff, kTenParOff): see TileSlot (labs_device.cuh).
  __device__ __forceinline__ void bind(uint64_t* raw, uint64_t* tempered, int i) {
    mt_s = static_cast<uint32_t>(__cvta_generic_to_shared(raw));
    out_s = static_cast<uint32_t>(__cvta_generic_to_shared(tempered));
    idx = i;
    tc_hi = 0;  // no window yet: begin_walk builds it
  }
  __device__ __forceinline__ uint64_t next() {
    if (idx >= kMtN) {
      tc_hi = mt_twist<T>(mt_s, out_s);
      idx = 0;
    }
    const uint64_t v = lds_u64(out_s + 8u * static_cast<uint32_t>(idx));
    ++idx;
    return v;
  }
  // Bulk: tile lane i (< count) receives draw i of the next `count` draws,
  // with count <= T and not crossing a twist (callers chunk on room()).
  __device__ __forceinline__ int room() {
    if (idx >= kMtN) {
      tc_hi = mt_twist<T>(mt_s, out_s);
      idx = 0;
    }
    return kMtN - idx;
  }
  // A walk's tenure window [min_t, min_t + range): tabulate the rest of the
  // block for it.
  __device__ __forceinline__ void begin_walk(int min_t, uint32_t range, int steps) {
    tc_hi = mt_tenure_table<T>(out_s, idx < kMtN ? idx : kMtN, min_t, range, steps);
  }
  // uniform_int(min_t, min_t + range - 1): one table byte, or the full draw.
  __device__ __forceinline__ int tenure();
  __device__ __forceinline__ uint64_t peek_lane(int i) const {
    return lds_u64(out_s + 8u * static_cast<uint32_t>(idx + i));
  }
  __device__ __forceinline__ void advance(int count) { idx += count; }
};
using MtRng = MtRngT<32>;

// ------------------------------------------------------------ PhiloxRng --
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0,
                                              uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
    uint32_t lo0 = 0xD2511F53u * c[0];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
    uint32_t lo1 = 0xCD9E8D57u * c[2];
    uint32_t n0 = hi1 ^ c[1] ^ k0;
    uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Draws are served from a per-tile block of 64 in shared memory: a refill
// has tile lane l compute Philox blocks base/2 + l + T q (q < 32/T), i.e.
// draws base + 2(l + T q) and base + 2(l + T q) + 1, so the 10-round cost is
// paid once per 64 draws and spread over the tile. The stream is defined per
// draw index d (block d >> 1, half d & 1), independent of the buffering.
//
// Shared layout after the 64-draw block (TileSlot, labs_device.cuh): the
// block's tenure table (64 bytes, as the MT table: min_t + Lemire reduction
// of each draw for the current walk's window, 0xFF where the reduction might
// reject), its parameters {min_t, range, -, -} and the key {k0, k1, s0, s1},
// so the generator itself is three registers (buffer, 64-bit counter) plus
// the count of table entries still valid from the counter on.
constexpr int kPhBlock = 64;
constexpr uint32_t kPhTabOff = 8u * kPhBlock;
constexpr uint32_t kPhParOff = kPhTabOff + kPhBlock;
constexpr uint32_t kPhKeyOff = kPhParOff + 16;

// Tabulate the tenure draw of block entries [lo, 64); returns the first
// entry >= lo not served from the table (64 when all are).
template <int T>
__device__ __forceinline__ int philox_tenure_fill(uint32_t buf, int lo) {
  const int min_t = lds_s32(buf + kPhParOff);
  const uint32_t r32 = static_cast<uint32_t>(lds_s32(buf + kPhParOff + 4));
  if (min_t + static_cast<int>(r32) - 1 > 254) return lo;
  int first = kPhBlock;
#pragma unroll
  for (int q = 0; q < kPhBlock / T; ++q) {
    const int i = tile_lane<T>() + T * q;
    bool rej = false;
    if (i >= lo) {
      const uint64_t x = lds_u64(buf + 8u * static_cast<uint32_t>(i));
      const uint64_t p0 = static_cast<uint64_t>(static_cast<uint32_t>(x)) * r32;
      const uint64_t p1 =
          static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * r32 + (p0 >> 32);
      rej = static_cast<uint32_t>(p1) == 0 && static_cast<uint32_t>(p0) < r32;
      sts_u8(buf + kPhTabOff + i, rej ? 0xFFu : static_cast<uint32_t>(min_t) +
                                                   static_cast<uint32_t>(p1 >> 32));
    }
    const uint32_t b = tile_ballot<T>(rej);
    if (b && first == kPhBlock) first = T * q + __ffs(b) - 1;
  }
  tile_sync<T>();
  return first;
}

// Refill the block holding draw `base` (a multiple of 64) and tabulate its
// tenures; returns the count of table entries valid from entry 0.
template <int T>
__device__ __noinline__ int philox_refill(uint32_t buf, uint64_t base) {
  const uint32_t k0 = static_cast<uint32_t>(lds_s32(buf + kPhKeyOff));
  const uint32_t k1 = static_cast<uint32_t>(lds_s32(buf + kPhKeyOff + 4));
  const uint32_t s0 = static_cast<uint32_t>(lds_s32(buf + kPhKeyOff + 8));
  const uint32_t s1 = static_cast<uint32_t>(lds_s32(buf + kPhKeyOff + 12));
#pragma unroll
  for (int q = 0; q < 32 / T; ++q) {
    const uint32_t rel = tile_lane<T>() + T * q;
    const uint64_t blk = (base >> 1) + static_cast<uint64_t>(rel);
    uint32_t c[4] = {static_cast<uint32_t>(blk), static_cast<uint32_t>(blk >> 32), s0, s1};
    philox4x32_10(c, k0, k1);
    sts_u64(buf + 16u * rel, static_cast<uint64_t>(c[1]) << 32 | c[0]);
    sts_u64(buf + 16u * rel + 8u, static_cast<uint64_t>(c[3]) << 32 | c[2]);
  }
  tile_sync<T>();
  return philox_tenure_fill<T>(buf, 0);
}

template <int T>
__device__ __noinline__ int philox_tenure_table(uint32_t buf, int lo, int min_t, uint32_t range) {
  if (tile_lane<T>() == 0) {
    sts_s32(buf + kPhParOff, min_t);
    sts_s32(buf + kPhParOff + 4, static_cast<int32_t>(range));
  }
  tile_sync<T>();
  return philox_tenure_fill<T>(buf, lo) - lo;
}

template <int T>
struct PhiloxRngT;
template <int T>
struct PhiloxTenure {
  int v;
  PhiloxRngT<T> rng;
};
template <int T>
__device__ __noinline__ PhiloxTenure<T> philox_tenure_slow(PhiloxRngT<T> r);

template <int T>
struct PhiloxRngT {
  static constexpr int kBlock = kPhBlock;
  uint32_t buf_s;  // shared-window address of the current 64-draw block
  uint64_t ctr;    // next draw index
  int t_rem;       // table entries valid from ctr on (<= 0: none)

  // Key and stream live in shared memory next to the block (tile-uniform
  // writes by lane 0; bind/set_stream order them before the next refill).
  __device__ __forceinline__ void set_key(uint64_t* buf, uint32_t k0, uint32_t k1, uint32_t s1) {
    buf_s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    if (tile_lane<T>() == 0) {
      sts_s32(buf_s + kPhKeyOff, static_cast<int32_t>(k0));
      sts_s32(buf_s + kPhKeyOff + 4, static_cast<int32_t>(k1));
      sts_s32(buf_s + kPhKeyOff + 12, static_cast<int32_t>(s1));
      sts_s32(buf_s + kPhParOff, 0);  // tenure window {0, 1} until a walk sets one
      sts_s32(buf_s + kPhParOff + 4, 1);
    }
    tile_sync<T>();
  }
  __device__ __forceinline__ void set_stream(uint32_t s0) {
    if (tile_lane<T>() == 0) sts_s32(buf_s + kPhKeyOff + 8, static_cast<int32_t>(s0));
    tile_sync<T>();
  }
  // Position at draw c and fill the block holding it (key and stream set).
  __device__ __forceinline__ void bind(uint64_t c) {
    ctr = c;
    const int valid = philox_refill<T>(buf_s, ctr & ~static_cast<uint64_t>(kBlock - 1));
    t_rem = valid - static_cast<int>(static_cast<uint32_t>(ctr) & (kBlock - 1));
  }
  __device__ __forceinline__ uint64_t next() {
    const uint32_t off = static_cast<uint32_t>(ctr) & (kBlock - 1);
    if (off == 0) t_rem = philox_refill<T>(buf_s, ctr);
    const uint64_t v = lds_u64(buf_s + 8u * off);
    ++ctr;
    --t_rem;
    return v;
  }
  __device__ __forceinline__ int room() {
    const uint32_t off = static_cast<uint32_t>(ctr) & (kBlock - 1);
    if (off == 0) t_rem = philox_refill<T>(buf_s, ctr);
    return kBlock - static_cast<int>(off);
  }
  __device__ __forceinline__ uint64_t peek_lane(int i) const {
    return lds_u64(buf_s + 8u * ((static_cast<uint32_t>(ctr) & (kBlock - 1)) + i));
  }
  __device__ __forceinline__ void advance(int count) {
    // crossing into a new block mid-way is impossible: count <= room()
    ctr += static_cast<uint64_t>(count);
    t_rem -= count;
  }
  // A walk's tenure window: tabulate the rest of the current block for it
  // (a block not yet filled is tabulated by its refill).
  __device__ __forceinline__ void begin_walk(int min_t, uint32_t range, int /*steps*/) {
    const int off = static_cast<int>(static_cast<uint32_t>(ctr) & (kBlock - 1));
    t_rem = philox_tenure_table<T>(buf_s, off == 0 ? kBlock : off, min_t, range);
  }
  __device__ __forceinline__ int tenure() {
    if (t_rem > 0) {
      const uint32_t off = static_cast<uint32_t>(ctr) & (kBlock - 1);
      const int v = static_cast<int>(lds_u8(buf_s + kPhTabOff + off));
      ++ctr;
      --t_rem;
      return v;
    }
    const PhiloxTenure<T> p = philox_tenure_slow<T>(*this);
    *this = p.rng;
    return p.v;
  }
};
using PhiloxRng = PhiloxRngT<32>;

// ---------------------------------------------------- distributions -------
// uniform_int_distribution<long long>(lo, hi) over a 64-bit engine: Lemire's
// nearly-divisionless method on the 128-bit product; at least one draw.
template <class R>
__device__ __forceinline__ long long uniform_int(R& rng, long long lo,
                                                 long long hi) {
  const uint64_t range =
      static_cast<uint64_t>(hi) - static_cast<uint64_t>(lo) + 1ULL;
  uint64_t x = rng.next();
  if (range >> 32 == 0) {
    // 64 x 32-bit product in two wide multiplies: low 64 bits and the
    // high word (the result), same arithmetic as the 128-bit product.
    const uint32_t r32 = static_cast<uint32_t>(range);
    uint64_t p0 = static_cast<uint64_t>(static_cast<uint32_t>(x)) * r32;
    uint64_t p1 = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * r32 + (p0 >> 32);
    if (static_cast<uint32_t>(p1) == 0 && static_cast<uint32_t>(p0) < r32) {
      const uint64_t thr = (0ULL - range) % range;
      uint64_t low = (p1 << 32) | static_cast<uint32_t>(p0);
      while (low < thr) {
        x = rng.next();
        p0 = static_cast<uint64_t>(static_cast<uint32_t>(x)) * r32;
        p1 = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * r32 + (p0 >> 32);
        low = (p1 << 32) | static_cast<uint32_t>(p0);
      }
    }
    return static_cast<long long>(static_cast<uint64_t>(lo) + (p1 >> 32));
  }
  uint64_t low = x * range;
  if (low < range) {
    const uint64_t thr = (0ULL - range) % range;
    while (low < thr) {
      x = rng.next();
      low = x * range;
    }
  }
  return static_cast<long long>(static_cast<uint64_t>(lo) + __umul64hi(x, range));
}

// Rejection tail of uniform_below (taken with probability < 2^-32 per
// draw), kept out of line so the tabu step's code stays compact (the L0
// instruction cache is ~6 KB per SM sub-partition).
template <class R>
struct DrawTail {
  uint32_t v;
  R rng;
};
template <class R>
__device__ __noinline__ DrawTail<R> uniform_below_tail(R rng, uint32_t r32, uint64_t p0,
                                                       uint64_t p1) {
  const uint64_t range = r32;
  const uint64_t thr = (0ULL - range) % range;
  uint64_t low = (p1 << 32) | static_cast<uint32_t>(p0);
  while (low < thr) {
    const uint64_t x = rng.next();
    p0 = static_cast<uint64_t>(static_cast<uint32_t>(x)) * r32;
    p1 = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * r32 + (p0 >> 32);
    low = (p1 << 32) | static_cast<uint32_t>(p0);
  }
  return {static_cast<uint32_t>(p1 >> 32), rng};
}

// Tenure draw outside the table (block end, a possibly-rejecting entry, or
// an uncached window): the full uniform_int, then the next table bound.
template <int T>
struct TenurePick {
  int v;
  MtRngT<T> rng;
};
template <int T>
__device__ __noinline__ TenurePick<T> mt_tenure_slow(MtRngT<T> r);
template <int T>
__device__ __forceinline__ TenurePick<T> mt_tenure_slow_body(MtRngT<T> r);

template <int T>
__device__ __forceinline__ int MtRngT<T>::tenure() {
  if (idx < tc_hi) {
    const int v = static_cast<int>(lds_u8(out_s + kTenOff + static_cast<uint32_t>(idx)));
    ++idx;
    return v;
  }
#if LABS_RARE_INLINE
  const TenurePick<T> p = mt_tenure_slow_body<T>(*this);
  *this = p.rng;
  return p.v;
#else
  const TenurePick<T> p = mt_tenure_slow<T>(*this);
  *this = p.rng;
  return p.v;
#endif
}

// uniform_int(0, r - 1) for a known 32-bit range r >= 1: the same Lemire
// arithmetic (and draw count) as uniform_int, without the range dispatch.
template <class R>
__device__ __forceinline__ int uniform_below(R& rng, uint32_t r32) {
  const uint64_t x = rng.next();
  const uint64_t p0 = static_cast<uint64_t>(static_cast<uint32_t>(x)) * r32;
  const uint64_t p1 = static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * r32 + (p0 >> 32);
  // low 64 bits of x * r below r needs the middle word to be zero: ~2^-32.
  if (__builtin_expect(static_cast<uint32_t>(p1) == 0, 0) && static_cast<uint32_t>(p0) < r32) {
    const DrawTail<R> d = uniform_below_tail(rng, r32, p0, p1);
    rng = d.rng;
    return static_cast<int>(d.v);
  }
  return static_cast<int>(p1 >> 32);
}

// Tenure outside the table: at a block start refill (which tabulates the
// block); a possibly-rejecting entry takes the full uniform_int, after which
// the rest of the block is re-tabulated.
template <int T>
__device__ __noinline__ PhiloxTenure<T> philox_tenure_slow(PhiloxRngT<T> r) {
  uint32_t off = static_cast<uint32_t>(r.ctr) & (kPhBlock - 1);
  if (off == 0) r.t_rem = philox_refill<T>(r.buf_s, r.ctr);
  if (r.t_rem > 0) {
    const int v = static_cast<int>(lds_u8(r.buf_s + kPhTabOff + off));
    ++r.ctr;
    --r.t_rem;
    return {v, r};
  }
  const int min_t = lds_s32(r.buf_s + kPhParOff);
  const uint32_t range = static_cast<uint32_t>(lds_s32(r.buf_s + kPhParOff + 4));
  const int v = min_t + uniform_below(r, range);
  off = static_cast<uint32_t>(r.ctr) & (kPhBlock - 1);
  r.t_rem = off == 0 ? 0 : philox_tenure_fill<T>(r.buf_s, static_cast<int>(off)) -
                               static_cast<int>(off);
  return {v, r};
}

// Outside the tabulated window: at the block end twist (which tabulates the
// new block's first window), at a window end tabulate the next window; a
// possibly-rejecting entry takes the full uniform_int.
template <int T>
__device__ __forceinline__ TenurePick<T> mt_tenure_slow_body(MtRngT<T> r) {
  if (r.idx >= kMtN) {
    r.tc_hi = mt_twist<T>(r.mt_s, r.out_s);
    r.idx = 0;
  }
  if (r.idx >= r.tc_hi) r.tc_hi = mt_tenure_window<T>(r.out_s, r.idx);
  if (r.idx < r.tc_hi) {
    const int v = static_cast<int>(lds_u8(r.out_s + kTenOff + static_cast<uint32_t>(r.idx)));
    ++r.idx;
    return {v, r};
  }
  const int min_t = lds_s32(r.out_s + kTenParOff);
  const uint32_t range = static_cast<uint32_t>(lds_s32(r.out_s + kTenParOff + 4));
  const int v = min_t + uniform_below(r, range);
  r.tc_hi = r.idx < kMtN ? mt_tenure_window<T>(r.out_s, r.idx) : r.idx;
  return {v, r};
}

template <int T>
__device__ __noinline__ TenurePick<T> mt_tenure_slow(MtRngT<T> r) {
  return mt_tenure_slow_body<T>(r);
}

template <class R>
__device__ __forceinline__ double uniform01(R& rng) {
  return u01_from_bits(rng.next());
}

}  // namespace labsk
