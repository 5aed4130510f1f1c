// labs_exhaustive.cuh — exhaustive ground truth on the device (K5).
//
// Restates the reference's Gray-code oracle (proj/src/oracle.cpp:23-151):
// position 0 is fixed to +1 (complement symmetry) and positions 1..n-1 walk
// the reflected Gray code of an index g in [0, 2^(n-1)). Thread t owns the
// block of indices [t*2^B, (t+1)*2^B): inside a block the low B bits follow
// the Gray code of the block offset, so every thread of a warp flips the same
// position ctz(l)+1 at step l (uniform control flow) while their high bits
// differ. Each thread keeps its C_k in registers and updates them in O(n) per
// flip (C_k -= 2 s_j (s_{j-k} + s_{j+k}); E += dC (2 C_k + dC)), with n <= 64
// so a sequence is one 64-bit register.
#pragma once
#include <cstdint>

namespace labsk {

// bits of gray(g) placed on positions 1..n-1 (position 0 stays +1).
__device__ __forceinline__ uint64_t gray_bits(uint64_t g) {
  return (g ^ (g >> 1)) << 1;
}

// C_k (k = 1..n-1) and E of a packed sequence, from scratch (popcounts).
template <int KMAX>
__device__ __forceinline__ int exh_build(uint64_t s, int n, int (&C)[KMAX]) {
  const uint64_t all = n == 64 ? ~0ULL : ((1ULL << n) - 1ULL);
  int e = 0;
#pragma unroll
  for (int k = 1; k < KMAX; ++k) {
    int c = 0;
    if (k < n) {
      const uint64_t valid = all >> k;  // i in [0, n-k)
      c = (n - k) - 2 * __popcll((s ^ (s >> k)) & valid);
    }
    C[k] = c;
    e += c * c;
  }
  return e;
}

// Flip position j (uniform across the warp) and return the new energy.
template <int KMAX>
__device__ __forceinline__ int exh_flip(uint64_t& s, int n, int j, int (&C)[KMAX], int e) {
  const int sj = ((s >> j) & 1ULL) ? -1 : 1;
  // bit k-1 of up = position j+k; bit k-1 of dn = position j-k.
  const uint64_t up = j + 1 < 64 ? (s >> (j + 1)) & ((1ULL << (n - 1 - j)) - 1ULL) : 0ULL;
  const uint64_t dn = (__brevll(s) >> (64 - j)) & ((1ULL << j) - 1ULL);
  const int m2s = -2 * sj;
#pragma unroll
  for (int k = 1; k < KMAX; ++k) {
    if (k < n) {
      const int cnt = (k <= n - 1 - j) + (k <= j);
      const int neg = static_cast<int>((up >> (k - 1)) & 1ULL) + static_cast<int>((dn >> (k - 1)) & 1ULL);
      const int d = m2s * (cnt - 2 * neg);  // dC_k = -2 s_j (s_{j-k} + s_{j+k})
      e += d * (2 * C[k] + d);
      C[k] += d;
    }
  }
  s ^= 1ULL << j;
  return e;
}

// Mode 0: per-thread minimum -> atomicMin(best). Mode 1: record every
// sequence with E == *target (s_0 = +1 half) into out[0..cap), count in *cnt.
// Mode 2: count strict local optima (every single flip strictly worse).
template <int KMAX>
__global__ void __launch_bounds__(128) k_exhaust(int n, int B, uint64_t blocks, int mode,
                                                 unsigned long long* best, const int* target,
                                                 uint64_t* out, unsigned long long cap,
                                                 unsigned long long* cnt) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= blocks) return;
  const uint64_t span = 1ULL << B;
  uint64_t s = gray_bits(t * span);
  int C[KMAX];
  int e = exh_build<KMAX>(s, n, C);
  int local_min = e;
  unsigned long long local_cnt = 0;
  const int tgt = mode == 1 ? *target : 0;
  for (uint64_t l = 0;; ++l) {
    if (mode == 0) {
      local_min = e < local_min ? e : local_min;
    } else if (mode == 1) {
      if (e == tgt) {
        const unsigned long long slot = atomicAdd(cnt, 1ULL);
        if (slot < cap) out[slot] = s;
      }
    } else {
      // strict local optimum: dE_j > 0 for every j (proj/src/oracle.cpp:119-129)
      bool opt = true;
      for (int j = 0; j < n && opt; ++j) {
        const int sj = ((s >> j) & 1ULL) ? -1 : 1;
        int de = 0;
#pragma unroll
        for (int k = 1; k < KMAX; ++k) {
          if (k < n) {
            int d = 0;
            if (j - k >= 0) d += ((s >> (j - k)) & 1ULL) ? -1 : 1;
            if (j + k < n) d += ((s >> (j + k)) & 1ULL) ? -1 : 1;
            d *= -2 * sj;
            de += d * (2 * C[k] + d);
          }
        }
        opt = de > 0;
      }
      local_cnt += opt ? 1 : 0;
    }
    if (l + 1 == span) break;
    e = exh_flip<KMAX>(s, n, __ffsll(static_cast<long long>(l + 1)), C, e);
  }
  if (mode == 0) {
    atomicMin(best, static_cast<unsigned long long>(local_min));
  } else if (mode == 2) {
    if (local_cnt) atomicAdd(cnt, local_cnt);
  }
}

}  // namespace labsk
