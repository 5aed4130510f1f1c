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

// Pass 1: the minimum energy of every thread's block of Gray indices.
template <int KMAX>
__global__ void __launch_bounds__(128) k_exhaust_min(int n, int B, uint64_t blocks,
                                                     int* block_min) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= blocks) return;
  const uint64_t span = 1ULL << B;
  uint64_t s = gray_bits(t * span);
  int C[KMAX];
  int e = exh_build<KMAX>(s, n, C);
  int best = e;
  for (uint64_t l = 1; l < span; ++l) {
    e = exh_flip<KMAX>(s, n, __ffsll(static_cast<long long>(l)), C, e);
    best = e < best ? e : best;
  }
  block_min[t] = best;
}

// Pass 2, over the few blocks whose minimum is the optimum: record every
// sequence of those blocks with E == target.
template <int KMAX>
__global__ void __launch_bounds__(128) k_exhaust_collect(int n, int B, const uint32_t* ids,
                                                         int count, int target, uint64_t* out,
                                                         unsigned long long cap,
                                                         unsigned long long* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t span = 1ULL << B;
  uint64_t s = gray_bits(static_cast<uint64_t>(ids[i]) * span);
  int C[KMAX];
  int e = exh_build<KMAX>(s, n, C);
  for (uint64_t l = 0;; ++l) {
    if (e == target) {
      const unsigned long long slot = atomicAdd(cnt, 1ULL);
      if (slot < cap) out[slot] = s;
    }
    if (l + 1 == span) break;
    e = exh_flip<KMAX>(s, n, __ffsll(static_cast<long long>(l + 1)), C, e);
  }
}

// Strict local optima (every single flip strictly worse) of every block
// (proj/src/oracle.cpp:112-151).
template <int KMAX>
__global__ void __launch_bounds__(128) k_local_optima(int n, int B, uint64_t blocks,
                                                      unsigned long long* cnt) {
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= blocks) return;
  const uint64_t span = 1ULL << B;
  uint64_t s = gray_bits(t * span);
  int C[KMAX];
  int e = exh_build<KMAX>(s, n, C);
  unsigned long long local = 0;
  for (uint64_t l = 0;; ++l) {
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
    local += opt ? 1 : 0;
    if (l + 1 == span) break;
    e = exh_flip<KMAX>(s, n, __ffsll(static_cast<long long>(l + 1)), C, e);
  }
  (void)e;
  if (local) atomicAdd(cnt, local);
}

}  // namespace labsk
