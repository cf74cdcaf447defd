// polymul.cuh -- the kernels around poly_mul (polymul.hpp:48-95) that are not
// transforms or ring products: the prime ring's pointwise products, the
// support scan (poly_support, polymul.hpp:26-30), Schoenhage-Strassen
// packing of Z[x] coefficients into Z/(2^N+1) elements, and
// the Nussbaumer reshapes x^(j + s k) <-> z^j y^k with the recombination
// h_j = C_j + y C_{j+s}.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace polymul {

// a[i] <- a[i] * b[i] * c mod p (prime ring elements: one u64 in [0, p))
__device__ __forceinline__ u64 mulmod_p(u64 a, u64 b, u64 p) {
  return (u64)(((unsigned __int128)a * b) % p);
}
__global__ void prime_pointwise_kernel(std::uint8_t* a, const std::uint8_t* b, u64 stride, u64 count, u64 p,
                                       u64 c) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x) {
    u64* pa = reinterpret_cast<u64*>(a + i * stride);
    const u64 x = mulmod_p(*pa, *reinterpret_cast<const u64*>(b + i * stride), p);
    *pa = c == 1 ? x : mulmod_p(x, c, p);
  }
}

// poly_support: 1 + the index of the last element with a nonzero word
// (elem_words u64 words per element), 0 for the zero polynomial.  One warp
// per element, atomicMax into *out (initialised to 0).
__global__ void support_kernel(const std::uint8_t* a, u64 stride, u64 len, u32 elem_words,
                               unsigned long long* out) {
  const u32 lane = threadIdx.x & 31;
  const u64 wpb = blockDim.x >> 5;
  for (u64 e = blockIdx.x * wpb + (threadIdx.x >> 5); e < len; e += (u64)gridDim.x * wpb) {
    const u64* w = reinterpret_cast<const u64*>(a + e * stride);
    u64 any = 0;
    for (u32 k = lane; k < elem_words; k += 32) any |= w[k];
    if (__any_sync(0xffffffffu, any != 0) && lane == 0) atomicMax(out, (unsigned long long)(e + 1));
  }
}

// Schoenhage-Strassen packing: element i of dst (D32 u32 words + the top
// word) takes the src_words u64 limbs of coefficient i, zero-extended; one
// CTA per element.
__global__ void pack_limbs_kernel(std::uint8_t* dst, u64 dst_stride, const std::uint8_t* src, u64 src_words,
                                  u32 elem_words) {
  u64* d = reinterpret_cast<u64*>(dst + (u64)blockIdx.x * dst_stride);
  const u64* s = reinterpret_cast<const u64*>(src + (u64)blockIdx.x * src_words * 8);
  for (u32 k = threadIdx.x; k < elem_words; k += blockDim.x) d[k] = k < src_words ? s[k] : 0ull;
}

// Nussbaumer split: f (K s residues, f[j + s k]) -> elements A_j (K words,
// word k = f[j + s k]) for j < s: a [K][s] -> [s][K] transpose through a
// 32 x 33 shared tile (coalesced on both sides).
__global__ void nuss_split_kernel(std::uint8_t* dst, u64 dst_stride, const u64* f, u32 K, u32 s) {
  __shared__ u64 tile[32][33];
  const u32 j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const u32 tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (u32 r = ty; r < 32; r += 8) {
    const u32 k = k0 + r, j = j0 + tx;
    if (k < K && j < s) tile[r][tx] = f[(u64)k * s + j];
  }
  __syncthreads();
  for (u32 r = ty; r < 32; r += 8) {
    const u32 j = j0 + r, k = k0 + tx;
    if (j < s && k < K) reinterpret_cast<u64*>(dst + (u64)j * dst_stride)[k] = tile[tx][r];
  }
}

// Nussbaumer join: h[j + s k] = (C_j + y C_{j+s})[k] mod m for j < s, where
// y X is the negacyclic word shift (word 0 takes -X[K-1]) and C_{j+s} = 0
// past the product's 2s - 1 elements; the transpose back as in the split.
__global__ void nuss_join_kernel(u64* h, const std::uint8_t* C, u64 c_stride, u32 K, u32 s, u64 m) {
  __shared__ u64 tile[32][33];
  const u32 j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const u32 tx = threadIdx.x, ty = threadIdx.y;
  for (u32 r = ty; r < 32; r += 8) {
    const u32 j = j0 + r, k = k0 + tx;
    if (j < s && k < K) {
      const u64* cj = reinterpret_cast<const u64*>(C + (u64)j * c_stride);
      u64 v = cj[k];
      if (j + 1 < s) {  // C_{j+s} exists (j + s <= 2s - 2)
        const u64* cs = reinterpret_cast<const u64*>(C + (u64)(j + s) * c_stride);
        u64 y = k ? cs[k - 1] : cs[K - 1];
        if (!k && y) y = m - y;
        v += y;  // both < m < 2^62: no overflow
        if (v >= m) v -= m;
      }
      tile[r][tx] = v;
    }
  }
  __syncthreads();
  for (u32 r = ty; r < 32; r += 8) {
    const u32 k = k0 + r, j = j0 + tx;
    if (k < K && j < s) h[(u64)k * s + j] = tile[tx][r];
  }
}

}  // namespace polymul
}  // namespace cftft_b200
