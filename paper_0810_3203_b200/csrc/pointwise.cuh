// pointwise.cuh -- sm_100a pointwise ring products (the middle stage of
// poly_mul, polymul.hpp:73-77) for the two big rings.
//
// Negacyclic R = (Z/mZ)[y]/(y^K+1): a[i] <- a[i] * b[i] is a negacyclic
// convolution of length K mod m.  One CTA per product, operands in shared
// memory; each thread owns output coefficients and accumulates the 128-bit
// products exactly (positive and wrapped parts separately, 192-bit
// accumulators), reducing mod m once at the end.  Optional extra factor c
// (e.g. L^-1 of poly_mul's final scale, polymul.hpp:82-87) is folded in.
//
// Fermat R = Z/(2^N+1): a * b mod 2^N+1 is a NEGACYCLIC convolution of the
// 16-bit digit vectors (2^(16 * N/16) = 2^N == -1).  One CTA per product runs
// it as a weighted NTT over the Goldilocks field p = 2^64 - 2^32 + 1 (the
// reference's default ring, field.hpp:84-98): digits < 2^16, so every
// convolution coefficient lies in (-2^(44+1), 2^(44+1)) and is recovered
// exactly from its residue mod p.  The coefficients are then folded into
// 512-bit chunks with signed tops and carry-resolved like the transform
// engine, and written in the engine's lazy element format.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace pointwise {

// ---------------------------------------------------------------------------
// negacyclic

__device__ __forceinline__ void acc192_add(u64& a0, u64& a1, u64& a2, u64 lo, u64 hi) {
  asm("add.cc.u64 %0, %0, %3;\n\t"
      "addc.cc.u64 %1, %1, %4;\n\t"
      "addc.u64 %2, %2, 0;"
      : "+l"(a0), "+l"(a1), "+l"(a2)
      : "l"(lo), "l"(hi));
}

__device__ __forceinline__ u64 mod192(u64 a0, u64 a1, u64 a2, u64 m) {
  // (a2 2^128 + a1 2^64 + a0) mod m with 128-bit remainders
  typedef unsigned __int128 u128;
  u128 t = ((u128)(a2 % m) << 64) | a1;
  t %= m;
  t = (t << 64) | a0;
  return (u64)(t % m);
}

__device__ __forceinline__ u64 mulmod64(u64 a, u64 b, u64 m) {
  typedef unsigned __int128 u128;
  return (u64)(((u128)a * b) % m);
}

// One CTA per product.  a, b: element pointers (K words each, stride bytes).
__global__ void __launch_bounds__(256) nega_pointwise_kernel(std::uint8_t* a, const std::uint8_t* b, u64 stride,
                                                              u32 K, u64 m, u64 scale) {
  extern __shared__ __align__(16) u64 s_ab[];
  u64* sa = s_ab;
  u64* sb = s_ab + K;
  u64* sc = s_ab + 2 * K;
  u64* pa = reinterpret_cast<u64*>(a + (u64)blockIdx.x * stride);
  const u64* pb = reinterpret_cast<const u64*>(b + (u64)blockIdx.x * stride);
  for (u32 i = threadIdx.x; i < K; i += blockDim.x) {
    sa[i] = pa[i];
    sb[i] = pb[i];
  }
  __syncthreads();
  for (u32 k = threadIdx.x; k < K; k += blockDim.x) {
    u64 p0 = 0, p1 = 0, p2 = 0, n0 = 0, n1 = 0, n2 = 0;
    for (u32 i = 0; i <= k; ++i) {
      const u64 x = sa[i], y = sb[k - i];
      acc192_add(p0, p1, p2, x * y, __umul64hi(x, y));
    }
    for (u32 i = k + 1; i < K; ++i) {  // y^K = -1
      const u64 x = sa[i], y = sb[K + k - i];
      acc192_add(n0, n1, n2, x * y, __umul64hi(x, y));
    }
    const u64 pv = mod192(p0, p1, p2, m), nv = mod192(n0, n1, n2, m);
    u64 r = pv >= nv ? pv - nv : pv + (m - nv);
    if (scale != 1) r = mulmod64(r, scale, m);
    sc[k] = r;
  }
  __syncthreads();
  for (u32 k = threadIdx.x; k < K; k += blockDim.x) pa[k] = sc[k];
}

// a[i] <- c * a[i] (word-wise mod m) over count elements of K words.
__global__ void nega_scale_kernel(std::uint8_t* a, u64 stride, u64 count, u32 K, u64 m, u64 c) {
  const u64 idx = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count * K) return;
  const u64 e = idx / K, w = idx % K;
  u64* p = reinterpret_cast<u64*>(a + e * stride) + w;
  *p = mulmod64(*p, c, m);
}

// ---------------------------------------------------------------------------
// Goldilocks field (p = 2^64 - 2^32 + 1)

constexpr u64 GP = 0xFFFFFFFF00000001ull;

__device__ __forceinline__ u64 g_add(u64 a, u64 b) {
  const u64 s = a + b;
  // overflow past 2^64 or >= p: subtract p (== add 2^32 - 1 mod 2^64)
  if (s < a) return s + 0xFFFFFFFFull;
  return s >= GP ? s - GP : s;
}
__device__ __forceinline__ u64 g_sub(u64 a, u64 b) { return a >= b ? a - b : a + (GP - b); }
__device__ __forceinline__ u64 g_mul(u64 a, u64 b) {
  const u64 lo = a * b, hi = __umul64hi(a, b);
  // x = hi 2^64 + lo; 2^64 == 2^32 - 1, 2^96 == -1 (field.hpp:154-167 restated)
  const u64 hh = hi >> 32, hl = hi & 0xFFFFFFFFull;
  u64 t = lo - hh;
  if (lo < hh) t -= 0xFFFFFFFFull;
  const u64 s = hl * 0xFFFFFFFFull;
  u64 r = t + s;
  if (r < t) r += 0xFFFFFFFFull;
  if (r >= GP) r -= GP;
  return r;
}

struct FermatMulArgs {
  std::uint8_t* a;
  const std::uint8_t* b;
  u64 stride;
  u32 D16;        // digits (16-bit) per element = N/16 = NTT length n
  u32 logn;
  u32 D32;        // u32 words per element = N/32
  const u64* tw;  // psi^i (i < n), then omega_n^j (j < n/2), then the inverses
  u64 n_inv;      // 1/n mod p
  u32 rot;        // extra factor 2^rot of every product (rot < 2N): poly_mul's L^-1 = 2^(2N - ell)
};

// In-place cyclic NTT of length n in shared memory: DIF (natural -> bit
// reversed) for the forward transform, DIT (bit reversed -> natural) for the
// inverse; w = omega_n^j table (n/2 entries) in shared memory.
// ws: per-level twiddle tables in global memory (level ls: omega^(j 2^ls),
// j < n >> (ls+1), at n - (n >> ls)) -- contiguous in j, so a warp's reads
// coalesce (the strided w[j << ls] of one table was a 32-way shared-memory
// bank conflict in the middle levels).
__device__ __forceinline__ void ntt_dif(u64* x, const u64* ws, u32 n, u32 logn) {
  for (u32 h = n >> 1, ls = 0; h >= 1; h >>= 1, ++ls) {
    const u32 lh = logn - 1 - ls;
    const u64* w = ws + (n - (n >> ls));
    for (u32 t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
      const u32 grp = t >> lh, j = t & (h - 1);
      const u32 i0 = grp * 2 * h + j, i1 = i0 + h;
      const u64 u = x[i0], v = x[i1];
      x[i0] = g_add(u, v);
      x[i1] = g_mul(g_sub(u, v), __ldg(w + j));
    }
    __syncthreads();
  }
}
__device__ __forceinline__ void ntt_dit(u64* x, const u64* ws, u32 n, u32 logn) {
  for (u32 h = 1, ls = logn - 1; h < n; h <<= 1, --ls) {
    const u32 lh = logn - 1 - ls;
    const u64* w = ws + (n - (n >> ls));
    for (u32 t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
      const u32 grp = t >> lh, j = t & (h - 1);
      const u32 i0 = grp * 2 * h + j, i1 = i0 + h;
      const u64 u = x[i0], v = g_mul(x[i1], __ldg(w + j));
      x[i0] = g_add(u, v);
      x[i1] = g_sub(u, v);
    }
    __syncthreads();
  }
}

// Adds each chunk's pending signed carry `pend` into the chunked value (chunk
// t = 16 words owned by thread t) and ripples until no carry moves; returns
// the carry out of the top chunk (block-uniform).  sh: chunks + 1 scratch slots.
__device__ __forceinline__ long long ripple(u32 (&wv)[16], long long* sh, u32 t, u32 chunks, long long pend) {
  long long tout = 0;
  for (;;) {
    long long outc = 0;
    if (t < chunks && pend != 0) {
      long long cy = pend;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const long long v = (long long)wv[k] + cy;
        wv[k] = (u32)v;
        cy = v >> 32;  // arithmetic
      }
      outc = cy;
    }
    if (t < chunks) {
      if (t == chunks - 1)
        tout += outc;
      else
        sh[t] = outc;
    }
    __syncthreads();
    pend = (t < chunks && t > 0) ? sh[t - 1] : 0;
    if (!__syncthreads_or(pend != 0)) break;
  }
  if (t == chunks - 1) sh[chunks] = tout;
  __syncthreads();
  const long long r = sh[chunks];
  __syncthreads();
  return r;
}

// One CTA per product: a[e] <- a[e] * b[e] mod 2^N + 1, canonical output
// (lo in [0, 2^N), top word 1 only for 2^N == -1), as the transforms expect.
__global__ void __launch_bounds__(512) fermat_pointwise_kernel(FermatMulArgs A) {
  extern __shared__ __align__(16) u64 s_f[];
  const u32 n = A.D16;
  u64* xa = s_f;
  u64* xb = s_f + n;
  const u64* w = A.tw + 7 * (u64)n / 2;   // per-level omega^(j 2^ls) (ntt_dif)
  const u64* wi = A.tw + 9 * (u64)n / 2;  // per-level omega^-(j 2^ls) (ntt_dit)
  std::uint8_t* ea = A.a + (u64)blockIdx.x * A.stride;
  const std::uint8_t* eb = A.b + (u64)blockIdx.x * A.stride;
  const u64* psi = A.tw;                 // psi^i
  const u64* psii = A.tw + n + n;        // psi^-i * (1/n)
  const std::uint16_t* da = reinterpret_cast<const std::uint16_t*>(ea);
  const std::uint16_t* db = reinterpret_cast<const std::uint16_t*>(eb);
  const long long topa = *reinterpret_cast<const long long*>(ea + (u64)A.D32 * 4);
  const long long topb = *reinterpret_cast<const long long*>(eb + (u64)A.D32 * 4);
  const u32 chunks = n / 32;  // thread t owns words [16t, 16t+16)
  const u32 t = threadIdx.x;
  long long* carry = reinterpret_cast<long long*>(xb);  // scratch once xb is consumed
  u32 wv[16];
  long long pend = 0;
  if (topa != 0 || topb != 0) {
    // canonical inputs: top = 1 means 2^N == -1 (all limbs zero), so the
    // product is -b, -a or 1: as negacyclic digit coefficients -x_i, or 1
    const bool one = topa != 0 && topb != 0;
    const std::uint16_t* other = topa ? db : da;
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      const u64 d = one ? (i == 0 ? 1u : 0u) : (u64)other[i];
      xa[i] = one ? d : (d ? GP - d : 0);
    }
    __syncthreads();
  } else {
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      xa[i] = g_mul((u64)da[i], psi[i]);
      xb[i] = g_mul((u64)db[i], psi[i]);
    }
    __syncthreads();
    ntt_dif(xa, w, n, A.logn);
    ntt_dif(xb, w, n, A.logn);
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) xa[i] = g_mul(xa[i], xb[i]);
    __syncthreads();
    ntt_dit(xa, wi, n, A.logn);
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) xa[i] = g_mul(xa[i], psii[i]);
    __syncthreads();
  }
  {
    // fold the signed digit coefficients c_i (|c_i| < 2^45) into 512-bit
    // chunks; the extra factor 2^rot = x^q 2^r (x = 2^16, x^n = -1): digit i
    // of the result takes coefficient i - q (negated past the wrap) times 2^r
    const u32 q = A.rot >> 4, r = A.rot & 15u;
    if (t < chunks) {
      long long acc[17];
#pragma unroll
      for (int k = 0; k < 17; ++k) acc[k] = 0;
#pragma unroll
      for (int d = 0; d < 32; ++d) {
        int src = (int)(32 * t + d) - (int)(q % (2 * n));
        bool neg = false;
        while (src < 0) {
          src += (int)n;
          neg = !neg;
        }
        const u64 v = xa[src];
        long long c = v > (GP >> 1) ? -(long long)(GP - v) : (long long)v;
        if (neg) c = -c;
        c *= (1ll << r);  // |c| < 2^60
        // c * 2^(16 d) -> word d/2, shifted by 16 (d odd)
        if (d & 1) {
          acc[d / 2] += (long long)((unsigned long long)(c & 0xFFFF) << 16);
          acc[d / 2 + 1] += c >> 16;
        } else {
          acc[d / 2] += c;
        }
      }
      long long cy = 0;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const long long v = acc[k] + cy;
        wv[k] = (u32)v;
        cy = v >> 32;  // arithmetic
      }
      carry[t] = cy + acc[16];
    }
    __syncthreads();
    // chunk t takes chunk t-1's carry; the top chunk's carry wraps to chunk 0
    // negated (2^N == -1)
    if (t < chunks) pend = t == 0 ? -carry[chunks - 1] : carry[t - 1];
    __syncthreads();
  }
  // value = lo + c 2^N == lo - c with the top carry c in {-1, 0, 1}
  const long long c = ripple(wv, carry, t, chunks, pend);
  long long top = 0;
  if (c != 0) {
    // lo - 1 with lo == 0, or lo + 1 with lo == 2^N - 1: the result is 2^N
    bool edge = true;
    if (t < chunks) {
#pragma unroll
      for (int k = 0; k < 16; ++k) edge &= wv[k] == (c > 0 ? 0u : 0xFFFFFFFFu);
    }
    if (__syncthreads_and(edge)) {
      top = 1;
      if (t < chunks) {
#pragma unroll
        for (int k = 0; k < 16; ++k) wv[k] = 0;
      }
    } else {
      ripple(wv, carry, t, chunks, t == 0 ? -c : 0);
    }
  }
  if (t < chunks) {
    uint4* dst = reinterpret_cast<uint4*>(ea) + 4 * t;
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = make_uint4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]);
    if (t == 0) *reinterpret_cast<long long*>(ea + (u64)A.D32 * 4) = top;
  }
}

}  // namespace pointwise
}  // namespace cftft_b200
