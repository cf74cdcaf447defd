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
// it as psi-weighted NTTs modulo two 30-bit primes (native 32-bit Shoup /
// Barrett arithmetic) and recovers every coefficient (|c| < n 2^32) by CRT;
// the coefficients are then folded into 512-bit chunks and carry-resolved,
// canonical output.
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
// Two NTT primes below 2^30 with roots of unity of every power-of-two order
// up to 2^23: 998244353 = 119 2^23 + 1 and 469762049 = 7 2^26 + 1 (primitive
// root 3 for both).  Their product (~2^58.7) exceeds twice the largest
// negacyclic convolution coefficient of 16-bit digits, n 2^32 <= 2^45
// (n = N/16 <= 8192), so each coefficient comes back exactly by CRT.
constexpr u32 Q1 = 998244353u, Q2 = 469762049u;

// Shoup product x w mod p for a fixed w (wp = floor(w 2^32 / p)): x < 2^32,
// result in [0, 2p)
__device__ __forceinline__ u32 shoup(u32 x, u32 w, u32 wp, u32 p) {
  const u32 q = __umulhi(x, wp);
  return x * w - q * p;
}
// x y mod p for variable x, y < 2^31 (Barrett with m64 = floor(2^64 / p)):
// result in [0, 2p)
__device__ __forceinline__ u32 mulmod_b(u32 x, u32 y, u32 p, u64 m64) {
  const u64 t = (u64)x * y;
  const u64 q = __umul64hi(t, m64);
  return (u32)(t - q * p);
}

struct FermatMulArgs {
  std::uint8_t* a;
  const std::uint8_t* b;
  u64 stride;
  u32 D16;        // digits (16-bit) per element = N/16 = NTT length n
  u32 logn;
  u32 D32;        // u32 words per element = N/32
  const uint4* tw;  // 4 n entries {w mod Q1, its Shoup factor, w mod Q2, its Shoup}: psi^i, psi^-i / n,
                    // the forward level twiddles (level ls: omega^(j 2^ls), j < n >> (ls+1), at
                    // n - (n >> ls)), the inverse ones
  u32 rot;        // extra factor 2^rot of every product (rot < 2N): poly_mul's L^-1 = 2^(2N - ell)
};

// Both primes' arrays of one operand advance together (independent work per
// thread); values stay lazily in [0, 2p) (Harvey's butterflies, p < 2^30).
template <u32 Q>
__device__ __forceinline__ void bf_dif(u32& u, u32& v, u32 w, u32 wp) {
  const u32 s = u + v, d = u - v + 2 * Q;
  u = s >= 2 * Q ? s - 2 * Q : s;
  v = shoup(d, w, wp, Q);
}
template <u32 Q>
__device__ __forceinline__ void bf_dit(u32& u, u32& v, u32 w, u32 wp) {
  const u32 t = shoup(v, w, wp, Q);
  const u32 s = u + t, d = u - t + 2 * Q;
  u = s >= 2 * Q ? s - 2 * Q : s;
  v = d >= 2 * Q ? d - 2 * Q : d;
}
// Shared arrays are padded one word per eight (index i at i + i/8): the
// radix-8 passes' strided sets then hit distinct banks for every span.
__device__ __forceinline__ u32 pd(u32 i) { return i + (i >> 3); }
__host__ __device__ constexpr u32 padded(u32 n) { return n + (n >> 3); }

// one radix-2 level (the passes' tail when log n is not a multiple of 3)
template <bool DIF>
__device__ __forceinline__ void level2(u32* x1, u32* x2, const uint4* tw, u32 n, u32 logn, u32 ls) {
  const u32 h = n >> (ls + 1), lh = logn - 1 - ls, off = n - (n >> ls);
  const uint4* tl = tw + (DIF ? 2 * n : 3 * n) + off;
  for (u32 t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
    const u32 grp = t >> lh, j = t & (h - 1);
    const u32 i0 = pd(grp * 2 * h + j), i1 = pd(grp * 2 * h + j + h);
    u32 a = x1[i0], b = x1[i1], c = x2[i0], d = x2[i1];
    const uint4 w = __ldg(tl + j);
    if (DIF) {
      bf_dif<Q1>(a, b, w.x, w.y);
      bf_dif<Q2>(c, d, w.z, w.w);
    } else {
      bf_dit<Q1>(a, b, w.x, w.y);
      bf_dit<Q2>(c, d, w.z, w.w);
    }
    x1[i0] = a;
    x1[i1] = b;
    x2[i0] = c;
    x2[i1] = d;
  }
  __syncthreads();
}
// Three levels in registers: the sets {base + m q, m < 8} (q the smallest
// span of the three) are closed under them.  DIF: spans 4q, 2q, q (levels
// ls, ls+1, ls+2); DIT: spans q, 2q, 4q (levels ls+2, ls+1, ls).  The
// twiddles a set needs: four at the 4q level, two at 2q, one at q.
template <bool DIF>
__device__ __forceinline__ void pass8(u32* x1, u32* x2, const uint4* tw, u32 n, u32 logn, u32 ls) {
  const u32 logq = logn - ls - 3, q = 1u << logq;
  const uint4* tl = tw + (DIF ? 2 * n : 3 * n);
  const u32 o0 = n - (n >> ls), o1 = n - (n >> (ls + 1)), o2 = n - (n >> (ls + 2));
  for (u32 st = threadIdx.x; st < (n >> 3); st += blockDim.x) {
    const u32 g = st >> logq, r = st & (q - 1), base = (g << (logq + 3)) + r;
    u32 v1[8], v2[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      v1[m] = x1[pd(base + m * q)];
      v2[m] = x2[pd(base + m * q)];
    }
    uint4 w[7];  // [0..3] the 4q level, [4..5] 2q, [6] q
#pragma unroll
    for (int k = 0; k < 7; ++k)
      w[k] = __ldg(tl + (k < 4 ? o0 + r + k * q : (k < 6 ? o1 + r + (k - 4) * q : o2 + r)));
    auto bf = [&](int k, int m0, int m1) {
      if (DIF) {
        bf_dif<Q1>(v1[m0], v1[m1], w[k].x, w[k].y);
        bf_dif<Q2>(v2[m0], v2[m1], w[k].z, w[k].w);
      } else {
        bf_dit<Q1>(v1[m0], v1[m1], w[k].x, w[k].y);
        bf_dit<Q2>(v2[m0], v2[m1], w[k].z, w[k].w);
      }
    };
    if (DIF) {
#pragma unroll
      for (int m = 0; m < 4; ++m) bf(m, m, m + 4);
#pragma unroll
      for (int m = 0; m < 8; m += 4) {
        bf(4, m, m + 2);
        bf(5, m + 1, m + 3);
      }
#pragma unroll
      for (int m = 0; m < 8; m += 2) bf(6, m, m + 1);
    } else {
#pragma unroll
      for (int m = 0; m < 8; m += 2) bf(6, m, m + 1);
#pragma unroll
      for (int m = 0; m < 8; m += 4) {
        bf(4, m, m + 2);
        bf(5, m + 1, m + 3);
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) bf(m, m, m + 4);
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      x1[pd(base + m * q)] = v1[m];
      x2[pd(base + m * q)] = v2[m];
    }
  }
  __syncthreads();
}
// cyclic NTTs of length n = 2^logn: DIF natural -> bit reversed (levels 0,
// 1, ...), DIT bit reversed -> natural (levels logn-1, ..., 0)
__device__ __forceinline__ void ntt_dif2(u32* x1, u32* x2, const uint4* tw, u32 n, u32 logn) {
  u32 ls = 0;
  for (; ls + 3 <= logn; ls += 3) pass8<true>(x1, x2, tw, n, logn, ls);
  for (; ls < logn; ++ls) level2<true>(x1, x2, tw, n, logn, ls);
}
__device__ __forceinline__ void ntt_dit2(u32* x1, u32* x2, const uint4* tw, u32 n, u32 logn) {
  int ls = (int)logn - 1;
  for (; ls >= 0 && (u32)ls + 1 > (logn / 3) * 3; --ls) level2<false>(x1, x2, tw, n, logn, (u32)ls);
  for (; ls >= 2; ls -= 3) pass8<false>(x1, x2, tw, n, logn, (u32)ls - 2);
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

// One CTA per product: a[e] <- a[e] * b[e] * 2^rot mod 2^N + 1, canonical
// output (lo in [0, 2^N), top word 1 only for 2^N == -1).  The digit
// vectors' negacyclic convolution runs as psi-weighted cyclic NTTs modulo Q1
// and Q2 in shared memory (four u32 arrays of n), then CRT to signed 64-bit
// coefficients, digit shift by rot, folding into 512-bit chunks and carry
// resolution.
__global__ void __launch_bounds__(512) fermat_pointwise_kernel(FermatMulArgs A) {
  extern __shared__ __align__(16) u32 s_f[];
  const u32 n = A.D16;
  const u32 np = padded(n);
  u32* a1 = s_f;
  u32* a2 = s_f + np;
  u32* b1 = s_f + 2 * np;
  u32* b2 = s_f + 3 * np;
  long long* cf = reinterpret_cast<long long*>(b1);  // signed coefficients, once b is consumed
  const uint4* tw = A.tw;
  std::uint8_t* ea = A.a + (u64)blockIdx.x * A.stride;
  const std::uint8_t* eb = A.b + (u64)blockIdx.x * A.stride;
  const std::uint16_t* da = reinterpret_cast<const std::uint16_t*>(ea);
  const std::uint16_t* db = reinterpret_cast<const std::uint16_t*>(eb);
  const long long topa = *reinterpret_cast<const long long*>(ea + (u64)A.D32 * 4);
  const long long topb = *reinterpret_cast<const long long*>(eb + (u64)A.D32 * 4);
  const u32 chunks = n / 32;  // thread t owns words [16t, 16t+16)
  const u32 t = threadIdx.x;
  long long* carry = reinterpret_cast<long long*>(a1);  // scratch once the coefficients are out
  u32 wv[16];
  long long pend = 0;
  if (topa != 0 || topb != 0) {
    // canonical inputs: top = 1 means 2^N == -1 (all limbs zero), so the
    // product is -b, -a or 1: as negacyclic digit coefficients -x_i, or 1
    const bool one = topa != 0 && topb != 0;
    const std::uint16_t* other = topa ? db : da;
    __syncthreads();
    for (u32 i = threadIdx.x; i < n; i += blockDim.x)
      cf[i] = one ? (i == 0 ? 1 : 0) : -(long long)other[i];
    __syncthreads();
  } else {
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      const u32 x = da[i], y = db[i], k = pd(i);
      const uint4 ps = __ldg(tw + i);
      a1[k] = shoup(x, ps.x, ps.y, Q1);
      a2[k] = shoup(x, ps.z, ps.w, Q2);
      b1[k] = shoup(y, ps.x, ps.y, Q1);
      b2[k] = shoup(y, ps.z, ps.w, Q2);
    }
    __syncthreads();
    ntt_dif2(a1, a2, tw, n, A.logn);
    ntt_dif2(b1, b2, tw, n, A.logn);
    constexpr u64 M1 = ~0ull / Q1, M2 = ~0ull / Q2;
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      const u32 k = pd(i);
      a1[k] = mulmod_b(a1[k], b1[k], Q1, M1);
      a2[k] = mulmod_b(a2[k], b2[k], Q2, M2);
    }
    __syncthreads();
    ntt_dit2(a1, a2, tw, n, A.logn);
    // unweight (psi^-i / n), CRT: c = r1 + Q1 ((r2 - r1) Q1^-1 mod Q2), signed
    constexpr u32 INV = 208783132u;               // Q1^-1 mod Q2
    constexpr u32 INVP = (u32)(((u64)INV << 32) / Q2);
    constexpr u64 P = (u64)Q1 * Q2;
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      const uint4 ip = __ldg(tw + n + i);
      u32 r1 = shoup(a1[pd(i)], ip.x, ip.y, Q1);
      u32 r2 = shoup(a2[pd(i)], ip.z, ip.w, Q2);
      r1 = r1 >= Q1 ? r1 - Q1 : r1;
      r2 = r2 >= Q2 ? r2 - Q2 : r2;
      u32 r1m = r1 >= Q2 ? r1 - Q2 : r1;
      r1m = r1m >= Q2 ? r1m - Q2 : r1m;
      u32 k = shoup(r2 + Q2 - r1m, INV, INVP, Q2);
      k = k >= Q2 ? k - Q2 : k;
      const u64 c = r1 + (u64)Q1 * k;
      cf[i] = c > P / 2 ? (long long)c - (long long)P : (long long)c;
    }
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
        long long c = cf[src];
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
