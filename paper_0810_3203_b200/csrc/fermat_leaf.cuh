// fermat_leaf.cuh -- sm_100a leaf kernel for R = Z/(2^N+1), omega = 2.
//
// One CTA runs one leaf: a sub-transform of <= 2^max_ell coefficients held
// entirely in shared memory (the reference's column/row sub-transforms,
// transform.hpp:175-185 / :215-238, cut where they fit on chip).
//
// Element representation in shared memory ("chunked, carry-deferred"):
//   D = N/32 u32 words, grouped in C = D/4 chunks of 128 bits, plus one signed
//   8-bit pending carry per chunk.  The value is
//       sum_j (chunk_j + pend_j * 2^128) * 2^(128 j)   (mod 2^N + 1),
//   the last chunk's pending carry sitting at 2^N == -1.  A butterfly output
//   chunk i is computed by ONE thread from chunk i of operand a (plus a's
//   pending carry from chunk i-1) and the matching window of the rotated
//   operand b (plus the one pending carry of b that lands inside it); the
//   thread's carry-out becomes the new pending carry of chunk i.  No
//   cross-thread carry propagation happens inside a leaf: it is resolved once,
//   when a slot is stored back to HBM (warp-level resolution loop below).
//
// Global (HBM) element format between passes: N/64 u64 limbs "lo" plus a
// signed top word hi, value = lo + hi*2^N (== lo - hi).  Canonical inputs
// (top in {0,1}) are a special case; the final pass canonicalises.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace fermat {

constexpr int kThreads = 512;
constexpr int kTasksPerThread = 8;

struct Args {
  std::uint8_t* data;      // view element 0
  u64 elem_bytes;          // bytes between consecutive view elements
  const DevLeaf* leaves;   // this wave's leaves (blockIdx.x indexes)
  const DevClass* classes;
  const DevOp* ops;
  const u32* levels;       // absolute op offsets
  const SymExp* stores;
  u64 N, M;
  u32 D, C;                // u32 words, 128-bit chunks per element
  u32 slot_bytes;          // 4*D + pending bytes (16B aligned)
};

__device__ __forceinline__ u32* slot_words(std::uint8_t* sm, const Args& A, u32 s) {
  return reinterpret_cast<u32*>(sm + (size_t)s * A.slot_bytes);
}
__device__ __forceinline__ signed char* slot_pend(std::uint8_t* sm, const Args& A, u32 s) {
  return reinterpret_cast<signed char*>(sm + (size_t)s * A.slot_bytes + 4u * A.D);
}

// Rotation r (0 <= r < 2N) decomposed for the windowed read of R_r(b).
struct Rot {
  int sigma;  // -1 when r >= N (2^N == -1)
  u32 w, sh;  // t = r mod N = 32 w + sh
  u32 q, o;   // t = 128 q + o
};
__device__ __forceinline__ Rot make_rot(u64 r, u64 N) {
  Rot R;
  R.sigma = (r >= N) ? -1 : 1;
  u64 t = (r >= N) ? r - N : r;
  R.w = (u32)(t >> 5);
  R.sh = (u32)(t & 31);
  R.q = (u32)(t >> 7);
  R.o = (u32)(t & 127);
  return R;
}

// Signed per-word contributions of chunk i of R_r(x) (x a shared-memory slot):
// bw[k] (k < 4) and the landed pending carry (value pterm at word pw).
__device__ __forceinline__ void rotated_chunk(const u32* xw, const signed char* xp, const Rot& R,
                                              u32 D, u32 C, u32 i, long long bw[4],
                                              long long& pterm, u32& pw) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    u32 g = 4 * i + k;
    u32 hi_idx = (g + D - R.w) % D;
    u32 lo_idx = (hi_idx + D - 1) % D;
    u32 hv = xw[hi_idx];
    u32 fv = R.sh ? ((hv << R.sh) | (xw[lo_idx] >> (32 - R.sh))) : hv;
    long long v;
    if (g > R.w) {
      v = (long long)fv;
    } else if (g < R.w) {
      v = -(long long)fv;
    } else {
      u32 mhi = 0xFFFFFFFFu << R.sh;
      v = (long long)(fv & mhi) - (long long)(fv & ~mhi);
    }
    bw[k] = v * R.sigma;
  }
  // the one pending carry landing inside output chunk i (at offset o)
  int j = (int)i - (int)R.q - 1;
  int sgn = R.sigma;
  if (j < 0) {
    j += (int)C;
    sgn = -sgn;
  }
  pterm = (long long)xp[j] * sgn * (long long)(1ll << (R.o & 31));
  pw = R.o >> 5;
}

struct TaskOut {
  u32 w0[4], w1[4];
  signed char p0, p1;
  std::uint8_t mask;  // bit0: out0 -> slot a, bit1: out1 -> slot b
  std::uint16_t sa, sb;
  u32 chunk;
};

__device__ __forceinline__ void run_task(std::uint8_t* sm, const Args& A, const DevOp& op, u64 s,
                                         u32 i, TaskOut& T) {
  const u32 D = A.D, C = A.C;
  T.sa = op.a;
  T.sb = op.b;
  T.chunk = i;
  const u32* aw = slot_words(sm, A, op.a);
  const signed char* ap = slot_pend(sm, A, op.a);
  if (op.type == OP_COPY) {
    uint4 v = reinterpret_cast<const uint4*>(aw)[i];
    T.w1[0] = v.x;
    T.w1[1] = v.y;
    T.w1[2] = v.z;
    T.w1[3] = v.w;
    T.p1 = ap[i];
    T.mask = 2;
    return;
  }
  const u64 r = (op.ra * s + op.rb) & (A.M - 1);
  const Rot R = make_rot(r, A.N);
  long long bw[4], pterm;
  u32 pw;
  rotated_chunk(slot_words(sm, A, op.b), slot_pend(sm, A, op.b), R, D, C, i, bw, pterm, pw);
  uint4 av4 = reinterpret_cast<const uint4*>(aw)[i];
  u32 av[4] = {av4.x, av4.y, av4.z, av4.w};
  long long pa_in = (i == 0) ? -(long long)ap[C - 1] : (long long)ap[i - 1];
  // out0 = alpha*A + beta*B ; out1 = A - B
  const int alpha = (op.type == OP_SUB2 || op.type == OP_SUB2DIFF) ? 2 : 1;
  const int beta = (op.type == OP_ADDSUB || op.type == OP_ADD) ? 1 : -1;
  const bool two = (op.type == OP_ADDSUB || op.type == OP_SUB2DIFF);
  long long c0 = 0, c1 = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    long long a = (long long)av[k] + (k == 0 ? pa_in : 0);
    long long b = bw[k] + ((u32)k == pw ? pterm : 0);
    long long s0 = c0 + alpha * a + beta * b;
    T.w0[k] = (u32)s0;
    c0 = s0 >> 32;
    long long s1 = c1 + a - b;
    T.w1[k] = (u32)s1;
    c1 = s1 >> 32;
  }
  T.p0 = (signed char)c0;
  T.p1 = (signed char)c1;
  T.mask = two ? 3 : 1;
}

__device__ __forceinline__ void write_task(std::uint8_t* sm, const Args& A, const TaskOut& T) {
  if (T.mask & 1) {
    reinterpret_cast<uint4*>(slot_words(sm, A, T.sa))[T.chunk] =
        make_uint4(T.w0[0], T.w0[1], T.w0[2], T.w0[3]);
    slot_pend(sm, A, T.sa)[T.chunk] = T.p0;
  }
  if (T.mask & 2) {
    reinterpret_cast<uint4*>(slot_words(sm, A, T.sb))[T.chunk] =
        make_uint4(T.w1[0], T.w1[1], T.w1[2], T.w1[3]);
    slot_pend(sm, A, T.sb)[T.chunk] = T.p1;
  }
}

// Adds a small signed carry into a 4-word chunk; returns the carry out (-1/0/1).
__device__ __forceinline__ int add_small(u32 w[4], long long cin) {
  long long c = cin;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    long long s = c + (long long)w[k];
    w[k] = (u32)s;
    c = s >> 32;
  }
  return (int)c;
}

__global__ void __launch_bounds__(kThreads, 1) leaf_kernel(Args A) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  const DevLeaf lf = A.leaves[blockIdx.x];
  const DevClass cl = A.classes[lf.cls];
  const u32 tid = threadIdx.x, nthr = blockDim.x;
  const u32 D = A.D, C = A.C;

  // ---- load slots [0, nload) ------------------------------------------------
  {
    const u32 q16 = D / 4;
    const u32 total = cl.nload * q16;
    for (u32 idx = tid; idx < total; idx += nthr) {
      u32 s = idx / q16, k = idx - s * q16;
      const uint4* src =
          reinterpret_cast<const uint4*>(A.data + (lf.base + (u64)s * lf.stride) * A.elem_bytes);
      reinterpret_cast<uint4*>(slot_words(sm, A, s))[k] = __ldg(src + k);
    }
    const u32 ptotal = cl.nload * C;
    for (u32 idx = tid; idx < ptotal; idx += nthr) {
      u32 s = idx / C, c = idx - s * C;
      signed char v = 0;
      if (c == C - 1) {
        const long long* top = reinterpret_cast<const long long*>(
            A.data + (lf.base + (u64)s * lf.stride) * A.elem_bytes + A.N / 8);
        v = (signed char)*top;
      }
      slot_pend(sm, A, s)[c] = v;
    }
  }
  __syncthreads();

  // ---- micro-op levels --------------------------------------------------------
  const u32 ops_per_batch = max(1u, (nthr * kTasksPerThread) / C);
  for (u32 l = 0; l < cl.nlevels; ++l) {
    const u32 o0 = A.levels[cl.level_begin + l], o1 = A.levels[cl.level_begin + l + 1];
    for (u32 ob = o0; ob < o1; ob += ops_per_batch) {
      const u32 oe = min(o1, ob + ops_per_batch);
      const u32 ntask = (oe - ob) * C;
      TaskOut T[kTasksPerThread];
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        T[k].mask = 0;
        u32 t = tid + k * nthr;
        if (t < ntask) {
          u32 oi = ob + t / C;
          DevOp op = A.ops[oi];
          run_task(sm, A, op, lf.s, t % C, T[k]);
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k)
        if (T[k].mask) write_task(sm, A, T[k]);
      __syncthreads();
    }
  }

  // ---- store slots [0, nstore): apply final rotation, resolve carries --------
  const u32 lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  for (u32 si = warp; si < cl.nstore; si += nwarps) {
    const SymExp P = A.stores[cl.store_begin + si];
    const u64 r = (P.a * lf.s + P.b) & (A.M - 1);
    const Rot R = make_rot(r, A.N);
    std::uint8_t* dst = A.data + (lf.base + (u64)si * lf.stride) * A.elem_bytes;
    const u32* xw = slot_words(sm, A, si);
    const signed char* xp = slot_pend(sm, A, si);
    long long seg_carry = 0;
    for (u32 seg = 0; seg < C; seg += 32) {
      const u32 i = seg + lane;
      const bool act = i < C;
      const u32 last = min(31u, C - 1 - seg);
      u32 w[4] = {0, 0, 0, 0};
      int pout = 0;
      if (act) {
        long long bw[4], pterm;
        u32 pw;
        rotated_chunk(xw, xp, R, D, C, i, bw, pterm, pw);
        long long c = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          long long sres = c + bw[k] + ((u32)k == pw ? pterm : 0);
          w[k] = (u32)sres;
          c = sres >> 32;
        }
        pout = (int)c;
      }
      long long cin_first = seg_carry;
      seg_carry = 0;
      for (;;) {
        int cin = __shfl_up_sync(0xffffffffu, pout, 1);
        int outgoing = __shfl_sync(0xffffffffu, pout, last);
        seg_carry += outgoing;
        long long cin_l = (lane == 0) ? cin_first : (long long)cin;
        cin_first = 0;
        pout = 0;
        if (act && lane <= last && cin_l != 0) pout = add_small(w, cin_l);
        if (!__any_sync(0xffffffffu, pout != 0)) break;
      }
      if (act) reinterpret_cast<uint4*>(dst)[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (lane == 0) *reinterpret_cast<long long*>(dst + A.N / 8) = seg_carry;
  }
}

// Final canonicalisation: value = lo + hi*2^N == lo - hi -> [0, 2^N].
// Thread per element; carry chains beyond word 0 are rare, handled serially.
__global__ void canonicalize_kernel(std::uint8_t* data, u64 elem_bytes, u64 count, u32 D) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  std::uint8_t* el = data + e * elem_bytes;
  long long* topp = reinterpret_cast<long long*>(el + (u64)D * 4);
  long long hi = *topp;
  if (hi == 0) return;
  u32* w = reinterpret_cast<u32*>(el);
  long long top = 0;
  if (hi > 0) {
    // subtract hi
    unsigned long long b = (unsigned long long)hi;
    u32 k = 0;
    for (; k < D && b; ++k) {
      unsigned long long v = w[k];
      unsigned long long lo32 = b & 0xFFFFFFFFull;
      unsigned long long hi32 = b >> 32;
      w[k] = (u32)(v - lo32);
      b = hi32 + (v < lo32 ? 1 : 0);
    }
    if (b) {  // negative: add 2^N + 1 -> +1 on the N-bit residue
      u32 c = 1;
      for (k = 0; k < D && c; ++k) {
        w[k] += 1;
        c = (w[k] == 0);
      }
      top = c;
    }
  } else {
    unsigned long long c = (unsigned long long)(-hi);
    u32 k = 0;
    for (; k < D && c; ++k) {
      unsigned long long v = (unsigned long long)w[k] + (c & 0xFFFFFFFFull);
      w[k] = (u32)v;
      c = (c >> 32) + (v >> 32);
    }
    if (c) {  // value = lo + 2^N == lo - 1
      u32 b = 1;
      for (k = 0; k < D && b; ++k) {
        u32 v = w[k];
        w[k] = v - 1;
        b = (v == 0);
      }
      if (b) {  // was zero: -1 == 2^N
        for (k = 0; k < D; ++k) w[k] = 0;
        top = 1;
      }
    }
  }
  *topp = top;
}

}  // namespace fermat
}  // namespace cftft_b200
