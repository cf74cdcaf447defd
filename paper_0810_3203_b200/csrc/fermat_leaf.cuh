// fermat_leaf.cuh -- sm_100a leaf engine for R = Z/(2^N+1), omega = 2.
//
// One persistent launch runs a whole transform.  Each CTA repeatedly takes a
// ticket (a leaf: a sub-transform of <= 2^max_ell coefficients that fits in
// shared memory), waits until the (node, phase) counter it depends on is
// complete, runs the leaf, and bumps the counters it completes.  Tickets are
// issued in a topological, L2-batched order by the planner.
//
// Element representation in shared memory ("chunked, carry-deferred"):
//   D = N/32 u32 words in C = D/4 chunks of 128 bits, plus one signed 8-bit
//   pending carry per chunk (the carry out of that chunk, not yet added to
//   the next).  The value is
//       sum_j (chunk_j + pend_j * 2^128) * 2^(128 j)   (mod 2^N + 1),
//   the last chunk's pending carry sitting at 2^N == -1.  One thread computes
//   one 128-bit output chunk of a butterfly from chunk i of operand a (plus
//   a's pending carry from chunk i-1) and the matching window of the rotated
//   operand b (plus the one pending carry of b landing inside it); its carry
//   out becomes the new pending carry of chunk i.  No cross-thread carry
//   propagation happens inside a leaf: carries are resolved once per stored
//   slot (parallel sweeps in shared memory).
//
// Global (HBM) element format between waves: N/64 u64 limbs "lo" plus a
// signed top word hi, value = lo + hi*2^N (== lo - hi).  Canonical inputs
// (top in {0,1}) are a special case; the last step canonicalises.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace fermat {

constexpr int kThreads = 512;
constexpr int kTasksPerThread = 4;

typedef unsigned __int128 u128;

struct Args {
  std::uint8_t* data;      // view element 0
  u64 elem_bytes;          // bytes between consecutive view elements
  const DevLeaf* leaves;   // ticket order
  u64 nleaves;
  const DevClass* classes;
  const DevOp* ops;
  const u32* levels;       // absolute op offsets
  const SymExp* rots;      // pre/post rotation tables
  u32* counters;           // [0]: ticket; [1 + k]: (node, phase) completion counters
  const DevCounter* cmeta;  // per-counter target and parent link
  u64 N, M;
  u32 D, C;                // u32 words, 128-bit chunks per element
  u32 slot_bytes;          // 4*D + pending bytes (16B aligned)
};

__device__ __forceinline__ uint4* slot_chunks(std::uint8_t* sm, const Args& A, u32 s) {
  return reinterpret_cast<uint4*>(sm + (size_t)s * A.slot_bytes);
}
__device__ __forceinline__ signed char* slot_pend(std::uint8_t* sm, const Args& A, u32 s) {
  return reinterpret_cast<signed char*>(sm + (size_t)s * A.slot_bytes + 4u * A.D);
}

__device__ __forceinline__ u128 to128(uint4 v) {
  return ((u128)v.w << 96) | ((u128)v.z << 64) | ((u128)v.y << 32) | (u128)v.x;
}
__device__ __forceinline__ uint4 from128(u128 x) {
  return make_uint4((u32)x, (u32)(x >> 32), (u32)(x >> 64), (u32)(x >> 96));
}

// value = lo + hi * 2^128
struct Val {
  u128 lo;
  int hi;
};
__device__ __forceinline__ Val vadd(Val a, Val b) {
  Val r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}
__device__ __forceinline__ Val vsub(Val a, Val b) {
  Val r;
  r.lo = a.lo - b.lo;
  r.hi = a.hi - b.hi - (a.lo < b.lo ? 1 : 0);
  return r;
}
__device__ __forceinline__ Val vneg(Val a) {
  Val r;
  r.lo = (u128)0 - a.lo;
  r.hi = -a.hi - (a.lo != 0 ? 1 : 0);
  return r;
}
// small signed p times 2^o, 0 <= o < 128
__device__ __forceinline__ Val vsmall(int p, u32 o) {
  Val r;
  __int128 sp = (__int128)p;
  r.lo = (u128)sp << o;
  r.hi = o ? (int)(sp >> (128 - o)) : (p < 0 ? -1 : 0);
  return r;
}

// Rotation r (0 <= r < 2N) for windowed reads of omega^r * x.
struct Rot {
  int sigma;  // -1 when r >= N (2^N == -1)
  u32 q, o;   // t = r mod N = 128 q + o
};
__device__ __forceinline__ Rot make_rot(u64 r, u64 N) {
  Rot R;
  R.sigma = (r >= N) ? -1 : 1;
  u64 t = (r >= N) ? r - N : r;
  R.q = (u32)(t >> 7);
  R.o = (u32)(t & 127);
  return R;
}

// Exact value of output chunk i of omega^r * x (x a shared-memory slot),
// including the one pending carry of x that lands inside it.
__device__ __forceinline__ Val rot_chunk(const uint4* xc, const signed char* xp, const Rot& R,
                                         u32 C, u32 i) {
  const u32 Cm = C - 1;
  const u32 j = (i - R.q) & Cm;  // source chunk of the upper part
  const u32 jm = (j - 1) & Cm;   // source chunk of the lower part / landed pending
  Val v;
  if (R.o == 0) {
    v.lo = to128(xc[j]);
    v.hi = 0;
    if (i < R.q) v = vneg(v);
  } else {
    const u128 up = to128(xc[j]) << R.o;
    const u128 dn = to128(xc[jm]) >> (128 - R.o);
    if (i > R.q) {
      v.lo = up | dn;
      v.hi = 0;
    } else if (i < R.q) {
      v.lo = up | dn;
      v.hi = 0;
      v = vneg(v);
    } else {
      Val a{up, 0}, b{dn, 0};
      v = vsub(a, b);
    }
  }
  int p = xp[jm];
  if (i <= R.q) p = -p;
  v = vadd(v, vsmall(p, R.o));
  if (R.sigma < 0) v = vneg(v);
  return v;
}

// Operand a, unrotated: chunk i plus its bottom pending carry.
__device__ __forceinline__ Val plain_chunk(const uint4* ac, const signed char* ap, u32 C, u32 i) {
  Val v{to128(ac[i]), 0};
  int p = i ? (int)ap[i - 1] : -(int)ap[C - 1];
  return vadd(v, vsmall(p, 0));
}

struct TaskOut {
  uint4 w0, w1;
  signed char p0, p1;
  std::uint8_t mask;  // bit0: out0 -> slot a, bit1: out1 -> slot b
  std::uint16_t sa, sb;
  u32 chunk;
};

__device__ __forceinline__ void run_op_task(std::uint8_t* sm, const Args& A, const DevOp& op, u32 i,
                                            TaskOut& T) {
  const u32 C = A.C;
  T.sa = op.a;
  T.sb = op.b;
  T.chunk = i;
  const uint4* ac = slot_chunks(sm, A, op.a);
  const signed char* ap = slot_pend(sm, A, op.a);
  if (op.type == OP_COPY) {
    T.w1 = ac[i];
    T.p1 = ap[i];
    T.mask = 2;
    return;
  }
  const Rot R = make_rot(op.r, A.N);
  const Val b = rot_chunk(slot_chunks(sm, A, op.b), slot_pend(sm, A, op.b), R, C, i);
  const Val a = plain_chunk(ac, ap, C, i);
  Val y0, y1;
  switch (op.type) {
    case OP_ADDSUB:
      y0 = vadd(a, b);
      y1 = vsub(a, b);
      T.mask = 3;
      break;
    case OP_ADD:
      y0 = vadd(a, b);
      T.mask = 1;
      break;
    case OP_SUB2:
      y0 = vsub(vadd(a, a), b);
      T.mask = 1;
      break;
    default:  // OP_SUB2DIFF
      y1 = vsub(a, b);
      y0 = vadd(a, y1);
      T.mask = 3;
      break;
  }
  T.w0 = from128(y0.lo);
  T.p0 = (signed char)y0.hi;
  if (T.mask & 2) {
    T.w1 = from128(y1.lo);
    T.p1 = (signed char)y1.hi;
  }
}

__device__ __forceinline__ void write_task(std::uint8_t* sm, const Args& A, const TaskOut& T) {
  if (T.mask & 1) {
    slot_chunks(sm, A, T.sa)[T.chunk] = T.w0;
    slot_pend(sm, A, T.sa)[T.chunk] = T.p0;
  }
  if (T.mask & 2) {
    slot_chunks(sm, A, T.sb)[T.chunk] = T.w1;
    slot_pend(sm, A, T.sb)[T.chunk] = T.p1;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ u32 ld_acquire(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Rotates slots [s0, s0+ns) in place by rot[k] (k = slot) -- batched so that
// every thread holds at most kTasksPerThread chunks.
__device__ __forceinline__ void rotate_slots(std::uint8_t* sm, const Args& A, u32 s0, u32 ns,
                                             const SymExp* rot, u64 s) {
  const u32 C = A.C, tid = threadIdx.x, nthr = blockDim.x;
  const u32 per_batch = max(1u, (nthr * kTasksPerThread) / C);
  for (u32 b0 = 0; b0 < ns; b0 += per_batch) {
    const u32 nb = min(ns - b0, per_batch);
    const u32 ntask = nb * C;
    uint4 w[kTasksPerThread];
    signed char p[kTasksPerThread];
#pragma unroll
    for (int k = 0; k < kTasksPerThread; ++k) {
      const u32 t = tid + k * nthr;
      if (t < ntask) {
        const u32 sl = s0 + b0 + t / C, i = t % C;
        const u64 r = (rot[sl].a * s + rot[sl].b) & (A.M - 1);
        const Rot R = make_rot(r, A.N);
        Val v = rot_chunk(slot_chunks(sm, A, sl), slot_pend(sm, A, sl), R, C, i);
        w[k] = from128(v.lo);
        p[k] = (signed char)v.hi;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTasksPerThread; ++k) {
      const u32 t = tid + k * nthr;
      if (t < ntask) {
        const u32 sl = s0 + b0 + t / C, i = t % C;
        slot_chunks(sm, A, sl)[i] = w[k];
        slot_pend(sm, A, sl)[i] = p[k];
      }
    }
    __syncthreads();
  }
}

// Resolves the pending carries of slots [0, ns) into exact limbs (the top
// pending carry stays: it is the element's signed top word).
__device__ __forceinline__ void resolve_slots(std::uint8_t* sm, const Args& A, u32 ns) {
  const u32 C = A.C, tid = threadIdx.x, nthr = blockDim.x;
  const u32 per_batch = max(1u, (nthr * kTasksPerThread) / C);
  for (u32 b0 = 0; b0 < ns; b0 += per_batch) {
    const u32 nb = min(ns - b0, per_batch);
    const u32 ntask = nb * C;
    for (;;) {
      u128 w[kTasksPerThread];
      int e[kTasksPerThread];
      int any = 0;
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        const u32 t = tid + k * nthr;
        e[k] = 0;
        if (t < ntask) {
          const u32 sl = b0 + t / C, i = t % C;
          const signed char* pp = slot_pend(sm, A, sl);
          const int in = i ? (int)pp[i - 1] : 0;
          w[k] = to128(slot_chunks(sm, A, sl)[i]);
          const u128 old = w[k];
          w[k] += (u128)(__int128)in;
          int carry = 0;
          if (in > 0 && w[k] < old) carry = 1;
          if (in < 0 && w[k] > old) carry = -1;
          e[k] = (i == C - 1) ? (int)pp[C - 1] + carry : carry;
          if (i != C - 1 && carry != 0) any = 1;
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        const u32 t = tid + k * nthr;
        if (t < ntask) {
          const u32 sl = b0 + t / C, i = t % C;
          slot_chunks(sm, A, sl)[i] = from128(w[k]);
          slot_pend(sm, A, sl)[i] = (signed char)e[k];
        }
      }
      if (!__syncthreads_or(any)) break;
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) leaf_kernel(Args A) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  __shared__ u32 s_ticket;
  const u32 tid = threadIdx.x, nthr = blockDim.x;
  const u32 D = A.D, C = A.C;

  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(&A.counters[0], 1u);
    __syncthreads();
    const u32 ticket = s_ticket;
    if (ticket >= A.nleaves) return;
    const DevLeaf lf = A.leaves[ticket];
    const DevClass cl = A.classes[lf.cls];
    if (lf.dep != kNoDep && tid == 0) {
      const u32* c = &A.counters[1 + lf.dep];
      while (ld_acquire(c) < lf.dep_target) __nanosleep(64);
    }
    __syncthreads();

    // ---- load slots [0, nload) (L2 path: data may come from other CTAs) ----
    {
      const u32 q16 = D / 4;
      const u32 total = cl.nload * q16;
      for (u32 idx = tid; idx < total; idx += nthr) {
        const u32 s = idx / q16, k = idx - s * q16;
        const uint4* src =
            reinterpret_cast<const uint4*>(A.data + (lf.base + (u64)s * lf.stride) * A.elem_bytes);
        cp_async16(slot_chunks(sm, A, s) + k, src + k);
      }
      for (u32 s = tid; s < cl.nload; s += nthr) {
        const long long* top = reinterpret_cast<const long long*>(
            A.data + (lf.base + (u64)s * lf.stride) * A.elem_bytes + A.N / 8);
        const long long hi = __ldcg(top);
        signed char* pp = slot_pend(sm, A, s);
        pp[C - 1] = (signed char)hi;
      }
      const u32 ptotal = cl.nload * (C - 1);
      for (u32 idx = tid; idx < ptotal; idx += nthr) {
        const u32 s = idx / (C - 1), c = idx - s * (C - 1);
        slot_pend(sm, A, s)[c] = 0;
      }
      cp_async_wait_all();
    }
    __syncthreads();
    if (cl.has_pre) rotate_slots(sm, A, 0, cl.nload, A.rots + cl.pre_begin, lf.s);

    // ---- micro-op levels ------------------------------------------------------
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
          const u32 t = tid + k * nthr;
          if (t < ntask) {
            const DevOp op = A.ops[ob + t / C];
            run_op_task(sm, A, op, t % C, T[k]);
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k)
          if (T[k].mask) write_task(sm, A, T[k]);
        __syncthreads();
      }
    }

    // ---- post-rotation, carry resolution, store --------------------------------
    rotate_slots(sm, A, 0, cl.nstore, A.rots + cl.post_begin, lf.s);
    resolve_slots(sm, A, cl.nstore);
    {
      const u32 q16 = D / 4;
      const u32 total = cl.nstore * q16;
      for (u32 idx = tid; idx < total; idx += nthr) {
        const u32 s = idx / q16, k = idx - s * q16;
        uint4* dst = reinterpret_cast<uint4*>(A.data + (lf.base + (u64)s * lf.stride) * A.elem_bytes);
        __stcg(dst + k, slot_chunks(sm, A, s)[k]);
      }
      for (u32 s = tid; s < cl.nstore; s += nthr) {
        long long* top = reinterpret_cast<long long*>(A.data + (lf.base + (u64)s * lf.stride) * A.elem_bytes +
                                                      A.N / 8);
        __stcg(top, (long long)slot_pend(sm, A, s)[C - 1]);
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0 && lf.comp != kNoDep) {
      // bump the phase counter; the last child of a node's last phase
      // finishes the node and reports to the parent phase in turn
      u32 k = lf.comp;
      for (;;) {
        const u32 old = atomicAdd(&A.counters[1 + k], 1u);
        const DevCounter cm = A.cmeta[k];
        if (old + 1 != cm.target || cm.next == kNoDep) break;
        __threadfence();
        k = cm.next;
      }
    }
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
