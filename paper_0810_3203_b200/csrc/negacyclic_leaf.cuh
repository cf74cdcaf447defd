// negacyclic_leaf.cuh -- sm_100a leaf engine for R = (Z/mZ)[y]/(y^K+1), omega = y.
//
// Same persistent ticket/leaf structure as the Fermat engine.  An element is
// K u64 words in [0, m); a twiddle y^r is a negacyclic rotation of the word
// vector (no carries), add/sub are word-wise mod m, and half/double are
// word-wise (ctx.half / ctx.add(x,x) of transform.hpp restated for m odd).
// A task is one output word of one micro-op.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace negacyclic {

constexpr int kThreads = 512;
constexpr int kTasksPerThread = 8;

struct Args {
  std::uint8_t* data;
  u64 elem_bytes;
  const DevLeaf* leaves;
  u64 nleaves;
  const DevClass* classes;
  const DevOp* ops;
  const u32* levels;
  const SymExp* rots;
  u32* counters;           // [0]: ticket; [1 + k]: (node, phase) completion counters
  const DevCounter* cmeta;
  u64 K, M, m;
  u32 slot_bytes;
};

__device__ __forceinline__ u64 addm(u64 a, u64 b, u64 m) {
  u64 s = a + b;
  return s >= m ? s - m : s;
}
__device__ __forceinline__ u64 subm(u64 a, u64 b, u64 m) { return a >= b ? a - b : a + (m - b); }
__device__ __forceinline__ u64 negm(u64 a, u64 m) { return a ? m - a : 0; }
__device__ __forceinline__ u64 halfm(u64 a, u64 m) { return (a & 1) ? (a >> 1) + (m >> 1) + 1 : a >> 1; }

// Word j of y^r * x (0 <= r < 2K).
__device__ __forceinline__ u64 rot_word(const u64* x, u64 r, u64 K, u64 m, u64 j) {
  bool neg = r >= K;
  const u64 t = neg ? r - K : r;
  u64 src;
  if (j >= t) {
    src = j - t;
  } else {
    src = j + K - t;
    neg = !neg;
  }
  const u64 v = x[src];
  return neg ? negm(v, m) : v;
}

__device__ __forceinline__ u32 ld_acquire(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct TaskOut {
  u64 v0, v1;
  std::uint16_t sa, sb;
  u32 j;
  std::uint8_t mask;
};

__global__ void __launch_bounds__(kThreads, 1) leaf_kernel(Args A) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  __shared__ u32 s_ticket;
  const u32 tid = threadIdx.x, nthr = blockDim.x;
  const u64 K = A.K, m = A.m;
  const u32 Kw = (u32)K;
  auto slot = [&](u32 s) { return reinterpret_cast<u64*>(sm + (size_t)s * A.slot_bytes); };

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

    {
      const u32 q16 = (u32)(K / 2);
      const u32 total = cl.nload * q16;
      for (u32 idx = tid; idx < total; idx += nthr) {
        const u32 s = idx / q16, k = idx - s * q16;
        const uint4* src =
            reinterpret_cast<const uint4*>(A.data + (lf.base + (u64)s * lf.stride) * A.elem_bytes);
        reinterpret_cast<uint4*>(slot(s))[k] = __ldcg(src + k);
      }
    }
    __syncthreads();

    // pre-rotations (ITFT spectral inputs), batched through registers
    if (cl.has_pre) {
      const u32 per = max(1u, (nthr * kTasksPerThread) / Kw);
      for (u32 b0 = 0; b0 < cl.nload; b0 += per) {
        const u32 ntask = min(cl.nload - b0, per) * Kw;
        u64 v[kTasksPerThread];
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          const u32 t = tid + k * nthr;
          if (t < ntask) {
            const u32 sl = b0 + t / Kw, j = t % Kw;
            const SymExp P = A.rots[cl.pre_begin + sl];
            v[k] = rot_word(slot(sl), (P.a * lf.s + P.b) & (A.M - 1), K, m, j);
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          const u32 t = tid + k * nthr;
          if (t < ntask) slot(b0 + t / Kw)[t % Kw] = v[k];
        }
        __syncthreads();
      }
    }

    const u32 ops_per_batch = max(1u, (nthr * kTasksPerThread) / Kw);
    for (u32 l = 0; l < cl.nlevels; ++l) {
      const u32 o0 = A.levels[cl.level_begin + l], o1 = A.levels[cl.level_begin + l + 1];
      for (u32 ob = o0; ob < o1; ob += ops_per_batch) {
        const u32 oe = min(o1, ob + ops_per_batch);
        const u32 ntask = (oe - ob) * Kw;
        TaskOut T[kTasksPerThread];
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          T[k].mask = 0;
          const u32 t = tid + k * nthr;
          if (t >= ntask) continue;
          const DevOp op = A.ops[ob + t / Kw];
          const u32 j = t % Kw;
          T[k].sa = op.a;
          T[k].sb = op.b;
          T[k].j = j;
          const u64 a = slot(op.a)[j];
          switch (op.type) {
            case OP_COPY:
              T[k].v1 = a;
              T[k].mask = 2;
              break;
            case OP_DBL:
              T[k].v0 = addm(a, a, m);
              T[k].mask = 1;
              break;
            case OP_HALF:
              T[k].v0 = halfm(a, m);
              T[k].mask = 1;
              break;
            default: {
              const u64 b = rot_word(slot(op.b), op.r, K, m, j);
              switch (op.type) {
                case OP_ADDSUB:
                  T[k].v0 = addm(a, b, m);
                  T[k].v1 = subm(a, b, m);
                  T[k].mask = 3;
                  break;
                case OP_ADD:
                  T[k].v0 = addm(a, b, m);
                  T[k].mask = 1;
                  break;
                case OP_SUB2:
                  T[k].v0 = subm(addm(a, a, m), b, m);
                  T[k].mask = 1;
                  break;
                case OP_SUB2DIFF:
                  T[k].v0 = subm(addm(a, a, m), b, m);
                  T[k].v1 = subm(a, b, m);
                  T[k].mask = 3;
                  break;
                case OP_ADDHALF:
                  T[k].v0 = halfm(addm(a, b, m), m);
                  T[k].mask = 1;
                  break;
                default:
                  break;
              }
            }
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          if (T[k].mask & 1) slot(T[k].sa)[T[k].j] = T[k].v0;
          if (T[k].mask & 2) slot(T[k].sb)[T[k].j] = T[k].v1;
        }
        __syncthreads();
      }
    }

    // store with the post-rotation
    const u32 total = cl.nstore * Kw;
    for (u32 idx = tid; idx < total; idx += nthr) {
      const u32 si = idx / Kw, j = idx - si * Kw;
      const SymExp P = A.rots[cl.post_begin + si];
      u64* dst = reinterpret_cast<u64*>(A.data + (lf.base + (u64)si * lf.stride) * A.elem_bytes);
      __stcg(dst + j, rot_word(slot(si), (P.a * lf.s + P.b) & (A.M - 1), K, m, j));
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

}  // namespace negacyclic
}  // namespace cftft_b200
