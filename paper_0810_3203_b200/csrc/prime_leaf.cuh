// prime_leaf.cuh -- sm_100a leaf engine for the reference's own ring: Z/pZ,
// p an odd 64-bit prime with 2^m | p - 1, omega of order M = 2^m (the
// reference's RingCtx, field.hpp:84-185; Goldilocks p = 2^64 - 2^32 + 1,
// m = 32 is its default).  One coefficient is one u64 word in [0, p).
//
// Same persistent ticket/leaf structure and the same ring-agnostic leaf
// programs as the negacyclic engine (negacyclic_leaf.cuh): a task is one
// micro-op; omega^r is a Montgomery product with a two-level table of powers
// (omega^(r mod 2^16) and omega^(2^16 floor(r / 2^16)), kept times 2^64 mod p,
// so a product with a table entry lands back in normal form); add / sub /
// half / double are mod p with the carry of p > 2^63 handled.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace prime {

constexpr int kThreads = 128;
constexpr int kTasksPerThread = 4;

struct Args {
  std::uint8_t* data;
  u64 elem_bytes;
  const DevLeaf* leaves;
  u64 nleaves;
  const DevClass* classes;
  const DevOp* ops;
  const u32* levels;
  const SymExp* rots;
  u32* counters;  // [0]: ticket; [1 + k]: (node, phase) completion counters
  const DevCounter* cmeta;
  u64 M, p, pinv;      // pinv = -p^-1 mod 2^64
  const u64* tw_lo;    // omega^i 2^64 mod p, i < 2^lo_bits
  const u64* tw_hi;    // omega^(i 2^lo_bits) 2^64 mod p
  u32 lo_bits;
  u32 slot_bytes;
  const u32* groups;  // tickets = {first leaf, count} (Plan::groups), or null: one leaf each
};

__device__ __forceinline__ u64 addp(u64 a, u64 b, u64 p) {
  const u64 s = a + b;
  return (s < a || s >= p) ? s - p : s;  // (a wrap past 2^64 is a value >= p)
}
__device__ __forceinline__ u64 subp(u64 a, u64 b, u64 p) { return a >= b ? a - b : a - b + p; }
__device__ __forceinline__ u64 halfp(u64 a, u64 p) { return (a & 1) ? (a >> 1) + (p >> 1) + 1 : a >> 1; }
// a b 2^-64 mod p (a, b < p)
__device__ __forceinline__ u64 montmul(u64 a, u64 b, u64 p, u64 pinv) {
  const u64 lo = a * b, hi = __umul64hi(a, b);
  const u64 mq = lo * pinv;
  const u64 mh = __umul64hi(mq, p);
  // (a b + mq p) / 2^64 = hi + mh + (lo != 0) < 2p
  const u64 s = hi + mh;
  const bool c1 = s < hi;
  const u64 s2 = s + (lo != 0 ? 1u : 0u);
  const bool c2 = s2 < s;
  return (c1 || c2 || s2 >= p) ? s2 - p : s2;
}

__device__ __forceinline__ u32 ld_acquire(const u32* c) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(c) : "memory");
  return v;
}

__global__ void __launch_bounds__(kThreads) leaf_kernel(Args A) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  __shared__ u32 s_ticket;
  __shared__ u64 s_w[32];  // weights of the ticket's leaves
  const u32 tid = threadIdx.x, nthr = blockDim.x;
  const u64 p = A.p, pinv = A.pinv;
  const u64 lomask = (u64{1} << A.lo_bits) - 1;
  u64* const slot = reinterpret_cast<u64*>(sm);
  // x omega^r (r < M)
  auto twiddle = [&](u64 x, u64 r) -> u64 {
    if (r == 0) return x;
    u64 t = A.tw_lo[r & lomask];
    if (r >> A.lo_bits) t = montmul(t, A.tw_hi[r >> A.lo_bits], p, pinv);
    return montmul(x, t, p, pinv);
  };

  for (;;) {
    if (tid == 0) s_ticket = atomicAdd(&A.counters[0], 1u);
    __syncthreads();
    const u32 ticket = s_ticket;
    if (ticket >= A.nleaves) return;
    // a ticket is G >= 1 leaves on adjacent coefficients (Planner::group_leaves):
    // leaf j starts at base + j, with its own weight, dependency and counter;
    // slot k of leaf j sits at k G + j
    const u32 first = A.groups ? A.groups[2 * ticket] : ticket;
    const u32 G = A.groups ? A.groups[2 * ticket + 1] : 1u;
    const DevLeaf lf = A.leaves[first];
    const DevClass cl = A.classes[lf.cls];
    if (tid < G) {
      const DevLeaf lj = A.leaves[first + tid];
      s_w[tid] = lj.s;
      if (lj.dep != kNoDep) {
        const u32* c = &A.counters[1 + lj.dep];
        while (ld_acquire(c) < lj.dep_target) __nanosleep(64);
      }
    }
    __syncthreads();
    auto wt = [&](u32 j) -> u64 { return s_w[j] & (A.M - 1); };
    // load through the pre-rotations (the ITFT's spectral inputs)
    for (u32 idx = tid; idx < cl.nload * G; idx += nthr) {
      const u32 k = idx / G, j = idx - k * G;
      const u64 v = __ldcg(reinterpret_cast<const u64*>(A.data + (lf.base + j + (u64)k * lf.stride) * A.elem_bytes));
      if (cl.has_pre) {
        const SymExp P = A.rots[cl.pre_begin + k];
        slot[idx] = twiddle(v, (P.a * wt(j) + P.b) & (A.M - 1));
      } else {
        slot[idx] = v;
      }
    }
    __syncthreads();

    // tasks = (op, leaf j), j fastest
    const u32 tasks_per_batch = nthr * kTasksPerThread;
    for (u32 l = 0; l < cl.nlevels; ++l) {
      const u32 o0 = A.levels[cl.level_begin + l], o1 = A.levels[cl.level_begin + l + 1];
      const u32 ntasks = (o1 - o0) * G;
      for (u32 tb = 0; tb < ntasks; tb += tasks_per_batch) {
        u64 v0[kTasksPerThread], v1[kTasksPerThread];
        u32 sa[kTasksPerThread], sb[kTasksPerThread], mask[kTasksPerThread];
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          mask[k] = 0;
          const u32 task = tb + tid + k * nthr;
          if (task >= ntasks) continue;
          const u32 oi = task / G, j = task - oi * G;
          const DevOp op = A.ops[o0 + oi];
          sa[k] = op.a * G + j;
          sb[k] = op.b * G + j;
          const u64 a = slot[sa[k]];
          switch (op.type) {
            case OP_COPY:
              v1[k] = a;
              mask[k] = 2;
              break;
            case OP_DBL:
              v0[k] = addp(a, a, p);
              mask[k] = 1;
              break;
            case OP_HALF:
              v0[k] = halfp(a, p);
              mask[k] = 1;
              break;
            default: {
              const u64 b = twiddle(slot[sb[k]], op.r);
              switch (op.type) {
                case OP_ADDSUB:
                  v0[k] = addp(a, b, p);
                  v1[k] = subp(a, b, p);
                  mask[k] = 3;
                  break;
                case OP_ADD:
                  v0[k] = addp(a, b, p);
                  mask[k] = 1;
                  break;
                case OP_SUB2:
                  v0[k] = subp(addp(a, a, p), b, p);
                  mask[k] = 1;
                  break;
                case OP_SUB2DIFF:
                  v0[k] = subp(addp(a, a, p), b, p);
                  v1[k] = subp(a, b, p);
                  mask[k] = 3;
                  break;
                case OP_ADDHALF:
                  v0[k] = halfp(addp(a, b, p), p);
                  mask[k] = 1;
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
          if (mask[k] & 1) slot[sa[k]] = v0[k];
          if (mask[k] & 2) slot[sb[k]] = v1[k];
        }
        __syncthreads();
      }
    }

    // store through the post-rotations
    for (u32 idx = tid; idx < cl.nstore * G; idx += nthr) {
      const u32 k = idx / G, j = idx - k * G;
      const SymExp P = A.rots[cl.post_begin + k];
      u64* dst = reinterpret_cast<u64*>(A.data + (lf.base + j + (u64)k * lf.stride) * A.elem_bytes);
      __stcg(dst, twiddle(slot[idx], (P.a * wt(j) + P.b) & (A.M - 1)));
    }
    __threadfence();
    __syncthreads();
    if (tid < G && A.leaves[first + tid].comp != kNoDep) {
      // bump the leaf's phase counter; the last child of a node's last phase
      // finishes the node and reports to the parent phase in turn
      u32 k = A.leaves[first + tid].comp;
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

}  // namespace prime
}  // namespace cftft_b200
