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
  // network classes (DevClass::wnet 1 DIF / 2 DIT): per butterfly (level l,
  // index j < L/2) omega^r 2^64 mod p at ntw[wop_begin + l L/2 + j]; 0 = r 0
  const u64* ntw;
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

// Shared-memory slot index, padded by one word per 16 (a warp's 8-byte
// accesses at any power-of-two stride spread over the banks)
__device__ __forceinline__ u32 pdx(u32 i) { return i + (i >> 4); }

// Radix-2^NL group of a full network (levels l0 .. l0 + NL - 1) on one
// element set {base + m hs} of leaf j (slot k of leaf j at k G + j).
template <int NL, bool DIF>
__device__ __forceinline__ void net_group(u64* slot, u32 G, u32 j, u32 base, u32 hs, u32 l0, u32 half,
                                          const u64* tw, u64 p, u64 pinv) {
  constexpr u32 R = 1u << NL;
  u64 v[R];
#pragma unroll
  for (u32 m = 0; m < R; ++m) v[m] = slot[pdx((base + m * hs) * G + j)];
#pragma unroll
  for (u32 t = 0; t < NL; ++t) {
    const u32 sp = DIF ? (R >> (t + 1)) : (1u << t);  // span in units of hs
    const u32 h = sp * hs;
    const u32 lvl = l0 + t;
#pragma unroll
    for (u32 m = 0; m < R; ++m) {
      if (m & sp) continue;
      const u32 a = base + m * hs;
      const u32 jb = (a / (2 * h)) * h + a % h;
      const u64 w = __ldg(tw + (u64)lvl * half + jb);
      const u64 b = w ? montmul(v[m + sp], w, p, pinv) : v[m + sp];
      const u64 x = v[m];
      v[m] = addp(x, b, p);
      v[m + sp] = subp(x, b, p);
    }
  }
#pragma unroll
  for (u32 m = 0; m < R; ++m) slot[pdx((base + m * hs) * G + j)] = v[m];
}

template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT < 4 ? 4 : 1024 / NT) leaf_kernel(Args A) {
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
    // x / G for x < 2^24 as a high product (G <= 16)
    const u32 ginv = (u32)((0x100000000ull + G - 1) / G);
    auto divg = [&](u32 x) -> u32 { return G == 1 ? x : __umulhi(x, ginv); };
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
      const u32 k = divg(idx), j = idx - k * G;
      const u64 v = __ldcg(reinterpret_cast<const u64*>(A.data + (lf.base + j + (u64)k * lf.stride) * A.elem_bytes));
      if (cl.has_pre) {
        const SymExp P = A.rots[cl.pre_begin + k];
        slot[pdx(idx)] = twiddle(v, (P.a * wt(j) + P.b) & (A.M - 1));
      } else {
        slot[pdx(idx)] = v;
      }
    }
    __syncthreads();

    if (cl.wnet) {
      // a full radix-2 network (DIF: spans L/2 .. 1, DIT: 1 .. L/2; truncated
      // TFT inputs read as zeros): register groups of three levels, one
      // shared-memory round trip and barrier per group
      for (u32 idx = cl.nload * G + tid; idx < cl.L * G; idx += nthr) slot[pdx(idx)] = 0;
      __syncthreads();
      const bool dif = cl.wnet == 1;
      const u32 ell = 31 - __clz(cl.L), half = cl.L >> 1;
      const u64* tw = A.ntw + cl.wop_begin;
      for (u32 l0 = 0; l0 < ell; l0 += 3) {
        const u32 nl = ell - l0 < 3 ? ell - l0 : 3;
        const u32 hs = dif ? (cl.L >> (l0 + nl)) : (1u << l0);  // span of the group's last / first level
        const u32 lhs = 31 - __clz(hs);
        const u32 nsets = cl.L >> nl;
        for (u32 task = tid; task < nsets * G; task += nthr) {
          const u32 set = divg(task), j = task - set * G;
          const u32 base = ((set >> lhs) << (lhs + nl)) | (set & (hs - 1));
          if (nl == 3) {
            if (dif) net_group<3, true>(slot, G, j, base, hs, l0, half, tw, p, pinv);
            else net_group<3, false>(slot, G, j, base, hs, l0, half, tw, p, pinv);
          } else if (nl == 2) {
            if (dif) net_group<2, true>(slot, G, j, base, hs, l0, half, tw, p, pinv);
            else net_group<2, false>(slot, G, j, base, hs, l0, half, tw, p, pinv);
          } else {
            if (dif) net_group<1, true>(slot, G, j, base, hs, l0, half, tw, p, pinv);
            else net_group<1, false>(slot, G, j, base, hs, l0, half, tw, p, pinv);
          }
        }
        __syncthreads();
      }
    }
    // tasks = (op, leaf j), j fastest; the ops of a level touch disjoint
    // slots (Planner: dependency levels), so each task writes its results
    // straight back and one barrier ends the level
    for (u32 l = 0; l < (cl.wnet ? 0u : cl.nlevels); ++l) {
      const u32 o0 = A.levels[cl.level_begin + l], o1 = A.levels[cl.level_begin + l + 1];
      const u32 ntasks = (o1 - o0) * G;
      for (u32 task = tid; task < ntasks; task += nthr) {
        const u32 oi = divg(task), j = task - oi * G;
        const DevOp op = A.ops[o0 + oi];
        const u32 sa = pdx(op.a * G + j), sb = pdx(op.b * G + j);
        const u64 a = slot[sa];
        switch (op.type) {
          case OP_COPY:
            slot[sb] = a;
            break;
          case OP_DBL:
            slot[sa] = addp(a, a, p);
            break;
          case OP_HALF:
            slot[sa] = halfp(a, p);
            break;
          default: {
            // op.pad2 = omega^r 2^64 mod p (host-computed, upload())
            const u64 b = op.r ? montmul(slot[sb], op.pad2, p, pinv) : slot[sb];
            switch (op.type) {
              case OP_ADDSUB:
                slot[sa] = addp(a, b, p);
                slot[sb] = subp(a, b, p);
                break;
              case OP_ADD:
                slot[sa] = addp(a, b, p);
                break;
              case OP_SUB2:
                slot[sa] = subp(addp(a, a, p), b, p);
                break;
              case OP_SUB2DIFF:
                slot[sa] = subp(addp(a, a, p), b, p);
                slot[sb] = subp(a, b, p);
                break;
              case OP_ADDHALF:
                slot[sa] = halfp(addp(a, b, p), p);
                break;
              default:
                break;
            }
          }
        }
      }
      __syncthreads();
    }

    // store through the post-rotations
    for (u32 idx = tid; idx < cl.nstore * G; idx += nthr) {
      const u32 k = divg(idx), j = idx - k * G;
      const SymExp P = A.rots[cl.post_begin + k];
      u64* dst = reinterpret_cast<u64*>(A.data + (lf.base + j + (u64)k * lf.stride) * A.elem_bytes);
      __stcg(dst, twiddle(slot[pdx(idx)], (P.a * wt(j) + P.b) & (A.M - 1)));
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
