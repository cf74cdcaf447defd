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
  u32 logC;
};

__device__ __forceinline__ uint4* slot_chunks(std::uint8_t* sm, const Args& A, u32 s) {
  return reinterpret_cast<uint4*>(sm + (size_t)s * A.slot_bytes);
}
__device__ __forceinline__ signed char* slot_pend(std::uint8_t* sm, const Args& A, u32 s) {
  return reinterpret_cast<signed char*>(sm + (size_t)s * A.slot_bytes + 4u * A.D);
}

// ---- 128-bit chunk arithmetic on u32 words with PTX carry chains -------------

struct Ch {
  u32 w[4];
};
__device__ __forceinline__ Ch ld_ch(const uint4* p) {
  const uint4 v = *p;
  return Ch{{v.x, v.y, v.z, v.w}};
}
__device__ __forceinline__ void st_ch(uint4* p, const Ch& c) { *p = make_uint4(c.w[0], c.w[1], c.w[2], c.w[3]); }

// r = a + b; returns the carry out (0/1)
__device__ __forceinline__ int ch_add(Ch& r, const Ch& a, const Ch& b) {
  u32 c;
  asm("add.cc.u32 %0, %5, %9;\n\t"
      "addc.cc.u32 %1, %6, %10;\n\t"
      "addc.cc.u32 %2, %7, %11;\n\t"
      "addc.cc.u32 %3, %8, %12;\n\t"
      "addc.u32 %4, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]),
        "r"(b.w[3]));
  return (int)c;
}
// r = a - b; returns the borrow as -1/0
__device__ __forceinline__ int ch_sub(Ch& r, const Ch& a, const Ch& b) {
  u32 c;
  asm("sub.cc.u32 %0, %5, %9;\n\t"
      "subc.cc.u32 %1, %6, %10;\n\t"
      "subc.cc.u32 %2, %7, %11;\n\t"
      "subc.cc.u32 %3, %8, %12;\n\t"
      "subc.u32 %4, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]),
        "r"(b.w[3]));
  return (int)c;
}
// r += k (k small signed, sign-extended); returns the signed carry (-1/0/1)
__device__ __forceinline__ int ch_add_small(Ch& r, int k) {
  const u32 e = (u32)(k >> 31);
  u32 c;
  asm("add.cc.u32 %0, %0, %5;\n\t"
      "addc.cc.u32 %1, %1, %6;\n\t"
      "addc.cc.u32 %2, %2, %6;\n\t"
      "addc.cc.u32 %3, %3, %6;\n\t"
      "addc.u32 %4, %6, 0;"
      : "+r"(r.w[0]), "+r"(r.w[1]), "+r"(r.w[2]), "+r"(r.w[3]), "=r"(c)
      : "r"((u32)k), "r"(e));
  return (int)c;
}
__device__ __forceinline__ Ch ch_not(const Ch& a) { return Ch{{~a.w[0], ~a.w[1], ~a.w[2], ~a.w[3]}}; }

// A chunk value in "open" form: value = c + pb + adj * 2^128, with pb a small
// signed integer at bit 0 of the chunk and adj the chunk's carry-out.
struct Open {
  Ch c;
  int pb, adj;
};
__device__ __forceinline__ Open open_neg(const Open& x) {
  // -(c + pb + adj 2^128) = ~c + 1 - 2^128 - pb - adj 2^128
  return Open{ch_not(x.c), 1 - x.pb, -1 - x.adj};
}

// Rotation r (0 <= r < 2N) for windowed reads of omega^r * x.
struct Rot {
  int sigma;  // -1 when r >= N (2^N == -1)
  u32 q, o;   // t = r mod N = 128 q + o
};
__device__ __forceinline__ Rot make_rot(u64 r, u64 N) {
  Rot R;
  R.sigma = (r >= N) ? -1 : 1;
  const u64 t = (r >= N) ? r - N : r;
  R.q = (u32)(t >> 7);
  R.o = (u32)(t & 127);
  return R;
}

// 128-bit window [lo:hi] >> (128 - o) ... i.e. bits [128-o, 256-o) of hi:lo
// (o in 1..127): the chunk of (hi:lo) << o that lands in the upper half.
__device__ __forceinline__ Ch funnel_up(const Ch& lo, const Ch& hi, u32 o) {
  u32 W[8] = {lo.w[0], lo.w[1], lo.w[2], lo.w[3], hi.w[0], hi.w[1], hi.w[2], hi.w[3]};
  const u32 ow = o >> 5, ob = o & 31;
  Ch r;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // output word k of the upper half = bits [32(4+k) - o, ...) of W
    const int hiw = 4 + k - (int)ow;  // word holding the high part
    u32 h = 0, l = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      if (x == hiw) h = W[x];
      if (x == hiw - 1) l = W[x];
    }
    r.w[k] = ob ? __funnelshift_l(l, h, ob) : h;
  }
  return r;
}

// Chunk i of omega^r * x in open form (x a shared-memory slot), including the
// one pending carry of x that lands inside it.
__device__ __forceinline__ Open rot_chunk(const uint4* xc, const signed char* xp, const Rot& R,
                                          u32 C, u32 i) {
  const u32 Cm = C - 1;
  const u32 j = (i - R.q) & Cm;  // source chunk of the upper part
  const u32 jm = (j - 1) & Cm;   // lower part / landed pending (top of chunk jm)
  Open v;
  if (R.o == 0) {
    // aligned: chunk j moves whole, its bottom pending (top of jm) with it
    v.c = ld_ch(xc + j);
    v.pb = (int)xp[jm];
    v.adj = 0;
    const bool neg = (i < R.q) != (R.sigma < 0);
    if (i == R.q) v.pb = -v.pb;  // the element's top carry wraps: 2^N == -1
    if (neg) v = open_neg(v);
    return v;
  }
  const Ch lo = ld_ch(xc + jm), hi = ld_ch(xc + j);
  const int p = (int)xp[jm];
  // p * 2^o as a 160-bit signed value folded into the window
  const u32 ow = R.o >> 5, ob = R.o & 31;
  const long long pw = (long long)p * (1ll << ob);  // < 2^40 in magnitude
  Ch P;
  const u32 ext = (u32)(p >> 31);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    P.w[k] = ((u32)k < ow) ? 0u : ((u32)k == ow ? (u32)pw : ((u32)k == ow + 1 ? (u32)(pw >> 32) : ext));
  }
  const int ptop = (ow == 3) ? (int)(pw >> 32) : (int)ext;  // word 4 of p*2^o (sign extension)
  if (i != R.q) {
    v.c = funnel_up(lo, hi, R.o);
    const int c = ch_add(v.c, v.c, P);
    v.pb = 0;
    v.adj = c + ptop;
    const bool neg = (i < R.q) != (R.sigma < 0);
    if (neg) v = open_neg(v);
    return v;
  }
  // the chunk holding bit t: upper bits from chunk 0 (positive), lower bits
  // from the top of chunk C-1 (wrapped, negative), and the wrapped top carry
  Ch up = funnel_up(Ch{{0, 0, 0, 0}}, hi, R.o);
  Ch dn = funnel_up(lo, Ch{{0, 0, 0, 0}}, R.o);
  // value = up - dn - p*2^o
  int c1 = ch_sub(v.c, up, dn);
  int c2 = ch_sub(v.c, v.c, P);
  v.pb = 0;
  v.adj = c1 + c2 - ptop;
  if (R.sigma < 0) v = open_neg(v);
  return v;
}

struct TaskOut {
  Ch w0, w1;
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
    T.w1 = ld_ch(ac + i);
    T.p1 = ap[i];
    T.mask = 2;
    return;
  }
  const Rot R = make_rot(op.r, A.N);
  const Open b = rot_chunk(slot_chunks(sm, A, op.b), slot_pend(sm, A, op.b), R, C, i);
  const Ch a = ld_ch(ac + i);
  const int pa = i ? (int)ap[i - 1] : -(int)ap[C - 1];
  // S = a + b, T = a - b (open form, exact)
  Ch S, D;
  int cs = ch_add(S, a, b.c);
  cs += ch_add_small(S, pa + b.pb);
  cs += b.adj;
  int cd = ch_sub(D, a, b.c);
  cd += ch_add_small(D, pa - b.pb);
  cd -= b.adj;
  switch (op.type) {
    case OP_ADDSUB:
      T.w0 = S;
      T.p0 = (signed char)cs;
      T.w1 = D;
      T.p1 = (signed char)cd;
      T.mask = 3;
      break;
    case OP_ADD:
      T.w0 = S;
      T.p0 = (signed char)cs;
      T.mask = 1;
      break;
    default: {  // OP_SUB2 / OP_SUB2DIFF: out0 = a + (a - b)
      Ch E;
      int ce = ch_add(E, a, D);
      ce += ch_add_small(E, pa);
      T.w0 = E;
      T.p0 = (signed char)(ce + cd);
      if (op.type == OP_SUB2DIFF) {
        T.w1 = D;
        T.p1 = (signed char)cd;
        T.mask = 3;
      } else {
        T.mask = 1;
      }
    }
  }
}

__device__ __forceinline__ void write_task(std::uint8_t* sm, const Args& A, const TaskOut& T) {
  if (T.mask & 1) {
    st_ch(slot_chunks(sm, A, T.sa) + T.chunk, T.w0);
    slot_pend(sm, A, T.sa)[T.chunk] = T.p0;
  }
  if (T.mask & 2) {
    st_ch(slot_chunks(sm, A, T.sb) + T.chunk, T.w1);
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
    Ch w[kTasksPerThread];
    signed char p[kTasksPerThread];
#pragma unroll
    for (int k = 0; k < kTasksPerThread; ++k) {
      const u32 t = tid + k * nthr;
      if (t < ntask) {
        const u32 sl = s0 + b0 + (t >> A.logC), i = t & (C - 1);
        const u64 r = (rot[sl].a * s + rot[sl].b) & (A.M - 1);
        const Open v = rot_chunk(slot_chunks(sm, A, sl), slot_pend(sm, A, sl), make_rot(r, A.N), C, i);
        w[k] = v.c;
        p[k] = (signed char)(v.adj + ch_add_small(w[k], v.pb));
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTasksPerThread; ++k) {
      const u32 t = tid + k * nthr;
      if (t < ntask) {
        const u32 sl = s0 + b0 + (t >> A.logC), i = t & (C - 1);
        st_ch(slot_chunks(sm, A, sl) + i, w[k]);
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
      Ch w[kTasksPerThread];
      int e[kTasksPerThread];
      int any = 0;
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        const u32 t = tid + k * nthr;
        e[k] = 0;
        if (t < ntask) {
          const u32 sl = b0 + (t >> A.logC), i = t & (C - 1);
          const signed char* pp = slot_pend(sm, A, sl);
          const int in = i ? (int)pp[i - 1] : 0;
          w[k] = ld_ch(slot_chunks(sm, A, sl) + i);
          const int carry = in ? ch_add_small(w[k], in) : 0;
          e[k] = (i == C - 1) ? (int)pp[C - 1] + carry : carry;
          if (i != C - 1 && carry != 0) any = 1;
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        const u32 t = tid + k * nthr;
        if (t < ntask) {
          const u32 sl = b0 + (t >> A.logC), i = t & (C - 1);
          st_ch(slot_chunks(sm, A, sl) + i, w[k]);
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
            const DevOp op = A.ops[ob + (t >> A.logC)];
            run_op_task(sm, A, op, t & (C - 1), T[k]);
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
