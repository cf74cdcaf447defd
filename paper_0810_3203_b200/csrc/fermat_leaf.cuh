// fermat_leaf.cuh -- sm_100a leaf engine for R = Z/(2^N+1), omega = 2.
//
// One persistent launch runs a whole transform.  Each CTA repeatedly takes a
// ticket (a leaf: a sub-transform of <= 2^max_ell coefficients that fits in
// shared memory), waits until the (node, phase) counter it depends on is
// complete, runs the leaf, and bumps the counter it completes.  Tickets are
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
//   operand b (plus the one pending carry of b landing inside it), with PTX
//   add.cc/addc chains; its carry out becomes the new pending carry of chunk
//   i.  No cross-thread carry propagation happens inside a leaf: carries are
//   resolved once per stored slot, fused with the final rotation and the
//   store to global memory.
//
// Global (HBM) element format between levels: N/64 u64 limbs "lo" plus a
// signed top word hi, value = lo + hi*2^N (== lo - hi).  Canonical inputs
// (top in {0,1}) are a special case; the last step canonicalises.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace fermat {

constexpr int kThreads = 512;
constexpr int kTasksPerThread = 4;
constexpr u32 kMaxBatch = 256;  // ops (or slots) staged per batch

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
  const DevCounter* cmeta; // per-counter target and parent link
  u64 N, M;
  u32 D, C;                // u32 words, 128-bit chunks per element
  u32 logC;
  u32 slot_bytes;          // 4*D + pending bytes (16B aligned)
  u32 scratch_off;         // byte offset of the carry scratch
};

// ---- 128-bit chunk arithmetic on u32 words with PTX carry chains -------------

struct Ch {
  u32 w[4];
};
__device__ __forceinline__ Ch lds_ch(u32 addr) {
  Ch c;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3])
               : "r"(addr));
  return c;
}
__device__ __forceinline__ void sts_ch(u32 addr, const Ch& c) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(c.w[0]), "r"(c.w[1]),
               "r"(c.w[2]), "r"(c.w[3])
               : "memory");
}
__device__ __forceinline__ int lds_s8(u32 addr) {
  int v;
  asm volatile("ld.shared.s8 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_s8(u32 addr, int v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

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
__device__ __forceinline__ Ch ch_xor(const Ch& a, u32 m) {
  return Ch{{a.w[0] ^ m, a.w[1] ^ m, a.w[2] ^ m, a.w[3] ^ m}};
}

// A chunk value in "open" form: value = c + pb + adj * 2^128, with pb a small
// signed integer at bit 0 of the chunk and adj the chunk's carry-out.
struct Open {
  Ch c;
  int pb, adj;
};
// conditional negation: -(c + pb + adj 2^128) = ~c + (1 - pb) + (-1 - adj) 2^128
__device__ __forceinline__ Open open_cneg(const Open& x, bool neg) {
  const u32 m = neg ? 0xFFFFFFFFu : 0u;
  return Open{ch_xor(x.c, m), neg ? 1 - x.pb : x.pb, neg ? -1 - x.adj : x.adj};
}

// Rotation r (0 <= r < 2N) for windowed reads of omega^r * x.
struct Rot {
  u32 q, o;   // t = r mod N = 128 q + o
  u32 sneg;   // 1 when r >= N (2^N == -1)
};
__device__ __forceinline__ Rot make_rot(u64 r, u64 N) {
  Rot R;
  R.sneg = (r >= N) ? 1u : 0u;
  const u64 t = R.sneg ? r - N : r;
  R.q = (u32)(t >> 7);
  R.o = (u32)(t & 127);
  return R;
}

// Upper 128 bits of (hi:lo) << o, 0 < o < 128.
__device__ __forceinline__ Ch funnel_up(const Ch& lo, const Ch& hi, u32 o) {
  const u32 W[8] = {lo.w[0], lo.w[1], lo.w[2], lo.w[3], hi.w[0], hi.w[1], hi.w[2], hi.w[3]};
  const u32 ow = o >> 5, ob = o & 31;
  Ch r;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    u32 h = 0, l = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      if (x == 4 + k - (int)ow) h = W[x];
      if (x == 3 + k - (int)ow) l = W[x];
    }
    r.w[k] = __funnelshift_l(l, h, ob);
  }
  return r;
}

// Chunk i of omega^r * x in open form; x = (chunk base address, pending base
// address) in shared memory.  Includes the one pending carry of x that lands
// inside the chunk.
__device__ __forceinline__ Open rot_chunk(u32 xw, u32 xp, const Rot& R, u32 Cm, u32 i) {
  const u32 j = (i - R.q) & Cm;  // source chunk of the upper part
  const u32 jm = (j - 1) & Cm;   // lower part / landed pending (top of chunk jm)
  Open v;
  if (R.o == 0) {
    // aligned: chunk j moves whole, its bottom pending (top of chunk jm) with it
    v.c = lds_ch(xw + 16 * j);
    v.pb = lds_s8(xp + jm);
    v.adj = 0;
    if (i == R.q) v.pb = -v.pb;  // the element's top carry wraps: 2^N == -1
    return open_cneg(v, ((i < R.q) ? 1u : 0u) != R.sneg);
  }
  const Ch lo = lds_ch(xw + 16 * jm), hi = lds_ch(xw + 16 * j);
  const int p = lds_s8(xp + jm);
  // p * 2^o as a 160-bit signed value P (+ ptop * 2^128)
  const u32 ow = R.o >> 5, ob = R.o & 31;
  const long long pw = (long long)p * (1ll << ob);
  const u32 ext = (u32)(p >> 31);
  Ch P;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    P.w[k] = ((u32)k < ow) ? 0u : ((u32)k == ow ? (u32)pw : ((u32)k == ow + 1 ? (u32)(pw >> 32) : ext));
  const int ptop = (ow == 3) ? (int)(pw >> 32) : (int)ext;
  if (i != R.q) {
    v.c = funnel_up(lo, hi, R.o);
    v.adj = ch_add(v.c, v.c, P) + ptop;
    v.pb = 0;
    return open_cneg(v, ((i < R.q) ? 1u : 0u) != R.sneg);
  }
  // the chunk holding bit t: upper bits from chunk 0 (positive), lower bits
  // from the top of chunk C-1 (wrapped, negative), and the wrapped top carry
  const Ch z{{0, 0, 0, 0}};
  const Ch up = funnel_up(z, hi, R.o);
  const Ch dn = funnel_up(lo, z, R.o);
  const int c1 = ch_sub(v.c, up, dn);
  const int c2 = ch_sub(v.c, v.c, P);
  v.pb = 0;
  v.adj = c1 + c2 - ptop;
  return open_cneg(v, R.sneg != 0);
}

// Per-op parameters staged in shared memory once per batch.
struct OpT {
  u32 aw, bw;  // smem addresses of slot a / slot b (pending arrays at +W4)
  u32 q, o;
  u32 sneg, type;
};

struct TaskOut {
  Ch w0, w1;
  int p0, p1;
  u32 d0, d1;  // smem chunk destinations
  u32 mask;
};

__device__ __forceinline__ void run_op_task(const OpT& op, u32 W4, u32 Cm, u32 i, TaskOut& T) {
  T.d0 = op.aw + 16 * i;
  T.d1 = op.bw + 16 * i;
  if (op.type == OP_COPY) {  // b <- a verbatim
    T.w1 = lds_ch(op.aw + 16 * i);
    T.p1 = lds_s8(op.aw + W4 + i);
    T.mask = 2;
    return;
  }
  const Rot R{op.q, op.o, op.sneg};
  const Open b = rot_chunk(op.bw, op.bw + W4, R, Cm, i);
  const Ch a = lds_ch(op.aw + 16 * i);
  const int pa_raw = lds_s8(op.aw + W4 + ((i - 1) & Cm));
  const int pa = i ? pa_raw : -pa_raw;
  Ch S, D;
  int cs = ch_add(S, a, b.c);
  cs += ch_add_small(S, pa + b.pb) + b.adj;
  int cd = ch_sub(D, a, b.c);
  cd += ch_add_small(D, pa - b.pb) - b.adj;
  if (op.type == OP_ADDSUB) {
    T.w0 = S;
    T.p0 = cs;
    T.w1 = D;
    T.p1 = cd;
    T.mask = 3;
  } else if (op.type == OP_ADD) {
    T.w0 = S;
    T.p0 = cs;
    T.mask = 1;
  } else {  // OP_SUB2 / OP_SUB2DIFF: out0 = a + (a - b)
    Ch E;
    int ce = ch_add(E, a, D);
    ce += ch_add_small(E, pa);
    T.w0 = E;
    T.p0 = ce + cd;
    T.w1 = D;
    T.p1 = cd;
    T.mask = (op.type == OP_SUB2DIFF) ? 3 : 1;
  }
}

__device__ __forceinline__ void write_task(const TaskOut& T, u32 W4, u32 i) {
  if (T.mask & 1) {
    sts_ch(T.d0, T.w0);
    sts_s8(T.d0 - 16 * i + W4 + i, T.p0);
  }
  if (T.mask & 2) {
    sts_ch(T.d1, T.w1);
    sts_s8(T.d1 - 16 * i + W4 + i, T.p1);
  }
}

__device__ __forceinline__ void cp_async16(u32 saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ u32 ld_acquire(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kThreads, 1) leaf_kernel(Args A) {
  extern __shared__ __align__(16) std::uint8_t sm[];
  __shared__ u32 s_ticket;
  __shared__ OpT s_ops[kMaxBatch];
  __shared__ Rot s_rot[kMaxBatch];
  const u32 tid = threadIdx.x, nthr = blockDim.x;
  const u32 C = A.C, Cm = C - 1, logC = A.logC;
  const u32 smb = (u32)__cvta_generic_to_shared(sm);
  const u32 SB = A.slot_bytes, W4 = 4 * A.D;
  const u32 scr = smb + A.scratch_off;
  const u32 per_batch = min(kMaxBatch, max(1u, (nthr * kTasksPerThread) >> logC));

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
    std::uint8_t* const gbase = A.data + lf.base * A.elem_bytes;
    const u64 gstride = lf.stride * A.elem_bytes;

    // ---- load slots [0, nload) through L2 (written by other CTAs) -------------
    {
      const u32 total = cl.nload << logC;
      for (u32 idx = tid; idx < total; idx += nthr) {
        const u32 s = idx >> logC, k = idx & Cm;
        cp_async16(smb + s * SB + 16 * k, gbase + s * gstride + 16 * (u64)k);
      }
      for (u32 idx = tid; idx < total; idx += nthr) {
        const u32 s = idx >> logC, c = idx & Cm;
        int v = 0;
        if (c == Cm) v = (int)__ldcg(reinterpret_cast<const long long*>(gbase + s * gstride + W4));
        sts_s8(smb + s * SB + W4 + c, v);
      }
      cp_async_wait_all();
    }
    __syncthreads();

    // ---- pre-rotations (ITFT spectral inputs), in place through registers ---
    if (cl.has_pre) {
      for (u32 b0 = 0; b0 < cl.nload; b0 += per_batch) {
        const u32 nb = min(cl.nload - b0, per_batch);
        for (u32 x = tid; x < nb; x += nthr) {
          const SymExp P = A.rots[cl.pre_begin + b0 + x];
          s_rot[x] = make_rot((P.a * lf.s + P.b) & (A.M - 1), A.N);
        }
        __syncthreads();
        const u32 ntask = nb << logC;
        Ch w[kTasksPerThread];
        int p[kTasksPerThread];
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          const u32 t = tid + k * nthr;
          if (t < ntask) {
            const u32 x = t >> logC, i = t & Cm, sw = smb + (b0 + x) * SB;
            const Open v = rot_chunk(sw, sw + W4, s_rot[x], Cm, i);
            w[k] = v.c;
            p[k] = v.adj + ch_add_small(w[k], v.pb);
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          const u32 t = tid + k * nthr;
          if (t < ntask) {
            const u32 i = t & Cm, sw = smb + (b0 + (t >> logC)) * SB;
            sts_ch(sw + 16 * i, w[k]);
            sts_s8(sw + W4 + i, p[k]);
          }
        }
        __syncthreads();
      }
    }

    // ---- micro-op levels ------------------------------------------------------
    for (u32 l = 0; l < cl.nlevels; ++l) {
      const u32 o0 = A.levels[cl.level_begin + l], o1 = A.levels[cl.level_begin + l + 1];
      for (u32 ob = o0; ob < o1; ob += per_batch) {
        const u32 nb = min(o1 - ob, per_batch);
        for (u32 x = tid; x < nb; x += nthr) {
          const DevOp op = A.ops[ob + x];
          const Rot R = make_rot(op.r, A.N);
          s_ops[x] = OpT{smb + op.a * SB, smb + op.b * SB, R.q, R.o, R.sneg, op.type};
        }
        __syncthreads();
        const u32 ntask = nb << logC;
        TaskOut T[kTasksPerThread];
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k) {
          T[k].mask = 0;
          const u32 t = tid + k * nthr;
          if (t < ntask) run_op_task(s_ops[t >> logC], W4, Cm, t & Cm, T[k]);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kTasksPerThread; ++k)
          if (T[k].mask) write_task(T[k], W4, (tid + k * nthr) & Cm);
        __syncthreads();
      }
    }

    // ---- post-rotation + carry resolution + store, fused ------------------------
    for (u32 b0 = 0; b0 < cl.nstore; b0 += per_batch) {
      const u32 nb = min(cl.nstore - b0, per_batch);
      for (u32 x = tid; x < nb; x += nthr) {
        const SymExp P = A.rots[cl.post_begin + b0 + x];
        s_rot[x] = make_rot((P.a * lf.s + P.b) & (A.M - 1), A.N);
      }
      __syncthreads();
      const u32 ntask = nb << logC;
      Ch w[kTasksPerThread];
      int top[kTasksPerThread];
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        const u32 t = tid + k * nthr;
        if (t < ntask) {
          const u32 x = t >> logC, i = t & Cm, sw = smb + (b0 + x) * SB;
          const Open v = rot_chunk(sw, sw + W4, s_rot[x], Cm, i);
          w[k] = v.c;
          top[k] = v.adj + ch_add_small(w[k], v.pb);
          sts_s8(scr + t, top[k]);
        }
      }
      __syncthreads();
      // absorb the carry of the chunk below (one step); carries that ripple
      // further (a chunk of all ones / all zeros) take the slow path
      int rare = 0;
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        const u32 t = tid + k * nthr;
        if (t < ntask) {
          const u32 i = t & Cm;
          const int in = i ? lds_s8(scr + t - 1) : 0;
          const int e = in ? ch_add_small(w[k], in) : 0;
          if (i == Cm) {
            top[k] += e;
          } else {
            if (e) rare = 1;
            top[k] = e;  // carry still owed to chunk i+1
          }
        }
      }
      if (__syncthreads_or(rare)) {
        // sequential sweeps through shared memory (the slots are free now)
        for (;;) {
#pragma unroll
          for (int k = 0; k < kTasksPerThread; ++k) {
            const u32 t = tid + k * nthr;
            if (t < ntask && (t & Cm) != Cm) sts_s8(scr + t, top[k]);
          }
          __syncthreads();
          int any = 0;
#pragma unroll
          for (int k = 0; k < kTasksPerThread; ++k) {
            const u32 t = tid + k * nthr;
            if (t < ntask) {
              const u32 i = t & Cm;
              const int in = i ? lds_s8(scr + t - 1) : 0;
              const int e = in ? ch_add_small(w[k], in) : 0;
              if (i == Cm) {
                top[k] += e;
              } else {
                if (e) any = 1;
                top[k] = e;
              }
            }
          }
          if (!__syncthreads_or(any)) break;
        }
      }
#pragma unroll
      for (int k = 0; k < kTasksPerThread; ++k) {
        const u32 t = tid + k * nthr;
        if (t < ntask) {
          const u32 i = t & Cm;
          std::uint8_t* g = gbase + (b0 + (t >> logC)) * gstride;
          __stcg(reinterpret_cast<uint4*>(g) + i, make_uint4(w[k].w[0], w[k].w[1], w[k].w[2], w[k].w[3]));
          if (i == Cm) __stcg(reinterpret_cast<long long*>(g + W4), (long long)top[k]);
        }
      }
      __syncthreads();  // scratch and s_rot reuse
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
