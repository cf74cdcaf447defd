// fermat_leaf.cuh -- sm_100a leaf engine for R = Z/(2^N+1), omega = 2.
//
// One persistent launch runs a whole transform.  Each CTA repeatedly takes a
// ticket (a leaf: a sub-transform of <= 2^max_ell coefficients that fits in
// shared memory), waits until the (node, phase) counter it depends on is
// complete, runs the leaf, and bumps the counter it completes.  Tickets are
// issued in a topological, L2-batched order by the planner.
//
// Element representation in shared memory ("chunked, carry-deferred"):
//   D = N/32 u32 words in C = D/CW chunks of CW words (CB = 32*CW bits), plus
//   one signed 32-bit carry per chunk that sits ON TOP of the chunk:
//       value = sum_j (chunk_j + top_j * 2^CB) * 2^(CB j)   (mod 2^N + 1),
//   the last chunk's top sitting at 2^N == -1.  A butterfly output chunk is
//   computed by one thread from chunk i of operand a and chunk i of the
//   rotated operand b with ONE add.cc chain and ONE sub.cc chain; the tops
//   just add (top0 = ta + tb + carry), so nothing ever crosses a chunk
//   boundary inside a leaf.  A rotation by a whole number of chunks moves
//   (chunk, top) pairs, negating those that wrap past 2^N; the negation costs
//   nothing because it turns the add chain into a sub chain and vice versa.
//   Tops grow by about one bit per level; they are folded into the limbs once
//   per stored slot, fused with the final rotation and the store to HBM.
//
// Global (HBM) element format between levels: N/64 u64 limbs "lo" plus a
// signed top word hi, value = lo + hi*2^N (== lo - hi).  Canonical inputs
// (top in {0,1}) are a special case; the last step canonicalises.
#pragma once
#include <cstdint>

#include "planner.hpp"

namespace cftft_b200 {
namespace fermat {

constexpr int kThreads = 512;  // default CTA size (the 2-CTA/SM variant uses 256)
constexpr u32 kMaxBatch = 256;    // ops (or slots) staged per batch
constexpr u32 kWordsPerThread = 32;  // live words per thread per batch

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
  u32 D, C;                // u32 words, chunks per element
  u32 logC;
  u32 slot_bytes;          // 4*D + 4*C (16B aligned)
  u32 scratch_off;         // byte offset of the carry scratch
  int* T;                  // carry-save tops, [buffer][view element][lane] (nullptr: not in use)
  std::uint8_t* data2;     // shadow buffer (same element stride), coset plans
  u64 tloc;                // tops entries per buffer
  const u64* locbits;      // per-slot buffer bits (DevLeaf::locoff)
  u32 nclasses;
  u32 no_deps;             // launch order already separates dependent tickets (wave engine)
  u32 half;                // bytes of one of the two ticket buffers (double buffering)
  u32 lanes, logLanes;     // lanes (chunks) per element
  u32 logS;                // tops-array lane interleave
  unsigned long long* prof;  // optional per-phase cycle totals (CFTFT_PROFILE=1)
  u32 debug_skip;            // perf experiments only (CFTFT_DEBUG_SKIP): 1 = levels, 2 = post maths
  const u32* xpre;           // wave engine: deferred pre-rotation bits of whole tickets (DevLeaf::c0 - 1)
};

// Phase timing (debug): thread 0 of each CTA accumulates clock64 deltas.
enum { PH_WAIT = 0, PH_LOAD, PH_PRE, PH_LEVELS, PH_POST, PH_STORE, PH_ISSUE, PH_CACHE, PH_N };
struct PhaseClock {
  unsigned long long acc[PH_N];
  unsigned long long t;
  bool on;
  __device__ void start(bool enable) {
    on = enable;
    for (int i = 0; i < PH_N; ++i) acc[i] = 0;
    t = clock64();
  }
  __device__ void mark(int ph) {
    if (!on) return;
    const unsigned long long n = clock64();
    acc[ph] += n - t;
    t = n;
  }
  __device__ void flush(unsigned long long* out) {
    if (!on) return;
    for (int i = 0; i < PH_N; ++i) atomicAdd(out + i, acc[i]);
  }
};

extern __shared__ __align__(16) std::uint8_t g_sm[];

template <int CW>
struct Ch {
  u32 w[CW];
};

// A slot stores its chunks PIECE-MAJOR and XOR-swizzled: 16-byte piece k of
// chunk i lives at slot + (k*C + (i ^ (k & (C-1))))*16.  Lanes of a warp
// (consecutive chunks, same k) touch distinct consecutive-ish 16-byte pieces,
// and so do lanes copying consecutive pieces of one chunk: both the compute
// accesses and the coalesced copies to/from HBM are bank-conflict free.
__device__ __forceinline__ u32 piece_off(u32 slot, u32 i, u32 k, u32 C) {
  return slot + ((k * C) + (i ^ (k & (C - 1)))) * 16;
}
template <int CW>
__device__ __forceinline__ void lds_ch(Ch<CW>& c, u32 slot, u32 i, u32 C) {
#pragma unroll
  for (int k = 0; k < CW; k += 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(g_sm + piece_off(slot, i, k / 4, C));
    c.w[k] = v.x;
    c.w[k + 1] = v.y;
    c.w[k + 2] = v.z;
    c.w[k + 3] = v.w;
  }
}
template <int CW>
__device__ __forceinline__ void sts_ch(u32 slot, u32 i, u32 C, const Ch<CW>& c) {
#pragma unroll
  for (int k = 0; k < CW; k += 4)
    *reinterpret_cast<uint4*>(g_sm + piece_off(slot, i, k / 4, C)) =
        make_uint4(c.w[k], c.w[k + 1], c.w[k + 2], c.w[k + 3]);
}

// X[m] = W[CW-1-OW+m] (m = 0..CW) of the window W = lo ++ hi.
template <int CW, int OW>
__device__ __forceinline__ void pick_window(u32 (&X)[CW + 1], const Ch<CW>& lo, const Ch<CW>& hi) {
#pragma unroll
  for (int m = 0; m <= CW; ++m) {
    const int idx = CW - 1 - OW + m;
    X[m] = idx < CW ? lo.w[idx] : hi.w[idx - CW];
  }
}
template <int CW, int OW = 0>
__device__ __forceinline__ void pick_window_rt(u32 (&X)[CW + 1], const Ch<CW>& lo, const Ch<CW>& hi, u32 ow) {
  if constexpr (OW < CW) {
    if (ow == OW)
      pick_window<CW, OW>(X, lo, hi);
    else
      pick_window_rt<CW, OW + 1>(X, lo, hi, ow);
  }
}

__device__ __forceinline__ int lds_i32(u32 off) { return *reinterpret_cast<const int*>(g_sm + off); }
__device__ __forceinline__ void sts_i32(u32 off, int v) { *reinterpret_cast<int*>(g_sm + off) = v; }

// ---- multi-word carry chains: ONE asm statement per chain (the carry flag
// is invisible to the compiler, so a chain must never be split) -----------
// (generated for CW = 4, 8, 16)
template <int CW> __device__ int ch_add(Ch<CW>& r, const Ch<CW>& a, const Ch<CW>& b);
template <int CW> __device__ int ch_sub(Ch<CW>& r, const Ch<CW>& a, const Ch<CW>& b);
template <int CW> __device__ int ch_add_small(Ch<CW>& r, int k);

// r = a + b; returns the carry out (0/1)
template <>
__device__ __forceinline__ int ch_add<4>(Ch<4>& r, const Ch<4>& a, const Ch<4>& b) {
  u32 c;
  asm("add.cc.u32 %0, %5, %9;\n\t"
      "addc.cc.u32 %1, %6, %10;\n\t"
      "addc.cc.u32 %2, %7, %11;\n\t"
      "addc.cc.u32 %3, %8, %12;\n\t"
      "addc.u32 %4, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
  return (int)c;
}

// r = a - b; returns the borrow as -1/0
template <>
__device__ __forceinline__ int ch_sub<4>(Ch<4>& r, const Ch<4>& a, const Ch<4>& b) {
  u32 c;
  asm("sub.cc.u32 %0, %5, %9;\n\t"
      "subc.cc.u32 %1, %6, %10;\n\t"
      "subc.cc.u32 %2, %7, %11;\n\t"
      "subc.cc.u32 %3, %8, %12;\n\t"
      "subc.u32 %4, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
  return (int)c;
}

// r += k (small signed, sign-extended); returns the signed carry out
template <>
__device__ __forceinline__ int ch_add_small<4>(Ch<4>& r, int k) {
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

// r = a + b; returns the carry out (0/1)
template <>
__device__ __forceinline__ int ch_add<8>(Ch<8>& r, const Ch<8>& a, const Ch<8>& b) {
  u32 c;
  asm("add.cc.u32 %0, %9, %17;\n\t"
      "addc.cc.u32 %1, %10, %18;\n\t"
      "addc.cc.u32 %2, %11, %19;\n\t"
      "addc.cc.u32 %3, %12, %20;\n\t"
      "addc.cc.u32 %4, %13, %21;\n\t"
      "addc.cc.u32 %5, %14, %22;\n\t"
      "addc.cc.u32 %6, %15, %23;\n\t"
      "addc.cc.u32 %7, %16, %24;\n\t"
      "addc.u32 %8, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(a.w[4]), "r"(a.w[5]), "r"(a.w[6]), "r"(a.w[7]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]), "r"(b.w[6]), "r"(b.w[7]));
  return (int)c;
}

// r = a - b; returns the borrow as -1/0
template <>
__device__ __forceinline__ int ch_sub<8>(Ch<8>& r, const Ch<8>& a, const Ch<8>& b) {
  u32 c;
  asm("sub.cc.u32 %0, %9, %17;\n\t"
      "subc.cc.u32 %1, %10, %18;\n\t"
      "subc.cc.u32 %2, %11, %19;\n\t"
      "subc.cc.u32 %3, %12, %20;\n\t"
      "subc.cc.u32 %4, %13, %21;\n\t"
      "subc.cc.u32 %5, %14, %22;\n\t"
      "subc.cc.u32 %6, %15, %23;\n\t"
      "subc.cc.u32 %7, %16, %24;\n\t"
      "subc.u32 %8, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(a.w[4]), "r"(a.w[5]), "r"(a.w[6]), "r"(a.w[7]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]), "r"(b.w[6]), "r"(b.w[7]));
  return (int)c;
}

// r += k (small signed, sign-extended); returns the signed carry out
template <>
__device__ __forceinline__ int ch_add_small<8>(Ch<8>& r, int k) {
  const u32 e = (u32)(k >> 31);
  u32 c;
  asm("add.cc.u32 %0, %0, %9;\n\t"
      "addc.cc.u32 %1, %1, %10;\n\t"
      "addc.cc.u32 %2, %2, %10;\n\t"
      "addc.cc.u32 %3, %3, %10;\n\t"
      "addc.cc.u32 %4, %4, %10;\n\t"
      "addc.cc.u32 %5, %5, %10;\n\t"
      "addc.cc.u32 %6, %6, %10;\n\t"
      "addc.cc.u32 %7, %7, %10;\n\t"
      "addc.u32 %8, %10, 0;"
      : "+r"(r.w[0]), "+r"(r.w[1]), "+r"(r.w[2]), "+r"(r.w[3]), "+r"(r.w[4]), "+r"(r.w[5]), "+r"(r.w[6]), "+r"(r.w[7]), "=r"(c)
      : "r"((u32)k), "r"(e));
  return (int)c;
}

// r = a + b; returns the carry out (0/1)
template <>
__device__ __forceinline__ int ch_add<16>(Ch<16>& r, const Ch<16>& a, const Ch<16>& b) {
  u32 c;
  asm("add.cc.u32 %0, %17, %33;\n\t"
      "addc.cc.u32 %1, %18, %34;\n\t"
      "addc.cc.u32 %2, %19, %35;\n\t"
      "addc.cc.u32 %3, %20, %36;\n\t"
      "addc.cc.u32 %4, %21, %37;\n\t"
      "addc.cc.u32 %5, %22, %38;\n\t"
      "addc.cc.u32 %6, %23, %39;\n\t"
      "addc.cc.u32 %7, %24, %40;\n\t"
      "addc.cc.u32 %8, %25, %41;\n\t"
      "addc.cc.u32 %9, %26, %42;\n\t"
      "addc.cc.u32 %10, %27, %43;\n\t"
      "addc.cc.u32 %11, %28, %44;\n\t"
      "addc.cc.u32 %12, %29, %45;\n\t"
      "addc.cc.u32 %13, %30, %46;\n\t"
      "addc.cc.u32 %14, %31, %47;\n\t"
      "addc.cc.u32 %15, %32, %48;\n\t"
      "addc.u32 %16, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]), "=r"(r.w[8]), "=r"(r.w[9]), "=r"(r.w[10]), "=r"(r.w[11]), "=r"(r.w[12]), "=r"(r.w[13]), "=r"(r.w[14]), "=r"(r.w[15]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(a.w[4]), "r"(a.w[5]), "r"(a.w[6]), "r"(a.w[7]), "r"(a.w[8]), "r"(a.w[9]), "r"(a.w[10]), "r"(a.w[11]), "r"(a.w[12]), "r"(a.w[13]), "r"(a.w[14]), "r"(a.w[15]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]), "r"(b.w[6]), "r"(b.w[7]), "r"(b.w[8]), "r"(b.w[9]), "r"(b.w[10]), "r"(b.w[11]), "r"(b.w[12]), "r"(b.w[13]), "r"(b.w[14]), "r"(b.w[15]));
  return (int)c;
}

// r = a - b; returns the borrow as -1/0
template <>
__device__ __forceinline__ int ch_sub<16>(Ch<16>& r, const Ch<16>& a, const Ch<16>& b) {
  u32 c;
  asm("sub.cc.u32 %0, %17, %33;\n\t"
      "subc.cc.u32 %1, %18, %34;\n\t"
      "subc.cc.u32 %2, %19, %35;\n\t"
      "subc.cc.u32 %3, %20, %36;\n\t"
      "subc.cc.u32 %4, %21, %37;\n\t"
      "subc.cc.u32 %5, %22, %38;\n\t"
      "subc.cc.u32 %6, %23, %39;\n\t"
      "subc.cc.u32 %7, %24, %40;\n\t"
      "subc.cc.u32 %8, %25, %41;\n\t"
      "subc.cc.u32 %9, %26, %42;\n\t"
      "subc.cc.u32 %10, %27, %43;\n\t"
      "subc.cc.u32 %11, %28, %44;\n\t"
      "subc.cc.u32 %12, %29, %45;\n\t"
      "subc.cc.u32 %13, %30, %46;\n\t"
      "subc.cc.u32 %14, %31, %47;\n\t"
      "subc.cc.u32 %15, %32, %48;\n\t"
      "subc.u32 %16, 0, 0;"
      : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]), "=r"(r.w[7]), "=r"(r.w[8]), "=r"(r.w[9]), "=r"(r.w[10]), "=r"(r.w[11]), "=r"(r.w[12]), "=r"(r.w[13]), "=r"(r.w[14]), "=r"(r.w[15]), "=r"(c)
      : "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(a.w[4]), "r"(a.w[5]), "r"(a.w[6]), "r"(a.w[7]), "r"(a.w[8]), "r"(a.w[9]), "r"(a.w[10]), "r"(a.w[11]), "r"(a.w[12]), "r"(a.w[13]), "r"(a.w[14]), "r"(a.w[15]), "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]), "r"(b.w[6]), "r"(b.w[7]), "r"(b.w[8]), "r"(b.w[9]), "r"(b.w[10]), "r"(b.w[11]), "r"(b.w[12]), "r"(b.w[13]), "r"(b.w[14]), "r"(b.w[15]));
  return (int)c;
}

// r += k (small signed, sign-extended); returns the signed carry out
template <>
__device__ __forceinline__ int ch_add_small<16>(Ch<16>& r, int k) {
  const u32 e = (u32)(k >> 31);
  u32 c;
  asm("add.cc.u32 %0, %0, %17;\n\t"
      "addc.cc.u32 %1, %1, %18;\n\t"
      "addc.cc.u32 %2, %2, %18;\n\t"
      "addc.cc.u32 %3, %3, %18;\n\t"
      "addc.cc.u32 %4, %4, %18;\n\t"
      "addc.cc.u32 %5, %5, %18;\n\t"
      "addc.cc.u32 %6, %6, %18;\n\t"
      "addc.cc.u32 %7, %7, %18;\n\t"
      "addc.cc.u32 %8, %8, %18;\n\t"
      "addc.cc.u32 %9, %9, %18;\n\t"
      "addc.cc.u32 %10, %10, %18;\n\t"
      "addc.cc.u32 %11, %11, %18;\n\t"
      "addc.cc.u32 %12, %12, %18;\n\t"
      "addc.cc.u32 %13, %13, %18;\n\t"
      "addc.cc.u32 %14, %14, %18;\n\t"
      "addc.cc.u32 %15, %15, %18;\n\t"
      "addc.u32 %16, %18, 0;"
      : "+r"(r.w[0]), "+r"(r.w[1]), "+r"(r.w[2]), "+r"(r.w[3]), "+r"(r.w[4]), "+r"(r.w[5]), "+r"(r.w[6]), "+r"(r.w[7]), "+r"(r.w[8]), "+r"(r.w[9]), "+r"(r.w[10]), "+r"(r.w[11]), "+r"(r.w[12]), "+r"(r.w[13]), "+r"(r.w[14]), "+r"(r.w[15]), "=r"(c)
      : "r"((u32)k), "r"(e));
  return (int)c;
}

// Rotation r (0 <= r < 2N) for windowed reads of omega^r * x.
struct Rot {
  u32 q, o;   // t = r mod N = CB q + o
  u32 sneg;   // 1 when r >= N (2^N == -1)
};
template <int CW>
__device__ __forceinline__ Rot make_rot(u64 r, u64 N) {
  constexpr u32 CB = 32 * CW;
  Rot R;
  R.sneg = (r >= N) ? 1u : 0u;
  const u64 t = R.sneg ? r - N : r;
  R.q = (u32)(t / CB);
  R.o = (u32)(t % CB);
  return R;
}

// p * 2^o (o < CB) as a (CW+1)-word signed value: words P and top ptop.
template <int CW>
__device__ __forceinline__ int small_shifted(Ch<CW>& P, int p, u32 o) {
  const u32 ow = o >> 5, ob = o & 31;
  const long long pw = (long long)p * (1ll << ob);
  const u32 ext = (u32)(p >> 31);
#pragma unroll
  for (int k = 0; k < CW; ++k)
    P.w[k] = ((u32)k < ow) ? 0u : ((u32)k == ow ? (u32)pw : ((u32)k == ow + 1 ? (u32)(pw >> 32) : ext));
  return (ow == CW - 1) ? (int)(pw >> 32) : (int)ext;
}

// Unaligned part of rot_chunk (the rotation is not a whole number of
// chunks): kept out of line so the hot aligned paths keep their registers.
// word g of the output takes source bits [32g - t, 32g + 32 - t) (mod N);
// words below t wrap past 2^N (negative).
template <int CW>
__device__ __noinline__ bool rot_chunk_unaligned(Ch<CW>& B, int& tb, u32 xw, u32 xt, Rot R, u32 Cm, u32 i) {
  const u32 C = Cm + 1;
  const u32 j = (i - R.q) & Cm;
  const u32 jm = (j - 1) & Cm;
  const u32 ow = R.o >> 5, sh = R.o & 31;
  Ch<CW> lo, hi;
  lds_ch(lo, xw, jm, C);
  lds_ch(hi, xw, j, C);
  u32 Wd[CW + 1];
  pick_window_rt<CW>(Wd, lo, hi, ow);
  Ch<CW> P;
  const int ptop = small_shifted(P, lds_i32(xt + 4 * jm), R.o);  // jm's top lands at offset o
  if (i != R.q) {
#pragma unroll
    for (int k = 0; k < CW; ++k) B.w[k] = __funnelshift_l(Wd[k], Wd[k + 1], sh);
    tb = ch_add(B, B, P) + ptop;
    return ((i < R.q) ? 1u : 0u) != R.sneg;
  }
  // the chunk holding bit t: words above t come from chunk 0 (positive),
  // words below from the top of chunk C-1 and its top carry (wrapped: negative)
  Ch<CW> up, dn;
#pragma unroll
  for (int k = 0; k < CW; ++k) {
    const u32 v = __funnelshift_l(Wd[k], Wd[k + 1], sh);
    const u32 mhi = ((u32)k > ow) ? 0xFFFFFFFFu : ((u32)k == ow ? (0xFFFFFFFFu << sh) : 0u);
    up.w[k] = v & mhi;
    dn.w[k] = v & ~mhi;
  }
  const int c1 = ch_sub(B, up, dn);
  const int c2 = ch_sub(B, B, P);
  tb = c1 + c2 - ptop;
  return R.sneg != 0;
}

// Chunk i of omega^r * x as (B, tb, neg): value = (-1)^neg (B + tb 2^CB).
// xw: smem offset of x's chunks, xt: of its tops.
template <int CW>
__device__ __forceinline__ bool rot_chunk(Ch<CW>& B, int& tb, u32 xw, u32 xt, const Rot& R, u32 Cm,
                                          u32 i) {
  if (R.o == 0) {  // whole chunks: (chunk, top) pairs move together
    const u32 j = (i - R.q) & Cm;
    lds_ch(B, xw, j, Cm + 1);
    tb = lds_i32(xt + 4 * j);
    return ((i < R.q) ? 1u : 0u) != R.sneg;
  }
  return rot_chunk_unaligned<CW>(B, tb, xw, xt, R, Cm, i);
}

// Exact form of (-1)^neg (B + tb 2^CB): chunk W and top.
template <int CW>
__device__ __forceinline__ int exact_from(Ch<CW>& W, int tb, bool neg) {
  if (!neg) return tb;
  // -(B + tb 2^CB) = (~B + 1) - (tb + 1) 2^CB
#pragma unroll
  for (int k = 0; k < CW; ++k) W.w[k] = ~W.w[k];
  return ch_add_small(W, 1) - tb - 1;
}

// Per-op parameters staged in shared memory.
struct OpT {
  u32 aw, bw;  // smem offsets of slot a / slot b (tops at +W4)
  u32 q, o;
  u32 sneg, type;
};

__device__ __forceinline__ void cp_async16(u32 saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async4(u32 saddr, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(u32 saddr, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ u32 ld_acquire(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Leaf-program cache: the micro-ops / rotations of the current leaf class
// live in shared memory, so consecutive leaves of one class (the common case)
// never touch the class tables in global memory again.
constexpr u32 kCacheOps = 256;
constexpr u32 kCacheLev = 64;
constexpr u32 kCacheRot = 512;  // pre + post rotations

// Chunk-i piece offsets (within a slot) for the thread's fixed chunk.
template <int CW>
struct Offs {
  u32 o[CW / 4];
  __device__ __forceinline__ void init(u32 i, u32 C) {
#pragma unroll
    for (int k = 0; k < CW / 4; ++k) o[k] = piece_off(0, i, k, C);
  }
};
template <int CW>
__device__ __forceinline__ void lds_at(Ch<CW>& c, u32 slot, const Offs<CW>& f) {
#pragma unroll
  for (int k = 0; k < CW; k += 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(g_sm + slot + f.o[k / 4]);
    c.w[k] = v.x;
    c.w[k + 1] = v.y;
    c.w[k + 2] = v.z;
    c.w[k + 3] = v.w;
  }
}
template <int CW>
__device__ __forceinline__ void sts_at(u32 slot, const Offs<CW>& f, const Ch<CW>& c) {
#pragma unroll
  for (int k = 0; k < CW; k += 4)
    *reinterpret_cast<uint4*>(g_sm + slot + f.o[k / 4]) = make_uint4(c.w[k], c.w[k + 1], c.w[k + 2], c.w[k + 3]);
}

// Per-leaf geometry (from the leaf's class and ticket).
struct Geo {
  u32 C, Cm, logC;  // chunks per slot
  u32 SB, W4, HO;   // slot bytes, offsets of the tops and of the element top word
  u32 coset;        // coset leaf
  u32 m, logm, step, c0;
};
__device__ __forceinline__ Geo geo_of(const DevClass& cl, const DevLeaf& lf, u32 CW) {
  Geo g;
  g.C = cl.cs;
  g.Cm = cl.cs - 1;
  g.logC = __ffs(cl.cs) - 1;
  g.SB = cl.slot_bytes;
  g.W4 = cl.cs * CW * 4;
  g.HO = g.W4 + ((4 * cl.cs + 7) & ~7u);
  g.coset = cl.kind;
  g.m = cl.m;
  g.logm = __ffs(cl.m) - 1;
  g.step = cl.step;
  g.c0 = lf.c0;
  return g;
}
// element lane of slot chunk j
__device__ __forceinline__ u32 lane_of(const Geo& g, u32 j) {
  return g.coset ? g.c0 + (j & (g.m - 1)) + g.step * (j >> g.logm) : j;
}
// tops-array index of lane p (lanes interleaved by S = 2^logS, so that the
// lanes of one coset are contiguous)
__device__ __forceinline__ u32 tops_ix(const Args& A, u32 p) {
  return ((p & ((1u << A.logS) - 1)) << (A.logLanes - A.logS)) | (p >> A.logS);
}

// Pre / post rotation (omega exponent) of slot k of a leaf.
__device__ __forceinline__ u64 pre_exp(const Args& A, const DevClass& cl, const DevLeaf& lf, const SymExp& P, u32 k) {
  return (P.a * lf.s + P.b + (k < cl.spec_n ? lf.tpre : 0)) & (A.M - 1);
}
__device__ __forceinline__ u64 post_exp(const Args& A, const DevClass& cl, const DevLeaf& lf, const SymExp& P,
                                        u32 k) {
  const bool tp = cl.inverse ? (k == cl.fslot) : true;
  return (P.a * lf.s + P.b + (tp ? lf.tpost : 0)) & (A.M - 1);
}

// Rotation of a micro-op: bits for whole leaves; for coset leaves the lane
// rotation r/lane (a multiple of the step) moves chunk j to j + m r/(lane step)
// in the slot's negacyclic ring of C chunks.
template <int CW>
__device__ __forceinline__ Rot op_rot(const Args& A, const Geo& g, u64 r) {
  if (!g.coset) return make_rot<CW>(r, A.N);
  constexpr u32 CB = 32 * CW;
  const u32 qv = (u32)((r / CB) / g.step) * g.m;
  Rot R;
  R.sneg = qv >= g.C ? 1u : 0u;
  R.q = qv - (R.sneg ? g.C : 0u);
  R.o = 0;
  return R;
}

// Moves whole elements between HBM and shared memory (piece-major swizzled
// slots), 16 bytes per thread per step, coalesced on the HBM side.  Element
// x of the range lives at g0 + x*gstride and in slot (s0 + x), x < nslots.
// The per-thread piece positions are fixed, so the loop body is a couple of
// adds (no division, no 64-bit multiply).
constexpr u32 kMaskWords = 16;  // per-slot buffer bits of up to 1024 slots
__device__ __forceinline__ u32 in_buf(const u64* m, u32 k) { return (u32)(m[2 * (k >> 6)] >> (k & 63)) & 1u; }
__device__ __forceinline__ u32 out_buf(const u64* m, u32 k) { return (u32)(m[2 * (k >> 6) + 1] >> (k & 63)) & 1u; }
__device__ __forceinline__ std::uint8_t* elem_ptr(const Args& A, u32 buf, u64 e) {
  return (buf ? A.data2 : A.data) + e * A.elem_bytes;
}
__device__ __forceinline__ int* tops_row(const Args& A, u32 buf, u64 e) {
  return A.T + (buf ? A.tloc : 0) + e * A.lanes;
}

template <int CW, bool kLoad, int NT>
__device__ __forceinline__ void copy_slots(const Args& A, const Geo& G, const DevLeaf& lf, const u64* locm, u32 k0,
                                           u32 k1, u32 smem_base, u32 boff, u32 tid) {
  constexpr u32 lpc = CW == 16 ? 2 : (CW == 8 ? 1 : 0);  // log2 pieces per chunk
  const u32 C = G.C, SB = G.SB;
  const u32 lq = G.logC + lpc, q16 = 1u << lq;  // pieces per slot
  auto slot_ptr = [&](u32 x) {
    const u32 b = kLoad ? in_buf(locm, x) : out_buf(locm, x);
    return elem_ptr(A, b, lf.base + (u64)x * lf.stride);
  };
  if (q16 >= (u32)NT) {
    // each thread copies pieces tid, tid+NT, ... of every slot
    for (u32 pp = tid; pp < q16; pp += NT) {
      const u32 so0 = piece_off(0, pp >> lpc, pp & ((1u << lpc) - 1), C);
      u32 so = boff + k0 * SB + so0;
      for (u32 x = k0; x < k1; ++x, so += SB) {
        std::uint8_t* g = slot_ptr(x) + 16u * pp;
        if (kLoad)
          cp_async16(smem_base + so, g);
        else
          __stcg(reinterpret_cast<uint4*>(g), *reinterpret_cast<const uint4*>(g_sm + so));
      }
    }
  } else {
    // NT/q16 slots side by side; each thread keeps one piece position
    const u32 pp = tid & (q16 - 1), x0 = tid >> lq, step = (u32)NT >> lq;
    const u32 so0 = piece_off(0, pp >> lpc, pp & ((1u << lpc) - 1), C);
    u32 so = boff + (k0 + x0) * SB + so0;
    for (u32 x = k0 + x0; x < k1; x += step, so += step * SB) {
      std::uint8_t* g = slot_ptr(x) + 16u * pp;
      if (kLoad)
        cp_async16(smem_base + so, g);
      else
        __stcg(reinterpret_cast<uint4*>(g), *reinterpret_cast<const uint4*>(g_sm + so));
    }
  }
}

// Slot layout (both leaf kinds): C chunks (piece-major, swizzled), then one
// int32 top per chunk at W4, then the element's 64-bit top word at W4 + 4C.
constexpr u32 kMaxSlots = 64;
constexpr u32 kClassTab = 48;

// Issues the loads of a ticket into the slot buffer at `boff`, all as
// cp.async in one commit group: the data chunks (coset tickets gather their
// lanes through the slot's lane pre-rotation), the 4-byte word of the tops
// array that holds each chunk's carry-save top (when in use), and each
// slot's element top word.  fixup() turns these into int32 tops once landed.
// Stages a ticket's per-slot buffer bits, (coset) lane pre-rotations and
// input element pointers in shared memory; ends with a barrier.
template <int CW, int NT>
__device__ __forceinline__ void stage_load(const Args& A, const DevLeaf& lf, const DevClass& cl, u32 tid, u32* rho,
                                           u64* locm, std::uint8_t** sp) {
  const Geo G = geo_of(cl, lf, CW);
  const u32 nl = cl.nload;
  constexpr u32 CB = 32 * CW;
  const u32 span = max(cl.nload, cl.nstore), nw = (span + 63) >> 6;
  for (u32 x = tid; x < 2 * kMaskWords; x += NT)
    locm[x] = (lf.locoff != kNoDep && x < 2 * nw) ? A.locbits[lf.locoff + x] : 0ull;
  if (G.coset) {
    for (u32 k = tid; k < nl; k += NT) {
      const SymExp P = A.rots[cl.pre_begin + k];
      rho[k] = (u32)(pre_exp(A, cl, lf, P, k) / CB);
      const u32 b = (lf.locoff != kNoDep) ? (u32)(A.locbits[lf.locoff + 2 * (k >> 6)] >> (k & 63)) & 1u : 0u;
      sp[k] = elem_ptr(A, b, lf.base + (u64)k * lf.stride);
    }
  }
  __syncthreads();
}

// Issues the cp.async loads of slots [k0, k1) of a staged ticket into the
// slot buffer at `boff`: the data chunks (coset tickets gather their lanes
// through the slot's lane pre-rotation), the tops-array word of each chunk
// (when in use), each slot's element top word.  fixup() finishes them.
template <int CW, int NT>
__device__ __forceinline__ void issue_slots(const Args& A, const DevLeaf& lf, const DevClass& cl, u32 smem_base,
                                            u32 boff, u32 tid, const u32* rho, const u64* locm,
                                            std::uint8_t* const* sp, u32 k0, u32 k1) {
  const Geo G = geo_of(cl, lf, CW);
  k1 = min(k1, cl.nload);
  if (k0 >= k1) return;
  constexpr u32 CB = 32 * CW;
  constexpr u32 lpc = CW == 16 ? 2 : (CW == 8 ? 1 : 0);
  const u32 CL = A.lanes;
  const u32 sb = smem_base + boff;
  if (G.coset) {
    // thread -> fixed piece position (chunk j, piece q); slots strided
    const u32 lq = G.logC + lpc, P = 1u << lq;
    const u32 kstep = NT > P ? NT / P : 1u;
    for (u32 pp = tid & (P - 1); pp < ((A.debug_skip & 16) ? 0u : P); pp += NT) {
      const u32 j = pp >> lpc, q = pp & ((1u << lpc) - 1);
      const u32 lj = lane_of(G, j) + 2 * CL;
      const u32 so0 = piece_off(0, j, q, G.C);
      for (u32 k = k0 + (NT > P ? tid / P : 0u); k < k1; k += kstep) {
        const u32 ln = (lj - rho[k]) & (CL - 1);
        cp_async16(sb + k * G.SB + so0, sp[k] + (u64)ln * (CB / 8) + 16u * q);
      }
    }
    if (A.T && !(A.debug_skip & 8)) {
      const u32 Pc = G.C;
      const u32 kstep = NT > Pc ? NT / Pc : 1u;
      for (u32 j = tid & (Pc - 1); j < Pc; j += NT) {
        const u32 lj = lane_of(G, j) + 2 * CL;
        for (u32 k = k0 + (NT > Pc ? tid / Pc : 0u); k < k1; k += kstep) {
          const u32 ln = (lj - rho[k]) & (CL - 1);
          const u32 b = in_buf(locm, k);
          const int* tr = A.T + (b ? A.tloc : 0) + (lf.base + (u64)k * lf.stride) * CL;
          cp_async4(sb + k * G.SB + G.W4 + 4 * j, tr + tops_ix(A, ln));
        }
      }
    }
    for (u32 k = k0 + tid; k < k1; k += NT) cp_async8(sb + k * G.SB + G.HO, sp[k] + 4ull * A.D);
  } else {
    copy_slots<CW, true, NT>(A, G, lf, locm, k0, k1, smem_base, boff, tid);
    if (A.T) {
      const u32 tt = (k1 - k0) << G.logC;
      for (u32 idx = tid; idx < tt; idx += NT) {
        const u32 k = k0 + (idx >> G.logC), j = idx & G.Cm;
        const int* tr = tops_row(A, in_buf(locm, k), lf.base + (u64)k * lf.stride);
        cp_async4(sb + k * G.SB + G.W4 + 4 * j, tr + tops_ix(A, j));
      }
    }
    for (u32 k = k0 + tid; k < k1; k += NT)
      cp_async8(sb + k * G.SB + G.HO, elem_ptr(A, in_buf(locm, k), lf.base + (u64)k * lf.stride) + 4ull * A.D);
  }
}

template <int CW, int NT>
__device__ __forceinline__ void issue_load(const Args& A, const DevLeaf& lf, const DevClass& cl, u32 smem_base,
                                           u32 boff, u32 tid, u32* rho, u64* locm, std::uint8_t** sp) {
  stage_load<CW, NT>(A, lf, cl, tid, rho, locm, sp);
  issue_slots<CW, NT>(A, lf, cl, smem_base, boff, tid, rho, locm, sp, 0, cl.nload);
  cp_async_commit();
}

// Once a ticket's loads have landed: int32 tops from the tops-array words and
// the element top word (on lane C-1), and coset lanes that wrapped past 2^N
// negated in place.
template <int CW, int NT>
__device__ __forceinline__ void fixup(const Args& A, const DevLeaf& lf, const DevClass& cl, u32 boff, u32 tid,
                                      const u32* rho) {
  const Geo G = geo_of(cl, lf, CW);
  const u32 CL = A.lanes;
  const u32 Pc = G.C, nl = cl.nload;
  const u32 kstep = NT > Pc ? NT / Pc : 1u;
  for (u32 j = tid & (Pc - 1); j < Pc; j += NT) {
    const u32 lj = G.coset ? lane_of(G, j) + 2 * CL : j;
    for (u32 k = NT > Pc ? tid / Pc : 0u; k < nl; k += kstep) {
      const u32 src = G.coset ? ((lj - rho[k]) & (2 * CL - 1)) : j;
      const u32 ln = src & (CL - 1);
      const u32 so = boff + k * G.SB;
      int top = 0;
      if (A.T) top = *reinterpret_cast<const int*>(g_sm + so + G.W4 + 4 * j);
      // the element's top word hi sits at 2^N == -1: fold -hi into lane 0
      // right here, so no lane top ever accumulates it
      const int hi = ln == 0 ? (int)*reinterpret_cast<const long long*>(g_sm + so + G.HO) : 0;
      if (hi != 0 || src >= CL) {
        Ch<CW> w;
        lds_ch(w, so, j, G.C);
        if (hi) top += ch_add_small<CW>(w, -hi);
        if (src >= CL) top = exact_from<CW>(w, top, true);
        sts_ch(so, j, G.C, w);
      }
      sts_i32(so + G.W4 + 4 * j, top);
    }
  }
}

__device__ __forceinline__ bool small_ticket(const Args& A, const DevClass& cl) {
  return cl.L * cl.slot_bytes <= A.half;
}

template <int CW, int NT>
__global__ void __launch_bounds__(NT, NT >= 512 ? 1 : 512 / NT) leaf_kernel(Args A) {
  constexpr int TPT = 2;  // ops per thread per round (each a CW-word chunk)
  constexpr u32 CB = 32 * CW;
  // ticket descriptors, a ring of three: the current ticket, the next one
  // (prefetched into the other buffer when its inputs are ready), and the one
  // after it, whose descriptor tid 0 fetches while the current one computes
  __shared__ u32 s_tk[3];
  __shared__ DevLeaf s_lf[3];
  __shared__ DevClass s_cl[3];
  __shared__ u32 s_boff[3];
  __shared__ int s_ready[3];  // dependency already satisfied (as last checked)
  __shared__ u32 s_cached;
  __shared__ OpT s_ops[kCacheOps];
  __shared__ u32 s_lev[kCacheLev + 1];
  __shared__ SymExp s_crot[kCacheRot];
  __shared__ u32 s_rho[3][kMaxSlots];  // coset: lane pre-rotation per loaded slot
  __shared__ u64 s_loc[3][2 * kMaskWords];  // per-slot buffer bits
  __shared__ std::uint8_t* s_sp[3][kMaxSlots];  // coset: input element pointer per slot
  __shared__ std::uint8_t* s_op[kMaxSlots];     // coset: output element pointer per slot
  __shared__ u32 s_rhp[kMaxSlots];     // coset: lane post-rotation per stored slot
  __shared__ DevClass s_ctab[kClassTab];  // the plan's first kClassTab classes
  const u32 tid = threadIdx.x;
  constexpr u32 nthr = NT;
  const u32 CL = A.lanes, CLm = CL - 1;
  const u32 W4e = 4 * A.D;
  const u32 scr = A.scratch_off;
  const u32 smem_base = (u32)__cvta_generic_to_shared(g_sm);
  PhaseClock pc;
  pc.start(tid == 0 && A.prof != nullptr);

  auto dep_met = [&](const DevLeaf& l) {
    return A.no_deps || (l.dep == kNoDep) || (ld_acquire(&A.counters[1 + l.dep]) >= l.dep_target);
  };
  auto fetch = [&](u32 r) {  // tid 0 only
    const u32 t = atomicAdd(&A.counters[0], 1u);
    s_tk[r] = t;
    s_ready[r] = 0;
    if (t < A.nleaves) {
      s_lf[r] = A.leaves[t];
      s_cl[r] = A.classes[s_lf[r].cls];
      s_ready[r] = dep_met(s_lf[r]);
    }
  };

  for (u32 x = tid; x < min(A.nclasses, kClassTab); x += NT) s_ctab[x] = A.classes[x];
  // ---- prologue: first two tickets, the first one's loads -------------------
  if (tid == 0) {
    fetch(0);
    s_boff[0] = 0;
    if (s_tk[0] < A.nleaves)
      while (!dep_met(s_lf[0])) __nanosleep(64);
    fetch(1);
    s_cached = 0xFFFFFFFFu;
  }
  __syncthreads();
  if (s_tk[0] < A.nleaves) issue_load<CW, NT>(A, s_lf[0], s_cl[0], smem_base, 0, tid, s_rho[0], s_loc[0], s_sp[0]);
  u32 cur = 0;

  for (;;) {
    const u32 ticket = s_tk[cur];
    if (ticket >= A.nleaves) break;
    const DevLeaf lf = s_lf[cur];
    const DevClass cl = s_cl[cur];
    const u32 boff = s_boff[cur];
    const Geo G = geo_of(cl, lf, CW);
    const u32 C = G.C, Cm = G.Cm, logC = G.logC, SB = G.SB, W4 = G.W4;
    // fixed thread geometry for this leaf: chunk i of group g; NG groups side by side
    const u32 i = tid & Cm, g = tid >> logC, NG = nthr >> logC;
    Offs<CW> fi;
    fi.init(i, C);
    const u32 ti = W4 + 4 * i;  // offset of chunk i's top within a slot
    const u32 nxt = cur == 2 ? 0 : cur + 1, nn = nxt == 2 ? 0 : nxt + 1;
    const bool have_next = s_tk[nxt] < A.nleaves;
    // the descriptor after next: its ticket number is claimed now, its leaf is
    // read once the prefetch is issued; everyone reads it next iteration
    u32 tnn = 0xFFFFFFFFu;
    if (tid == 0 && have_next) tnn = atomicAdd(&A.counters[0], 1u);
    // the next ticket streams into the other buffer while this one computes
    bool prefetched = false, rolled = false;
    if (have_next && s_ready[nxt] && small_ticket(A, cl) && small_ticket(A, s_cl[nxt])) {
      if (tid == 0) s_boff[nxt] = boff ^ A.half;
      issue_load<CW, NT>(A, s_lf[nxt], s_cl[nxt], smem_base, boff ^ A.half, tid, s_rho[nxt], s_loc[nxt], s_sp[nxt]);
      prefetched = true;
    }
    pc.mark(PH_ISSUE);
    if (tid == 0 && have_next) {
      s_tk[nn] = tnn;
      s_ready[nn] = 0;  // checked at the end of this iteration
      if (tnn < A.nleaves) {
        s_lf[nn] = A.leaves[tnn];
        const u32 c = s_lf[nn].cls;
        s_cl[nn] = c < kClassTab ? s_ctab[c] : A.classes[c];
      }
    }
    // leaf-program cache
    const bool cached = cl.nops <= kCacheOps && cl.nlevels <= kCacheLev && cl.nload + cl.nstore <= kCacheRot;
    if (cached && s_cached != lf.cls) {
      const u32 op0 = cl.op_begin;
      for (u32 x = tid; x < cl.nops; x += nthr) {
        const DevOp op = A.ops[op0 + x];
        const Rot R = op_rot<CW>(A, G, op.r);
        s_ops[x] = OpT{op.a * SB, op.b * SB, R.q, R.o, R.sneg, op.type};
      }
      for (u32 x = tid; x <= cl.nlevels; x += nthr) s_lev[x] = A.levels[cl.level_begin + x] - op0;
      for (u32 x = tid; x < cl.nload; x += nthr) s_crot[x] = A.rots[cl.pre_begin + x];
      for (u32 x = tid; x < cl.nstore; x += nthr) s_crot[cl.nload + x] = A.rots[cl.post_begin + x];
    }
    if (G.coset) {
      for (u32 k = tid; k < cl.nstore; k += nthr) {
        const SymExp P = A.rots[cl.post_begin + k];
        s_rhp[k] = (u32)(post_exp(A, cl, lf, P, k) / CB);
        const u32 b = (lf.locoff != kNoDep) ? (u32)(A.locbits[lf.locoff + 2 * (k >> 6) + 1] >> (k & 63)) & 1u : 0u;
        s_op[k] = elem_ptr(A, b, lf.base + (u64)k * lf.stride);
      }
    }
    pc.mark(PH_CACHE);
    if (prefetched)
      cp_async_wait<1>();
    else
      cp_async_wait<0>();
    __syncthreads();
    if (tid == 0 && cached) s_cached = lf.cls;
    pc.mark(PH_LOAD);
    fixup<CW, NT>(A, lf, cl, boff, tid, s_rho[cur]);
    __syncthreads();
    const u64* const locm = s_loc[cur];

    const u32* const xp = (!G.coset && A.xpre && lf.c0) ? A.xpre + (lf.c0 - 1) : nullptr;
    if (!G.coset && (cl.has_pre || lf.tpre || xp)) {
      // ---- pre-rotations (whole tickets), in place: NG slots per round --------------
      for (u32 b0 = 0; b0 < cl.nload; b0 += NG) {
        const u32 sl = b0 + g;
        const bool act = sl < cl.nload;
        Ch<CW> w;
        int tp = 0;
        if (act) {
          const SymExp P = cached ? s_crot[sl] : A.rots[cl.pre_begin + sl];
          const u64 r = pre_exp(A, cl, lf, P, sl) + (xp ? xp[sl] : 0u);
          const Rot R = make_rot<CW>(r & (A.M - 1), A.N);
          const u32 so = boff + sl * SB;
          const bool neg = rot_chunk<CW>(w, tp, so, so + W4, R, Cm, i);
          tp = exact_from<CW>(w, tp, neg);
        }
        __syncthreads();
        if (act) {
          sts_at<CW>(boff + sl * SB, fi, w);
          sts_i32(boff + sl * SB + ti, tp);
        }
        __syncthreads();
      }
    }
    pc.mark(PH_PRE);

    // ---- micro-op levels: each thread runs chunk i of up to TPT ops per round ----
    for (u32 l = 0; l < ((A.debug_skip & 1) ? 0u : cl.nlevels); ++l) {
      u32 o0, o1;
      if (cached) {
        o0 = s_lev[l];
        o1 = s_lev[l + 1];
      } else {
        o0 = A.levels[cl.level_begin + l] - cl.op_begin;
        o1 = A.levels[cl.level_begin + l + 1] - cl.op_begin;
      }
      for (u32 ob = o0; ob < o1; ob += NG * TPT) {
        const u32 nb = min(o1 - ob, NG * TPT);
        u32 sbase = ob;
        if (!cached) {  // stage this round's ops
          for (u32 x = tid; x < nb; x += nthr) {
            const DevOp op = A.ops[cl.op_begin + ob + x];
            const Rot R = op_rot<CW>(A, G, op.r);
            s_ops[x] = OpT{op.a * SB, op.b * SB, R.q, R.o, R.sneg, op.type};
          }
          __syncthreads();
          sbase = 0;
        }
        // out0 goes to slot a in place right away (only this thread reads a's
        // chunk i); out1 goes to slot b after the barrier (b is read rotated)
        Ch<CW> hold[TPT];
        int htop[TPT];
        u32 hdst[TPT];
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          hdst[k] = 0xFFFFFFFFu;
          const u32 x = g + NG * k;
          if (x >= nb) continue;
          OpT op = s_ops[sbase + x];
          op.aw += boff;
          op.bw += boff;
          Ch<CW> a;
          lds_at(a, op.aw, fi);
          const int pa = lds_i32(op.aw + ti);
          if (op.type == OP_COPY) {
            hold[k] = a;
            htop[k] = pa;
            hdst[k] = op.bw;
            continue;
          }
          Ch<CW> b;
          int pb;
          bool neg;
          if (op.o == 0) {  // whole-chunk rotation: the common case inside a leaf
            const u32 j = (i - op.q) & Cm;
            lds_ch(b, op.bw, j, C);
            pb = lds_i32(op.bw + W4 + 4 * j);
            neg = ((i < op.q) ? 1u : 0u) != op.sneg;
          } else {
            neg = rot_chunk<CW>(b, pb, op.bw, op.bw + W4, Rot{op.q, op.o, op.sneg}, Cm, i);
          }
          Ch<CW> y0;
          int t0, t1;
          // y0 = a + s b, y1 = a - s b with s = (-1)^neg
          if (!neg) {
            t0 = ch_add(y0, a, b) + pa + pb;
            t1 = ch_sub(hold[k], a, b) + pa - pb;
          } else {
            t0 = ch_sub(y0, a, b) + pa - pb;
            t1 = ch_add(hold[k], a, b) + pa + pb;
          }
          if (op.type == OP_SUB2 || op.type == OP_SUB2DIFF) {  // y0 = a + y1 = 2a - s b
            t0 = ch_add(y0, a, hold[k]) + pa + t1;
          }
          sts_at<CW>(op.aw, fi, y0);
          sts_i32(op.aw + ti, t0);
          if (op.type == OP_ADDSUB || op.type == OP_SUB2DIFF) {
            htop[k] = t1;
            hdst[k] = op.bw;
          }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < TPT; ++k) {
          if (hdst[k] != 0xFFFFFFFFu) {
            sts_at<CW>(hdst[k], fi, hold[k]);
            sts_i32(hdst[k] + ti, htop[k]);
          }
        }
        __syncthreads();
      }
    }
    pc.mark(PH_LEVELS);

    if (G.coset) {
      // ---- coset ticket: lanes out through the post-rotation, carry-save -----------
      // (1) per chunk: negate wrapped lanes in place, write the tops array, and
      //     clear the element top word where this ticket owns lane C-1
      for (u32 idx = tid; idx < (cl.nstore << logC); idx += nthr) {
        const u32 k = idx >> logC, j = idx & Cm;
        const u32 rho = s_rhp[k];
        const u32 dst = (lane_of(G, j) + rho) & (2 * CL - 1);
        const u32 d = dst & CLm;
        const u32 so = boff + k * SB;
        int tp = lds_i32(so + W4 + 4 * j);
        if (dst >= CL) {
          Ch<CW> w;
          lds_ch(w, so, j, C);
          tp = exact_from<CW>(w, tp, true);
          sts_ch(so, j, C, w);
        }
        const u64 e = lf.base + (u64)k * lf.stride;
        const u32 ob = out_buf(locm, k);
        __stcg(tops_row(A, ob, e) + tops_ix(A, d), tp);
        if (j == 0) {
          // one ticket per slot (the one that read lane 0, which took the
          // element top word, or for an output-only slot writes lane 0) sets
          // the output's element top word to zero: the value now lives in the
          // lanes and their tops
          const u32 pstar = k < cl.nload ? (s_rho[cur][k] & CLm) : ((2 * CL - rho) & CLm);
          if (((pstar & (G.step - 1)) - G.c0) < G.m)
            __stcg(reinterpret_cast<long long*>(elem_ptr(A, ob, e) + W4e), 0ll);
        }
      }
      __syncthreads();
      // (2) coalesced copy of the lanes to their rotated positions.  When the
      //     next ticket is ready and lands in this buffer, the copy runs in two
      //     halves: the next ticket's loads stream into the freed first half
      //     while the second half is stored.
      auto store_range = [&](u32 k0, u32 k1) {
        constexpr u32 lpc = CW == 16 ? 2 : (CW == 8 ? 1 : 0);
        const u32 lq = logC + lpc, P = 1u << lq;
        const u32 kstep = nthr > P ? nthr / P : 1u;
        for (u32 pp = tid & (P - 1); pp < P; pp += nthr) {
          const u32 j = pp >> lpc, q = pp & ((1u << lpc) - 1);
          const u32 lj = lane_of(G, j);
          const u32 so0 = piece_off(0, j, q, C);
          for (u32 k = k0 + (nthr > P ? tid / P : 0u); k < k1; k += kstep) {
            const u32 d = (lj + s_rhp[k]) & CLm;
            __stcg(reinterpret_cast<uint4*>(s_op[k] + (u64)d * (CB / 8) + 16u * q),
                   *reinterpret_cast<const uint4*>(g_sm + boff + k * SB + so0));
          }
        }
      };
      if (have_next && !prefetched && boff == 0 && s_ready[nxt] && cl.nstore >= 2) {
        const u32 h = cl.nstore / 2;
        store_range(0, h);
        __syncthreads();
        if (tid == 0) s_boff[nxt] = 0;
        stage_load<CW, NT>(A, s_lf[nxt], s_cl[nxt], tid, s_rho[nxt], s_loc[nxt], s_sp[nxt]);
        const u32 h2 = (h * SB) / s_cl[nxt].slot_bytes;
        issue_slots<CW, NT>(A, s_lf[nxt], s_cl[nxt], smem_base, 0, tid, s_rho[nxt], s_loc[nxt], s_sp[nxt], 0, h2);
        store_range(h, cl.nstore);
        __syncthreads();
        issue_slots<CW, NT>(A, s_lf[nxt], s_cl[nxt], smem_base, 0, tid, s_rho[nxt], s_loc[nxt], s_sp[nxt], h2,
                            0xFFFFFFFFu);
        cp_async_commit();
        rolled = true;
      } else {
        store_range(0, cl.nstore);
        __syncthreads();  // slot reuse
      }
      pc.mark(PH_STORE);
    } else {
      // ---- post-rotation + carry resolution + store: NG slots per round ------------
      for (u32 b0 = 0; b0 < cl.nstore; b0 += NG) {
        const u32 nb = min(cl.nstore - b0, NG);
        const u32 sl = b0 + g;
        const bool act = g < nb;
        const u32 so = boff + sl * SB;
        Ch<CW> w;
        int top = 0;
        if (act && (A.debug_skip & 2)) {
          lds_at(w, so, fi);
          sts_i32(scr + 4 * tid, 0);
        } else if (act) {
          const SymExp P = cached ? s_crot[cl.nload + sl] : A.rots[cl.post_begin + sl];
          const Rot R = make_rot<CW>(post_exp(A, cl, lf, P, sl), A.N);
          bool neg;
          if (R.o == 0) {
            const u32 j = (i - R.q) & Cm;
            lds_ch(w, so, j, C);
            top = lds_i32(so + W4 + 4 * j);
            neg = ((i < R.q) ? 1u : 0u) != R.sneg;
          } else {
            neg = rot_chunk<CW>(w, top, so, so + W4, R, Cm, i);
          }
          top = exact_from<CW>(w, top, neg);
          sts_i32(scr + 4 * tid, top);
        }
        __syncthreads();
        pc.mark(PH_POST);
        // fold in the top of the chunk below (one step); carries that ripple
        // further (a chunk of all ones / all zeros) take the slow path
        int rare = 0;
        if (act) {
          const int in = i ? lds_i32(scr + 4 * (tid - 1)) : 0;
          const int e = in ? ch_add_small<CW>(w, in) : 0;
          if (i == Cm) {
            top += e;
          } else {
            if (e) rare = 1;
            top = e;  // carry still owed to chunk i+1
          }
        }
        if (__syncthreads_or(rare)) {
          for (;;) {
            if (act && i != Cm) sts_i32(scr + 4 * tid, top);
            __syncthreads();
            int any = 0;
            if (act) {
              const int in = i ? lds_i32(scr + 4 * (tid - 1)) : 0;
              const int e = in ? ch_add_small<CW>(w, in) : 0;
              if (i == Cm) {
                top += e;
              } else {
                if (e) any = 1;
                top = e;
              }
            }
            if (!__syncthreads_or(any)) break;
          }
        }
        // resolved chunks back into their (free) slots, then a coalesced copy
        // of whole elements to HBM (full 32-byte sectors per request)
        if (act) {
          sts_at<CW>(so, fi, w);
          if (i == Cm) sts_i32(so + W4, top);
        }
        __syncthreads();  // scratch reuse
        pc.mark(PH_STORE);
      }
      // the whole leaf is resolved in shared memory: one coalesced copy to HBM
      copy_slots<CW, false, NT>(A, G, lf, locm, 0, cl.nstore, smem_base, boff, tid);
      for (u32 x = tid; x < cl.nstore; x += nthr)
        __stcg(reinterpret_cast<long long*>(elem_ptr(A, out_buf(locm, x), lf.base + (u64)x * lf.stride) + W4e),
               (long long)lds_i32(boff + x * SB + W4));
      if (A.T) {  // element format out: the lanes carry no tops
        if ((CL & 3) == 0) {
          const u32 per = CL / 4;  // 16-byte groups of int32 tops per element
          for (u32 x = tid; x < cl.nstore * per; x += nthr) {
            const u32 k = x / per, q = x - k * per;
            __stcg(reinterpret_cast<uint4*>(tops_row(A, out_buf(locm, k), lf.base + (u64)k * lf.stride)) + q,
                   make_uint4(0, 0, 0, 0));
          }
        } else {
          for (u32 x = tid; x < cl.nstore * CL; x += nthr) {
            const u32 k = x / CL, q = x - k * CL;
            tops_row(A, out_buf(locm, k), lf.base + (u64)k * lf.stride)[q] = 0;
          }
        }
      }
      __syncthreads();  // slot reuse
    }
    pc.mark(PH_STORE);
    // publish completion: bump the phase counter; the last child of a node's
    // last phase finishes the node and reports to the parent phase in turn
    if (tid == 0 && lf.comp != kNoDep && !A.no_deps) {
      if (!(A.debug_skip & 4)) __threadfence();
      u32 k = lf.comp;
      for (;;) {
        const u32 old = atomicAdd(&A.counters[1 + k], 1u);
        const DevCounter cm = A.cmeta[k];
        if (old + 1 != cm.target || cm.next == kNoDep) break;
        __threadfence();
        k = cm.next;
      }
    }
    if (have_next && !prefetched && !rolled) {
      if (tid == 0) {
        while (!dep_met(s_lf[nxt])) __nanosleep(64);
        s_boff[nxt] = 0;
      }
      __syncthreads();
      issue_load<CW, NT>(A, s_lf[nxt], s_cl[nxt], smem_base, 0, tid, s_rho[nxt], s_loc[nxt], s_sp[nxt]);
    }
    // refresh the readiness of the ticket after next (prefetch decision)
    if (tid == 0 && have_next && s_tk[nn] < A.nleaves && !s_ready[nn]) s_ready[nn] = dep_met(s_lf[nn]);
    __syncthreads();
    pc.mark(PH_WAIT);
    cur = nxt;
  }
  pc.mark(PH_WAIT);
  pc.flush(A.prof);
}

// Final canonicalisation: value = lo + hi*2^N == lo - hi -> [0, 2^N].
// Carry chains beyond word 0 are rare, handled serially.
__device__ void canon_element(std::uint8_t* el, u32 D) {
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

// Thread per element.
__global__ void canonicalize_kernel(std::uint8_t* data, u64 elem_bytes, u64 count, u32 D) {
  u64 e = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= count) return;
  canon_element(data + e * elem_bytes, D);
}

// x <- x * 2^e mod 2^N + 1 for `count` canonical elements (x in [0, 2^N],
// the top word 1 only for 2^N == -1): one CTA per element.  With t = e mod N,
// x 2^t = (lo << t mod 2^N) - (lo >> (N - t)) - top 2^t: the shifted words in
// parallel, the borrow chain by a block scan; for e mod 2N >= N (2^N == -1)
// the difference is taken the other way round.  poly_mul's 1/L = 2^(2N - ell) (polymul.hpp:82-87).
__global__ void __launch_bounds__(256) rotate_kernel(std::uint8_t* base, u64 stride, u64 e, u32 D) {
  extern __shared__ u32 s_x[];  // lo (D words), difference (D), borrow masks (<= D)
  u32* const s_d = s_x + D;
  u32* const s_b = s_x + 2 * D;
  std::uint8_t* el = base + (u64)blockIdx.x * stride;
  u32* w = reinterpret_cast<u32*>(el);
  long long* hip = reinterpret_cast<long long*>(el + (u64)D * 4);
  const u64 N = 32ull * D;
  e %= 2 * N;
  const bool neg = e >= N;
  const u64 t = neg ? e - N : e;
  const u32 ws = (u32)(t >> 5), b = (u32)(t & 31);
  const u32 nT = (u32)((t + 31) >> 5);
  const long long top = *hip;
  for (u32 i = threadIdx.x; i < D; i += blockDim.x) s_x[i] = w[i];
  __syncthreads();
  if (top != 0) {
    // x = 2^N == -1 (lo = 0): x 2^t = -2^t = (2^N - 2^t) - 2^N, or 2^N for t = 0
    for (u32 i = threadIdx.x; i < D; i += blockDim.x)
      w[i] = t == 0 ? 0u : i < ws ? 0u : (i == ws ? (0xFFFFFFFFu << b) : 0xFFFFFFFFu);
    __syncthreads();
    if (threadIdx.x == 0) {
      *hip = t ? -1 : 1;
      canon_element(el, D);
    }
  } else {
    // d = A - S word by word: A = lo << t mod 2^N, S = lo >> (N - t) (t bits).
    // Borrows: each warp owns a contiguous segment, 32 words a step; within a
    // step the borrow-in bits are the carries of (g | p) + g + cin (g: word
    // borrows, p: word is zero), across warps a scan of segment maps.
    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const u32 seg = ((D + nw * 32 - 1) / (nw * 32)) * 32, steps = seg >> 5;
    u32* const s_g = s_b;              // D / 32 + steps * nw masks
    u32* const s_p = s_b + steps * nw;  // (fits in the D-word flag area)
    u32 c0 = 0, c1 = 1;  // segment borrow out for borrow in 0 / 1
    for (u32 k = 0; k < steps; ++k) {
      const u32 i = warp * seg + k * 32 + lane;
      u32 g = 0, pr = 1;
      if (i < D) {
        const u32 x0 = i >= ws ? s_x[i - ws] : 0u;
        const u32 x1 = i >= ws + 1 ? s_x[i - ws - 1] : 0u;
        const u32 a = b ? (x0 << b) | (x1 >> (32 - b)) : x0;
        u32 sv = 0;
        if (i < nT) {
          const u64 st = N - t + 32ull * i;
          const u32 q = (u32)(st >> 5), sh = (u32)(st & 31);
          const u32 l0 = q < D ? s_x[q] : 0u, l1 = q + 1 < D ? s_x[q + 1] : 0u;
          sv = sh ? (l0 >> sh) | (l1 << (32 - sh)) : l0;
        }
        // e mod 2N >= N: x 2^e = -(A - S) = S - A
        const u32 d = neg ? sv - a : a - sv;
        s_d[i] = d;
        g = neg ? sv < a : a < sv;
        pr = d == 0;
      }
      const u32 gm = __ballot_sync(0xFFFFFFFFu, g), pm = __ballot_sync(0xFFFFFFFFu, pr);
      if (lane == 0) {
        s_g[warp * steps + k] = gm;
        s_p[warp * steps + k] = pm;
      }
      c0 = (u32)(((u64)(gm | pm) + gm + c0) >> 32);
      c1 = (u32)(((u64)(gm | pm) + gm + c1) >> 32);
    }
    __shared__ u32 s_c0[32], s_c1[32];
    if (lane == 0) {
      s_c0[warp] = c0;
      s_c1[warp] = c1;
    }
    __syncthreads();
    u32 c = 0;
    for (u32 k = 0; k < warp; ++k) c = c ? s_c1[k] : s_c0[k];
    for (u32 k = 0; k < steps; ++k) {
      const u32 i = warp * seg + k * 32 + lane;
      const u32 gm = s_g[warp * steps + k], am = gm | s_p[warp * steps + k];
      const u64 sum = (u64)am + gm + c;
      const u32 bin = (((u32)sum ^ am ^ gm) >> lane) & 1u;
      c = (u32)(sum >> 32);
      if (i < D) s_d[i] -= bin;
    }
    __shared__ u32 s_out;
    if (threadIdx.x == blockDim.x - 1) s_out = c;  // borrow out of the top word
    __syncthreads();
    const long long out = s_out;
    for (u32 i = threadIdx.x; i < D; i += blockDim.x) w[i] = s_d[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      *hip = -out;  // value = lo - out 2^N
      canon_element(el, D);
    }
  }
  if (!neg || top == 0) return;  // (the sign is in the difference above)
  __syncthreads();
  // -x = 2^N + 1 - x (x canonical): 0 -> 0, 2^N -> 1, else ~lo + 2
  const long long h = *hip;
  int nz = 0;
  for (u32 i = threadIdx.x; i < D; i += blockDim.x) nz |= w[i] != 0;
  nz = __syncthreads_or(nz);
  if (h) {
    for (u32 i = threadIdx.x; i < D; i += blockDim.x) w[i] = i == 0 ? 1u : 0u;
    if (threadIdx.x == 0) *hip = 0;
    return;
  }
  if (!nz) return;
  for (u32 i = threadIdx.x; i < D; i += blockDim.x) w[i] = ~w[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 c = 2;
    for (u32 i = 0; i < D && c; ++i) {
      const u64 v = (u64)w[i] + c;
      w[i] = (u32)v;
      c = v >> 32;
    }
    *hip = c ? 1 : 0;  // only for x = 1: ~1 + 2 = 2^N
  }
}

// Outputs the schedule left in the shadow buffer: element (lanes, top word)
// and its tops row back to the caller's view.
__global__ void shadow_copy_kernel(std::uint8_t* data, const std::uint8_t* data2, u64 eb, int* T, u64 tloc, u32 CL,
                                   const u64* idx, u32 D) {
  const u64 e = idx[blockIdx.x];
  const uint4* src = reinterpret_cast<const uint4*>(data2 + e * eb);
  uint4* dst = reinterpret_cast<uint4*>(data + e * eb);
  const u32 pieces = (4 * D + 8 + 15) / 16;
  for (u32 x = threadIdx.x; x < pieces; x += blockDim.x) dst[x] = __ldcg(src + x);
  for (u32 x = threadIdx.x; x < CL; x += blockDim.x) T[e * CL + x] = T[tloc + e * CL + x];
}

// Carry-save lanes -> canonical element format, one CTA per element: lane p
// takes the top of lane p-1 (lane 0 takes minus the top of lane C-1 and the
// element top word: 2^N == -1).  Only word 0 of a lane is touched unless a
// carry ripples; lanes whose carry-in is zero are not touched at all.
//
// frot (wave engine): per element, a sub-lane rotation 2^o its last writer
// deferred (Plan::final_rot), applied here after the fold: x = lo + h 2^N
// times 2^o is (lo << o mod 2^N) - S with S = (lo >> (N - o)) + h 2^o, a
// number of about o bits -- the shifted words in parallel, then S subtracted
// serially (the borrow stops after a few words unless a run of zero words).
// Dynamic shared memory: 4 D bytes when frot is set.
//
// idx (optional): the element of CTA b is idx[b] (else idx0 + b istride);
// src (optional): the element lives in this buffer (the shadow copy; T then
// points at that buffer's tops) -- it is copied into place first.
__global__ void __launch_bounds__(256) cs_fold_kernel(std::uint8_t* data, u64 eb, const int* T, u32 CL, u32 CW,
                                                      u32 logLanes, u32 logS, u32 D, u64 idx0, u64 istride,
                                                      const u32* frot, const u64* idx, const std::uint8_t* src,
                                                      u32 src_cm = 0) {
  __shared__ int s_pend[1024];
  extern __shared__ u32 s_old[];  // D words (frot only)
  const u64 e = idx ? idx[blockIdx.x] : idx0 + (u64)blockIdx.x * istride;
  std::uint8_t* el = data + e * eb;
  const int* Te = T + e * CL;
  auto tix = [&](u32 p) { return ((p & ((1u << logS) - 1)) << (logLanes - logS)) | (p >> logS); };
  bool fused = false;  // pass 1 done while copying
  if (src && CW == 8) {
    // 256-bit lanes: every lane is read from the source once, takes its
    // carry-in in registers and is written into place (no second visit).
    // Coset-major source (wave_tma.cuh): lane p = coset p mod 2^src_cm, row
    // p >> src_cm, 1 KB per coset, 16-byte halves swapped on rows with bit 2
    // set; the top word follows the lanes as usual.  (Reading in source order
    // and scattering the writes, or staging through shared memory, measured
    // slower: profiles/r02_experiments.md.)
    const std::uint8_t* se = src + e * eb;
    const long long hsrc = *reinterpret_cast<const long long*>(se + (u64)D * 4);
    for (u32 p = threadIdx.x; p < CL; p += blockDim.x) {
      u32 off = 32u * p, sw = 0;
      if (src_cm) {
        const u32 row = p >> src_cm, cs = p & ((1u << src_cm) - 1);
        off = (cs << 10) | (row << 5);
        sw = (row >> 2) & 1u;
      }
      const uint4* sp = reinterpret_cast<const uint4*>(se + off);
      const uint4 lo = __ldcg(sp + sw), hi = __ldcg(sp + (sw ^ 1u));
      u32 v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
      const long long cin = p ? (long long)Te[tix(p - 1)] : -((long long)Te[tix(CL - 1)] + hsrc);
      long long c = cin;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const long long x = (long long)v[k] + c;
        v[k] = (u32)x;
        c = x >> 32;
      }
      uint4* dp = reinterpret_cast<uint4*>(el + 32u * p);
      dp[0] = make_uint4(v[0], v[1], v[2], v[3]);
      dp[1] = make_uint4(v[4], v[5], v[6], v[7]);
      s_pend[p] = (int)c;
    }
    fused = true;
  } else if (src) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src + e * eb);
    uint4* d4 = reinterpret_cast<uint4*>(el);
    const u32 pieces = (4 * D + 8 + 15) / 16;
    for (u32 x = threadIdx.x; x < pieces; x += blockDim.x) d4[x] = __ldcg(s4 + x);
    __syncthreads();
  }
  long long* hip = reinterpret_cast<long long*>(el + (u64)D * 4);
  u32* w = reinterpret_cast<u32*>(el);
  const u32 o = frot ? frot[e] : 0u;
  // pass 1: every lane takes its carry-in
  for (u32 p = threadIdx.x; !fused && p < CL; p += blockDim.x) {
    long long cin;
    if (p) {
      cin = Te[tix(p - 1)];
    } else {
      cin = -((long long)Te[tix(CL - 1)] + *hip);
    }
    int co = 0;
    if (cin) {
      u32* lw = w + (u64)p * CW;
      long long v = (long long)lw[0] + cin;
      lw[0] = (u32)v;
      long long c = v >> 32;
      for (u32 k = 1; k < CW && c; ++k) {
        v = (long long)lw[k] + c;
        lw[k] = (u32)v;
        c = v >> 32;
      }
      co = (int)c;
    }
    s_pend[p] = co;
  }
  // carries out of a lane come from a lane of all ones / all zeros (sparse
  // values: every high lane).  A lane passes carry x in {-1, 0, 1} on as
  // own + [x = 1, lane all ones] - [x = -1, lane all zeros]; those maps are
  // composed by a block scan over per-thread lane chunks, then every lane
  // takes its carry; the top lane's goes to the element top word
  int any = 0;
  for (u32 p = threadIdx.x; p < CL; p += blockDim.x) any |= s_pend[p];
  if (!__syncthreads_or(any)) {
    if (threadIdx.x == 0) *hip = 0;  // lo is canonical: every lane in [0, 2^lane)
  } else {
    // map m: 2-bit fields m(x) + 1 at bit 2 (x + 1); identity 0x24
    auto apply = [](u32 m, int x) { return (int)((m >> (2 * (x + 1))) & 3u) - 1; };
    auto compose = [&](u32 lo, u32 up) {  // up after lo
      u32 r = 0;
      for (int x = -1; x <= 1; ++x) r |= (u32)(apply(up, apply(lo, x)) + 1) << (2 * (x + 1));
      return r;
    };
    const u32 per = (CL + blockDim.x - 1) / blockDim.x;
    const u32 p0 = min(CL, threadIdx.x * per), p1 = min(CL, p0 + per);
    u32 M = 0x24;
    for (u32 p = p0; p < p1; ++p) {
      const u32* lw = w + (u64)p * CW;
      u32 and_ = 0xFFFFFFFFu, or_ = 0;
      for (u32 k = 0; k < CW; ++k) {
        and_ &= lw[k];
        or_ |= lw[k];
      }
      const int own = s_pend[p];
      const int fm = own - (or_ == 0 ? 1 : 0), fp = own + (and_ == 0xFFFFFFFFu ? 1 : 0);
      M = compose(M, (u32)(fm + 1) | ((u32)(own + 1) << 2) | ((u32)(fp + 1) << 4));
    }
    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (u32 d = 1; d < 32; d <<= 1) {
      const u32 m2 = __shfl_up_sync(0xFFFFFFFFu, M, d);
      if (lane >= d) M = compose(m2, M);
    }
    __shared__ u32 s_wm[32];
    if (lane == 31) s_wm[warp] = M;
    __syncthreads();
    int pre = 0;  // carry into this warp's first lane
    for (u32 k = 0; k < warp; ++k) pre = apply(s_wm[k], pre);
    const int incl = apply(M, pre);
    const int up = __shfl_up_sync(0xFFFFFFFFu, incl, 1);
    int x = lane ? up : pre;
    for (u32 p = p0; p < p1; ++p) {
      if (x) {
        u32* lw = w + (u64)p * CW;
        long long c = x;
        for (u32 k = 0; k < CW && c; ++k) {
          const long long v = (long long)lw[k] + c;
          lw[k] = (u32)v;
          c = v >> 32;
        }
        x = s_pend[p] + (int)c;
      } else {
        x = s_pend[p];
      }
    }
    __shared__ int s_h;
    if (threadIdx.x == blockDim.x - 1) s_h = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      // value = lo + h 2^N; the lane-0 term already took the old element top
      *hip = s_h;
      canon_element(el, D);
    }
  }
  if (!o) return;
  __syncthreads();
  for (u32 i = threadIdx.x; i < D; i += blockDim.x) s_old[i] = w[i];
  __syncthreads();
  const u32 ws = o >> 5, b = o & 31;
  for (u32 i = threadIdx.x; i < D; i += blockDim.x) {
    const u32 x0 = i >= ws ? s_old[i - ws] : 0u;
    const u32 x1 = i >= ws + 1 ? s_old[i - ws - 1] : 0u;
    w[i] = b ? (x0 << b) | (x1 >> (32 - b)) : x0;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const u32 N = 32 * D, nT = (o + 31) >> 5;
  const long long h = *hip;
  __int128 acc = 0;
  for (u32 i = 0; i < D; ++i) {
    acc += w[i];
    if (i < nT) {  // word i of lo >> (N - o)
      const u32 st = N - o + 32 * i, q = st >> 5, sh = st & 31;
      const u32 lo0 = s_old[q], lo1 = q + 1 < D ? s_old[q + 1] : 0u;
      acc -= sh ? (lo0 >> sh) | (lo1 << (32 - sh)) : lo0;
    }
    if (i == ws) acc -= (__int128)h << b;
    w[i] = (u32)acc;
    acc >>= 32;
    if (i + 1 >= nT && i >= ws && acc == 0) break;
  }
  *hip = (long long)acc;
  if (acc) canon_element(el, D);
}

}  // namespace fermat
}  // namespace cftft_b200
