// wave_coset.cuh -- warp-level engine for small coset leaves (2^lambda <= 8
// coefficients), one launch per wave of independent leaves.
//
// A coset leaf's rotations are whole multiples of its coset step (planner.hpp,
// DevClass), so lane p of every output depends only on the lanes
// p' == p (mod step) of its inputs.  Here one warp owns 2^cb cosets x C'
// positions (cb = 6 - lambda, C' = 2^(lambda-1)): lane l holds the 256-bit
// chunk of element lane  c + step * pos  (c = coset, pos = l >> cb) of every
// slot of the leaf.  A butterfly reads its own chunk of `a` and the chunk of
// the rotated `b` from the lane (pos - q) of the same coset -- a permutation
// inside the warp -- so the whole leaf runs with __syncwarp only: no CTA
// barriers, no tickets, no dependency counters (launch order separates the
// waves).  Chunks live in a per-warp shared-memory tile [slot][word][lane]
// (conflict-free: a warp always touches 32 distinct lanes of one row).
//
// Formats are the persistent engine's (fermat_leaf.cuh): carry-save lanes
// with an int32 top per lane in the tops array, the coefficient's top word
// folded into lane 0 by the lane that reads it, the two-buffer ping-pong of
// DevLeaf::locoff, the pre / post rotations of DevClass / DevLeaf.
#pragma once

#include "fermat_leaf.cuh"

namespace cftft_b200 {
namespace fermat {

struct WaveArgs {
  const DevLeaf* leaves;  // this wave's coset tickets (one per leaf)
  u32 nleaves;
  const DevClass* classes;
  const DevOp* ops;
  const SymExp* rots;
  std::uint8_t* data;   // caller's view
  std::uint8_t* data2;  // shadow buffer
  u64 elem_bytes;
  int* T;               // tops, [buffer][element][lane] (natural lane order); always set (coset plans)
  u64 tloc;
  const u64* locbits;
  const u32* wops;      // packed micro-ops (Plan::wave_ops)
  const u32* levels;    // class level tables (absolute op indices; coset_wide_kernel)
  const u32* wslots;    // per-slot {pre, post} lane rotations | buffer bits (Plan::wave_slots)
  u32 lanes;            // lanes per coefficient (C)
  u32 D;                // u32 words per coefficient
  u64 M;
  u32 gpl;              // work items per ticket: its most warp groups (Plan::waves)
  u32 logS, logLanes;   // tops-array lane interleave (fermat_leaf.cuh, tops_ix)
  u32 debug;            // CFTFT_DEBUG_SKIP bits (experiments; results wrong when set)
  const void* tdesc;    // coset_tma_kernel: per-leaf descriptors of the wave (TmaLeafDesc)
  const std::uint8_t* tlay;  // coset_tma_kernel: per slot entry of wslots, bit 0 input / bit 1 output coset-major
  u32 runlog;                // coset_tma_kernel: a CTA takes runs of 2^runlog consecutive items
};
__device__ __forceinline__ u32 wave_tix(const WaveArgs& A, u32 p) {
  return ((p & ((1u << A.logS) - 1)) << (A.logLanes - A.logS)) | (p >> A.logS);
}


// y0 = a + s b, y1 = a - s b with s = (-1)^neg varying per lane, branch-free:
// -(B + tb 2^CB) = (B ^ ~0) + 1 + (tb ^ ~0) 2^CB, so with x = B ^ m, tx = tb ^ m
// (m = neg ? ~0 : 0), y0 = a + x + neg and y1 = a - x - neg as carry chains
// with a carry / borrow in.
__device__ __forceinline__ void ch_pm8(Ch<8>& y0, int& t0, Ch<8>& y1, int& t1, const Ch<8>& a, int ta,
                                       const Ch<8>& b, int tb, bool neg) {
  const u32 m = neg ? ~0u : 0u, ci = neg ? 1u : 0u;
  Ch<8> x;
#pragma unroll
  for (int w = 0; w < 8; ++w) x.w[w] = b.w[w] ^ m;
  const int tx = tb ^ (int)m;
  u32 c0, c1, d0, d1;
  asm("add.cc.u32 %9, %10, -1;\n\t"
      "addc.cc.u32 %0, %11, %19;\n\t"
      "addc.cc.u32 %1, %12, %20;\n\t"
      "addc.cc.u32 %2, %13, %21;\n\t"
      "addc.cc.u32 %3, %14, %22;\n\t"
      "addc.cc.u32 %4, %15, %23;\n\t"
      "addc.cc.u32 %5, %16, %24;\n\t"
      "addc.cc.u32 %6, %17, %25;\n\t"
      "addc.cc.u32 %7, %18, %26;\n\t"
      "addc.u32 %8, 0, 0;"
      : "=r"(y0.w[0]), "=r"(y0.w[1]), "=r"(y0.w[2]), "=r"(y0.w[3]), "=r"(y0.w[4]), "=r"(y0.w[5]), "=r"(y0.w[6]),
        "=r"(y0.w[7]), "=r"(c0), "=r"(d0)
      : "r"(ci), "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(a.w[4]), "r"(a.w[5]), "r"(a.w[6]),
        "r"(a.w[7]), "r"(x.w[0]), "r"(x.w[1]), "r"(x.w[2]), "r"(x.w[3]), "r"(x.w[4]), "r"(x.w[5]), "r"(x.w[6]),
        "r"(x.w[7]));
  asm("sub.cc.u32 %9, 0, %10;\n\t"
      "subc.cc.u32 %0, %11, %19;\n\t"
      "subc.cc.u32 %1, %12, %20;\n\t"
      "subc.cc.u32 %2, %13, %21;\n\t"
      "subc.cc.u32 %3, %14, %22;\n\t"
      "subc.cc.u32 %4, %15, %23;\n\t"
      "subc.cc.u32 %5, %16, %24;\n\t"
      "subc.cc.u32 %6, %17, %25;\n\t"
      "subc.cc.u32 %7, %18, %26;\n\t"
      "subc.u32 %8, 0, 0;"
      : "=r"(y1.w[0]), "=r"(y1.w[1]), "=r"(y1.w[2]), "=r"(y1.w[3]), "=r"(y1.w[4]), "=r"(y1.w[5]), "=r"(y1.w[6]),
        "=r"(y1.w[7]), "=r"(c1), "=r"(d1)
      : "r"(ci), "r"(a.w[0]), "r"(a.w[1]), "r"(a.w[2]), "r"(a.w[3]), "r"(a.w[4]), "r"(a.w[5]), "r"(a.w[6]),
        "r"(a.w[7]), "r"(x.w[0]), "r"(x.w[1]), "r"(x.w[2]), "r"(x.w[3]), "r"(x.w[4]), "r"(x.w[5]), "r"(x.w[6]),
        "r"(x.w[7]));
  t0 = ta + tx + (int)c0;
  t1 = ta - tx + (int)c1;
}


// Sub-lane part of a rotation by o = 32 OW + sh bits (0 < o < 256), for one
// lane of the result: bits [256 - o, 512 - o) of (B ++ A) -- A the source
// lane, B the lane below it -- plus B's top tb shifted to bit o; returns the
// result's top.  One specialisation per word offset OW (o is warp-uniform):
// the window and the shifted top are compile-time register picks.
template <int OW>
__device__ __forceinline__ int unal_ow8(Ch<8>& out, const Ch<8>& b, const Ch<8>& a, int tb, u32 sh) {
  u32 W[16];
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    W[m] = b.w[m];
    W[8 + m] = a.w[m];
  }
#pragma unroll
  for (int x = 0; x < 8; ++x) out.w[x] = __funnelshift_l(W[7 - OW + x], W[8 - OW + x], sh);
  const long long pw = (long long)tb * (1ll << sh);  // |tb| < 2^31: fits
  const u32 lo = (u32)pw, hi = (u32)((unsigned long long)pw >> 32), ext = (u32)(tb >> 31);
  Ch<8> P;
#pragma unroll
  for (int k = 0; k < 8; ++k) P.w[k] = k < OW ? 0u : (k == OW ? lo : (k == OW + 1 ? hi : ext));
  return ch_add<8>(out, out, P) + (OW == 7 ? (int)hi : (int)ext);
}
__device__ __forceinline__ int unal_combine8(Ch<8>& out, const Ch<8>& b, const Ch<8>& a, int tb, u32 o) {
  const u32 sh = o & 31;
  switch (o >> 5) {
    case 0: return unal_ow8<0>(out, b, a, tb, sh);
    case 1: return unal_ow8<1>(out, b, a, tb, sh);
    case 2: return unal_ow8<2>(out, b, a, tb, sh);
    case 3: return unal_ow8<3>(out, b, a, tb, sh);
    case 4: return unal_ow8<4>(out, b, a, tb, sh);
    case 5: return unal_ow8<5>(out, b, a, tb, sh);
    case 6: return unal_ow8<6>(out, b, a, tb, sh);
    default: return unal_ow8<7>(out, b, a, tb, sh);
  }
}


// cp.async of 16 bytes with an L2 prefetch-size hint (a warp row reads runs
// of 8 consecutive 32-byte lanes: the first miss brings in the whole run)
__device__ __forceinline__ void cp_async16_l2(u32 saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}

constexpr int kWaveWarps = 4;  // warps per CTA, at most (the launch may use fewer)

// per warp: data rows [slot][lane] of CW words, their 16-byte halves swapped
// on lanes with bit 2 set (so the 8 lanes of a 16-byte access phase hit 32
// distinct banks); tops [slot][lane]; the slots' top words; extra rows of
// unaligned rotations [slot][position] (CW words + top, padded to 16 bytes)
template <int CW>
__host__ __device__ constexpr u32 wave_xrow_words() {
  return (CW + 1 + 3) & ~3u;
}
// per ticket and slot: source / destination element and tops row (buffer
// resolved), the slot's pre / post entry of Plan::wave_slots
struct WaveSlot {
  const std::uint8_t* in;
  const int* tin;
  std::uint8_t* out;
  int* tout;
  u32 pre, post, pad0, pad1;
};
// per warp, S slots (8, or 16 for radix-16 leaves): rows [S][32] x CW words,
// tops [S][32], top words [S] (u64), extra rows [S][S/2], slot table [S]
template <int CW, int S = 8>
__host__ __device__ constexpr u32 wave_tile_words() {
  return (u32)S * 32u * CW + (u32)S * 32u + 2u * S + (u32)S * (S / 2) * wave_xrow_words<CW>() +
         (u32)S * (sizeof(WaveSlot) / 4);
}

// TIX: the tops arrays are lane-interleaved (wide plans, A.logS > 0); the
// radix-8 plans keep natural lane order and skip the index mapping
template <int CW, bool TIX, int S = 8>
__global__ void __launch_bounds__(32 * kWaveWarps, 4) coset_wave_kernel(WaveArgs A) {
  auto tix = [&](u32 p) -> u32 { return TIX ? wave_tix(A, p) : p; };
  static_assert(CW == 8, "the wave engine runs 256-bit lanes");
  extern __shared__ __align__(16) u32 wsm[];
  constexpr u32 CB = 32 * CW;
  constexpr u32 XR = wave_xrow_words<CW>();
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  u32* const tile = wsm + warp * wave_tile_words<CW, S>();
  const u32 CL = A.lanes;
  auto rowp = [&](u32 slot, u32 l) -> u32* { return tile + (slot * 32u + l) * CW; };
  constexpr u32 TW = (u32)S * 32u * CW;  // tops follow the rows
  int* const tops = reinterpret_cast<int*>(tile + TW);
  long long* const hiw = reinterpret_cast<long long*>(tile + TW + S * 32u);  // per slot top word
  u32* const xtile = tile + TW + S * 32u + 2u * S;  // extra rows: [slot][position]
  auto xrow = [&](u32 slot, u32 p) -> u32* { return xtile + (slot * (S / 2) + p) * XR; };
  WaveSlot* const si = reinterpret_cast<WaveSlot*>(xtile + (u32)S * (S / 2) * XR);
  auto swz = [](u32 l) -> u32 { return (l >> 2) & 1u; };
  auto ldw = [&](Ch<CW>& c, const u32* r, u32 sw) {
#pragma unroll
    for (u32 q = 0; q < CW / 4; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(r + 4 * (q ^ sw));
      c.w[4 * q] = v.x;
      c.w[4 * q + 1] = v.y;
      c.w[4 * q + 2] = v.z;
      c.w[4 * q + 3] = v.w;
    }
  };
  auto stw = [&](u32* r, u32 sw, const Ch<CW>& c) {
#pragma unroll
    for (u32 q = 0; q < CW / 4; ++q)
      *reinterpret_cast<uint4*>(r + 4 * (q ^ sw)) =
          make_uint4(c.w[4 * q], c.w[4 * q + 1], c.w[4 * q + 2], c.w[4 * q + 3]);
  };
  auto ld = [&](Ch<CW>& c, u32 slot, u32 l) -> int {
    ldw(c, rowp(slot, l), swz(l));
    return tops[slot * 32u + l];
  };
  auto st = [&](u32 slot, u32 l, const Ch<CW>& c, int top) {
    stw(rowp(slot, l), swz(l), c);
    tops[slot * 32u + l] = top;
  };
  const u32 tile_s = (u32)__cvta_generic_to_shared(tile);

  // descriptors one ticket ahead: the next ticket's load overlaps this one
  struct Desc {
    u64 base, stride;
    u32 cls, c0;
  };
  auto fetch = [&](u32 t) {
    Desc d{0, 0, 0, 0};
    if (t < A.nleaves) {
      const DevLeaf* p = A.leaves + t;
      d.base = p->base;
      d.stride = p->stride;
      d.cls = p->cls;
      d.c0 = p->c0;
    }
    return d;
  };
  // work items (ticket, warp group), gpl per ticket: a contiguous run per
  // CTA, dealt round-robin to its warps -- the CTA's warps stream adjacent
  // cosets of the same coefficients at once (DRAM locality), consecutive
  // items of a warp mostly share a ticket (descriptor and tables)
  const u64 gpl = A.gpl, items = (u64)A.nleaves * gpl;
  const u64 c1i = (blockIdx.x + 1ull) * items / gridDim.x;
  u64 i = blockIdx.x * items / gridDim.x + warp;
  Desc lf_next = fetch(i < c1i ? (u32)(i / gpl) : A.nleaves);
  while (i < c1i) {
    const u32 t = (u32)(i / gpl);
    const Desc lf = lf_next;
    const u64 tend = c1i < (t + 1ull) * gpl ? c1i : (t + 1ull) * gpl;
    const u64 inext = i + (tend - i + nwarps - 1) / nwarps * nwarps;  // this warp's first item past t
    lf_next = fetch(inext < c1i ? (u32)(inext / gpl) : A.nleaves);
    const DevClass cl = A.classes[lf.cls];
    const u32 ell = 31 - __clz(cl.L);
    const u32 cp = 1u << (ell - 1);   // positions per coset
    const u32 cb = 6 - ell;           // coset bits of the lane index
    const u32 cmask = (1u << cb) - 1;
    const u32 step = cl.step;
    const u32 groups = max(1u, step >> cb);
    // the ticket's slot table and the class's first 32 packed ops, one word
    // per lane, broadcast by shuffles (no dependent global loads in the loops)
    const u32 span = max(cl.nload, cl.nstore);
    const u32 nwo = cl.nops;
    const u32 opv0 = lane < nwo ? A.wops[cl.wop_begin + lane] : 0u;
    // the ticket's slots, resolved once (lane k: slot k) and read back by
    // broadcast; the previous ticket's groups are done with the table
    __syncwarp();
    const u32 pre_l = lane < cl.nload ? A.wslots[lf.c0 + 2 * lane] : 0u;
    // any unaligned pre-rotation in the ticket (warp-uniform)
    const bool tunal = __any_sync(0xffffffffu, ((pre_l & 0x3FFFFFFFu) % CB) != 0);
    if (lane < span) {
      const u32 pre = A.wslots[lf.c0 + 2 * lane], post = A.wslots[lf.c0 + 2 * lane + 1];
      const u64 e = lf.base + (u64)lane * lf.stride;
      WaveSlot w;
      w.in = (pre >> 31 ? A.data2 : A.data) + e * A.elem_bytes;
      w.tin = A.T + (pre >> 31 ? A.tloc : 0) + e * CL;
      w.out = (post >> 31 ? A.data2 : A.data) + e * A.elem_bytes;
      w.tout = A.T + (post >> 31 ? A.tloc : 0) + e * CL;
      w.pre = pre;
      w.post = post;
      w.pad0 = w.pad1 = 0;
      si[lane] = w;
    }
    __syncwarp();
    for (; i < tend; i += nwarps) {
      const u32 g = (u32)(i - (u64)t * gpl);
      if (g >= groups) continue;
      const u32 c = (g << cb) + (lane & cmask);
      const u32 pos = lane >> cb;
      const bool act = c < step && pos < cp;
      const u32 L0 = c + step * pos;  // this lane's element lane (frame)

      // ---- load: gather through the pre-rotation (all slots in flight at
      //      once), then fold the top word and negate wrapped lanes
      // A pre-rotation by r = q*lane + o bits reads source lane L0 - q ("A");
      // when o != 0 the output lane also takes the top o bits of lane
      // L0 - q - 1 ("B") -- the A of the previous lane of this warp, or, for a
      // warp's first coset, an extra row this lane loads itself.
      u32 wrapA = 0, wrapB = 0, zeroA = 0, zeroB = 0, unal = 0;  // per-slot bit masks
      // slot table: {pre bits | in-buffer << 31, post lanes | out-buffer << 31}
      const bool first = (lane & cmask) == 0;
#pragma unroll
      for (u32 k = 0; k < (u32)S; ++k) {
        if (!act || k >= cl.nload) break;
        const u32 r = si[k].pre & 0x3FFFFFFFu;
        const u32 q = r / CB, o = r % CB;
        const u32 srcA = (L0 + 2 * CL - q) & (2 * CL - 1);
        const u32 lnA = srcA & (CL - 1);
        const std::uint8_t* el = si[k].in;
        const int* tr = si[k].tin;
        const bool fresh = (si[k].pre >> 30) & 1u;  // never written: tops are zero
        const u32 so = tile_s + (k * 32u + lane) * CW * 4u, sw = swz(lane);
#pragma unroll
        for (u32 x = 0; x < CW / 4; ++x) cp_async16_l2(so + 16u * (x ^ sw), el + (u64)lnA * (CB / 8) + 16u * x);
        if (fresh)
          tops[k * 32u + lane] = 0;
        else
          cp_async4(tile_s + (TW + k * 32u + lane) * 4u, tr + tix(lnA));
        if (lane == 0) cp_async8(tile_s + (TW + S * 32u) * 4u + 8u * k, el + 4ull * A.D);
        if (lnA == 0) zeroA |= 1u << k;
        if (srcA >= CL) wrapA |= 1u << k;
        if (o) {
          unal |= 1u << k;
          const u32 srcB = (srcA + 2 * CL - 1) & (2 * CL - 1);
          const u32 lnB = srcB & (CL - 1);
          if (lnB == 0) zeroB |= 1u << k;
          if (srcB >= CL) wrapB |= 1u << k;
          if (first) {
            const u32 xo = (u32)__cvta_generic_to_shared(xrow(k, pos));
#pragma unroll
            for (int x = 0; x < CW / 4; ++x) cp_async16(xo + 16u * x, el + (u64)lnB * (CB / 8) + 16u * x);
            if (fresh)
              xrow(k, pos)[CW] = 0u;
            else
              cp_async4(xo + 4u * CW, tr + tix(lnB));
          }
        }
      }
      cp_async_wait_all();
      __syncwarp();
      // full networks without unaligned pre-rotations settle their rows as
      // they first read them into registers (no separate pass)
      const bool fused = cl.wnet && !tunal;
      // rows -> true carry-save values of their source lanes: the coefficient's
      // top word folded into (every copy of) source lane 0, wrapped lanes negated
      auto settle = [&](u32* rw, u32 sw, int* tp, u32 k, bool zero, bool neg) {
        int top = *tp;
        if (!zero && !neg) return;
        Ch<CW> w;
        ldw(w, rw, sw);
        if (zero) {
          const int hi = (int)hiw[k];
          if (hi) top += ch_add_small<CW>(w, -hi);
        }
        if (neg) top = exact_from<CW>(w, top, true);
        stw(rw, sw, w);
        *tp = top;
      };
      for (u32 k = 0; k < (fused ? 0u : cl.nload); ++k) {
        if (!act) break;
        settle(rowp(k, lane), swz(lane), tops + k * 32u + lane, k, (zeroA >> k) & 1u, (wrapA >> k) & 1u);
        if (((unal >> k) & 1u) && first)
          settle(xrow(k, pos), 0u, reinterpret_cast<int*>(xrow(k, pos) + CW), k, (zeroB >> k) & 1u,
                 (wrapB >> k) & 1u);
      }
      __syncwarp();
      // unaligned slots: lane L0 = bits [Λ - o, 2Λ - o) of (B ++ A) plus B's top at bit o
      for (u32 k = 0; k < (tunal ? cl.nload : 0u); ++k) {
        const u32 o = (si[k].pre & 0x3FFFFFFFu) % CB;  // uniform across the warp
        if (o == 0) continue;
        Ch<CW> out;
        int otop = 0;
        if (act) {
          Ch<CW> a, b;
          ld(a, k, lane);
          int tb;
          if (first) {
            ldw(b, xrow(k, pos), 0u);
            tb = (int)xrow(k, pos)[CW];
          } else {
            tb = ld(b, k, lane - 1);
          }
          otop = unal_combine8(out, b, a, tb, o);
          if (L0 == 0) {
            // Lane 0's B is lane C-1's A seen through 2^N == -1: the split of
            // -v must be -(split of v), and floor(-v 2^o / 2^Λ) is one short
            // of that whenever v's low Λ-o bits (the part lane C-1 keeps) are
            // nonzero (negation preserves that).
            const u32 nb = CB - o;
            u32 nz = 0;
#pragma unroll
            for (int x = 0; x < CW; ++x) {
              const u32 lo = 32u * x;
              const u32 m = lo + 32u <= nb ? ~0u : (lo < nb ? (1u << (nb - lo)) - 1u : 0u);
              nz |= b.w[x] & m;
            }
            if (nz) otop += ch_add_small<CW>(out, 1);
          }
        }
        __syncwarp();
        if (act) st(k, lane, out, otop);
        __syncwarp();
      }
      // ---- store: scatter through the post-rotation, carry-save out
      // (called by every lane of the warp)
      auto store_slot = [&](u32 k, Ch<CW>& w, int top) {
        const WaveSlot* sk = si + k;
        const u32 post = sk->post;
        const u32 dst = (L0 + (post & 0x3FFFFFFFu)) & (2 * CL - 1);
        const u32 d = dst & (CL - 1);
        std::uint8_t* el = sk->out;
        if (dst >= CL) top = exact_from<CW>(w, top, true);
        if (post & (1u << 30)) {
          // a final output (warp-uniform): output lane d takes the top of
          // lane d-1 (lane 0: minus lane C-1's, 2^N == -1) from the warp lane
          // before it when that lane holds it -- the final fold then only
          // touches lanes at warp-group edges and rare carries
          const int up = __shfl_up_sync(0xffffffffu, top, 1);
          const bool takes = (lane & cmask) != 0;
          const bool gives = (lane & cmask) != cmask && c + 1 < step;
          const int cin = takes ? (d == 0 ? -up : up) : 0;
          const int co = cin ? ch_add_small<CW>(w, cin) : 0;
          top = co + (gives ? 0 : top);
        }
        if (!act) return;
        uint4* gp = reinterpret_cast<uint4*>(el + (u64)d * (CB / 8));
#pragma unroll
        for (int q = 0; q < CW / 4; ++q)
          __stcg(gp + q, make_uint4(w.w[4 * q], w.w[4 * q + 1], w.w[4 * q + 2], w.w[4 * q + 3]));
        __stcg(sk->tout + tix(d), top);
        // the lane that took the top word (source lane 0), or for an
        // output-only slot the lane writing lane 0, clears the output's
        const bool owner = k < cl.nload ? ((L0 + 2 * CL - (sk->pre & 0x3FFFFFFFu) / CB) & (CL - 1)) == 0 : d == 0;
        if (owner) __stcg(reinterpret_cast<long long*>(el + 4ull * A.D), 0ll);
      };

      if (cl.wnet) {
        // ---- the full 8-point network in registers: a butterfly's b comes
        //      from the lane `q` positions back in the same coset (a shuffle,
        //      none when q = 0).  Rows are lane-private from here on (no
        //      __syncwarp): the span-4 level runs pairwise through the rows,
        //      the two 4-point halves in registers, and outputs go straight
        //      from registers to global memory.
        auto bfly = [&](Ch<CW>& a, int& ta, Ch<CW>& b, int& tb, u32 oi) {
          const u32 qv = __shfl_sync(0xffffffffu, opv0, (int)oi) >> 16;
          Ch<CW> y0;
          int t0;
          if (qv == 0) {  // warp-uniform
            t0 = ch_add(y0, a, b) + ta + tb;
            Ch<CW> y1;
            tb = ch_sub(y1, a, b) + ta - tb;
            b = y1;
          } else {
            const u32 sneg = qv >= cp ? 1u : 0u;
            const u32 qq = qv - (sneg ? cp : 0u);
            const u32 pl = (((pos - qq) & (cp - 1)) << cb) | (lane & cmask);
            const bool neg = ((pos < qq) ? 1u : 0u) != sneg;
            Ch<CW> bp;
#pragma unroll
            for (int w = 0; w < CW; ++w) bp.w[w] = __shfl_sync(0xffffffffu, b.w[w], (int)pl);
            const int tbp = __shfl_sync(0xffffffffu, tb, (int)pl);
            ch_pm8(y0, t0, b, tb, a, ta, bp, tbp, neg);
          }
          a = y0;
          ta = t0;
        };
        // span-4 level (op 0..3 or 8..11): pairs (j, j + 4) through the rows
        // a row read into registers; `fresh` (fused settle): first read of the slot
        // first: the slot's first read (slots >= nload are truncated inputs: zero)
        auto ldx = [&](Ch<CW>& c, u32 k, bool first, bool fresh) -> int {
          if (first && k >= cl.nload) {  // warp-uniform
#pragma unroll
            for (int w = 0; w < CW; ++w) c.w[w] = 0;
            return 0;
          }
          int top = ld(c, k, lane);
          if (fresh) {
            if ((zeroA >> k) & 1u) {
              const int hi = (int)hiw[k];
              if (hi) top += ch_add_small<CW>(c, -hi);
            }
            if ((wrapA >> k) & 1u) top = exact_from<CW>(c, top, true);
          }
          return top;
        };
        // np pairs (b0 + j, b0 + j + sp), ops o0 + j, through the rows
        auto spanp = [&](u32 np, u32 sp, u32 b0, u32 o0, bool out, bool first, bool fresh) {
#pragma unroll 1
          for (u32 j = 0; j < np; ++j) {
            Ch<CW> a, b;
            const u32 ka = b0 + j, kb = ka + sp;
            int ta = ldx(a, ka, first, fresh), tb = ldx(b, kb, first, fresh);
            bfly(a, ta, b, tb, o0 + j);
            if (out) {
              if (ka < cl.nstore) store_slot(ka, a, ta);
              if (kb < cl.nstore) store_slot(kb, b, tb);
            } else {
              st(ka, lane, a, ta);
              st(kb, lane, b, tb);
            }
          }
        };
        // a 4-point half (slots b0+4h..b0+4h+3) of the 8-point network whose
        // ops start at ob: spans 1,2 (DIT: ops 2h, 2h+1 then 4+2h, 5+2h) or
        // 2,1 (DIF: ops 4+2h, 5+2h then 8+2h, 9+2h)
        auto half4 = [&](u32 b0, u32 ob, u32 h, bool dit, bool out, bool first, bool fresh) {
          Ch<CW> x[4];
          int tx[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) tx[k] = ldx(x[k], b0 + 4 * h + k, first, fresh);
          if (dit) {
            bfly(x[0], tx[0], x[1], tx[1], ob + 2 * h);
            bfly(x[2], tx[2], x[3], tx[3], ob + 2 * h + 1);
            bfly(x[0], tx[0], x[2], tx[2], ob + 4 + 2 * h);
            bfly(x[1], tx[1], x[3], tx[3], ob + 5 + 2 * h);
          } else {
            bfly(x[0], tx[0], x[2], tx[2], ob + 4 + 2 * h);
            bfly(x[1], tx[1], x[3], tx[3], ob + 5 + 2 * h);
            bfly(x[0], tx[0], x[1], tx[1], ob + 8 + 2 * h);
            bfly(x[2], tx[2], x[3], tx[3], ob + 9 + 2 * h);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const u32 sk = b0 + 4 * h + k;
            if (out) {
              if (sk < cl.nstore) store_slot(sk, x[k], tx[k]);
            } else {
              st(sk, lane, x[k], tx[k]);
            }
          }
        };
        // the 8-point network of slots b0..b0+7, ops ob..ob+11
        auto net8 = [&](u32 b0, u32 ob, bool dif, bool out, bool first, bool fresh) {
          if (dif) {  // span 4, then the halves
            spanp(4, 4, b0, ob, false, first, fresh);
            half4(b0, ob, 0, false, out, false, false);
            half4(b0, ob, 1, false, out, false, false);
          } else {  // the halves, then span 4
            half4(b0, ob, 0, true, false, first, fresh);
            half4(b0, ob, 1, true, false, first, fresh);
            spanp(4, 4, b0, ob + 8, out, false, false);
          }
        };
        net8(0, 0, cl.wnet == 1, true, true, fused);
        __syncwarp();
        continue;
      }

      // ---- the leaf program: every lane runs every micro-op on its chunk
      u32 opv = opv0;
      for (u32 o = 0; o < cl.nops; ++o) {
        if (o && (o & 31) == 0) opv = o + lane < cl.nops ? A.wops[cl.wop_begin + o + lane] : 0u;
        const u32 wop = __shfl_sync(0xffffffffu, opv, (int)(o & 31));
        struct {
          u32 type, a, b, q;
        } op{wop & 15u, (wop >> 4) & 63u, (wop >> 10) & 63u, wop >> 16};
        Ch<CW> a, b, y0, y1;
        int pa = 0, pb = 0, t0 = 0, t1 = 0;
        if (act) {
          pa = ld(a, op.a, lane);
          if (op.type == OP_COPY) {
            y1 = a;
            t1 = pa;
          } else {
            const u32 qv = op.q;  // positions, < 2 cp
            const u32 sneg = qv >= cp ? 1u : 0u;
            const u32 qq = qv - (sneg ? cp : 0u);
            const u32 pl = (((pos - qq) & (cp - 1)) << cb) | (lane & cmask);
            const bool neg = ((pos < qq) ? 1u : 0u) != sneg;
            pb = ld(b, op.b, pl);
            // y0 = a + s b, y1 = a - s b with s = (-1)^neg
            ch_pm8(y0, t0, y1, t1, a, pa, b, pb, neg);
            if (op.type == OP_SUB2 || op.type == OP_SUB2DIFF) t0 = ch_add(y0, a, y1) + pa + t1;
          }
        }
        __syncwarp();
        if (act) {
          if (op.type != OP_COPY) st(op.a, lane, y0, t0);
          if (op.type == OP_ADDSUB || op.type == OP_SUB2DIFF || op.type == OP_COPY) st(op.b, lane, y1, t1);
        }
        __syncwarp();
      }

      for (u32 k = 0; k < cl.nstore; ++k) {
        Ch<CW> w;
        const int top = ld(w, k, lane);
        store_slot(k, w, top);
      }
      __syncwarp();
    }
  }
}

}  // namespace fermat
}  // namespace cftft_b200
