// wave_tma.cuh -- radix-64 coset passes as a TMA-fed, warp-specialised
// persistent kernel (the default engine for radix-64 network waves).
//
// Same plan formats as coset_wide_kernel (wave_wide.cuh): one work item =
// (coset leaf of 64 coefficients, one lane coset c < step); the 64 slots x 32
// positions of the item are lanes c + step * pos of its coefficients (256-bit
// lanes, carry-save with an int32 top per lane); the leaf is a full 64-point
// network (DIF for the TFT, DIT for the ITFT) = two stages of eight 8-point
// register networks (Planner::wide_network).  What differs is how the data
// moves and who waits for whom:
//
//  * one CTA per SM, 8 warps; warp w owns stage-A network w and its buffer
//    of the input ring;
//  * the inputs of an item arrive by TMA (cp.async.bulk.tensor): per slot one
//    32-position box of the source coset (and, for a sub-lane pre-rotation,
//    one box of the coset below it), the 128-byte tops rows and, when a lane
//    of the item reads source lane 0, the element's top word -- completing on
//    the network's mbarrier (expect_tx).  Each warp issues its own network's
//    copies for the CTA's NEXT item as soon as it has read the current one
//    out of its buffer: a one-item-deep pipeline with no producer warp and no
//    release barriers;
//  * a warp settles its 8 slots one at a time (pre-rotation by whole cosets
//    = a row index; sub-lane part = a funnel of the two boxes; the top word
//    folded into source lane 0; lanes past 2^N negated) in place in its
//    buffer, loads them into registers, runs the stage-A network, and after a
//    CTA barrier the stage-B networks read the exchange tile and store their
//    outputs straight from registers (post-rotation = the output lane index).
//
// Shared memory (bytes, 1024-aligned base):
//   ring rows   8 networks x 16 boxes (8 slots A, 8 slots B) x 1 KB   131072
//   exchange    64 slots x 32 rows x 32 B                              65536
//   ring tops   8 networks x 8 slots x (128 B below + 128 B own)       16384
//   top words   8 networks x 8 slots x 16 B                              1024
//   exch tops   64 slots x 32 int                                         8192
//   mbarriers   8 x 8 B                                                     64
// Rows of 32 bytes are stored with the 32-byte swizzle (the 16-byte half of
// row r is swapped when bit 2 of r is set: CU_TENSOR_MAP_SWIZZLE_32B for the
// TMA boxes, the same XOR by hand for the exchange): a warp's 32 lanes reading
// 32 rows hit distinct banks.
#pragma once

#include <cuda.h>

#include "wave_coset.cuh"

namespace cftft_b200 {
namespace fermat {

constexpr int kTmaNets = 8;                // warps (= networks per stage)
constexpr int kTmaThreads = 32 * kTmaNets;
constexpr u32 kTmaRing = 0;  // per slot [B 1 KB | A 1 KB]
constexpr u32 kTmaExch = kTmaRing + 8u * 16u * 1024u;
constexpr u32 kTmaRingTops = kTmaExch + 64u * 1024u;
constexpr u32 kTmaHiw = kTmaRingTops + 8u * 8u * 256u;
constexpr u32 kTmaExchTops = kTmaHiw + 8u * 8u * 16u;
constexpr u32 kTmaBars = kTmaExchTops + 64u * 32u * 4u;
constexpr u32 kTmaSmem = kTmaBars + 8u * 8u + 1024u;  // + alignment slack

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u32 bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// one 32-position box (8 words x 32 rows) of element e, coset cls
__device__ __forceinline__ void tma_box(u32 dst, const CUtensorMap* tm, u32 cls, u32 e, u32 bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          dst),
      "l"(tm), "r"(8u * cls), "r"(0u), "r"(e), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(u32 dst, const void* src, u32 bytes, u32 bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void named_bar(u32 id, u32 n) { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }

// 32-byte row r of a tile: 16-byte half h at 32 r + 16 h (coset-major chunks
// arrive as plain 1 KB copies, so the tiles are linear; a warp reading 32 rows
// pays a 2-way bank conflict)
__device__ __forceinline__ u32 sw_off(u32 r, u32 h) { return 32u * r + 16u * h; }
__device__ __forceinline__ void lds_row(Ch<8>& c, u32 tile, u32 r) {
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3])
               : "r"(tile + sw_off(r, 0)));
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(c.w[4]), "=r"(c.w[5]), "=r"(c.w[6]), "=r"(c.w[7])
               : "r"(tile + sw_off(r, 1)));
}
__device__ __forceinline__ void sts_row(u32 tile, u32 r, const Ch<8>& c) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(tile + sw_off(r, 0)), "r"(c.w[0]), "r"(c.w[1]),
               "r"(c.w[2]), "r"(c.w[3])
               : "memory");
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(tile + sw_off(r, 1)), "r"(c.w[4]), "r"(c.w[5]),
               "r"(c.w[6]), "r"(c.w[7])
               : "memory");
}
__device__ __forceinline__ int sh_ld32(u32 a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];\n" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sh_st32(u32 a, int v) { asm volatile("st.shared.s32 [%0], %1;\n" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ long long sh_ld64(u32 a) {
  long long v;
  asm volatile("ld.shared.s64 %0, [%1];\n" : "=l"(v) : "r"(a));
  return v;
}

// (W, t) <- -(W + t 2^256) when neg, branch-free: (W ^ ~0) + 1 with the
// carry into the complemented top (exact_from's representation)
__device__ __forceinline__ void neg_if8(Ch<8>& W, int& t, bool neg) {
  const u32 m = neg ? ~0u : 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) W.w[k] ^= m;
  u32 c;
  asm("add.cc.u32 %0, %0, %9;\n\t"
      "addc.cc.u32 %1, %1, 0;\n\t"
      "addc.cc.u32 %2, %2, 0;\n\t"
      "addc.cc.u32 %3, %3, 0;\n\t"
      "addc.cc.u32 %4, %4, 0;\n\t"
      "addc.cc.u32 %5, %5, 0;\n\t"
      "addc.cc.u32 %6, %6, 0;\n\t"
      "addc.cc.u32 %7, %7, 0;\n\t"
      "addc.u32 %8, 0, 0;"
      : "+r"(W.w[0]), "+r"(W.w[1]), "+r"(W.w[2]), "+r"(W.w[3]), "+r"(W.w[4]), "+r"(W.w[5]), "+r"(W.w[6]), "+r"(W.w[7]),
        "=r"(c)
      : "r"(m & 1u));
  t = (t ^ (int)m) + (int)c;
}

// Source of one thread's lane under a slot's pre-rotation by q whole lanes:
// lane L0 = c + step pos reads srcA = L0 - q (mod 2C) = c' + step rho with
// rho in [0, 64) (rho >= 32: past 2^N, negated) -- coset c' = (c - q) mod step.
struct PreSrc {
  u32 cls;   // source coset c'
  u32 row;   // rho mod 32
  bool neg;  // rho >= 32
};
__device__ __forceinline__ PreSrc pre_src(u32 c, u32 pos, u32 q, u32 logS) {
  const u32 step = 1u << logS;
  const u32 qa = q >> logS, qb = q & (step - 1);
  const bool wrap = c < qb;
  PreSrc s;
  s.cls = wrap ? c + step - qb : c - qb;
  const u32 rho = (pos - qa - (wrap ? 1u : 0u)) & 63u;
  s.row = rho & 31u;
  s.neg = rho >= 32;
  return s;
}

// Butterflies: (a, b) <- (a + R b, a - R b).  Plain (R = 1): two carry
// chains.  Rotated: R = rotation by q coset positions (q from lane oi of opv,
// warp-uniform, < 64; q >= 32 includes 2^N == -1): b's rotated lane comes
// from warp lane pos - q, negated when that wraps -- branch-free (ch_pm8).
__device__ __forceinline__ void bfly_plain(Ch<8>& a, int& ta, Ch<8>& b, int& tb) {
  Ch<8> y0, y1;
  const int t0 = ch_add<8>(y0, a, b) + ta + tb;
  const int t1 = ch_sub<8>(y1, a, b) + ta - tb;
  a = y0;
  ta = t0;
  b = y1;
  tb = t1;
}
__device__ __forceinline__ void bfly_rot(Ch<8>& a, int& ta, Ch<8>& b, int& tb, u32 opv, int oi, u32 pos) {
  const u32 qv = (__shfl_sync(0xffffffffu, opv, oi) >> 16) & 63u;
  const u32 qq = qv & 31u;
  const u32 pl = (pos - qq) & 31u;
  const bool neg = (pos < qq) != (qv >= 32u);
  Ch<8> bp, y0, y1;
#pragma unroll
  for (int wd = 0; wd < 8; ++wd) bp.w[wd] = __shfl_sync(0xffffffffu, b.w[wd], (int)pl);
  const int tbp = __shfl_sync(0xffffffffu, tb, (int)pl);
  int t0, t1;
  ch_pm8(y0, t0, y1, t1, a, ta, bp, tbp, neg);
  a = y0;
  ta = t0;
  b = y1;
  tb = t1;
}
// Which ops of a stage-A network rotate (Planner::wide_network, unweighted
// leaves): bit j of the mask = op j.  The host checks every stage-A op
// outside the mask has q = 0 (DevicePlan::tma_wave); ops inside read q.
constexpr u32 kRotDif = (1u << 6) | (1u << 7) | (1u << 9) | (1u << 10) | (1u << 11);
constexpr u32 kRotDit = (1u << 5) | (1u << 7) | (1u << 9) | (1u << 10) | (1u << 11);
template <u32 MASK, int J>
__device__ __forceinline__ void bfly_m(Ch<8>& a, int& ta, Ch<8>& b, int& tb, u32 opv, u32 pos) {
  if constexpr ((MASK >> J) & 1u)
    bfly_rot(a, ta, b, tb, opv, J, pos);
  else
    bfly_plain(a, ta, b, tb);
}
// the 8-point network (lane j < 12 of opv: op j); DIF spans 4, 2, 1 / DIT 1, 2, 4
template <bool DIF, u32 MASK>
__device__ __forceinline__ void net8(Ch<8> (&x)[8], int (&t)[8], u32 opv, u32 pos) {
  if constexpr (DIF) {
    bfly_m<MASK, 0>(x[0], t[0], x[4], t[4], opv, pos);
    bfly_m<MASK, 1>(x[1], t[1], x[5], t[5], opv, pos);
    bfly_m<MASK, 2>(x[2], t[2], x[6], t[6], opv, pos);
    bfly_m<MASK, 3>(x[3], t[3], x[7], t[7], opv, pos);
    bfly_m<MASK, 4>(x[0], t[0], x[2], t[2], opv, pos);
    bfly_m<MASK, 5>(x[1], t[1], x[3], t[3], opv, pos);
    bfly_m<MASK, 6>(x[4], t[4], x[6], t[6], opv, pos);
    bfly_m<MASK, 7>(x[5], t[5], x[7], t[7], opv, pos);
    bfly_m<MASK, 8>(x[0], t[0], x[1], t[1], opv, pos);
    bfly_m<MASK, 9>(x[2], t[2], x[3], t[3], opv, pos);
    bfly_m<MASK, 10>(x[4], t[4], x[5], t[5], opv, pos);
    bfly_m<MASK, 11>(x[6], t[6], x[7], t[7], opv, pos);
  } else {
    bfly_m<MASK, 0>(x[0], t[0], x[1], t[1], opv, pos);
    bfly_m<MASK, 1>(x[2], t[2], x[3], t[3], opv, pos);
    bfly_m<MASK, 2>(x[4], t[4], x[5], t[5], opv, pos);
    bfly_m<MASK, 3>(x[6], t[6], x[7], t[7], opv, pos);
    bfly_m<MASK, 4>(x[0], t[0], x[2], t[2], opv, pos);
    bfly_m<MASK, 5>(x[1], t[1], x[3], t[3], opv, pos);
    bfly_m<MASK, 6>(x[4], t[4], x[6], t[6], opv, pos);
    bfly_m<MASK, 7>(x[5], t[5], x[7], t[7], opv, pos);
    bfly_m<MASK, 8>(x[0], t[0], x[4], t[4], opv, pos);
    bfly_m<MASK, 9>(x[1], t[1], x[5], t[5], opv, pos);
    bfly_m<MASK, 10>(x[2], t[2], x[6], t[6], opv, pos);
    bfly_m<MASK, 11>(x[3], t[3], x[7], t[7], opv, pos);
  }
}

// Per-leaf descriptor of a TMA wave (host-built: one load per item).
struct TmaLeafDesc {
  u64 base, stride;  // view index of slot 0, distance between slots
  u32 c0;            // offset of the leaf's {pre, post} slot entries (Plan::wave_slots)
  u32 wop_begin;     // the class's packed ops
  u32 nload;
  u32 nstore_wnet;   // nstore | wnet << 16
};
static_assert(sizeof(TmaLeafDesc) == 32, "TmaLeafDesc layout");
__device__ __forceinline__ u32 slot_a(u32 wnet, u32 w, u32 j) { return wnet == 2 ? 8u * w + j : w + 8u * j; }
__device__ __forceinline__ u32 slot_b(u32 wnet, u32 w, u32 j) { return wnet == 2 ? w + 8u * j : 8u * w + j; }

// Per-lane registers of an item: lanes 0..7 the stage-A slots, lanes 8..15
// the stage-B slots of this warp's networks (with their output addresses);
// lanes < 12 the packed ops of both networks.
struct TmaLane {
  u32 pre, post;
  u64 e;
  u32 opa, opb;
  u32 lay;  // bit 0: the slot's input is coset-major, bit 1: its output is
};
__device__ __forceinline__ TmaLane tma_lane(const WaveArgs& A, const TmaLeafDesc& d, bool valid, u32 w, u32 lane) {
  TmaLane l{};
  if (!valid) return l;
  const u32 wnet = d.nstore_wnet >> 16;
  if (lane < 16) {
    const u32 j = lane & 7u;
    const u32 slot = lane < 8 ? slot_a(wnet, w, j) : slot_b(wnet, w, j);
    l.e = d.base + (u64)slot * d.stride;
    if (slot < max(d.nload, d.nstore_wnet & 0xFFFFu)) {
      l.pre = __ldg(A.wslots + d.c0 + 2 * slot);
      l.post = __ldg(A.wslots + d.c0 + 2 * slot + 1);
      l.lay = __ldg(A.tlay + d.c0 + 2 * slot);
    }
  }
  if (lane < 12) {
    l.opa = __ldg(A.wops + d.wop_begin + w * 12u + lane);
    l.opb = __ldg(A.wops + d.wop_begin + (8u + w) * 12u + lane);
  }
  return l;
}

// TMA copies of network w's inputs of an item (coset g) into the warp's ring
// buffer (lanes 0..7: one slot each), completing on the network's mbarrier.
__device__ __forceinline__ void tma_issue(const WaveArgs& A, const CUtensorMap* tmv, const CUtensorMap* tms,
                                          const TmaLeafDesc& d, u32 g, const TmaLane& l, u32 w, u32 lane, u32 sm_s,
                                          u32 bar, u32 step) {
  const u32 slot = slot_a(d.nstore_wnet >> 16, w, lane & 7u);
  const bool ld = lane < 8 && slot < d.nload;
  u32 bytes = 0, cA = 0, cB = 0;
  bool unal = false, fresh = false, hiw = false;
  if (ld) {
    const u32 r = l.pre & 0x3FFFFFFFu;
    const u32 qb = (r >> 8) & (step - 1);
    unal = (r & 255u) != 0;
    fresh = (l.pre >> 30) & 1u;
    cA = g >= qb ? g - qb : g + step - qb;
    cB = cA ? cA - 1 : step - 1;
    hiw = cA == 0 || (unal && cA == 1);  // a lane of the item reads source lane 0
    bytes = (unal ? 2048u : 1024u) + (fresh ? 0u : (unal ? 256u : 128u)) + (hiw ? 16u : 0u);
  }
  u32 tot = bytes;
#pragma unroll
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0) mbar_expect_tx(bar, tot);
  __syncwarp();
  if (ld) {
    const bool sh = l.pre >> 31;
    const u32 sb = sm_s + kTmaRing + (w * 8u + lane) * 2048u;  // [B | A]
    const std::uint8_t* el = (sh ? A.data2 : A.data) + l.e * A.elem_bytes;
    if (l.lay & 1u) {  // coset-major: coset k of the element is the 1 KB chunk k
      if (unal && cA) {
        bulk_g2s(sb, el + (u64)cB * 1024u, 2048u, bar);
      } else {
        bulk_g2s(sb + 1024u, el + (u64)cA * 1024u, 1024u, bar);
        if (unal) bulk_g2s(sb, el + (u64)cB * 1024u, 1024u, bar);
      }
    } else {  // natural lane order: one 32-row box per coset
      const CUtensorMap* tm = sh ? tms : tmv;
      tma_box(sb + 1024u, tm, cA, (u32)l.e, bar);
      if (unal) tma_box(sb, tm, cB, (u32)l.e, bar);
    }
    if (!fresh) {
      const int* tin = A.T + (sh ? A.tloc : 0) + l.e * A.lanes;
      const u32 tdst = sm_s + kTmaRingTops + (w * 8u + lane) * 256u;  // [below | own]
      if (unal && cA) {
        bulk_g2s(tdst, tin + (u64)cB * 32u, 256u, bar);
      } else {
        bulk_g2s(tdst + 128u, tin + (u64)cA * 32u, 128u, bar);
        if (unal) bulk_g2s(tdst, tin + (u64)cB * 32u, 128u, bar);
      }
    }
    if (hiw) bulk_g2s(sm_s + kTmaHiw + (w * 8u + lane) * 16u, el + 4ull * A.D, 16u, bar);
  }
}

// The stage-B networks (every op through the rotated path) and the stores.
template <bool DIF>
__device__ __forceinline__ void stage_b_and_store(const WaveArgs& A, Ch<8> (&x)[8], int (&tx)[8], const TmaLane& ln,
                                                  const TmaLeafDesc& d, u32 c, u32 w, u32 pos, u32 exch, u32 etops,
                                                  u32 step, u32 logS) {
  const u32 wnet = DIF ? 1u : 2u;
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_b(wnet, w, j);
    lds_row(x[j], exch + slot * 1024u, pos);
    tx[j] = sh_ld32(etops + (slot * 32u + pos) * 4u);
  }
  net8<DIF, 0xFFFu>(x, tx, ln.opb, pos);
  const u32 CL = A.lanes, L0 = c + step * pos, nstore = d.nstore_wnet & 0xFFFFu;
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_b(wnet, w, j);
    if (slot >= nstore) continue;  // (warp-uniform)
    const u32 post = __shfl_sync(0xffffffffu, ln.post, (int)(8 + j));
    const u32 pre = __shfl_sync(0xffffffffu, ln.pre, (int)(8 + j));
    const u32 lay = __shfl_sync(0xffffffffu, ln.lay, (int)(8 + j));
    const u64 e = __shfl_sync(0xffffffffu, ln.e, (int)(8 + j));
    const u32 dst = (L0 + (post & 0x3FFFFFFFu)) & (2 * CL - 1);
    const u32 dl = dst & (CL - 1);
    const bool ng = dst >= CL;
    if (__any_sync(0xffffffffu, ng)) neg_if8(x[j], tx[j], ng);
    const bool osh = post >> 31;
    std::uint8_t* el = (osh ? A.data2 : A.data) + e * A.elem_bytes;
    int* tout = A.T + (osh ? A.tloc : 0) + e * CL;
    const u32 at = (lay & 2u) ? ((dl & (step - 1)) << 5) | (dl >> logS) : dl;  // coset-major: chunk, row
    uint4* gp = reinterpret_cast<uint4*>(el + (u64)at * 32u);
    __stcg(gp, make_uint4(x[j].w[0], x[j].w[1], x[j].w[2], x[j].w[3]));
    __stcg(gp + 1, make_uint4(x[j].w[4], x[j].w[5], x[j].w[6], x[j].w[7]));
    __stcg(tout + (((dl & (step - 1)) << (A.logLanes - logS)) | (dl >> logS)), tx[j]);
    bool owner;
    if (slot < d.nload) {  // the lane that read source lane 0 clears the output's top word
      const u32 q = (pre & 0x3FFFFFFFu) >> 8;
      if (q == 0) {
        owner = c == 0 && pos == 0;
      } else {
        const PreSrc s = pre_src(c, pos, q, logS);
        owner = s.cls == 0 && s.row == 0;
      }
    } else {
      owner = dl == 0;
    }
    if (owner) __stcg(reinterpret_cast<long long*>(el + 4ull * A.D), 0ll);
  }
}

template <bool DIF>
__device__ __forceinline__ void tma_item_run(const WaveArgs& A, const TmaLeafDesc& d, const TmaLane& ln, u32 c,
                                             u32 w, u32 pos, u32 sm_s, u32 step, u32 logS, Ch<8> (&x)[8],
                                             int (&tx)[8]) {
  // ---- stage-A inputs: settle the slots that need it in place, then load
  const u32 wnet = DIF ? 1u : 2u;
  const u32 ring = sm_s + kTmaRing + w * 16u * 1024u;  // slot j: [B | A] at ring + 2 KB j
  const u32 rtops = sm_s + kTmaRingTops + w * 8u * 256u;
  const u32 L0 = c + step * pos;
#pragma unroll 1
  for (u32 j = 0; j < 8; ++j) {
    if (slot_a(wnet, w, j) >= d.nload) break;  // (warp-uniform; later slots are truncated too)
    const u32 pre = __shfl_sync(0xffffffffu, ln.pre, (int)j);
    const u32 r = pre & 0x3FFFFFFFu;
    if (r == 0) continue;  // read in place below
    const u32 o = r & 255u;
    const bool fresh = (pre >> 30) & 1u;
    const PreSrc sa = pre_src(c, pos, r >> 8, logS);
    const u32 rowsB = ring + j * 2048u, rowsA = rowsB + 1024u;
    const u32 tp = rtops + j * 256u;
    const u32 hw = sm_s + kTmaHiw + (w * 8u + j) * 16u;
    Ch<8> a;
    lds_row(a, rowsA, sa.row);
    int ta = fresh ? 0 : sh_ld32(tp + 128u + 4u * sa.row);
    if (sa.cls == 0) {  // warp-uniform: the item reads source lane 0 (row 0)
      const long long hi = sh_ld64(hw);
      if (sa.row == 0 && hi) ta += ch_add_small<8>(a, -(int)hi);
    }
    if (__any_sync(0xffffffffu, sa.neg)) neg_if8(a, ta, sa.neg);
    if (o) {
      // the lane below the source: coset c'-1 on the same row, or coset
      // step-1 one row down (srcA - 1 = (step - 1) + step (rho - 1))
      u32 rowB = sa.row;
      bool negB = sa.neg;
      if (sa.cls == 0) {
        const u32 rhoB = ((sa.neg ? 32u : 0u) + sa.row - 1u) & 63u;
        rowB = rhoB & 31u;
        negB = rhoB >= 32;
      }
      Ch<8> b;
      lds_row(b, rowsB, rowB);
      int tb = fresh ? 0 : sh_ld32(tp + 4u * rowB);
      if (sa.cls == 1) {
        const long long hi = sh_ld64(hw);
        if (rowB == 0 && hi) tb += ch_add_small<8>(b, -(int)hi);
      }
      if (__any_sync(0xffffffffu, negB)) neg_if8(b, tb, negB);
      Ch<8> out;
      int otop = unal_combine8(out, b, a, tb, o);
      if (L0 == 0) {
        // lane 0's B is lane C-1's A seen through 2^N == -1 (wave_coset.cuh)
        const u32 nbits = 256u - o;
        u32 nz = 0;
#pragma unroll
        for (int xw = 0; xw < 8; ++xw) {
          const u32 lo = 32u * xw;
          const u32 m = lo + 32u <= nbits ? ~0u : (lo < nbits ? (1u << (nbits - lo)) - 1u : 0u);
          nz |= b.w[xw] & m;
        }
        if (nz) otop += ch_add_small<8>(out, 1);
      }
      a = out;
      ta = otop;
    }
    __syncwarp();
    sts_row(rowsA, pos, a);
    sh_st32(tp + 128u + 4u * pos, ta);
  }
  __syncwarp();
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    if (slot_a(wnet, w, j) >= d.nload) {  // truncated input (warp-uniform)
#pragma unroll
      for (int wd = 0; wd < 8; ++wd) x[j].w[wd] = 0;
      tx[j] = 0;
      continue;
    }
    const u32 pre = __shfl_sync(0xffffffffu, ln.pre, (int)j);
    lds_row(x[j], ring + j * 2048u + 1024u, pos);
    const bool inplace = (pre & 0x3FFFFFFFu) == 0;
    tx[j] = (inplace && ((pre >> 30) & 1u)) ? 0 : sh_ld32(rtops + j * 256u + 128u + 4u * pos);
    if (inplace && c == 0) {  // source lane 0 is this item's row 0: fold the top word in
      const long long hi = sh_ld64(sm_s + kTmaHiw + (w * 8u + j) * 16u);
      if (pos == 0 && hi) tx[j] += ch_add_small<8>(x[j], -(int)hi);
    }
  }
  __syncwarp();
}

template <int DUMMY = 0>
__global__ void __launch_bounds__(kTmaThreads, 1)
    coset_tma_kernel(const __grid_constant__ CUtensorMap tm_view, const __grid_constant__ CUtensorMap tm_shadow,
                     WaveArgs A) {
  extern __shared__ std::uint8_t tsm_raw[];
  const u32 sm_s = ((u32)__cvta_generic_to_shared(tsm_raw) + 1023u) & ~1023u;
  const u32 w = threadIdx.x >> 5, lane = threadIdx.x & 31, pos = lane;
  const u32 logS = A.logS, step = 1u << logS;
  const u32 bar = sm_s + kTmaBars + 8u * w;
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  // items: (leaf t, coset g), g fastest (the host guarantees gpl == step)
  const u32 items = A.nleaves << logS;
  const TmaLeafDesc* descs = static_cast<const TmaLeafDesc*>(A.tdesc);
  auto load_desc = [&](u32 item) {
    TmaLeafDesc d{};
    if (item < items) d = descs[item >> logS];
    return d;
  };
  // descriptors two items ahead, lane registers one item ahead
  u32 i1 = blockIdx.x, i2 = i1 + gridDim.x;
  TmaLeafDesc d1 = load_desc(i1), d2 = load_desc(i2);
  TmaLane l1 = tma_lane(A, d1, i1 < items, w, lane);
  if (i1 < items) tma_issue(A, &tm_view, &tm_shadow, d1, i1 & (step - 1), l1, w, lane, sm_s, bar, step);
  const u32 exch = sm_s + kTmaExch, etops = sm_s + kTmaExchTops;
  for (u32 k = 0; i1 < items; ++k) {
    const TmaLeafDesc d = d1;
    const TmaLane ln = l1;
    const u32 c = i1 & (step - 1);
    i1 = i2;
    d1 = d2;
    l1 = tma_lane(A, d1, i1 < items, w, lane);
    i2 += gridDim.x;
    d2 = load_desc(i2);
    const bool dif = (d.nstore_wnet >> 16) == 1;
    mbar_wait(bar, k & 1u);
    Ch<8> x[8];
    int tx[8];
    if (dif)
      tma_item_run<true>(A, d, ln, c, w, pos, sm_s, step, logS, x, tx);
    else
      tma_item_run<false>(A, d, ln, c, w, pos, sm_s, step, logS, x, tx);
    // the buffer is free: the next item's inputs start moving now
    if (i1 < items) tma_issue(A, &tm_view, &tm_shadow, d1, i1 & (step - 1), l1, w, lane, sm_s, bar, step);
    if (dif)
      net8<true, kRotDif>(x, tx, ln.opa, pos);
    else
      net8<false, kRotDit>(x, tx, ln.opa, pos);
    named_bar(1, kTmaThreads);  // every warp is done reading the previous item's exchange tile
#pragma unroll
    for (u32 j = 0; j < 8; ++j) {
      const u32 slot = dif ? w + 8u * j : 8u * w + j;
      sts_row(exch + slot * 1024u, pos, x[j]);
      sh_st32(etops + (slot * 32u + pos) * 4u, tx[j]);
    }
    named_bar(1, kTmaThreads);  // stage A complete
    if (dif)
      stage_b_and_store<true>(A, x, tx, ln, d, c, w, pos, exch, etops, step, logS);
    else
      stage_b_and_store<false>(A, x, tx, ln, d, c, w, pos, exch, etops, step, logS);
  }
}

}  // namespace fermat
}  // namespace cftft_b200
