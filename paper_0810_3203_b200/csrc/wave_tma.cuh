// wave_tma.cuh -- radix-64 coset passes as a TMA-fed, warp-specialised
// persistent kernel (the engine of radix-64 network waves).
//
// Same plan formats as coset_wide_kernel (wave_wide.cuh): one work item =
// (coset leaf of 64 coefficients, one lane coset c < step); the 64 slots x 32
// positions of the item are lanes c + step * pos of its coefficients (256-bit
// lanes, carry-save with an int32 top per lane); the leaf is a full 64-point
// network (DIF for the TFT, DIT for the ITFT) = two stages of eight 8-point
// register networks (Planner::wide_network).
//
// One 16-warp CTA per SM, two groups of 8 warps, each with its own item tile:
// group g runs stage A then stage B of items k = g (mod 2), so one group's
// stage B overlaps the other's stage A.  Per item, warp w of the group
//  * stage A: waits for its own cp.async loads (its 8 stage-A slots: rows,
//    tops, the element's top word) and the lane-below rows of unaligned slots
//    (TMA bulk copies / tensor boxes into a per-network ring, issued one item
//    ahead), settles each slot in place (pre-rotation by whole cosets = a row
//    index; a sub-lane part = a funnel with the lane below; the top word
//    folded into source lane 0; lanes past 2^N negated), runs its 8-point
//    network in registers and writes the outputs back into its own slots;
//  * stage B (after the group's named barrier): reads its 8 slots re-gauged
//    (a rotation by whole coset positions is a row index and a sign, so only
//    five of the twelve butterflies shuffle: net8_g), releases the tile and
//    starts the loads of the group's next item into it, runs the network and
//    stores straight from registers through the post-rotation (carry-save,
//    coset-major or natural order).
// Tiles and coset-major chunks are stored with the 32-byte swizzle (the
// 16-byte halves of row r swapped when bit 2 of r is set -- the writers' own
// addressing, CU_TENSOR_MAP_SWIZZLE_32B for tensor boxes): a warp's 32 rows
// hit distinct banks.
//
// Shared memory (bytes, 1024-aligned base):
//   tile t (x2)  rows 64 slots x 1 KB | tops 64 x 128 B | top words 64 x 16 B
//   ring rows    8 warps x 8 slots x 1 KB   (stage A: the lane-below cosets)
//   ring tops    8 warps x 8 slots x 128 B
//   store tables 16 warps x 8 descriptors of 32 B
//   mbarriers    ring[2][8]
#pragma once

#include <cuda.h>

#include "wave_coset.cuh"

namespace cftft_b200 {
namespace fermat {

constexpr int kTmaWarpsA = 8;
constexpr int kTmaThreads = 32 * 2 * kTmaWarpsA;
constexpr u32 kTileRows = 0;
constexpr u32 kTileTops = 64u * 1024u;
constexpr u32 kTileHiw = kTileTops + 64u * 128u;
constexpr u32 kTileBytes = kTileHiw + 64u * 16u;  // 74752 (a multiple of 1024)
constexpr u32 kRingRows = 2u * kTileBytes;
constexpr u32 kRingTops = kRingRows + 64u * 1024u;
constexpr u32 kSlotTab = kRingTops + 64u * 128u;  // per warp: 8 store descriptors of 32 B
constexpr u32 kTmaBars = kSlotTab + 128u * 32u;
constexpr u32 kTmaSmem = kTmaBars + 16u * 8u + 1024u;  // + alignment slack
static_assert(kTileBytes % 1024u == 0, "tile alignment");

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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
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

// 32-byte row r of a tile: 16-byte half h at 32 r + 16 (h ^ bit 2 of r)
__device__ __forceinline__ u32 sw_off(u32 r, u32 h) { return 32u * r + 16u * (h ^ ((r >> 2) & 1u)); }
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

__device__ __forceinline__ TmaLeafDesc tma_desc(const WaveArgs& A, u32 item, u32 items) {
  TmaLeafDesc d{};
  if (item < items) d = static_cast<const TmaLeafDesc*>(A.tdesc)[item >> A.logS];
  return d;
}
// source coset of a slot's pre-rotation for item coset g
__device__ __forceinline__ u32 src_coset(u32 pre, u32 g, u32 step) {
  const u32 qb = ((pre & 0x3FFFFFFFu) >> 8) & (step - 1);
  return g >= qb ? g - qb : g + step - qb;
}
__device__ __forceinline__ u32 warp_sum(u32 v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Stage-A warp w: cp.async loads of its own slots of item (d, g) into the
// group's tile -- rows (swizzled), tops, the element's top word where the
// item reads source lane 0 (lane j < 8 holds slot j's pre / layout entry).
// Lanes 4j .. 4j+3 resolve slot j: for natural-layout rows lane 4j + 2b + h
// copies the 16-byte half h of rows 2i + b (i < 16), so one instruction moves
// whole 32-byte sectors (two lanes per row); coset-major chunks are copied by
// the whole warp, 512 contiguous bytes per instruction.
template <bool DIF>
__device__ __forceinline__ void warp_load(const WaveArgs& A, const TmaLeafDesc& d, u32 g, u32 w, u32 lane, u32 apre,
                                           u32 alay, u32 tile, u32 step) {
  const u32 j = lane >> 2, qd = lane & 3u, b = qd >> 1, h = qd & 1u;
  const u32 pre = __shfl_sync(0xffffffffu, apre, (int)j), lay = __shfl_sync(0xffffffffu, alay, (int)j);
  const u32 slot = slot_a(DIF ? 1u : 2u, w, j);
  u64 chunk = 0;  // coset-major slots: the source chunk (copied by the whole warp below)
  if (slot < d.nload) {
    const u32 r = pre & 0x3FFFFFFFu;
    const u32 cA = src_coset(pre, g, step);
    const bool unal = (r & 255u) != 0, fresh = (pre >> 30) & 1u, sh = pre >> 31;
    const u64 e = d.base + (u64)slot * d.stride;
    const std::uint8_t* el = (sh ? A.data2 : A.data) + e * A.elem_bytes;
    if (lay & 1u) {
      chunk = reinterpret_cast<u64>(el + (u64)cA * 1024u);
    } else {
      const u32 dst = tile + kTileRows + slot * 1024u + 32u * b;
      const std::uint8_t* src = el + 32ull * cA + (u64)(32u * step) * b + 16u * h;
      const u64 inc = 64ull * step;
      const u32 d0 = dst + 16u * h, d1 = dst + 16u * (h ^ 1u);
#pragma unroll
      for (u32 i = 0; i < 16; ++i) {
        cp_async16_l2(((i >> 1) & 1u ? d1 : d0) + 64u * i, src);
        src += inc;
      }
    }
    if (!fresh) {
      const int* tr = A.T + (sh ? A.tloc : 0) + e * A.lanes + cA * 32u + 8u * qd;
      const u32 td = tile + kTileTops + slot * 128u + 32u * qd;
      cp_async16(td, tr);
      cp_async16(td + 16u, tr + 4);
    }
    if (qd == 0 && (cA == 0 || (unal && cA == 1))) cp_async8(tile + kTileHiw + slot * 16u, el + 4ull * A.D);
  }
  // coset-major chunks are stored swizzled: a linear copy, 512 contiguous
  // bytes per instruction
  const u32 cm = __ballot_sync(0xffffffffu, chunk != 0);
  if (cm) {
#pragma unroll
    for (u32 k = 0; k < 8; ++k) {
      const u64 cp = __shfl_sync(0xffffffffu, chunk, (int)(4u * k));
      if (!cp) continue;  // (warp-uniform)
      const u32 dst = tile + kTileRows + slot_a(DIF ? 1u : 2u, w, k) * 1024u + 16u * lane;
      const std::uint8_t* src = reinterpret_cast<const std::uint8_t*>(cp) + 16u * lane;
      cp_async16(dst, src);
      cp_async16(dst + 512u, src + 512u);
    }
  }
  cp_async_commit();
}

// Stage-A warp w: the lane-below rows of its unaligned slots of item (d, g)
// into the warp's ring (lane j < 8: slot j of the warp's network).
template <bool DIF>
__device__ __forceinline__ void ring_issue(const WaveArgs& A, const CUtensorMap* tmv, const CUtensorMap* tms,
                                           const TmaLeafDesc& d, u32 g, bool valid, u32 w, u32 lane, u32 pre,
                                           u32 lay, u32 sm_s, u32 bar, u32 step) {
  const u32 slot = slot_a(DIF ? 1u : 2u, w, lane & 7u);
  const u32 r = pre & 0x3FFFFFFFu;
  const bool ld = valid && lane < 8 && slot < d.nload && (r & 255u) != 0;
  const bool fresh = (pre >> 30) & 1u;
  const u32 tot = warp_sum(ld ? 1024u + (fresh ? 0u : 128u) : 0u);
  if (lane == 0) mbar_expect_tx(bar, tot);
  __syncwarp();
  if (ld) {
    const u32 cA = src_coset(pre, g, step);
    const u32 cB = cA ? cA - 1 : step - 1;
    const bool sh = pre >> 31;
    const u64 e = d.base + (u64)slot * d.stride;
    const std::uint8_t* el = (sh ? A.data2 : A.data) + e * A.elem_bytes;
    const u32 dst = sm_s + kRingRows + (w * 8u + lane) * 1024u;
    if (lay & 1u)
      bulk_g2s(dst, el + (u64)cB * 1024u, 1024u, bar);
    else
      tma_box(dst, sh ? tms : tmv, cB, (u32)e, bar);
    if (!fresh)
      bulk_g2s(sm_s + kRingTops + (w * 8u + lane) * 128u, A.T + (sh ? A.tloc : 0) + e * A.lanes + (u64)cB * 32u,
               128u, bar);
  }
}

// Settle one slot in place: row pos of the slot becomes the true carry-save
// value of this lane's rotated source lane (x = lane L0 - r, r = q lanes + o
// bits), the element's top word folded into source lane 0, lanes past 2^N
// negated; its top goes to tops[pos].  A sub-lane rotation takes the low
// 256 - o bits of source lane A = L0 - q shifted up and the high o bits (and
// the top) of the lane below it, B; each part carries the sign its source
// lane has as seen from this lane, applied after the split -- so the lane
// that reads X as A and the lane that reads X as B always split X the same
// way, and across 2^N == -1 (output lane 0 taking lane C-1's high bits) the
// parts are exact negatives.
template <bool FAST>
__device__ __forceinline__ void settle_slot(u32 pre, u32 c, u32 pos, u32 rows, u32 tops, u32 hiw, u32 brows,
                                            u32 btops, u32 logS) {
  const u32 r = pre & 0x3FFFFFFFu;
  const bool fresh = (pre >> 30) & 1u;
  Ch<8> x;
  int t;
  if (FAST && r < 256u && c >= 2) {
    // the common case of the TFT's unaligned waves (warp-uniform; FAST: the
    // kernel instance those waves run): no whole-lane rotation and no lane-0
    // neighbourhood -- source lane = this lane, the lane below it = the
    // ring's row of the same position, no signs, no top word
    Ch<8> b;
    lds_row(x, rows, pos);
    lds_row(b, brows, pos);
    const int tb = fresh ? 0 : sh_ld32(btops + 4u * pos);
    Ch<8> out;
    t = unal_combine8(out, b, x, tb, r);
    sts_row(rows, pos, out);
    sh_st32(tops + 4u * pos, t);
    return;
  }
  if (r == 0) {  // c == 0: only the top word of row 0 to fold
    lds_row(x, rows, pos);
    t = fresh ? 0 : sh_ld32(tops + 4u * pos);
    const long long hi = sh_ld64(hiw);
    if (pos == 0 && hi) t += ch_add_small<8>(x, -(int)hi);
  } else {
    const u32 o = r & 255u;
    const PreSrc sa = pre_src(c, pos, r >> 8, logS);
    lds_row(x, rows, sa.row);
    t = fresh ? 0 : sh_ld32(tops + 4u * sa.row);
    if (sa.cls == 0) {  // warp-uniform
      const long long hi = sh_ld64(hiw);
      if (sa.row == 0 && hi) t += ch_add_small<8>(x, -(int)hi);
    }
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
      lds_row(b, brows, rowB);
      int tb = fresh ? 0 : sh_ld32(btops + 4u * rowB);
      if (sa.cls == 1) {
        const long long hi = sh_ld64(hiw);
        if (rowB == 0 && hi) tb += ch_add_small<8>(b, -(int)hi);
      }
      // signs differ only where the source index wraps between B and A
      const bool mixed = negB != sa.neg;
      const bool anym = __any_sync(0xffffffffu, mixed);
      Ch<8> out;
      if (anym) {
        Ch<8> bs;
#pragma unroll
        for (int k = 0; k < 8; ++k) bs.w[k] = mixed ? 0u : b.w[k];
        t = unal_combine8(out, bs, x, mixed ? 0 : tb, o);  // the whole lane, or low(A) where mixed
      } else {
        t = unal_combine8(out, b, x, tb, o);
      }
      if (__any_sync(0xffffffffu, sa.neg)) neg_if8(out, t, sa.neg);
      if (anym) {
        Ch<8> z, h;
#pragma unroll
        for (int k = 0; k < 8; ++k) z.w[k] = 0;
        int th = unal_combine8(h, b, z, tb, o);  // high(B)
        if (__any_sync(0xffffffffu, negB)) neg_if8(h, th, negB);
        if (mixed) t += th + ch_add<8>(out, out, h);
      }
      x = out;
    } else if (__any_sync(0xffffffffu, sa.neg)) {
      neg_if8(x, t, sa.neg);
    }
  }
  __syncwarp();  // every lane has read the slot's rows
  sts_row(rows, pos, x);
  sh_st32(tops + 4u * pos, t);
}

// ---- stage B with re-gauged inputs.  A rotation of a whole slot by g coset
// positions is a row index (and a per-lane sign) when the slot is read from
// the tile, so stage B reads slot j as x^{g_j} * slot j with the g_j chosen
// (Planner::wide_network, bits 4..9 of op j < 8) such that seven of the twelve
// butterflies need no rotation at all; the other five (the ops of kRotDif /
// kRotDit) keep a residual rotation (bits 10..15).  Signs are carried per slot
// (sg bit j: this lane's row of slot j is held negated) and folded into the
// butterflies' +- (ch_pm8): both outputs of a butterfly take a's gauge and
// sign, every chain ends in slot 0 (g_0 = 0), so the outputs are the plain
// network's.
template <bool DIF>
__device__ __forceinline__ void stage_b_load_g(Ch<8> (&x)[8], int (&tx)[8], u32& sg, u32 wb, u32 pos, u32 opb,
                                               u32 tile) {
  const u32 wnet = DIF ? 1u : 2u;
  sg = 0;
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_b(wnet, wb, j);
    const u32 g = (__shfl_sync(0xffffffffu, opb, (int)j) >> 4) & 63u;
    const u32 gq = g & 31u, row = (pos - gq) & 31u;
    sg |= (u32)((pos < gq) != (g >= 32u)) << j;
    lds_row(x[j], tile + kTileRows + slot * 1024u, row);
    tx[j] = sh_ld32(tile + kTileTops + slot * 128u + 4u * row);
  }
}
template <u32 MASK, int J, int IA, int IB>
__device__ __forceinline__ void bfly_g(Ch<8> (&x)[8], int (&t)[8], u32& sg, u32 opv, u32 pos) {
  Ch<8> y0, y1;
  int t0, t1;
  if constexpr ((MASK >> J) & 1u) {
    const u32 qv = (__shfl_sync(0xffffffffu, opv, J) >> 10) & 63u;
    const u32 qq = qv & 31u;
    const u32 pl = (pos - qq) & 31u;
    Ch<8> bp;
#pragma unroll
    for (int wd = 0; wd < 8; ++wd) bp.w[wd] = __shfl_sync(0xffffffffu, x[IB].w[wd], (int)pl);
    const int tbp = __shfl_sync(0xffffffffu, t[IB], (int)pl);
    const u32 sb = __shfl_sync(0xffffffffu, sg, (int)pl) >> IB;
    const bool neg = (((sg >> IA) ^ sb) & 1u) != (u32)((pos < qq) != (qv >= 32u));
    ch_pm8(y0, t0, y1, t1, x[IA], t[IA], bp, tbp, neg);
  } else {
    const bool neg = ((sg >> IA) ^ (sg >> IB)) & 1u;
    ch_pm8(y0, t0, y1, t1, x[IA], t[IA], x[IB], t[IB], neg);
  }
  x[IA] = y0;
  t[IA] = t0;
  x[IB] = y1;
  t[IB] = t1;
  sg = (sg & ~(1u << IB)) | (((sg >> IA) & 1u) << IB);
}
template <bool DIF>
__device__ __forceinline__ void net8_g(Ch<8> (&x)[8], int (&t)[8], u32& sg, u32 opv, u32 pos) {
  if constexpr (DIF) {
    bfly_g<kRotDif, 0, 0, 4>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 1, 1, 5>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 2, 2, 6>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 3, 3, 7>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 4, 0, 2>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 5, 1, 3>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 6, 4, 6>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 7, 5, 7>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 8, 0, 1>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 9, 2, 3>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 10, 4, 5>(x, t, sg, opv, pos);
    bfly_g<kRotDif, 11, 6, 7>(x, t, sg, opv, pos);
  } else {
    bfly_g<kRotDit, 0, 0, 1>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 1, 2, 3>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 2, 4, 5>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 3, 6, 7>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 4, 0, 2>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 5, 1, 3>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 6, 4, 6>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 7, 5, 7>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 8, 0, 4>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 9, 1, 5>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 10, 2, 6>(x, t, sg, opv, pos);
    bfly_g<kRotDit, 11, 3, 7>(x, t, sg, opv, pos);
  }
}

// stage A of one item for warp w (tile `tile`): settle in place, load,
// network, write back
template <bool DIF, bool FAST, class Settled>
__device__ __forceinline__ void stage_a(const TmaLeafDesc& d, u32 c, u32 w, u32 pos, u32 apre, u32 opa, u32 tile,
                                        u32 sm_s, u32 logS, Settled settled) {
  const u32 wnet = DIF ? 1u : 2u;
  u32 tvalid = 0;  // bit j: the slot's tops row is valid
#pragma unroll 1
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_a(wnet, w, j);
    if (slot >= d.nload) break;  // (warp-uniform; later slots are truncated too)
    const u32 pre = __shfl_sync(0xffffffffu, apre, (int)j);
    if ((pre & 0x3FFFFFFFu) == 0 && c != 0) {  // read in place
      if (!((pre >> 30) & 1u)) tvalid |= 1u << j;
      continue;
    }
    settle_slot<FAST>(pre, c, pos, tile + kTileRows + slot * 1024u, tile + kTileTops + slot * 128u,
                tile + kTileHiw + slot * 16u, sm_s + kRingRows + (w * 8u + j) * 1024u,
                sm_s + kRingTops + (w * 8u + j) * 128u, logS);
    tvalid |= 1u << j;
  }
  __syncwarp();
  settled();  // the warp's ring is free
  Ch<8> x[8];
  int tx[8];
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_a(wnet, w, j);
    if (slot >= d.nload) {  // truncated input (warp-uniform)
#pragma unroll
      for (int wd = 0; wd < 8; ++wd) x[j].w[wd] = 0;
      tx[j] = 0;
      continue;
    }
    lds_row(x[j], tile + kTileRows + slot * 1024u, pos);
    tx[j] = ((tvalid >> j) & 1u) ? sh_ld32(tile + kTileTops + slot * 128u + 4u * pos) : 0;
  }
  if (DIF)
    net8<true, kRotDif>(x, tx, opa, pos);
  else
    net8<false, kRotDit>(x, tx, opa, pos);
  __syncwarp();  // every lane is done reading the warp's slots
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_a(wnet, w, j);
    sts_row(tile + kTileRows + slot * 1024u, pos, x[j]);
    sh_st32(tile + kTileTops + slot * 128u + 4u * pos, tx[j]);
  }
}

// Store descriptor of one output slot (stage-B warp table in shared memory)
struct SlotOut {
  u64 el;    // output element base (buffer resolved)
  u64 tout;  // its tops row
  u32 post;  // post-rotation in lanes
  u32 lown;  // the lane (L0) that clears the output's top word
  u32 flags; // bit 0: stored (slot < nstore), bit 1: coset-major output
  u32 pad;
};
static_assert(sizeof(SlotOut) == 32, "SlotOut layout");

template <bool DIF>
__device__ __forceinline__ void slot_table(const WaveArgs& A, const TmaLeafDesc& d, u32 wb, u32 lane, u32 tab) {
  if (lane < 8) {
    const u32 slot = slot_b(DIF ? 1u : 2u, wb, lane);
    SlotOut so{};
    if (slot < (d.nstore_wnet & 0xFFFFu)) {
      const u32 post = __ldg(A.wslots + d.c0 + 2 * slot + 1);
      const u32 CL = A.lanes;
      const u64 e = d.base + (u64)slot * d.stride;
      const bool osh = post >> 31;
      so.el = reinterpret_cast<u64>((osh ? A.data2 : A.data) + e * A.elem_bytes);
      so.tout = reinterpret_cast<u64>(A.T + (osh ? A.tloc : 0) + e * CL);
      so.post = post & 0x3FFFFFFFu;
      so.flags = 1u | (((u32)__ldg(A.tlay + d.c0 + 2 * slot) & 2u));
      if (slot < d.nload) {  // the lane that read source lane 0 (L0 == q mod C)
        const u32 q = (__ldg(A.wslots + d.c0 + 2 * slot) & 0x3FFFFFFFu) >> 8;
        so.lown = q & (CL - 1);
      } else {  // the lane writing output lane 0
        so.lown = (CL - (so.post & (CL - 1))) & (CL - 1);
      }
    }
    uint4* p = reinterpret_cast<uint4*>(__cvta_shared_to_generic(tab + 32u * lane));
    const uint4* sp = reinterpret_cast<const uint4*>(&so);
    p[0] = sp[0];
    p[1] = sp[1];
  }
}

template <bool DIF>
__device__ __forceinline__ void stage_b_load(Ch<8> (&x)[8], int (&tx)[8], u32 wb, u32 pos, u32 tile) {
  const u32 wnet = DIF ? 1u : 2u;
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_b(wnet, wb, j);
    lds_row(x[j], tile + kTileRows + slot * 1024u, pos);
    tx[j] = sh_ld32(tile + kTileTops + slot * 128u + 4u * pos);
  }
}
// store the 8 slots of a stage-B warp through its slot table (post-rotation,
// carry-save, coset-major or natural order)
__device__ __forceinline__ void stage_b_store(const WaveArgs& A, Ch<8> (&x)[8], int (&tx)[8], u32 c, u32 pos, u32 tab,
                                              u32 logS) {
  const u32 CL = A.lanes, L0 = c + (pos << logS), step = 1u << logS;
  const u32 tsh = A.logLanes - logS;
#pragma unroll
  for (u32 j = 0; j < 8; ++j) {
    const SlotOut* so = reinterpret_cast<const SlotOut*>(__cvta_shared_to_generic(tab + 32u * j));
    const uint4 h1 = reinterpret_cast<const uint4*>(so)[1];  // post, lown, flags, pad
    if (!(h1.z & 1u)) continue;  // slot >= nstore (warp-uniform)
    const uint4 h0 = reinterpret_cast<const uint4*>(so)[0];
    std::uint8_t* el = reinterpret_cast<std::uint8_t*>(((u64)h0.y << 32) | h0.x);
    int* tout = reinterpret_cast<int*>(((u64)h0.w << 32) | h0.z);
    const u32 dst = (L0 + h1.x) & (2 * CL - 1);
    const u32 dl = dst & (CL - 1);
    const bool ng = dst >= CL;
    if (__any_sync(0xffffffffu, ng)) neg_if8(x[j], tx[j], ng);
    const u32 cs = dl & (step - 1), rw = dl >> logS;
    if (h1.z & 2u) {  // coset-major, swizzled: chunk cs, row rw
      uint4* gp = reinterpret_cast<uint4*>(el + (cs << 10) + 32u * rw);
      const u32 sw = (rw >> 2) & 1u;
      __stcg(gp + sw, make_uint4(x[j].w[0], x[j].w[1], x[j].w[2], x[j].w[3]));
      __stcg(gp + (sw ^ 1u), make_uint4(x[j].w[4], x[j].w[5], x[j].w[6], x[j].w[7]));
    } else {
      uint4* gp = reinterpret_cast<uint4*>(el + 32u * dl);
      __stcg(gp, make_uint4(x[j].w[0], x[j].w[1], x[j].w[2], x[j].w[3]));
      __stcg(gp + 1, make_uint4(x[j].w[4], x[j].w[5], x[j].w[6], x[j].w[7]));
    }
    __stcg(tout + ((cs << tsh) | rw), tx[j]);
    if (L0 == h1.y) __stcg(reinterpret_cast<long long*>(el + 4ull * A.D), 0ll);
  }
}
// ---- phase programs (Planner::tma_program): 64-slot classes that are not
// full networks, e.g. the truncated ITFT leaves.  Stage A only settles the
// warp's slots in the tile; then every phase runs its ops on the tile, warp w
// the ops of its row / column (disjoint slots), a group barrier between
// phases; stage B stores from the tile.

// stage A of a program item: settle warp w's slots in place; the tops rows of
// slots read in place that were never written are zeroed
template <bool DIF>
__device__ __forceinline__ void stage_a_settle(const TmaLeafDesc& d, u32 c, u32 w, u32 pos, u32 apre, u32 tile,
                                               u32 sm_s, u32 logS) {
  const u32 wnet = DIF ? 1u : 2u;
#pragma unroll 1
  for (u32 j = 0; j < 8; ++j) {
    const u32 slot = slot_a(wnet, w, j);
    if (slot >= d.nload) break;
    const u32 pre = __shfl_sync(0xffffffffu, apre, (int)j);
    if ((pre & 0x3FFFFFFFu) == 0 && c != 0) {
      if ((pre >> 30) & 1u) sh_st32(tile + kTileTops + slot * 128u + 4u * pos, 0);
      continue;
    }
    settle_slot<false>(pre, c, pos, tile + kTileRows + slot * 1024u, tile + kTileTops + slot * 128u,
                tile + kTileHiw + slot * 16u, sm_s + kRingRows + (w * 8u + j) * 1024u,
                sm_s + kRingTops + (w * 8u + j) * 128u, logS);
  }
}

// warp w's ops of one phase: micro-ops on the tile's rows (a butterfly's b is
// row b read at position pos - q, negated across 2^N == -1).  An ADDSUB
// flagged as paired (bit 22) runs together with the next op, also an ADDSUB
// on other slots: two independent carry chains in flight.
__device__ __forceinline__ void prog_addsub_load(u32 wop, u32 tile, u32 pos, Ch<8>& x, int& ta, Ch<8>& yb, int& tb,
                                                 bool& neg) {
  const u32 a = (wop >> 4) & 63u, b = (wop >> 10) & 63u, q = (wop >> 16) & 63u;
  const u32 qq = q & 31u, pl = (pos - qq) & 31u;
  neg = (pos < qq) != (q >= 32u);
  lds_row(x, tile + kTileRows + a * 1024u, pos);
  ta = sh_ld32(tile + kTileTops + a * 128u + 4u * pos);
  lds_row(yb, tile + kTileRows + b * 1024u, pl);
  tb = sh_ld32(tile + kTileTops + b * 128u + 4u * pl);
}
__device__ __forceinline__ void prog_addsub_store(u32 wop, u32 tile, u32 pos, const Ch<8>& y0, int t0,
                                                  const Ch<8>& y1, int t1) {
  const u32 a = (wop >> 4) & 63u, b = (wop >> 10) & 63u;
  sts_row(tile + kTileRows + a * 1024u, pos, y0);
  sh_st32(tile + kTileTops + a * 128u + 4u * pos, t0);
  sts_row(tile + kTileRows + b * 1024u, pos, y1);
  sh_st32(tile + kTileTops + b * 128u + 4u * pos, t1);
}
__device__ __forceinline__ void prog_ops(const u32* prog, u32 desc, u32 lane, u32 tile) {
  const u32 first = desc >> 16, count = desc & 0xFFFFu;
  const u32 pos = lane;
#pragma unroll 1
  for (u32 o0 = 0; o0 < count; o0 += 32) {
    const u32 opv = o0 + lane < count ? __ldg(prog + first + o0 + lane) : 0u;
    const u32 m = count - o0 < 32u ? count - o0 : 32u;
#pragma unroll 1
    for (u32 o = 0; o < m; ++o) {
      const u32 wop = __shfl_sync(0xffffffffu, opv, (int)o);
      if (wop & (1u << 22)) {  // a pair of ADDSUBs or of ADDs (warp-uniform)
        const u32 wop2 = __shfl_sync(0xffffffffu, opv, (int)o + 1);
        Ch<8> x0, b0, x1, b1, y0, y1, z0, z1;
        int ta0, tb0, ta1, tb1, s0, s1, r0, r1;
        bool n0, n1;
        prog_addsub_load(wop, tile, pos, x0, ta0, b0, tb0, n0);
        prog_addsub_load(wop2, tile, pos, x1, ta1, b1, tb1, n1);
        ch_pm8(y0, s0, y1, s1, x0, ta0, b0, tb0, n0);
        ch_pm8(z0, r0, z1, r1, x1, ta1, b1, tb1, n1);
        __syncwarp();
        if ((wop & 15u) == OP_ADDSUB) {
          prog_addsub_store(wop, tile, pos, y0, s0, y1, s1);
          prog_addsub_store(wop2, tile, pos, z0, r0, z1, r1);
        } else {  // ADD: a only
          const u32 a0 = (wop >> 4) & 63u, a1 = (wop2 >> 4) & 63u;
          sts_row(tile + kTileRows + a0 * 1024u, pos, y0);
          sh_st32(tile + kTileTops + a0 * 128u + 4u * pos, s0);
          sts_row(tile + kTileRows + a1 * 1024u, pos, z0);
          sh_st32(tile + kTileTops + a1 * 128u + 4u * pos, r0);
        }
        __syncwarp();
        ++o;
        continue;
      }
      const u32 type = wop & 15u, a = (wop >> 4) & 63u, b = (wop >> 10) & 63u, q = (wop >> 16) & 63u;
      const u32 ra = tile + kTileRows + a * 1024u, rb = tile + kTileRows + b * 1024u;
      Ch<8> x, y0, y1;
      const int ta = sh_ld32(tile + kTileTops + a * 128u + 4u * pos);
      lds_row(x, ra, pos);
      int t0 = 0, t1 = ta;
      if (type == OP_COPY) {
        y1 = x;
      } else {
        const u32 qq = q & 31u;
        const u32 pl = (pos - qq) & 31u;
        const bool neg = (pos < qq) != (q >= 32u);
        Ch<8> yb;
        lds_row(yb, rb, pl);
        const int tb = sh_ld32(tile + kTileTops + b * 128u + 4u * pl);
        ch_pm8(y0, t0, y1, t1, x, ta, yb, tb, neg);
        if (type == OP_SUB2 || type == OP_SUB2DIFF) t0 = ch_add<8>(y0, x, y1) + ta + t1;
      }
      __syncwarp();
      if (type != OP_COPY) {
        sts_row(ra, pos, y0);
        sh_st32(tile + kTileTops + a * 128u + 4u * pos, t0);
      }
      if (type == OP_ADDSUB || type == OP_SUB2DIFF || type == OP_COPY) {
        sts_row(rb, pos, y1);
        sh_st32(tile + kTileTops + b * 128u + 4u * pos, t1);
      }
      __syncwarp();
    }
  }
}

// PROG: the wave has phase-program items (a separate instance, so the
// network-only kernels keep their register allocation)
// UNAL: the instance of the TFT's network waves with sub-lane pre-rotations
// (settle_slot's fast path)
template <bool DIF, bool PROG, bool UNAL = false>
__global__ void __launch_bounds__(kTmaThreads, 1)
    coset_tma_kernel(const __grid_constant__ CUtensorMap tm_view, const __grid_constant__ CUtensorMap tm_shadow,
                     WaveArgs A) {
  extern __shared__ std::uint8_t tsm_raw[];
  const u32 sm_s = ((u32)__cvta_generic_to_shared(tsm_raw) + 1023u) & ~1023u;
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31, pos = lane;
  const u32 grp = warp >> 3, w = warp & 7u;
  const u32 logS = A.logS, step = 1u << logS;
  // mbarriers ring[g][w]: network w's lane-below rows for group g's items
  const u32 bar0 = sm_s + kTmaBars;
  auto ringbar = [&](u32 g) { return bar0 + 64u * g + 8u * w; };
  if (threadIdx.x == 0) {
    for (int b = 0; b < 16; ++b) mbar_init(bar0 + 8u * b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const u32 items = A.nleaves << logS, G = gridDim.x;
  // Runs of 2^runlog consecutive items (cosets of one leaf) per CTA and
  // round: the lane-below rows of an item are the rows its neighbour item
  // loads, so with runs they are in L2 (the host picks the run per wave).
  const u32 runlog = A.runlog, runmask = (1u << runlog) - 1u;
  auto item_of = [&](u32 k) { return (blockIdx.x << runlog) + (k & runmask) + (k >> runlog) * (G << runlog); };
  const u32 tile = sm_s + grp * kTileBytes;
  const u32 tab = sm_s + kSlotTab + 256u * warp;
  // lane j < 8: slot j of this warp's stage-A network (pre, layout)
  auto lane_info = [&](const TmaLeafDesc& d, bool valid, u32& pre, u32& lay) {
    pre = lay = 0;
    const u32 slot = slot_a(DIF ? 1u : 2u, w, lane & 7u);
    if (valid && lane < 8 && slot < d.nload) {
      pre = __ldg(A.wslots + d.c0 + 2 * slot);
      lay = __ldg(A.tlay + d.c0 + 2 * slot);
    }
  };
  // Group g runs stage A then stage B of items k = g, g + 2, ...: while one
  // group is in stage B of item k the other settles and transforms item k+1.
  // Each warp loads its own stage-A slots (cp.async) as soon as the group's
  // tile is free; the lane-below rings are shared: the group that finishes
  // settling item k starts the rows of item k+1 (the other group's) into them.
  u32 i = item_of(grp);
  TmaLeafDesc d = tma_desc(A, i, items);
  u32 pre, lay;
  lane_info(d, i < items, pre, lay);
  if (i < items) warp_load<DIF>(A, d, i & (step - 1), w, lane, pre, lay, tile, step);
  if (grp == 0)
    ring_issue<DIF>(A, &tm_view, &tm_shadow, d, i & (step - 1), i < items, w, lane, pre, lay, sm_s, ringbar(0),
                    step);
  u32 n = 0;  // this group's item count
  for (u32 k = grp; i < items; k += 2, ++n) {
    const u32 c = i & (step - 1);
    const u32 in = item_of(k + 1);
    const TmaLeafDesc dn = tma_desc(A, in, items);
    u32 npre, nlay;
    lane_info(dn, in < items, npre, nlay);
    const u32 i2 = item_of(k + 2);
    const TmaLeafDesc d2 = tma_desc(A, i2, items);
    u32 pre2, lay2;
    lane_info(d2, i2 < items, pre2, lay2);
    // group-uniform: a phase program (wnet 3) instead of the two networks
    const bool prog = PROG && (d.nstore_wnet >> 16) == 3u;
    const u32 opa = !prog && lane < 12 ? __ldg(A.wops + d.wop_begin + w * 12u + lane) : 0u;
    const u32 opb = !prog && lane < 12 ? __ldg(A.wops + d.wop_begin + (8u + w) * 12u + lane) : 0u;
    // (the store table first: off the path between stage A and stage B, and
    // it overlaps the wait for the loads)
    slot_table<DIF>(A, d, w, lane, tab);
    // ---- stage A
    cp_async_wait<0>();
    __syncwarp();
    mbar_wait(ringbar(grp), n & 1u);
    // program items: word 0 = phases | network rows << 8 (the DIT kernel runs
    // phase 0 of those rows as stage-A networks in registers)
    const u32 phdr = prog ? __ldg(A.wops + d.wop_begin) : 0u;
    const bool pnet = prog && !DIF && ((phdr >> (8 + w)) & 1u);
    // As soon as the warp has settled its slots its ring is free: the next
    // item's lane-below rows (the other group's) start moving, and that
    // group's stage A may begin -- this hand-off also keeps the two groups
    // half an item apart.
    auto ring_next = [&]() {
      ring_issue<DIF>(A, &tm_view, &tm_shadow, dn, in & (step - 1), in < items, w, lane, npre, nlay, sm_s,
                      ringbar(grp ^ 1u), step);
    };
    if (pnet) {
      const u32 opn = lane < 12 ? __ldg(A.wops + d.wop_begin + 1 + 8 * (phdr & 0xFFu) + 12 * w + lane) : 0u;
      stage_a<DIF, false>(d, c, w, pos, pre, opn, tile, sm_s, logS, ring_next);
    } else if (prog) {
      stage_a_settle<DIF>(d, c, w, pos, pre, tile, sm_s, logS);
      ring_next();
    } else if (A.debug & 256u) {
      ring_next();
    } else {
      stage_a<DIF, UNAL>(d, c, w, pos, pre, opa, tile, sm_s, logS, ring_next);
    }
    named_bar(1u + grp, 256u);  // the group's stage-A outputs are in the tile
    if (prog) {
      const u32* pg = A.wops + d.wop_begin;
      const u32 P = phdr & 0xFFu;
#pragma unroll 1
      for (u32 p = 0; p < P; ++p) {
        if ((p || !pnet) && !((A.debug & 1024u) && p >= 2)) prog_ops(pg, __ldg(pg + 1 + 8 * p + w), lane, tile);
        named_bar(1u + grp, 256u);
      }
    }
    // ---- stage B
    Ch<8> x[8];
    int tx[8];
    u32 sg = 0;
    if (prog)
      stage_b_load<DIF>(x, tx, w, pos, tile);
    else
      stage_b_load_g<DIF>(x, tx, sg, w, pos, opb, tile);
    named_bar(1u + grp, 256u);  // every warp of the group holds its rows: the tile is free
    if (i2 < items) warp_load<DIF>(A, d2, i2 & (step - 1), w, lane, pre2, lay2, tile, step);
    if (prog)
      stage_b_store(A, x, tx, c, pos, tab, logS);
    else if (!(A.debug & 512u)) {
      net8_g<DIF>(x, tx, sg, opb, pos);
      stage_b_store(A, x, tx, c, pos, tab, logS);
    }
    __syncwarp();  // the slot table is rewritten for the next item
    i = i2;
    d = d2;
    pre = pre2;
  }
}

}  // namespace fermat
}  // namespace cftft_b200
