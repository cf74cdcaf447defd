// wave_wide.cuh -- CTA-level engine for coset leaves of 16..64 coefficients
// (2^lambda, lambda = 4..6), one launch per wave of independent leaves.
//
// Same formats and conventions as the warp kernel (wave_coset.cuh): a leaf's
// rotations are whole multiples of its coset step, so lane p of every output
// depends only on lanes p' == p (mod step) of its inputs; carry-save lanes
// with an int32 top per lane; the coefficient's top word folded into lane 0;
// per-ticket slot tables {pre, post | buffers} (Plan::wave_slots).
//
// One work item = (ticket, group of 2^(6 - lambda) cosets) is owned by the
// whole CTA (8 warps).  Its 2^lambda slots x 32 lanes sit in one shared tile
// [slot][lane] of 256-bit rows; lane l of a row is element lane
// c + step * pos, c = coset (l & cmask), pos = l >> cb.  Warp w loads,
// settles and pre-rotates its own slots, so no CTA barrier separates the
// loads from the first compute stage:
//
//  * full 64-point networks (wnet 1 = DIF, the TFT's; 2 = DIT, the ITFT's;
//    Planner::wide_network): stage A = eight independent 8-point networks
//    (warp w: slots w + 8i (DIF) / 8w + i (DIT)) in registers, rows back to
//    the tile, one __syncthreads, stage B = the eight 8-point networks of
//    the other stride (slots 8w + i / w + 8i), straight from registers to
//    global memory.  Rotations of a butterfly's b by q coset positions are
//    warp shuffles (all positions of a coset sit in one warp row);
//  * any other program (truncated ITFT leaves, 16/32-point leaves): the
//    leaf's micro-ops level by level, ops of a level dealt to the warps,
//    one __syncthreads per level.
//
// Unaligned pre-rotations (deferred sub-lane twiddles) need, for a row's
// first coset, the neighbouring lane of another coset: it is fetched straight
// from global memory into registers (mostly L2 hits: the CTAs running the
// neighbouring cosets of the same leaf read it at the same time).
#pragma once

#include "wave_coset.cuh"

namespace cftft_b200 {
namespace fermat {

constexpr int kWideWarps = 8;

template <int CW>
__host__ __device__ constexpr u32 wide_tile_words() {
  // rows [64][32] x CW words, tops [64][32], top words [64] (u64), slot table [64]
  return 64u * 32u * CW + 64u * 32u + 128u + 64u * (sizeof(WaveSlot) / 4);
}

template <int CW>
__global__ void __launch_bounds__(32 * kWideWarps, 2) coset_wide_kernel(WaveArgs A) {
  static_assert(CW == 8, "the wave engine runs 256-bit lanes");
  extern __shared__ __align__(16) u32 wsm[];
  constexpr u32 CB = 32 * CW;
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  u32* const tile = wsm;
  int* const tops = reinterpret_cast<int*>(wsm + 64u * 32u * CW);
  long long* const hiw = reinterpret_cast<long long*>(wsm + 64u * 32u * CW + 64u * 32u);
  WaveSlot* const si = reinterpret_cast<WaveSlot*>(wsm + 64u * 32u * CW + 64u * 32u + 128u);
  const u32 tile_s = (u32)__cvta_generic_to_shared(tile);
  const u32 CL = A.lanes;
  auto rowp = [&](u32 slot, u32 l) -> u32* { return tile + (slot * 32u + l) * CW; };
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

  const u64 gpl = A.gpl, items = (u64)A.nleaves * gpl;
  // items dealt round-robin over the CTAs: the CTAs running at the same time
  // read neighbouring cosets -- adjacent 32-byte pieces of the same
  // coefficients -- together (DRAM bursts are shared; a contiguous run of
  // items per CTA reads 2.5-4x the bytes from DRAM)
  u32 cur_t = 0xFFFFFFFFu;
  for (u64 item = blockIdx.x; item < items; item += gridDim.x) {
    const u32 t = (u32)(item / gpl), g = (u32)(item - (u64)t * gpl);
    const DevLeaf* lp = A.leaves + t;
    const u64 lbase = lp->base, lstride = lp->stride;
    const u32 lc0 = lp->c0;
    const DevClass cl = A.classes[lp->cls];
    const u32 ell = 31 - __clz(cl.L);
    const u32 nsl = cl.L;               // slots
    const u32 per = nsl >> 3;           // slots per warp
    const u32 cp = 1u << (ell - 1);     // positions per coset
    const u32 cb = 6 - ell;             // coset bits of the lane index
    const u32 cmask = (1u << cb) - 1;
    const u32 step = cl.step;
    const u32 groups = max(1u, step >> cb);
    if (g >= groups) continue;  // (uniform over the CTA)
    const u32 wnet = cl.wnet;
    // slot of the warp's i-th own slot: stage A's slots for the networks
    auto own = [&](u32 i) -> u32 { return wnet == 2 ? warp * per + i : warp + 8u * i; };
    const u32 span = max(cl.nload, cl.nstore);
    __syncthreads();  // the previous item is done with the tile and the slot table
    if (t != cur_t) {
      cur_t = t;
      if (threadIdx.x < span) {
      const u32 k = threadIdx.x;
      const u32 pre = A.wslots[lc0 + 2 * k], post = A.wslots[lc0 + 2 * k + 1];
      const u64 e = lbase + (u64)k * lstride;
      WaveSlot w;
      w.in = (pre >> 31 ? A.data2 : A.data) + e * A.elem_bytes;
      w.tin = A.T + (pre >> 31 ? A.tloc : 0) + e * CL;
      w.out = (post >> 31 ? A.data2 : A.data) + e * A.elem_bytes;
      w.tout = A.T + (post >> 31 ? A.tloc : 0) + e * CL;
      w.pre = pre;
      w.post = post;
      w.pad0 = w.pad1 = 0;
      si[k] = w;
      }
      __syncthreads();
    }

    const u32 c = (g << cb) + (lane & cmask);
    const u32 pos = lane >> cb;
    const bool act = c < step && pos < cp;
    const u32 L0 = c + step * pos;  // this lane's element lane (frame)
    const bool first = (lane & cmask) == 0;

    // ---- load the warp's own slots through their pre-rotations
    u32 wrapA = 0, zeroA = 0, unal = 0;  // bit i: own slot i
    for (u32 i = 0; i < per; ++i) {
      const u32 k = own(i);
      if (k >= cl.nload) continue;  // (warp-uniform)
      const u32 r = si[k].pre & 0x3FFFFFFFu;
      const u32 q = r / CB, o = r % CB;
      if (o) unal |= 1u << i;
      if (!act) continue;
      const u32 srcA = (L0 + 2 * CL - q) & (2 * CL - 1);
      const u32 lnA = srcA & (CL - 1);
      const std::uint8_t* el = si[k].in;
      const u32 so = tile_s + (k * 32u + lane) * CW * 4u, sw = swz(lane);
#pragma unroll
      for (u32 x = 0; x < CW / 4; ++x) cp_async16(so + 16u * (x ^ sw), el + (u64)lnA * (CB / 8) + 16u * x);
      if ((si[k].pre >> 30) & 1u)  // never written: tops are zero
        tops[k * 32u + lane] = 0;
      else
        cp_async4(tile_s + (64u * 32u * CW + k * 32u + lane) * 4u, si[k].tin + wave_tix(A, lnA));
      if (lane == 0) cp_async8(tile_s + (64u * 32u * CW + 64u * 32u) * 4u + 8u * k, el + 4ull * A.D);
      if (lnA == 0) zeroA |= 1u << i;
      if (srcA >= CL) wrapA |= 1u << i;
    }
    // neighbour lanes of unaligned slots for a row's first coset: straight
    // into registers, in batches of kNb own slots (the first batch overlaps
    // the tile loads)
    constexpr u32 kNb = 2;
    Ch<CW> nb[kNb];
    int nbt[kNb];
    u32 nbz = 0, nbw = 0;
    auto fetch_nb = [&](u32 i0) {
#pragma unroll
      for (u32 j = 0; j < kNb; ++j) {
        const u32 i = i0 + j;
        if (i >= per || !((unal >> i) & 1u) || !act || !first || (A.debug & 64)) continue;
        const u32 k = own(i);
        const u32 r = si[k].pre & 0x3FFFFFFFu;
        const u32 q = r / CB;
        const u32 srcA = (L0 + 2 * CL - q) & (2 * CL - 1);
        const u32 srcB = (srcA + 2 * CL - 1) & (2 * CL - 1);
        const u32 lnB = srcB & (CL - 1);
        const uint4* gp = reinterpret_cast<const uint4*>(si[k].in + (u64)lnB * (CB / 8));
#pragma unroll
        for (u32 x = 0; x < CW / 4; ++x) {
          const uint4 v = __ldcg(gp + x);
          nb[j].w[4 * x] = v.x;
          nb[j].w[4 * x + 1] = v.y;
          nb[j].w[4 * x + 2] = v.z;
          nb[j].w[4 * x + 3] = v.w;
        }
        nbt[j] = ((si[k].pre >> 30) & 1u) ? 0 : __ldcg(si[k].tin + wave_tix(A, lnB));
        if (lnB == 0) nbz |= 1u << i;
        if (srcB >= CL) nbw |= 1u << i;
      }
    };
    if (unal) fetch_nb(0);
    cp_async_wait_all();
    __syncwarp();

    const bool tunal = unal != 0;  // (warp-uniform)
    const bool fused = wnet && !tunal;  // stage A reads only the warp's own slots
    // rows -> true carry-save values of their source lanes: the coefficient's
    // top word folded into (every copy of) source lane 0, wrapped lanes negated
    auto settle_regs = [&](Ch<CW>& w, int top, u32 k, bool zero, bool neg) -> int {
      if (zero) {
        const int hi = (int)hiw[k];
        if (hi) top += ch_add_small<CW>(w, -hi);
      }
      if (neg) top = exact_from<CW>(w, top, true);
      return top;
    };
    if (!fused) {
      for (u32 i = 0; i < per; ++i) {
        const u32 k = own(i);
        if (k >= cl.nload || !act) continue;
        const bool zero = (zeroA >> i) & 1u, neg = (wrapA >> i) & 1u;
        if (!zero && !neg) continue;
        Ch<CW> w;
        int top = ld(w, k, lane);
        top = settle_regs(w, top, k, zero, neg);
        st(k, lane, w, top);
      }
      __syncwarp();
    }
    // unaligned slots: lane L0 = bits [CB - o, 2 CB - o) of (B ++ A) plus B's
    // top at bit o, B = the source lane below A (wave_coset.cuh)
    if (tunal) {
      for (u32 i0 = 0; i0 < per; i0 += kNb) {
        if (i0) {
          nbz = nbw = 0;
          fetch_nb(i0);
        }
#pragma unroll
        for (u32 j = 0; j < kNb; ++j) {
          const u32 i = i0 + j;
          if (i >= per || !((unal >> i) & 1u)) continue;  // (warp-uniform)
          const u32 k = own(i);
          const u32 o = (si[k].pre & 0x3FFFFFFFu) % CB;
          Ch<CW> out;
          int otop = 0;
          if (act) {
            Ch<CW> a, b;
            ld(a, k, lane);
            int tb;
            if (first) {
              b = nb[j];
              tb = settle_regs(b, nbt[j], k, (nbz >> i) & 1u, (nbw >> i) & 1u);
            } else {
              tb = ld(b, k, lane - 1);
            }
            otop = unal_combine8(out, b, a, tb, o);
            if (L0 == 0) {
              // lane 0's B is lane C-1's A seen through 2^N == -1 (wave_coset.cuh)
              const u32 nbits = CB - o;
              u32 nz = 0;
#pragma unroll
              for (int x = 0; x < CW; ++x) {
                const u32 lo = 32u * x;
                const u32 m = lo + 32u <= nbits ? ~0u : (lo < nbits ? (1u << (nbits - lo)) - 1u : 0u);
                nz |= b.w[x] & m;
              }
              if (nz) otop += ch_add_small<CW>(out, 1);
            }
          }
          __syncwarp();
          if (act) st(k, lane, out, otop);
          __syncwarp();
        }
      }
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
        // a final output: output lane d takes the top of lane d-1 from the
        // warp lane before it when that lane holds it (wave_coset.cuh)
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
      __stcg(sk->tout + wave_tix(A, d), top);
      const bool owner = k < cl.nload ? ((L0 + 2 * CL - (sk->pre & 0x3FFFFFFFu) / CB) & (CL - 1)) == 0 : d == 0;
      if (owner) __stcg(reinterpret_cast<long long*>(el + 4ull * A.D), 0ll);
    };

    if (wnet) {
      // ---- two stages of 8-point networks in registers
      u32 opv = 0;
      auto bfly = [&](Ch<CW>& a, int& ta, Ch<CW>& b, int& tb, u32 oi) {
        const u32 qv = __shfl_sync(0xffffffffu, opv, (int)oi) >> 16;
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
      // local slot i of stage st (0: the warp's own slots, 1: the other stride)
      auto sl = [&](u32 stg, u32 i) -> u32 {
        const bool strided = (wnet == 1) == (stg == 0);
        return strided ? warp + 8u * i : 8u * warp + i;
      };
      auto ldx = [&](Ch<CW>& x, u32 k, bool firstread) -> int {
        if (firstread && k >= cl.nload) {  // truncated inputs: zero (warp-uniform)
#pragma unroll
          for (int w = 0; w < CW; ++w) x.w[w] = 0;
          return 0;
        }
        int top = ld(x, k, lane);
        if (firstread && fused) {
          const u32 i = wnet == 2 ? k - warp * per : (k - warp) / 8u;
          top = settle_regs(x, top, k, (zeroA >> i) & 1u, (wrapA >> i) & 1u);
        }
        return top;
      };
      // span-4 level (ops o0..o0+3): pairs (j, j+4) through the rows
      auto span4 = [&](u32 stg, u32 o0, bool out, bool firstread) {
#pragma unroll 1
        for (u32 j = 0; j < 4; ++j) {
          Ch<CW> a, b;
          const u32 ka = sl(stg, j), kb = sl(stg, j + 4);
          int ta = ldx(a, ka, firstread), tb = ldx(b, kb, firstread);
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
      // a 4-point half (local slots 4h..4h+3), DIT: spans 1,2; DIF: spans 2,1
      auto half4 = [&](u32 stg, u32 h, bool dit, bool out, bool firstread) {
        Ch<CW> x[4];
        int tx[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) tx[k] = ldx(x[k], sl(stg, 4 * h + k), firstread);
        if (dit) {
          bfly(x[0], tx[0], x[1], tx[1], 2 * h);
          bfly(x[2], tx[2], x[3], tx[3], 2 * h + 1);
          bfly(x[0], tx[0], x[2], tx[2], 4 + 2 * h);
          bfly(x[1], tx[1], x[3], tx[3], 5 + 2 * h);
        } else {
          bfly(x[0], tx[0], x[2], tx[2], 4 + 2 * h);
          bfly(x[1], tx[1], x[3], tx[3], 5 + 2 * h);
          bfly(x[0], tx[0], x[1], tx[1], 8 + 2 * h);
          bfly(x[2], tx[2], x[3], tx[3], 9 + 2 * h);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const u32 sk = sl(stg, 4 * h + k);
          if (out) {
            if (sk < cl.nstore) store_slot(sk, x[k], tx[k]);
          } else {
            st(sk, lane, x[k], tx[k]);
          }
        }
      };
      auto net8 = [&](u32 stg, bool out, bool firstread) {
        opv = lane < 12 ? A.wops[cl.wop_begin + (stg * 8u + warp) * 12u + lane] : 0u;
        if (wnet == 1) {  // DIF: span 4, then the halves
          span4(stg, 0, false, firstread);
          half4(stg, 0, false, out, false);
          half4(stg, 1, false, out, false);
        } else {  // DIT: the halves, then span 4
          half4(stg, 0, true, false, firstread);
          half4(stg, 1, true, false, firstread);
          span4(stg, 8, out, false);
        }
      };
      net8(0, false, true);
      __syncthreads();
      net8(1, true, false);
      continue;
    }

    // ---- generic leaf program: levels of micro-ops, ops dealt to the warps
    __syncthreads();
    for (u32 lv = 0; lv < cl.nlevels; ++lv) {
      const u32 ob = A.levels[cl.level_begin + lv] - cl.op_begin;
      const u32 oe = A.levels[cl.level_begin + lv + 1] - cl.op_begin;
      for (u32 o = ob + warp; o < oe; o += kWideWarps) {
        const u32 wop = A.wops[cl.wop_begin + o];
        const u32 ty = wop & 15u, oa = (wop >> 4) & 63u, ob2 = (wop >> 10) & 63u, qv = wop >> 16;
        Ch<CW> a, b, y0, y1;
        int pa = 0, pb = 0, t0 = 0, t1 = 0;
        if (act) {
          pa = ld(a, oa, lane);
          if (ty == OP_COPY) {
            y1 = a;
            t1 = pa;
          } else {
            const u32 sneg = qv >= cp ? 1u : 0u;
            const u32 qq = qv - (sneg ? cp : 0u);
            const u32 pl = (((pos - qq) & (cp - 1)) << cb) | (lane & cmask);
            const bool neg = ((pos < qq) ? 1u : 0u) != sneg;
            pb = ld(b, ob2, pl);
            ch_pm8(y0, t0, y1, t1, a, pa, b, pb, neg);
            if (ty == OP_SUB2 || ty == OP_SUB2DIFF) t0 = ch_add(y0, a, y1) + pa + t1;
          }
        }
        __syncwarp();
        if (act) {
          if (ty != OP_COPY) st(oa, lane, y0, t0);
          if (ty == OP_ADDSUB || ty == OP_SUB2DIFF || ty == OP_COPY) st(ob2, lane, y1, t1);
        }
        __syncwarp();
      }
      __syncthreads();
    }
    for (u32 i = 0; i < per; ++i) {
      const u32 k = own(i);
      if (k >= cl.nstore) continue;
      Ch<CW> w;
      const int top = act ? ld(w, k, lane) : 0;
      store_slot(k, w, top);
    }
  }
}

}  // namespace fermat
}  // namespace cftft_b200
