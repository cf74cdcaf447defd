// planner.hpp -- host-side schedule builder for the GPU TFT/ITFT.
//
// The reference runs Algorithms 1 and 2 as a recursion over strided views
// (transform.hpp:154-239).  On the GPU the recursion is cut at "leaves":
// sub-transforms small enough that all their coefficients sit in one CTA's
// shared memory.  The planner
//   (1) replays the reference recursion above the leaves -- the reference's
//       own split at the top level, an SMEM-sized near-balanced split below
//       it (outputs are unique, so any inner split gives the same bits;
//       transform_test.cpp:248-272) -- and records, for every leaf, the one
//       (node, phase) completion counter it must wait for and the counters
//       it completes: within a node all columns finish before any row starts
//       (TFT), and the ITFT's phases i..iv run in order (transform.hpp:215-238);
//   (2) replays the reference recursion INSIDE a leaf with zeta = 1, turning
//       every base case (transform.hpp:94-150) into a micro-op on SMEM slots.
//       Multiplications by powers of omega are never executed eagerly: each
//       slot carries a pending exponent P (true value = omega^P * stored), so
//       a butterfly applies one relative rotation to one operand.  The leaf
//       weight zeta = omega^s enters only as a pre-rotation of the ITFT's
//       spectral inputs (x_j <- zeta^-j' x_j) and a post-rotation of the
//       outputs (TFT: zeta^j'; ITFT: the f-output), because
//       TFT_zeta(a)[j] = zeta^j' TFT_1(a)[j] (transform.hpp:288-311).  Inside
//       a leaf of length L' every relative rotation is then a multiple of
//       M/L' bits, i.e. whole 128-bit chunks for all BASELINE shapes;
//   (3) groups micro-ops into dependency levels (ops in a level touch
//       disjoint slots and run concurrently);
//   (4) orders leaves into a ticket list for one persistent launch: batches
//       of top-level sub-transforms small enough to stay L2 resident are run
//       level by level, so intermediate levels hit L2 instead of HBM.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace cftft_b200 {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

// Exponent a*s + b of omega, symbolic in a leaf weight s (all mod M).
struct SymExp {
  u64 a = 0, b = 0;
  SymExp operator+(const SymExp& o) const { return {a + o.a, b + o.b}; }
  SymExp operator-(const SymExp& o) const { return {a - o.a, b - o.b}; }
};

enum OpType : std::uint8_t {
  OP_ADDSUB = 0,    // a <- a + R(b);            b <- a - R(b)
  OP_ADD = 1,       // a <- a + R(b)
  OP_SUB2 = 2,      // a <- 2a - R(b)
  OP_SUB2DIFF = 3,  // a <- 2a - R(b);           b <- a - R(b)
  OP_COPY = 4,      // b <- a   (verbatim; the planner sets b's pending exponent)
  OP_DBL = 5,       // a <- 2a             (negacyclic only)
  OP_HALF = 6,      // a <- a/2            (negacyclic only)
  OP_ADDHALF = 7,   // a <- (a + R(b))/2   (negacyclic only)
};

// One micro-op; R = multiplication by omega^r (r concrete, reduced mod M).
struct DevOp {
  std::uint8_t type;
  std::uint8_t pad0;
  std::uint16_t a, b;
  std::uint16_t pad1;
  u64 r;
  u64 pad2;  // prime rings: omega^r 2^64 mod p (upload)
};
static_assert(sizeof(DevOp) == 24, "DevOp layout");

// A leaf class program, device layout (indices into the plan's tables).
struct DevClass {
  u32 L;            // leaf length (slots)
  u32 nload;        // slots [0, nload) are loaded from global memory
  u32 nstore;       // slots [0, nstore) are stored back
  u32 nlevels;
  u32 level_begin;  // index into level table (nlevels + 1 entries)
  u32 pre_begin;    // index into rotation table: nload pre-rotations
  u32 post_begin;   // index into rotation table: nstore post-rotations
  u32 has_pre;      // any nonzero pre-rotation coefficient
  u32 op_begin;     // first op of the class in the op table
  u32 nops;         // number of ops
  // leaf geometry (Fermat).  A leaf works on `cs` chunks of every slot:
  //   whole leaves (kind 0): cs = C, all lanes, any rotation, carries resolved
  //     at the store (element format out);
  //   coset leaves (kind 1): the lanes p == c0 .. c0+m-1 (mod step) of every
  //     slot, step = (M >> ell) / lane_bits; lane-aligned rotations only,
  //     carry-save format out (lanes + per-lane tops).
  u32 kind;
  u32 cs;          // chunks per slot in shared memory
  u32 m;           // cosets per ticket (coset leaves)
  u32 step;        // coset step in lanes (coset leaves)
  u32 slot_bytes;  // shared-memory bytes per slot
  u32 inverse;     // ITFT program: tpre goes to pre slots < spec_n, tpost to post slot fslot;
  u32 spec_n;      // TFT program: tpost goes to every post slot
  u32 fslot;
  u32 wop_begin;   // wave engine, coset classes: first packed op in Plan::wave_ops
  u32 wnet;        // wave engine: 0 generic ops, 1 / 2 the full 8-point network with
                   // butterfly spans 4,2,1 / 1,2,4 (ADDSUB only; run in registers)
};

constexpr u32 kNoDep = 0xFFFFFFFFu;

// Completion tracking: one counter per (node, phase) of the decomposition.
// A counter counts finished children (leaves or whole sub-nodes) of its
// phase; when it reaches `target` and the phase is its node's last, the node
// is finished and the counter `next` (the parent's phase) is bumped in turn.
struct DevCounter {
  u32 target;
  u32 next;  // kNoDep: none
};

struct DevLeaf {
  u32 cls;
  u32 dep;         // counter to wait for (kNoDep: none)
  u32 dep_target;  // ... until it reaches this value
  u32 comp;        // counter to bump when done (kNoDep: none)
  u64 base;        // view index of slot 0
  u64 stride;      // view-index distance between slots
  u64 s;           // leaf weight (omega exponent), reduced mod M
  // extra rotations of a leaf on the boundary of a factored node (see
  // Planner::node): added to the pre-rotation of the ITFT's spectral inputs
  // (tpre) and to the post-rotation of the TFT's outputs / the ITFT's f-output
  // (tpost); 0 elsewhere
  u64 tpre, tpost;
  u32 c0;          // coset leaves: first coset of this ticket
  // Buffer of each slot (plans with coset leaves): the tickets of one coset
  // leaf read and write different lanes of the same coefficients, so a coset
  // leaf reads each slot from one of two buffers (the caller's view, a shadow
  // copy) and writes it to the other.  locbits[locoff + 2w] / [+ 2w + 1]: bit
  // k%64 of word w = slot k's input / output buffer.  kNoDep: all in the view.
  u32 locoff;
};
static_assert(sizeof(DevLeaf) == 64, "DevLeaf layout");

struct ClassKey {
  int inverse;
  unsigned ell;
  u64 z, n;
  int f;
  int kind = 0;  // 0 whole, 1 coset
  bool operator<(const ClassKey& o) const {
    return std::tie(inverse, ell, z, n, f, kind) < std::tie(o.inverse, o.ell, o.z, o.n, o.f, o.kind);
  }
};

struct LeafProgram {
  ClassKey key;
  std::vector<DevOp> ops;          // sorted by level
  std::vector<u32> level_begin;    // nlevels + 1 offsets into ops
  std::vector<SymExp> pre;         // per loaded slot (a*s + b)
  std::vector<SymExp> post;        // per stored slot
  u32 nload = 0, nstore = 0;
  bool has_pre = false;
  // geometry (DevClass)
  u32 kind = 0, cs = 0, m = 1, step = 1, slot_bytes = 0;
};

struct Plan {
  bool inverse = false;
  u64 L = 0, s = 0, z = 0, n = 0;
  int f = 0, policy = 0;
  std::vector<LeafProgram> classes;
  std::vector<DevLeaf> leaves;  // ticket order (topological)
  std::vector<u32> leaf_wave;   // merged wave index of each leaf (debug / waves view)
  std::vector<DevCounter> counters;
  unsigned max_ell = 0;
  u64 final_count = 0;  // outputs [0, final_count) are canonicalised at the end
  u64 max_slot_area = 0;  // shared-memory bytes of the largest leaf
  bool coset = false;     // some leaves write carry-save lanes (tops array in use)
  u64 extent = 0;         // view indices [0, extent) touched (tops array rows)
  std::vector<u64> locbits;        // per-slot buffer bits (see DevLeaf::locoff)
  std::vector<u64> shadow_finals;  // outputs the schedule leaves in the shadow buffer
  // the fold visits listed outputs (fold_list in place, shadow_finals from the
  // shadow buffer into place) instead of the index range [0, final_count)
  bool use_fold_list = false;
  std::vector<u64> fold_list;
  // small-coefficient plans: tickets are groups {first leaf, count} of
  // consecutive leaves (Planner::group_leaves); empty: one leaf per ticket
  std::vector<u32> groups;
  // wave engine: ticket ranges of mutually independent leaves, launched in
  // order; {first ticket, count, kind (0 whole, 1 coset), coset ranges: the
  // most warp groups of lane cosets a ticket of the range has}
  std::vector<std::array<u64, 4>> waves;
  // wave engine, coset classes: micro-ops packed as type | a << 4 | b << 10 |
  // q << 16, q the rotation in coset positions (class order, see wop_begin)
  std::vector<u32> wave_ops;
  std::vector<u32> wave_op_begin;  // per class
  std::vector<u32> wave_net;       // per class, DevClass::wnet
  // per class: its TMA phase program in wave_ops (Planner::tma_program), or
  // kNoDep (64-slot classes that are not full networks)
  std::vector<u32> wave_prog;
  // wave engine, coset tickets: per slot {pre bits | fresh << 30 | in-buffer << 31,
  // post lanes | final output << 30 | out-buffer << 31}, at DevLeaf::c0 (reused as the offset);
  // fresh: the element was never written by the plan before (its tops are zero, not loaded);
  // whole tickets with deferred rotations on their inputs: per loaded slot
  // the extra pre-rotation bits, at DevLeaf::c0 - 1 (c0 = 0: none)
  std::vector<u32> wave_slots;
  // outputs whose last writer deferred a sub-lane rotation: bits per view
  // element [0, extent), applied by the final fold (empty: none)
  std::vector<u32> final_rot;
  bool wide = false;  // some waves run on coset_wide_kernel (kind 2)
  // the tops arrays must start zeroed: some kernel reads the tops of an
  // element the plan has not written (wave plans: whole leaves only)
  bool tops_clear = true;
};

// Ring-dependent planning parameters.
struct RingShape {
  bool fermat = true;  // false: negacyclic (or prime)
  // prime rings (one u64 per coefficient): up to this many identical leaves
  // on adjacent coefficients share a ticket (Planner::group_leaves)
  u32 group = 1;
  u64 M = 0;           // root order
  unsigned max_leaf_ell = 3;
  u64 elem_bytes = 0;          // bytes per coefficient (for L2 batching)
  // bytes of top-level sub-transforms per ticket-order batch: the engine is
  // issue bound, so batches favour parallelism over L2 residency
  u64 l2_budget = 512ull << 20;
  // whole-leaf geometry (Fermat): chunks per element and slot bytes
  u32 C = 0;
  u32 slot_bytes = 0;
  // coset mode (Fermat): lanes of lane_bits bits (= chunks), 0 = off
  u64 lane_bits = 0;
  unsigned coset_max_ell = 0;
  u64 slot_budget = 0;  // shared-memory bytes available for a leaf's slots
  u32 wave_overlap = 0;  // waves by which consecutive L2 batches overlap in the ticket order
  u64 ticket_budget = 0;  // shared-memory bytes a coset ticket may fill (default: one of two buffers)
  // wave engine: leaves of <= 8 coefficients, one launch per independent wave;
  // coset leaves run on the warp-level kernel (csrc/wave_coset.cuh)
  bool wave_engine = false;
  bool wave_unaligned = true;  // coset leaves may take unaligned pre-rotations (warp kernel)
  // wave engine with coset leaves of up to 64 coefficients: leaves of 2^4..2^6
  // run on the CTA kernel (csrc/wave_wide.cuh); the top-level split leaves
  // row nodes of 2^(6k) coefficients (three radix-64 passes at L = 2^18)
  bool wide = false;
  // 64-slot ITFT classes that are not full networks stay radix-64 leaves when
  // they have a phase program (the TMA kernel runs them in one pass)
  bool tma_programs = true;
};

// Fermat shared-memory slot: cs chunks of lane_bytes, an int32 top per chunk,
// the element's 64-bit top word; 16-byte aligned.
inline u32 fermat_slot_bytes(u64 cs, u64 lane_bytes) {
  return (u32)((cs * lane_bytes + ((cs * 4 + 7) & ~u64(7)) + 8 + 15) & ~u64(15));
}

inline u64 bitrev(u64 j, unsigned ell) {
  u64 r = 0;
  for (unsigned i = 0; i < ell; ++i) {
    r = (r << 1) | (j & 1);
    j >>= 1;
  }
  return r;
}

// ---------------------------------------------------------------------------
class Planner {
 public:
  explicit Planner(const RingShape& rs) : rs_(rs) {}

  // Independent sub-transforms in one schedule (one launch): the building
  // block of the multi-GPU column / row passes.
  struct Item {
    u64 L, s, z, n;
    int f;
    u64 base, stride;
  };
  Plan build_batch(bool inverse, const std::vector<Item>& items, int policy) {
    Plan p;
    p.inverse = inverse;
    p.policy = policy;
    reset();
    u64 item_bytes = items.empty() ? 1 : (items[0].L * std::max<u64>(1, rs_.elem_bytes));
    u64 batch = std::max<u64>(1, rs_.l2_budget / std::max<u64>(1, item_bytes));
    for (size_t k = 0; k < items.size(); ++k) {
      const Item& it = items[k];
      Ctx c;
      c.dep = kNoDep;
      c.report = kNoDep;
      c.top_phase = 0;
      c.top_batch = k / batch;
      c.top_child = k;
      node(inverse, it.L, it.s, it.z, it.n, it.f, it.base, it.stride, policy, /*depth=*/1, c, 0, Bnd{});
    }
    std::vector<u64> finals;
    for (const Item& it : items)
      for (u64 k = 0; k < it.n + (u64)(inverse ? it.f : 0); ++k) finals.push_back(it.base + k * it.stride);
    finish(p, finals);
    p.final_count = 0;  // caller canonicalises
    fold_lists(p, finals, true);
    return p;
  }

  Plan build(bool inverse, u64 L, u64 s, u64 z, u64 n, int f, int policy) {
    Plan p;
    p.inverse = inverse;
    p.L = L;
    p.s = s;
    p.z = z;
    p.n = n;
    p.f = f;
    p.policy = policy;
    reset();
    Ctx root;
    root.dep = kNoDep;
    root.dep_target = 0;
    root.report = kNoDep;
    node(inverse, L, s, z, n, f, 0, 1, policy, /*depth=*/0, root, /*wave0=*/0, Bnd{});
    p.final_count = inverse ? n + (u64)f : n;
    std::vector<u64> finals(p.final_count);
    for (u64 k = 0; k < p.final_count; ++k) finals[k] = k;
    finish(p, finals);
    fold_lists(p, finals, false);
    return p;
  }

 private:
  static unsigned ctz(u64 x) { return (unsigned)__builtin_ctzll(x); }

  // Which outputs the fold visits, and from where: a batch folds its outputs
  // only (not every element in [0, extent)); outputs left in the shadow buffer
  // are folded from there straight into place (no separate copy back).
  static void fold_lists(Plan& p, const std::vector<u64>& finals, bool batch) {
    if (!p.coset || (!batch && p.shadow_finals.empty())) return;
    p.use_fold_list = true;
    std::vector<u64> sh = p.shadow_finals;
    std::sort(sh.begin(), sh.end());
    p.fold_list.clear();
    for (u64 e : finals)
      if (!std::binary_search(sh.begin(), sh.end(), e)) p.fold_list.push_back(e);
  }

  void reset() {
    class_index_.clear();
    classes_.clear();
    progs_.clear();
    lin_progs_.clear();
    leaves_.clear();
    keys_.clear();
    counters_.clear();
    max_ell_ = 0;
    max_area_ = 0;
    coset_used_ = false;
    extent_ = 0;
  }

  // Buffers of every slot (plans with coset leaves).  A coset leaf reads each
  // slot from one buffer and writes it to the other; a whole leaf (one
  // ticket) may read and write either.  Backward over the leaves (emission
  // order is topological), whole leaves pick the output buffer that brings
  // the element back to the caller's view after the coset leaves that
  // follow; forward, the actual buffers are assigned.  Outputs that still end
  // in the shadow buffer (an odd run of coset leaves from the inputs) are
  // listed for the final fold to copy back.
  void assign_buffers(Plan& p, const std::vector<u64>& finals) {
    const size_t nt = leaves_.size();
    std::vector<size_t> gs;
    for (size_t t = 0; t < nt; ++t) {
      if (t > 0) {
        const DevLeaf &a = leaves_[t - 1], &b = leaves_[t];
        if (classes_[b.cls].kind == 1 && a.cls == b.cls && a.base == b.base && a.stride == b.stride && b.c0 != 0)
          continue;
      }
      gs.push_back(t);
    }
    constexpr std::uint8_t ANY = 2;
    std::vector<std::uint8_t> req(extent_, ANY);
    for (u64 e : finals) req[e] = 0;
    std::vector<std::vector<u64>> pref(gs.size());
    for (size_t gi = gs.size(); gi-- > 0;) {
      const DevLeaf& lf = leaves_[gs[gi]];
      const LeafProgram& c = classes_[lf.cls];
      const u32 nl = c.nload, ns = c.nstore, span = std::max(nl, ns);
      pref[gi].assign((span + 63) / 64, 0);
      for (u32 k = 0; k < span; ++k) {
        const u64 e = lf.base + (u64)k * lf.stride;
        if (k < ns) {
          const std::uint8_t want = req[e] == ANY ? 0 : req[e];
          if (c.kind == 0) {
            if (want) pref[gi][k / 64] |= u64{1} << (k % 64);
            req[e] = ANY;
          } else {
            req[e] = k < nl ? (std::uint8_t)(1 - want) : ANY;
          }
        } else {
          req[e] = ANY;
        }
      }
    }
    std::vector<std::uint8_t> loc(extent_, 0);
    p.locbits.clear();
    for (size_t gi = 0; gi < gs.size(); ++gi) {
      const size_t t0 = gs[gi], t1 = gi + 1 < gs.size() ? gs[gi + 1] : nt;
      const DevLeaf& lf = leaves_[t0];
      const LeafProgram& c = classes_[lf.cls];
      const u32 nl = c.nload, ns = c.nstore, span = std::max(nl, ns), nw = (span + 63) / 64;
      const u32 off = (u32)p.locbits.size();
      p.locbits.resize(off + 2 * (size_t)nw, 0);
      for (u32 k = 0; k < nl; ++k)
        if (loc[lf.base + (u64)k * lf.stride]) p.locbits[off + 2 * (k / 64)] |= u64{1} << (k % 64);
      for (u32 k = 0; k < ns; ++k) {
        const u64 e = lf.base + (u64)k * lf.stride;
        const std::uint8_t o = c.kind == 1 ? (std::uint8_t)(1 - loc[e]) : (std::uint8_t)((pref[gi][k / 64] >> (k % 64)) & 1);
        if (o) p.locbits[off + 2 * (k / 64) + 1] |= u64{1} << (k % 64);
        loc[e] = o;
      }
      for (size_t t = t0; t < t1; ++t) leaves_[t].locoff = off;
    }
    p.shadow_finals.clear();
    for (u64 e : finals)
      if (loc[e]) p.shadow_finals.push_back(e);
  }

  // Host-side precomputation for the warp-level kernel: packed micro-ops per
  // coset class and per-slot rotations / buffers per coset ticket.
  //
  // Deferred rotations: a coset leaf applies the whole-lane part q of a
  // post-rotation by r = q*lane + o bits and leaves 2^o pending on the
  // element; the element's next reader (emission order is topological, and
  // every element is read by at most one later leaf) adds o to its
  // pre-rotation -- any bits on the warp kernel, a per-slot table on the whole
  // leaf kernel -- and outputs still pending at the end are rotated after the
  // fold.  2^o commutes with everything in between: the element is only
  // copied between buffers.  (A slot read but not written keeps its value,
  // and so its pending rotation.)
  void wave_tables(Plan& p, const std::vector<u64>& finals) {
    const u64 M = rs_.M, lb = rs_.lane_bits;
    p.wave_ops.clear();
    p.wave_op_begin.assign(classes_.size(), 0);
    p.wave_net.assign(classes_.size(), 0);
    p.wave_prog.assign(classes_.size(), kNoDep);
    for (size_t c = 0; c < classes_.size(); ++c) {
      const LeafProgram& cl = classes_[c];
      p.wave_op_begin[c] = (u32)p.wave_ops.size();
      if (cl.kind != 1) continue;
      if (cl.key.ell >= 4) {
        // CTA kernel: the radix-64 network's rotations per (stage, warp, op),
        // or the class's micro-ops
        std::vector<u32> net;
        p.wave_net[c] = wide_network(cl, M, net);
        if (p.wave_net[c]) {
          p.wave_ops.insert(p.wave_ops.end(), net.begin(), net.end());
          continue;
        }
      } else {
        p.wave_net[c] = full_network(cl);
      }
      for (const auto& op : cl.ops) {
        const u64 q = op.type == OP_COPY ? 0 : (op.r / lb) / cl.step;
        p.wave_ops.push_back((u32)op.type | ((u32)op.a << 4) | ((u32)op.b << 10) | ((u32)q << 16));
      }
      std::vector<u32> prog;
      if (cl.key.ell == 6 && tma_program(cl, lb, prog)) {
        p.wave_prog[c] = (u32)p.wave_ops.size();
        p.wave_ops.insert(p.wave_ops.end(), prog.begin(), prog.end());
      }
    }
    p.wave_slots.clear();
    p.final_rot.clear();
    std::vector<u32> pend(extent_, 0);
    std::vector<u64> last(extent_, ~u64{0});  // wave_slots index of the element's last coset write
    std::vector<std::uint8_t> written(extent_, 0);  // tops rows valid (written by a leaf)
    p.tops_clear = false;
    for (auto& lf : leaves_) {
      const LeafProgram& cl = classes_[lf.cls];
      const bool inv = cl.key.inverse != 0;
      if (cl.kind != 1) {
        bool any = false;
        for (u32 k = 0; k < cl.nload; ++k) any |= pend[lf.base + (u64)k * lf.stride] != 0;
        for (u32 k = 0; k < cl.nload; ++k) p.tops_clear = p.tops_clear || !written[lf.base + (u64)k * lf.stride];
        for (u32 k = 0; k < cl.nstore; ++k) written[lf.base + (u64)k * lf.stride] = 1;  // tops rows zeroed
        if (any) {
          lf.c0 = (u32)p.wave_slots.size() + 1;
          for (u32 k = 0; k < cl.nload; ++k) p.wave_slots.push_back(pend[lf.base + (u64)k * lf.stride]);
        }
        for (u32 k = 0; k < cl.nstore; ++k) {
          pend[lf.base + (u64)k * lf.stride] = 0;
          last[lf.base + (u64)k * lf.stride] = ~u64{0};
        }
        continue;
      }
      const u32 off = (u32)p.wave_slots.size();
      const u32 span = std::max(cl.nload, cl.nstore);
      for (u32 k = 0; k < span; ++k) {
        const u64 e = lf.base + (u64)k * lf.stride;
        u32 pre = 0, post = 0;
        if (k < cl.nload) {
          const u64 r = cl.pre[k].a * lf.s + cl.pre[k].b + ((inv && k < cl.key.n) ? lf.tpre : 0) + pend[e];
          pre = (u32)(r & (M - 1));  // bits: the warp kernel takes unaligned pre-rotations
          if (!written[e]) pre |= 1u << 30;
        }
        if (k < cl.nstore) written[e] = 1;
        if (k < cl.nstore) {
          const bool tp = inv ? (cl.key.f && k == cl.key.n) : true;
          const u64 r = (cl.post[k].a * lf.s + cl.post[k].b + (tp ? lf.tpost : 0)) & (M - 1);
          post = (u32)(r / lb);
          pend[e] = (u32)(r % lb);
          last[e] = p.wave_slots.size() + 1;
        }
        if (lf.locoff != kNoDep) {
          if ((p.locbits[lf.locoff + 2 * (k / 64)] >> (k % 64)) & 1) pre |= 1u << 31;
          if ((p.locbits[lf.locoff + 2 * (k / 64) + 1] >> (k % 64)) & 1) post |= 1u << 31;
        }
        p.wave_slots.push_back(pre);
        p.wave_slots.push_back(post);
      }
      lf.c0 = off;
    }
    for (u64 e : finals) {
      if (pend[e]) {
        if (p.final_rot.empty()) p.final_rot.assign(extent_, 0);
        p.final_rot[e] = pend[e];
      }
      // the last writer of an output absorbs lane tops into the next lane
      // where the warp holds both (wave_coset.cuh, store_slot)
      if (last[e] != ~u64{0}) p.wave_slots[last[e]] |= 1u << 30;
    }
  }

  // launch kind of a leaf class in the wave engine: 0 whole (leaf_kernel),
  // 1 coset leaf of <= 8 coefficients (coset_wave_kernel), 2 coset leaf of
  // 16..64 coefficients (coset_wide_kernel)
  u32 wave_kind(const LeafProgram& cl) const {
    if (cl.kind != 1) return 0;
    if (cl.key.ell <= 3) return 1u;
    return 2u;
  }

  // 1 / 2: the 64-slot class runs as the radix-2 DIF (spans 32..1, the TFT's)
  // / DIT (spans 1..32, the ITFT's) network of ADDSUB butterflies, as two
  // stages of eight 8-point networks in registers (coset_wide_kernel); 0:
  // anything else.  `net` gets the rotation (coset positions << 16) of every
  // butterfly, ordered (stage, warp, op) with ops in the 8-point network order
  // of wave_coset.cuh.  Truncated programs qualify when every op lies on a
  // network pair in network order and the network -- missing inputs read as
  // zeros, butterflies the program skips run with rotation 0, outputs >= n
  // not stored -- reproduces the program exactly: both are evaluated over
  // Z[x]/(x^32+1) (x = the leaf's rotation unit, x^32 = -1) on random inputs.
  static u32 wide_network(const LeafProgram& cl, u64 M, std::vector<u32>& net) {
    if (cl.key.ell != 6 || cl.nload == 0 || cl.ops.empty()) return 0;
    const u64 unit = M >> 6;
    using V = std::array<long long, 32>;
    auto rot = [](const V& v, u64 q) {  // x^q v
      V r{};
      for (u32 d = 0; d < 32; ++d) {
        const u64 t = d + q;
        const bool neg = ((t / 32) & 1) != 0;
        r[t % 32] = neg ? -v[d] : v[d];
      }
      return r;
    };
    auto ilog = [](u32 h) { u32 l = 0; while ((1u << l) < h) ++l; return l; };
    for (u32 kind = 1; kind <= 2; ++kind) {
      int qn[6][32];
      for (auto& row : qn)
        for (int& q : row) q = -1;
      std::array<int, 64> last;
      last.fill(-1);
      bool ok = true;
      for (const DevOp& op : cl.ops) {
        const u32 a = op.a, b = op.b, h = b - a;
        if (op.type > OP_COPY || b <= a || b >= 64 || (h & (h - 1)) || (a & h)) { ok = false; break; }
        const int lvl = kind == 1 ? 5 - (int)ilog(h) : (int)ilog(h);
        if (last[a] >= lvl || last[b] >= lvl) { ok = false; break; }
        last[a] = last[b] = lvl;
        if (op.type != OP_COPY && op.r % unit) { ok = false; break; }
        const u32 j = (a / (2 * h)) * h + a % h;
        qn[lvl][j] = op.type == OP_COPY ? 0 : (int)((op.r / unit) % 64);
      }
      if (!ok) continue;
      // exact evaluation: the program, then the network
      std::vector<V> x0(64), x1;
      u64 seed = 0x9E3779B97F4A7C15ull * (cl.key.z * 131 + cl.key.n * 7 + kind);
      for (u32 k = 0; k < 64; ++k)
        for (u32 d = 0; d < 32; ++d) {
          seed = seed * 6364136223846793005ull + 1442695040888963407ull;
          x0[k][d] = k < cl.nload ? (long long)((seed >> 33) % 2001) - 1000 : 0;
        }
      x1 = x0;
      for (const DevOp& op : cl.ops) {
        V& A = x1[op.a];
        V& B = x1[op.b];
        if (op.type == OP_COPY) { B = A; continue; }
        const V rb = rot(B, (op.r / unit) % 64);
        V s0, s1;
        for (u32 d = 0; d < 32; ++d) {
          s0[d] = (op.type == OP_SUB2 || op.type == OP_SUB2DIFF ? 2 * A[d] - rb[d] : A[d] + rb[d]);
          s1[d] = A[d] - rb[d];
        }
        A = s0;
        if (op.type == OP_ADDSUB || op.type == OP_SUB2DIFF) B = s1;
      }
      std::vector<V> y = x0;
      for (int lvl = 0; lvl < 6; ++lvl) {
        const u32 h = kind == 1 ? (32u >> lvl) : (1u << lvl);
        for (u32 j = 0; j < 32; ++j) {
          const u32 a = (j / h) * 2 * h + j % h;
          const V rb = rot(y[a + h], (u64)std::max(0, qn[lvl][j]));
          for (u32 d = 0; d < 32; ++d) {
            const long long av = y[a][d];
            y[a][d] = av + rb[d];
            y[a + h][d] = av - rb[d];
          }
        }
      }
      for (u32 k = 0; k < cl.nstore && ok; ++k) ok = y[k] == x1[k];
      if (!ok) continue;
      net.assign(2 * 8 * 12, 0);
      for (u32 st = 0; st < 2; ++st)
        for (u32 w = 0; w < 8; ++w)
          for (u32 o = 0; o < 12; ++o) {
            const u32 ll = o / 4, jj = o % 4;
            const u32 hl = kind == 1 ? (4u >> ll) : (1u << ll);
            const u32 al = (jj / hl) * 2 * hl + jj % hl;
            // stage slots: DIF stage 0 / DIT stage 1 take w + 8i, the others 8w + i
            const bool strided = (kind == 1) == (st == 0);
            const u32 a = strided ? w + 8 * al : 8 * w + al, h = strided ? 8 * hl : hl;
            const u32 lvl = 3 * st + ll;
            const u32 j = (a / (2 * h)) * h + a % h;
            net[(st * 8 + w) * 12 + o] = (u32)std::max(0, qn[lvl][j]) << 16;
          }
      // Stage B re-gauged (wave_tma.cuh, net8_g): slot j of a stage-B network
      // is read as x^{g_j} * slot j (a row index and a sign), the g_j chosen
      // so that seven butterflies need no rotation (both outputs of a
      // butterfly keep a's gauge; q' = q + G_a - G_b); bits 4..9 of op j < 8:
      // g_j, bits 10..15 of the other five ops: the residual rotation.
      for (u32 w = 0; w < 8; ++w) {
        u32* e = &net[(8 + w) * 12];
        u32 q[12], g[8], res[12] = {};
        for (u32 o = 0; o < 12; ++o) q[o] = (e[o] >> 16) & 63u;
        g[0] = 0;
        if (kind == 1) {  // DIF: pairs (k, k+4), then (0,2) (1,3) (4,6) (5,7), then (2k, 2k+1)
          g[1] = q[8]; g[2] = q[4]; g[3] = g[1] + q[5]; g[4] = q[0];
          g[5] = g[1] + q[1]; g[6] = g[2] + q[2]; g[7] = g[3] + q[3];
          res[6] = q[6] - q[4]; res[7] = q[7] - q[5];
        } else {          // DIT: pairs (2k, 2k+1), then (0,2) (1,3) (4,6) (5,7), then (k, k+4)
          g[1] = q[0]; g[2] = q[4]; g[3] = g[2] + q[1]; g[4] = q[8];
          g[5] = g[4] + q[2]; g[6] = g[4] + q[6]; g[7] = g[6] + q[3];
          res[5] = q[5] - q[4]; res[7] = q[7] - q[6];
        }
        for (u32 o = 9; o < 12; ++o) res[o] = q[o] - q[8];
        for (u32 o = 0; o < 12; ++o) e[o] |= (o < 8 ? (g[o] & 63u) << 4 : 0u) | ((res[o] & 63u) << 10);
      }
      return kind;
    }
    return 0;
  }

  // A 64-slot coset class that is not a full network (the truncated ITFT
  // leaves: the reference's phases i..iv over an 8 x 8 grid, slot 8r + c,
  // transform.hpp:215-238) as a phase program for the TMA kernel's warp
  // groups (wave_tma.cuh, prog_ops): each op lies inside one row or one
  // column of the grid; in a row phase warp w runs the ops of row w, in a
  // column phase those of column w, in level order; a phase starts when the
  // previous one is done on every warp.  Phases alternate row / column; an
  // op goes to the first phase of its kind after the phases of every earlier
  // op on its slots (the same phase when that op is of its kind: then it is
  // the same warp's).  Layout: word 0 = phase count P | network rows << 8,
  // words 1 + 8p + w = (first op << 16) | op count of warp w in phase p
  // (offsets from word 0), words 1 + 8P + 12w: row w's network ops, then the
  // ops packed as in wave_ops (bit 22: runs paired with the next op).  Returns false when an op spans rows
  // and columns, reads a slot nothing has defined (slots >= nload are never
  // loaded), or needs more than 8 phases.
  static bool tma_program(const LeafProgram& cl, u64 lane_bits, std::vector<u32>& out) {
    if (cl.key.ell != 6 || cl.kind != 1 || cl.nload == 0 || cl.ops.empty()) return false;
    constexpr int kMaxPhases = 8;
    std::array<int, 64> lastp;  // phase of the last op on the slot (-1: none)
    lastp.fill(-1);
    std::array<bool, 64> defined{};
    for (u32 k = 0; k < 64; ++k) defined[k] = k < cl.nload;
    const int t0 = (cl.ops[0].a % 8 != cl.ops[0].b % 8) ? 0 : 1;  // kind of phase 0 (0 rows, 1 columns)
    std::vector<std::array<std::vector<u32>, 8>> ph;
    for (const DevOp& op : cl.ops) {
      const u32 a = op.a, b = op.b;
      if (a >= 64 || b >= 64) return false;
      int kind;
      if (a == b && (op.type == OP_ADDSUB || op.type == OP_SUB2DIFF || op.type == OP_COPY)) return false;
      if (a == b)  // a <- a +- R(a): either kind; stay in the slot's last phase
        kind = lastp[a] < 0 ? t0 : (((lastp[a] & 1) == 0) ? t0 : 1 - t0);
      else if (a / 8 == b / 8)
        kind = 0;
      else if (a % 8 == b % 8)
        kind = 1;
      else
        return false;
      if (!defined[a] || (op.type != OP_COPY && !defined[b])) return false;
      if (op.type != OP_COPY && op.type != OP_ADDSUB && op.type != OP_ADD && op.type != OP_SUB2 &&
          op.type != OP_SUB2DIFF)
        return false;
      const u32 owner = kind == 0 ? a / 8 : a % 8;
      int p = (kind == t0) ? 0 : 1;
      for (u32 s : {a, b}) {
        if (lastp[s] < 0) continue;
        const int q = lastp[s];
        const int qk = ((q & 1) == 0) ? t0 : 1 - t0;
        const int need = qk == kind ? q : q + 1;
        while (p < need) p += 2;
      }
      if (p >= kMaxPhases) return false;
      if ((int)ph.size() <= p) ph.resize(p + 1);
      const u64 q = op.type == OP_COPY ? 0 : (op.r / lane_bits) / cl.step;
      ph[p][owner].push_back((u32)op.type | (a << 4) | (b << 10) | ((u32)q << 16));
      lastp[a] = lastp[b] = p;
      defined[b] = defined[b] || op.type == OP_ADDSUB || op.type == OP_SUB2DIFF || op.type == OP_COPY;
    }
    for (u32 k = 0; k < cl.nstore; ++k)
      if (!defined[k]) return false;
    const u32 P = (u32)ph.size();
    // phase 0 rows that are full 8-point DIT networks (the ITFT's phase i) run
    // in registers on the DIT kernel (stage_a: ADDSUB on the network's pairs,
    // rotations only where kRotDit has them); their ops stay in the list for
    // the DIF kernel
    static const u32 pr[12][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {0, 2}, {1, 3},
                                  {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};
    constexpr u32 kRotDitMask = (1u << 5) | (1u << 7) | (1u << 9) | (1u << 10) | (1u << 11);
    u32 netmask = 0;
    for (u32 w = 0; w < 8 && t0 == 0 && P > 0; ++w) {
      const auto& v = ph[0][w];
      bool net = v.size() == 12;
      for (u32 j = 0; j < 12 && net; ++j) {
        const u32 wop = v[j];
        net = (wop & 15u) == OP_ADDSUB && ((wop >> 4) & 63u) == 8 * w + pr[j][0] &&
              ((wop >> 10) & 63u) == 8 * w + pr[j][1] && (((kRotDitMask >> j) & 1u) || (wop >> 16) == 0);
      }
      if (net) netmask |= 1u << w;
    }
    // pairs: an ADDSUB (ADD) followed by an ADDSUB (ADD) on other slots (bit
    // 22 on the first) run together (two independent carry chains), within a
    // 32-op chunk
    for (auto& phase : ph)
      for (auto& v : phase)
        for (size_t k = 0; k + 1 < v.size();) {
          const u32 x = v[k], y = v[k + 1];
          const u32 xa = (x >> 4) & 63u, xb = (x >> 10) & 63u, ya = (y >> 4) & 63u, yb = (y >> 10) & 63u;
          const u32 tx = x & 15u, ty = y & 15u;
          if ((k & 31) != 31 && tx == ty && (tx == OP_ADDSUB || tx == OP_ADD) && xa != ya && xa != yb &&
              xb != ya && xb != yb) {
            v[k] |= 1u << 22;
            k += 2;
          } else {
            k += 1;
          }
        }
    out.assign(1 + 8 * P + 96, 0);
    out[0] = P | (netmask << 8);
    for (u32 w = 0; w < 8; ++w)
      if ((netmask >> w) & 1u)
        for (u32 j = 0; j < 12; ++j) out[1 + 8 * P + 12 * w + j] = ph[0][w][j] & ~(1u << 22);
    for (u32 p = 0; p < P; ++p)
      for (u32 w = 0; w < 8; ++w) {
        out[1 + 8 * p + w] = ((u32)out.size() << 16) | (u32)ph[p][w].size();
        out.insert(out.end(), ph[p][w].begin(), ph[p][w].end());
      }
    return out.size() < 65536;
  }

  // 1 / 2: the class runs as the full 8-point network of ADDSUB butterflies
  // with spans 4,2,1 (the TFT's) / 1,2,4 (the ITFT's) in level order -- the
  // warp kernel then keeps it in registers; 0: anything else.  Truncated
  // programs (z or n < 8) qualify when every op is an ADDSUB on the network's
  // pairs, a COPY into a slot that still holds a truncated (zero) input, or an
  // ADD whose b is never read again: with the missing inputs read as zeros
  // and outputs >= n not stored, the ADDSUB network computes the same values.
  static u32 full_network(const LeafProgram& cl) {
    if (cl.key.ell != 3 || cl.ops.size() != 12 || cl.nload == 0) return 0;
    for (u32 net = 1; net <= 2; ++net) {
      bool ok = true;
      bool zero[8];
      for (u32 k = 0; k < 8; ++k) zero[k] = k >= cl.nload;
      for (u32 o = 0; o < 12 && ok; ++o) {
        const u32 lvl = o >> 2, j = o & 3, h = net == 1 ? (4u >> lvl) : (1u << lvl);
        const u32 a = (j / h) * 2 * h + (j % h);
        const DevOp& op = cl.ops[o];
        ok = op.a == a && op.b == a + h;
        if (!ok) break;
        if (op.type == OP_COPY) {
          ok = zero[op.b];
        } else if (op.type == OP_ADD) {
          for (u32 o2 = o + 1; o2 < 12 && ok; ++o2) ok = cl.ops[o2].a != op.b && cl.ops[o2].b != op.b;
          ok = ok && op.b >= cl.nstore;
        } else {
          ok = op.type == OP_ADDSUB;
        }
        const bool z = zero[op.a] && zero[op.b];
        zero[op.a] = zero[op.b] = z;
      }
      if (ok) return net;
    }
    return 0;
  }

  // ticket order: (top phase, batch, wave, top child, emission order), with
  // the waves of consecutive L2 batches overlapped by `overlap` waves: batch
  // b's wave w is ranked at w + (W - overlap) b (W = waves per batch), so the
  // next batch's first waves fill the CTAs that the tail of a batch (its few
  // late tickets) leaves idle.  Any such order is topological: batches are
  // independent, and each keeps its own wave order.
  void finish(Plan& p, const std::vector<u64>& finals) {
    if (coset_used_) assign_buffers(p, finals);
    if (rs_.wave_engine) wave_tables(p, finals);
    std::vector<u32> idx(leaves_.size());
    for (u32 i = 0; i < idx.size(); ++i) idx[i] = i;
    u32 W = 1;
    for (const auto& k : keys_) W = std::max(W, std::get<2>(k) + 1);
    const u32 ov = std::min(W - 1, rs_.wave_overlap);
    auto rank = [&](u32 x) {
      const auto& k = keys_[x];
      if (rs_.wave_engine)  // (top phase, wave, kind): every range is independent
        return std::make_tuple(std::get<0>(k), (u64)std::get<2>(k), (u64)wave_kind(classes_[leaves_[x].cls]),
                               std::get<3>(k), std::get<4>(k));
      // (grouped small-coefficient plans: a wave's leaves are independent --
      // ordered by element address, adjacent columns become consecutive tickets)
      return std::make_tuple(std::get<0>(k), (u64)std::get<2>(k) + (u64)(W - ov) * std::get<1>(k), std::get<1>(k),
                             rs_.group > 1 ? leaves_[x].base : std::get<3>(k), std::get<4>(k));
    };
    std::stable_sort(idx.begin(), idx.end(), [&](u32 x, u32 y) { return rank(x) < rank(y); });
    p.waves.clear();
    p.wide = false;
    if (rs_.wave_engine) {
      for (size_t t = 0; t < idx.size(); ++t) {
        const auto& k = keys_[idx[t]];
        const u64 kind = wave_kind(classes_[leaves_[idx[t]].cls]);
        if (t == 0 || std::get<0>(keys_[idx[t - 1]]) != std::get<0>(k) ||
            std::get<2>(keys_[idx[t - 1]]) != std::get<2>(k) || p.waves.back()[2] != kind)
          p.waves.push_back({(u64)t, 0, kind, 0});
        p.waves.back()[1] += 1;
        if (kind == 2) p.wide = true;
        if (kind >= 1) {  // a warp row takes 2^(6 - ell) cosets of all positions (wave_coset.cuh, wave_wide.cuh)
          const LeafProgram& c = classes_[leaves_[idx[t]].cls];
          const u64 groups = std::max<u64>(1, (u64)c.step >> (6 - c.key.ell));
          p.waves.back()[3] = std::max(p.waves.back()[3], groups);
        }
      }
    }
    p.leaves.reserve(idx.size());
    p.leaf_wave.reserve(idx.size());
    for (u32 i : idx) {
      p.leaves.push_back(leaves_[i]);
      p.leaf_wave.push_back(std::get<2>(keys_[i]));
    }
    if (rs_.group > 1 && !rs_.wave_engine) group_leaves(p);
    p.classes = std::move(classes_);
    p.counters = std::move(counters_);
    p.max_ell = max_ell_;
    p.max_slot_area = max_area_;
    p.coset = coset_used_;
    p.extent = extent_;
  }

  // Small coefficients (one u64): consecutive leaves of one class on adjacent
  // coefficients (base, base + 1, ...: the columns u, u+1, ... of one phase,
  // same stride) share a ticket of up to rs_.group leaves, so that a slot
  // access covers whole 32-byte sectors (PAPER.md:837-839 processes several
  // columns at once for the same reason).  Each member keeps its own weight,
  // dependency and completion counter.
  void group_leaves(Plan& p) const {
    p.groups.clear();
    // at most 4096 slots per ticket: big leaves (2^9..2^11) group fewer
    const size_t cap = std::max<size_t>(1, std::min<size_t>(rs_.group, size_t{4096} >> max_ell_));
    for (size_t t = 0; t < p.leaves.size();) {
      const DevLeaf& g = p.leaves[t];
      size_t n = 1;
      while (n < cap && t + n < p.leaves.size()) {
        const DevLeaf& x = p.leaves[t + n];
        if (x.cls != g.cls || x.stride != g.stride || x.base != g.base + n || p.leaf_wave[t + n] != p.leaf_wave[t])
          break;
        ++n;
      }
      p.groups.push_back((u32)t);
      p.groups.push_back((u32)n);
      t += n;
    }
  }

  // Split for a node: the reference's policy at the top (transform.hpp:83-87),
  // an SMEM-sized near-balanced split below it.
  void split(unsigned ell, int policy, bool top, unsigned& l1, unsigned& l2) const {
    if (top && rs_.wide && !policy_everywhere_ && ell > 6) {
      // any split gives the same outputs (transform_test.cpp:248-272): the
      // row nodes get 2^(6k) coefficients (radix-64 passes), the columns the rest
      l1 = ell - 6 * ((ell - 1) / 6);
      l2 = ell - l1;
      return;
    }
    if (top || policy_everywhere_) {
      if (policy == 1) {
        l1 = 1;
        l2 = ell - 1;
      } else {
        l1 = ell / 2;
        l2 = ell - ell / 2;
      }
      return;
    }
    unsigned lam = rs_.max_leaf_ell;
    if (rs_.fermat && rs_.lane_bits) lam = std::max(lam, rs_.coset_max_ell);
    unsigned k = (ell + lam - 1) / lam;  // levels needed
    l1 = (ell + k - 1) / k;
    if (l1 >= ell) l1 = ell - 1;
    if (l1 < 1) l1 = 1;
    l2 = ell - l1;
  }

  struct Ctx {
    u32 dep = kNoDep, dep_target = 0;
    u32 report = kNoDep;  // counter of the parent phase this subtree reports to
    // top-level bookkeeping for ticket ordering
    u32 top_phase = 0;
    u64 top_batch = 0, top_child = 0;
  };

  // A "factored" node: the first node on a path whose internal rotations
  // (multiples of M/L) are whole lanes.  Its weight zeta = omega^sigma is
  // taken out -- TFT_zeta = diag(zeta^[j]) TFT_1 and ITFT_zeta = ITFT_1 after
  // x_j <- zeta^-[j] x_j (j < n), with the f-output times zeta^[n]
  // (transform.hpp:288-311) -- so every leaf inside runs with a lane-aligned
  // weight and only the leaves on the node's boundary carry the (possibly
  // unaligned) rotations zeta^[j].
  struct Bnd {
    bool active = false;
    u64 sigma = 0;
    unsigned ell = 0;
    u64 base = 0, stride = 1;
    bool out = false;  // TFT: this sub-node's outputs are the node's outputs
    bool in = false;   // ITFT: its spectral inputs are the node's spectral inputs
    bool fo = false;   // ITFT: its f-output is the node's f-output
  };

  using Key = std::tuple<u32, u64, u32, u64, u64>;  // phase, batch, wave, child, seq

  // One node of the GPU decomposition (base/stride in view elements).
  // Returns the number of completion events it reports to cx.report and the
  // number of waves (leaf levels) it spans.
  std::pair<u64, u32> node(bool inv, u64 L, u64 s, u64 z, u64 n, int f, u64 base, u64 stride,
                           int policy, int depth, const Ctx& cx, u32 wave0, Bnd bnd) {
    const u64 M = rs_.M;
    s &= (M - 1);
    unsigned ell = ctz(L);
    extent_ = std::max(extent_, base + (L - 1) * stride + 1);
    const bool coset_on = rs_.fermat && rs_.lane_bits != 0;
    if (coset_on && !bnd.active && (M >> ell) % rs_.lane_bits == 0) {
      bnd.active = true;
      bnd.sigma = s;
      bnd.ell = ell;
      bnd.base = base;
      bnd.stride = stride;
      bnd.out = !inv;
      bnd.in = inv;
      bnd.fo = inv && f;
      s = 0;
    }
    if (bnd.active) {
      u64 units = 0;
      if (try_leaf(inv, L, s, z, n, f, base, stride, policy, cx, wave0, bnd, units)) return {units, 1};
    } else if (ell <= rs_.max_leaf_ell) {
      DevLeaf lf{};
      lf.s = s;
      emit_whole(inv, ell, z, n, f, base, stride, policy, cx, wave0, lf);
      return {1, 1};
    }
    unsigned l1, l2;
    if (bnd.active) {
      const bool unal = (bnd.sigma % rs_.lane_bits) != 0;
      if (unal && !(rs_.wave_engine && rs_.wave_unaligned) && ((!inv && bnd.out) || (inv && bnd.in))) {
        // the boundary rows (TFT: last level, ITFT: first level) carry
        // unaligned rotations: make them whole leaves
        l2 = std::min(rs_.max_leaf_ell, ell - 1);
        l1 = ell - l2;
      } else {
        const unsigned lam = std::max(1u, rs_.coset_max_ell);
        const unsigned k = std::max(2u, (ell + lam - 1) / lam);
        l1 = (ell + k - 1) / k;
        if (l1 >= ell) l1 = ell - 1;
        l2 = ell - l1;
      }
    } else if (coset_on && depth > 0) {
      l1 = ell / 2;
      l2 = ell - l1;
    } else {
      split(ell, policy, depth == 0, l1, l2);
    }
    const u64 cols = u64{1} << l2, rows = u64{1} << l1;
    const u64 col_step = M >> ell;
    const u64 s_row = s << l1;

    // a phase = list of child sub-transforms
    struct Child {
      u64 L, s, z, n;
      int f;
      u64 base, stride;
      Bnd b;
    };
    Bnd colb = bnd, rowb = bnd;
    colb.out = colb.in = colb.fo = false;  // columns never touch the node boundary
    std::vector<std::vector<Child>> phases;
    if (!inv) {  // transform.hpp:154-186
      const u64 n2 = n & (cols - 1), n1 = n >> l2, n1c = n1 + (n2 ? 1 : 0);
      const u64 z2 = z & (cols - 1), z1 = z >> l2, z2e = z1 ? cols : z2;
      std::vector<Child> c, r;
      for (u64 u = 0; u < z2e; ++u)
        c.push_back({rows, s + u * col_step, u < z2 ? z1 + 1 : z1, n1c, 0, base + u * stride,
                     stride * cols, colb});
      for (u64 u = 0; u < n1c; ++u)
        r.push_back({cols, s_row, z2e, u < n1 ? cols : n2, 0, base + u * cols * stride, stride, rowb});
      phases.push_back(std::move(c));
      phases.push_back(std::move(r));
    } else {  // transform.hpp:188-239
      const u64 n2 = n & (cols - 1), n1 = n >> l2, z2 = z & (cols - 1), z1 = z >> l2;
      const int fm = (n2 + (u64)f > 0) ? 1 : 0;
      const u64 z2e = z1 ? cols : z2;
      const u64 lo = std::min(n2, z2), hi = std::max(n2, z2);
      Bnd r1 = bnd;  // phase i rows: full rows of node spectral inputs, no f-output
      r1.fo = false;
      Bnd r3 = bnd;  // phase iii row: its first n2 inputs and its f-output are the node's
      std::vector<Child> p1, p2, p3, p4;
      for (u64 u = 0; u < n1; ++u)
        p1.push_back({cols, s_row, cols, cols, 0, base + u * cols * stride, stride, r1});
      for (u64 u = n2; u < z2e; ++u)
        p2.push_back({rows, s + u * col_step, u < hi ? z1 + 1 : z1, n1, fm, base + u * stride, stride * cols,
                      colb});
      if (fm) p3.push_back({cols, s_row, z2e, n2, f, base + n1 * cols * stride, stride, r3});
      for (u64 u = 0; u < n2; ++u)
        p4.push_back({rows, s + u * col_step, u < lo ? z1 + 1 : z1, n1 + 1, 0, base + u * stride, stride * cols,
                      colb});
      for (auto* ph : {&p1, &p2, &p3, &p4})
        if (!ph->empty()) phases.push_back(std::move(*ph));
    }

    u32 wave = wave0;
    u32 prev_counter = kNoDep;
    u32 prev_target = 0;
    u32 phase_index = 0;
    for (auto& ph : phases) {
      const u32 cid = (u32)counters_.size();
      counters_.push_back(DevCounter{0, kNoDep});
      Ctx c2;
      if (phase_index == 0) {
        c2.dep = cx.dep;
        c2.dep_target = cx.dep_target;
      } else {
        c2.dep = prev_counter;
        c2.dep_target = prev_target;
      }
      c2.report = cid;
      u32 maxw = 0;
      u64 units = 0;
      // L2 batching of top-level children
      u64 child_bytes = (u64{1} << ctz(ph.front().L)) * rs_.elem_bytes;
      u64 batch = std::max<u64>(1, rs_.l2_budget / std::max<u64>(1, child_bytes));
      for (u64 ci = 0; ci < ph.size(); ++ci) {
        const Child& ch = ph[ci];
        if (depth == 0) {
          c2.top_phase = phase_index;
          c2.top_batch = ci / batch;
          c2.top_child = ci;
        } else {
          c2.top_phase = cx.top_phase;
          c2.top_batch = cx.top_batch;
          c2.top_child = cx.top_child;
        }
        u32 w0 = depth == 0 ? 0 : wave;
        auto [k, w] = node(inv, ch.L, ch.s, ch.z, ch.n, ch.f, ch.base, ch.stride, policy, depth + 1,
                           c2, w0, ch.b);
        units += k;
        maxw = std::max(maxw, w);
      }
      counters_[cid].target = (u32)units;
      prev_counter = cid;
      prev_target = (u32)units;
      wave += maxw;
      ++phase_index;
    }
    // the node is finished when its last phase is: report to the parent phase
    counters_[prev_counter].next = cx.report;
    return {1, wave - wave0};
  }

  // Boundary rotations of a leaf inside a factored node (see Bnd): leaf slot k
  // sits at node position j = rb + k * 2^a, so zeta^[j] = omega^(t + [k] s2)
  // with t = sigma [rb] and s2 = sigma 2^(ell_node - a - ell_leaf).
  void boundary(const Bnd& bnd, bool inv, unsigned ell, u64 base, u64 stride, DevLeaf& lf) const {
    const u64 M = rs_.M;
    if (!bnd.active) return;
    const bool tft_out = !inv && bnd.out;
    const bool itft_b = inv && (bnd.in || bnd.fo);
    if (!tft_out && !itft_b) return;
    const u64 rb = (base - bnd.base) / bnd.stride, rt = stride / bnd.stride;
    const unsigned a = ctz(rt);
    const u64 s2 = (bnd.sigma << (bnd.ell - a - ell)) & (M - 1);
    const u64 t = (bnd.sigma * bitrev(rb, bnd.ell)) & (M - 1);
    // boundary leaves have a zero weight of their own inside the factored node
    if (lf.s != 0) throw std::logic_error("planner: boundary leaf with a nonzero weight");
    lf.s = s2;
    if (tft_out) lf.tpost = t;
    if (inv && bnd.in) lf.tpre = (M - t) & (M - 1);
    if (inv && bnd.fo) lf.tpost = t;
  }

  // A leaf inside a factored node: a coset leaf when every rotation it
  // performs is lane aligned, else a whole leaf when it fits; false: split.
  bool try_leaf(bool inv, u64 L, u64 s, u64 z, u64 n, int f, u64 base, u64 stride, int policy,
                const Ctx& cx, u32 wave0, const Bnd& bnd, u64& units) {
    const unsigned ell = ctz(L);
    DevLeaf lf{};
    lf.s = s;
    boundary(bnd, inv, ell, base, stride, lf);
    if (coset_fits(ell)) {
      const ClassKey key{inv ? 1 : 0, ell, z, n, f, 1};
      const LeafProgram& prog = coset_program(key, policy);
      // a 64-coefficient ITFT leaf that is neither a full network nor a
      // phase program for the TMA kernel (tma_program) would run its
      // micro-ops on the CTA kernel, an order of magnitude slower per byte
      // than the radix-8 warp waves: cut it into radix-8 leaves instead
      bool take = aligned(prog, inv, ell, lf);
      if (take && inv && ell == 6 && rs_.wide) {
        auto it = full_net_.find(key);
        if (it == full_net_.end()) {
          std::vector<u32> net;
          bool ok = wide_network(prog, rs_.M, net) != 0;
          if (!ok && rs_.tma_programs) {
            LeafProgram cp = prog;  // the class's coset geometry (class_of)
            cp.kind = 1;
            cp.step = (u32)(lanes2() >> ell);
            ok = cp.step >= 2 && tma_program(cp, rs_.lane_bits, net);
          }
          it = full_net_.emplace(key, ok).first;
        }
        take = it->second;
      }
      if (take) {
        units = emit_coset(key, policy, base, stride, cx, wave0, lf);
        return true;
      }
    }
    if (ell <= rs_.max_leaf_ell) {
      emit_whole(inv, ell, z, n, f, base, stride, policy, cx, wave0, lf);
      units = 1;
      return true;
    }
    return false;
  }

  u64 lanes2() const { return rs_.M / rs_.lane_bits; }  // 2C
  u32 coset_slot_bytes(u64 cs) const { return fermat_slot_bytes(cs, rs_.lane_bits / 8); }

  // coset tickets must fit one of the two ticket buffers (double buffering)
  bool coset_fits(unsigned ell) const {
    if (!rs_.lane_bits || ell > rs_.coset_max_ell || ell < 1) return false;
    if ((u64{1} << ell) > lanes2()) return false;  // step >= 1
    const u64 cs = u64{1} << (ell - 1);
    return (u64{1} << ell) * coset_slot_bytes(cs) <= rs_.slot_budget / 2;
  }

  // every op rotation a multiple of the coset step, every pre/post rotation a
  // whole number of lanes
  bool aligned(const LeafProgram& prog, bool inv, unsigned ell, const DevLeaf& lf) const {
    const u64 M = rs_.M, inner = M >> ell, lb = rs_.lane_bits;
    for (const auto& op : prog.ops)
      if (op.type != OP_COPY && (op.r % inner) != 0) return false;
    for (u32 k = 0; k < prog.nload && !(rs_.wave_engine && rs_.wave_unaligned); ++k) {  // the warp kernel takes any pre-rotation
      u64 r = prog.pre[k].a * lf.s + prog.pre[k].b + ((inv && k < prog.key.n) ? lf.tpre : 0);
      if ((r & (M - 1)) % lb) return false;
    }
    // the warp kernel applies the lane part of a post-rotation and defers the
    // sub-lane rest to the next reader of the element (see wave_tables)
    for (u32 k = 0; k < prog.nstore && !(rs_.wave_engine && rs_.wave_unaligned); ++k) {
      const bool tp = inv ? (prog.key.f && k == prog.key.n) : true;
      u64 r = prog.post[k].a * lf.s + prog.post[k].b + (tp ? lf.tpost : 0);
      if ((r & (M - 1)) % lb) return false;
    }
    return true;
  }

  void push_leaf(const DevLeaf& lf, const Ctx& cx, u32 wave0) {
    leaves_.push_back(lf);
    keys_.push_back(Key{cx.top_phase, cx.top_batch, wave0, cx.top_child, (u64)keys_.size()});
  }

  void emit_whole(bool inv, unsigned ell, u64 z, u64 n, int f, u64 base, u64 stride, int policy, const Ctx& cx,
                  u32 wave0, DevLeaf lf) {
    lf.cls = class_of(ClassKey{inv ? 1 : 0, ell, z, n, f, 0}, policy);
    lf.locoff = kNoDep;
    lf.dep = cx.dep;
    lf.dep_target = cx.dep_target;
    lf.comp = cx.report;
    lf.base = base;
    lf.stride = stride;
    lf.c0 = 0;
    push_leaf(lf, cx, wave0);
    max_ell_ = std::max(max_ell_, ell);
  }

  u64 emit_coset(const ClassKey& key, int policy, u64 base, u64 stride, const Ctx& cx, u32 wave0, DevLeaf lf) {
    lf.cls = class_of(key, policy);
    const LeafProgram& c = classes_[lf.cls];
    lf.dep = cx.dep;
    lf.dep_target = cx.dep_target;
    lf.comp = cx.report;
    lf.base = base;
    lf.stride = stride;
    const u64 groups = c.step / c.m;
    lf.locoff = kNoDep;
    for (u64 g = 0; g < groups; ++g) {
      lf.c0 = (u32)(g * c.m);
      push_leaf(lf, cx, wave0);
    }
    coset_used_ = true;
    return groups;
  }

  // ---- leaf programs -------------------------------------------------------
  const LeafProgram& program(ClassKey k, int policy) {
    k.kind = 0;
    auto it = progs_.find(k);
    if (it == progs_.end()) it = progs_.emplace(k, build_leaf(k, policy)).first;
    return it->second;
  }

  // The program a coset leaf runs: the leaf program, or -- when its op
  // rotations are not lane aligned (the ITFT's halvings) and the wave engine
  // takes sub-lane pre-rotations -- its linear form, if it has one.
  const LeafProgram& coset_program(ClassKey k, int policy) {
    k.kind = 0;
    auto it = lin_progs_.find(k);
    if (it != lin_progs_.end()) return it->second;
    const LeafProgram& src = program(k, policy);
    LeafProgram lin;
    const u64 inner = rs_.M >> k.ell;
    bool al = true;
    for (const auto& op : src.ops) al = al && (op.type == OP_COPY || op.r % inner == 0);
    const bool use = !al && rs_.wave_engine && rs_.wave_unaligned && rs_.fermat &&
                     (linearize(src, lin) || realign(src, lin));
    return lin_progs_.emplace(k, use ? lin : src).first->second;
  }

  // Sub-unit offsets: the same program with every op rotation a multiple of
  // the leaf's unit U = M >> ell, when offsets d_k (true value of slot k =
  // omega^d_k * stored) absorb the rest.  The ITFT's divisions by 2 (omega =
  // 2 in the Fermat ring, 2^-1 = omega^(M-1)) leave chains such as
  // x <- 2x - omega^(2U-3) y, x <- 2x - omega^(4U-2) y', ... (the row n1 of
  // a truncated 64-point ITFT, transform.hpp:227-230): x starts with an
  // offset of -4 (taken by its load's pre-rotation, any bits on the TMA and
  // warp kernels) and each step is computed as omega (x - omega^(r-1) y),
  // raising the offset by one.  Per op, in order: the exact form when it is
  // aligned; else a slot still holding its loaded value takes the offset
  // that aligns it (its pre-rotation changes); else SUB2 as the shifted
  // subtraction.  Loads and stores absorb the offsets (pre - d, post + d).
  bool realign(const LeafProgram& src, LeafProgram& dst) const {
    const u64 M = rs_.M, U = M >> src.key.ell, H = M / 2;
    const u32 L = 1u << src.key.ell;
    if (U < 2) return false;
    std::vector<u64> d(L, 0), dload(L, 0);
    std::vector<char> fresh(L, 0);  // loaded, not yet read or written by an op
    for (u32 k = 0; k < src.nload; ++k) fresh[k] = 1;
    dst = src;
    for (auto& op : dst.ops) {
      const u32 a = op.a, b = op.b;
      if (op.type == OP_COPY) {
        d[b] = d[a];
        fresh[a] = fresh[b] = 0;
        continue;
      }
      if (op.type != OP_ADD && op.type != OP_ADDSUB && op.type != OP_SUB2 && op.type != OP_SUB2DIFF) return false;
      u64 rr = (op.r + d[b] - d[a]) & (M - 1);
      if (rr % U) {
        if (fresh[a] && a != b) {
          const u64 m = rr % U;  // d_a += m
          d[a] = (d[a] + m) & (M - 1);
          dload[a] = d[a];
          rr -= m;
        } else if (fresh[b] && a != b) {
          const u64 m = rr % U;  // d_b -= m
          d[b] = (d[b] - m) & (M - 1);
          dload[b] = d[b];
          rr -= m;
        } else if (op.type == OP_SUB2 && ((rr + M - 1) & (M - 1)) % U == 0) {
          // 2x - R y = omega (x - omega^-1 R y): an ADD of -omega^(r-1) y, offset + 1
          op.type = OP_ADD;
          op.r = (rr + M - 1 + H) & (M - 1);
          d[a] = (d[a] + 1) & (M - 1);
          fresh[a] = fresh[b] = 0;
          continue;
        } else {
          return false;
        }
      }
      op.r = rr;
      if (op.type == OP_ADDSUB || op.type == OP_SUB2DIFF) d[b] = d[a];
      fresh[a] = fresh[b] = 0;
    }
    for (u32 k = 0; k < dst.nload; ++k) dst.pre[k].b = (dst.pre[k].b - dload[k]) & (M - 1);
    for (u32 k = 0; k < dst.nstore; ++k) dst.post[k].b = (dst.post[k].b + d[k]) & (M - 1);
    return true;
  }

  // A one-output program whose output is a sum of +-omega^e multiples of its
  // (loaded) inputs, each input in at most one term, as that sum: the inputs
  // pre-rotated by their e (any bits: the wave kernel's sub-lane loads), then
  // added with rotation 0 (lane aligned).  The program's ops are replayed on
  // symbolic stored values -- lists of (input, exponent) -- with the kernel's
  // semantics (ADD a += R b, ADDSUB, SUB2 a = 2a - R b, SUB2DIFF, COPY b = a;
  // 2 = omega^1, -1 = omega^(M/2)).  False: not such a program.
  bool linearize(const LeafProgram& src, LeafProgram& dst) const {
    if (src.nstore != 1 || src.nload == 0) return false;
    const u64 M = rs_.M, H = M / 2;
    const u32 L = 1u << src.key.ell;
    using Terms = std::vector<std::pair<u32, u64>>;
    std::vector<Terms> t(L);
    for (u32 k = 0; k < src.nload; ++k) t[k].push_back({k, 0});
    bool ok = true;
    auto add_into = [&](Terms acc, const Terms& x, u64 sh) {
      for (const auto& [in, e0] : x) {
        const u64 e = (e0 + sh) & (M - 1);
        auto it = std::find_if(acc.begin(), acc.end(), [&](const auto& q) { return q.first == in; });
        if (it == acc.end()) {
          acc.push_back({in, e});
        } else if (it->second == e) {
          it->second = (e + 1) & (M - 1);  // 2 omega^e
        } else if (it->second == ((e + H) & (M - 1))) {
          acc.erase(it);  // cancels
        } else {
          ok = false;
        }
      }
      return acc;
    };
    auto shifted = [&](const Terms& x, u64 sh) {
      Terms r = x;
      for (auto& q : r) q.second = (q.second + sh) & (M - 1);
      return r;
    };
    for (const DevOp& op : src.ops) {
      const u32 a = op.a, b = op.b;
      switch (op.type) {
        case OP_ADD: t[a] = add_into(t[a], t[b], op.r); break;
        case OP_COPY: t[b] = t[a]; break;
        case OP_ADDSUB: {
          Terms ta = add_into(t[a], t[b], op.r), tb = add_into(t[a], t[b], op.r + H);
          t[a] = std::move(ta);
          t[b] = std::move(tb);
          break;
        }
        case OP_SUB2: t[a] = add_into(shifted(t[a], 1), t[b], op.r + H); break;
        case OP_SUB2DIFF: {
          Terms ta = add_into(shifted(t[a], 1), t[b], op.r + H), tb = add_into(t[a], t[b], op.r + H);
          t[a] = std::move(ta);
          t[b] = std::move(tb);
          break;
        }
        default: return false;
      }
      if (!ok) return false;
    }
    const Terms& out = t[0];
    if (out.empty()) return false;
    dst = LeafProgram{};
    dst.key = src.key;
    dst.nload = src.nload;
    dst.nstore = 1;
    dst.pre = src.pre;
    dst.post = src.post;
    dst.has_pre = true;
    Emit e;
    e.M = M;
    e.last.assign(L, 0);
    e.P.assign(L, 0);
    bool has0 = false;
    for (const auto& [in, ex] : out) {
      dst.pre[in].b = (dst.pre[in].b + ex) & (M - 1);
      has0 = has0 || in == 0;
    }
    if (!has0) e.push(OP_COPY, out[0].first, 0, 0, true);
    for (const auto& [in, ex] : out)
      if (in != 0 && (has0 || in != out[0].first)) e.push(OP_ADD, 0, in, 0, true);
    u32 nlev = 0;
    for (auto& r : e.ops) nlev = std::max(nlev, r.level);
    for (auto& r : e.ops) dst.ops.push_back(r.op);  // emitted in level order (a chain on slot 0)
    dst.level_begin.assign(nlev + 1, 0);
    size_t idx = 0;
    for (u32 l = 0; l <= nlev; ++l) {
      while (idx < e.ops.size() && e.ops[idx].level <= l) ++idx;
      dst.level_begin[l] = (u32)idx;
    }
    return true;
  }

  u32 class_of(const ClassKey& k, int policy) {
    auto it = class_index_.find(k);
    if (it != class_index_.end()) return it->second;
    LeafProgram prog = k.kind == 1 ? coset_program(k, policy) : program(k, policy);
    prog.key = k;
    const u64 L = u64{1} << k.ell;
    prog.kind = (u32)k.kind;
    if (k.kind == 1) {
      prog.step = (u32)(lanes2() >> k.ell);
      const u64 cl = u64{1} << (k.ell - 1);  // lanes per coset
      u64 m = 1;
      while (m * 2 <= prog.step && m * 2 * cl <= 512 && L * coset_slot_bytes(m * 2 * cl) <= rs_.ticket_budget)
        m *= 2;
      if (rs_.wave_engine) m = prog.step;  // one ticket per leaf: the warp kernel covers all cosets
      prog.m = (u32)m;
      prog.cs = (u32)(m * cl);
      prog.slot_bytes = coset_slot_bytes(prog.cs);
    } else {
      prog.step = 1;
      prog.m = 1;
      prog.cs = rs_.C;
      prog.slot_bytes = rs_.slot_bytes;
    }
    // shared memory of the persistent leaf kernel (the wave engine runs coset
    // classes on its own kernels)
    if (!(rs_.wave_engine && k.kind == 1)) max_area_ = std::max<u64>(max_area_, L * prog.slot_bytes);
    u32 id = (u32)classes_.size();
    classes_.push_back(std::move(prog));
    class_index_[k] = id;
    return id;
  }

  struct Emit {
    struct Raw {
      DevOp op;
      u32 level;
    };
    std::vector<Raw> ops;
    std::vector<u32> last;  // last level touching each slot
    std::vector<u64> P;     // pending exponent per slot (concrete, zeta = 1)
    u64 M = 0;
    void push(std::uint8_t type, u32 a, u32 b, u64 r, bool two_slots) {
      u32 lv = last[a];
      if (two_slots) lv = std::max(lv, last[b]);
      lv += 1;
      last[a] = lv;
      if (two_slots) last[b] = lv;
      DevOp op{};
      op.type = type;
      op.a = (std::uint16_t)a;
      op.b = (std::uint16_t)b;
      op.r = r & (M - 1);
      ops.push_back({op, lv});
    }
  };

  void leaf_tft(Emit& e, u64 L, u64 s, u64 z, u64 n, u64 base, u64 stride, int policy) {
    if (L == 2) {
      u32 i = (u32)base, j = (u32)(base + stride);
      if (n == 2) {
        if (z == 2) {  // (x0+x1, zeta(x0-x1))
          e.push(OP_ADDSUB, i, j, e.P[j] - e.P[i], true);
          e.P[j] = e.P[i] + s;
        } else {  // x1 = zeta x0
          e.push(OP_COPY, i, j, 0, true);
          e.P[j] = e.P[i] + s;
        }
      } else if (z == 2) {  // x0 = x0 + x1
        e.push(OP_ADD, i, j, e.P[j] - e.P[i], true);
      }
      return;
    }
    unsigned ell = ctz(L), l1, l2;
    split_ref(ell, policy, l1, l2);
    const u64 cols = u64{1} << l2, rows = u64{1} << l1;
    const u64 n2 = n & (cols - 1), n1 = n >> l2, n1c = n1 + (n2 ? 1 : 0);
    const u64 z2 = z & (cols - 1), z1 = z >> l2, z2e = z1 ? cols : z2;
    const u64 col_step = rs_.M >> ell;
    for (u64 u = 0; u < z2; ++u)
      leaf_tft(e, rows, s + u * col_step, z1 + 1, n1c, base + u * stride, stride * cols, policy);
    for (u64 u = z2; u < z2e; ++u)
      leaf_tft(e, rows, s + u * col_step, z1, n1c, base + u * stride, stride * cols, policy);
    const u64 s_row = s << l1;
    for (u64 u = 0; u < n1; ++u) leaf_tft(e, cols, s_row, z2e, cols, base + u * cols * stride, stride, policy);
    if (n2 > 0) leaf_tft(e, cols, s_row, z2e, n2, base + n1 * cols * stride, stride, policy);
  }

  void leaf_itft(Emit& e, u64 L, u64 s, u64 z, u64 n, int f, u64 base, u64 stride, int policy) {
    const bool fermat = rs_.fermat;
    if (L == 2) {
      u32 i = (u32)base, j = (u32)(base + stride);
      if (n == 2) {  // (x0 + zeta^-1 x1, x0 - zeta^-1 x1)
        e.push(OP_ADDSUB, i, j, e.P[j] - e.P[i] - s, true);
        e.P[j] = e.P[i];
      } else if (n == 1) {
        if (f == 1) {
          if (z == 2) {  // (2x0 - x1, zeta(x0 - x1))
            e.push(OP_SUB2DIFF, i, j, e.P[j] - e.P[i], true);
            e.P[j] = e.P[i] + s;
          } else {  // (2x0, zeta x0)
            e.push(OP_COPY, i, j, 0, true);
            e.P[j] = e.P[i] + s;
            // the doubling as arithmetic (x0 + x0), not as a pending 1-bit
            // rotation: lane-local, so it never makes a later rotation (or
            // the element's final value) sub-lane
            if (fermat)
              e.push(OP_ADD, i, i, 0, true);
            else
              e.push(OP_DBL, i, i, 0, false);
          }
        } else {
          if (z == 2) {  // 2x0 - x1
            e.push(OP_SUB2, i, j, e.P[j] - e.P[i], true);
          } else {  // 2x0 (as x0 + x0, see above)
            if (fermat)
              e.push(OP_ADD, i, i, 0, true);
            else
              e.push(OP_DBL, i, i, 0, false);
          }
        }
      } else {  // n == 0: half(x0 + x1) or half(x0)
        if (z == 2) {
          if (fermat) {
            e.push(OP_ADD, i, j, e.P[j] - e.P[i], true);
            e.P[i] = e.P[i] + (rs_.M - 1);
          } else {
            e.push(OP_ADDHALF, i, j, e.P[j] - e.P[i], true);
          }
        } else {
          if (fermat)
            e.P[i] = e.P[i] + (rs_.M - 1);
          else
            e.push(OP_HALF, i, i, 0, false);
        }
      }
      return;
    }
    unsigned ell = ctz(L), l1, l2;
    split_ref(ell, policy, l1, l2);
    const u64 cols = u64{1} << l2, rows = u64{1} << l1;
    const u64 n2 = n & (cols - 1), n1 = n >> l2, z2 = z & (cols - 1), z1 = z >> l2;
    const int fm = (n2 + (u64)f > 0) ? 1 : 0;
    const u64 z2e = z1 ? cols : z2;
    const u64 lo = std::min(n2, z2), hi = std::max(n2, z2);
    const u64 col_step = rs_.M >> ell;
    const u64 s_row = s << l1;
    for (u64 u = 0; u < n1; ++u) leaf_itft(e, cols, s_row, cols, cols, 0, base + u * cols * stride, stride, policy);
    for (u64 u = n2; u < hi; ++u)
      leaf_itft(e, rows, s + u * col_step, z1 + 1, n1, fm, base + u * stride, stride * cols, policy);
    for (u64 u = hi; u < z2e; ++u)
      leaf_itft(e, rows, s + u * col_step, z1, n1, fm, base + u * stride, stride * cols, policy);
    if (fm) leaf_itft(e, cols, s_row, z2e, n2, f, base + n1 * cols * stride, stride, policy);
    for (u64 u = 0; u < lo; ++u)
      leaf_itft(e, rows, s + u * col_step, z1 + 1, n1 + 1, 0, base + u * stride, stride * cols, policy);
    for (u64 u = lo; u < n2; ++u)
      leaf_itft(e, rows, s + u * col_step, z1, n1 + 1, 0, base + u * stride, stride * cols, policy);
  }

  static void split_ref(unsigned ell, int policy, unsigned& l1, unsigned& l2) {
    if (policy == 1) {
      l1 = 1;
      l2 = ell - 1;
    } else {
      l1 = ell / 2;
      l2 = ell - ell / 2;
    }
  }

  LeafProgram build_leaf(const ClassKey& k, int policy) {
    const u64 L = u64{1} << k.ell;
    Emit e;
    e.M = rs_.M;
    e.last.assign(L, 0);
    e.P.assign(L, 0);
    // zeta = 1 inside the leaf; the weight is applied by pre/post rotations
    if (k.inverse)
      leaf_itft(e, L, 0, k.z, k.n, k.f, 0, 1, policy);
    else
      leaf_tft(e, L, 0, k.z, k.n, 0, 1, policy);
    LeafProgram prog;
    prog.key = k;
    prog.nload = (u32)k.z;
    prog.nstore = (u32)(k.inverse ? k.n + (u64)k.f : k.n);
    u32 nlev = 0;
    for (auto& r : e.ops) nlev = std::max(nlev, r.level);
    std::stable_sort(e.ops.begin(), e.ops.end(),
                     [](const Emit::Raw& x, const Emit::Raw& y) { return x.level < y.level; });
    prog.ops.reserve(e.ops.size());
    for (auto& r : e.ops) prog.ops.push_back(r.op);
    // level l (1-based) spans [level_begin[l-1], level_begin[l])
    prog.level_begin.assign(nlev + 1, 0);
    size_t idx = 0;
    for (u32 l = 0; l <= nlev; ++l) {
      while (idx < e.ops.size() && e.ops[idx].level <= l) ++idx;
      prog.level_begin[l] = (u32)idx;
    }
    const u64 M = rs_.M;
    prog.pre.assign(prog.nload, SymExp{});
    prog.post.assign(prog.nstore, SymExp{});
    for (u32 j = 0; j < prog.nstore; ++j) prog.post[j].b = e.P[j] & (M - 1);
    if (!k.inverse) {
      // TFT_zeta(a)[j] = zeta^{j'} TFT_1(a)[j]
      for (u32 j = 0; j < prog.nstore; ++j) prog.post[j].a = bitrev(j, k.ell);
    } else {
      // spectral inputs x_j (j < n) are pre-rotated by zeta^{-j'}; the
      // f-output is a spectral value: post-rotated by zeta^{n'}
      for (u32 j = 0; j < prog.nload && j < k.n; ++j) {
        prog.pre[j].a = (u64)0 - bitrev(j, k.ell);
        if (bitrev(j, k.ell)) prog.has_pre = true;
      }
      if (k.f) prog.post[k.n].a = bitrev(k.n, k.ell);
    }
    return prog;
  }

  RingShape rs_;
  bool policy_everywhere_ = false;
  std::map<ClassKey, u32> class_index_;
  std::map<ClassKey, LeafProgram> progs_;
  std::map<ClassKey, LeafProgram> lin_progs_;  // coset_program
  std::map<ClassKey, bool> full_net_;          // try_leaf: the class is a full radix-64 network
  std::vector<LeafProgram> classes_;
  std::vector<DevLeaf> leaves_;
  std::vector<Key> keys_;
  std::vector<DevCounter> counters_;
  unsigned max_ell_ = 0;
  u64 max_area_ = 0;
  bool coset_used_ = false;
  u64 extent_ = 0;
};

// Estimated device cost of a plan: bytes its leaves move (the wave kernels are
// bound by their data movement, profiles/r01_experiments.md) -- coset leaves
// their slots' lanes and carry-save tops, whole leaves weighted by the slower
// persistent kernel.
inline double plan_cost(const Plan& p, u64 elem_bytes) {
  double c = 0;
  for (const DevLeaf& lf : p.leaves) {
    const LeafProgram& cl = p.classes[lf.cls];
    const double b = (double)(cl.nload + cl.nstore) * (double)elem_bytes;
    c += cl.kind == 1 ? 1.125 * b : 4.0 * b;
  }
  return c;
}

// ---------------------------------------------------------------------------
// Base-case counts of the REFERENCE recursion (policy at every level), by
// replay without arithmetic; memoised since counts are data independent
// (verify.hpp:175-199).
class CountReplay {
 public:
  u64 tft(u64 L, u64 z, u64 n, int policy) {
    if (L == 2) return 1;
    auto key = std::make_tuple(0, L, z, n, 0, policy);
    auto it = memo_.find(key);
    if (it != memo_.end()) return it->second;
    unsigned ell = (unsigned)__builtin_ctzll(L), l1, l2;
    if (policy == 1) {
      l1 = 1;
      l2 = ell - 1;
    } else {
      l1 = ell / 2;
      l2 = ell - ell / 2;
    }
    const u64 cols = u64{1} << l2, rows = u64{1} << l1;
    const u64 n2 = n & (cols - 1), n1 = n >> l2, n1c = n1 + (n2 ? 1 : 0);
    const u64 z2 = z & (cols - 1), z1 = z >> l2, z2e = z1 ? cols : z2;
    u64 c = 0;
    if (z2) c += z2 * tft(rows, z1 + 1, n1c, policy);
    if (z2e > z2) c += (z2e - z2) * tft(rows, z1, n1c, policy);
    if (n1) c += n1 * tft(cols, z2e, cols, policy);
    if (n2) c += tft(cols, z2e, n2, policy);
    memo_[key] = c;
    return c;
  }
  u64 itft(u64 L, u64 z, u64 n, int f, int policy) {
    if (L == 2) return 1;
    auto key = std::make_tuple(1, L, z, n, f, policy);
    auto it = memo_.find(key);
    if (it != memo_.end()) return it->second;
    unsigned ell = (unsigned)__builtin_ctzll(L), l1, l2;
    if (policy == 1) {
      l1 = 1;
      l2 = ell - 1;
    } else {
      l1 = ell / 2;
      l2 = ell - ell / 2;
    }
    const u64 cols = u64{1} << l2, rows = u64{1} << l1;
    const u64 n2 = n & (cols - 1), n1 = n >> l2, z2 = z & (cols - 1), z1 = z >> l2;
    const int fm = (n2 + (u64)f > 0) ? 1 : 0;
    const u64 z2e = z1 ? cols : z2;
    const u64 lo = std::min(n2, z2), hi = std::max(n2, z2);
    u64 c = 0;
    if (n1) c += n1 * itft(cols, cols, cols, 0, policy);
    if (hi > n2) c += (hi - n2) * itft(rows, z1 + 1, n1, fm, policy);
    if (z2e > hi) c += (z2e - hi) * itft(rows, z1, n1, fm, policy);
    if (fm) c += itft(cols, z2e, n2, f, policy);
    if (lo) c += lo * itft(rows, z1 + 1, n1 + 1, 0, policy);
    if (n2 > lo) c += (n2 - lo) * itft(rows, z1, n1 + 1, 0, policy);
    memo_[key] = c;
    return c;
  }

 private:
  std::map<std::tuple<int, u64, u64, u64, int, int>, u64> memo_;
};

}  // namespace cftft_b200
