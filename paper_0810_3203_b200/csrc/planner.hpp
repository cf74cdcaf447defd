// planner.hpp -- host-side schedule builder for the GPU TFT/ITFT.
//
// The reference runs Algorithms 1 and 2 as a recursion over strided views
// (transform.hpp:154-239).  On the GPU the recursion is cut at "leaves":
// sub-transforms small enough that all their coefficients sit in one CTA's
// shared memory.  The planner
//   (1) replays the reference recursion above the leaves, with the
//       reference's own split at the top level and an SMEM-sized split
//       below it (outputs are unique, so any inner split gives the same
//       bits: transform_test.cpp:248-272), producing WAVES of independent
//       leaves (all columns of a node before its rows; ITFT phases i..iv);
//   (2) replays the reference recursion INSIDE a leaf symbolically in the
//       leaf weight s, turning every base case (transform.hpp:94-150) into a
//       micro-op on SMEM slots.  Multiplications by powers of omega are never
//       executed eagerly: each slot carries a pending exponent P (its true
//       value is omega^P * stored), so a butterfly applies exactly one
//       relative rotation to one operand, and the leaf's store applies the
//       final P of each output slot;
//   (3) groups micro-ops into dependency levels (ops in a level touch
//       disjoint slots and run concurrently).
// Leaf programs depend only on (kind, ell, z, n, f), so they are shared by
// all leaves of a class; per-leaf data is (class, base, stride, s).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

namespace cftft_b200 {

using u64 = std::uint64_t;
using u32 = std::uint32_t;

// Exponent a*s + b of omega, symbolic in the leaf weight s (all mod M).
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
  OP_COPY = 4,      // b <- a   (verbatim, pending exponent set by planner)
  OP_DBL = 5,       // a <- 2a             (negacyclic only)
  OP_HALF = 6,      // a <- a/2            (negacyclic only)
  OP_ADDHALF = 7,   // a <- (a + R(b))/2   (negacyclic only)
};

// One micro-op; R = multiplication by omega^(ra*s + rb).  Device layout.
struct DevOp {
  std::uint8_t type;
  std::uint8_t pad0;
  std::uint16_t a, b;
  std::uint16_t pad1;
  u64 ra, rb;
};
static_assert(sizeof(DevOp) == 24, "DevOp layout");

// A leaf class program, device layout (indices into the plan's tables).
struct DevClass {
  u32 L;            // leaf length (slots)
  u32 nload;        // slots [0, nload) are loaded from global memory
  u32 nstore;       // slots [0, nstore) are stored back
  u32 nlevels;
  u32 level_begin;  // index into level table (nlevels + 1 entries)
  u32 store_begin;  // index into store-rotation table (nstore entries)
};

struct DevLeaf {
  u32 cls;
  u32 pad;
  u64 base;    // view index of slot 0
  u64 stride;  // view-index distance between slots
  u64 s;       // leaf weight (omega exponent), reduced mod M
};
static_assert(sizeof(DevLeaf) == 32, "DevLeaf layout");

struct ClassKey {
  int inverse;
  unsigned ell;
  u64 z, n;
  int f;
  bool operator<(const ClassKey& o) const {
    return std::tie(inverse, ell, z, n, f) < std::tie(o.inverse, o.ell, o.z, o.n, o.f);
  }
};

struct LeafProgram {
  ClassKey key;
  std::vector<DevOp> ops;          // sorted by level
  std::vector<u32> level_begin;    // nlevels + 1 offsets into ops
  std::vector<SymExp> store_rot;   // final pending exponent per stored slot
  u32 nload = 0, nstore = 0;
};

struct Wave {
  std::vector<DevLeaf> leaves;
  unsigned max_ell = 0;  // largest leaf in the wave (sizes shared memory)
};

struct Plan {
  bool inverse = false;
  u64 L = 0, s = 0, z = 0, n = 0;
  int f = 0, policy = 0;
  std::vector<LeafProgram> classes;
  std::vector<Wave> waves;
  u64 final_count = 0;  // outputs [0, final_count) are canonicalised at the end
};

// Ring-dependent planning parameters.
struct RingShape {
  bool fermat = true;  // false: negacyclic
  u64 M = 0;           // root order
  unsigned max_leaf_ell = 3;
};

// ---------------------------------------------------------------------------
class Planner {
 public:
  explicit Planner(const RingShape& rs) : rs_(rs) {}

  Plan build(bool inverse, u64 L, u64 s, u64 z, u64 n, int f, int policy) {
    Plan p;
    p.inverse = inverse;
    p.L = L;
    p.s = s;
    p.z = z;
    p.n = n;
    p.f = f;
    p.policy = policy;
    class_index_.clear();
    classes_.clear();
    std::vector<Wave> waves;
    node(inverse, L, s, z, n, f, 0, 1, policy, true, waves);
    p.waves = std::move(waves);
    p.classes = std::move(classes_);
    p.final_count = inverse ? n + (u64)f : n;
    return p;
  }

 private:
  static unsigned ctz(u64 x) { return (unsigned)__builtin_ctzll(x); }

  // Split for a node: the reference's policy at the top (transform.hpp:83-87),
  // an SMEM-sized near-balanced split below it.
  void split(unsigned ell, int policy, bool top, unsigned& l1, unsigned& l2) const {
    if (top) {
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
    unsigned k = (ell + lam - 1) / lam;  // waves needed
    l1 = (ell + k - 1) / k;
    if (l1 >= ell) l1 = ell - 1;
    if (l1 < 1) l1 = 1;
    l2 = ell - l1;
  }

  static void merge_into(std::vector<Wave>& acc, std::vector<Wave>&& w) {
    if (acc.size() < w.size()) acc.resize(w.size());
    for (size_t i = 0; i < w.size(); ++i) {
      auto& dst = acc[i].leaves;
      dst.insert(dst.end(), w[i].leaves.begin(), w[i].leaves.end());
      acc[i].max_ell = std::max(acc[i].max_ell, w[i].max_ell);
    }
  }

  static void append(std::vector<Wave>& out, std::vector<Wave>&& w) {
    for (auto& x : w) out.push_back(std::move(x));
  }

  // One node of the GPU decomposition.  base/stride are in view elements.
  void node(bool inv, u64 L, u64 s, u64 z, u64 n, int f, u64 base, u64 stride, int policy,
            bool top, std::vector<Wave>& out) {
    const u64 M = rs_.M;
    s &= (M - 1);
    unsigned ell = ctz(L);
    // A leaf when it fits on chip.  At the top level a transform that fits is
    // still a single leaf (the leaf program replays the policy's recursion).
    if (ell <= rs_.max_leaf_ell) {
      Wave w;
      w.max_ell = ell;
      DevLeaf lf{};
      lf.cls = class_of(ClassKey{inv ? 1 : 0, ell, z, n, f}, policy);
      lf.base = base;
      lf.stride = stride;
      lf.s = s;
      w.leaves.push_back(lf);
      out.push_back(std::move(w));
      return;
    }
    unsigned l1, l2;
    split(ell, policy, top, l1, l2);
    const u64 cols = u64{1} << l2, rows = u64{1} << l1;
    const u64 col_step = M >> ell;
    const u64 s_row = s << l1;
    if (!inv) {  // transform.hpp:154-186
      const u64 n2 = n & (cols - 1), n1 = n >> l2, n1c = n1 + (n2 ? 1 : 0);
      const u64 z2 = z & (cols - 1), z1 = z >> l2, z2e = z1 ? cols : z2;
      std::vector<Wave> colw, roww;
      for (u64 u = 0; u < z2e; ++u) {
        std::vector<Wave> w;
        node(false, rows, s + u * col_step, u < z2 ? z1 + 1 : z1, n1c, 0, base + u * stride,
             stride * cols, policy, false, w);
        merge_into(colw, std::move(w));
      }
      for (u64 u = 0; u < n1c; ++u) {
        std::vector<Wave> w;
        node(false, cols, s_row, z2e, u < n1 ? cols : n2, 0, base + u * cols * stride, stride,
             policy, false, w);
        merge_into(roww, std::move(w));
      }
      append(out, std::move(colw));
      append(out, std::move(roww));
      return;
    }
    // transform.hpp:188-239
    const u64 n2 = n & (cols - 1), n1 = n >> l2, z2 = z & (cols - 1), z1 = z >> l2;
    const int fm = (n2 + (u64)f > 0) ? 1 : 0;
    const u64 z2e = z1 ? cols : z2;
    const u64 lo = std::min(n2, z2), hi = std::max(n2, z2);
    std::vector<Wave> ph1, ph2, ph3, ph4;
    for (u64 u = 0; u < n1; ++u) {
      std::vector<Wave> w;
      node(true, cols, s_row, cols, cols, 0, base + u * cols * stride, stride, policy, false, w);
      merge_into(ph1, std::move(w));
    }
    for (u64 u = n2; u < z2e; ++u) {
      std::vector<Wave> w;
      node(true, rows, s + u * col_step, u < hi ? z1 + 1 : z1, n1, fm, base + u * stride,
           stride * cols, policy, false, w);
      merge_into(ph2, std::move(w));
    }
    if (fm) {
      std::vector<Wave> w;
      node(true, cols, s_row, z2e, n2, f, base + n1 * cols * stride, stride, policy, false, w);
      merge_into(ph3, std::move(w));
    }
    for (u64 u = 0; u < n2; ++u) {
      std::vector<Wave> w;
      node(true, rows, s + u * col_step, u < lo ? z1 + 1 : z1, n1 + 1, 0, base + u * stride,
           stride * cols, policy, false, w);
      merge_into(ph4, std::move(w));
    }
    append(out, std::move(ph1));
    append(out, std::move(ph2));
    append(out, std::move(ph3));
    append(out, std::move(ph4));
  }

  // ---- leaf programs -------------------------------------------------------
  u32 class_of(const ClassKey& k, int policy) {
    auto it = class_index_.find(k);
    if (it != class_index_.end()) return it->second;
    LeafProgram prog = build_leaf(k, policy);
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
    std::vector<u32> last;     // last level touching each slot
    std::vector<SymExp> P;     // pending exponent per slot
    void push(std::uint8_t type, u32 a, u32 b, SymExp r, bool two_slots) {
      u32 lv = last[a];
      if (two_slots) lv = std::max(lv, last[b]);
      lv += 1;
      last[a] = lv;
      if (two_slots) last[b] = lv;
      DevOp op{};
      op.type = type;
      op.a = (std::uint16_t)a;
      op.b = (std::uint16_t)b;
      op.ra = r.a;
      op.rb = r.b;
      ops.push_back({op, lv});
    }
  };

  // Symbolic twiddles: the leaf is called with s = 1*s + 0.
  void leaf_tft(Emit& e, u64 L, SymExp s, u64 z, u64 n, u64 base, u64 stride, int policy) {
    if (L == 2) {
      u32 i = (u32)base, j = (u32)(base + stride);
      if (n == 2) {
        if (z == 2) {  // (x0+x1, zeta(x0-x1))
          e.push(OP_ADDSUB, i, j, e.P[j] - e.P[i], true);
          e.P[j] = e.P[i] + s;
        } else {  // x1 = zeta x0
          e.push(OP_COPY, i, j, SymExp{}, true);
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
      leaf_tft(e, rows, s + SymExp{0, u * col_step}, z1 + 1, n1c, base + u * stride,
               stride * cols, policy);
    for (u64 u = z2; u < z2e; ++u)
      leaf_tft(e, rows, s + SymExp{0, u * col_step}, z1, n1c, base + u * stride, stride * cols,
               policy);
    const SymExp s_row{s.a << l1, s.b << l1};
    for (u64 u = 0; u < n1; ++u)
      leaf_tft(e, cols, s_row, z2e, cols, base + u * cols * stride, stride, policy);
    if (n2 > 0) leaf_tft(e, cols, s_row, z2e, n2, base + n1 * cols * stride, stride, policy);
  }

  void leaf_itft(Emit& e, u64 L, SymExp s, u64 z, u64 n, int f, u64 base, u64 stride,
                 int policy) {
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
            e.push(OP_COPY, i, j, SymExp{}, true);
            e.P[j] = e.P[i] + s;
            if (fermat)
              e.P[i] = e.P[i] + SymExp{0, 1};
            else
              e.push(OP_DBL, i, i, SymExp{}, false);
          }
        } else {
          if (z == 2) {  // 2x0 - x1
            e.push(OP_SUB2, i, j, e.P[j] - e.P[i], true);
          } else {  // 2x0
            if (fermat)
              e.P[i] = e.P[i] + SymExp{0, 1};
            else
              e.push(OP_DBL, i, i, SymExp{}, false);
          }
        }
      } else {  // n == 0: half(x0 + x1) or half(x0)
        if (z == 2) {
          if (fermat) {
            e.push(OP_ADD, i, j, e.P[j] - e.P[i], true);
            e.P[i] = e.P[i] + SymExp{0, rs_.M - 1};
          } else {
            e.push(OP_ADDHALF, i, j, e.P[j] - e.P[i], true);
          }
        } else {
          if (fermat)
            e.P[i] = e.P[i] + SymExp{0, rs_.M - 1};
          else
            e.push(OP_HALF, i, i, SymExp{}, false);
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
    const SymExp s_row{s.a << l1, s.b << l1};
    for (u64 u = 0; u < n1; ++u)
      leaf_itft(e, cols, s_row, cols, cols, 0, base + u * cols * stride, stride, policy);
    for (u64 u = n2; u < hi; ++u)
      leaf_itft(e, rows, s + SymExp{0, u * col_step}, z1 + 1, n1, fm, base + u * stride,
                stride * cols, policy);
    for (u64 u = hi; u < z2e; ++u)
      leaf_itft(e, rows, s + SymExp{0, u * col_step}, z1, n1, fm, base + u * stride,
                stride * cols, policy);
    if (fm) leaf_itft(e, cols, s_row, z2e, n2, f, base + n1 * cols * stride, stride, policy);
    for (u64 u = 0; u < lo; ++u)
      leaf_itft(e, rows, s + SymExp{0, u * col_step}, z1 + 1, n1 + 1, 0, base + u * stride,
                stride * cols, policy);
    for (u64 u = lo; u < n2; ++u)
      leaf_itft(e, rows, s + SymExp{0, u * col_step}, z1, n1 + 1, 0, base + u * stride,
                stride * cols, policy);
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
    e.last.assign(L, 0);
    e.P.assign(L, SymExp{});
    if (k.inverse)
      leaf_itft(e, L, SymExp{1, 0}, k.z, k.n, k.f, 0, 1, policy);
    else
      leaf_tft(e, L, SymExp{1, 0}, k.z, k.n, 0, 1, policy);
    LeafProgram prog;
    prog.key = k;
    prog.nload = (u32)k.z;
    prog.nstore = (u32)(k.inverse ? k.n + (u64)k.f : k.n);
    u32 nlev = 0;
    for (auto& r : e.ops) nlev = std::max(nlev, r.level);
    std::stable_sort(e.ops.begin(), e.ops.end(),
                     [](const Emit::Raw& x, const Emit::Raw& y) { return x.level < y.level; });
    prog.level_begin.assign(nlev + 1, 0);
    prog.ops.reserve(e.ops.size());
    u32 cur = 1;
    for (size_t i = 0; i < e.ops.size(); ++i) {
      while (cur < e.ops[i].level) prog.level_begin[cur++] = (u32)i;
      prog.ops.push_back(e.ops[i].op);
    }
    while (cur <= nlev) prog.level_begin[cur++] = (u32)e.ops.size();
    prog.level_begin[0] = 0;
    // level_begin[l] = first op of level l+1; entry nlev = total
    std::vector<u32> lb(nlev + 1);
    // recompute cleanly: lb[i] = first op index with level > i
    size_t idx = 0;
    for (u32 l = 0; l <= nlev; ++l) {
      while (idx < e.ops.size() && e.ops[idx].level <= l) ++idx;
      lb[l] = (u32)idx;
    }
    // lb[0] = 0 (no op has level 0); level l (1-based) spans [lb[l-1], lb[l])
    prog.level_begin = std::move(lb);
    prog.store_rot.assign(e.P.begin(), e.P.begin() + prog.nstore);
    return prog;
  }

  RingShape rs_;
  std::map<ClassKey, u32> class_index_;
  std::vector<LeafProgram> classes_;
};

// ---------------------------------------------------------------------------
// Base-case counts of the REFERENCE recursion (policy at every level), by
// replay without arithmetic; memoised since counts are data independent
// (verify.hpp:459-483).
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
