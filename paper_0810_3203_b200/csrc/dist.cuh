// dist.cuh -- one transform partitioned over the GPUs of a box (SURVEY.md
// §8e): Bailey column slabs -> NCCL transpose -> row slabs, and back for the
// ITFT, as native host code over an NCCL communicator (the C ABI's
// cftft_gpu_dist_tft / cftft_gpu_dist_itft; paper_0810_3203_b200/dist.py is
// the same partition over torch.distributed, kept for the CPU (gloo) tests).
//
//   TFT  rank p: its columns [c0, c1) (balanced over L2) -> column TFTs
//        (transform.hpp:175-180, one batched launch) -> every rank q gets
//        rows R_q (a balanced split of the n1' active output rows) of p's
//        columns (grouped ncclSend / ncclRecv) -> unpack into the row slab ->
//        row TFTs (transform.hpp:182-185).
//   ITFT phase i on the row owners (transform.hpp:215-216) -> rows [0, z1')
//        back to the column owners (received straight into the column slab)
//        -> phase ii (right columns, :219-224) -> phase iii: row n1's right
//        part gathered to its owner, transformed, its left part scattered
//        back (:227-230) -> phase iv (left columns, :233-238).
//
// Slabs (elements of elem_stride_bytes): column slab [L1][W_p] (element
// (r, c) of the rank's columns at r W_p + c); row slab [R_p][L2].
// NCCL is loaded at run time (dlopen of libnccl.so.2: the process's own copy,
// e.g. torch's, when one is loaded), so the library has no link dependency.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <vector>

namespace cftft_b200 {
namespace dist {

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok() const { return h && GetUniqueId && CommInitRank && Send && Recv && GroupStart && GroupEnd; }
};

inline Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (n.h) {
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(n.h, "ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(n.h, "ncclCommInitRank"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(n.h, "ncclCommDestroy"));
      n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(n.h, "ncclGroupStart"));
      n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(n.h, "ncclGroupEnd"));
      n.Send = reinterpret_cast<decltype(n.Send)>(dlsym(n.h, "ncclSend"));
      n.Recv = reinterpret_cast<decltype(n.Recv)>(dlsym(n.h, "ncclRecv"));
      n.CommCount = reinterpret_cast<decltype(n.CommCount)>(dlsym(n.h, "ncclCommCount"));
      n.CommUserRank = reinterpret_cast<decltype(n.CommUserRank)>(dlsym(n.h, "ncclCommUserRank"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(n.h, "ncclGetErrorString"));
    }
  }
  return n;
}

inline void balanced(u64 total, u64 parts, u64 k, u64& lo, u64& hi) {
  const u64 q = total / parts, r = total % parts;
  lo = k * q + std::min(k, r);
  hi = lo + q + (k < r ? 1 : 0);
}

// Partition of one (L, z, n[, f]) transform (dist.py: DistGeometry)
struct Geometry {
  u64 M, L, z, n, world;
  unsigned l1, l2;
  u64 L1, L2, n1, n2, n1c, z1, z2, z2e, zrows, col_step, R;
  std::vector<u64> c0, c1, r0, r1;
  // wide: the ring runs radix-64 coset leaves (shape_of): columns of 64
  // coefficients (one radix-64 pass) and rows of L / 64 (the single-GPU
  // plan's own top split) instead of the balanced split
  Geometry(u64 M_, u64 L_, u64 z_, u64 n_, u64 world_, int policy, bool inverse, int f, bool wide = false)
      : M(M_), L(L_), z(z_), n(n_), world(world_) {
    unsigned ell = 0;
    while ((u64{1} << ell) < L) ++ell;
    l1 = policy ? 1 : (wide && ell >= 12) ? 6 : ell / 2;
    l2 = ell - l1;
    L1 = u64{1} << l1;
    L2 = u64{1} << l2;
    n2 = n & (L2 - 1);
    n1 = n >> l2;
    n1c = n1 + (n2 ? 1 : 0);
    z2 = z & (L2 - 1);
    z1 = z >> l2;
    z2e = z1 ? L2 : z2;
    col_step = M >> ell;
    zrows = z1 + (z2 ? 1 : 0);
    if (inverse) {
      const u64 fm = (n2 + (u64)f) > 0 ? 1 : 0;
      R = std::max(zrows, n1 + fm);
    } else {
      R = n1c;
    }
    c0.resize(world);
    c1.resize(world);
    r0.resize(world);
    r1.resize(world);
    for (u64 p = 0; p < world; ++p) {
      balanced(L2, world, p, c0[p], c1[p]);
      balanced(R, world, p, r0[p], r1[p]);
    }
  }
  u64 width(u64 p) const { return c1[p] - c0[p]; }
  u64 nrows(u64 p) const { return r1[p] - r0[p]; }
};

// ---- transpose schedules (pure host code: what cftft_gpu_dist_tft / _itft
// hand to NCCL, and what tests/test_dist.py replays over simulated ranks).
// One transpose = a few chunks; the pieces of a chunk form one NCCL group, in
// this order; piece = one row's columns of one rank, contiguous on both sides.
struct Piece {
  u64 send;   // 1: ncclSend, 0: ncclRecv
  u64 peer;
  u64 buf;    // 0: column slab, 1: row slab
  u64 off;    // element offset into the slab
  u64 count;  // elements
};
// chunks of the distributed TFT (chunk k's transpose overlaps chunk k+1's
// column pass): a few, each still a machine's worth of columns; the same on
// every rank
inline u64 tft_chunks(const Geometry& g) { return std::max<u64>(1, std::min<u64>(4, (g.L2 / g.world) / 256)); }
// rank p's columns of chunk k: [a, b) of its slab
inline void tft_chunk_cols(const Geometry& g, u64 p, u64 k, u64& a, u64& b) {
  const u64 K = tft_chunks(g), W = g.width(p);
  a = W * k / K;
  b = W * (k + 1) / K;
}
// TFT: row r of R_q, my chunk's columns -> rank q, straight into q's row slab
inline std::vector<Piece> tft_transpose(const Geometry& g, u64 me, u64 k) {
  std::vector<Piece> v;
  const u64 W = g.width(me), nr = g.nrows(me);
  u64 a, b;
  tft_chunk_cols(g, me, k, a, b);
  for (u64 q = 0; q < g.world; ++q) {
    u64 qa, qb;
    tft_chunk_cols(g, q, k, qa, qb);
    for (u64 r = g.r0[q]; r < g.r1[q] && b > a; ++r) v.push_back(Piece{1, q, 0, r * W + a, b - a});
    for (u64 r = 0; r < nr && qb > qa; ++r) v.push_back(Piece{0, q, 1, r * g.L2 + g.c0[q] + qa, qb - qa});
  }
  return v;
}
// ITFT: rows [0, zrows) to the column owners, in chunks of rows; every rank
// cuts every rank's rows [r0_q, min(r1_q, zrows)) the same way
inline u64 itft_chunks(const Geometry& g) {
  u64 K = 1;
  for (u64 q = 0; q < g.world; ++q) {
    const u64 m = g.r0[q] < g.zrows ? std::min(g.r1[q], g.zrows) - g.r0[q] : 0;
    K = std::max(K, std::min<u64>(4, m));
  }
  return K;
}
inline void itft_chunk_rows(const Geometry& g, u64 q, u64 k, u64& a, u64& b) {  // global rows
  const u64 K = itft_chunks(g), lo = g.r0[q], m = lo < g.zrows ? std::min(g.r1[q], g.zrows) - lo : 0;
  a = lo + m * k / K;
  b = lo + m * (k + 1) / K;
}
inline std::vector<Piece> itft_transpose(const Geometry& g, u64 me, u64 k) {
  std::vector<Piece> v;
  const u64 W = g.width(me);
  u64 a, b;
  itft_chunk_rows(g, me, k, a, b);
  for (u64 q = 0; q < g.world; ++q) {
    u64 qa, qb;
    itft_chunk_rows(g, q, k, qa, qb);
    for (u64 u = a; u < b && g.width(q); ++u)
      v.push_back(Piece{1, q, 1, (u - g.r0[me]) * g.L2 + g.c0[q], g.width(q)});
    for (u64 u = qa; u < qb && W; ++u) v.push_back(Piece{0, q, 0, u * W, W});
  }
  return v;
}

}  // namespace dist
}  // namespace cftft_b200
