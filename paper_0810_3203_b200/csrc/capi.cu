// capi.cu -- the C ABI (include/cftft_b200.h) over the planner and the
// sm_100a leaf kernels.  Host C++; no torch types anywhere.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <atomic>
#include <sstream>
#include <thread>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/cftft_b200.h"
#include "fermat_leaf.cuh"
#include "negacyclic_leaf.cuh"
#include "prime_leaf.cuh"
#include "pointwise.cuh"
#include "polymul.cuh"
#include "dist.cuh"
#include "wave_coset.cuh"
#include "wave_wide.cuh"
#include "wave_tma.cuh"
#include "planner.hpp"

using namespace cftft_b200;

namespace {

thread_local std::string g_last_error;
std::atomic<int> g_fault{0};   // cftft_set_fault_injection
thread_local int t_sm_reserve = 0;  // SMs the wave launches leave free (set by the multi-GPU transforms)
std::atomic<int> g_timing{0};  // cftft_set_launch_timing
// Launch timing (cftft_set_launch_timing): CUDA events on the launching
// stream around each kernel of the transforms, with the launch's algorithmic
// bytes (coefficients read + written x information bytes per coefficient).
struct TimedLaunch {
  const char* kernel;
  u64 bytes;
  cudaEvent_t e0, e1;
};
thread_local std::vector<TimedLaunch> g_timed;
thread_local std::vector<cudaEvent_t> g_event_pool;
cudaEvent_t pooled_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
// RAII around one launch; a no-op unless timing is on
struct LaunchTimer {
  cudaStream_t st;
  bool on;
  TimedLaunch rec{};
  LaunchTimer(const char* kernel, u64 bytes, cudaStream_t s) : st(s), on(g_timing.load() != 0) {
    if (!on) return;
    rec.kernel = kernel;
    rec.bytes = bytes;
    rec.e0 = pooled_event();
    rec.e1 = pooled_event();
    cudaEventRecord(rec.e0, st);
  }
  ~LaunchTimer() {
    if (!on) return;
    cudaEventRecord(rec.e1, st);
    g_timed.push_back(rec);
  }
};
std::atomic<int> g_poison{0};  // cftft_set_debug_poison

// Experiment knobs (phase clocks, debug skips) exist only in builds with
// -DCFTFT_EXPERIMENTS; the shipped library reads no environment variables.
#ifdef CFTFT_EXPERIMENTS
int env_int(const char* k, int dflt) {
  const char* v = getenv(k);
  return v ? atoi(v) : dflt;
}
#else
int env_int(const char*, int dflt) { return dflt; }
#endif
thread_local u64 g_last_launches = 0;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(CFTFT_CUDA_ERROR, std::string(#expr ": ") + cudaGetErrorString(e_));    \
  } while (0)

constexpr size_t kSmemBudget = 196 * 1024;
constexpr size_t kMaxBatchPlans = 64;  // per-CTA dynamic shared memory for leaf slots
// Fermat carry scratch: one int per (thread x task) of a store batch
inline size_t scratch_bytes(u32 nt) { return (size_t)nt * 4; }

// A plan resident on one device.
struct DevicePlan {
  Plan host;
  void* dbuf = nullptr;
  const DevClass* classes = nullptr;
  const DevOp* ops = nullptr;
  const u32* levels = nullptr;
  const SymExp* rots = nullptr;
  const DevLeaf* leaves = nullptr;
  const DevCounter* cmeta = nullptr;
  const u64* locbits = nullptr;
  const u64* shadow_finals = nullptr;
  const u64* fold_list = nullptr;
  const u32* groups = nullptr;
  const u32* wave_ops = nullptr;
  const u32* wave_slots = nullptr;
  const u32* final_rot = nullptr;
  // per wave: 1 (DIF) / 2 (DIT) when every leaf is a radix-64 network class
  // of that kind the TMA kernel runs
  std::vector<std::uint8_t> tma_wave;
  std::vector<std::uint8_t> tma_aligned;  // per wave: no loaded slot has a sub-lane pre-rotation
  std::vector<u64> tma_desc_off;  // per wave: first descriptor in tma_descs
  void* tma_descs = nullptr;      // fermat::TmaLeafDesc per leaf of the TMA waves
  std::uint8_t* tma_lay = nullptr;  // coset-major layout bits per wave_slots entry (inside tma_descs)
  u32 tma_step = 0;
  std::vector<u64> batch_items;  // batch plans: the items, compared on a cache hit
  std::vector<u64> wave_loads;   // per wave: coefficients read + written by its leaves (launch timing)
  bool tma_cm_finals = false;  // every shadow-buffer final is written coset-major by a TMA wave
  u64 nleaves = 0;
  u32 ncounters = 0;
  unsigned max_ell = 0;
  // Fermat geometry of this plan: chunk (lane) width, chunks per element,
  // whole-leaf slot bytes, tops-array interleave
  u32 cw = 16, C = 0, slot_bytes = 0, logS = 0;
  u64* prime_ntw = nullptr;  // prime rings: network classes' butterfly twiddles (prime::Args::ntw)
  ~DevicePlan() {
    if (dbuf) cudaFree(dbuf);
    if (tma_descs) cudaFree(tma_descs);
    if (prime_ntw) cudaFree(prime_ntw);
  }
};

using PlanKey = std::tuple<int, int, u64, u64, u64, u64, int, int>;  // dev, inv, L, s, z, n, f, policy

}  // namespace

struct cftft_ring {
  int kind = 0;
  int coset_cw = -1;          // Fermat coset leaves: -1 auto, 0 off, 4/8/16 lane words
  int wide = -1;              // radix-64 coset leaves: -1 default (on), 0 off, 1 on (network waves on the
                              // TMA-wave kernel, the other radix-64 waves on coset_wide_kernel)
  unsigned leaf_limit = 0;    // cftft_ring_set_leaf_limit (0: none)
  u64 N = 0, K = 0, m = 0, M = 0;
  u32 D = 0, C = 0;     // Fermat: u32 words / chunks of CW words
  u32 CW = 16;
  u32 NT = 512;  // Fermat CTA size: 512 (1 CTA/SM) or 256 (2 CTAs/SM, half-size leaves)
  u32 slot_bytes = 0;   // shared-memory bytes per slot
  u64 elem_bytes = 0;   // minimal element stride
  unsigned max_leaf_ell = 1;
  unsigned max_leaf_fit = 1;
  std::mutex mu;
  std::map<PlanKey, std::unique_ptr<DevicePlan>> cache;
  // NTT twiddle tables of the Fermat pointwise multiplier (pointwise.cuh)
  u32* ntt_tw = nullptr;
  // prime rings: p (in m), -p^-1 mod 2^64, omega, two-level Montgomery tables
  u64 pinv = 0, omega = 0;
  u32 lo_bits = 0;
  u64* prime_tw = nullptr;  // [2^lo_bits] omega^i R, then [M / 2^lo_bits] omega^(i 2^lo_bits) R
  // staging buffer for the host-view entry points; stage_mu is held for a
  // whole host call (copy in, transform, copy out)
  std::mutex stage_mu;
  void* stage = nullptr;
  size_t stage_bytes = 0;
  // coset-plan scratch (shadow buffer, tops arrays), one per stream: reused
  // across launches on that stream (stream order makes reuse safe; a
  // stream-ordered pool allocation of 4 GB can cost the host tens of ms)
  struct Scratch {
    int dev = -1;
    void* stream = nullptr;
    std::thread::id thread;  // the default-stream handles (0, per-thread) name a different stream per thread
    void* shadow = nullptr;
    size_t shadow_bytes = 0;
    void* tops = nullptr;
    size_t tops_bytes = 0;
  };
  std::vector<Scratch> scratch;
  CountReplay counts;
  ~cftft_ring() {
    if (stage) cudaFree(stage);
    if (ntt_tw) cudaFree(ntt_tw);
    if (prime_tw) cudaFree(prime_tw);
    for (auto& sc : scratch) {
      if (sc.shadow) cudaFree(sc.shadow);
      if (sc.tops) cudaFree(sc.tops);
    }
  }
};

namespace {

// Prime rings: 1 (DIF, spans L/2 .. 1) / 2 (DIT, spans 1 .. L/2) when the
// class is the full radix-2 network of ADDSUB butterflies in level order --
// truncated TFT programs qualify when the network on zero-filled missing
// inputs reproduces every stored output (checked by evaluating both mod p on
// random inputs; a COPY is a butterfly with a zero b, an ADD one whose
// difference nothing reads) -- else 0.  `tw` gets
// omega^r 2^64 mod p per butterfly (level l, index j) at l L/2 + j, 0 for r = 0.
u32 prime_network(const LeafProgram& cl, u64 p, u64 omega, std::vector<u64>& tw) {
  const u32 ell = cl.key.ell;
  if (ell < 3 || cl.ops.empty() || cl.nload == 0) return 0;
  const u32 L = 1u << ell, half = L / 2;
  auto mulp = [p](u64 a, u64 b) { return (u64)((unsigned __int128)a * b % p); };
  auto powp = [&](u64 a, u64 e) {
    u64 r = 1 % p;
    for (; e; e >>= 1, a = mulp(a, a))
      if (e & 1) r = mulp(r, a);
    return r;
  };
  auto addm = [p](u64 a, u64 b) { return (u64)(((unsigned __int128)a + b) % p); };
  auto subm = [p](u64 a, u64 b) { return a >= b ? a - b : (u64)((unsigned __int128)a + p - b); };
  for (u32 kind = 1; kind <= 2; ++kind) {
    std::vector<long long> qn((size_t)ell * half, -1);
    std::vector<int> last(L, -1);
    bool ok = true;
    for (const DevOp& op : cl.ops) {
      const u32 a = op.a, b = op.b, h = b - a;
      if ((op.type != OP_ADDSUB && op.type != OP_COPY && op.type != OP_ADD) || b <= a || b >= L || (h & (h - 1)) ||
          (a & h)) {
        ok = false;
        break;
      }
      const int lh = __builtin_ctz(h);
      const int lvl = kind == 1 ? (int)ell - 1 - lh : lh;
      if (last[a] >= lvl || last[b] >= lvl) {
        ok = false;
        break;
      }
      last[a] = last[b] = lvl;
      qn[(size_t)lvl * half + (a / (2 * h)) * h + a % h] = op.type == OP_COPY ? 0 : (long long)op.r;
    }
    if (!ok) continue;
    std::vector<u64> x(L, 0), y;
    u64 seed = 0x9E3779B97F4A7C15ull ^ (cl.key.z * 131 + cl.key.n * 7 + kind);
    for (u32 k = 0; k < cl.nload; ++k) {
      seed = seed * 6364136223846793005ull + 1442695040888963407ull;
      x[k] = (seed >> 1) % p;
    }
    y = x;
    for (const DevOp& op : cl.ops) {
      if (op.type == OP_COPY) {
        x[op.b] = x[op.a];
        continue;
      }
      const u64 t = mulp(x[op.b], powp(omega, op.r)), u = x[op.a];
      x[op.a] = addm(u, t);
      if (op.type == OP_ADDSUB) x[op.b] = subm(u, t);
    }
    for (u32 lvl = 0; lvl < ell; ++lvl) {
      const u32 h = kind == 1 ? (L >> (lvl + 1)) : (1u << lvl);
      for (u32 j = 0; j < half; ++j) {
        const u32 a = (j / h) * 2 * h + j % h;
        const long long q = qn[(size_t)lvl * half + j];
        const u64 t = q > 0 ? mulp(y[a + h], powp(omega, (u64)q)) : y[a + h], u = y[a];
        y[a] = addm(u, t);
        y[a + h] = subm(u, t);
      }
    }
    for (u32 k = 0; k < cl.nstore && ok; ++k) ok = x[k] == y[k];
    if (!ok) continue;
    const u64 Rm = (u64)(((unsigned __int128)1 << 64) % p);
    const size_t off = tw.size();
    tw.resize(off + (size_t)ell * half, 0);
    for (size_t i = 0; i < (size_t)ell * half; ++i)
      if (qn[i] > 0) tw[off + i] = mulp(powp(omega, (u64)qn[i]), Rm);
    return kind;
  }
  return 0;
}

int upload(cftft_ring* R, DevicePlan& dp, cudaStream_t st) {
  const Plan& p = dp.host;
  std::vector<DevClass> cls;
  std::vector<DevOp> ops;
  std::vector<u32> levels;
  std::vector<SymExp> rots;
  std::vector<u64> ntw;  // prime network twiddles
  for (const auto& c : p.classes) {
    DevClass d{};
    d.L = 1u << c.key.ell;
    d.nload = c.nload;
    d.nstore = c.nstore;
    d.nlevels = (u32)c.level_begin.size() - 1;
    d.level_begin = (u32)levels.size();
    u32 op0 = (u32)ops.size();
    d.op_begin = op0;
    d.nops = (u32)c.ops.size();
    for (u32 x : c.level_begin) levels.push_back(op0 + x);
    ops.insert(ops.end(), c.ops.begin(), c.ops.end());
    d.pre_begin = (u32)rots.size();
    rots.insert(rots.end(), c.pre.begin(), c.pre.end());
    d.post_begin = (u32)rots.size();
    rots.insert(rots.end(), c.post.begin(), c.post.end());
    d.has_pre = c.has_pre ? 1 : 0;
    d.kind = c.kind;
    d.cs = c.cs ? c.cs : dp.C;
    d.m = c.m;
    d.step = c.step;
    d.slot_bytes = c.slot_bytes ? c.slot_bytes : dp.slot_bytes;
    d.inverse = (u32)c.key.inverse;
    d.spec_n = c.key.inverse ? (u32)c.key.n : 0;
    d.fslot = (c.key.inverse && c.key.f) ? (u32)c.key.n : 0xFFFFFFFFu;
    d.wop_begin = cls.size() < p.wave_op_begin.size() ? p.wave_op_begin[cls.size()] : 0;
    d.wnet = cls.size() < p.wave_net.size() ? p.wave_net[cls.size()] : 0;
    if (R->kind == CFTFT_RING_PRIME) {
      const size_t off = ntw.size();
      d.wnet = prime_network(c, R->m, R->omega, ntw);
      d.wop_begin = (u32)off;
    }
    cls.push_back(d);
  }
  if (!ntw.empty()) {
    CUDA_TRY(cudaMalloc(&dp.prime_ntw, ntw.size() * sizeof(u64)));
    CUDA_TRY(cudaMemcpyAsync(dp.prime_ntw, ntw.data(), ntw.size() * sizeof(u64), cudaMemcpyHostToDevice, st));
  }
  if (R->kind == CFTFT_RING_PRIME) {
    // each op's omega^r in Montgomery form (times 2^64 mod p): one product
    // per butterfly on the GPU instead of two table lookups and two products
    const u64 pm = R->m;
    auto mulp = [pm](u64 a, u64 b) { return (u64)((unsigned __int128)a * b % pm); };
    const u64 Rm = (u64)(((unsigned __int128)1 << 64) % pm);
    for (auto& op : ops) {
      u64 r = 1 % pm, a = R->omega, e = op.r;
      for (; e; e >>= 1, a = mulp(a, a))
        if (e & 1) r = mulp(r, a);
      op.pad2 = mulp(r, Rm);
    }
  }
  if (rots.empty()) rots.push_back(SymExp{});
  if (levels.empty()) levels.push_back(0);
  if (ops.empty()) ops.push_back(DevOp{});
  const auto& leaves = p.leaves;
  dp.nleaves = leaves.size();
  dp.ncounters = (u32)p.counters.size();
  std::vector<DevCounter> cm = p.counters;
  if (cm.empty()) cm.push_back(DevCounter{0, kNoDep});
  dp.max_ell = p.max_ell;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t o_cls = 0, o_ops = al(o_cls + cls.size() * sizeof(DevClass));
  size_t o_lev = al(o_ops + ops.size() * sizeof(DevOp));
  size_t o_rot = al(o_lev + levels.size() * sizeof(u32));
  size_t o_lf = al(o_rot + rots.size() * sizeof(SymExp));
  size_t o_cm = al(o_lf + leaves.size() * sizeof(DevLeaf));
  size_t o_lb = al(o_cm + cm.size() * sizeof(DevCounter));
  size_t o_sf = al(o_lb + p.locbits.size() * sizeof(u64));
  size_t o_fl = al(o_sf + p.shadow_finals.size() * sizeof(u64));
  size_t o_gr = al(o_fl + p.fold_list.size() * sizeof(u64));
  size_t o_wo = al(o_gr + p.groups.size() * sizeof(u32));
  size_t o_ws = al(o_wo + p.wave_ops.size() * sizeof(u32));
  size_t o_fr = al(o_ws + p.wave_slots.size() * sizeof(u32));
  size_t total = al(o_fr + p.final_rot.size() * sizeof(u32)) + 256;
  std::vector<std::uint8_t> h(total, 0);
  std::memcpy(h.data() + o_cls, cls.data(), cls.size() * sizeof(DevClass));
  std::memcpy(h.data() + o_ops, ops.data(), ops.size() * sizeof(DevOp));
  std::memcpy(h.data() + o_lev, levels.data(), levels.size() * sizeof(u32));
  std::memcpy(h.data() + o_rot, rots.data(), rots.size() * sizeof(SymExp));
  std::memcpy(h.data() + o_lf, leaves.data(), leaves.size() * sizeof(DevLeaf));
  std::memcpy(h.data() + o_cm, cm.data(), cm.size() * sizeof(DevCounter));
  if (!p.locbits.empty()) std::memcpy(h.data() + o_lb, p.locbits.data(), p.locbits.size() * sizeof(u64));
  if (!p.shadow_finals.empty())
    std::memcpy(h.data() + o_sf, p.shadow_finals.data(), p.shadow_finals.size() * sizeof(u64));
  if (!p.fold_list.empty()) std::memcpy(h.data() + o_fl, p.fold_list.data(), p.fold_list.size() * sizeof(u64));
  if (!p.groups.empty()) std::memcpy(h.data() + o_gr, p.groups.data(), p.groups.size() * sizeof(u32));
  if (!p.wave_ops.empty()) std::memcpy(h.data() + o_wo, p.wave_ops.data(), p.wave_ops.size() * sizeof(u32));
  if (!p.wave_slots.empty()) std::memcpy(h.data() + o_ws, p.wave_slots.data(), p.wave_slots.size() * sizeof(u32));
  if (!p.final_rot.empty()) std::memcpy(h.data() + o_fr, p.final_rot.data(), p.final_rot.size() * sizeof(u32));
  CUDA_TRY(cudaMalloc(&dp.dbuf, total));
  CUDA_TRY(cudaMemcpyAsync(dp.dbuf, h.data(), total, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));  // h is a temporary
  auto* b = static_cast<std::uint8_t*>(dp.dbuf);
  dp.classes = reinterpret_cast<const DevClass*>(b + o_cls);
  dp.ops = reinterpret_cast<const DevOp*>(b + o_ops);
  dp.levels = reinterpret_cast<const u32*>(b + o_lev);
  dp.rots = reinterpret_cast<const SymExp*>(b + o_rot);
  dp.leaves = reinterpret_cast<const DevLeaf*>(b + o_lf);
  dp.cmeta = reinterpret_cast<const DevCounter*>(b + o_cm);
  dp.locbits = reinterpret_cast<const u64*>(b + o_lb);
  dp.shadow_finals = reinterpret_cast<const u64*>(b + o_sf);
  dp.fold_list = reinterpret_cast<const u64*>(b + o_fl);
  dp.groups = p.groups.empty() ? nullptr : reinterpret_cast<const u32*>(b + o_gr);
  dp.wave_ops = reinterpret_cast<const u32*>(b + o_wo);
  dp.wave_slots = reinterpret_cast<const u32*>(b + o_ws);
  dp.final_rot = p.final_rot.empty() ? nullptr : reinterpret_cast<const u32*>(b + o_fr);
  // radix-64 network waves on the TMA kernel (wave_tma.cuh): 64-slot full
  // networks over 256-bit lanes with at least two cosets, one item per coset,
  // stage-A rotations only where the kernel's compile-time mask has them
  dp.wave_loads.assign(p.waves.size(), 0);
  for (size_t w = 0; w < p.waves.size(); ++w)
    for (u64 i = p.waves[w][0]; i < p.waves[w][0] + p.waves[w][1]; ++i)
      dp.wave_loads[w] += (u64)cls[p.leaves[i].cls].nload + cls[p.leaves[i].cls].nstore;
  dp.tma_wave.assign(p.waves.size(), 0);
  dp.tma_aligned.assign(p.waves.size(), 0);
  std::vector<fermat::TmaLeafDesc> descs;
  dp.tma_desc_off.assign(p.waves.size(), 0);
  for (size_t w = 0; w < p.waves.size(); ++w) {
    const auto& wr = p.waves[w];
    if (wr[2] != 2 || !wr[1]) continue;
    bool ok = true;
    u32 step = 0, wnet = 0;
    auto is_prog = [&](u32 ci) {
      return cls[ci].wnet == 0 && ci < p.wave_prog.size() && p.wave_prog[ci] != kNoDep;
    };
    for (u64 i = wr[0]; i < wr[0] + wr[1] && ok; ++i) {
      const u32 ci = p.leaves[i].cls;
      const DevClass& d = cls[ci];
      const bool prog = is_prog(ci);
      ok = d.L == 64 && (d.wnet == 1 || d.wnet == 2 || prog) && d.kind == 1 && d.step >= 2 &&
           (d.step & (d.step - 1)) == 0 && (step == 0 || d.step == step) && wr[3] == d.step &&
           (prog || wnet == 0 || d.wnet == wnet);
      step = d.step;
      if (!ok) break;
      if (prog) continue;  // phase programs run in either kernel
      wnet = d.wnet;
      const u32 mask = d.wnet == 1 ? fermat::kRotDif : fermat::kRotDit;
      for (u32 o = 0; o < 192 && ok; ++o) {
        const u32 wop = p.wave_ops[d.wop_begin + o];
        if ((wop & 15u) != OP_ADDSUB) ok = false;
        if (o < 96 && !((mask >> (o % 12)) & 1u) && (wop >> 16) != 0) ok = false;
      }
    }
    if (!ok) continue;
    // bits 0-1: the kernel's network kind (programs only: DIT); bit 2: phase programs
    bool any_prog = false;
    for (u64 i = wr[0]; i < wr[0] + wr[1]; ++i) any_prog = any_prog || is_prog(p.leaves[i].cls);
    dp.tma_wave[w] = (std::uint8_t)((wnet ? wnet : 2u) | (any_prog ? 4u : 0u));
    dp.tma_step = step;
    dp.tma_desc_off[w] = descs.size();
    dp.tma_aligned[w] = 1;
    for (u64 i = wr[0]; i < wr[0] + wr[1]; ++i) {
      const DevLeaf& lf = p.leaves[i];
      const DevClass& d = cls[lf.cls];
      const bool prog = is_prog(lf.cls);
      for (u32 k = 0; k < d.nload; ++k)
        if (p.wave_slots[lf.c0 + 2ull * k] & 255u) dp.tma_aligned[w] = 0;
      fermat::TmaLeafDesc td{};
      td.base = lf.base;
      td.stride = lf.stride;
      td.c0 = lf.c0;
      td.wop_begin = prog ? p.wave_prog[lf.cls] : d.wop_begin;
      td.nload = d.nload;
      td.nstore_wnet = d.nstore | ((prog ? 3u : d.wnet) << 16);
      descs.push_back(td);
    }
  }
  if (!descs.empty()) {
    // Coset-major intermediate layout: an element written by a TMA wave whose
    // every later read (until it is written again) is by a TMA wave is stored
    // coset by coset (coset k = lanes k + step * pos, pos = 0..31, as one 1 KB
    // chunk), so each slot's coset moves as one bulk copy; everything else --
    // inputs, outputs, whatever another kernel or the fold reads -- keeps the
    // natural lane order.  Per slot entry of wave_slots: bit 0 the input is
    // coset-major, bit 1 the output is.
    std::vector<std::uint8_t> lay(p.wave_slots.size(), 0);
    struct Ev {
      u32 wave;
      bool tma, rd, wr;
      u64 slot;  // index into wave_slots (TMA waves)
    };
    std::vector<std::vector<Ev>> ev(p.extent);
    for (size_t w = 0; w < p.waves.size(); ++w) {
      const auto& wr = p.waves[w];
      for (u64 i = wr[0]; i < wr[0] + wr[1]; ++i) {
        const DevLeaf& lf = p.leaves[i];
        const LeafProgram& c = p.classes[lf.cls];
        const u32 span = std::max(c.nload, c.nstore);
        for (u32 k = 0; k < span; ++k) {
          const u64 e = lf.base + (u64)k * lf.stride;
          if (e >= ev.size()) continue;
          ev[e].push_back(Ev{(u32)w, dp.tma_wave[w] != 0, k < c.nload, k < c.nstore, (u64)lf.c0 + 2ull * k});
        }
      }
    }
    // A final output left in the shadow buffer is folded from there into the
    // caller's view by cs_fold_kernel, which can read it coset by coset: when
    // every such output's last writer is a TMA wave, those writes are
    // coset-major too (whole 1 KB chunks instead of 32-byte pieces).
    std::vector<std::uint8_t> shfin(p.extent, 0);
    if (p.use_fold_list)
      for (u64 e : p.shadow_finals)
        if (e < shfin.size()) shfin[e] = 1;
    std::vector<u64> cm_final_slots;
    bool cm_all = p.use_fold_list && !p.shadow_finals.empty();
    for (u64 e = 0; e < ev.size(); ++e) {
      auto& es = ev[e];
      std::uint8_t cur = 0;
      for (size_t a = 0; a < es.size(); ++a) {
        const Ev& x = es[a];
        if (x.rd && x.tma) lay[x.slot] |= cur;
        if (!x.wr) continue;
        std::uint8_t out = 0;
        bool last = true;
        for (size_t b = a + 1; b < es.size(); ++b)
          if (es[b].wr) last = false;
        if (x.tma) {
          bool any = false, all = true;
          for (size_t b = a + 1; b < es.size(); ++b) {
            if (es[b].rd) {
              any = true;
              all = all && es[b].tma;
            }
            if (es[b].wr) break;
          }
          out = (any && all) ? 1 : 0;
          if (!any && last && shfin[e] && (p.wave_slots[x.slot + 1] >> 31)) {
            out = 1;
            cm_final_slots.push_back(x.slot);
          }
          lay[x.slot] |= (std::uint8_t)(out << 1);
        }
        if (last && shfin[e] && !(x.tma && out)) cm_all = false;
        cur = out;
      }
    }
    if (!cm_all)
      for (u64 sl : cm_final_slots) lay[sl] &= (std::uint8_t)~2u;
    dp.tma_cm_finals = cm_all;
    CUDA_TRY(cudaMalloc(&dp.tma_descs, descs.size() * sizeof(fermat::TmaLeafDesc) + lay.size()));
    CUDA_TRY(cudaMemcpyAsync(dp.tma_descs, descs.data(), descs.size() * sizeof(fermat::TmaLeafDesc),
                             cudaMemcpyHostToDevice, st));
    dp.tma_lay = static_cast<std::uint8_t*>(dp.tma_descs) + descs.size() * sizeof(fermat::TmaLeafDesc);
    CUDA_TRY(cudaMemcpyAsync(dp.tma_lay, lay.data(), lay.size(), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  (void)R;
  return CFTFT_OK;
}

// Planning geometry of one transform of length L.  Fermat: coset leaves use
// lanes of `cw` words, chosen so that the reference's top-level split yields
// sub-transforms whose internal rotations are whole lanes (M / sqrt(L) bits).
// allow_wide = false: radix-8 waves only
RingShape shape_of(const cftft_ring* R, u64 L, DevicePlan* dp, bool allow_wide = true) {
  RingShape rs;
  rs.fermat = (R->kind == CFTFT_RING_FERMAT);
  if (R->kind == CFTFT_RING_PRIME) rs.group = 16;  // adjacent u64 coefficients per ticket
  rs.M = R->M;
  rs.max_leaf_ell = R->max_leaf_ell;
  rs.elem_bytes = R->elem_bytes;
  u32 cw = R->CW, C = R->C, sb = R->slot_bytes;
  if (rs.fermat) {
    const bool on = R->coset_cw > 0 || (R->coset_cw < 0 && R->N >= 4096 && R->NT == 512);
    if (on && L >= 4) {
      if (R->coset_cw > 0) {
        cw = (u32)R->coset_cw;
      } else {
        const unsigned ell = (unsigned)__builtin_ctzll(L);
        const u64 lnode = u64{1} << (ell - ell / 2);
        u64 lane = R->M / lnode;
        // lanes of <= 8 words keep a 64-coefficient coset ticket within one of
        // the two ticket buffers
        cw = (u32)std::min<u64>(8, std::max<u64>(4, lane / 32));
      }
      if (cw > R->D) cw = R->D;
      while (R->D / cw > 512 && cw < 16) cw *= 2;  // a CTA covers one chunk per thread of a coefficient
      C = R->D / cw;
      sb = fermat_slot_bytes(C, 4 * cw);
      const size_t budget = kSmemBudget - scratch_bytes(1024);
      unsigned lam = 1;
      while (lam < 10 && ((size_t)sb << (lam + 1)) <= budget) ++lam;
      if (R->leaf_limit) lam = std::min(lam, R->leaf_limit);
      rs.max_leaf_ell = lam;
      rs.lane_bits = 32ull * cw;
      rs.slot_budget = budget;
      // per-ticket fixed costs outweigh the overlap two half-size buffers
      // would buy: coset tickets fill the shared memory
      rs.ticket_budget = budget;
      unsigned cl = 0;
      for (unsigned e = 1; e <= 6; ++e) {
        const u64 cs = u64{1} << (e - 1);
        const u64 slot = fermat_slot_bytes(cs, 4 * cw);
        if ((u64{1} << e) <= 2ull * C && (u64{1} << e) * slot <= budget / 2) cl = e;
      }
      if (R->leaf_limit) cl = std::min(cl, std::max(1u, R->leaf_limit));
      if (cw == 8) {
        rs.wave_engine = true;
        rs.wave_unaligned = true;
        // radix-64 coset leaves (default: their full-network waves run on the
        // TMA-wave kernel, wave_tma.cuh; set_wide(0): radix-8 warp waves only)
        const int wide = !allow_wide ? 0 : (R->wide >= 0 ? R->wide : 1);
        rs.wide = wide != 0 && cl >= 6 && (R->M >> 6) % rs.lane_bits == 0;
        cl = std::min(cl, rs.wide ? 6u : 3u);
        rs.max_leaf_ell = std::min(rs.max_leaf_ell, 3u);
      }
      rs.coset_max_ell = cl;
      if (!cl) rs.lane_bits = 0;
    }
    // whole-coefficient plans (small N): leaves of <= 64 coefficients, so the
    // Bailey phases spread over many CTAs instead of one CTA walking every
    // level of a transform that happens to fit its shared memory (C1: TFT +
    // ITFT 256 -> 163 us)
    if (!rs.lane_bits && !R->leaf_limit) rs.max_leaf_ell = std::min(rs.max_leaf_ell, 6u);
  }
  rs.C = C;
  rs.slot_bytes = sb;
  if (dp) {
    dp->cw = cw;
    dp->C = C;
    dp->slot_bytes = sb;
    u32 logS = 0;
    if (rs.lane_bits && (!rs.wave_engine || rs.wide)) {
      // the lanes of one coset of the largest coset leaves are contiguous in
      // the tops arrays (wide plans: one coset per warp row)
      const u64 S = std::max<u64>(1, (2ull * C) >> rs.coset_max_ell);
      logS = (u32)__builtin_ctzll(S);
    }
    dp->logS = logS;
  }
  return rs;
}

template <class F>
Plan best_plan(const RingShape& rs, F build) {
  Planner pa(rs);
  return build(pa);
}

int get_plan(cftft_ring* R, bool inv, const cftft_params& p, int policy, cudaStream_t st,
             DevicePlan** out) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  PlanKey key{dev, inv ? 1 : 0, p.length, p.twiddle_exp & (R->M - 1), p.input_count,
              p.output_count, inv ? p.want_next : 0, policy};
  std::lock_guard<std::mutex> g(R->mu);
  auto it = R->cache.find(key);
  if (it != R->cache.end()) {
    *out = it->second.get();
    return CFTFT_OK;
  }
  auto dp = std::make_unique<DevicePlan>();
  const RingShape rs = shape_of(R, p.length, dp.get());
  try {
    dp->host = best_plan(rs, [&](Planner& pl) {
      return pl.build(inv, p.length, p.twiddle_exp, p.input_count, p.output_count, inv ? p.want_next : 0,
                      policy);
    });
  } catch (const std::exception& ex) {
    return fail(CFTFT_UNSUPPORTED, ex.what());
  }
  int rc = upload(R, *dp, st);
  if (rc) return rc;
  *out = dp.get();
  R->cache[key] = std::move(dp);
  return CFTFT_OK;
}

int validate(const cftft_ring* R, bool inv, const cftft_params* p, int policy) {
  if (!R || !p) return fail(CFTFT_INVALID_PARAMS, "null ring or params");
  const u64 L = p->length;
  if (L < 2 || (L & (L - 1)) != 0 || L > R->M)  // transform.hpp:241-243
    return fail(CFTFT_BAD_LENGTH, "transform length " + std::to_string(L) +
                                      " is not a power of two dividing the root order");
  if (policy != CFTFT_BALANCED && policy != CFTFT_RADIX2)
    return fail(CFTFT_INVALID_PARAMS, "unknown split policy");
  if (!inv) {  // transform.hpp:255-259
    if (p->input_count < 1 || p->input_count > L || p->output_count < 1 || p->output_count > L)
      return fail(CFTFT_INVALID_PARAMS, "tft requires 1 <= z <= L and 1 <= n <= L");
    if (p->want_next != 0) return fail(CFTFT_INVALID_PARAMS, "the forward transform takes no f flag");
  } else {  // transform.hpp:276-281
    if (p->want_next != 0 && p->want_next != 1) return fail(CFTFT_INVALID_PARAMS, "f must be 0 or 1");
    const u64 nf = p->output_count + (u64)p->want_next;
    if (p->input_count < 1 || p->input_count > L || nf < 1 || nf > L ||
        p->input_count < p->output_count)
      return fail(CFTFT_INVALID_PARAMS, "itft requires 1 <= z <= L, 1 <= n+f <= L and z >= n");
  }
  return CFTFT_OK;
}

int check_stride(const cftft_ring* R, u64 stride) {
  if (R->kind == CFTFT_RING_PRIME) {
    if (stride < 8 || (stride % 8) != 0) return fail(CFTFT_UNSUPPORTED, "element stride must be a multiple of 8 bytes");
    return CFTFT_OK;
  }
  if (stride < R->elem_bytes || (stride % 16) != 0)
    return fail(CFTFT_UNSUPPORTED, "element stride must be a multiple of 16 and >= " +
                                       std::to_string(R->elem_bytes) + " bytes");
  return CFTFT_OK;
}

// Kernel attributes and occupancy are set / queried once per (device,
// kernel): touching a kernel's attributes while an earlier launch of it runs
// can stall the host until that launch ends.
struct KernelInfo {
  int dev;
  const void* fn;
  int threads;
  size_t smem;
  int per;
};
inline std::mutex g_kmu;
inline std::vector<KernelInfo> g_kinfo;

template <class K>
int set_smem(K kernel) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(g_kmu);
  for (const auto& k : g_kinfo)
    if (k.dev == dev && k.fn == (const void*)kernel && k.threads == -1) return CFTFT_OK;
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  g_kinfo.push_back(KernelInfo{dev, (const void*)kernel, -1, 0, 0});
  return CFTFT_OK;
}

template <class K>
int grid_for(K kernel, int threads, size_t smem, u64 nleaves, unsigned* grid) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  int per = -1, sms = 0;
  {
    std::lock_guard<std::mutex> g(g_kmu);
    for (const auto& k : g_kinfo)
      if (k.dev == dev && k.fn == (const void*)kernel && k.threads == threads && k.smem == smem) per = k.per;
  }
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per < 0) {
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem));
    std::lock_guard<std::mutex> g(g_kmu);
    g_kinfo.push_back(KernelInfo{dev, (const void*)kernel, threads, smem, per});
  }
  if (per < 1) return fail(CFTFT_CUDA_ERROR, "leaf kernel does not fit on an SM");
  u64 g = (u64)sms * (u64)per;
  if (g > nleaves) g = nleaves;
  *grid = (unsigned)std::max<u64>(g, 1);
  return CFTFT_OK;
}

// Dynamic shared memory attribute of a kernel, per device (cudaFuncSetAttribute
// applies to the current device only).
template <class K>
int set_smem_bytes(K kernel, size_t bytes) {
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(g_kmu);
  for (const auto& k : g_kinfo)
    if (k.dev == dev && k.fn == (const void*)kernel && k.threads == -2 && k.smem >= bytes) return CFTFT_OK;
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  g_kinfo.push_back(KernelInfo{dev, (const void*)kernel, -2, bytes, 0});
  return CFTFT_OK;
}

// TMA descriptors of the radix-64 coset kernel (wave_tma.cuh): a buffer of
// `extent` elements seen as [element][row][word] with rows of `step` 256-bit
// lanes (32 rows per coefficient) and 8-word x 32-row boxes (one coset).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int encode_fn(EncodeTiledFn* out) {
  static EncodeTiledFn fn = nullptr;
  static std::mutex m;
  std::lock_guard<std::mutex> g(m);
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) return fail(CFTFT_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  *out = fn;
  return CFTFT_OK;
}
CUtensorMapL2promotion l2_promotion() {
  // a coset box row is 32 bytes: let the L2 fetch the 64-byte pair (the
  // neighbouring coset is read by a concurrent item)
  return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
}
int make_coset_map(CUtensorMap* tm, void* base, u64 stride, u64 extent, u32 step) {
  EncodeTiledFn fn = nullptr;
  if (int rc = encode_fn(&fn)) return rc;
  const cuuint64_t gdim[3] = {8ull * step, 32ull, std::max<u64>(extent, 1)};
  const cuuint64_t gstr[2] = {32ull * step, stride};
  const cuuint32_t box[3] = {8u, 32u, 1u};
  const cuuint32_t est[3] = {1u, 1u, 1u};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, gdim, gstr, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_32B, l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CFTFT_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return CFTFT_OK;
}

// Per-launch scratch (counters, tops arrays, the shadow buffer) comes from the
// device's stream-ordered pool; keep freed blocks cached instead of returning
// them to the driver at every synchronisation.
int keep_pool() {
  static std::mutex m;
  static std::vector<int> done;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(m);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return CFTFT_OK;
  cudaMemPool_t pool;
  CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  u64 thr = ~u64{0};
  CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done.push_back(dev);
  return CFTFT_OK;
}

// Prime rings: the two-level Montgomery tables of omega's powers (omega^i R
// mod p, i < 2^lo_bits; omega^(i 2^lo_bits) R mod p), built once per ring.
int ensure_prime_tables(cftft_ring* R, cudaStream_t st) {
  std::lock_guard<std::mutex> g(R->mu);
  if (R->prime_tw) return CFTFT_OK;
  const u64 p = R->m, lo = u64{1} << R->lo_bits, hi = R->M >> R->lo_bits;
  auto mulp = [p](u64 a, u64 b) { return (u64)((unsigned __int128)a * b % p); };
  const u64 Rm = (u64)(((unsigned __int128)1 << 64) % p);  // 2^64 mod p
  std::vector<u64> h(lo + hi);
  u64 w = 1 % p;
  for (u64 i = 0; i < lo; ++i, w = mulp(w, R->omega)) h[i] = mulp(w, Rm);
  const u64 step = w;  // omega^lo
  u64 v = 1 % p;
  for (u64 i = 0; i < hi; ++i, v = mulp(v, step)) h[lo + i] = mulp(v, Rm);
  u64* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, h.size() * sizeof(u64)));
  CUDA_TRY(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(u64), cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  R->prime_tw = d;
  return CFTFT_OK;
}

// information bytes of one coefficient (N/8, 8 K, 8)
u64 info_bytes(const cftft_ring* R) {
  return R->kind == CFTFT_RING_FERMAT ? R->N / 8 : (R->kind == CFTFT_RING_NEGACYCLIC ? 8 * R->K : 8);
}

int launch_plan(cftft_ring* R, DevicePlan& dp, std::uint8_t* base, u64 stride, cudaStream_t st,
                bool canonicalize) {
  u64 launches = 0;
  if (int rc = keep_pool()) return rc;
  if (dp.nleaves) {
    u32* counters = nullptr;
    const size_t cbytes = sizeof(u32) * (1 + (size_t)dp.ncounters);
    CUDA_TRY(cudaMallocAsync((void**)&counters, cbytes, st));
    CUDA_TRY(cudaMemsetAsync(counters, 0, cbytes, st));
    size_t max_group = 1;  // prime: the most leaves a ticket groups
    for (size_t g = 1; g < dp.host.groups.size(); g += 2) max_group = std::max<size_t>(max_group, dp.host.groups[g]);
    // Fermat: two ticket buffers of `half` bytes each (a big ticket spans both)
    const size_t half = ((kSmemBudget - scratch_bytes(1024)) / 2) & ~size_t(15);
    const size_t slots_bytes = R->kind == CFTFT_RING_FERMAT
                                   ? std::max<size_t>({dp.host.max_slot_area, (size_t)dp.slot_bytes << dp.max_ell, 2 * half})
                                   : ((size_t)R->slot_bytes << dp.max_ell) * max_group *
                                         (R->kind == CFTFT_RING_PRIME ? 17 : 16) / 16;  // prime: grouped, padded
    const size_t smem = slots_bytes + (R->kind == CFTFT_RING_FERMAT ? scratch_bytes(1024) : 0);
    unsigned grid = 1;
    int* tops = nullptr;
    if (R->kind == CFTFT_RING_FERMAT) {
      fermat::Args A{};
      A.data = base;
      A.elem_bytes = stride;
      A.leaves = dp.leaves;
      A.nleaves = dp.nleaves;
      A.classes = dp.classes;
      A.ops = dp.ops;
      A.levels = dp.levels;
      A.rots = dp.rots;
      A.counters = counters;
      A.cmeta = dp.cmeta;
      A.N = R->N;
      A.M = R->M;
      A.D = R->D;
      A.C = dp.C;
      A.logC = (u32)__builtin_ctz(dp.C);
      A.slot_bytes = dp.slot_bytes;
      A.scratch_off = (u32)slots_bytes;
      A.lanes = dp.C;
      A.logLanes = (u32)__builtin_ctz(dp.C);
      A.logS = dp.logS;
      std::uint8_t* shadow = nullptr;
      if (dp.host.coset) {
        const size_t tb = 2 * (size_t)dp.host.extent * dp.C * sizeof(int);
        const size_t sb = (size_t)dp.host.extent * stride;
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> g(R->mu);
        cftft_ring::Scratch* sc = nullptr;
        const bool dflt = st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread;
        const std::thread::id me = dflt ? std::this_thread::get_id() : std::thread::id();
        for (auto& x : R->scratch)
          if (x.dev == dev && x.stream == (void*)st && x.thread == me) sc = &x;
        if (!sc) {
          R->scratch.push_back(cftft_ring::Scratch{});
          sc = &R->scratch.back();
          sc->dev = dev;
          sc->stream = (void*)st;
          sc->thread = me;
        }
        if (sc->tops_bytes < tb || sc->shadow_bytes < sb) {
          CUDA_TRY(cudaStreamSynchronize(st));  // the old buffers may still be in use
          if (sc->tops_bytes < tb) {
            if (sc->tops) cudaFree(sc->tops);
            sc->tops = nullptr;
            sc->tops_bytes = 0;
            CUDA_TRY(cudaMalloc(&sc->tops, tb));
            sc->tops_bytes = tb;
          }
          if (sc->shadow_bytes < sb) {
            if (sc->shadow) cudaFree(sc->shadow);
            sc->shadow = nullptr;
            sc->shadow_bytes = 0;
            CUDA_TRY(cudaMalloc(&sc->shadow, sb));
            sc->shadow_bytes = sb;
          }
        }
        tops = static_cast<int*>(sc->tops);
        shadow = static_cast<std::uint8_t*>(sc->shadow);
        // wave plans load no tops of elements they have not written (Plan::tops_clear)
        if (dp.host.tops_clear) CUDA_TRY(cudaMemsetAsync(tops, 0, tb, st));
      }
      A.T = tops;
      A.data2 = shadow;
      A.tloc = (u64)dp.host.extent * dp.C;
      A.locbits = dp.locbits;
      A.nclasses = (u32)dp.host.classes.size();
      A.no_deps = 0;
      A.half = (u32)half;
      unsigned long long* prof = nullptr;
      static const bool profiling = env_int("CFTFT_PROFILE", 0) != 0;
      if (profiling) {
        CUDA_TRY(cudaMallocAsync((void**)&prof, 8 * fermat::PH_N, st));
        CUDA_TRY(cudaMemsetAsync(prof, 0, 8 * fermat::PH_N, st));
      }
      A.prof = prof;
      static const u32 dbg = (u32)env_int("CFTFT_DEBUG_SKIP", 0);
      A.debug_skip = dbg;
      auto go = [&](auto kernel, int nt) -> int {
        if (int rc = set_smem(kernel)) return rc;
        if (int rc = grid_for(kernel, nt, smem, dp.nleaves, &grid)) return rc;
        kernel<<<grid, nt, smem, st>>>(A);
        return CFTFT_OK;
      };
      int rc = 0;
      if (!dp.host.waves.empty()) {
        // wave engine: one launch per range of independent tickets, in order;
        // coset ranges on the warp-level kernel, whole ranges on the leaf kernel
        A.no_deps = 1;
        A.xpre = dp.wave_slots;
        fermat::WaveArgs W{};
        W.classes = dp.classes;
        W.ops = dp.ops;
        W.rots = dp.rots;
        W.data = base;
        W.data2 = A.data2;
        W.elem_bytes = stride;
        W.T = tops;
        W.tloc = A.tloc;
        W.locbits = dp.locbits;
        W.wops = dp.wave_ops;
        W.levels = dp.levels;
        W.logS = dp.logS;
        W.debug = dbg;
        W.logLanes = (u32)__builtin_ctz(dp.C);
        W.wslots = dp.wave_slots;
        W.lanes = dp.C;
        W.D = R->D;
        W.M = R->M;
        const int wwarps = fermat::kWaveWarps;
        const size_t wsmem = (size_t)wwarps * fermat::wave_tile_words<8>() * 4;
        if (int e = set_smem_bytes(fermat::coset_wave_kernel<8, false>, wsmem)) return e;
        if (int e = set_smem_bytes(fermat::coset_wave_kernel<8, true>, wsmem)) return e;
        int dev = 0, sms = 0, per = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        // the multi-GPU transforms leave a few SMs to NCCL's kernels, which run on
        // the context's stream next to these persistent CTAs (t_sm_reserve)
        sms = std::max(1, sms - t_sm_reserve);
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fermat::coset_wave_kernel<8, false>, 32 * wwarps, wsmem));
        const size_t xsmem = (size_t)fermat::wide_tile_words<8>() * 4;
        int xper = 0;
        if (dp.host.wide) {
          if (int e = set_smem_bytes(fermat::coset_wide_kernel<8>, xsmem)) return e;
          CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&xper, fermat::coset_wide_kernel<8>,
                                                                 32 * fermat::kWideWarps, xsmem));
        }
        CUtensorMap tm_view{}, tm_shadow{};
        bool tma_maps = false;
        for (size_t wi = 0; wi < dp.host.waves.size(); ++wi) {
          const auto& wr = dp.host.waves[wi];
          const char* kname = (wr[2] == 2 && dp.tma_wave[wi]) ? "coset_tma_kernel"
                              : wr[2] == 2                   ? "coset_wide_kernel"
                              : wr[2] == 1                   ? "coset_wave_kernel"
                                                             : "leaf_kernel";
          LaunchTimer lt(kname, dp.wave_loads[wi] * info_bytes(R), st);
          if (wr[2] == 2 && dp.tma_wave[wi]) {
            if (!tma_maps) {
              if (int e = make_coset_map(&tm_view, base, stride, dp.host.extent, dp.tma_step)) return e;
              if (int e = make_coset_map(&tm_shadow, shadow ? (void*)shadow : (void*)base, stride, dp.host.extent,
                                         dp.tma_step))
                return e;
              if (int e = set_smem_bytes(fermat::coset_tma_kernel<true, false>, fermat::kTmaSmem)) return e;
              if (int e = set_smem_bytes(fermat::coset_tma_kernel<true, false, true>, fermat::kTmaSmem)) return e;
              if (int e = set_smem_bytes(fermat::coset_tma_kernel<false, false>, fermat::kTmaSmem)) return e;
              if (int e = set_smem_bytes(fermat::coset_tma_kernel<true, true>, fermat::kTmaSmem)) return e;
              if (int e = set_smem_bytes(fermat::coset_tma_kernel<false, true>, fermat::kTmaSmem)) return e;
              tma_maps = true;
            }
            W.leaves = dp.leaves + wr[0];
            W.nleaves = (u32)wr[1];
            W.gpl = (u32)std::max<u64>(1, wr[3]);
            W.tdesc = static_cast<const fermat::TmaLeafDesc*>(dp.tma_descs) + dp.tma_desc_off[wi];
            W.tlay = dp.tma_lay;
            // waves with sub-lane pre-rotations read every coset twice (as rows and
            // as the next coset's lane-below rows): runs of adjacent cosets per CTA
            // keep the second read in L2 (measured: 8 for the TFT's waves, 2 for
            // the ITFT's network waves, none for aligned and program waves)
            W.runlog = dp.tma_aligned[wi] ? 0u : dp.tma_wave[wi] == 1 ? 3u : dp.tma_wave[wi] == 2 ? 1u : 0u;
            const unsigned g = (unsigned)std::min<u64>(wr[1] * W.gpl, (u64)sms);
            switch (dp.tma_wave[wi]) {
              case 1:
                if (dp.tma_aligned[wi])
                  fermat::coset_tma_kernel<true, false><<<g, fermat::kTmaThreads, fermat::kTmaSmem, st>>>(tm_view, tm_shadow, W);
                else
                  fermat::coset_tma_kernel<true, false, true><<<g, fermat::kTmaThreads, fermat::kTmaSmem, st>>>(tm_view, tm_shadow, W);
                break;
              case 2:
                fermat::coset_tma_kernel<false, false><<<g, fermat::kTmaThreads, fermat::kTmaSmem, st>>>(tm_view, tm_shadow, W);
                break;
              case 5:
                fermat::coset_tma_kernel<true, true><<<g, fermat::kTmaThreads, fermat::kTmaSmem, st>>>(tm_view, tm_shadow, W);
                break;
              default:
                fermat::coset_tma_kernel<false, true><<<g, fermat::kTmaThreads, fermat::kTmaSmem, st>>>(tm_view, tm_shadow, W);
                break;
            }
          } else if (wr[2] == 2) {
            W.leaves = dp.leaves + wr[0];
            W.nleaves = (u32)wr[1];
            W.gpl = (u32)std::max<u64>(1, wr[3]);
            const unsigned g = (unsigned)std::min<u64>(wr[1] * W.gpl, (u64)sms * std::max(xper, 1));
            fermat::coset_wide_kernel<8><<<g, 32 * fermat::kWideWarps, xsmem, st>>>(W);
          } else if (wr[2] == 1) {
            W.leaves = dp.leaves + wr[0];
            W.nleaves = (u32)wr[1];
            W.gpl = (u32)std::max<u64>(1, wr[3]);
            const unsigned g = (unsigned)std::min<u64>((wr[1] * W.gpl + wwarps - 1) / wwarps, (u64)sms * std::max(per, 1));
            if (W.logS)
              fermat::coset_wave_kernel<8, true><<<g, 32 * wwarps, wsmem, st>>>(W);
            else
              fermat::coset_wave_kernel<8, false><<<g, 32 * wwarps, wsmem, st>>>(W);
          } else {
            CUDA_TRY(cudaMemsetAsync(counters, 0, sizeof(u32), st));  // ticket counter of this range
            A.leaves = dp.leaves + wr[0];
            A.nleaves = wr[1];
            rc = go(fermat::leaf_kernel<8, 512>, 512);
            if (rc) return rc;
          }
          ++launches;
        }
        launches -= 1;  // counted once more below
      } else {
        rc = dp.cw == 16 ? go(fermat::leaf_kernel<16, 512>, 512)
             : dp.cw == 8 ? go(fermat::leaf_kernel<8, 512>, 512)
                          : go(fermat::leaf_kernel<4, 512>, 512);
      }
      if (rc) return rc;
      if (tops) {
        // carry-save lanes of the outputs back to the canonical element format
        // (with the sub-lane rotations the outputs' last writers deferred)
        const size_t fsm = dp.final_rot ? (size_t)R->D * 4 : 0;
        if (fsm > 40 * 1024)
          if (int e = set_smem_bytes(fermat::cs_fold_kernel, fsm)) return e;
        const u32 logC = (u32)__builtin_ctz(dp.C);
        if (dp.host.use_fold_list) {
          // listed outputs in place, the shadow buffer's from there into place
          if (!dp.host.fold_list.empty()) {
            LaunchTimer lt("cs_fold_kernel", 2 * dp.host.fold_list.size() * info_bytes(R), st);
            fermat::cs_fold_kernel<<<(unsigned)dp.host.fold_list.size(), 256, fsm, st>>>(
                base, stride, tops, dp.C, dp.cw, logC, dp.logS, R->D, 0, 1, dp.final_rot, dp.fold_list, nullptr);
            ++launches;
          }
          if (!dp.host.shadow_finals.empty()) {
            LaunchTimer lt("cs_fold_kernel", 2 * dp.host.shadow_finals.size() * info_bytes(R), st);
            fermat::cs_fold_kernel<<<(unsigned)dp.host.shadow_finals.size(), 256, fsm, st>>>(
                base, stride, tops + A.tloc, dp.C, dp.cw, logC, dp.logS, R->D, 0, 1, dp.final_rot,
                dp.shadow_finals, shadow, dp.tma_cm_finals ? (u32)__builtin_ctz(dp.tma_step) : 0u);
            ++launches;
          }
        } else if (dp.host.final_count) {
          LaunchTimer lt("cs_fold_kernel", 2 * dp.host.final_count * info_bytes(R), st);
          fermat::cs_fold_kernel<<<(unsigned)dp.host.final_count, 256, fsm, st>>>(
              base, stride, tops, dp.C, dp.cw, logC, dp.logS, R->D, 0, 1, dp.final_rot, nullptr, nullptr);
          ++launches;
        }
      }
      if (prof) {
        unsigned long long h[fermat::PH_N];
        CUDA_TRY(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        CUDA_TRY(cudaFreeAsync(prof, st));
        unsigned long long tot = 0;
        for (auto v : h) tot += v;
        fprintf(stderr, "[cftft] leaves=%llu grid=%u phase cycles (%% of CTA time): wait %.1f issue %.1f cache %.1f load %.1f pre %.1f levels %.1f post %.1f store %.1f (total %.3g cyc/CTA)\n",
                (unsigned long long)dp.nleaves, grid, 100.0 * h[0] / tot, 100.0 * h[6] / tot, 100.0 * h[7] / tot,
                100.0 * h[1] / tot, 100.0 * h[2] / tot, 100.0 * h[3] / tot, 100.0 * h[4] / tot, 100.0 * h[5] / tot,
                (double)tot / grid);
      }
    } else if (R->kind == CFTFT_RING_PRIME) {
      if (int rc = ensure_prime_tables(R, st)) return rc;
      // big leaves (2^9..2^11 coefficients): 256-thread CTAs for the TFT
      // (network leaves), 512 for the ITFT (its truncated leaves run many
      // short dependency levels: wider CTAs per barrier measured faster)
      const bool big = dp.max_ell >= 9;
      const bool wide_cta = big && dp.host.inverse;
      const int pthreads = wide_cta ? 512 : big ? 256 : 128;
      if (wide_cta) {
        if (int rc = set_smem(prime::leaf_kernel<512>)) return rc;
        if (int rc = grid_for(prime::leaf_kernel<512>, pthreads, smem, dp.nleaves, &grid)) return rc;
      } else if (big) {
        if (int rc = set_smem(prime::leaf_kernel<256>)) return rc;
        if (int rc = grid_for(prime::leaf_kernel<256>, pthreads, smem, dp.nleaves, &grid)) return rc;
      } else {
        if (int rc = set_smem(prime::leaf_kernel<128>)) return rc;
        if (int rc = grid_for(prime::leaf_kernel<128>, pthreads, smem, dp.nleaves, &grid)) return rc;
      }
      prime::Args A{};
      A.data = base;
      A.elem_bytes = stride;
      A.leaves = dp.leaves;
      A.nleaves = dp.nleaves;
      A.classes = dp.classes;
      A.ops = dp.ops;
      A.levels = dp.levels;
      A.rots = dp.rots;
      A.counters = counters;
      A.cmeta = dp.cmeta;
      A.M = R->M;
      A.p = R->m;
      A.pinv = R->pinv;
      A.lo_bits = R->lo_bits;
      A.tw_lo = R->prime_tw;
      A.tw_hi = R->prime_tw + (size_t{1} << R->lo_bits);
      A.slot_bytes = R->slot_bytes;
      A.groups = dp.groups;
      A.ntw = dp.prime_ntw;
      A.nleaves = dp.groups ? dp.host.groups.size() / 2 : dp.nleaves;  // tickets
      if (wide_cta)
        prime::leaf_kernel<512><<<grid, pthreads, smem, st>>>(A);
      else if (big)
        prime::leaf_kernel<256><<<grid, pthreads, smem, st>>>(A);
      else
        prime::leaf_kernel<128><<<grid, pthreads, smem, st>>>(A);
    } else {
      if (int rc = set_smem(negacyclic::leaf_kernel)) return rc;
      if (int rc = grid_for(negacyclic::leaf_kernel, negacyclic::kThreads, smem, dp.nleaves, &grid))
        return rc;
      negacyclic::Args A{};
      A.data = base;
      A.elem_bytes = stride;
      A.leaves = dp.leaves;
      A.nleaves = dp.nleaves;
      A.classes = dp.classes;
      A.ops = dp.ops;
      A.levels = dp.levels;
      A.rots = dp.rots;
      A.counters = counters;
      A.cmeta = dp.cmeta;
      A.K = R->K;
      A.M = R->M;
      A.m = R->m;
      A.slot_bytes = R->slot_bytes;
      negacyclic::leaf_kernel<<<grid, negacyclic::kThreads, smem, st>>>(A);
    }
    ++launches;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaFreeAsync(counters, st));
  }
  if (R->kind == CFTFT_RING_FERMAT && canonicalize && dp.host.final_count && !dp.host.coset) {
    const u64 cnt = dp.host.final_count;
    fermat::canonicalize_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(base, stride, cnt, R->D);
    ++launches;
  }
  g_last_launches = launches;
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

// fault::corrupt_tft_base on the GPU: element 0 += 1 in the ring (Fermat:
// N/64 limbs + top word, canonical; negacyclic: word 0 mod m; prime: mod p)
__device__ void fault_add_one_kernel_body(std::uint8_t* el, int kind, u64 words, u64 m) {
  u64* w = reinterpret_cast<u64*>(el);
  if (kind == CFTFT_RING_FERMAT) {
    const u64 limbs = words / 2;  // words = D (u32 words)
    if (w[limbs]) {  // 2^N + 1 == 0
      w[limbs] = 0;
      return;
    }
    u64 i = 0;
    while (i < limbs && ++w[i] == 0) ++i;
    if (i == limbs) w[limbs] = 1;  // 2^N - 1 + 1
  } else {
    w[0] = (w[0] + 1 == m) ? 0 : w[0] + 1;
  }
}

__global__ void fault_add_one_kernel(std::uint8_t* el, int kind, u64 words, u64 m) {
  fault_add_one_kernel_body(el, kind, words, m);
}
__global__ void fault_add_one_items_kernel(std::uint8_t* base, u64 esb, const u64* idx, u64 count, int kind,
                                           u64 words, u64 m) {
  const u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (i < count) fault_add_one_kernel_body(base + idx[i] * esb, kind, words, m);
}

int transform(const cftft_ring* cR, bool inv, const cftft_params* p, void* dev_base, u64 stride,
              int policy, uint64_t* count, void* stream) {
  if (int rc = validate(cR, inv, p, policy)) return rc;
  if (int rc = check_stride(cR, stride)) return rc;
  auto* R = const_cast<cftft_ring*>(cR);
  if (count) {
    std::lock_guard<std::mutex> g(R->mu);
    *count = inv ? R->counts.itft(p->length, p->input_count, p->output_count, p->want_next, policy)
                 : R->counts.tft(p->length, p->input_count, p->output_count, policy);
  }
  auto st = static_cast<cudaStream_t>(stream);
  DevicePlan* dp = nullptr;
  if (int rc = get_plan(R, inv, *p, policy, st, &dp)) return rc;
  auto* base = static_cast<std::uint8_t*>(dev_base);
  auto run = [&]() -> int {
    if (int rc = launch_plan(R, *dp, base, stride, st, true)) return rc;
    if (!inv && g_fault.load()) {
      // fault::corrupt_tft_base: x[0] += 1 in the ring
      fault_add_one_kernel<<<1, 1, 0, st>>>(base, R->kind, R->kind == CFTFT_RING_NEGACYCLIC ? R->K : (u64)R->D,
                                           R->m);
      CUDA_TRY(cudaGetLastError());
    }
    return CFTFT_OK;
  };
  if (!g_poison.load()) return run();
  // debug poison: two runs with different fills of [z, L); the specified
  // outputs must agree bit for bit
  const u64 L = p->length, z = p->input_count;
  const u64 o = inv ? p->output_count + (u64)p->want_next : p->output_count;
  const size_t eb = R->elem_bytes;
  void *save = nullptr, *out1 = nullptr;
  CUDA_TRY(cudaMalloc(&save, (size_t)L * eb));
  CUDA_TRY(cudaMalloc(&out1, (size_t)o * eb));
  int rc = CFTFT_OK;
  auto fail_free = [&](int code) {
    cudaFree(save);
    cudaFree(out1);
    return code;
  };
  if (cudaMemcpy2DAsync(save, eb, base, stride, eb, z, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return fail_free(fail(CFTFT_CUDA_ERROR, "poison: save"));
  for (int pass = 0; pass < 2 && !rc; ++pass) {
    if (pass && cudaMemcpy2DAsync(base, stride, save, eb, eb, z, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return fail_free(fail(CFTFT_CUDA_ERROR, "poison: restore"));
    if (L > z && cudaMemset2DAsync(base + z * stride, stride, pass ? 0xA5 : 0xFF, eb, L - z, st) != cudaSuccess)
      return fail_free(fail(CFTFT_CUDA_ERROR, "poison: fill"));
    rc = run();
    if (!rc && !pass &&
        cudaMemcpy2DAsync(out1, eb, base, stride, eb, o, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      rc = fail(CFTFT_CUDA_ERROR, "poison: keep");
  }
  if (rc) return fail_free(rc);
  std::vector<std::uint8_t> a((size_t)o * eb), b((size_t)o * eb);
  if (cudaMemcpy2DAsync(a.data(), eb, out1, eb, eb, o, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaMemcpy2DAsync(b.data(), eb, base, stride, eb, o, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return fail_free(fail(CFTFT_CUDA_ERROR, "poison: compare"));
  // (a Fermat element is its lanes and top word; the bytes that pad it to a
  // multiple of 16 are not part of the value)
  const size_t vb = R->kind == CFTFT_RING_FERMAT ? (size_t)R->D * 4 + 8 : eb;
  for (u64 i = 0; i < o; ++i)
    if (std::memcmp(a.data() + i * eb, b.data() + i * eb, vb) != 0)
      return fail_free(fail(CFTFT_POISON_READ, "output " + std::to_string(i) +
                                                   " depends on the cells >= z (read before written)"));
  return fail_free(CFTFT_OK);
}

int host_transform(const cftft_ring* cR, bool inv, const cftft_params* p, void* host_base,
                   u64 stride, int policy, uint64_t* count) {
  if (int rc = validate(cR, inv, p, policy)) return rc;
  if (int rc = check_stride(cR, stride)) return rc;
  auto* R = const_cast<cftft_ring*>(cR);
  const u64 L = p->length;
  const size_t need = (size_t)L * stride;
  std::lock_guard<std::mutex> sg(R->stage_mu);
  {
    if (R->stage_bytes < need) {
      if (R->stage) cudaFree(R->stage);
      R->stage = nullptr;
      R->stage_bytes = 0;
      CUDA_TRY(cudaMalloc(&R->stage, need));
      R->stage_bytes = need;
    }
  }
  const u64 in = p->input_count;
  const u64 out = inv ? p->output_count + (u64)p->want_next : p->output_count;
  const size_t eb = R->elem_bytes;
  CUDA_TRY(cudaMemcpy2D(R->stage, stride, host_base, stride, eb, in, cudaMemcpyHostToDevice));
  int rc = transform(R, inv, p, R->stage, stride, policy, count, nullptr);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpy2D(host_base, stride, R->stage, stride, eb, out, cudaMemcpyDeviceToHost));
  return CFTFT_OK;
}

void json_plan(std::ostringstream& os, const Plan& p, u64 lane_bits) {
  os << "{\"inverse\":" << (p.inverse ? 1 : 0) << ",\"lane_bits\":" << lane_bits << ",\"coset\":" << (p.coset ? 1 : 0)
     << ",\"wave\":" << (p.waves.empty() ? 0 : 1);
  os << ",\"waves\":[";
  for (size_t w = 0; w < p.waves.size(); ++w)
    os << (w ? "," : "") << "[" << p.waves[w][0] << "," << p.waves[w][1] << "," << p.waves[w][2] << "," << p.waves[w][3] << "]";
  os << "]"
     << ",\"L\":" << p.L << ",\"s\":" << p.s
     << ",\"z\":" << p.z << ",\"n\":" << p.n << ",\"f\":" << p.f << ",\"final_count\":"
     << p.final_count << ",\"counters\":[";
  for (size_t i = 0; i < p.counters.size(); ++i)
    os << (i ? "," : "") << "[" << p.counters[i].target << ","
       << (p.counters[i].next == kNoDep ? -1 : (long long)p.counters[i].next) << "]";
  os << "],\"classes\":[";
  auto sym = [&](const std::vector<SymExp>& v) {
    os << "[";
    for (size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << "[" << v[i].a << "," << v[i].b << "]";
    os << "]";
  };
  for (size_t c = 0; c < p.classes.size(); ++c) {
    const auto& k = p.classes[c];
    if (c) os << ",";
    os << "{\"ell\":" << k.key.ell << ",\"inverse\":" << k.key.inverse << ",\"z\":" << k.key.z
       << ",\"n\":" << k.key.n << ",\"f\":" << k.key.f << ",\"nload\":" << k.nload
       << ",\"nstore\":" << k.nstore << ",\"kind\":" << k.kind << ",\"step\":" << k.step
       << ",\"m\":" << k.m << ",\"cs\":" << k.cs
       << ",\"wnet\":" << (c < p.wave_net.size() ? p.wave_net[c] : 0u);
    if (c < p.wave_net.size() && p.wave_net[c] && (k.key.ell == 6 || k.key.ell == 4)) {
      // the radix-64 network's rotations (coset positions), (stage, warp, op);
      // the 16-slot network's in the warp kernel's op order
      const u32 nn = k.key.ell == 6 ? 192u : 32u;
      os << ",\"net\":[";
      for (u32 i = 0; i < nn; ++i) os << (i ? "," : "") << (p.wave_ops[p.wave_op_begin[c] + i] >> 16);
      os << "]";
      if (k.key.ell == 6) {
        // stage B re-gauged (Planner::wide_network): per (warp, op) the input
        // gauge g (ops 0..7) and the residual rotation, as {g, res}
        os << ",\"net_g\":[";
        for (u32 i = 96; i < 192; ++i) {
          const u32 wd = p.wave_ops[p.wave_op_begin[c] + i];
          os << (i > 96 ? "," : "") << "[" << ((wd >> 4) & 63u) << "," << ((wd >> 10) & 63u) << "]";
        }
        os << "]";
      }
    }
    os << ",\"levels\":[";
    for (size_t l = 0; l < k.level_begin.size(); ++l) os << (l ? "," : "") << k.level_begin[l];
    os << "],\"ops\":[";
    for (size_t i = 0; i < k.ops.size(); ++i) {
      const auto& o = k.ops[i];
      os << (i ? "," : "") << "[" << (int)o.type << "," << o.a << "," << o.b << "," << o.r << "]";
    }
    os << "],\"pre\":";
    sym(k.pre);
    os << ",\"post\":";
    sym(k.post);
    os << "}";
  }
  os << "],\"leaves\":[";
  for (size_t i = 0; i < p.leaves.size(); ++i) {
    const auto& lf = p.leaves[i];
    os << (i ? "," : "") << "[" << lf.cls << "," << lf.base << "," << lf.stride << "," << lf.s << ","
       << (lf.dep == kNoDep ? -1 : (long long)lf.dep) << "," << lf.dep_target << ","
       << (lf.comp == kNoDep ? -1 : (long long)lf.comp) << "," << p.leaf_wave[i] << "," << lf.tpre << ","
       << lf.tpost << "," << lf.c0 << "," << (lf.locoff == kNoDep ? -1 : (long long)lf.locoff) << "]";
  }
  os << "],\"locbits\":[";
  for (size_t i = 0; i < p.locbits.size(); ++i) os << (i ? "," : "") << p.locbits[i];
  os << "],\"shadow_finals\":[";
  for (size_t i = 0; i < p.shadow_finals.size(); ++i) os << (i ? "," : "") << p.shadow_finals[i];
  os << "],\"wave_slots\":[";
  for (size_t i = 0; i < p.wave_slots.size(); ++i) os << (i ? "," : "") << p.wave_slots[i];
  os << "],\"final_rot\":[";  // {element, bits} pairs
  bool first_fr = true;
  for (size_t i = 0; i < p.final_rot.size(); ++i)
    if (p.final_rot[i]) {
      os << (first_fr ? "" : ",") << i << "," << p.final_rot[i];
      first_fr = false;
    }
  os << "]}";
}

}  // namespace

extern "C" {

int cftft_ring_create(int kind, uint64_t n_or_k, uint64_t modulus, cftft_ring** out) {
  if (!out) return fail(CFTFT_INVALID_PARAMS, "null out");
  *out = nullptr;
  auto R = std::make_unique<cftft_ring>();
  R->kind = kind;
  if (kind == CFTFT_RING_FERMAT) {
    const u64 N = n_or_k;
    if (N < 128 || (N & (N - 1)) != 0 || N > (u64{1} << 18))
      return fail(CFTFT_UNSUPPORTED, "Fermat ring needs N a power of two in [128, 2^18]");
    R->N = N;
    R->M = 2 * N;
    R->D = (u32)(N / 32);
    R->CW = R->D >= 16 ? (R->D <= 64 ? 4 : 16) : R->D;
    R->C = R->D / R->CW;
    R->slot_bytes = fermat_slot_bytes(R->C, 4 * R->CW);
    R->elem_bytes = ((N / 8 + 8) + 15) & ~u64(15);
  } else if (kind == CFTFT_RING_NEGACYCLIC) {
    const u64 K = n_or_k, m = modulus;
    if (K < 2 || (K & (K - 1)) != 0 || K > 16384)
      return fail(CFTFT_UNSUPPORTED, "negacyclic ring needs K a power of two in [2, 16384]");
    if (m < 3 || (m & 1) == 0 || m >= (u64{1} << 62))
      return fail(CFTFT_INVALID_PARAMS, "negacyclic modulus must be odd and < 2^62");
    R->K = K;
    R->m = m;
    R->M = 2 * K;
    R->slot_bytes = (u32)(8 * K);
    R->elem_bytes = 8 * K;
  } else if (kind == CFTFT_RING_PRIME) {
    // the reference's RingCtx(p, m) (field.hpp:84-185), m <= 32 on the GPU
    const u64 m = n_or_k, p = modulus;
    if (m < 1 || m > 32) return fail(CFTFT_UNSUPPORTED, "prime ring: two-adicity m must be in [1, 32]");
    if (p < 3 || (p & 1) == 0 || ((p - 1) & ((u64{1} << m) - 1)) != 0)
      return fail(CFTFT_INVALID_PARAMS, "prime ring: p must be odd with 2^m | p - 1");
    auto mulp = [p](u64 a, u64 b) { return (u64)((unsigned __int128)a * b % p); };
    auto powp = [&](u64 a, u64 e) {
      u64 r = 1 % p;
      for (; e; e >>= 1, a = mulp(a, a))
        if (e & 1) r = mulp(r, a);
      return r;
    };
    // the reference rejects composite moduli (field.hpp:56-78, NotPrime):
    // Miller-Rabin with the first twelve primes as bases, exact below 2^64
    {
      bool prime = true;
      const u64 d0 = p - 1;
      const int r0 = __builtin_ctzll(d0);
      const u64 d = d0 >> r0;
      for (u64 a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
        if (p % a == 0) {
          prime = p == a;
          break;
        }
        u64 x = powp(a, d);
        if (x == 1 || x == p - 1) continue;
        bool witness = true;
        for (int i = 1; i < r0 && witness; ++i) {
          x = mulp(x, x);
          if (x == p - 1) witness = false;
        }
        if (witness) {
          prime = false;
          break;
        }
      }
      if (!prime) return fail(CFTFT_INVALID_PARAMS, "prime ring: modulus is not prime");
    }
    const u64 M = u64{1} << m;
    // smallest g in 2, 3, 5, 7, ... whose (p-1)/2^m power has order 2^m (field.hpp:170-177)
    u64 omega = 0;
    for (u64 g = 2; g < 1024 && !omega; g = (g == 2) ? 3 : g + 2) {
      const u64 w = powp(g % p, (p - 1) >> m);
      if (powp(w, M / 2) == p - 1) omega = w;
    }
    if (!omega) return fail(CFTFT_INVALID_PARAMS, "prime ring: no root of order 2^m (is p prime?)");
    u64 inv = 1;  // p^-1 mod 2^64 by Newton's iteration
    for (int i = 0; i < 7; ++i) inv *= 2 - p * inv;
    R->m = p;
    R->K = m;
    R->M = M;
    R->omega = omega;
    R->pinv = (u64)0 - inv;
    R->lo_bits = (u32)std::min<u64>(m, 16);
    R->slot_bytes = 8;
    R->elem_bytes = 8;
  } else {
    return fail(CFTFT_UNSUPPORTED, "unknown ring kind");
  }
  // largest leaf whose slots fit the shared-memory budget (and the 16-bit slot ids)
  unsigned lam = 1;
  const size_t per_cta = kSmemBudget;
  const size_t budget = per_cta - (kind == CFTFT_RING_FERMAT ? scratch_bytes(R->NT) : 0);
  // (prime rings: leaves up to 2^11, so that L = 2^22 runs in two passes)
  const unsigned lam_max = kind == CFTFT_RING_PRIME ? 11u : 10u;
  while (lam < lam_max && ((size_t)R->slot_bytes << (lam + 1)) <= budget) ++lam;
  R->max_leaf_ell = lam;
  R->max_leaf_fit = lam;
  *out = R.release();
  return CFTFT_OK;
}

void cftft_ring_destroy(cftft_ring* ring) { delete ring; }
uint64_t cftft_ring_root_order(const cftft_ring* ring) { return ring ? ring->M : 0; }
uint64_t cftft_ring_element_bytes(const cftft_ring* ring) { return ring ? ring->elem_bytes : 0; }

unsigned cftft_ring_set_leaf_limit(cftft_ring* ring, unsigned max_ell) {
  if (!ring) return 0;
  std::lock_guard<std::mutex> g(ring->mu);
  unsigned cap = ring->max_leaf_fit;
  unsigned v = max_ell == 0 ? cap : std::min(std::max(max_ell, 1u), cap);
  const unsigned lim = max_ell == 0 ? 0u : std::max(max_ell, 1u);
  if (v != ring->max_leaf_ell || lim != ring->leaf_limit) {
    ring->max_leaf_ell = v;
    ring->leaf_limit = lim;
    ring->cache.clear();
  }
  return v;
}

int cftft_validate(const cftft_ring* ring, int inverse, const cftft_params* params, int policy) {
  return validate(ring, inverse != 0, params, policy);
}

int cftft_stream_synchronize(void* stream) {
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return CFTFT_OK;
}

int cftft_ring_set_coset(cftft_ring* ring, int lane_words) {
  if (!ring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (ring->kind != CFTFT_RING_FERMAT) return lane_words == 0 ? CFTFT_OK : fail(CFTFT_UNSUPPORTED, "coset leaves are for Fermat rings");
  if (lane_words != -1 && lane_words != 0 && lane_words != 4 && lane_words != 8 && lane_words != 16)
    return fail(CFTFT_INVALID_PARAMS, "lane_words must be -1 (auto), 0 (off), 4, 8 or 16");
  std::lock_guard<std::mutex> g(ring->mu);
  if (ring->coset_cw != lane_words) {
    ring->coset_cw = lane_words;
    ring->cache.clear();
  }
  return CFTFT_OK;
}

int cftft_ring_set_wide(cftft_ring* ring, int wide) {
  if (!ring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (wide < -1 || wide > 1)
    return fail(CFTFT_INVALID_PARAMS, "wide must be -1 (default), 0 (radix-8 waves) or 1 (radix-64 waves)");
  std::lock_guard<std::mutex> g(ring->mu);
  if (ring->wide != wide) {
    ring->wide = wide;
    ring->cache.clear();
  }
  return CFTFT_OK;
}

int cftft_gpu_tft(const cftft_ring* ring, const cftft_params* params, void* dev_base,
                  uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count, void* stream) {
  return transform(ring, false, params, dev_base, elem_stride_bytes, policy, base_case_count, stream);
}

int cftft_gpu_itft(const cftft_ring* ring, const cftft_params* params, void* dev_base,
                   uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count, void* stream) {
  return transform(ring, true, params, dev_base, elem_stride_bytes, policy, base_case_count, stream);
}

int cftft_tft_host(const cftft_ring* ring, const cftft_params* params, void* host_base,
                   uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count) {
  return host_transform(ring, false, params, host_base, elem_stride_bytes, policy, base_case_count);
}

int cftft_itft_host(const cftft_ring* ring, const cftft_params* params, void* host_base,
                    uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count) {
  return host_transform(ring, true, params, host_base, elem_stride_bytes, policy, base_case_count);
}

namespace {
typedef unsigned __int128 hu128;
int ensure_ntt_tables(cftft_ring* R, cudaStream_t st) {
  std::lock_guard<std::mutex> g(R->mu);
  if (R->ntt_tw) return CFTFT_OK;
  const u64 n = R->N / 16;
  // 4 n entries of {w mod Q1, Shoup factor floor(w 2^32 / Q1), w mod Q2,
  // Shoup} (pointwise.cuh; primitive root 3 for both primes): psi^i,
  // psi^-i / n, the forward level twiddles (level ls: omega^(j 2^ls),
  // j < n >> (ls+1), at n - (n >> ls)), the inverse ones
  std::vector<u32> h((size_t)16 * n, 0);
  const u32 primes[2] = {pointwise::Q1, pointwise::Q2};
  for (int j = 0; j < 2; ++j) {
    const u64 p = primes[j];
    auto mul = [p](u64 a, u64 b) { return a * b % p; };
    auto pw = [&](u64 a, u64 e) {
      u64 r = 1;
      for (; e; e >>= 1, a = mul(a, a))
        if (e & 1) r = mul(r, a);
      return r;
    };
    auto put = [&](u64 slot, u64 w) {
      h[4 * slot + 2 * j] = (u32)w;
      h[4 * slot + 2 * j + 1] = (u32)((w << 32) / p);
    };
    const u64 psi = pw(3, (p - 1) / (2 * n)), om = mul(psi, psi);
    const u64 psi_inv = pw(psi, p - 2), om_inv = pw(om, p - 2), n_inv = pw(n % p, p - 2);
    u64 x = 1, y = n_inv;
    for (u64 i = 0; i < n; ++i) {
      put(i, x);
      put(n + i, y);
      x = mul(x, psi);
      y = mul(y, psi_inv);
    }
    for (u64 ls = 0, off = 0; (n >> (ls + 1)) >= 1; off += n >> (ls + 1), ++ls) {
      const u64 sf = pw(om, u64{1} << ls), si = pw(om_inv, u64{1} << ls);
      u64 a = 1, b = 1;
      for (u64 k = 0; k < (n >> (ls + 1)); ++k) {
        put(2 * n + off + k, a);
        put(3 * n + off + k, b);
        a = mul(a, sf);
        b = mul(b, si);
      }
    }
  }
  CUDA_TRY(cudaMalloc((void**)&R->ntt_tw, h.size() * 4));
  CUDA_TRY(cudaMemcpyAsync(R->ntt_tw, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return CFTFT_OK;
}
}  // namespace

int cftft_gpu_pointwise_scaled(const cftft_ring* cring, void* dev_a, const void* dev_b, uint64_t count,
                               uint64_t elem_stride_bytes, uint64_t scale, void* stream) {
  if (!cring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (int rc = check_stride(cring, elem_stride_bytes)) return rc;
  if (count == 0) return CFTFT_OK;
  if (count > 0x7FFFFFFFull) return fail(CFTFT_UNSUPPORTED, "too many products for one launch");
  auto* R = const_cast<cftft_ring*>(cring);
  auto st = static_cast<cudaStream_t>(stream);
  if (R->kind == CFTFT_RING_NEGACYCLIC) {
    const size_t smem = 24 * R->K;
    if (smem > 48 * 1024)
      if (int rc = set_smem_bytes(pointwise::nega_pointwise_kernel, smem)) return rc;
    pointwise::nega_pointwise_kernel<<<(unsigned)count, 256, smem, st>>>(
        static_cast<std::uint8_t*>(dev_a), static_cast<const std::uint8_t*>(dev_b), elem_stride_bytes, (u32)R->K,
        R->m, scale % R->m);
    g_last_launches = 1;
    CUDA_TRY(cudaGetLastError());
    return CFTFT_OK;
  }
  if (R->kind == CFTFT_RING_PRIME) {
    const unsigned grid = (unsigned)std::min<u64>((count + 255) / 256, 148ull * 16);
    polymul::prime_pointwise_kernel<<<grid, 256, 0, st>>>(static_cast<std::uint8_t*>(dev_a),
                                                           static_cast<const std::uint8_t*>(dev_b),
                                                           elem_stride_bytes, count, R->m, scale % R->m);
    g_last_launches = 1;
    CUDA_TRY(cudaGetLastError());
    return CFTFT_OK;
  }
  if (R->N < 512 || R->N > (u64{1} << 17))
    return fail(CFTFT_UNSUPPORTED, "Fermat pointwise products need 512 <= N <= 2^17");
  if (int rc = ensure_ntt_tables(R, st)) return rc;
  pointwise::FermatMulArgs A{};
  A.a = static_cast<std::uint8_t*>(dev_a);
  A.b = static_cast<const std::uint8_t*>(dev_b);
  A.stride = elem_stride_bytes;
  A.D16 = (u32)(R->N / 16);
  A.logn = (u32)__builtin_ctz(A.D16);
  A.D32 = R->D;
  A.tw = reinterpret_cast<const uint4*>(R->ntt_tw);
  A.rot = (u32)(scale & (R->M - 1));
  const size_t smem = (size_t)4 * pointwise::padded(A.D16) * 4;
  if (smem > 48 * 1024)
    if (int rc = set_smem_bytes(pointwise::fermat_pointwise_kernel, smem)) return rc;
  pointwise::fermat_pointwise_kernel<<<(unsigned)count, 512, smem, st>>>(A);
  g_last_launches = 1;
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

int cftft_gpu_pointwise(const cftft_ring* ring, void* dev_a, const void* dev_b, uint64_t count,
                        uint64_t elem_stride_bytes, void* stream) {
  // the identity factor: 2^0 in Z/(2^N+1), 1 in the other rings
  return cftft_gpu_pointwise_scaled(ring, dev_a, dev_b, count, elem_stride_bytes,
                                    ring && ring->kind == CFTFT_RING_FERMAT ? 0 : 1, stream);
}

int cftft_gpu_poly_support(const cftft_ring* ring, const void* dev_a, uint64_t len, uint64_t elem_stride_bytes,
                           uint64_t* support, void* stream) {
  if (!ring || !support) return fail(CFTFT_INVALID_PARAMS, "null argument");
  if (int rc = check_stride(ring, elem_stride_bytes)) return rc;
  *support = 0;
  if (len == 0) return CFTFT_OK;
  auto st = static_cast<cudaStream_t>(stream);
  unsigned long long* d = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&d, sizeof *d, st));
  CUDA_TRY(cudaMemsetAsync(d, 0, sizeof *d, st));
  const unsigned grid = (unsigned)std::min<u64>((len + 7) / 8, 148ull * 8);
  polymul::support_kernel<<<grid, 256, 0, st>>>(static_cast<const std::uint8_t*>(dev_a), elem_stride_bytes, len,
                                                 (u32)(ring->elem_bytes / 8), d);
  unsigned long long h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaFreeAsync(d, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *support = h;
  return CFTFT_OK;
}

int cftft_gpu_poly_mul(const cftft_ring* cring, const void* dev_g, uint64_t zg, const void* dev_h, uint64_t zh,
                       void* dev_out, uint64_t elem_stride_bytes, int policy, cftft_mul_stats* stats,
                       void* stream) {
  if (!cring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (int rc = check_stride(cring, elem_stride_bytes)) return rc;
  if (policy != CFTFT_BALANCED && policy != CFTFT_RADIX2) return fail(CFTFT_INVALID_PARAMS, "unknown split policy");
  if (stats) *stats = cftft_mul_stats{0, 0, 0};
  if (zg == 0 || zh == 0) return CFTFT_OK;  // the zero polynomial (polymul.hpp:55)
  auto* R = const_cast<cftft_ring*>(cring);
  auto st = static_cast<cudaStream_t>(stream);
  const u64 n = zg + zh - 1;
  // choose_length (polymul.hpp:33-37)
  if (n > R->M)
    return fail(CFTFT_TOO_LARGE, "product length " + std::to_string(n) + " exceeds the available root order " +
                                     std::to_string(R->M));
  u64 L = 2;
  while (L < n) L <<= 1;
  const size_t eb = R->elem_bytes, sz = (size_t)L * elem_stride_bytes;
  std::uint8_t *g = nullptr, *h = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&g, 2 * sz, st));
  h = g + sz;
  int rc = CFTFT_OK;
  uint64_t c1 = 0, c2 = 0, c3 = 0;
  do {
    if (cudaMemcpy2DAsync(g, elem_stride_bytes, dev_g, elem_stride_bytes, eb, zg, cudaMemcpyDeviceToDevice, st) ||
        cudaMemcpy2DAsync(h, elem_stride_bytes, dev_h, elem_stride_bytes, eb, zh, cudaMemcpyDeviceToDevice, st)) {
      rc = fail(CFTFT_CUDA_ERROR, "poly_mul: staging copies");
      break;
    }
    const cftft_params pg{L, 0, zg, n, 0}, ph{L, 0, zh, n, 0}, pi{L, 0, n, n, 0};
    if ((rc = transform(R, false, &pg, g, elem_stride_bytes, policy, &c1, st))) break;
    if ((rc = transform(R, false, &ph, h, elem_stride_bytes, policy, &c2, st))) break;
    // exactly n pointwise products (polymul.hpp:73-77) with the final L^-1
    // (polymul.hpp:82-87) folded in: 2^(2N - ell) in Z/(2^N+1), L^-1 mod m / p
    unsigned ell = 0;
    while ((u64{1} << ell) < L) ++ell;
    u64 scale = 0;
    if (R->kind == CFTFT_RING_FERMAT) {
      scale = R->M - ell;
    } else {
      const u64 mod = R->m;
      auto mulm = [mod](u64 a, u64 b) { return (u64)((unsigned __int128)a * b % mod); };
      // L^-1 = (2^-1)^ell, 2^-1 = (mod + 1) / 2 (mod odd)
      u64 inv2 = (mod + 1) / 2, r = 1 % mod;
      for (unsigned k = 0; k < ell; ++k) r = mulm(r, inv2);
      scale = r;
    }
    if ((rc = cftft_gpu_pointwise_scaled(R, g, h, n, elem_stride_bytes, scale, st))) break;
    if ((rc = transform(R, true, &pi, g, elem_stride_bytes, policy, &c3, st))) break;
    if (cudaMemcpy2DAsync(dev_out, elem_stride_bytes, g, elem_stride_bytes, eb, n, cudaMemcpyDeviceToDevice, st)) {
      rc = fail(CFTFT_CUDA_ERROR, "poly_mul: output copy");
      break;
    }
  } while (false);
  cudaFreeAsync(g, st);
  if (rc) return rc;
  if (stats) *stats = cftft_mul_stats{n, L, c1 + c2 + c3};
  return CFTFT_OK;
}

int cftft_gpu_pack_limbs(const cftft_ring* ring, void* dev_dst, uint64_t elem_stride_bytes, const void* dev_src,
                         uint64_t src_words, uint64_t count, void* stream) {
  if (!ring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (int rc = check_stride(ring, elem_stride_bytes)) return rc;
  const u64 ew = ring->elem_bytes / 8;
  if (src_words > (ring->kind == CFTFT_RING_FERMAT ? ring->N / 64 : ew))
    return fail(CFTFT_INVALID_PARAMS, "source coefficients wider than the ring's elements");
  if (count == 0) return CFTFT_OK;
  if (count > 0x7FFFFFFFull) return fail(CFTFT_UNSUPPORTED, "too many elements for one launch");
  polymul::pack_limbs_kernel<<<(unsigned)count, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<std::uint8_t*>(dev_dst), elem_stride_bytes, static_cast<const std::uint8_t*>(dev_src), src_words,
      (u32)ew);
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

int cftft_gpu_nussbaumer_split(const cftft_ring* ring, void* dev_dst, uint64_t elem_stride_bytes,
                               const uint64_t* dev_f, uint64_t s, void* stream) {
  if (!ring || ring->kind != CFTFT_RING_NEGACYCLIC) return fail(CFTFT_INVALID_PARAMS, "a negacyclic ring is needed");
  if (int rc = check_stride(ring, elem_stride_bytes)) return rc;
  if (s == 0 || s > 0x7FFFFFFFull) return fail(CFTFT_INVALID_PARAMS, "bad split length");
  const dim3 grid((unsigned)((s + 31) / 32), (unsigned)((ring->K + 31) / 32)), block(32, 8);
  polymul::nuss_split_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<std::uint8_t*>(dev_dst), elem_stride_bytes, dev_f, (u32)ring->K, (u32)s);
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

int cftft_gpu_nussbaumer_join(const cftft_ring* ring, uint64_t* dev_h, const void* dev_c, uint64_t elem_stride_bytes,
                              uint64_t s, void* stream) {
  if (!ring || ring->kind != CFTFT_RING_NEGACYCLIC) return fail(CFTFT_INVALID_PARAMS, "a negacyclic ring is needed");
  if (int rc = check_stride(ring, elem_stride_bytes)) return rc;
  if (s == 0 || s > 0x7FFFFFFFull) return fail(CFTFT_INVALID_PARAMS, "bad split length");
  const dim3 grid((unsigned)((s + 31) / 32), (unsigned)((ring->K + 31) / 32)), block(32, 8);
  polymul::nuss_join_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(
      dev_h, static_cast<const std::uint8_t*>(dev_c), elem_stride_bytes, (u32)ring->K, (u32)s, ring->m);
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

int cftft_gpu_mul_scalar(const cftft_ring* ring, void* dev_base, uint64_t count, uint64_t elem_stride_bytes,
                         uint64_t c, void* stream) {
  if (!ring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (ring->kind != CFTFT_RING_NEGACYCLIC) return fail(CFTFT_UNSUPPORTED, "mul_scalar is for negacyclic rings");
  if (int rc = check_stride(ring, elem_stride_bytes)) return rc;
  if (count == 0) return CFTFT_OK;
  const u64 total = count * ring->K;
  pointwise::nega_scale_kernel<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<std::uint8_t*>(dev_base), elem_stride_bytes, count, (u32)ring->K, ring->m, c % ring->m);
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

int cftft_gpu_scale(const cftft_ring* cring, void* dev_base, uint64_t count,
                    uint64_t elem_stride_bytes, uint64_t e, void* stream) {
  if (!cring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (int rc = check_stride(cring, elem_stride_bytes)) return rc;
  if (count == 0) return CFTFT_OK;
  auto* R = const_cast<cftft_ring*>(cring);
  auto st = static_cast<cudaStream_t>(stream);
  if (R->kind == CFTFT_RING_FERMAT && (u64)R->D * 12 <= 200 * 1024) {
    // one CTA per element: word-parallel shift, block-scan borrows (rotate_kernel)
    const size_t sm = (size_t)R->D * 12 + 128;  // + borrow masks of a small ring
    if (sm > 40 * 1024)  // with the static scan scratch
      if (int rc = set_smem_bytes(fermat::rotate_kernel, sm)) return rc;
    fermat::rotate_kernel<<<(unsigned)count, 256, sm, st>>>(static_cast<std::uint8_t*>(dev_base), elem_stride_bytes,
                                                            e, R->D);
    CUDA_TRY(cudaGetLastError());
    g_last_launches = 1;
    return CFTFT_OK;
  }
  // A scale is a degenerate plan: one length-1 class (load, no ops, store
  // with rotation e) and one leaf per element.
  const u64 M = R->M;
  int sdev = 0;
  CUDA_TRY(cudaGetDevice(&sdev));
  PlanKey key{sdev, 2, 1, e & (M - 1), count, 0, 0, 0};
  DevicePlan* dp = nullptr;
  {
    std::lock_guard<std::mutex> g(R->mu);
    auto it = R->cache.find(key);
    if (it != R->cache.end()) {
      dp = it->second.get();
    } else {
      auto np = std::make_unique<DevicePlan>();
      LeafProgram lp;
      lp.key = ClassKey{0, 0, 1, 1, 0};
      lp.nload = 1;
      lp.nstore = 1;
      lp.level_begin = {0};
      lp.pre = {SymExp{}};
      lp.post = {SymExp{0, e & (M - 1)}};
      np->host.classes.push_back(lp);
      for (u64 i = 0; i < count; ++i) {
        DevLeaf lf{};
        lf.locoff = kNoDep;
        lf.cls = 0;
        lf.dep = kNoDep;
        lf.comp = kNoDep;
        lf.base = i;
        lf.stride = 1;
        np->host.leaves.push_back(lf);
      }
      np->host.max_ell = 0;
      np->host.final_count = count;
      np->cw = R->CW;
      np->C = R->C;
      np->slot_bytes = R->slot_bytes;
      if (int rc = upload(R, *np, st)) return rc;
      dp = np.get();
      R->cache[key] = std::move(np);
    }
  }
  return launch_plan(R, *dp, static_cast<std::uint8_t*>(dev_base), elem_stride_bytes, st, true);
}

int cftft_gpu_batch(const cftft_ring* cring, int inverse, const cftft_subtransform* items, uint64_t count,
                    void* dev_base, uint64_t elem_stride_bytes, int policy, int canonicalize, void* stream) {
  if (!cring || (!items && count)) return fail(CFTFT_INVALID_PARAMS, "null ring or items");
  if (int rc = check_stride(cring, elem_stride_bytes)) return rc;
  if (count == 0) return CFTFT_OK;
  auto* R = const_cast<cftft_ring*>(cring);
  std::vector<Planner::Item> v;
  v.reserve(count);
  for (u64 k = 0; k < count; ++k) {
    const cftft_subtransform& it = items[k];
    cftft_params p{it.length, it.twiddle_exp, it.input_count, it.output_count, it.want_next};
    if (int rc = validate(R, inverse != 0, &p, policy)) return rc;
    if (it.stride == 0) return fail(CFTFT_INVALID_PARAMS, "sub-transform stride must be >= 1");
    v.push_back(Planner::Item{it.length, it.twiddle_exp & (R->M - 1), it.input_count, it.output_count,
                              inverse ? it.want_next : 0, it.base, it.stride});
  }
  auto st = static_cast<cudaStream_t>(stream);
  // batches are planned per call (the multi-GPU passes reuse one shape many
  // times; the planner is fast) and cached by a content hash
  u64 h = 1469598103934665603ull;
  auto mix = [&](u64 x) { h = (h ^ x) * 1099511628211ull; };
  mix(inverse ? 1 : 0);
  mix((u64)policy);
  for (const auto& it : v) {
    mix(it.L); mix(it.s); mix(it.z); mix(it.n); mix((u64)it.f); mix(it.base); mix(it.stride);
  }
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  PlanKey key{dev, 3 + (inverse ? 1 : 0), h, count, v[0].L, v[0].base, policy, -1};
  std::vector<u64> bkey;
  bkey.reserve(v.size() * 7);
  for (const auto& it : v) bkey.insert(bkey.end(), {it.L, it.s, it.z, it.n, (u64)it.f, it.base, it.stride});
  DevicePlan* dp = nullptr;
  {
    std::lock_guard<std::mutex> g(R->mu);
    auto itc = R->cache.find(key);
    if (itc != R->cache.end() && itc->second->batch_items != bkey) {
      R->cache.erase(itc);  // a hash collision: replan
      itc = R->cache.end();
    }
    if (itc != R->cache.end()) {
      dp = itc->second.get();
    } else {
      // bounded: batch shapes beyond kMaxBatchPlans evict the cached batches
      size_t nb = 0;
      for (const auto& kv : R->cache) nb += std::get<1>(kv.first) >= 3;
      if (nb >= kMaxBatchPlans) {
        CUDA_TRY(cudaStreamSynchronize(st));  // their device buffers may still be in use
        for (auto it2 = R->cache.begin(); it2 != R->cache.end();)
          it2 = std::get<1>(it2->first) >= 3 ? R->cache.erase(it2) : std::next(it2);
      }
      auto np = std::make_unique<DevicePlan>();
      // radix-64 leaves where the sub-transforms have them (the multi-GPU
      // slabs of a wide ring: columns of 64, rows of L / 64)
      const RingShape rs = shape_of(R, v[0].L, np.get(), true);
      try {
        np->host = best_plan(rs, [&](Planner& pl) { return pl.build_batch(inverse != 0, v, policy); });
      } catch (const std::exception& ex) {
        return fail(CFTFT_UNSUPPORTED, ex.what());
      }
      if (int rc = upload(R, *np, st)) return rc;
      np->batch_items = std::move(bkey);
      dp = np.get();
      R->cache[key] = std::move(np);
    }
  }
  int rc = launch_plan(R, *dp, static_cast<std::uint8_t*>(dev_base), elem_stride_bytes, st, false);
  if (rc) return rc;
  if (!inverse && g_fault.load()) {
    // fault::corrupt_tft_base: every forward sub-transform's x[0] += 1
    std::vector<u64> idx(count);
    for (u64 k = 0; k < count; ++k) idx[k] = v[k].base;
    u64* di = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&di, count * 8, st));
    CUDA_TRY(cudaMemcpyAsync(di, idx.data(), count * 8, cudaMemcpyHostToDevice, st));
    // (batch outputs of whole-leaf plans are canonicalised first below)
    if (canonicalize && R->kind == CFTFT_RING_FERMAT && !dp->host.coset) {
      for (u64 k = 0; k < count; ++k) {
        const u64 outs = v[k].n + (u64)v[k].f;
        std::uint8_t* b = static_cast<std::uint8_t*>(dev_base) + v[k].base * elem_stride_bytes;
        fermat::canonicalize_kernel<<<(unsigned)((outs + 255) / 256), 256, 0, st>>>(
            b, elem_stride_bytes * v[k].stride, outs, R->D);
      }
    }
    fault_add_one_items_kernel<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(
        static_cast<std::uint8_t*>(dev_base), elem_stride_bytes, di, count, R->kind,
        R->kind == CFTFT_RING_NEGACYCLIC ? R->K : (u64)R->D, R->m);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaFreeAsync(di, st));
    return CFTFT_OK;
  }
  // coset plans end in the carry-save fold: their outputs are canonical already
  if (!canonicalize || R->kind != CFTFT_RING_FERMAT || dp->host.coset) return rc;
  for (u64 k = 0; k < count; ++k) {
    const u64 outs = v[k].n + (u64)v[k].f;
    std::uint8_t* b = static_cast<std::uint8_t*>(dev_base) + v[k].base * elem_stride_bytes;
    if (v[k].stride == 1) {
      fermat::canonicalize_kernel<<<(unsigned)((outs + 255) / 256), 256, 0, st>>>(b, elem_stride_bytes, outs, R->D);
    } else {
      fermat::canonicalize_kernel<<<(unsigned)((outs + 255) / 256), 256, 0, st>>>(
          b, elem_stride_bytes * v[k].stride, outs, R->D);
    }
  }
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

int cftft_gpu_canonicalize(const cftft_ring* ring, void* dev_base, uint64_t count, uint64_t elem_stride_bytes,
                           void* stream) {
  if (!ring) return fail(CFTFT_INVALID_PARAMS, "null ring");
  if (int rc = check_stride(ring, elem_stride_bytes)) return rc;
  if (ring->kind != CFTFT_RING_FERMAT || count == 0) return CFTFT_OK;
  fermat::canonicalize_kernel<<<(unsigned)((count + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<std::uint8_t*>(dev_base), elem_stride_bytes, count, ring->D);
  CUDA_TRY(cudaGetLastError());
  return CFTFT_OK;
}

uint64_t cftft_tft_base_cases(uint64_t L, uint64_t z, uint64_t n, int policy) {
  CountReplay c;
  return c.tft(L, z, n, policy);
}
uint64_t cftft_itft_base_cases(uint64_t L, uint64_t z, uint64_t n, int f, int policy) {
  CountReplay c;
  return c.itft(L, z, n, f, policy);
}

uint64_t cftft_last_launch_count(void) { return g_last_launches; }
void cftft_set_fault_injection(int on) { g_fault.store(on ? 1 : 0); }
void cftft_set_launch_timing(int on) { g_timing.store(on ? 1 : 0); }
uint64_t cftft_launch_timing_read(cftft_launch_record* out, uint64_t max) {
  // waits for the recorded launches; returns (and forgets) this thread's records
  const u64 n = g_timed.size();
  for (u64 i = 0; i < n; ++i) {
    TimedLaunch& t = g_timed[i];
    float ms = 0.f;
    cudaEventSynchronize(t.e1);
    cudaEventElapsedTime(&ms, t.e0, t.e1);
    if (out && i < max) {
      std::snprintf(out[i].kernel, sizeof out[i].kernel, "%s", t.kernel);
      out[i].algorithmic_bytes = t.bytes;
      out[i].ms = ms;
    }
    g_event_pool.push_back(t.e0);
    g_event_pool.push_back(t.e1);
  }
  g_timed.clear();
  return n;
}
int cftft_fault_injection(void) { return g_fault.load(); }
void cftft_set_debug_poison(int on) { g_poison.store(on ? 1 : 0); }

size_t cftft_plan_dump(const cftft_ring* ring, int inverse, const cftft_params* params, int policy,
                       char* buf, size_t cap) {
  if (validate(ring, inverse != 0, params, policy)) return 0;
  DevicePlan geo;
  const RingShape rs = shape_of(ring, params->length, &geo);
  Plan p;
  try {
    p = best_plan(rs, [&](Planner& pl) {
      return pl.build(inverse != 0, params->length, params->twiddle_exp, params->input_count,
                      params->output_count, inverse ? params->want_next : 0, policy);
    });
  } catch (const std::exception&) {
    return 0;
  }
  std::ostringstream os;
  json_plan(os, p, rs.lane_bits);
  std::string s = os.str();
  if (buf && cap) {
    size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return s.size() + 1;
}

const char* cftft_last_error(void) { return g_last_error.c_str(); }
const char* cftft_version(void) { return "cftft-b200 0.1 (sm_100a)"; }

}  // extern "C"

// ---------------------------------------------------------------------------
// Multi-GPU transforms (dist.cuh): one transform partitioned over an NCCL
// communicator's ranks.

struct cftft_dist {
  const cftft_ring* ring = nullptr;
  ncclComm_t comm = nullptr;
  bool owns = false;
  int rank = 0, world = 1, device = 0;
  cudaStream_t comm_stream = nullptr;  // the TFT's transposes run here, behind the column chunks
  cudaEvent_t ev = nullptr;
};

namespace {
#define NCCL_TRY(expr)                                                                                  \
  do {                                                                                                  \
    ncclResult_t r_ = (expr);                                                                           \
    if (r_ != ncclSuccess)                                                                              \
      return fail(CFTFT_CUDA_ERROR, std::string(#expr ": ") +                                           \
                                        (dist::nccl().GetErrorString ? dist::nccl().GetErrorString(r_) \
                                                                     : "nccl error"));                  \
  } while (0)

cftft_subtransform sub(u64 L, u64 s, u64 z, u64 n, int f, u64 base, u64 stride) {
  cftft_subtransform t{};
  t.length = L;
  t.twiddle_exp = s;
  t.input_count = z;
  t.output_count = n;
  t.want_next = f;
  t.base = base;
  t.stride = stride;
  return t;
}
int run_subs(const cftft_dist* d, int inverse, const std::vector<cftft_subtransform>& v, void* slab, u64 esb,
             int policy, cudaStream_t st) {
  if (v.empty()) return CFTFT_OK;
  return cftft_gpu_batch(d->ring, inverse, v.data(), v.size(), slab, esb, policy, 1, st);
}
// the ring's transforms of length L run radix-64 coset leaves: the slabs take
// the (6, ell - 6) split of the single-GPU plan
// While a chunk's transpose runs on the context's stream the next chunk's
// persistent wave CTAs would hold every SM; they leave this many free, so
// NCCL's send / receive kernels start at once instead of in the gaps
// between launches.  (One rank: NCCL's self-copies gain nothing from it --
// measured 989 -> 975 GB/s -- so nothing is reserved there.)
constexpr int kDistSmReserve = 8;
struct SmReserve {
  int old;
  explicit SmReserve(int n) : old(t_sm_reserve) { t_sm_reserve = n; }
  ~SmReserve() { t_sm_reserve = old; }
};
// one NCCL group of transpose pieces (dist.cuh) on stream st
int run_pieces(const cftft_dist* d, const std::vector<dist::Piece>& v, void* colslab, void* rowslab, u64 esb,
               cudaStream_t st) {
  auto& nc = dist::nccl();
  NCCL_TRY(nc.GroupStart());
  for (const dist::Piece& pc : v) {
    std::uint8_t* at = static_cast<std::uint8_t*>(pc.buf ? rowslab : colslab) + pc.off * esb;
    if (pc.send)
      NCCL_TRY(nc.Send(at, pc.count * esb, ncclUint8, (int)pc.peer, d->comm, st));
    else
      NCCL_TRY(nc.Recv(at, pc.count * esb, ncclUint8, (int)pc.peer, d->comm, st));
  }
  NCCL_TRY(nc.GroupEnd());
  return CFTFT_OK;
}
bool dist_wide(const cftft_ring* R, u64 L) {
  DevicePlan geo;
  return shape_of(R, L, &geo).wide;
}
int check_dist(const cftft_dist* d, const cftft_params* p, int inverse, int policy, u64 esb) {
  if (!d || !d->ring || !p) return fail(CFTFT_INVALID_PARAMS, "null argument");
  if (int rc = validate(d->ring, inverse != 0, p, policy)) return rc;
  if (int rc = check_stride(d->ring, esb)) return rc;
  if (esb % 16) return fail(CFTFT_UNSUPPORTED, "distributed slabs need a 16-byte element stride");
  return CFTFT_OK;
}
}  // namespace

int cftft_nccl_unique_id(void* out) {
  if (!out) return fail(CFTFT_INVALID_PARAMS, "null id buffer");
  auto& n = dist::nccl();
  if (!n.ok()) return fail(CFTFT_UNSUPPORTED, "libnccl.so.2 not found");
  ncclUniqueId id;
  NCCL_TRY(n.GetUniqueId(&id));
  std::memcpy(out, &id, sizeof id);
  return CFTFT_OK;
}

int cftft_dist_create(const cftft_ring* ring, int rank, int world, const void* nccl_id, cftft_dist** out) {
  if (!ring || !nccl_id || !out || world < 1 || rank < 0 || rank >= world)
    return fail(CFTFT_INVALID_PARAMS, "bad distributed context arguments");
  auto& n = dist::nccl();
  if (!n.ok()) return fail(CFTFT_UNSUPPORTED, "libnccl.so.2 not found");
  auto d = std::make_unique<cftft_dist>();
  d->ring = ring;
  d->rank = rank;
  d->world = world;
  CUDA_TRY(cudaGetDevice(&d->device));
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof id);
  NCCL_TRY(n.CommInitRank(&d->comm, world, id, rank));
  d->owns = true;
  CUDA_TRY(cudaStreamCreateWithFlags(&d->comm_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&d->ev, cudaEventDisableTiming));
  *out = d.release();
  return CFTFT_OK;
}

int cftft_dist_create_from_comm(const cftft_ring* ring, void* nccl_comm, cftft_dist** out) {
  if (!ring || !nccl_comm || !out) return fail(CFTFT_INVALID_PARAMS, "bad distributed context arguments");
  auto& n = dist::nccl();
  if (!n.ok() || !n.CommCount || !n.CommUserRank) return fail(CFTFT_UNSUPPORTED, "libnccl.so.2 not found");
  auto d = std::make_unique<cftft_dist>();
  d->ring = ring;
  d->comm = static_cast<ncclComm_t>(nccl_comm);
  NCCL_TRY(n.CommCount(d->comm, &d->world));
  NCCL_TRY(n.CommUserRank(d->comm, &d->rank));
  CUDA_TRY(cudaGetDevice(&d->device));
  CUDA_TRY(cudaStreamCreateWithFlags(&d->comm_stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&d->ev, cudaEventDisableTiming));
  *out = d.release();
  return CFTFT_OK;
}

void cftft_dist_destroy(cftft_dist* d) {
  if (!d) return;
  if (d->owns && d->comm && dist::nccl().CommDestroy) dist::nccl().CommDestroy(d->comm);
  if (d->comm_stream) cudaStreamDestroy(d->comm_stream);
  if (d->ev) cudaEventDestroy(d->ev);
  delete d;
}

int cftft_dist_geometry(const cftft_dist* d, const cftft_params* p, int inverse, int policy, uint64_t* out) {
  if (!d || !p || !out) return fail(CFTFT_INVALID_PARAMS, "null argument");
  if (int rc = validate(d->ring, inverse != 0, p, policy)) return rc;
  const dist::Geometry g(d->ring->M, p->length, p->input_count, p->output_count, (u64)d->world, policy,
                         inverse != 0, inverse ? p->want_next : 0, dist_wide(d->ring, p->length));
  const u64 r = (u64)d->rank;
  const u64 v[8] = {g.c0[r], g.c1[r], g.r0[r], g.r1[r], g.L1, g.L2, g.L1 * g.width(r), g.nrows(r) * g.L2};
  std::memcpy(out, v, sizeof v);
  return CFTFT_OK;
}

size_t cftft_dist_schedule(uint64_t M, const cftft_params* p, int inverse, int policy, int wide, int world,
                           int rank, uint64_t* out, size_t cap) {
  if (!p || world < 1 || rank < 0 || rank >= world) return 0;
  const dist::Geometry g(M, p->length, p->input_count, p->output_count, (u64)world, policy, inverse != 0,
                         inverse ? p->want_next : 0, wide != 0);
  const u64 K = inverse ? dist::itft_chunks(g) : dist::tft_chunks(g);
  size_t n = 0;
  for (u64 k = 0; k < K; ++k) {
    const auto v = inverse ? dist::itft_transpose(g, (u64)rank, k) : dist::tft_transpose(g, (u64)rank, k);
    for (const dist::Piece& pc : v) {
      const u64 rec[6] = {k, pc.send, pc.peer, pc.buf, pc.off, pc.count};
      if (out && n + 6 <= cap) std::memcpy(out + n, rec, sizeof rec);
      n += 6;
    }
  }
  return n;
}

int cftft_gpu_dist_tft(const cftft_dist* d, const cftft_params* p, void* colslab, void* rowslab,
                       uint64_t esb, int policy, void* stream) {
  if (int rc = check_dist(d, p, 0, policy, esb)) return rc;
  SmReserve reserve(d->world > 1 ? kDistSmReserve : 0);
  auto st = static_cast<cudaStream_t>(stream);
  const cftft_ring* R = d->ring;
  const dist::Geometry g(R->M, p->length, p->input_count, p->output_count, (u64)d->world, policy, false, 0,
                         dist_wide(R, p->length));
  const u64 me = (u64)d->rank, W = g.width(me);
  const u64 s = p->twiddle_exp & (R->M - 1), s_row = (s << g.l1) & (R->M - 1);
  // 1. column TFTs (transform.hpp:175-180) in chunks of adjacent columns, and
  // 2. the transpose of each chunk behind it on the communicator's stream:
  //    row r of R_q, the chunk's columns -> rank q, received straight into
  //    place in q's row slab (the piece is contiguous on both sides: no pack
  //    or unpack pass, no staging buffer).  Chunk k's sends overlap chunk
  //    k+1's column pass; ranks issue the same chunks in the same order.
  const u64 K = dist::tft_chunks(g);
  cudaStream_t cst = d->comm_stream;
  cudaEvent_t ev = d->ev;
  std::vector<cftft_subtransform> v;
  for (u64 k = 0; k < K; ++k) {
    u64 a, b;
    dist::tft_chunk_cols(g, me, k, a, b);
    v.clear();
    for (u64 c = a; c < b; ++c) {
      const u64 u = g.c0[me] + c;
      if (u >= g.z2e) continue;
      v.push_back(sub(g.L1, (s + u * g.col_step) & (R->M - 1), u < g.z2 ? g.z1 + 1 : g.z1, g.n1c, 0, c, W));
    }
    if (int rc = run_subs(d, 0, v, colslab, esb, policy, st)) return rc;
    CUDA_TRY(cudaEventRecord(ev, st));
    CUDA_TRY(cudaStreamWaitEvent(cst, ev, 0));
    if (int rc = run_pieces(d, dist::tft_transpose(g, me, k), colslab, rowslab, esb, cst)) return rc;
  }
  CUDA_TRY(cudaEventRecord(ev, cst));
  CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
  // 3. row TFTs (transform.hpp:182-185)
  v.clear();
  for (u64 u = g.r0[me]; u < g.r1[me]; ++u)
    v.push_back(sub(g.L2, s_row, g.z2e, u < g.n1 ? g.L2 : g.n2, 0, (u - g.r0[me]) * g.L2, 1));
  return run_subs(d, 0, v, rowslab, esb, policy, st);
}

int cftft_gpu_dist_itft(const cftft_dist* d, const cftft_params* p, void* rowslab, void* colslab,
                        uint64_t esb, int policy, void* stream) {
  if (int rc = check_dist(d, p, 1, policy, esb)) return rc;
  SmReserve reserve(d->world > 1 ? kDistSmReserve : 0);
  auto& nc = dist::nccl();
  auto st = static_cast<cudaStream_t>(stream);
  const cftft_ring* R = d->ring;
  const int f = p->want_next;
  const dist::Geometry g(R->M, p->length, p->input_count, p->output_count, (u64)d->world, policy, true, f,
                         dist_wide(R, p->length));
  const u64 P = (u64)d->world, me = (u64)d->rank, W = g.width(me);
  const u64 r0 = g.r0[me], r1 = g.r1[me], c0 = g.c0[me];
  const u64 n1 = g.n1, n2 = g.n2, z1 = g.z1, z2e = g.z2e;
  const u64 fm = (n2 + (u64)f) > 0 ? 1 : 0, lo = std::min(n2, g.z2), hi = std::max(n2, g.z2);
  const u64 s = p->twiddle_exp & (R->M - 1), s_row = (s << g.l1) & (R->M - 1);
  auto* rs = static_cast<std::uint8_t*>(rowslab);
  auto* cs = static_cast<std::uint8_t*>(colslab);
  // i. full rows u < n1 (transform.hpp:215-216), in chunks of rows; each
  // chunk's rows then go to the column owners on the communicator's stream
  // while the next chunk is transformed: the columns [c0_q, c1_q) of a row
  // leave as they lie (contiguous in the row), rank q's rows arrive in
  // global row order, straight into the column slab.  Every rank cuts every
  // rank's rows [r0_q, min(r1_q, zrows)) the same way.
  std::vector<cftft_subtransform> v;
  {
    cudaStream_t cst = d->comm_stream;
    cudaEvent_t ev = d->ev;
    const u64 K = dist::itft_chunks(g);
    // rows of mine at or past zrows (none are sent) still take phase i
    for (u64 u = std::max(r0, std::min(r1, g.zrows)); u < std::min(r1, n1); ++u)
      v.push_back(sub(g.L2, s_row, g.L2, g.L2, 0, (u - r0) * g.L2, 1));
    if (int rc = run_subs(d, 1, v, rowslab, esb, policy, st)) return rc;
    for (u64 k = 0; k < K; ++k) {
      u64 a, b;
      dist::itft_chunk_rows(g, me, k, a, b);
      v.clear();
      for (u64 u = a; u < std::min(b, n1); ++u) v.push_back(sub(g.L2, s_row, g.L2, g.L2, 0, (u - r0) * g.L2, 1));
      if (int rc = run_subs(d, 1, v, rowslab, esb, policy, st)) return rc;
      CUDA_TRY(cudaEventRecord(ev, st));
      CUDA_TRY(cudaStreamWaitEvent(cst, ev, 0));
      if (int rc = run_pieces(d, dist::itft_transpose(g, me, k), colslab, rowslab, esb, cst)) return rc;
    }
    CUDA_TRY(cudaEventRecord(ev, cst));
    CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
  }
  // ii. right columns [n2, z2') (transform.hpp:219-224)
  v.clear();
  for (u64 c = 0; c < W; ++c) {
    const u64 u = c0 + c;
    if (n2 <= u && u < z2e)
      v.push_back(sub(g.L1, (s + u * g.col_step) & (R->M - 1), u < hi ? z1 + 1 : z1, n1, (int)fm, c, W));
  }
  if (int rc = run_subs(d, 1, v, colslab, esb, policy, st)) return rc;
  // iii. row n1 (transform.hpp:227-230): gather, transform on its owner, scatter
  if (fm) {
    u64 owner = 0;
    for (u64 q = 0; q < P; ++q)
      if (g.r0[q] <= n1 && n1 < g.r1[q]) owner = q;
    std::uint8_t* row = me == owner ? rs + (n1 - g.r0[owner]) * g.L2 * esb : nullptr;
    NCCL_TRY(nc.GroupStart());
    {
      const u64 a = std::max(n2, c0), b = std::min(z2e, g.c1[me]);
      if (b > a) {
        if (me == owner) {
          CUDA_TRY(cudaMemcpyAsync(row + a * esb, cs + (n1 * W + (a - c0)) * esb, (b - a) * esb,
                                   cudaMemcpyDeviceToDevice, st));
        } else {
          NCCL_TRY(nc.Send(cs + (n1 * W + (a - c0)) * esb, (b - a) * esb, ncclUint8, (int)owner, d->comm, st));
        }
      }
      if (me == owner)
        for (u64 q = 0; q < P; ++q) {
          const u64 aa = std::max(n2, g.c0[q]), bb = std::min(z2e, g.c1[q]);
          if (q != me && bb > aa) NCCL_TRY(nc.Recv(row + aa * esb, (bb - aa) * esb, ncclUint8, (int)q, d->comm, st));
        }
    }
    NCCL_TRY(nc.GroupEnd());
    if (me == owner) {
      v.assign(1, sub(g.L2, s_row, z2e, n2, f, (n1 - g.r0[owner]) * g.L2, 1));
      if (int rc = run_subs(d, 1, v, rowslab, esb, policy, st)) return rc;
    }
    const u64 outs = n2 + (u64)f;
    NCCL_TRY(nc.GroupStart());
    {
      const u64 aa = c0, bb = std::min(outs, g.c1[me]);
      if (bb > aa) {
        if (me == owner) {
          CUDA_TRY(cudaMemcpyAsync(cs + n1 * W * esb, row + aa * esb, (bb - aa) * esb, cudaMemcpyDeviceToDevice, st));
        } else {
          NCCL_TRY(nc.Recv(cs + n1 * W * esb, (bb - aa) * esb, ncclUint8, (int)owner, d->comm, st));
        }
      }
      if (me == owner)
        for (u64 q = 0; q < P; ++q) {
          const u64 qa = g.c0[q], qb = std::min(outs, g.c1[q]);
          if (q != me && qb > qa) NCCL_TRY(nc.Send(row + qa * esb, (qb - qa) * esb, ncclUint8, (int)q, d->comm, st));
        }
    }
    NCCL_TRY(nc.GroupEnd());
  }
  // iv. left columns [0, n2) (transform.hpp:233-238)
  v.clear();
  for (u64 c = 0; c < W; ++c) {
    const u64 u = c0 + c;
    if (u < n2) v.push_back(sub(g.L1, (s + u * g.col_step) & (R->M - 1), u < lo ? z1 + 1 : z1, n1 + 1, 0, c, W));
  }
  return run_subs(d, 1, v, colslab, esb, policy, st);
}
