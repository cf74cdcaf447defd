// cftft_cli.cpp -- the command-line workbench (the reference's
// tools/cftft_cli.cpp contract: subcommands verify / count / bench / compare,
// the same flags, CSV headers and exit codes) on the GPU engine, for the
// reference's own prime field and the two big rings:
//
//   cftft verify  [--max-ell K] [--seed S] [--inject-fault] RING
//   cftft count   --length L [--policy balanced|radix2] RING
//   cftft bench   [--min A --max B --step-pct P --trials T --seed S] [--policy P] RING
//   cftft compare [--min A --max B --step-pct P --trials T --seed S] RING
//   RING: [--ring prime|fermat:N|negacyclic:K,M] [--modulus P] [--two-adicity M]
//         [--device cuda]
//
// verify runs the reference's five suites (verify.hpp:85-269): the GPU
// transforms against a host naive DFT (dft_naive, transform.hpp:292-311,
// restated here over each ring), ITFT inversion, and the base-case count
// bounds; every (L <= 2^K, z, n[, f], policy) case of a suite and length runs
// in one batched launch (cftft_gpu_batch).  bench times GPU poly_mul over the
// reference's geometric grid (bench.hpp:18-98).  Exit status: 0 pass, 1 a
// suite failed, 2 bad arguments / errors (the reference's CLI11 parse errors
// also exit nonzero).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cerrno>
#include <cstring>
#include <memory>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "../../include/cftft_b200.hpp"

namespace cf = cftft_b200;
using u64 = std::uint64_t;

namespace {

struct ArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

u64 mix_seed(u64 a, u64 b) {  // verify.hpp:17-25
  u64 x = a + 0x9e3779b97f4a7c15ull * (b + 1);
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

u64 bit_reverse(u64 j, unsigned ell) {
  u64 r = 0;
  for (unsigned i = 0; i < ell; ++i, j >>= 1) r = (r << 1) | (j & 1);
  return r;
}

// ---------------------------------------------------------------------------
// Host rings: element = words (u64) in the engine's format; add, twiddle
// (omega^k x), L x, random elements, the poison fill of unspecified cells.
struct HostRing {
  virtual ~HostRing() = default;
  virtual u64 words() const = 0;   // u64 words per element (the engine's stride / 8)
  virtual u64 M() const = 0;       // root order
  virtual void random(std::mt19937_64& g, u64* x) const = 0;
  virtual void add(u64* acc, const u64* x) const = 0;              // acc += x
  virtual void twiddle(u64* out, const u64* x, u64 k) const = 0;   // out = omega^k x
  virtual void mul_small(u64* x, u64 c) const = 0;                  // x *= c (c small)
  virtual bool is_zero(const u64* x) const = 0;
  virtual u64 value_words() const { return words(); }  // the words that carry the value (no padding)
  // elements [0, count) of two arrays of `words()`-word elements agree
  bool same(const u64* a, const u64* b, u64 count) const {
    const u64 W = words(), V = value_words();
    for (u64 e = 0; e < count; ++e)
      if (!std::equal(a + e * W, a + e * W + V, b + e * W)) return false;
    return true;
  }
};

struct HostPrime : HostRing {
  u64 p, om, m2;
  HostPrime(u64 p_, unsigned m) : p(p_) {
    m2 = u64{1} << m;
    om = 0;  // the reference's root (field.hpp:170-177): smallest g with g^((p-1)/2^m) of order 2^m
    for (u64 g = 2; g < 1024 && !om; g = (g == 2) ? 3 : g + 2) {
      const u64 w = pw(g % p, (p - 1) >> m);
      if (pw(w, m2 / 2) == p - 1) om = w;
    }
  }
  u64 mul(u64 a, u64 b) const { return (u64)((unsigned __int128)a * b % p); }
  u64 pw(u64 a, u64 e) const {
    u64 r = 1 % p;
    for (; e; e >>= 1, a = mul(a, a))
      if (e & 1) r = mul(r, a);
    return r;
  }
  u64 words() const override { return 1; }
  u64 M() const override { return m2; }
  void random(std::mt19937_64& g, u64* x) const override { x[0] = g() % p; }
  void add(u64* acc, const u64* x) const override {
    const u64 s = acc[0] + x[0];
    acc[0] = (s < acc[0] || s >= p) ? s - p : s;
  }
  void twiddle(u64* out, const u64* x, u64 k) const override { out[0] = mul(pw(om, k % m2), x[0]); }
  void mul_small(u64* x, u64 c) const override { x[0] = mul(x[0], c % p); }
  bool is_zero(const u64* x) const override { return x[0] == 0; }
};

// Z/(2^N+1): N/64 limbs then a top word; canonical values in [0, 2^N]
struct HostFermat : HostRing {
  u64 N, lim, w;
  explicit HostFermat(u64 N_, u64 stride_words) : N(N_), lim(N_ / 64), w(stride_words) {}
  u64 words() const override { return w; }
  u64 value_words() const override { return lim + 1; }
  u64 M() const override { return 2 * N; }
  void random(std::mt19937_64& g, u64* x) const override {
    for (u64 k = 0; k < w; ++k) x[k] = k < lim ? g() : 0;
  }
  // value of x as (lo limbs, top in {0, 1}); add two canonical values
  void add(u64* acc, const u64* x) const override {
    unsigned __int128 cy = 0;
    for (u64 k = 0; k < lim; ++k) {
      cy += (unsigned __int128)acc[k] + x[k];
      acc[k] = (u64)cy;
      cy >>= 64;
    }
    const long long top = (long long)cy + (long long)acc[lim] + (long long)x[lim];  // 0..3
    acc[lim] = 0;
    normalize(acc, top);
  }
  // lo + top 2^N with top in [-3, 3] -> canonical
  void normalize(u64* x, long long top) const {
    // 2^N == -1: lo + top 2^N == lo - top
    if (top > 0) {
      u64 b = (u64)top;
      for (u64 k = 0; k < lim && b; ++k) {
        const u64 v = x[k];
        x[k] = v - b;
        b = v < b ? 1 : 0;
      }
      if (b) {  // negative: add 2^N + 1
        unsigned __int128 cy = 1;
        for (u64 k = 0; k < lim && cy; ++k) {
          cy += x[k];
          x[k] = (u64)cy;
          cy >>= 64;
        }
        // lo - top + 2^N + 1 with lo - top in [-3, 0): result < 2^N + 1; if it overflowed past 2^N...
        if (cy) x[lim] = 1;  // exactly 2^N (all limbs wrapped to 0)
      }
    } else if (top < 0) {
      unsigned __int128 cy = (u64)(-top);
      for (u64 k = 0; k < lim && cy; ++k) {
        cy += x[k];
        x[k] = (u64)cy;
        cy >>= 64;
      }
      if (cy) normalize(x, 1);  // carried into 2^N
    }
    // lo == 2^N exactly is represented as top 1, limbs 0: only reachable via the wrap above
  }
  // out = 2^k x (k mod 2N): rotation with the wrapped bits subtracted
  void twiddle(u64* out, const u64* x, u64 k) const override {
    k %= 2 * N;
    // value v in [0, 2^N]; 2^N v == -v
    bool neg = false;
    if (k >= N) {
      k -= N;
      neg = true;
    }
    std::vector<u64> v(x, x + lim + 1);
    if (v[lim]) {  // v = 2^N == -1: 2^k (-1)
      std::fill(v.begin(), v.end(), 0);
      v[0] = 1;
      neg = !neg;
    }
    // v 2^k = lo part (v << k mod 2^N) + hi part (v >> (N - k)) 2^N == lo - hi
    std::vector<u64> lo(lim, 0), hi(lim, 0);
    const u64 ws = k / 64, bs = k % 64;
    for (u64 i = 0; i < lim; ++i) {
      // bit position of limb i after the shift: i*64 + k
      const u64 a = v[i];
      const u64 t = i + ws;
      const u64 p0 = bs ? a << bs : a, p1 = bs ? a >> (64 - bs) : 0;
      if (t < lim) lo[t] |= p0; else hi[t - lim] |= p0;
      if (t + 1 < lim) lo[t + 1] |= p1; else if (t + 1 - lim < lim) hi[t + 1 - lim] |= p1;
    }
    // r = lo - hi (mod 2^N + 1)
    std::vector<u64> r(lim + 1, 0);
    u64 b = 0;
    for (u64 i = 0; i < lim; ++i) {
      const unsigned __int128 d = (unsigned __int128)lo[i] - hi[i] - b;
      r[i] = (u64)d;
      b = (u64)(d >> 127) & 1;
    }
    if (b) {  // negative: + 2^N + 1
      unsigned __int128 cy = 1;
      for (u64 i = 0; i < lim && cy; ++i) {
        cy += r[i];
        r[i] = (u64)cy;
        cy >>= 64;
      }
      if (cy) r[lim] = 1;
    }
    if (neg) negate(r.data());
    std::copy(r.begin(), r.end(), out);
    for (u64 i = lim + 1; i < w; ++i) out[i] = 0;
  }
  void negate(u64* r) const {
    bool zero = r[lim] == 0;
    for (u64 i = 0; i < lim && zero; ++i) zero = r[i] == 0;
    if (zero) return;
    if (r[lim]) {  // -(2^N) = 1
      for (u64 i = 0; i < lim; ++i) r[i] = 0;
      r[lim] = 0;
      r[0] = 1;
      return;
    }
    // 2^N + 1 - v = ~v + 2 (limbs), v in (0, 2^N)
    unsigned __int128 cy = 2;
    for (u64 i = 0; i < lim; ++i) {
      cy += (u64)~r[i];
      r[i] = (u64)cy;
      cy >>= 64;
    }
    r[lim] = (u64)cy;  // 1 only when v == 1 (result 2^N)
    if (r[lim]) for (u64 i = 0; i < lim; ++i) r[i] = 0;
  }
  void mul_small(u64* x, u64 c) const override {
    std::vector<u64> acc(w, 0), t(x, x + w);
    for (; c; c >>= 1) {
      if (c & 1) add(acc.data(), t.data());
      std::vector<u64> d(t);
      add(t.data(), d.data());
    }
    std::copy(acc.begin(), acc.end(), x);
  }
  bool is_zero(const u64* x) const override {
    for (u64 i = 0; i <= lim; ++i)
      if (x[i]) return false;
    return true;
  }
};

// (Z/mZ)[y]/(y^K+1): K words in [0, m); omega = y
struct HostNega : HostRing {
  u64 K, m;
  HostNega(u64 K_, u64 m_) : K(K_), m(m_) {}
  u64 words() const override { return K; }
  u64 M() const override { return 2 * K; }
  void random(std::mt19937_64& g, u64* x) const override {
    for (u64 k = 0; k < K; ++k) x[k] = g() % m;
  }
  void add(u64* acc, const u64* x) const override {
    for (u64 k = 0; k < K; ++k) {
      const u64 s = acc[k] + x[k];
      acc[k] = s >= m ? s - m : s;
    }
  }
  void twiddle(u64* out, const u64* x, u64 r) const override {
    r %= 2 * K;
    for (u64 k = 0; k < K; ++k) {
      const u64 t = k + r;
      const u64 v = x[k];
      const bool neg = (t / K) & 1;
      out[t % K] = neg ? (v ? m - v : 0) : v;
    }
  }
  void mul_small(u64* x, u64 c) const override {
    for (u64 k = 0; k < K; ++k) x[k] = (u64)((unsigned __int128)x[k] * c % m);
  }
  bool is_zero(const u64* x) const override {
    for (u64 k = 0; k < K; ++k)
      if (x[k]) return false;
    return true;
  }
};

// ---------------------------------------------------------------------------
struct Options {
  std::string cmd;
  std::string ring = "prime", device = "cuda";
  u64 modulus = 0xFFFFFFFF00000001ull;
  unsigned two_adicity = 32;
  unsigned max_ell = 6;
  u64 seed = 42;
  bool inject_fault = false;
  u64 length = 0;
  int policy = CFTFT_BALANCED;
  u64 min_n = 512, max_n = 16384;
  unsigned step_pct = 5, trials = 3;
};

u64 parse_u64(const std::string& flag, const char* v) {
  if (!v) throw ArgError(flag + " needs a value");
  char* end = nullptr;
  errno = 0;
  const unsigned long long x = std::strtoull(v, &end, 10);
  if (errno || !end || *end || v[0] == '-') throw ArgError(flag + ": not a non-negative integer: " + v);
  return x;
}

Options parse(int argc, char** argv) {
  if (argc < 2) throw ArgError("a subcommand is required: verify, count, bench or compare");
  Options o;
  o.cmd = argv[1];
  if (o.cmd != "verify" && o.cmd != "count" && o.cmd != "bench" && o.cmd != "compare")
    throw ArgError("unknown subcommand " + o.cmd);
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    const char* v = i + 1 < argc ? argv[i + 1] : nullptr;
    auto take = [&]() {
      ++i;
      return v;
    };
    if (a == "--inject-fault" && o.cmd == "verify") {
      o.inject_fault = true;
    } else if (a == "--max-ell" && o.cmd == "verify") {
      o.max_ell = (unsigned)parse_u64(a, take());
      if (o.max_ell < 1 || o.max_ell > 8) throw ArgError("--max-ell must be in [1, 8]");
    } else if (a == "--seed" && o.cmd != "count") {
      o.seed = parse_u64(a, take());
    } else if (a == "--length" && o.cmd == "count") {
      o.length = parse_u64(a, take());
    } else if (a == "--policy" && (o.cmd == "count" || o.cmd == "bench")) {
      std::string p = take() ? v : "";
      std::transform(p.begin(), p.end(), p.begin(), ::tolower);
      if (p == "balanced") o.policy = CFTFT_BALANCED;
      else if (p == "radix2") o.policy = CFTFT_RADIX2;
      else throw ArgError("--policy must be balanced or radix2");
    } else if (a == "--min" && (o.cmd == "bench" || o.cmd == "compare")) {
      o.min_n = parse_u64(a, take());
    } else if (a == "--max" && (o.cmd == "bench" || o.cmd == "compare")) {
      o.max_n = parse_u64(a, take());
    } else if (a == "--step-pct" && (o.cmd == "bench" || o.cmd == "compare")) {
      o.step_pct = (unsigned)parse_u64(a, take());
      if (o.step_pct < 1) throw ArgError("--step-pct must be positive");
    } else if (a == "--trials" && (o.cmd == "bench" || o.cmd == "compare")) {
      o.trials = (unsigned)parse_u64(a, take());
      if (o.trials < 1) throw ArgError("--trials must be positive");
    } else if (a == "--modulus") {
      o.modulus = parse_u64(a, take());
    } else if (a == "--two-adicity") {
      o.two_adicity = (unsigned)parse_u64(a, take());
    } else if (a == "--ring") {
      if (!take()) throw ArgError("--ring needs a value");
      o.ring = v;
    } else if (a == "--device") {
      if (!take()) throw ArgError("--device needs a value");
      o.device = v;
      if (o.device != "cuda") throw ArgError("--device: this build runs the transforms on cuda only");
    } else {
      throw ArgError("unknown option " + a + " for " + o.cmd);
    }
  }
  if (o.cmd == "count" && o.length == 0) throw ArgError("count needs --length");
  return o;
}

// the ring context (GPU) and its host mirror
struct Rings {
  std::unique_ptr<cf::Ring> dev;
  std::unique_ptr<HostRing> host;
  u64 stride = 0;  // element stride, bytes
};

Rings make_rings(const Options& o) {
  Rings r;
  if (o.ring == "prime") {
    r.dev.reset(new cf::PrimeRing(o.modulus, o.two_adicity));
    r.host.reset(new HostPrime(o.modulus, o.two_adicity));
    r.stride = 8;
  } else if (o.ring.rfind("fermat:", 0) == 0) {
    const u64 N = parse_u64("--ring fermat:N", o.ring.c_str() + 7);
    r.dev.reset(new cf::FermatRing(N));
    r.stride = r.dev->element_bytes();
    r.host.reset(new HostFermat(N, r.stride / 8));
  } else if (o.ring.rfind("negacyclic:", 0) == 0) {
    const std::string s = o.ring.substr(11);
    const auto comma = s.find(',');
    if (comma == std::string::npos) throw ArgError("--ring negacyclic:K,M");
    const u64 K = parse_u64("--ring negacyclic:K", s.substr(0, comma).c_str());
    const u64 m = parse_u64("--ring negacyclic:M", s.substr(comma + 1).c_str());
    r.dev.reset(new cf::NegacyclicRing(K, m));
    r.host.reset(new HostNega(K, m));
    r.stride = r.dev->element_bytes();
  } else {
    throw ArgError("--ring must be prime, fermat:N or negacyclic:K,M");
  }
  return r;
}

// naive weighted DFT (transform.hpp:292-311): out[j] = sum_i omega^(j' (s + i M/L)) a_i
std::vector<u64> dft_naive(const HostRing& R, u64 L, u64 s, const std::vector<u64>& a, u64 z) {
  const u64 W = R.words(), M = R.M();
  unsigned ell = 0;
  while ((u64{1} << ell) < L) ++ell;
  std::vector<u64> out(L * W, 0), t(W);
  for (u64 j = 0; j < L; ++j) {
    const u64 jr = bit_reverse(j, ell);
    for (u64 i = 0; i < z; ++i) {
      R.twiddle(t.data(), a.data() + i * W, (jr * ((s + i * (M / L)) % M)) % M);
      R.add(out.data() + j * W, t.data());
    }
  }
  return out;
}

struct Suite {
  std::string name;
  u64 cases = 0, failures = 0;
  std::string first;
};

std::string describe(u64 L, u64 z, u64 n, int f, int policy, u64 seed) {
  return "L=" + std::to_string(L) + " z=" + std::to_string(z) + " n=" + std::to_string(n) +
         " f=" + std::to_string(f) + " policy=" + (policy ? "radix2" : "balanced") + " seed=" + std::to_string(seed);
}

// One batch of sub-transforms over a device slab: items (with their slab
// inputs already in `host`), run, read back.
void run_batch(const Rings& R, int inverse, const std::vector<cftft_subtransform>& items, int policy,
               std::vector<u64>& host) {
  void* d = nullptr;
  const size_t bytes = host.size() * 8;
  cf::check(cudaMalloc(&d, bytes) == cudaSuccess ? CFTFT_OK : CFTFT_CUDA_ERROR);
  cudaMemcpy(d, host.data(), bytes, cudaMemcpyHostToDevice);
  const int rc = cftft_gpu_batch(R.dev->handle(), inverse, items.data(), items.size(), d, R.stride, policy, 1, nullptr);
  if (rc == CFTFT_OK) cudaMemcpy(host.data(), d, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d);
  cf::check(rc);
  cf::check(cftft_stream_synchronize(nullptr));
}

Suite tft_oracle_suite(const Rings& R, unsigned max_ell, u64 seed, unsigned samples = 8) {
  Suite res{"tft-oracle"};
  const HostRing& H = *R.host;
  const u64 W = H.words();
  for (unsigned ell = 1; ell <= max_ell; ++ell) {
    const u64 L = u64{1} << ell;
    for (int policy = 0; policy < 2; ++policy) {
      // one batch per (L, policy): items (z, k, n)
      std::vector<cftft_subtransform> items;
      std::vector<u64> slab;
      std::vector<std::vector<u64>> wants;
      std::vector<u64> seeds, zs;
      for (u64 z = 1; z <= L; ++z)
        for (unsigned k = 0; k < samples; ++k) {
          const u64 cs = mix_seed(mix_seed(mix_seed(seed, L), z), k);
          std::mt19937_64 g(cs);
          std::vector<u64> a(z * W);
          for (u64 i = 0; i < z; ++i) H.random(g, a.data() + i * W);
          const u64 s = g() % H.M();
          wants.push_back(dft_naive(H, L, s, a, z));
          seeds.push_back(cs);
          zs.push_back(z);
          for (u64 n = 1; n <= L; ++n) {
            cftft_subtransform t{};
            t.length = L;
            t.twiddle_exp = s;
            t.input_count = z;
            t.output_count = n;
            t.base = slab.size() / W;
            t.stride = 1;
            items.push_back(t);
            const size_t at = slab.size();
            slab.resize(at + L * W, ~u64{0});  // cells >= z: a non-canonical poison
            std::copy(a.begin(), a.end(), slab.begin() + at);
          }
        }
      run_batch(R, 0, items, policy, slab);
      for (size_t t = 0; t < items.size(); ++t) {
        const auto& it = items[t];
        const auto& want = wants[t / L];
        ++res.cases;
        const bool good = H.same(slab.data() + it.base * W, want.data(), it.output_count);
        if (!good && !res.failures++) res.first = describe(L, zs[t / L], it.output_count, 0, policy, seeds[t / L]);
      }
    }
  }
  return res;
}

Suite itft_inversion_suite(const Rings& R, unsigned max_ell, u64 seed, unsigned samples = 3) {
  Suite res{"itft-inversion"};
  const HostRing& H = *R.host;
  const u64 W = H.words();
  for (unsigned ell = 1; ell <= max_ell; ++ell) {
    const u64 L = u64{1} << ell;
    for (int policy = 0; policy < 2; ++policy) {
      std::vector<cftft_subtransform> items;
      std::vector<u64> slab;
      struct Want {
        std::vector<u64> spectrum, scaled;
        u64 z, seed;
      };
      std::vector<Want> wants;
      std::vector<size_t> which;
      for (u64 z = 1; z <= L; ++z)
        for (unsigned k = 0; k < samples; ++k) {
          const u64 cs = mix_seed(mix_seed(mix_seed(seed, L), z), k);
          std::mt19937_64 g(cs);
          std::vector<u64> a(z * W);
          for (u64 i = 0; i < z; ++i) H.random(g, a.data() + i * W);
          const u64 s = g() % H.M();
          Want w{dft_naive(H, L, s, a, z), a, z, cs};
          for (u64 i = 0; i < z; ++i) H.mul_small(w.scaled.data() + i * W, L);
          for (u64 n = 0; n <= z; ++n)
            for (int f = 0; f <= 1; ++f) {
              const u64 nf = n + (u64)f;
              if (nf < 1 || nf > L) continue;
              cftft_subtransform t{};
              t.length = L;
              t.twiddle_exp = s;
              t.input_count = z;
              t.output_count = n;
              t.want_next = f;
              t.base = slab.size() / W;
              t.stride = 1;
              items.push_back(t);
              which.push_back(wants.size());
              const size_t at = slab.size();
              slab.resize(at + L * W, ~u64{0});
              std::copy(w.spectrum.begin(), w.spectrum.begin() + n * W, slab.begin() + at);
              std::copy(w.scaled.begin() + n * W, w.scaled.end(), slab.begin() + at + n * W);
            }
          wants.push_back(std::move(w));
        }
      run_batch(R, 1, items, policy, slab);
      for (size_t t = 0; t < items.size(); ++t) {
        const auto& it = items[t];
        const Want& w = wants[which[t]];
        ++res.cases;
        const u64 n = it.output_count;
        bool good = H.same(slab.data() + it.base * W, w.scaled.data(), n);
        if (good && it.want_next) good = H.same(slab.data() + (it.base + n) * W, w.spectrum.data() + n * W, 1);
        if (!good && !res.failures++) res.first = describe(L, w.z, n, it.want_next, policy, w.seed);
      }
    }
  }
  return res;
}

u64 tft_bound_2x(u64 L, unsigned ell, u64 n) { return std::min((n - 1) * ell + 2 * (L - 1), L * (u64)ell); }
u64 itft_bound_2x(u64 L, unsigned ell, u64 n, int f) {
  return std::min((n + (u64)f - 1) * ell + 2 * (L - 1), L * (u64)ell);
}

Suite count_suite(const char* name, unsigned max_ell, int kind) {  // 0 tft bounds, 1 itft bounds, 2 smoothness
  Suite res{name};
  for (unsigned ell = 1; ell <= max_ell; ++ell) {
    const u64 L = u64{1} << ell;
    for (u64 z = 1; z <= L; ++z)
      for (u64 n = (kind == 1 ? 0 : 1); n <= (kind == 1 ? z : L); ++n)
        for (int f = 0; f <= (kind == 1 ? 1 : 0); ++f) {
          if (kind == 1 && (n + f < 1 || n + f > L)) continue;
          for (int policy = 0; policy < 2; ++policy) {
            ++res.cases;
            bool good;
            if (kind == 1) {
              const u64 c = cftft_itft_base_cases(L, z, n, f, policy);
              good = 2 * c <= itft_bound_2x(L, ell, n, f);
              if (good && n == L && z == L && f == 0) good = 2 * c == L * ell;
            } else {
              const u64 c = cftft_tft_base_cases(L, z, n, policy);
              if (kind == 0) {
                good = 2 * c <= tft_bound_2x(L, ell, n);
                if (good && n == L && z == L) good = 2 * c == L * ell;
              } else {
                good = 2 * c <= n * ell + 2 * L;
              }
            }
            if (!good && !res.failures++) res.first = describe(L, z, n, f, policy, 0);
          }
        }
  }
  return res;
}

int run_verify(const Options& o) {
  Rings R = make_rings(o);
  if ((u64{1} << o.max_ell) > R.host->M())
    throw ArgError("sweep depth 2^" + std::to_string(o.max_ell) + " exceeds the root order " +
                   std::to_string(R.host->M()));
  cf::fault::set_corrupt_tft_base(o.inject_fault);
  std::vector<Suite> suites;
  suites.push_back(tft_oracle_suite(R, o.max_ell, o.seed));
  suites.push_back(itft_inversion_suite(R, o.max_ell, o.seed));
  suites.push_back(count_suite("tft-bounds", o.max_ell, 0));
  suites.push_back(count_suite("itft-bounds", o.max_ell, 1));
  suites.push_back(count_suite("tft-smoothness", o.max_ell, 2));
  cf::fault::set_corrupt_tft_base(false);
  unsigned failed = 0;
  for (const Suite& s : suites) {
    if (!s.failures) {
      std::printf("%-16s PASS  %" PRIu64 " cases\n", s.name.c_str(), s.cases);
    } else {
      ++failed;
      std::printf("%-16s FAIL  %" PRIu64 " of %" PRIu64 " cases, first: %s\n", s.name.c_str(), s.failures, s.cases,
                  s.first.c_str());
    }
  }
  if (!failed) {
    std::printf("all %zu suites passed (max L = %" PRIu64 ", seed %" PRIu64 ")\n", suites.size(), u64{1} << o.max_ell,
                o.seed);
    return 0;
  }
  std::printf("%u of %zu suites failed\n", failed, suites.size());
  return 1;
}

int run_count(const Options& o) {
  Rings R = make_rings(o);
  const u64 L = o.length;
  if (L < 2 || (L & (L - 1)) || L > R.host->M() || L > (u64{1} << 16))
    throw cf::BadLength("transform length " + std::to_string(L) + " must be a power of two in [2, min(M, 2^16)]");
  unsigned ell = 0;
  while ((u64{1} << ell) < L) ++ell;
  std::printf("n,tft_count,tft_bound,itft_count,itft_bound\n");
  for (u64 n = 1; n <= L; ++n)
    std::printf("%" PRIu64 ",%" PRIu64 ",%" PRIu64 ",%" PRIu64 ",%" PRIu64 "\n", n,
                cftft_tft_base_cases(L, n, n, o.policy), tft_bound_2x(L, ell, n) / 2,
                cftft_itft_base_cases(L, n, n, 0, o.policy), itft_bound_2x(L, ell, n, 0) / 2);
  return 0;
}

std::vector<u64> sweep_grid(u64 min_n, u64 max_n, unsigned step_pct) {  // bench.hpp:18-30
  std::vector<u64> grid;
  const double ratio = 1.0 + step_pct / 100.0;
  for (double exact = (double)min_n;; exact *= ratio) {
    const u64 v = (u64)std::llround(exact);
    if (v >= max_n) break;
    if (grid.empty() || v > grid.back()) grid.push_back(v);
  }
  grid.push_back(max_n);
  return grid;
}

struct BenchRecord {
  u64 n, L, wall_ns, butterflies;
};

// bench_point (bench.hpp:54-98): seeded inputs with the product length n
// (zg = (n+2)/2, zh = n+1-zg, leading coefficients nonzero), one warm-up
// poly_mul, the median of `trials` timed ones (inputs already on the GPU).
BenchRecord bench_point(const Rings& R, u64 n, int policy, unsigned trials, u64 seed) {
  const HostRing& H = *R.host;
  const u64 W = H.words();
  std::mt19937_64 g(mix_seed(seed, n));
  const u64 zg = (n + 2) / 2, zh = n + 1 - zg;
  std::vector<u64> a(zg * W), b(zh * W);
  for (u64 i = 0; i < zg; ++i) H.random(g, a.data() + i * W);
  for (u64 i = 0; i < zh; ++i) H.random(g, b.data() + i * W);
  auto force_nonzero = [&](u64* x) {
    while (H.is_zero(x)) H.random(g, x);
  };
  force_nonzero(a.data() + (zg - 1) * W);
  force_nonzero(b.data() + (zh - 1) * W);
  void *dg = nullptr, *dh = nullptr, *dout = nullptr;
  cudaMalloc(&dg, zg * R.stride);
  cudaMalloc(&dh, zh * R.stride);
  cudaMalloc(&dout, n * R.stride);
  cudaMemcpy(dg, a.data(), zg * R.stride, cudaMemcpyHostToDevice);
  cudaMemcpy(dh, b.data(), zh * R.stride, cudaMemcpyHostToDevice);
  cf::MulStats st;
  cf::DeviceView vg(dg, R.stride, zg), vh(dh, R.stride, zh), vo(dout, R.stride, n);
  cf::poly_mul(*R.dev, vg, vh, vo, policy ? cf::SplitPolicy::radix2 : cf::SplitPolicy::balanced, &st);
  std::vector<u64> ns;
  for (unsigned t = 0; t < trials; ++t) {
    const auto t0 = std::chrono::steady_clock::now();
    cf::poly_mul(*R.dev, vg, vh, vo, policy ? cf::SplitPolicy::radix2 : cf::SplitPolicy::balanced, &st);
    ns.push_back((u64)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0)
                     .count());
  }
  cudaFree(dg);
  cudaFree(dh);
  cudaFree(dout);
  std::sort(ns.begin(), ns.end());
  const u64 med = ns.size() % 2 ? ns[ns.size() / 2] : (ns[ns.size() / 2 - 1] + ns[ns.size() / 2]) / 2;
  return BenchRecord{n, st.transform_length, med, st.butterflies.base_case_count};
}

void check_grid(const Rings& R, const Options& o) {
  if (o.min_n < 1 || o.min_n > o.max_n || o.max_n > R.host->M())
    throw cf::InvalidParams("sweep requires 1 <= min <= max <= root order");
}

int run_bench(const Options& o) {
  Rings R = make_rings(o);
  check_grid(R, o);
  std::printf("n,L,policy,wall_ns,butterflies\n");
  for (u64 n : sweep_grid(o.min_n, o.max_n, o.step_pct)) {
    const BenchRecord r = bench_point(R, n, o.policy, o.trials, o.seed);
    std::printf("%" PRIu64 ",%" PRIu64 ",%s,%" PRIu64 ",%" PRIu64 "\n", r.n, r.L, o.policy ? "radix2" : "balanced",
                r.wall_ns, r.butterflies);
    std::fflush(stdout);
  }
  return 0;
}

int run_compare(const Options& o) {
  Rings R = make_rings(o);
  check_grid(R, o);
  std::printf("n,wall_ns_balanced,wall_ns_radix2,ratio\n");
  for (u64 n : sweep_grid(o.min_n, o.max_n, o.step_pct)) {
    const BenchRecord a = bench_point(R, n, CFTFT_BALANCED, o.trials, o.seed);
    const BenchRecord b = bench_point(R, n, CFTFT_RADIX2, o.trials, o.seed);
    std::printf("%" PRIu64 ",%" PRIu64 ",%" PRIu64 ",%.4f\n", n, a.wall_ns, b.wall_ns,
                (double)b.wall_ns / (double)a.wall_ns);
    std::fflush(stdout);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Options o = parse(argc, argv);
    if (o.cmd == "verify") return run_verify(o);
    if (o.cmd == "count") return run_count(o);
    if (o.cmd == "bench") return run_bench(o);
    return run_compare(o);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
