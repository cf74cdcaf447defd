// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference library
// (/root/reference/proj/include/cftft, header-only C++20).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/ (git
// ignored) when /root/reference is present; it includes the reference
// headers in place (-I/root/reference/proj/include), nothing is copied.
// Used to (1) pin the C oracle's recursion to the reference bit for bit over
// the reference's own prime-field ring, and (2) generate the golden fixtures
// in tests/golden/ (scripts/make_golden.py), and as the "reference" CPU arm.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

#include "cftft/cftft.hpp"

using namespace cftft;

namespace {
int code_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const BadLength&) {
    return 1;
  } catch (const InvalidParams&) {
    return 2;
  } catch (...) {
    return 3;
  }
}
SplitPolicy pol(int p) { return p ? SplitPolicy::radix2 : SplitPolicy::balanced; }
}  // namespace

extern "C" {

// Transforms over data[base + i*stride], i < L, with the reference's RingCtx(p, m).
int ref_tft(uint64_t p, unsigned m, uint64_t L, uint64_t s, uint64_t z, uint64_t n,
            uint64_t* data, uint64_t size, uint64_t base, uint64_t stride, int policy,
            uint64_t* count) {
  try {
    const RingCtx ctx(p, m);
    std::span<Fp> buf(reinterpret_cast<Fp*>(data), size);
    StridedView v(buf, base, stride, L);
    ButterflyStats st;
    cf_tft(ctx, {.length = L, .twiddle_exp = s, .input_count = z, .output_count = n}, v,
           pol(policy), &st);
    if (count) *count = st.base_case_count;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_itft(uint64_t p, unsigned m, uint64_t L, uint64_t s, uint64_t z, uint64_t n, int f,
             uint64_t* data, uint64_t size, uint64_t base, uint64_t stride, int policy,
             uint64_t* count) {
  try {
    const RingCtx ctx(p, m);
    std::span<Fp> buf(reinterpret_cast<Fp*>(data), size);
    StridedView v(buf, base, stride, L);
    ButterflyStats st;
    cf_itft(ctx,
            {.length = L, .twiddle_exp = s, .input_count = z, .output_count = n, .want_next = f},
            v, pol(policy), &st);
    if (count) *count = st.base_case_count;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_dft_naive(uint64_t p, unsigned m, uint64_t L, uint64_t s, const uint64_t* coeffs,
                  uint64_t z, uint64_t* out) {
  try {
    const RingCtx ctx(p, m);
    std::span<const Fp> c(reinterpret_cast<const Fp*>(coeffs), z);
    auto r = dft_naive(ctx, L, s, c);
    for (uint64_t j = 0; j < L; ++j) out[j] = r[j].v;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

uint64_t ref_omega(uint64_t p, unsigned m) { return RingCtx(p, m).omega().v; }

// Runs the five verify.hpp suites; fills cases[5], failures[5].
int ref_run_all_suites(uint64_t p, unsigned m, unsigned max_ell, uint64_t seed, uint64_t* cases,
                       uint64_t* failures) {
  try {
    const RingCtx ctx(p, m);
    auto res = run_all_suites(ctx, max_ell, seed);
    for (size_t i = 0; i < res.size() && i < 5; ++i) {
      cases[i] = res[i].cases;
      failures[i] = res[i].failures;
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

uint64_t ref_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }

// poly_mul (polymul.hpp:48-95): out must hold zg+zh-1 words; returns the length.
int64_t ref_poly_mul(uint64_t p, unsigned m, const uint64_t* g, uint64_t ng, const uint64_t* h,
                     uint64_t nh, uint64_t* out, int policy, uint64_t* stats3) {
  try {
    const RingCtx ctx(p, m);
    Polynomial G(ng), H(nh);
    for (uint64_t i = 0; i < ng; ++i) G[i] = Fp{g[i]};
    for (uint64_t i = 0; i < nh; ++i) H[i] = Fp{h[i]};
    MulStats st;
    auto r = poly_mul(ctx, G, H, pol(policy), &st);
    for (size_t i = 0; i < r.size(); ++i) out[i] = r[i].v;
    if (stats3) {
      stats3[0] = st.pointwise_mults;
      stats3[1] = st.transform_length;
      stats3[2] = st.butterflies.base_case_count;
    }
    return static_cast<int64_t>(r.size());
  } catch (...) {
    return -code_of(std::current_exception());
  }
}

}  // extern "C"
