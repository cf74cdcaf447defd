// api_test.cpp -- the C++ host API (include/cftft_b200.hpp) used the way the
// reference's own tests use cftft:: (transform_test.cpp:122-130, 228-246,
// 360-390): validation errors thrown before any work, and (--gpu) round trips
// ITFT(TFT(a)) = L a on device and host buffers.  Exit status 0 = pass.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/cftft_b200.hpp"

namespace cf = cftft_b200;

static int failures = 0;
#define EXPECT(cond)                                              \
  do {                                                            \
    if (!(cond)) {                                                \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                 \
    }                                                             \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void validation() {
  cf::FermatRing ring(128);  // M = 256
  EXPECT(ring.root_order() == 256);
  cf::DeviceView v8(nullptr, ring.element_bytes(), 8);
  // transform_test.cpp:360-390, in the reference's order
  EXPECT(throws<cf::BadLength>([&] { cf::cf_tft(ring, {12, 0, 1, 1, 0}, v8); }));
  EXPECT(throws<cf::BadLength>([&] { cf::cf_tft(ring, {512, 0, 1, 1, 0}, v8); }));
  EXPECT(throws<cf::InvalidParams>([&] { cf::cf_tft(ring, {8, 0, 0, 1, 0}, v8); }));
  EXPECT(throws<cf::InvalidParams>([&] { cf::cf_tft(ring, {8, 0, 9, 1, 0}, v8); }));
  EXPECT(throws<cf::InvalidParams>([&] { cf::cf_tft(ring, {8, 0, 1, 1, 1}, v8); }));
  EXPECT(throws<cf::InvalidParams>([&] { cf::cf_tft(ring, {4, 0, 1, 1, 0}, v8); }));  // view length
  EXPECT(throws<cf::InvalidParams>([&] { cf::cf_itft(ring, {8, 0, 2, 3, 0}, v8); }));  // z < n
  EXPECT(throws<cf::InvalidParams>([&] { cf::cf_itft(ring, {8, 0, 8, 8, 1}, v8); }));  // n + f > L
  EXPECT(throws<std::invalid_argument>([&] { cf::cf_tft(ring, {6, 0, 1, 1, 0}, v8); }));
  EXPECT(throws<cf::Unsupported>([] { cf::FermatRing bad(100); }));
  EXPECT(cf::bit_reverse(1, 3) == 4 && cf::bit_reverse(6, 3) == 3);
  // choose_length / TooLarge (polymul.hpp:33-37, 13-18)
  cf::PrimeRing small(97, 4);  // root order 16
  EXPECT(cf::choose_length(small, 1) == 2 && cf::choose_length(small, 9) == 16);
  EXPECT(throws<cf::TooLarge>([&] { cf::choose_length(small, 17); }));
  EXPECT(throws<std::length_error>([&] { cf::choose_length(small, 17); }));
  EXPECT(throws<cf::InvalidParams>([&] { cf::choose_length(small, 0); }));
  EXPECT(throws<cf::InvalidParams>([] { cf::PrimeRing composite(97 * 193, 2); }));
}

// poly_mul on the GPU against a schoolbook product (polymul_test.cpp:11-19,
// 81-162): the reference's own ring, then Z/(2^1024+1) with small
// coefficients (exact integer products); exactly n pointwise products,
// the zero polynomial, TooLarge.
static void poly_mul_gpu() {
  const std::uint64_t p = 0xFFFFFFFF00000001ull;
  cf::PrimeRing ring(p, 32);
  std::mt19937_64 rng(7);
  const std::uint64_t zg = 300, zh = 257, len = 320;
  std::vector<std::uint64_t> g(len, 0), h(len, 0);
  for (std::uint64_t i = 0; i < zg; ++i) g[i] = rng() % p;
  for (std::uint64_t i = 0; i < zh; ++i) h[i] = rng() % p;
  g[zg - 1] = 5;  // nonzero leading coefficients: supports zg, zh
  h[zh - 1] = 9;
  const std::uint64_t n = zg + zh - 1;
  std::vector<std::uint64_t> want(n, 0);
  for (std::uint64_t i = 0; i < zg; ++i)
    for (std::uint64_t j = 0; j < zh; ++j)
      want[i + j] = (std::uint64_t)(((unsigned __int128)g[i] * h[j] + want[i + j]) % p);
  std::uint64_t *dg = nullptr, *dh = nullptr, *dout = nullptr;
  EXPECT(cudaMalloc(&dg, len * 8) == cudaSuccess && cudaMalloc(&dh, len * 8) == cudaSuccess &&
         cudaMalloc(&dout, n * 8) == cudaSuccess);
  EXPECT(cudaMemcpy(dg, g.data(), len * 8, cudaMemcpyHostToDevice) == cudaSuccess);
  EXPECT(cudaMemcpy(dh, h.data(), len * 8, cudaMemcpyHostToDevice) == cudaSuccess);
  cf::MulStats st;
  const std::uint64_t got_n = cf::poly_mul(ring, cf::DeviceView(dg, 8, len), cf::DeviceView(dh, 8, len),
                                           cf::DeviceView(dout, 8, n), cf::SplitPolicy::balanced, &st);
  EXPECT(got_n == n);
  EXPECT(st.pointwise_mults == n && st.transform_length == 1024);
  EXPECT(st.butterflies.base_case_count == cftft_tft_base_cases(1024, zg, n, 0) +
                                               cftft_tft_base_cases(1024, zh, n, 0) +
                                               cftft_itft_base_cases(1024, n, n, 0, 0));
  std::vector<std::uint64_t> out(n);
  EXPECT(cudaMemcpy(out.data(), dout, n * 8, cudaMemcpyDeviceToHost) == cudaSuccess);
  EXPECT(out == want);
  // the zero polynomial: nothing written, stats zero
  EXPECT(cudaMemset(dh, 0, len * 8) == cudaSuccess);
  EXPECT(cf::poly_mul(ring, cf::DeviceView(dg, 8, len), cf::DeviceView(dh, 8, len), cf::DeviceView(dout, 8, n),
                      cf::SplitPolicy::radix2, &st) == 0);
  EXPECT(st.pointwise_mults == 0 && st.transform_length == 0);
  // TooLarge: root order 16
  cf::PrimeRing small(97, 4);
  EXPECT(cudaMemcpy(dh, h.data(), len * 8, cudaMemcpyHostToDevice) == cudaSuccess);
  EXPECT(throws<cf::TooLarge>([&] {
    cf::poly_mul(small, cf::DeviceView(dg, 8, 10), cf::DeviceView(dh, 8, 10), cf::DeviceView(dout, 8, 19));
  }));
  cudaFree(dg);
  cudaFree(dh);
  cudaFree(dout);

  // Z/(2^1024+1): coefficients < 2^62, products exact below 2^1024
  const std::uint64_t N = 1024;
  cf::FermatRing fr(N);
  const std::uint64_t eb = fr.element_bytes(), words = eb / 8, fz = 200;
  std::vector<std::uint64_t> fg(fz * words, 0), fh(fz * words, 0);
  std::vector<std::uint64_t> sg(fz), sh(fz);
  for (std::uint64_t i = 0; i < fz; ++i) {
    sg[i] = rng() >> 2;
    sh[i] = rng() >> 2;
    fg[i * words] = sg[i];
    fh[i * words] = sh[i];
  }
  const std::uint64_t fn = 2 * fz - 1;
  std::vector<unsigned __int128> acc(fn, 0);
  std::vector<std::uint64_t> hi(fn, 0);
  for (std::uint64_t i = 0; i < fz; ++i)
    for (std::uint64_t j = 0; j < fz; ++j) {
      const unsigned __int128 t = (unsigned __int128)sg[i] * sh[j];
      const unsigned __int128 old = acc[i + j];
      acc[i + j] += t;
      if (acc[i + j] < old) ++hi[i + j];
    }
  void *fdg = nullptr, *fdh = nullptr, *fdo = nullptr;
  EXPECT(cudaMalloc(&fdg, fz * eb) == cudaSuccess && cudaMalloc(&fdh, fz * eb) == cudaSuccess &&
         cudaMalloc(&fdo, fn * eb) == cudaSuccess);
  EXPECT(cudaMemcpy(fdg, fg.data(), fz * eb, cudaMemcpyHostToDevice) == cudaSuccess);
  EXPECT(cudaMemcpy(fdh, fh.data(), fz * eb, cudaMemcpyHostToDevice) == cudaSuccess);
  EXPECT(cf::poly_mul(fr, cf::DeviceView(fdg, eb, fz), cf::DeviceView(fdh, eb, fz), cf::DeviceView(fdo, eb, fn)) ==
         fn);
  std::vector<std::uint64_t> fo(fn * words);
  EXPECT(cudaMemcpy(fo.data(), fdo, fn * eb, cudaMemcpyDeviceToHost) == cudaSuccess);
  bool same = true;
  for (std::uint64_t i = 0; i < fn; ++i) {
    same &= fo[i * words] == (std::uint64_t)acc[i] && fo[i * words + 1] == (std::uint64_t)(acc[i] >> 64) &&
            fo[i * words + 2] == hi[i];
    for (std::uint64_t k = 3; k < words; ++k) same &= fo[i * words + k] == 0;
  }
  EXPECT(same);
  cudaFree(fdg);
  cudaFree(fdh);
  cudaFree(fdo);
}

static void round_trip_gpu() {
  // config 1 shape: Z/(2^1024+1), L = 2^10, z = n = 700, zeta = 1
  const std::uint64_t N = 1024, L = 1024, z = 700;
  cf::FermatRing ring(N);
  const std::uint64_t eb = ring.element_bytes(), words = eb / 8, lim = N / 64;
  std::vector<std::uint64_t> a(L * words, 0);
  std::mt19937_64 rng(42);
  for (std::uint64_t i = 0; i < z; ++i)
    for (std::uint64_t k = 0; k < lim; ++k) a[i * words + k] = rng();
  void* d = nullptr;
  EXPECT(cudaMalloc(&d, L * eb) == cudaSuccess);
  EXPECT(cudaMemcpy(d, a.data(), L * eb, cudaMemcpyHostToDevice) == cudaSuccess);
  cf::DeviceView x(d, eb, L);
  cf::ButterflyStats st;
  cf::cf_tft(ring, {L, 0, z, z, 0}, x, cf::SplitPolicy::balanced, &st);
  EXPECT(st.base_case_count == 3900);  // SURVEY.md §8 config table (reference instrumentation)
  cf::cf_itft(ring, {L, 0, z, z, 0}, x, cf::SplitPolicy::radix2, &st);
  EXPECT(st.base_case_count == 7800);
  // x = L a: scale by 1/L = omega^(2N - 10) and compare with a
  cf::check(cftft_gpu_scale(ring.handle(), d, z, eb, 2 * N - 10, nullptr));
  std::vector<std::uint64_t> back(L * words, 0);
  EXPECT(cudaMemcpy(back.data(), d, L * eb, cudaMemcpyDeviceToHost) == cudaSuccess);
  bool same = true;
  for (std::uint64_t i = 0; i < z; ++i)
    for (std::uint64_t k = 0; k <= lim; ++k) same &= back[i * words + k] == a[i * words + k];
  EXPECT(same);
  // column / row views of a 32 x 32 matrix: a length-32 sub-transform in place
  cf::DeviceView col = x.column(3, 32, 32);
  EXPECT(col.size() == 32 && col.stride() == 32);
  cf::cf_tft(ring, {32, 5, 20, 32, 0}, col);
  cf::cf_itft(ring, {32, 5, 32, 32, 0}, col);
  // host-buffer entry points (the reference's synchronous convention)
  std::vector<std::uint64_t> h = a;
  cf::cf_tft_host(ring, {L, 0, z, z, 0}, h.data(), eb);
  cf::cf_itft_host(ring, {L, 0, z, z, 0}, h.data(), eb);
  EXPECT(cudaMemcpy(d, h.data(), L * eb, cudaMemcpyHostToDevice) == cudaSuccess);
  cf::check(cftft_gpu_scale(ring.handle(), d, z, eb, 2 * N - 10, nullptr));
  EXPECT(cudaMemcpy(back.data(), d, L * eb, cudaMemcpyDeviceToHost) == cudaSuccess);
  same = true;
  for (std::uint64_t i = 0; i < z; ++i)
    for (std::uint64_t k = 0; k <= lim; ++k) same &= back[i * words + k] == a[i * words + k];
  EXPECT(same);
  cudaFree(d);
}

int main(int argc, char** argv) {
  validation();
  if (argc > 1 && std::string(argv[1]) == "--gpu") {
    round_trip_gpu();
    poly_mul_gpu();
  }
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}
