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
  if (argc > 1 && std::string(argv[1]) == "--gpu") round_trip_gpu();
  std::printf("%s (%d failures)\n", failures ? "FAIL" : "OK", failures);
  return failures ? 1 : 0;
}
