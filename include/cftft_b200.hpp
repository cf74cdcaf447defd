// cftft_b200.hpp -- C++ host API over the C ABI (cftft_b200.h), mirroring the
// reference library's transform interface so that a caller of
//   cftft::cf_tft / cftft::cf_itft   (proj/include/cftft/transform.hpp:252-286)
// switches by changing the namespace, the ring context and the view type:
//
//   reference (cftft::)                         here (cftft_b200::)
//   ------------------------------------------  ------------------------------------------
//   TransformParams        (transform.hpp:39-45) TransformParams (same fields, same meaning)
//   SplitPolicy            (:27-30)             SplitPolicy
//   ButterflyStats         (:49-51)             ButterflyStats (filled by schedule replay)
//   BadLength, InvalidParams (:16-24)           BadLength, InvalidParams (same bases)
//   RingCtx                (field.hpp:84)       FermatRing(N), NegacyclicRing(K, m)
//   StridedView            (view.hpp:14-51)     DeviceView (device memory, same column/row)
//   cf_tft / cf_itft       (:252-286)           cf_tft / cf_itft (same checks, same order)
//
// Semantics follow the reference: in place over the view; x[0..z) in,
// x[0..n) (+ x[n] for an ITFT with f = 1) out; other cells unspecified;
// errors are thrown before any work.  The reference is synchronous; these
// calls enqueue on `stream` and, by default, synchronise it before returning.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "cftft_b200.h"

namespace cftft_b200 {

using u64 = std::uint64_t;

struct BadLength : std::invalid_argument {
  explicit BadLength(const std::string& what) : std::invalid_argument(what) {}
};
struct InvalidParams : std::invalid_argument {
  explicit InvalidParams(const std::string& what) : std::invalid_argument(what) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& what) : std::runtime_error(what) {}
};
struct Unsupported : std::runtime_error {
  explicit Unsupported(const std::string& what) : std::runtime_error(what) {}
};
// cftft::TooLarge (polymul.hpp:13-18): the product does not fit the root order
struct TooLarge : std::length_error {
  explicit TooLarge(const std::string& what) : std::length_error(what) {}
};
// debug poison (cftft_set_debug_poison): an output depended on a cell >= z
struct PoisonRead : std::logic_error {
  explicit PoisonRead(const std::string& what) : std::logic_error(what) {}
};

// cftft::fault::corrupt_tft_base (transform.hpp:53-56): the reference's hook
// is a global flag; here it is the library's (forward transforms add 1 to
// x[0] while set).
namespace fault {
inline void set_corrupt_tft_base(bool on) { cftft_set_fault_injection(on ? 1 : 0); }
inline bool corrupt_tft_base() { return cftft_fault_injection() != 0; }
}  // namespace fault

inline void check(int rc) {
  if (rc == CFTFT_OK) return;
  const std::string msg = cftft_last_error();
  switch (rc) {
    case CFTFT_BAD_LENGTH: throw BadLength(msg);
    case CFTFT_INVALID_PARAMS: throw InvalidParams(msg);
    case CFTFT_CUDA_ERROR: throw CudaError(msg);
    case CFTFT_POISON_READ: throw PoisonRead(msg);
    case CFTFT_TOO_LARGE: throw TooLarge(msg);
    default: throw Unsupported(msg);
  }
}

enum class SplitPolicy { balanced = CFTFT_BALANCED, radix2 = CFTFT_RADIX2 };

struct TransformParams {
  u64 length = 0;        // L = 2^ell, divides the root order
  u64 twiddle_exp = 0;   // s: zeta = omega^s
  u64 input_count = 0;   // z
  u64 output_count = 0;  // n
  int want_next = 0;     // f (inverse only)
};

struct ButterflyStats {
  u64 base_case_count = 0;
};

/// A ring context: immutable after construction, shareable between threads.
class Ring {
 public:
  Ring(const Ring&) = delete;
  Ring& operator=(const Ring&) = delete;
  Ring(Ring&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  ~Ring() {
    if (h_) cftft_ring_destroy(h_);
  }
  u64 root_order() const { return cftft_ring_root_order(h_); }
  u64 element_bytes() const { return cftft_ring_element_bytes(h_); }
  const cftft_ring* handle() const { return h_; }

 protected:
  Ring(int kind, u64 n_or_k, u64 m) { check(cftft_ring_create(kind, n_or_k, m, &h_)); }
  cftft_ring* h_ = nullptr;
};

/// Z/(2^N+1), omega = 2 (root order 2N).  Element: N/64 little-endian u64
/// limbs then a top word, canonical value in [0, 2^N].
class FermatRing : public Ring {
 public:
  explicit FermatRing(u64 N) : Ring(CFTFT_RING_FERMAT, N, 0) {}
};

/// (Z/mZ)[y]/(y^K+1), omega = y (root order 2K), m odd < 2^62.  Element: K
/// u64 words in [0, m).
class NegacyclicRing : public Ring {
 public:
  NegacyclicRing(u64 K, u64 m) : Ring(CFTFT_RING_NEGACYCLIC, K, m) {}
};

/// Non-owning strided window onto device memory: element i at
/// base + i * stride * elem_stride_bytes (view.hpp:14-51 over device bytes).
class DeviceView {
 public:
  DeviceView(void* base, u64 elem_stride_bytes, std::size_t len, std::size_t stride = 1)
      : base_(static_cast<std::uint8_t*>(base)), esb_(elem_stride_bytes), stride_(stride), len_(len) {}
  std::size_t size() const noexcept { return len_; }
  std::size_t stride() const noexcept { return stride_; }
  std::uint8_t* base() const noexcept { return base_; }
  u64 elem_stride_bytes() const noexcept { return esb_; }
  /// Column u of this view read as a rows x cols matrix.
  DeviceView column(std::size_t u, std::size_t rows, std::size_t cols) const {
    return DeviceView(base_ + u * stride_ * esb_, esb_, rows, stride_ * cols);
  }
  /// Row u of this view read as a matrix with the given row width.
  DeviceView row(std::size_t u, std::size_t cols) const {
    return DeviceView(base_ + u * cols * stride_ * esb_, esb_, cols, stride_);
  }

 private:
  std::uint8_t* base_;
  u64 esb_;
  std::size_t stride_, len_;
};

namespace detail {
inline cftft_params to_c(const TransformParams& p) {
  return cftft_params{p.length, p.twiddle_exp, p.input_count, p.output_count, p.want_next};
}
inline void run(int (*fn)(const cftft_ring*, const cftft_params*, void*, uint64_t, int, uint64_t*, void*),
                int inverse, const Ring& ring, const TransformParams& params, const DeviceView& x, SplitPolicy policy,
                ButterflyStats* stats, void* stream, bool synchronize) {
  cftft_params p = to_c(params);
  // the reference's order: length, then counts, then the view (transform.hpp:253-260)
  check(cftft_validate(ring.handle(), inverse, &p, static_cast<int>(policy)));
  if (x.size() != params.length) throw InvalidParams("view length does not match the transform length");
  uint64_t count = 0;
  check(fn(ring.handle(), &p, x.base(), x.elem_stride_bytes() * x.stride(), static_cast<int>(policy),
           stats ? &count : nullptr, stream));
  if (stats) stats->base_case_count += count;
  if (synchronize) check(cftft_stream_synchronize(stream));
}
}  // namespace detail

/// Forward truncated transform, in place over the view (transform.hpp:252-264).
inline void cf_tft(const Ring& ring, const TransformParams& params, DeviceView x,
                   SplitPolicy policy = SplitPolicy::balanced, ButterflyStats* stats = nullptr,
                   void* stream = nullptr, bool synchronize = true) {
  detail::run(cftft_gpu_tft, 0, ring, params, x, policy, stats, stream, synchronize);
}

/// Inverse truncated transform, in place over the view (transform.hpp:273-286).
inline void cf_itft(const Ring& ring, const TransformParams& params, DeviceView x,
                    SplitPolicy policy = SplitPolicy::balanced, ButterflyStats* stats = nullptr,
                    void* stream = nullptr, bool synchronize = true) {
  detail::run(cftft_gpu_itft, 1, ring, params, x, policy, stats, stream, synchronize);
}

/// The reference's calling convention on host memory: `buffer` holds L
/// elements of `elem_stride_bytes`; copies in, transforms, copies out.
inline void cf_tft_host(const Ring& ring, const TransformParams& params, void* buffer, u64 elem_stride_bytes,
                        SplitPolicy policy = SplitPolicy::balanced, ButterflyStats* stats = nullptr) {
  cftft_params p = detail::to_c(params);
  uint64_t count = 0;
  check(cftft_tft_host(ring.handle(), &p, buffer, elem_stride_bytes, static_cast<int>(policy),
                       stats ? &count : nullptr));
  if (stats) stats->base_case_count += count;
}
inline void cf_itft_host(const Ring& ring, const TransformParams& params, void* buffer, u64 elem_stride_bytes,
                         SplitPolicy policy = SplitPolicy::balanced, ButterflyStats* stats = nullptr) {
  cftft_params p = detail::to_c(params);
  uint64_t count = 0;
  check(cftft_itft_host(ring.handle(), &p, buffer, elem_stride_bytes, static_cast<int>(policy),
                        stats ? &count : nullptr));
  if (stats) stats->base_case_count += count;
}

/// The reference's own ring: Z/pZ, omega of order 2^m (field.hpp:84-185).
class PrimeRing : public Ring {
 public:
  explicit PrimeRing(u64 p = 0xFFFFFFFF00000001ull, unsigned m = 32) : Ring(CFTFT_RING_PRIME, m, p) {}
};

// ---------------------------------------------------------------------------
// poly_mul (polymul.hpp:26-95) over device memory

struct MulStats {
  u64 pointwise_mults = 0;   // exactly the product length, never the padded L
  u64 transform_length = 0;  // L, or 0 when a zero input short-circuits
  ButterflyStats butterflies;  // all three transforms combined
};

/// A polynomial on the device: coefficient i is element i of `view`
/// (contiguous: view.stride() == 1).
inline u64 poly_support(const Ring& ring, const DeviceView& a, void* stream = nullptr) {
  uint64_t k = 0;
  check(cftft_gpu_poly_support(ring.handle(), a.base(), a.size(), a.elem_stride_bytes() * a.stride(), &k, stream));
  return k;
}

/// Smallest power-of-two transform length >= max(n, 2) within the root order.
inline u64 choose_length(const Ring& ring, u64 n) {
  if (n < 1) throw InvalidParams("choose_length requires n >= 1");
  if (n > ring.root_order())
    throw TooLarge("product length " + std::to_string(n) + " exceeds the available root order " +
                   std::to_string(ring.root_order()));
  u64 L = 2;
  while (L < n) L <<= 1;
  return L;
}

/// g * h into `out` (>= zg + zh - 1 elements; supports by poly_support);
/// returns the product length n (0 for a zero input: nothing written).
inline u64 poly_mul(const Ring& ring, const DeviceView& g, const DeviceView& h, DeviceView out,
                    SplitPolicy policy = SplitPolicy::balanced, MulStats* stats = nullptr, void* stream = nullptr,
                    bool synchronize = true) {
  if (stats) *stats = MulStats{};
  if (g.stride() != 1 || h.stride() != 1 || out.stride() != 1 ||
      g.elem_stride_bytes() != out.elem_stride_bytes() || h.elem_stride_bytes() != out.elem_stride_bytes())
    throw InvalidParams("poly_mul takes contiguous views of one element stride");
  const u64 zg = poly_support(ring, g, stream), zh = poly_support(ring, h, stream);
  if (zg == 0 || zh == 0) return 0;
  const u64 n = zg + zh - 1;
  choose_length(ring, n);
  if (out.size() < n) throw InvalidParams("output view shorter than the product");
  cftft_mul_stats cs{};
  check(cftft_gpu_poly_mul(ring.handle(), g.base(), zg, h.base(), zh, out.base(), out.elem_stride_bytes(),
                           static_cast<int>(policy), &cs, stream));
  if (synchronize) check(cftft_stream_synchronize(stream));
  if (stats) {
    stats->pointwise_mults = cs.pointwise_mults;
    stats->transform_length = cs.transform_length;
    stats->butterflies.base_case_count = cs.base_case_count;
  }
  return n;
}

/// Bit reversal of the low ell bits (transform.hpp:73-80).
inline u64 bit_reverse(u64 j, unsigned ell) {
  u64 r = 0;
  for (unsigned i = 0; i < ell; ++i, j >>= 1) r = (r << 1) | (j & 1);
  return r;
}

}  // namespace cftft_b200
