/*
 * cftft_oracle.h -- CPU oracle for the truncated Fourier transform (TFT) and
 * its inverse (ITFT) of Harvey, "A cache-friendly truncated FFT"
 * (arxiv 0810.3203).
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker the GPU path is
 * compared against; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_0810_3203_b200) never links or calls it.
 *
 * It restates, in plain C, the reference's algorithm:
 *   tft_base2   /root/reference/proj/include/cftft/transform.hpp:94-110
 *   itft_base2  transform.hpp:120-150
 *   tft_rec     transform.hpp:154-186   (Algorithm 1)
 *   itft_rec    transform.hpp:188-239   (Algorithm 2)
 *   cf_tft      transform.hpp:252-264   (validation, exceptions -> codes)
 *   cf_itft     transform.hpp:273-286
 *   dft_naive   transform.hpp:292-311
 *   bounds      transform.hpp:316-333
 * generically over three rings, each exposing only the operations the
 * recursion uses (add, sub, multiply-by-omega^s, half, root order):
 *   PRIME       Z/p with a principal 2^m-th root omega found exactly as
 *               field.hpp:170-177 does (pins the schedule to the reference)
 *   FERMAT      Z/(2^N+1), omega = 2, M = 2N (Schoenhage-Strassen ring)
 *   NEGACYCLIC  (Z/mZ)[y]/(y^K+1), omega = y, M = 2K (Nussbaumer ring)
 *
 * Element storage (u64 words, little endian):
 *   PRIME       1 word, canonical in [0,p)
 *   FERMAT      N/64 limbs then one top word; canonical value in [0, 2^N]
 *               (top = 1 only for 2^N == -1, with all limbs zero)
 *   NEGACYCLIC  K words, each canonical in [0,m)
 * Views are strided exactly like cftft::StridedView (view.hpp:14-51): element
 * i of a view lives at base + i * stride_words.
 */
#ifndef CFTFT_ORACLE_H
#define CFTFT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_PRIME = 0, OR_FERMAT = 1, OR_NEGACYCLIC = 2 };
enum { OR_OK = 0, OR_BAD_LENGTH = 1, OR_INVALID_PARAMS = 2, OR_NOMEM = 3 };
enum { OR_BALANCED = 0, OR_RADIX2 = 1 };

typedef struct or_ring {
  int kind;
  uint64_t M;          /* root order: omega has order M */
  uint64_t words;      /* u64 words of one element value */
  /* PRIME */
  uint64_t p, omega, inv2;
  unsigned two_adicity;
  /* FERMAT */
  uint64_t N;          /* bits; multiple of 64 */
  /* NEGACYCLIC */
  uint64_t K, m;
} or_ring;

/* Ring construction.  Returns OR_OK or OR_INVALID_PARAMS. */
int or_ring_init_prime(or_ring* r, uint64_t p, unsigned two_adicity);
int or_ring_init_fermat(or_ring* r, uint64_t N);
int or_ring_init_negacyclic(or_ring* r, uint64_t K, uint64_t m);

/* Element operations (out may alias inputs).  Exposed for the ring-axiom
 * tests (restating field_test.cpp:117-144 for the new rings). */
void or_add(const or_ring* r, uint64_t* out, const uint64_t* a, const uint64_t* b);
void or_sub(const or_ring* r, uint64_t* out, const uint64_t* a, const uint64_t* b);
void or_twiddle(const or_ring* r, uint64_t s, uint64_t* out, const uint64_t* x);
void or_half(const or_ring* r, uint64_t* out, const uint64_t* x);
/* Full ring product (pointwise stage of poly_mul, polymul.hpp:73-77). */
void or_mul(const or_ring* r, uint64_t* out, const uint64_t* a, const uint64_t* b);

/* Base cases (transform.hpp:94-150).  count may be NULL. */
void or_tft_base2(const or_ring* r, uint64_t s, uint64_t z, uint64_t n, uint64_t* x0,
                  uint64_t* x1, uint64_t* count);
void or_itft_base2(const or_ring* r, uint64_t s, uint64_t z, uint64_t n, int f, uint64_t* x0,
                   uint64_t* x1, uint64_t* count);

/* cf_tft / cf_itft over the strided view [base, base + (L-1)*stride].
 * threads > 1 runs the independent top-level column/row sub-transforms on
 * that many POSIX threads ("the column loops are embarrassingly
 * parallel"); results are identical to threads == 1.  count may be NULL. */
int or_tft(const or_ring* r, uint64_t L, uint64_t s, uint64_t z, uint64_t n, uint64_t* base,
           uint64_t stride_words, int policy, uint64_t* count, int threads);
int or_itft(const or_ring* r, uint64_t L, uint64_t s, uint64_t z, uint64_t n, int f,
            uint64_t* base, uint64_t stride_words, int policy, uint64_t* count, int threads);

/* dft_naive (transform.hpp:292-311): out[j] = zeta^j' sum_i omega_L^(i j') a_i,
 * j' = bitrev(j).  out receives L elements at out_stride. */
int or_dft_naive(const or_ring* r, uint64_t L, uint64_t s, const uint64_t* coeffs, uint64_t z,
                 uint64_t coeff_stride, uint64_t* out, uint64_t out_stride);

uint64_t or_bit_reverse(uint64_t j, unsigned ell);
uint64_t or_tft_bound_2x(uint64_t L, uint64_t n);
uint64_t or_itft_bound_2x(uint64_t L, uint64_t n, int f);

/* Test hook mirroring fault::corrupt_tft_base (transform.hpp:53-56, 109). */
void or_set_fault(int on);

#ifdef __cplusplus
}
#endif
#endif
