/*
 * cftft_b200.h -- C ABI of the B200-native truncated Fourier transform engine.
 *
 * Drop-in boundary for the reference's transform entry points
 * (/root/reference/proj/include/cftft/transform.hpp), re-targeted at the
 * large-coefficient rings of the BASELINE north star:
 *
 *   FERMAT      R = Z/(2^N+1), omega = 2, root order M = 2N   (Schoenhage-Strassen)
 *   NEGACYCLIC  R = (Z/mZ)[y]/(y^K+1), omega = y, M = 2K      (Nussbaumer)
 *
 * Plain pointers and sizes only; no torch or C++ types cross this boundary.
 *
 * Element format (little-endian u64 words):
 *   FERMAT      N/64 limbs followed by one top word; canonical value in
 *               [0, 2^N] (top == 1 only for 2^N == -1, all limbs zero).
 *   NEGACYCLIC  K words, each canonical in [0, m).
 * Element i of a view lives at base + i * elem_stride_bytes; the stride must
 * be a multiple of 16 and at least cftft_ring_element_bytes(ring).  This is
 * the byte-level form of cftft::StridedView (view.hpp:14-51): a reference
 * view (buffer, base, stride) maps to base_ptr = buffer + base*size and
 * elem_stride_bytes = stride*size.
 *
 * Errors map 1:1 onto the reference's exceptions:
 *   CFTFT_BAD_LENGTH      <- cftft::BadLength      (transform.hpp:16-20)
 *   CFTFT_INVALID_PARAMS  <- cftft::InvalidParams  (transform.hpp:22-24)
 * and are raised before any work is enqueued.  cftft_last_error() returns
 * the message of the last failure on the calling thread.
 */
#ifndef CFTFT_B200_H
#define CFTFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum cftft_status {
  CFTFT_OK = 0,
  CFTFT_BAD_LENGTH = 1,     /* L not a power of two in [2, M]               */
  CFTFT_INVALID_PARAMS = 2, /* z, n, f outside the reference's contract      */
  CFTFT_CUDA_ERROR = 3,     /* CUDA runtime failure (no GPU, launch error)  */
  CFTFT_UNSUPPORTED = 4,    /* ring/stride the engine does not implement    */
  CFTFT_NO_MEMORY = 5,
  CFTFT_POISON_READ = 6,    /* debug poison: a cell >= z was read (below)    */
  CFTFT_TOO_LARGE = 7       /* poly_mul: product longer than the root order  */
};

/* CFTFT_RING_PRIME: the reference's own ring, Z/pZ for an odd prime p < 2^64
 * with 2^m | p - 1 and omega the reference's root of order M = 2^m
 * (field.hpp:84-185; Goldilocks p = 2^64 - 2^32 + 1, m = 32 by default):
 * cftft_ring_create(CFTFT_RING_PRIME, m, p, &ring), m <= 32; one u64 word
 * per coefficient, element stride a multiple of 8 bytes. */
enum cftft_ring_kind { CFTFT_RING_FERMAT = 1, CFTFT_RING_NEGACYCLIC = 2, CFTFT_RING_PRIME = 3 };

/* cftft::SplitPolicy (transform.hpp:27-30). */
enum cftft_split_policy { CFTFT_BALANCED = 0, CFTFT_RADIX2 = 1 };

/* cftft::TransformParams (transform.hpp:39-45). */
typedef struct cftft_params {
  uint64_t length;       /* L = 2^ell, 2 <= L <= M                    */
  uint64_t twiddle_exp;  /* s: zeta = omega^s, reduced mod M on use   */
  uint64_t input_count;  /* z                                         */
  uint64_t output_count; /* n                                         */
  int32_t want_next;     /* f (inverse transform only)                */
} cftft_params;

typedef struct cftft_ring cftft_ring;

/* Ring contexts replace cftft::RingCtx (field.hpp:84-185).  For FERMAT,
 * n_or_k = N (a power of two in [128, 2^18]) and modulus is ignored.  For
 * NEGACYCLIC, n_or_k = K (a power of two in [2, 16384]) and modulus = m
 * (odd, < 2^62).  For PRIME, n_or_k = m (two-adicity, 1..32) and modulus =
 * p (a prime with 2^m | p - 1; a composite p is CFTFT_INVALID_PARAMS, the
 * reference's NotPrime).  Out-of-range sizes: CFTFT_UNSUPPORTED.  Immutable
 * and shareable across threads once created (concurrent host-view calls on
 * one ring are serialised). */
int cftft_ring_create(int kind, uint64_t n_or_k, uint64_t modulus, cftft_ring** out);
void cftft_ring_destroy(cftft_ring* ring);
uint64_t cftft_ring_root_order(const cftft_ring* ring);    /* M */
uint64_t cftft_ring_element_bytes(const cftft_ring* ring); /* minimal stride */

/* Tuning/testing knob: caps the on-chip leaf size at 2^max_ell coefficients
 * (default: the largest that fits the shared-memory budget).  Smaller caps
 * force deeper Bailey decompositions (more waves); results are unchanged.
 * Returns the cap in effect.  Must not race with transforms on the ring. */
unsigned cftft_ring_set_leaf_limit(cftft_ring* ring, unsigned max_ell);

/* Validation only (transform.hpp:241-286: length, then counts), no work. */
int cftft_validate(const cftft_ring* ring, int inverse, const cftft_params* params, int policy);

/* cudaStreamSynchronize for callers that do not include the CUDA runtime. */
int cftft_stream_synchronize(void* stream);

/* Fermat rings: leaf layout.  lane_words = 0 runs every leaf on whole
 * coefficients; 4, 8 or 16 enables coset leaves over lanes of that many
 * 32-bit words (a leaf whose rotations are whole lanes works
 * on one residue class of lanes of many coefficients, carries kept per
 * lane); -1 (the default) picks the lane width per transform length.
 * Results are bit-identical in every mode. */
int cftft_ring_set_coset(cftft_ring* ring, int lane_words);

/* Fermat rings with coset leaves: 1 (and -1, the default) cuts the
 * transform into coset leaves of up to 64 coefficients, whose full-network
 * waves run on the TMA-wave kernel (three passes over the data at L = 2^18
 * instead of six); 0 keeps leaves of <= 8 coefficients on the radix-8 warp
 * engine.  Bit-identical results; other values: CFTFT_INVALID_PARAMS. */
int cftft_ring_set_wide(cftft_ring* ring, int wide);

/* Forward truncated transform, in place over a DEVICE view
 * (replaces cftft::cf_tft, transform.hpp:252-264).  On entry x[0..z) hold
 * the coefficients (cells beyond are never read); on exit x[0..n) hold the
 * first n transformed values in bit-reversed order; x[n..L) are unspecified.
 * Asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 * base_case_count (nullable) receives the reference's ButterflyStats count
 * (transform.hpp:47-51), computed by schedule replay on the host. */
int cftft_gpu_tft(const cftft_ring* ring, const cftft_params* params, void* dev_base,
                  uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count,
                  void* stream);

/* Inverse truncated transform, in place over a DEVICE view
 * (replaces cftft::cf_itft, transform.hpp:273-286).  On entry x[0..n) hold
 * transformed values and x[n..z) hold L times the coefficients; on exit
 * x[0..n) hold L times the coefficients and, if f = 1, x[n] holds the next
 * transformed value. */
int cftft_gpu_itft(const cftft_ring* ring, const cftft_params* params, void* dev_base,
                   uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count,
                   void* stream);

/* Host-buffer forms: the same contract as cf_tft/cf_itft on a HOST view
 * (synchronous, like the reference).  The engine stages x[0..z) to the GPU,
 * transforms, and copies back x[0..n) (+ x[n] for f = 1).  Pinned host
 * memory gives full PCIe bandwidth but is not required. */
int cftft_tft_host(const cftft_ring* ring, const cftft_params* params, void* host_base,
                   uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count);
int cftft_itft_host(const cftft_ring* ring, const cftft_params* params, void* host_base,
                    uint64_t elem_stride_bytes, int policy, uint64_t* base_case_count);

/* One independent sub-transform of a batch (cftft_gpu_batch): a TFT or ITFT
 * of `length` elements of the device view, element i at view index
 * base + i*stride (the Bailey columns / rows of a distributed transform). */
typedef struct cftft_subtransform {
  uint64_t length, twiddle_exp, input_count, output_count;
  int32_t want_next;
  int32_t pad;
  uint64_t base, stride;
} cftft_subtransform;

/* Runs `count` independent sub-transforms (all forward, or all inverse) of
 * the view [dev_base, elem_stride_bytes] in ONE launch.  Outputs are left in
 * the engine's lazy element format (limbs + signed top word) unless
 * canonicalize != 0; cftft_gpu_canonicalize finishes them later.  Used by the
 * multi-GPU column and row passes. */
int cftft_gpu_batch(const cftft_ring* ring, int inverse, const cftft_subtransform* items, uint64_t count,
                    void* dev_base, uint64_t elem_stride_bytes, int policy, int canonicalize, void* stream);

/* Canonicalises x[0..count) (lazy engine format -> [0, 2^N]); Fermat only. */
int cftft_gpu_canonicalize(const cftft_ring* ring, void* dev_base, uint64_t count,
                           uint64_t elem_stride_bytes, void* stream);

/* Pointwise ring products a[i] <- a[i] * b[i], i < count, on device views
 * with the same element stride (the pointwise stage of cftft::poly_mul,
 * polymul.hpp:73-77).  Inputs and outputs canonical.  Fermat rings need
 * 512 <= N <= 2^17. */
int cftft_gpu_pointwise(const cftft_ring* ring, void* dev_a, const void* dev_b, uint64_t count,
                        uint64_t elem_stride_bytes, void* stream);

/* Negacyclic rings: x[i] <- c * x[i] word-wise mod m (e.g. poly_mul's final
 * L^-1 scale, polymul.hpp:82-87). */
/* The same with an extra factor on every product: Z/(2^N+1): 2^scale
 * (scale < 2N; poly_mul's L^-1 = 2^(2N - ell)); negacyclic and prime rings:
 * the scalar `scale` mod m / p.  cftft_gpu_pointwise is scale = 2^0 / 1. */
int cftft_gpu_pointwise_scaled(const cftft_ring* ring, void* dev_a, const void* dev_b, uint64_t count,
                               uint64_t elem_stride_bytes, uint64_t scale, void* stream);

/* cftft::MulStats (polymul.hpp:39-43): exactly n pointwise products, the
 * transform length L, and the base cases of all three transforms. */
typedef struct cftft_mul_stats {
  uint64_t pointwise_mults;
  uint64_t transform_length;
  uint64_t base_case_count;
} cftft_mul_stats;

/* cftft::poly_mul (polymul.hpp:48-95) on the GPU: g (zg elements) times h
 * (zh elements), both DEVICE arrays at elem_stride_bytes, into dev_out
 * (n = zg + zh - 1 canonical elements); the caller passes the supports
 * (cftft_gpu_poly_support computes poly_support, polymul.hpp:26-30).  TFT,
 * TFT, n pointwise products with the final L^-1 folded in, ITFT -- all on
 * the GPU, asynchronous on `stream` (workspace is stream-ordered).  zg or
 * zh = 0 gives the zero polynomial (nothing written, stats zero); n > M is
 * CFTFT_TOO_LARGE (cftft::TooLarge, polymul.hpp:13-18). */
int cftft_gpu_poly_mul(const cftft_ring* ring, const void* dev_g, uint64_t zg, const void* dev_h, uint64_t zh,
                       void* dev_out, uint64_t elem_stride_bytes, int policy, cftft_mul_stats* stats,
                       void* stream);
/* poly_support (polymul.hpp:26-30): 1 + the index of the last nonzero
 * element of a DEVICE array of len elements (0: zero polynomial).  Waits. */
int cftft_gpu_poly_support(const cftft_ring* ring, const void* dev_a, uint64_t len, uint64_t elem_stride_bytes,
                           uint64_t* support, void* stream);

/* Schoenhage-Strassen packing: count coefficients of
 * src_words little-endian u64 limbs each (contiguous) zero-extended into
 * ring elements at elem_stride_bytes. */
int cftft_gpu_pack_limbs(const cftft_ring* ring, void* dev_dst, uint64_t elem_stride_bytes, const void* dev_src,
                         uint64_t src_words, uint64_t count, void* stream);

/* Nussbaumer, negacyclic rings (Z/mZ)[y]/(y^K+1), y = x^s:
 * split: f (K s residues) -> s elements A_j with word k = f[j + s k];
 * join: h[j + s k] = (C_j + y C_{j+s})[k] mod m for j < s, from the 2s - 1
 * product elements C (C_{j+s} = 0 past them). */
int cftft_gpu_nussbaumer_split(const cftft_ring* ring, void* dev_dst, uint64_t elem_stride_bytes,
                               const uint64_t* dev_f, uint64_t s, void* stream);
int cftft_gpu_nussbaumer_join(const cftft_ring* ring, uint64_t* dev_h, const void* dev_c, uint64_t elem_stride_bytes,
                              uint64_t s, void* stream);

int cftft_gpu_mul_scalar(const cftft_ring* ring, void* dev_base, uint64_t count, uint64_t elem_stride_bytes,
                         uint64_t c, void* stream);

/* Scales x[0..count) by omega^e (e.g. 1/L = omega^(M - ell) in the Fermat
 * ring, or the SS final 2^-k scale); device view, asynchronous. */
int cftft_gpu_scale(const cftft_ring* ring, void* dev_base, uint64_t count,
                    uint64_t elem_stride_bytes, uint64_t e, void* stream);

/* Multi-GPU transforms: one transform partitioned over the
 * ranks of an NCCL communicator, one GPU per rank.  Rank p owns top-level
 * columns [c0, c1) of the Bailey split L = L1 x L2 (a "column slab": L1 x
 * (c1 - c0) elements, element (r, c) at r (c1 - c0) + c) and rows [r0, r1)
 * of the active rows (a "row slab": (r1 - r0) x L2, each row contiguous).
 * cftft_gpu_dist_tft: column slab (inputs x[r L2 + c] for the rank's
 * columns) -> column TFTs -> NCCL transpose -> row TFTs -> row slab (the
 * first n outputs, in the reference's bit-reversed order, row by row).
 * cftft_gpu_dist_itft: row slab (x[0, n) transformed values, x[n, z) L a)
 * -> phases i-iv with the transposes and the phase-iii row exchange ->
 * column slab (L a[0, n), plus x[n] if f = 1).  Asynchronous on `stream`;
 * every rank calls with the same parameters.  NCCL is loaded at run time
 * (libnccl.so.2).
 * The split L1 x L2 is the library's: the policy's (transform.hpp:150-152),
 * except that rings whose single-GPU plans run radix-64 leaves take columns
 * of L1 = 64 (outputs do not depend on the split); cftft_dist_geometry
 * reports it together with the slabs.  Each transpose piece (one row's
 * columns of one rank) is contiguous on both sides and moves by one
 * ncclSend / ncclRecv straight into place; the column pass (TFT) and the
 * full-row pass (ITFT) run in chunks, a chunk's transpose on the context's
 * own stream overlapping the next chunk's transforms. */
typedef struct cftft_dist cftft_dist;
int cftft_nccl_unique_id(void* out128);  /* ncclGetUniqueId: rank 0 makes it, all ranks get a copy */
int cftft_dist_create(const cftft_ring* ring, int rank, int world, const void* nccl_id128, cftft_dist** out);
int cftft_dist_create_from_comm(const cftft_ring* ring, void* nccl_comm, cftft_dist** out);
void cftft_dist_destroy(cftft_dist* d);
/* this rank's slabs: out[8] = {c0, c1, r0, r1, L1, L2, column-slab elements, row-slab elements} */
int cftft_dist_geometry(const cftft_dist* d, const cftft_params* params, int inverse, int policy, uint64_t* out);
/* Debug (pure host code, no GPU, no NCCL): the transpose schedule rank `rank`
 * of `world` hands to NCCL for one transform over a ring of root order M --
 * records of 6 words {chunk, 1 = send / 0 = recv, peer, 0 = column slab / 1 =
 * row slab, element offset, element count}, in issue order; the pieces of one
 * chunk form one NCCL group.  `wide` = the ring runs radix-64 leaves (columns
 * of 64).  Returns the number of words (writes at most cap). */
size_t cftft_dist_schedule(uint64_t M, const cftft_params* params, int inverse, int policy, int wide, int world,
                           int rank, uint64_t* out, size_t cap);
int cftft_gpu_dist_tft(const cftft_dist* d, const cftft_params* params, void* dev_colslab, void* dev_rowslab,
                       uint64_t elem_stride_bytes, int policy, void* stream);
int cftft_gpu_dist_itft(const cftft_dist* d, const cftft_params* params, void* dev_rowslab, void* dev_colslab,
                        uint64_t elem_stride_bytes, int policy, void* stream);

/* Base-case counts of the reference recursion (data independent;
 * verify.hpp:175-199), by host replay.  No GPU needed. */
uint64_t cftft_tft_base_cases(uint64_t L, uint64_t z, uint64_t n, int policy);
uint64_t cftft_itft_base_cases(uint64_t L, uint64_t z, uint64_t n, int f, int policy);

/* Launch statistics of the last transform issued on this thread: number of
 * kernels enqueued (for bench.py's gpu_launches). */
uint64_t cftft_last_launch_count(void);

/* cftft::fault::corrupt_tft_base (transform.hpp:53-56, 109): while set,
 * every forward transform ends with a one-thread kernel that adds the ring's
 * 1 to output x[0] (a corrupted butterfly), so verification sweeps must
 * fail.  Process-global, like the reference's hook (cftft_cli.cpp:41). */
void cftft_set_fault_injection(int on);
int cftft_fault_injection(void);

/* Launch timing for the bench (roofline of the dominant kernel): while set,
 * every kernel of a transform is bracketed by CUDA events on its launching
 * stream and logged with its ALGORITHMIC bytes (coefficients its leaves read
 * plus write, times the coefficient's information bytes: N/8, 8 K, 8).
 * cftft_launch_timing_read waits for the logged launches of the calling
 * thread, copies up to max records and returns how many there were. */
typedef struct cftft_launch_record {
  char kernel[40];
  uint64_t algorithmic_bytes;
  float ms;
} cftft_launch_record;
void cftft_set_launch_timing(int on);
uint64_t cftft_launch_timing_read(cftft_launch_record* out, uint64_t max);

/* Debug poison (transform.hpp:58-70, poison_tail): while set, cftft_gpu_tft
 * / cftft_gpu_itft run each transform twice, with two different
 * non-canonical fills of the cells [z, L) (inputs [0, z) restored in
 * between), and return CFTFT_POISON_READ if any specified output (x[0, n),
 * plus x[n] for an ITFT with f = 1) differs: a cell the contract leaves
 * unspecified was read before it was written.  Synchronous; debug only. */
void cftft_set_debug_poison(int on);

/* Debug: JSON description of the GPU schedule (leaves, waves, micro-ops) a
 * transform would run.  Pure host code (no GPU).  Returns the number of
 * bytes needed (including the terminating NUL); writes at most cap bytes. */
size_t cftft_plan_dump(const cftft_ring* ring, int inverse, const cftft_params* params,
                       int policy, char* buf, size_t cap);

const char* cftft_last_error(void);
const char* cftft_version(void);

#ifdef __cplusplus
}
#endif
#endif
