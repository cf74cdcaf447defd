/*
 * cftft_oracle.c -- CPU oracle (TEST INFRASTRUCTURE ONLY; see the header).
 *
 * A plain-C restatement of the reference's TFT/ITFT recursion
 * (/root/reference/proj/include/cftft/transform.hpp) made generic over the
 * ring, plus the three ring instances the GPU path is checked against.
 */
#include "cftft_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static int g_fault = 0;
void or_set_fault(int on) { g_fault = on; }

/* ------------------------------------------------------------------------ */
/* Per-call scratch.  Ring ops need temporaries; one scratch per thread.    */
typedef struct scratch {
  uint64_t* t0;  /* >= 2*words + 4 */
  uint64_t* t1;
  uint64_t* t2;
} scratch;

static int scratch_init(scratch* sc, const or_ring* r) {
  size_t w = 2 * r->words + 8;
  sc->t0 = (uint64_t*)calloc(w, 8);
  sc->t1 = (uint64_t*)calloc(w, 8);
  sc->t2 = (uint64_t*)calloc(w, 8);
  return (sc->t0 && sc->t1 && sc->t2) ? OR_OK : OR_NOMEM;
}
static void scratch_free(scratch* sc) {
  free(sc->t0);
  free(sc->t1);
  free(sc->t2);
}

/* ------------------------------------------------------------------------ */
/* PRIME field Z/p (restates field.hpp:38-51, 108-150, 170-177).            */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((u128)a * b % p); }
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t acc = 1 % p;
  a %= p;
  while (e) {
    if (e & 1) acc = mulmod(acc, a, p);
    e >>= 1;
    if (e) a = mulmod(a, a, p);
  }
  return acc;
}
static int is_prime_u64(uint64_t n) { /* deterministic Miller-Rabin, field.hpp:56-78 */
  static const uint64_t bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i)
    if (n % bases[i] == 0) return n == bases[i];
  int rr = __builtin_ctzll(n - 1);
  uint64_t d = (n - 1) >> rr;
  for (int i = 0; i < 12; ++i) {
    uint64_t x = powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int witness = 1;
    for (int k = 1; k < rr; ++k) {
      x = mulmod(x, x, n);
      if (x == n - 1) {
        witness = 0;
        break;
      }
    }
    if (witness) return 0;
  }
  return 1;
}

int or_ring_init_prime(or_ring* r, uint64_t p, unsigned m) {
  memset(r, 0, sizeof *r);
  if (m < 1 || !is_prime_u64(p) || m > 63 || ((p - 1) & ((1ull << m) - 1)) != 0)
    return OR_INVALID_PARAMS;
  r->kind = OR_PRIME;
  r->p = p;
  r->two_adicity = m;
  r->M = 1ull << m;
  r->words = 1;
  r->inv2 = (p + 1) / 2;
  /* smallest g in 2,3,5,7,... whose (p-1)/2^m power has order 2^m (field.hpp:170-177) */
  uint64_t e = (p - 1) >> m;
  for (uint64_t g = 2; g < 1024; g = (g == 2) ? 3 : g + 2) {
    uint64_t w = powmod(g % p, e, p);
    if (powmod(w, r->M / 2, p) == p - 1) {
      r->omega = w;
      return OR_OK;
    }
  }
  return OR_INVALID_PARAMS;
}

/* ------------------------------------------------------------------------ */
/* FERMAT ring Z/(2^N+1): W = N/64 limbs + top word.                        */
int or_ring_init_fermat(or_ring* r, uint64_t N) {
  memset(r, 0, sizeof *r);
  if (N < 64 || (N % 64) != 0 || (N & (N - 1)) != 0) return OR_INVALID_PARAMS;
  r->kind = OR_FERMAT;
  r->N = N;
  r->M = 2 * N; /* omega = 2 has order 2N */
  r->words = N / 64 + 1;
  return OR_OK;
}

/* Reduce value = x[0..W) + hi * 2^N (hi signed, small) to canonical form. */
static void f_norm(uint64_t* x, uint64_t W, int64_t hi) {
  /* 2^N == -1, so value == x - hi */
  if (hi > 0) {
    uint64_t b = (uint64_t)hi;
    for (uint64_t i = 0; i < W && b; ++i) {
      uint64_t v = x[i];
      x[i] = v - b;
      b = (v < b);
    }
    if (b) { /* went negative: x now holds value + 2^N; add 2^N + 1 -> +1 */
      uint64_t c = 1;
      for (uint64_t i = 0; i < W && c; ++i) {
        x[i] += 1;
        c = (x[i] == 0);
      }
      x[W] = c; /* c == 1 iff the result is exactly 2^N */
      return;
    }
    x[W] = 0;
  } else if (hi < 0) {
    uint64_t c = (uint64_t)(-hi);
    for (uint64_t i = 0; i < W && c; ++i) {
      uint64_t v = x[i] + c;
      c = (v < c);
      x[i] = v;
    }
    x[W] = 0;
    if (c) { /* x + 2^N == x - 1 */
      uint64_t b = 1;
      for (uint64_t i = 0; i < W && b; ++i) {
        uint64_t v = x[i];
        x[i] = v - 1;
        b = (v == 0);
      }
      if (b) { /* x was 0: -1 == 2^N */
        memset(x, 0, W * 8);
        x[W] = 1;
      }
    }
  } else {
    x[W] = 0;
  }
}

static void f_add(const or_ring* r, uint64_t* out, const uint64_t* a, const uint64_t* b) {
  uint64_t W = r->N / 64, c = 0;
  int64_t hi = (int64_t)a[W] + (int64_t)b[W];
  for (uint64_t i = 0; i < W; ++i) {
    u128 s = (u128)a[i] + b[i] + c;
    out[i] = (uint64_t)s;
    c = (uint64_t)(s >> 64);
  }
  f_norm(out, W, hi + (int64_t)c);
}

static void f_sub(const or_ring* r, uint64_t* out, const uint64_t* a, const uint64_t* b) {
  uint64_t W = r->N / 64, bw = 0;
  int64_t hi = (int64_t)a[W] - (int64_t)b[W];
  for (uint64_t i = 0; i < W; ++i) {
    uint64_t ai = a[i], bi = b[i];
    uint64_t d = ai - bi - bw;
    bw = (ai < bi) || (ai == bi && bw);
    out[i] = d;
  }
  f_norm(out, W, hi - (int64_t)bw);
}

/* 2^s * x mod 2^N+1.  Shift into a 2W+2 limb temporary, then fold the bits
 * at and above 2^N back with a subtraction (2^N == -1). */
static void f_twiddle(const or_ring* r, scratch* sc, uint64_t s, uint64_t* out, const uint64_t* x) {
  uint64_t N = r->N, W = N / 64;
  s &= (2 * N - 1);
  int neg = s >= N;
  uint64_t t = s % N;
  uint64_t* tmp = sc->t0;
  memset(tmp, 0, (2 * W + 2) * 8);
  uint64_t q = t / 64, b = t % 64;
  for (uint64_t i = 0; i <= W; ++i) { /* x has W+1 words including top */
    uint64_t v = x[i];
    tmp[i + q] |= v << b;
    if (b) tmp[i + q + 1] |= v >> (64 - b);
  }
  /* value = lo - hi where lo = tmp[0..W), hi = tmp[W..2W+2) (< 2^(t+1) <= 2^N) */
  uint64_t bw = 0;
  for (uint64_t i = 0; i < W; ++i) {
    uint64_t hi_i = (W + i < 2 * W + 2) ? tmp[W + i] : 0;
    uint64_t ai = tmp[i];
    uint64_t d = ai - hi_i - bw;
    bw = (ai < hi_i) || (ai == hi_i && bw);
    tmp[i] = d;
  }
  /* the limbs of hi beyond W words (index >= 2W) are zero since hi < 2^(N+1)
   * only when t = N-1 and top = 1: hi = 2^N exactly -> tmp[2W] = 1 */
  int64_t extra = (int64_t)tmp[2 * W]; /* bit N of hi: contributes -2^N == +1 */
  memcpy(out, tmp, W * 8);
  /* value = out - bw*2^N + extra  ==  out + bw + extra  (2^N == -1) */
  f_norm(out, W, -(int64_t)bw - extra);
  if (neg) {
    /* -v = 0 - v */
    uint64_t* z = sc->t2;
    memset(z, 0, (W + 1) * 8);
    f_sub(r, out, z, out);
  }
}

/* Schoolbook product mod 2^N+1 (pointwise stage; test sizes only). */
static void f_mul(const or_ring* r, uint64_t* out, const uint64_t* a, const uint64_t* b) {
  uint64_t W = r->N / 64;
  if (a[W] || b[W]) { /* one operand is 2^N == -1 */
    uint64_t* z = (uint64_t*)calloc(W + 1, 8);
    const uint64_t* other = a[W] ? b : a;
    if (a[W] && b[W]) { /* (-1)(-1) = 1 */
      memset(out, 0, (W + 1) * 8);
      out[0] = 1;
    } else {
      f_sub(r, out, z, other);
    }
    free(z);
    return;
  }
  uint64_t* prod = (uint64_t*)calloc(2 * W + 1, 8);
  for (uint64_t i = 0; i < W; ++i) {
    uint64_t c = 0;
    for (uint64_t j = 0; j < W; ++j) {
      u128 t = (u128)a[i] * b[j] + prod[i + j] + c;
      prod[i + j] = (uint64_t)t;
      c = (uint64_t)(t >> 64);
    }
    prod[i + W] = c;
  }
  /* lo - hi */
  uint64_t bw = 0;
  for (uint64_t i = 0; i < W; ++i) {
    uint64_t ai = prod[i], hi_i = prod[W + i];
    uint64_t d = ai - hi_i - bw;
    bw = (ai < hi_i) || (ai == hi_i && bw);
    out[i] = d;
  }
  f_norm(out, W, -(int64_t)bw);
  free(prod);
}

/* ------------------------------------------------------------------------ */
/* NEGACYCLIC ring (Z/mZ)[y]/(y^K+1), omega = y.                             */
int or_ring_init_negacyclic(or_ring* r, uint64_t K, uint64_t m) {
  memset(r, 0, sizeof *r);
  if (K < 1 || (K & (K - 1)) != 0 || m < 3 || (m & 1) == 0 || m >= (1ull << 63))
    return OR_INVALID_PARAMS;
  r->kind = OR_NEGACYCLIC;
  r->K = K;
  r->m = m;
  r->M = 2 * K; /* y has order 2K */
  r->words = K;
  return OR_OK;
}

static inline uint64_t n_addw(uint64_t a, uint64_t b, uint64_t m) {
  u128 s = (u128)a + b;
  return (uint64_t)(s >= m ? s - m : s);
}
static inline uint64_t n_subw(uint64_t a, uint64_t b, uint64_t m) { return a >= b ? a - b : a + (m - b); }

static void n_twiddle(const or_ring* r, scratch* sc, uint64_t s, uint64_t* out, const uint64_t* x) {
  uint64_t K = r->K, m = r->m;
  s &= (2 * K - 1);
  uint64_t* tmp = sc->t0;
  for (uint64_t i = 0; i < K; ++i) {
    uint64_t e = i + s; /* < 3K */
    uint64_t v = x[i];
    int neg = 0;
    while (e >= K) {
      e -= K;
      neg ^= 1;
    }
    tmp[e] = neg ? n_subw(0, v, m) : v;
  }
  memcpy(out, tmp, K * 8);
}

static void n_mul(const or_ring* r, uint64_t* out, const uint64_t* a, const uint64_t* b) {
  uint64_t K = r->K, m = r->m;
  uint64_t* acc = (uint64_t*)calloc(K, 8);
  for (uint64_t i = 0; i < K; ++i) {
    if (!a[i]) continue;
    for (uint64_t j = 0; j < K; ++j) {
      uint64_t p = mulmod(a[i], b[j], m);
      uint64_t e = i + j;
      if (e < K)
        acc[e] = n_addw(acc[e], p, m);
      else
        acc[e - K] = n_subw(acc[e - K], p, m);
    }
  }
  memcpy(out, acc, K * 8);
  free(acc);
}

/* ------------------------------------------------------------------------ */
/* Generic ring dispatch (scratch-carrying internal versions).              */
static void r_add(const or_ring* r, scratch* sc, uint64_t* o, const uint64_t* a, const uint64_t* b) {
  (void)sc;
  switch (r->kind) {
    case OR_PRIME: {
      uint64_t gap = r->p - b[0]; /* field.hpp:108-112 */
      o[0] = a[0] >= gap ? a[0] - gap : a[0] + b[0];
      break;
    }
    case OR_FERMAT: f_add(r, o, a, b); break;
    default:
      for (uint64_t i = 0; i < r->K; ++i) o[i] = n_addw(a[i], b[i], r->m);
  }
}
static void r_sub(const or_ring* r, scratch* sc, uint64_t* o, const uint64_t* a, const uint64_t* b) {
  (void)sc;
  switch (r->kind) {
    case OR_PRIME: o[0] = a[0] >= b[0] ? a[0] - b[0] : a[0] + (r->p - b[0]); break;
    case OR_FERMAT: f_sub(r, o, a, b); break;
    default:
      for (uint64_t i = 0; i < r->K; ++i) o[i] = n_subw(a[i], b[i], r->m);
  }
}
/* omega^s * x; s reduced mod M on use (field.hpp:148-150). */
static void r_twiddle(const or_ring* r, scratch* sc, uint64_t s, uint64_t* o, const uint64_t* x) {
  switch (r->kind) {
    case OR_PRIME: o[0] = mulmod(powmod(r->omega, s & (r->M - 1), r->p), x[0], r->p); break;
    case OR_FERMAT: f_twiddle(r, sc, s, o, x); break;
    default: n_twiddle(r, sc, s, o, x);
  }
}
static void r_half(const or_ring* r, scratch* sc, uint64_t* o, const uint64_t* x) {
  switch (r->kind) {
    case OR_PRIME: o[0] = mulmod(x[0], r->inv2, r->p); break;
    case OR_FERMAT: f_twiddle(r, sc, 2 * r->N - 1, o, x); break; /* 2^-1 = 2^(2N-1) */
    default:
      for (uint64_t i = 0; i < r->K; ++i) {
        uint64_t c = x[i];
        o[i] = (c & 1) ? (uint64_t)(((u128)c + r->m) >> 1) : c >> 1;
      }
  }
}
static void r_zero(const or_ring* r, uint64_t* o) { memset(o, 0, r->words * 8); }

static void r_mul(const or_ring* r, uint64_t* o, const uint64_t* a, const uint64_t* b) {
  switch (r->kind) {
    case OR_PRIME: o[0] = mulmod(a[0], b[0], r->p); break;
    case OR_FERMAT: f_mul(r, o, a, b); break;
    default: n_mul(r, o, a, b);
  }
}

/* Public element ops (allocate their own scratch). */
#define WITH_SCRATCH(stmt)            \
  do {                                \
    scratch sc;                       \
    if (scratch_init(&sc, r)) return; \
    stmt;                             \
    scratch_free(&sc);                \
  } while (0)
void or_add(const or_ring* r, uint64_t* o, const uint64_t* a, const uint64_t* b) { WITH_SCRATCH(r_add(r, &sc, o, a, b)); }
void or_sub(const or_ring* r, uint64_t* o, const uint64_t* a, const uint64_t* b) { WITH_SCRATCH(r_sub(r, &sc, o, a, b)); }
void or_twiddle(const or_ring* r, uint64_t s, uint64_t* o, const uint64_t* x) { WITH_SCRATCH(r_twiddle(r, &sc, s, o, x)); }
void or_half(const or_ring* r, uint64_t* o, const uint64_t* x) { WITH_SCRATCH(r_half(r, &sc, o, x)); }
void or_mul(const or_ring* r, uint64_t* o, const uint64_t* a, const uint64_t* b) { r_mul(r, o, a, b); }

/* ------------------------------------------------------------------------ */
/* Base cases: transform.hpp:94-110 and :120-150.                           */
static void fault_bump(const or_ring* r, scratch* sc, uint64_t* x0) {
  /* fault::corrupt_tft_base adds the ring's 1 to x0 (transform.hpp:109) */
  uint64_t* one = sc->t2;
  r_zero(r, one);
  one[0] = 1;
  r_add(r, sc, x0, x0, one);
}

static void tft_base2(const or_ring* r, scratch* sc, uint64_t s, uint64_t z, uint64_t n,
                      uint64_t* x0, uint64_t* x1, uint64_t* count) {
  if (count) ++*count;
  if (n == 2) {
    if (z == 2) {
      uint64_t* diff = sc->t1;
      r_sub(r, sc, diff, x0, x1);
      r_add(r, sc, x0, x0, x1);
      r_twiddle(r, sc, s, x1, diff);
    } else {
      r_twiddle(r, sc, s, x1, x0);
    }
  } else if (z == 2) {
    r_add(r, sc, x0, x0, x1);
  }
  if (g_fault) fault_bump(r, sc, x0);
}

static void itft_base2(const or_ring* r, scratch* sc, uint64_t s, uint64_t z, uint64_t n, int f,
                       uint64_t* x0, uint64_t* x1, uint64_t* count) {
  if (count) ++*count;
  uint64_t* t = sc->t1;
  if (n == 2) {
    r_twiddle(r, sc, 0 - s, t, x1); /* zeta^-1 = omega^(0-s), transform.hpp:126 */
    r_sub(r, sc, x1, x0, t);
    r_add(r, sc, x0, x0, t);
  } else if (n == 1) {
    if (f == 1) {
      if (z == 2) {
        r_sub(r, sc, t, x0, x1);
        r_add(r, sc, x0, x0, t);
        r_twiddle(r, sc, s, x1, t);
      } else {
        r_twiddle(r, sc, s, x1, x0);
        r_add(r, sc, x0, x0, x0);
      }
    } else {
      if (z == 2) {
        r_add(r, sc, t, x0, x0);
        r_sub(r, sc, x0, t, x1);
      } else {
        r_add(r, sc, x0, x0, x0);
      }
    }
  } else {
    if (z == 2) {
      r_add(r, sc, t, x0, x1);
      r_half(r, sc, x0, t);
    } else {
      r_half(r, sc, x0, x0);
    }
  }
}

void or_tft_base2(const or_ring* r, uint64_t s, uint64_t z, uint64_t n, uint64_t* x0, uint64_t* x1,
                  uint64_t* count) {
  WITH_SCRATCH(tft_base2(r, &sc, s, z, n, x0, x1, count));
}
void or_itft_base2(const or_ring* r, uint64_t s, uint64_t z, uint64_t n, int f, uint64_t* x0,
                   uint64_t* x1, uint64_t* count) {
  WITH_SCRATCH(itft_base2(r, &sc, s, z, n, f, x0, x1, count));
}

/* ------------------------------------------------------------------------ */
/* Strided view (view.hpp:14-51): element i at base + i*stride.             */
typedef struct view {
  uint64_t* base;
  uint64_t stride; /* in u64 words */
  uint64_t len;
} view;
static inline uint64_t* at(view v, uint64_t i) { return v.base + i * v.stride; }
static inline view v_column(view v, uint64_t u, uint64_t rows, uint64_t cols) {
  view c = {v.base + u * v.stride, v.stride * cols, rows};
  return c;
}
static inline view v_row(view v, uint64_t u, uint64_t cols) {
  view c = {v.base + u * cols * v.stride, v.stride, cols};
  return c;
}

static void split(unsigned ell, int policy, unsigned* l1, unsigned* l2) { /* transform.hpp:83-87 */
  if (policy == OR_RADIX2) {
    *l1 = 1;
    *l2 = ell - 1;
  } else {
    *l1 = ell / 2;
    *l2 = ell - ell / 2;
  }
}

/* Algorithm 1 (transform.hpp:154-186). */
static void tft_rec(const or_ring* r, scratch* sc, uint64_t L, uint64_t s, uint64_t z, uint64_t n,
                    view x, int policy, uint64_t* count) {
  if (L == 2) {
    tft_base2(r, sc, s, z, n, at(x, 0), at(x, 1), count);
    return;
  }
  unsigned ell = (unsigned)__builtin_ctzll(L), l1, l2;
  split(ell, policy, &l1, &l2);
  uint64_t cols = 1ull << l2, rows = 1ull << l1;
  uint64_t n2 = n & (cols - 1), n1 = n >> l2, n1c = n1 + (n2 ? 1 : 0);
  uint64_t z2 = z & (cols - 1), z1 = z >> l2, z2e = z1 ? cols : z2;
  uint64_t col_step = r->M >> ell;
  for (uint64_t u = 0; u < z2; ++u)
    tft_rec(r, sc, rows, s + u * col_step, z1 + 1, n1c, v_column(x, u, rows, cols), policy, count);
  for (uint64_t u = z2; u < z2e; ++u)
    tft_rec(r, sc, rows, s + u * col_step, z1, n1c, v_column(x, u, rows, cols), policy, count);
  uint64_t s_row = s << l1;
  for (uint64_t u = 0; u < n1; ++u) tft_rec(r, sc, cols, s_row, z2e, cols, v_row(x, u, cols), policy, count);
  if (n2 > 0) tft_rec(r, sc, cols, s_row, z2e, n2, v_row(x, n1, cols), policy, count);
}

/* Algorithm 2 (transform.hpp:188-239). */
static void itft_rec(const or_ring* r, scratch* sc, uint64_t L, uint64_t s, uint64_t z, uint64_t n,
                     int f, view x, int policy, uint64_t* count) {
  if (L == 2) {
    itft_base2(r, sc, s, z, n, f, at(x, 0), at(x, 1), count);
    return;
  }
  unsigned ell = (unsigned)__builtin_ctzll(L), l1, l2;
  split(ell, policy, &l1, &l2);
  uint64_t cols = 1ull << l2, rows = 1ull << l1;
  uint64_t n2 = n & (cols - 1), n1 = n >> l2, z2 = z & (cols - 1), z1 = z >> l2;
  int fm = (n2 + (uint64_t)f > 0) ? 1 : 0;
  uint64_t z2e = z1 ? cols : z2;
  uint64_t lo = n2 < z2 ? n2 : z2, hi = n2 > z2 ? n2 : z2;
  uint64_t col_step = r->M >> ell, s_row = s << l1;
  for (uint64_t u = 0; u < n1; ++u) itft_rec(r, sc, cols, s_row, cols, cols, 0, v_row(x, u, cols), policy, count);
  for (uint64_t u = n2; u < hi; ++u)
    itft_rec(r, sc, rows, s + u * col_step, z1 + 1, n1, fm, v_column(x, u, rows, cols), policy, count);
  for (uint64_t u = hi; u < z2e; ++u)
    itft_rec(r, sc, rows, s + u * col_step, z1, n1, fm, v_column(x, u, rows, cols), policy, count);
  if (fm) itft_rec(r, sc, cols, s_row, z2e, n2, f, v_row(x, n1, cols), policy, count);
  for (uint64_t u = 0; u < lo; ++u)
    itft_rec(r, sc, rows, s + u * col_step, z1 + 1, n1 + 1, 0, v_column(x, u, rows, cols), policy, count);
  for (uint64_t u = lo; u < n2; ++u)
    itft_rec(r, sc, rows, s + u * col_step, z1, n1 + 1, 0, v_column(x, u, rows, cols), policy, count);
}

/* ------------------------------------------------------------------------ */
/* Top-level parallel driver: a job is one sub-transform of the top split.  */
typedef struct job {
  int inverse;
  uint64_t L, s, z, n;
  int f;
  view x;
} job;

typedef struct pool_arg {
  const or_ring* r;
  const job* jobs;
  uint64_t njobs;
  uint64_t next; /* atomic cursor */
  int policy;
  uint64_t count;
  int err;
} pool_arg;

static void* pool_worker(void* p) {
  pool_arg* a = (pool_arg*)p;
  scratch sc;
  if (scratch_init(&sc, a->r)) {
    __atomic_store_n(&a->err, 1, __ATOMIC_RELAXED);
    return NULL;
  }
  uint64_t cnt = 0;
  for (;;) {
    uint64_t i = __atomic_fetch_add(&a->next, 1, __ATOMIC_RELAXED);
    if (i >= a->njobs) break;
    const job* j = &a->jobs[i];
    if (j->inverse)
      itft_rec(a->r, &sc, j->L, j->s, j->z, j->n, j->f, j->x, a->policy, &cnt);
    else
      tft_rec(a->r, &sc, j->L, j->s, j->z, j->n, j->x, a->policy, &cnt);
  }
  __atomic_fetch_add(&a->count, cnt, __ATOMIC_RELAXED);
  scratch_free(&sc);
  return NULL;
}

static int run_jobs(const or_ring* r, const job* jobs, uint64_t njobs, int policy, int threads,
                    uint64_t* count) {
  if (njobs == 0) return OR_OK;
  pool_arg a = {r, jobs, njobs, 0, policy, 0, 0};
  int nt = threads < 1 ? 1 : threads;
  if ((uint64_t)nt > njobs) nt = (int)njobs;
  pthread_t tid[256];
  if (nt > 256) nt = 256;
  int started = 0;
  for (int t = 1; t < nt; ++t)
    if (pthread_create(&tid[t], NULL, pool_worker, &a) == 0) started = t;
    else break;
  pool_worker(&a);
  for (int t = 1; t <= started; ++t) pthread_join(tid[t], NULL);
  if (count) *count += a.count;
  return a.err ? OR_NOMEM : OR_OK;
}

static int check_length(const or_ring* r, uint64_t L) { /* transform.hpp:241-243 */
  return (L < 2 || (L & (L - 1)) != 0 || L > r->M) ? OR_BAD_LENGTH : OR_OK;
}

int or_tft(const or_ring* r, uint64_t L, uint64_t s, uint64_t z, uint64_t n, uint64_t* base,
           uint64_t stride, int policy, uint64_t* count, int threads) {
  if (check_length(r, L)) return OR_BAD_LENGTH;
  if (z < 1 || z > L || n < 1 || n > L) return OR_INVALID_PARAMS;
  if (stride < r->words) return OR_INVALID_PARAMS;
  view x = {base, stride, L};
  if (threads <= 1 || L == 2) {
    scratch sc;
    if (scratch_init(&sc, r)) return OR_NOMEM;
    tft_rec(r, &sc, L, s, z, n, x, policy, count);
    scratch_free(&sc);
    return OR_OK;
  }
  /* one level of the recursion by hand, sub-transforms as parallel jobs */
  unsigned ell = (unsigned)__builtin_ctzll(L), l1, l2;
  split(ell, policy, &l1, &l2);
  uint64_t cols = 1ull << l2, rows = 1ull << l1;
  uint64_t n2 = n & (cols - 1), n1 = n >> l2, n1c = n1 + (n2 ? 1 : 0);
  uint64_t z2 = z & (cols - 1), z1 = z >> l2, z2e = z1 ? cols : z2;
  uint64_t col_step = r->M >> ell;
  job* jobs = (job*)malloc(sizeof(job) * (cols + rows + 1));
  if (!jobs) return OR_NOMEM;
  uint64_t nj = 0;
  for (uint64_t u = 0; u < z2e; ++u) {
    job j = {0, rows, s + u * col_step, u < z2 ? z1 + 1 : z1, n1c, 0, v_column(x, u, rows, cols)};
    jobs[nj++] = j;
  }
  int rc = run_jobs(r, jobs, nj, policy, threads, count);
  nj = 0;
  uint64_t s_row = s << l1;
  for (uint64_t u = 0; u < n1; ++u) {
    job j = {0, cols, s_row, z2e, cols, 0, v_row(x, u, cols)};
    jobs[nj++] = j;
  }
  if (n2 > 0) {
    job j = {0, cols, s_row, z2e, n2, 0, v_row(x, n1, cols)};
    jobs[nj++] = j;
  }
  if (!rc) rc = run_jobs(r, jobs, nj, policy, threads, count);
  free(jobs);
  return rc;
}

int or_itft(const or_ring* r, uint64_t L, uint64_t s, uint64_t z, uint64_t n, int f, uint64_t* base,
            uint64_t stride, int policy, uint64_t* count, int threads) {
  if (check_length(r, L)) return OR_BAD_LENGTH;
  if (f != 0 && f != 1) return OR_INVALID_PARAMS;
  uint64_t nf = n + (uint64_t)f;
  if (z < 1 || z > L || nf < 1 || nf > L || z < n) return OR_INVALID_PARAMS;
  if (stride < r->words) return OR_INVALID_PARAMS;
  view x = {base, stride, L};
  if (threads <= 1 || L == 2) {
    scratch sc;
    if (scratch_init(&sc, r)) return OR_NOMEM;
    itft_rec(r, &sc, L, s, z, n, f, x, policy, count);
    scratch_free(&sc);
    return OR_OK;
  }
  unsigned ell = (unsigned)__builtin_ctzll(L), l1, l2;
  split(ell, policy, &l1, &l2);
  uint64_t cols = 1ull << l2, rows = 1ull << l1;
  uint64_t n2 = n & (cols - 1), n1 = n >> l2, z2 = z & (cols - 1), z1 = z >> l2;
  int fm = (n2 + (uint64_t)f > 0) ? 1 : 0;
  uint64_t z2e = z1 ? cols : z2;
  uint64_t lo = n2 < z2 ? n2 : z2, hi = n2 > z2 ? n2 : z2;
  uint64_t col_step = r->M >> ell, s_row = s << l1;
  job* jobs = (job*)malloc(sizeof(job) * (cols + rows + 1));
  if (!jobs) return OR_NOMEM;
  uint64_t nj = 0;
  int rc = OR_OK;
  for (uint64_t u = 0; u < n1; ++u) {
    job j = {1, cols, s_row, cols, cols, 0, v_row(x, u, cols)};
    jobs[nj++] = j;
  }
  rc = run_jobs(r, jobs, nj, policy, threads, count);
  nj = 0;
  for (uint64_t u = n2; u < z2e; ++u) {
    job j = {1, rows, s + u * col_step, u < hi ? z1 + 1 : z1, n1, fm, v_column(x, u, rows, cols)};
    jobs[nj++] = j;
  }
  if (!rc) rc = run_jobs(r, jobs, nj, policy, threads, count);
  if (!rc && fm) {
    job j = {1, cols, s_row, z2e, n2, f, v_row(x, n1, cols)};
    rc = run_jobs(r, &j, 1, policy, 1, count);
  }
  nj = 0;
  for (uint64_t u = 0; u < n2; ++u) {
    job j = {1, rows, s + u * col_step, u < lo ? z1 + 1 : z1, n1 + 1, 0, v_column(x, u, rows, cols)};
    jobs[nj++] = j;
  }
  if (!rc) rc = run_jobs(r, jobs, nj, policy, threads, count);
  free(jobs);
  return rc;
}

/* ------------------------------------------------------------------------ */
uint64_t or_bit_reverse(uint64_t j, unsigned ell) { /* transform.hpp:73-80 */
  uint64_t rr = 0;
  for (unsigned i = 0; i < ell; ++i) {
    rr = (rr << 1) | (j & 1);
    j >>= 1;
  }
  return rr;
}

/* dft_naive (transform.hpp:292-311), restated with twiddles only:
 * omega_L^e = omega^(e*M/L), zeta^j' = omega^(s*j'). */
int or_dft_naive(const or_ring* r, uint64_t L, uint64_t s, const uint64_t* coeffs, uint64_t z,
                 uint64_t cstride, uint64_t* out, uint64_t ostride) {
  if (L < 1 || (L & (L - 1)) != 0 || L > r->M) return OR_BAD_LENGTH;
  if (z < 1 || z > L) return OR_INVALID_PARAMS;
  scratch sc;
  if (scratch_init(&sc, r)) return OR_NOMEM;
  unsigned ell = (unsigned)__builtin_ctzll(L);
  uint64_t step = r->M / L;
  uint64_t* acc = (uint64_t*)calloc(r->words + 2, 8);
  uint64_t* term = (uint64_t*)calloc(2 * r->words + 8, 8);
  for (uint64_t j = 0; j < L; ++j) {
    uint64_t jr = or_bit_reverse(j, ell);
    r_zero(r, acc);
    for (uint64_t i = 0; i < z; ++i) {
      uint64_t e = (uint64_t)(((u128)i * jr) % L);
      r_twiddle(r, &sc, e * step, term, coeffs + i * cstride);
      r_add(r, &sc, acc, acc, term);
    }
    r_twiddle(r, &sc, (uint64_t)(((u128)s * jr) % r->M), out + j * ostride, acc);
  }
  free(acc);
  free(term);
  scratch_free(&sc);
  return OR_OK;
}

uint64_t or_tft_bound_2x(uint64_t L, uint64_t n) { /* transform.hpp:316-320 */
  uint64_t ell = (uint64_t)__builtin_ctzll(L);
  uint64_t a = (n - 1) * ell + 2 * (L - 1), b = L * ell;
  return a < b ? a : b;
}
uint64_t or_itft_bound_2x(uint64_t L, uint64_t n, int f) { /* transform.hpp:322-327 */
  uint64_t ell = (uint64_t)__builtin_ctzll(L);
  uint64_t a = (n + (uint64_t)f - 1) * ell + 2 * (L - 1), b = L * ell;
  return a < b ? a : b;
}
