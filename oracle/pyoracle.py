"""ctypes bindings for the CPU oracle (liboracle.so) and the reference shim.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package never
imports this module.

Element buffers are numpy uint64 arrays shaped (L, stride_words); element i of
a view is row i.  Fermat elements are N/64 limbs + a top word (canonical value
in [0, 2^N]); negacyclic elements are K words in [0, m); prime elements are one
word (cftft::Fp, field.hpp:31-34).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libcftft_ref.so")

PRIME, FERMAT, NEGACYCLIC = 0, 1, 2
BALANCED, RADIX2 = 0, 1
OK, BAD_LENGTH, INVALID_PARAMS = 0, 1, 2

GOLDILOCKS = 0xFFFFFFFF00000001


class OrRing(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("M", C.c_uint64),
        ("words", C.c_uint64),
        ("p", C.c_uint64),
        ("omega", C.c_uint64),
        ("inv2", C.c_uint64),
        ("two_adicity", C.c_uint),
        ("N", C.c_uint64),
        ("K", C.c_uint64),
        ("m", C.c_uint64),
    ]


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None
_ref = None
U64P = C.POINTER(C.c_uint64)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = C.CDLL(_LIB)
        rp = C.POINTER(OrRing)
        L.or_ring_init_prime.argtypes = [rp, C.c_uint64, C.c_uint]
        L.or_ring_init_fermat.argtypes = [rp, C.c_uint64]
        L.or_ring_init_negacyclic.argtypes = [rp, C.c_uint64, C.c_uint64]
        for f in ("or_add", "or_sub", "or_mul"):
            getattr(L, f).argtypes = [rp, U64P, U64P, U64P]
            getattr(L, f).restype = None
        L.or_twiddle.argtypes = [rp, C.c_uint64, U64P, U64P]
        L.or_twiddle.restype = None
        L.or_half.argtypes = [rp, U64P, U64P]
        L.or_half.restype = None
        L.or_tft_base2.argtypes = [rp, C.c_uint64, C.c_uint64, C.c_uint64, U64P, U64P, U64P]
        L.or_tft_base2.restype = None
        L.or_itft_base2.argtypes = [rp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, U64P, U64P, U64P]
        L.or_itft_base2.restype = None
        L.or_tft.argtypes = [rp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, U64P, C.c_uint64,
                             C.c_int, U64P, C.c_int]
        L.or_itft.argtypes = [rp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, U64P,
                              C.c_uint64, C.c_int, U64P, C.c_int]
        L.or_dft_naive.argtypes = [rp, C.c_uint64, C.c_uint64, U64P, C.c_uint64, C.c_uint64, U64P,
                                   C.c_uint64]
        L.or_bit_reverse.argtypes = [C.c_uint64, C.c_uint]
        L.or_bit_reverse.restype = C.c_uint64
        L.or_tft_bound_2x.argtypes = [C.c_uint64, C.c_uint64]
        L.or_tft_bound_2x.restype = C.c_uint64
        L.or_itft_bound_2x.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.or_itft_bound_2x.restype = C.c_uint64
        L.or_set_fault.argtypes = [C.c_int]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF)


def ref():
    global _ref
    if _ref is None:
        R = C.CDLL(_REF)
        R.ref_tft.argtypes = [C.c_uint64, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                              U64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, U64P]
        R.ref_itft.argtypes = [C.c_uint64, C.c_uint, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                               C.c_int, U64P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, U64P]
        R.ref_dft_naive.argtypes = [C.c_uint64, C.c_uint, C.c_uint64, C.c_uint64, U64P, C.c_uint64,
                                    U64P]
        R.ref_omega.argtypes = [C.c_uint64, C.c_uint]
        R.ref_omega.restype = C.c_uint64
        R.ref_run_all_suites.argtypes = [C.c_uint64, C.c_uint, C.c_uint, C.c_uint64, U64P, U64P]
        R.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        R.ref_mix_seed.restype = C.c_uint64
        R.ref_poly_mul.argtypes = [C.c_uint64, C.c_uint, U64P, C.c_uint64, U64P, C.c_uint64, U64P,
                                   C.c_int, U64P]
        R.ref_poly_mul.restype = C.c_int64
        _ref = R
    return _ref


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(U64P)


class OracleError(Exception):
    def __init__(self, code: int):
        super().__init__({BAD_LENGTH: "BadLength", INVALID_PARAMS: "InvalidParams"}.get(code, str(code)))
        self.code = code


class Ring:
    """A ring instance of the oracle."""

    def __init__(self, kind: int, **kw):
        self.r = OrRing()
        if kind == PRIME:
            rc = lib().or_ring_init_prime(C.byref(self.r), kw["p"], kw["m"])
        elif kind == FERMAT:
            rc = lib().or_ring_init_fermat(C.byref(self.r), kw["N"])
        else:
            rc = lib().or_ring_init_negacyclic(C.byref(self.r), kw["K"], kw["m"])
        if rc:
            raise OracleError(rc)
        self.kind = kind

    @staticmethod
    def prime(p: int, m: int) -> "Ring":
        return Ring(PRIME, p=p, m=m)

    @staticmethod
    def fermat(N: int) -> "Ring":
        return Ring(FERMAT, N=N)

    @staticmethod
    def negacyclic(K: int, m: int) -> "Ring":
        return Ring(NEGACYCLIC, K=K, m=m)

    @property
    def M(self) -> int:
        return self.r.M

    @property
    def words(self) -> int:
        return self.r.words

    # --- element helpers -------------------------------------------------
    def zeros(self, L: int, stride: int | None = None) -> np.ndarray:
        return np.zeros((L, stride or self.words), dtype=np.uint64)

    def _e(self):
        return np.zeros(2 * self.words + 8, dtype=np.uint64)

    def add(self, a, b):
        o = self._e()
        lib().or_add(C.byref(self.r), _p(o), _p(np.ascontiguousarray(a, np.uint64)),
                     _p(np.ascontiguousarray(b, np.uint64)))
        return o[: self.words]

    def sub(self, a, b):
        o = self._e()
        lib().or_sub(C.byref(self.r), _p(o), _p(np.ascontiguousarray(a, np.uint64)),
                     _p(np.ascontiguousarray(b, np.uint64)))
        return o[: self.words]

    def mul(self, a, b):
        o = self._e()
        lib().or_mul(C.byref(self.r), _p(o), _p(np.ascontiguousarray(a, np.uint64)),
                     _p(np.ascontiguousarray(b, np.uint64)))
        return o[: self.words]

    def twiddle(self, s, x):
        o = self._e()
        lib().or_twiddle(C.byref(self.r), s % (1 << 64), _p(o), _p(np.ascontiguousarray(x, np.uint64)))
        return o[: self.words]

    def half(self, x):
        o = self._e()
        lib().or_half(C.byref(self.r), _p(o), _p(np.ascontiguousarray(x, np.uint64)))
        return o[: self.words]

    # --- transforms ------------------------------------------------------
    def tft(self, buf: np.ndarray, L, s, z, n, policy=BALANCED, threads=1, count=False):
        """In place on buf (shape (L, stride)); returns the base-case count."""
        c = C.c_uint64(0)
        rc = lib().or_tft(C.byref(self.r), L, s % (1 << 64), z, n, _p(buf), buf.shape[1], policy,
                          C.byref(c), threads)
        if rc:
            raise OracleError(rc)
        return c.value

    def itft(self, buf: np.ndarray, L, s, z, n, f=0, policy=BALANCED, threads=1):
        c = C.c_uint64(0)
        rc = lib().or_itft(C.byref(self.r), L, s % (1 << 64), z, n, f, _p(buf), buf.shape[1], policy,
                           C.byref(c), threads)
        if rc:
            raise OracleError(rc)
        return c.value

    def tft_at(self, buf: np.ndarray, base: int, stride: int, L, s, z, n, policy=BALANCED):
        """In place on the strided view buf[base + i * stride], i < L (element
        rows of a 2-D buffer): the sub-transforms of a Bailey decomposition."""
        W = buf.shape[1]
        ptr = C.cast(buf.ctypes.data + 8 * W * base, U64P)
        c = C.c_uint64(0)
        rc = lib().or_tft(C.byref(self.r), L, s % (1 << 64), z, n, ptr, W * stride, policy, C.byref(c), 1)
        if rc:
            raise OracleError(rc)
        return c.value

    def itft_at(self, buf: np.ndarray, base: int, stride: int, L, s, z, n, f=0, policy=BALANCED):
        W = buf.shape[1]
        ptr = C.cast(buf.ctypes.data + 8 * W * base, U64P)
        c = C.c_uint64(0)
        rc = lib().or_itft(C.byref(self.r), L, s % (1 << 64), z, n, f, ptr, W * stride, policy, C.byref(c), 1)
        if rc:
            raise OracleError(rc)
        return c.value

    def dft_naive(self, L, s, coeffs: np.ndarray) -> np.ndarray:
        coeffs = np.ascontiguousarray(coeffs, np.uint64)
        out = np.zeros((L, self.words), dtype=np.uint64)
        rc = lib().or_dft_naive(C.byref(self.r), L, s % (1 << 64), _p(coeffs), coeffs.shape[0],
                                coeffs.shape[1], _p(out), self.words)
        if rc:
            raise OracleError(rc)
        return out


def bit_reverse(j: int, ell: int) -> int:
    return lib().or_bit_reverse(j, ell)


def tft_bound(L: int, n: int) -> int:
    return lib().or_tft_bound_2x(L, n) // 2


def itft_bound(L: int, n: int, f: int) -> int:
    return lib().or_itft_bound_2x(L, n, f) // 2


def set_fault(on: bool) -> None:
    lib().or_set_fault(1 if on else 0)


# ---------------------------------------------------------------------------
# Seeded inputs (verify.hpp:17-37): mix_seed + std::mt19937_64.


def mix_seed(a: int, b: int) -> int:
    """splitmix64-style mixer, restated from verify.hpp:17-25."""
    M = (1 << 64) - 1
    x = (a + 0x9E3779B97F4A7C15 * (b + 1)) & M
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & M
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & M
    x ^= x >> 31
    return x


class MT19937_64:
    """std::mt19937_64, restated (the engine behind verify.hpp:27-37)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def next(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEEA00000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF

    def below(self, bound: int) -> int:
        return self.next() % bound

    def words(self, count: int) -> np.ndarray:
        return np.array([self.next() for _ in range(count)], dtype=np.uint64)


def fast_words(seed: int, count: int) -> np.ndarray:
    """Bulk uniform u64 words for the large configs (numpy PCG64 seeded from the
    reference's mixer; the oracle and the GPU consume identical bytes)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.integers(0, 1 << 64, size=count, dtype=np.uint64, endpoint=False)
