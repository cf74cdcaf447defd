"""Independent big-integer model of the target rings (pure Python ints).

TEST INFRASTRUCTURE ONLY.  Shares nothing with the C oracle but the
mathematics: it evaluates the weighted transform straight from its definition
(transform.hpp:288-311) and the ITFT's defining relations
(transform.hpp:266-272), for small rings, to pin the big-ring arithmetic that
the reference's own tests cannot pin (the reference only implements a 64-bit
prime field).  tests/golden/make_golden.py uses it to write the
committed fixtures.

Element <-> u64-word conversions follow the GPU/oracle storage formats:
  Fermat Z/(2^N+1):  N/64 limbs + top word, value in [0, 2^N]
  negacyclic (Z/mZ)[y]/(y^K+1): K words in [0, m)
"""
from __future__ import annotations

import numpy as np


def bitrev(j: int, ell: int) -> int:
    r = 0
    for _ in range(ell):
        r = (r << 1) | (j & 1)
        j >>= 1
    return r


class FermatModel:
    """R = Z/(2^N+1), omega = 2 of order M = 2N."""

    def __init__(self, N: int):
        self.N = N
        self.P = (1 << N) + 1
        self.M = 2 * N
        self.words = N // 64 + 1

    def tw(self, s: int, x: int) -> int:
        return (x * pow(2, s % self.M, self.P)) % self.P

    def to_words(self, x: int) -> np.ndarray:
        assert 0 <= x <= (1 << self.N)
        return np.array([(x >> (64 * i)) & ((1 << 64) - 1) for i in range(self.words)], dtype=np.uint64)

    def from_words(self, w) -> int:
        v = 0
        for i in range(self.words):
            v |= int(w[i]) << (64 * i)
        return v

    def dft(self, L: int, s: int, coeffs: list[int]) -> list[int]:
        ell = L.bit_length() - 1
        step = self.M // L
        out = []
        for j in range(L):
            jr = bitrev(j, ell)
            acc = 0
            for i, a in enumerate(coeffs):
                acc += a * pow(2, (step * i * jr) % self.M, self.P)
            out.append(self.tw(s * jr, acc % self.P))
        return out


class NegacyclicModel:
    """R = (Z/mZ)[y]/(y^K+1), omega = y of order M = 2K.  Elements are lists."""

    def __init__(self, K: int, m: int):
        self.K, self.m, self.M = K, m, 2 * K
        self.words = K

    def tw(self, s: int, x: list[int]) -> list[int]:
        s %= self.M
        out = [0] * self.K
        for i, v in enumerate(x):
            e = i + s
            sign = 1
            while e >= self.K:
                e -= self.K
                sign = -sign
            out[e] = (sign * v) % self.m
        return out

    def add(self, a, b):
        return [(x + y) % self.m for x, y in zip(a, b)]

    def scale(self, c: int, a):
        return [(c * x) % self.m for x in a]

    def dft(self, L: int, s: int, coeffs: list[list[int]]) -> list[list[int]]:
        ell = L.bit_length() - 1
        step = self.M // L
        out = []
        for j in range(L):
            jr = bitrev(j, ell)
            acc = [0] * self.K
            for i, a in enumerate(coeffs):
                acc = self.add(acc, self.tw(step * i * jr, a))
            out.append(self.tw(s * jr, acc))
        return out

    def to_words(self, x) -> np.ndarray:
        return np.array(x, dtype=np.uint64)

    def from_words(self, w) -> list[int]:
        return [int(v) for v in w[: self.K]]
