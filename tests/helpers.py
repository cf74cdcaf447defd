"""Shared helpers for the parity tests (seeded inputs, GPU <-> numpy plumbing)."""
from __future__ import annotations

import numpy as np

import pyoracle as po


def fermat_inputs(N: int, L: int, z: int, W: int, seed: int, special: bool = False) -> np.ndarray:
    """(L, W) uint64 buffer: rows [0,z) hold canonical residues of Z/(2^N+1)
    (uniform limbs, top word 0); rows >= z hold a poison pattern that is not a
    canonical residue (transform.hpp:58-70: those cells must never be read)."""
    lim = N // 64
    rng = np.random.default_rng(seed)
    buf = np.full((L, W), 0xDEADBEEFDEADBEEF, dtype=np.uint64)
    buf[:z, :lim] = rng.integers(0, 1 << 64, size=(z, lim), dtype=np.uint64, endpoint=False)
    buf[:z, lim:] = 0
    if special and z >= 4:
        # carry/borrow stress: 0, 2^N (== -1), 2^N - 1 (all ones), 1
        buf[0, :] = 0
        buf[1, :] = 0
        buf[1, lim] = 1
        buf[2, :lim] = np.uint64(0xFFFFFFFFFFFFFFFF)
        buf[2, lim:] = 0
        buf[3, :] = 0
        buf[3, 0] = 1
    return buf


def negacyclic_inputs(K: int, m: int, L: int, z: int, W: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    buf = np.full((L, W), 0xDEADBEEFDEADBEEF, dtype=np.uint64)
    buf[:z, :K] = rng.integers(0, m, size=(z, K), dtype=np.uint64)
    return buf


def random_modulus(seed: int) -> int:
    """m = (next() & (2^62-1)) | 2^61 | 1: odd, exactly 62 bits."""
    g = po.MT19937_64(seed)
    return (g.next() & ((1 << 62) - 1)) | (1 << 61) | 1


def to_dev(buf: np.ndarray):
    import torch

    return torch.from_numpy(np.ascontiguousarray(buf).view(np.int64)).cuda()


def from_dev(t) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)
