"""Polynomial multiplication over the big rings (polymul.hpp:48-95 restated
for R = Z/(2^N+1) and R = (Z/mZ)[y]/(y^K+1)), and the two BASELINE
multiplication pipelines built on it:

  config 3  Schoenhage-Nussbaumer: negacyclic product in (Z/mZ)[x] mod
            x^(K s) + 1 via R = (Z/mZ)[y]/(y^K+1), y = x^s
  config 4  Schoenhage-Strassen: product in Z[x] via R = Z/(2^N+1),
            N = k L / 2 the smallest size holding the output coefficients
            

Everything runs on the GPU: the transforms (cf_tft / cf_itft), the pointwise
ring products (cftft_gpu_pointwise), the final L^-1 scale, packing and
recombination (torch tensor ops on device memory).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import (ButterflyStats, DeviceView, FermatRingCtx, InvalidParams, NegacyclicRingCtx, SplitPolicy,
               TransformParams, _check, _stream_ptr, cf_itft, cf_tft, lib, scale)


class TooLarge(ValueError):
    """polymul.hpp:13-18: the product does not fit the root order."""


@dataclass
class MulStats:
    """polymul.hpp:39-43."""
    pointwise_mults: int = 0
    transform_length: int = 0
    butterflies: ButterflyStats = field(default_factory=ButterflyStats)


def choose_length(ctx, n: int) -> int:
    """Smallest power-of-two length >= max(n, 2) within the root order (polymul.hpp:33-37)."""
    if n < 1:
        raise InvalidParams("choose_length requires n >= 1")
    if n > ctx.root_order():
        raise TooLarge(f"product length {n} exceeds the available root order {ctx.root_order()}")
    L = 2
    while L < n:
        L <<= 1
    return L


def pointwise(ctx, a: torch.Tensor, b: torch.Tensor, count: int, stream=None) -> None:
    """a[i] <- a[i] * b[i] for i < count (device tensors of elements, rows)."""
    assert a.shape[1] == b.shape[1]
    _check(lib().cftft_gpu_pointwise(ctx._h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), count,
                                     a.shape[1] * 8, C.c_void_p(_stream_ptr(stream))))


def mul_scalar(ctx, a: torch.Tensor, count: int, c: int, stream=None) -> None:
    _check(lib().cftft_gpu_mul_scalar(ctx._h, C.c_void_p(a.data_ptr()), count, a.shape[1] * 8, c,
                                      C.c_void_p(_stream_ptr(stream))))


def poly_mul(ctx, G: torch.Tensor, H: torch.Tensor, zg: int, zh: int, policy=SplitPolicy.balanced,
             stats: MulStats | None = None) -> torch.Tensor:
    """Product of two polynomials over the ring (polymul.hpp:48-95): G, H are
    CUDA tensors of elements (rows) with supports zg, zh.  Returns the n =
    zg + zh - 1 coefficients of the product (canonical elements)."""
    if stats is not None:
        stats.__init__()
    if zg == 0 or zh == 0:
        return G[:0]
    n = zg + zh - 1
    L = choose_length(ctx, n)
    W = ctx.element_words
    g = torch.zeros((L, W), dtype=torch.int64, device=G.device)
    h = torch.zeros((L, W), dtype=torch.int64, device=G.device)
    g[:zg] = G[:zg]
    h[:zh] = H[:zh]
    bs = ButterflyStats()
    cf_tft(ctx, TransformParams(L, 0, zg, n), DeviceView(g), policy, bs)
    cf_tft(ctx, TransformParams(L, 0, zh, n), DeviceView(h), policy, bs)
    pointwise(ctx, g, h, n)
    cf_itft(ctx, TransformParams(L, 0, n, n, 0), DeviceView(g), policy, bs)
    ell = L.bit_length() - 1
    if isinstance(ctx, FermatRingCtx):
        scale(ctx, DeviceView(g), n, ctx.root_order() - ell)  # 1/L = omega^(M - ell)
    else:
        mul_scalar(ctx, g, n, pow(L, -1, ctx.m))
    if stats is not None:
        stats.pointwise_mults = n
        stats.transform_length = L
        stats.butterflies = bs
    return g[:n]


# ---------------------------------------------------------------------------
# config 3: Nussbaumer


def nussbaumer_negacyclic_mul(f: torch.Tensor, g: torch.Tensor, m: int, K: int, s: int,
                              policy=SplitPolicy.balanced, stats: MulStats | None = None) -> torch.Tensor:
    """h = f * g mod (x^(K s) + 1) over Z/mZ for int64 CUDA tensors of K*s
    residues.  Split x^(j + s k) -> z^j y^k with y = x^s (y^K = -1), multiply
    in R[z] with R = (Z/mZ)[y]/(y^K+1) (TFT length L = 2s, omega = y), and
    recombine h_j = C_j + y C_{j+s}."""
    assert f.numel() == K * s and g.numel() == K * s
    ctx = _RINGS.get(("negacyclic", K, m))
    if ctx is None:
        ctx = _RINGS[("negacyclic", K, m)] = NegacyclicRingCtx(K, m)
    A = f.view(K, s).t().contiguous()  # A[j][k] = f[j + s k]
    B = g.view(K, s).t().contiguous()
    Cz = poly_mul(ctx, A, B, s, s, policy, stats)  # 2s - 1 elements of R
    top = torch.zeros((s, K), dtype=torch.int64, device=f.device)
    top[: s - 1] = Cz[s:]
    # y * C: negacyclic shift by one word
    yC = torch.roll(top, 1, dims=1)
    yC[:, 0] = torch.where(yC[:, 0] == 0, yC[:, 0], m - yC[:, 0])
    hb = Cz[:s] + yC
    hb = torch.where(hb >= m, hb - m, hb)
    return hb.t().contiguous().view(-1)


# ---------------------------------------------------------------------------
# config 4: Schoenhage-Strassen


_RINGS: dict = {}


def _fermat_ring(N: int) -> "FermatRingCtx":
    """One ring context per N, kept: a ring owns its plan cache and scratch
    (the reference's callers likewise build a RingCtx once, field.hpp:84-100),
    so repeated products re-plan nothing."""
    r = _RINGS.get(("fermat", N))
    if r is None:
        r = _RINGS[("fermat", N)] = FermatRingCtx(N)
    return r


def ss_ring_bits(L: int, out_bits: int) -> int:
    """N = k L / 2 for the smallest k with N > out_bits, N a power
    of two here (so that M = 2N is a power of two); at least 512, the smallest
    ring the GPU pointwise multiplier takes."""
    N = max(L // 2, 512)
    while N <= out_bits:
        N *= 2
    return N


def ss_mul(F: torch.Tensor, G: torch.Tensor, coeff_bits: int, policy=SplitPolicy.balanced,
           stats: MulStats | None = None):
    """Product of two polynomials in Z[x] with unsigned coefficients < 2^coeff_bits.
    F, G: uint64-limb CUDA tensors [len, limbs] (int64 dtype).  Returns
    (H, N): H [lenF + lenG - 1, N/64] limbs of the product coefficients."""
    zf, zg = F.shape[0], G.shape[0]
    n = zf + zg - 1
    L = 2
    while L < n:
        L <<= 1
    out_bits = 2 * coeff_bits + (min(zf, zg)).bit_length()
    N = ss_ring_bits(L, out_bits)
    ctx = _fermat_ring(N)
    W = ctx.element_words
    limbs = F.shape[1]
    A = torch.zeros((zf, W), dtype=torch.int64, device=F.device)
    B = torch.zeros((zg, W), dtype=torch.int64, device=F.device)
    A[:, :limbs] = F
    B[:, :limbs] = G
    H = poly_mul(ctx, A, B, zf, zg, policy, stats)
    return H[:, : N // 64], N
