"""Polynomial multiplication over the big rings (polymul.hpp:48-95 restated
for R = Z/(2^N+1) and R = (Z/mZ)[y]/(y^K+1)), and the two BASELINE
multiplication pipelines built on it:

  config 3  Schoenhage-Nussbaumer: negacyclic product in (Z/mZ)[x] mod
            x^(K s) + 1 via R = (Z/mZ)[y]/(y^K+1), y = x^s
  config 4  Schoenhage-Strassen: product in Z[x] via R = Z/(2^N+1),
            N = k L / 2 the smallest size holding the output coefficients
            

Everything runs on the GPU through the C ABI (include/cftft_b200.h):
cftft_gpu_poly_mul (two TFTs, the n pointwise products with L^-1 folded in,
the ITFT), cftft_gpu_pack_limbs (SS packing), cftft_gpu_nussbaumer_split /
_join (the x^(j+sk) <-> z^j y^k reshapes and the y C recombination).  torch
only allocates device memory.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import (ButterflyStats, FermatRingCtx, InvalidParams, NegacyclicRingCtx, SplitPolicy, _check, _stream_ptr,
               lib)


class TooLarge(ValueError):
    """polymul.hpp:13-18: the product does not fit the root order."""


@dataclass
class MulStats:
    """polymul.hpp:39-43."""
    pointwise_mults: int = 0
    transform_length: int = 0
    butterflies: ButterflyStats = field(default_factory=ButterflyStats)


class _CMulStats(C.Structure):
    _fields_ = [("pointwise_mults", C.c_uint64), ("transform_length", C.c_uint64),
                ("base_case_count", C.c_uint64)]


def _bind():
    L = lib()
    if not getattr(L, "_polymul_bound", False):
        vp, u64 = C.c_void_p, C.c_uint64
        L.cftft_gpu_poly_mul.argtypes = [vp, vp, u64, vp, u64, vp, u64, C.c_int, C.POINTER(_CMulStats), vp]
        L.cftft_gpu_poly_support.argtypes = [vp, vp, u64, u64, C.POINTER(u64), vp]
        L.cftft_gpu_pointwise_scaled.argtypes = [vp, vp, vp, u64, u64, u64, vp]
        L.cftft_gpu_pack_limbs.argtypes = [vp, vp, u64, vp, u64, u64, vp]
        L.cftft_gpu_nussbaumer_split.argtypes = [vp, vp, u64, vp, u64, vp]
        L.cftft_gpu_nussbaumer_join.argtypes = [vp, vp, vp, u64, u64, vp]
        L._polymul_bound = True
    return L


def _call(rc: int) -> None:
    if rc == 7:
        raise TooLarge(lib().cftft_last_error().decode())
    _check(rc)


def poly_support(ctx, A: torch.Tensor, stream=None) -> int:
    """1 + deg (trailing zero elements ignored), polymul.hpp:26-30."""
    out = C.c_uint64()
    _call(_bind().cftft_gpu_poly_support(ctx._h, C.c_void_p(A.data_ptr()), A.shape[0], A.shape[1] * 8,
                                         C.byref(out), C.c_void_p(_stream_ptr(stream))))
    return out.value


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


def poly_mul(ctx, G: torch.Tensor, H: torch.Tensor, zg: int | None = None, zh: int | None = None,
             policy=SplitPolicy.balanced, stats: MulStats | None = None, stream=None) -> torch.Tensor:
    """Product of two polynomials over the ring (polymul.hpp:48-95) through
    cftft_gpu_poly_mul: G, H are CUDA tensors of elements (rows); supports
    zg, zh default to poly_support.  Returns the n = zg + zh - 1
    coefficients of the product (canonical elements)."""
    if stats is not None:
        stats.__init__()
    if zg is None:
        zg = poly_support(ctx, G, stream)
    if zh is None:
        zh = poly_support(ctx, H, stream)
    if zg == 0 or zh == 0:
        return G[:0]
    n = zg + zh - 1
    out = torch.empty((n, ctx.element_words), dtype=torch.int64, device=G.device)
    cs = _CMulStats()
    _call(_bind().cftft_gpu_poly_mul(ctx._h, C.c_void_p(G.data_ptr()), zg, C.c_void_p(H.data_ptr()), zh,
                                     C.c_void_p(out.data_ptr()), ctx.element_words * 8, int(policy), C.byref(cs),
                                     C.c_void_p(_stream_ptr(stream))))
    if stats is not None:
        stats.pointwise_mults = cs.pointwise_mults
        stats.transform_length = cs.transform_length
        stats.butterflies = ButterflyStats(cs.base_case_count)
    return out


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
    L = _bind()
    eb = ctx.element_words * 8
    f, g = f.contiguous(), g.contiguous()
    A = torch.empty((s, K), dtype=torch.int64, device=f.device)
    B = torch.empty((s, K), dtype=torch.int64, device=f.device)
    _call(L.cftft_gpu_nussbaumer_split(ctx._h, C.c_void_p(A.data_ptr()), eb, C.c_void_p(f.data_ptr()), s, None))
    _call(L.cftft_gpu_nussbaumer_split(ctx._h, C.c_void_p(B.data_ptr()), eb, C.c_void_p(g.data_ptr()), s, None))
    Cz = poly_mul(ctx, A, B, s, s, policy, stats)  # 2s - 1 elements of R
    h = torch.empty(K * s, dtype=torch.int64, device=f.device)
    _call(L.cftft_gpu_nussbaumer_join(ctx._h, C.c_void_p(h.data_ptr()), C.c_void_p(Cz.data_ptr()), eb, s, None))
    return h


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
    L = _bind()
    A = torch.empty((zf, W), dtype=torch.int64, device=F.device)
    B = torch.empty((zg, W), dtype=torch.int64, device=F.device)
    Fc, Gc = F.contiguous(), G.contiguous()
    _call(L.cftft_gpu_pack_limbs(ctx._h, C.c_void_p(A.data_ptr()), W * 8, C.c_void_p(Fc.data_ptr()), limbs, zf, None))
    _call(L.cftft_gpu_pack_limbs(ctx._h, C.c_void_p(B.data_ptr()), W * 8, C.c_void_p(Gc.data_ptr()), limbs, zg, None))
    H = poly_mul(ctx, A, B, zf, zg, policy, stats)
    return H[:, : N // 64], N
