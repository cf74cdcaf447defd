"""GPU multiplication pipelines (BASELINE configs 3 and 4) and the pointwise
ring products, against the CPU oracle / schoolbook products
(polymul_test.cpp:11-19, 81-162 restated for the big rings)."""
from __future__ import annotations

import ctypes as C
import random
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import pyoracle as po
from helpers import from_dev, random_modulus, to_dev

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_0810_3203_b200 as cf  # noqa: E402
from paper_0810_3203_b200 import polymul as pm  # noqa: E402


@pytest.mark.parametrize("N", [512, 1024, 65536])
def test_fermat_pointwise_matches_oracle(N):
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    W = ctx.element_words
    lim = N // 64
    cnt = 24 if N == 65536 else 200
    rng = np.random.default_rng(N)
    a = np.zeros((cnt, W), dtype=np.uint64)
    b = np.zeros((cnt, W), dtype=np.uint64)
    a[:, :lim] = rng.integers(0, 1 << 64, size=(cnt, lim), dtype=np.uint64, endpoint=False)
    b[:, :lim] = rng.integers(0, 1 << 64, size=(cnt, lim), dtype=np.uint64, endpoint=False)
    # edge values: 0, 1, 2^N (== -1), 2^N - 1
    a[0, :] = 0
    a[1, :] = 0
    a[1, lim] = 1
    b[2, :] = 0
    b[2, lim] = 1
    a[3, :lim] = np.uint64(0xFFFFFFFFFFFFFFFF)
    a[4, :] = 0
    a[4, 0] = 1
    a[5, :] = 0  # (-1) * 1 = -1 (top word 1)
    a[5, lim] = 1
    b[5, :] = 0
    b[5, 0] = 1
    a[6, :lim] = np.uint64(0xFFFFFFFFFFFFFFFF)  # (-2) * (-2) = 4
    b[6, :lim] = np.uint64(0xFFFFFFFFFFFFFFFF)
    a[7, :] = 0  # (-1) * (-1) = 1
    a[7, lim] = 1
    b[7, :] = 0
    b[7, lim] = 1
    da, db = to_dev(a), to_dev(b)
    pm.pointwise(ctx, da, db, cnt)  # outputs canonical, no canonicalize pass
    got = from_dev(da)
    for i in range(cnt):
        want = ring.mul(a[i, : lim + 1], b[i, : lim + 1])
        assert np.array_equal(got[i, : lim + 1], want), i


def test_negacyclic_pointwise_matches_oracle():
    for K in (4, 64, 1024):
        m = random_modulus(K + 1)
        ctx = cf.NegacyclicRingCtx(K, m)
        ring = po.Ring.negacyclic(K, m)
        cnt = 8
        rng = np.random.default_rng(K)
        a = rng.integers(0, m, size=(cnt, K), dtype=np.uint64)
        b = rng.integers(0, m, size=(cnt, K), dtype=np.uint64)
        da, db = to_dev(a), to_dev(b)
        pm.pointwise(ctx, da, db, cnt)
        got = from_dev(da)
        for i in range(cnt):
            assert np.array_equal(got[i], ring.mul(a[i], b[i])), (K, i)


def _negacyclic_schoolbook(f, g, m):
    n = len(f)
    out = [0] * n
    for i, x in enumerate(f):
        if x == 0:
            continue
        for j, y in enumerate(g):
            k = i + j
            if k < n:
                out[k] = (out[k] + x * y) % m
            else:
                out[k - n] = (out[k - n] - x * y) % m
    return out


@pytest.mark.parametrize("K,s", [(4, 4), (8, 8), (16, 16), (32, 8)])
def test_nussbaumer_small_matches_schoolbook(K, s):
    m = random_modulus(K * s)
    rnd = random.Random(K * s)
    f = [rnd.randrange(m) for _ in range(K * s)]
    g = [rnd.randrange(m) for _ in range(K * s)]
    ft = torch.tensor(np.array(f, dtype=np.uint64).view(np.int64), device="cuda")
    gt = torch.tensor(np.array(g, dtype=np.uint64).view(np.int64), device="cuda")
    st = pm.MulStats()
    h = pm.nussbaumer_negacyclic_mul(ft, gt, m, K, s, stats=st)
    got = [int(v) for v in h.cpu().numpy().view(np.uint64)]
    assert got == _negacyclic_schoolbook(f, g, m)
    assert st.pointwise_mults == 2 * s - 1 and st.transform_length == 2 * s  # polymul.hpp:39-43


def test_ss_small_matches_schoolbook():
    """SS multiplication in Z[x] against Python integers (polymul_test.cpp:81-97)."""
    rnd = random.Random(7)
    for zf, zg, bits in [(60, 45, 100), (17, 1, 200), (1, 1, 64), (33, 31, 300)]:
        F = [rnd.getrandbits(bits) for _ in range(zf)]
        G = [rnd.getrandbits(bits) for _ in range(zg)]
        limbs = (bits + 63) // 64
        Ft = np.array([[(x >> (64 * k)) & ((1 << 64) - 1) for k in range(limbs)] for x in F], dtype=np.uint64)
        Gt = np.array([[(x >> (64 * k)) & ((1 << 64) - 1) for k in range(limbs)] for x in G], dtype=np.uint64)
        H, N = pm.ss_mul(to_dev(Ft), to_dev(Gt), bits)
        Hn = from_dev(H)
        want = [0] * (zf + zg - 1)
        for i, x in enumerate(F):
            for j, y in enumerate(G):
                want[i + j] += x * y
        got = [sum(int(Hn[i, k]) << (64 * k) for k in range(Hn.shape[1])) for i in range(Hn.shape[0])]
        assert got == want, (zf, zg, bits)


@pytest.mark.slow
def test_config3_full_size_matches_oracle():
    """BASELINE config 3: two length-2^20 polynomials mod an odd 62-bit m,
    R = (Z/mZ)[y]/(y^1024+1), TFT length 2^11 with omega = y: product
    bit-exact against the oracle pipeline (oracle TFT / schoolbook ring
    products / ITFT)."""
    K = s = 1024
    m = random_modulus(po.mix_seed(42, 3))
    rng = np.random.default_rng(po.mix_seed(42, 3))
    f = rng.integers(0, m, size=K * s, dtype=np.uint64)
    g = rng.integers(0, m, size=K * s, dtype=np.uint64)
    h = pm.nussbaumer_negacyclic_mul(to_dev(f.reshape(-1, 1)).view(-1), to_dev(g.reshape(-1, 1)).view(-1), m, K, s)
    got = h.cpu().numpy().view(np.uint64)
    # oracle: same mapping on the CPU
    ring = po.Ring.negacyclic(K, m)
    L, n = 2 * s, 2 * s - 1
    A = np.zeros((L, K), dtype=np.uint64)
    B = np.zeros((L, K), dtype=np.uint64)
    A[:s] = f.reshape(K, s).T
    B[:s] = g.reshape(K, s).T
    ring.tft(A, L, 0, s, n, threads=8)
    ring.tft(B, L, 0, s, n, threads=8)
    with ThreadPoolExecutor(8) as ex:
        prods = list(ex.map(lambda i: ring.mul(A[i], B[i]), range(n)))
    for i in range(n):
        A[i] = prods[i]
    ring.itft(A, L, 0, n, n, 0, threads=8)
    inv = pow(L, -1, m)
    Cz = [[(int(v) * inv) % m for v in A[i]] for i in range(n)]
    want = np.zeros(K * s, dtype=np.uint64)
    for j in range(s):
        blk = Cz[j]
        if j + s < n:
            c2 = Cz[j + s]
            yc = [(m - c2[K - 1]) % m] + c2[: K - 1]
            blk = [(x + y) % m for x, y in zip(blk, yc)]
        want[j::s] = blk
    assert np.array_equal(got, want)


def _gmp():
    import ctypes.util
    name = ctypes.util.find_library("gmp") or "libgmp.so.10"
    g = C.CDLL(name)
    g.__gmpn_mul.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_void_p, C.c_long]
    g.__gmpn_mul.restype = C.c_uint64
    return g


def _kronecker_product(F, G, slot_limbs):
    """Z[x] product by Kronecker substitution and GMP's mpn_mul (an independent
    check of the config-4 pipeline): coefficients < 2^(64 slot_limbs) never
    overlap, so the product integer's slots are the product coefficients."""
    zf, zg = F.shape[0], G.shape[0]
    a = np.zeros((zf, slot_limbs), dtype=np.uint64)
    b = np.zeros((zg, slot_limbs), dtype=np.uint64)
    a[:, : F.shape[1]] = F
    b[:, : G.shape[1]] = G
    if zf < zg:
        a, b, zf, zg = b, a, zg, zf
    out = np.zeros((zf + zg) * slot_limbs, dtype=np.uint64)
    _gmp().__gmpn_mul(out.ctypes.data, a.ctypes.data, zf * slot_limbs, b.ctypes.data, zg * slot_limbs)
    return out.reshape(zf + zg, slot_limbs)[: zf + zg - 1]


def _limbs(rng, count, bits):
    limbs = (bits + 63) // 64
    x = rng.integers(0, 1 << 64, size=(count, limbs), dtype=np.uint64, endpoint=False)
    if bits % 64:
        x[:, -1] &= np.uint64((1 << (bits % 64)) - 1)
    return x


def test_ss_medium_matches_gmp():
    rng = np.random.default_rng(11)
    for zf, zg, bits in [(3000, 2500, 500), (4096, 4096, 1000), (1, 5000, 1000)]:
        F, G = _limbs(rng, zf, bits), _limbs(rng, zg, bits)
        H, N = pm.ss_mul(to_dev(F), to_dev(G), bits)
        want = _kronecker_product(F, G, N // 64)
        assert np.array_equal(from_dev(H), want), (zf, zg, bits)


@pytest.mark.slow
def test_config4_full_size_matches_gmp():
    """BASELINE config 4: two length-60000 polynomials with 1000-bit
    coefficients, R = Z/(2^65536+1), L = 2^17: the product in Z[x], bit-exact."""
    rng = np.random.default_rng(po.mix_seed(42, 4))
    F, G = _limbs(rng, 60000, 1000), _limbs(rng, 60000, 1000)
    st = pm.MulStats()
    H, N = pm.ss_mul(to_dev(F), to_dev(G), 1000, stats=st)
    assert N == 65536 and st.transform_length == 1 << 17 and st.pointwise_mults == 119999
    want = _kronecker_product(F, G, N // 64)
    assert np.array_equal(from_dev(H), want)
