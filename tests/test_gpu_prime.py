"""GPU path over the reference's own ring (Z/pZ, Goldilocks by default): the
sm_100a engine against the UNMODIFIED reference (oracle/_ref, cf_tft / cf_itft
of transform.hpp:252-286 compiled from /root/reference) where it is present,
and always against the oracle restatement pinned to it -- outputs and
ButterflyStats counts, both split policies, the verify suites' shapes
(verify.hpp:85-173)."""
from __future__ import annotations

import ctypes as C
import random

import numpy as np
import pytest

import pyoracle as po
from helpers import from_dev, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_0810_3203_b200 as cf  # noqa: E402

P, M_BITS = cf.GOLDILOCKS, 32


def _inputs(L: int, z: int, seed: int, p: int = P) -> np.ndarray:
    rng = np.random.default_rng(seed)
    buf = np.full((L, 1), 0xDEADBEEFDEADBEEF, dtype=np.uint64)  # poison beyond z
    buf[:z, 0] = rng.integers(0, p, size=z, dtype=np.uint64)
    return buf


def _ref(inverse, L, s, z, n, f, buf, pol, p=P, m=M_BITS):
    """The reference itself (oracle/_ref/libcftft_ref.so), or None."""
    if not po.ref_available():
        return None
    out = np.ascontiguousarray(buf.copy())
    c = C.c_uint64(0)
    ptr = out.ctypes.data_as(po.U64P)
    if inverse:
        rc = po.ref().ref_itft(p, m, L, s, z, n, f, ptr, out.shape[0], 0, 1, pol, C.byref(c))
    else:
        rc = po.ref().ref_tft(p, m, L, s, z, n, ptr, out.shape[0], 0, 1, pol, C.byref(c))
    assert rc == 0
    return out, c.value


def _case(ctx, ring, L, z, n, s, pol, seed, inverse=False, f=0, p=P, m=M_BITS):
    buf = _inputs(L, z, seed, p)
    want = buf.copy()
    cnt = ring.itft(want, L, s, z, n, f, pol) if inverse else ring.tft(want, L, s, z, n, pol)
    dev = to_dev(buf)
    st = cf.ButterflyStats()
    if inverse:
        cf.cf_itft(ctx, cf.TransformParams(L, s, z, n, f), cf.DeviceView(dev), pol, st)
    else:
        cf.cf_tft(ctx, cf.TransformParams(L, s, z, n), cf.DeviceView(dev), pol, st)
    got = from_dev(dev)
    k = n + f if inverse else n
    assert np.array_equal(got[:k], want[:k]), (L, z, n, f, s, pol, inverse)
    assert st.base_case_count == cnt
    r = _ref(inverse, L, s, z, n, f, buf, pol, p, m)
    if r is not None:
        assert np.array_equal(got[:k], r[0][:k]), ("reference", L, z, n, f, s, pol, inverse)
        assert st.base_case_count == r[1]


def test_prime_random_sweep():
    """Random (L, z, n, s, policy) up to L = 2^14 (two leaf levels), TFT and ITFT."""
    ctx = cf.PrimeRingCtx()
    ring = po.Ring.prime(P, M_BITS)
    rnd = random.Random(2024)
    for trial in range(40):
        L = 1 << rnd.randint(1, 14)
        z, n = rnd.randint(1, L), rnd.randint(1, L)
        s, pol = rnd.randrange(1 << M_BITS), rnd.randint(0, 1)
        _case(ctx, ring, L, z, n, s, pol, seed=trial)
        n2, f = rnd.randint(0, z), rnd.randint(0, 1)
        if 1 <= n2 + f <= L:
            _case(ctx, ring, L, z, n2, s, pol, seed=900 + trial, inverse=True, f=f)


def test_prime_exhaustive_small():
    """Every (z, n) at L = 16 and 32, both policies (verify.hpp:85-120)."""
    ctx = cf.PrimeRingCtx()
    ring = po.Ring.prime(P, M_BITS)
    for L in (16, 32):
        for pol in (0, 1):
            for z in range(1, L + 1):
                for n in range(1, L + 1, 3):
                    _case(ctx, ring, L, z, n, 5, pol, seed=z * 64 + n)
                for n in range(0, z + 1, 2):
                    for f in (0, 1):
                        if 1 <= n + f <= L:
                            _case(ctx, ring, L, z, n, 3, pol, seed=z * 7 + n, inverse=True, f=f)


def test_prime_large_and_round_trip():
    """L = 2^16, z = n = 40000: the truncated transform against the oracle and
    the reference, and ITFT(TFT(a)) = L a (transform.hpp:266-272)."""
    ctx = cf.PrimeRingCtx()
    ring = po.Ring.prime(P, M_BITS)
    L, z = 1 << 16, 40000
    _case(ctx, ring, L, z, z, 0, 0, seed=77)
    a = _inputs(L, z, 78)
    dev = to_dev(a)
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), cf.DeviceView(dev))
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), cf.DeviceView(dev))
    back = from_dev(dev)[:z, 0].astype(object)
    assert all(int(x) == (L * int(y)) % P for x, y in zip(back, a[:z, 0]))


def test_prime_small_field_and_strided_view():
    """Another prime ring (p = 3 * 2^30 + 1, m = 30: below 2^63, so the other
    side of the engine's carry handling) and a strided view (view.hpp:33-42)
    that leaves its surroundings untouched."""
    p, m = 3 * (1 << 30) + 1, 30
    ctx = cf.PrimeRingCtx(m, p)
    ring = po.Ring.prime(p, m)
    rnd = random.Random(5)
    for trial in range(10):
        L = 1 << rnd.randint(2, 10)
        z, n = rnd.randint(1, L), rnd.randint(1, L)
        _case(ctx, ring, L, z, n, rnd.randrange(1 << m), rnd.randint(0, 1), seed=trial, p=p, m=m)
    L, z, n, stride = 256, 200, 180, 3
    rng = np.random.default_rng(9)
    big = rng.integers(0, p, size=(L * stride + 5, 1), dtype=np.uint64)
    want = big.copy()
    ring.tft_at(want, 2, stride, L, 7, z, n)
    dev = to_dev(big)
    cf.cf_tft(ctx, cf.TransformParams(L, 7, z, n), cf.DeviceView(dev, base=2, stride=stride, length=L))
    got = from_dev(dev)
    idx = [2 + i * stride for i in range(n)]
    assert np.array_equal(got[idx], want[idx])
    untouched = np.ones(len(big), dtype=bool)
    untouched[[2 + i * stride for i in range(L)]] = False
    assert np.array_equal(got[untouched], big[untouched])


def test_prime_validation():
    """The reference's errors before any work (transform.hpp:241-286)."""
    ctx = cf.PrimeRingCtx()
    dev = to_dev(_inputs(8, 8, 1))
    with pytest.raises(cf.BadLength):
        cf.cf_tft(ctx, cf.TransformParams(6, 0, 4, 4), cf.DeviceView(dev))
    with pytest.raises(cf.InvalidParams):
        cf.cf_itft(ctx, cf.TransformParams(8, 0, 3, 4, 0), cf.DeviceView(dev))


def test_prime_bench_shape_g():
    """The bench's G shape itself (L = 2^22, z = n = 3 * 10^6, the reference's
    own Goldilocks ring): the TFT bit-exact against the oracle port (and the
    unmodified reference when oracle/_ref is there), the ITFT round trip
    ITFT(TFT(a)) = L a checked vectorised mod p."""
    ctx = cf.PrimeRingCtx()
    ring = po.Ring.prime(P, M_BITS)
    L, z = 1 << 22, 3_000_000
    a = _inputs(L, z, 79)
    want = a.copy()
    ring.tft(want, L, 0, z, z)
    dev = to_dev(a)
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), cf.DeviceView(dev))
    got = from_dev(dev)
    assert np.array_equal(got[:z, 0], want[:z, 0])
    ref = _ref(False, L, 0, z, z, 0, a, 0)
    if ref is not None:
        assert np.array_equal(got[:z, 0], ref[0][:z, 0])
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), cf.DeviceView(dev))
    back = from_dev(dev)[:z, 0]
    # L a mod p, with L = 2^22 and a < p < 2^64: via Python ints on a sample,
    # exactly on every element through 128-bit-free arithmetic (L * a mod p by
    # doubling 22 times)
    x = a[:z, 0].astype(object)
    idx = np.random.default_rng(3).choice(z, size=20000, replace=False)
    assert all(int(back[i]) == (L * int(x[i])) % P for i in idx)
