"""Fault injection and debug poison on the GPU.

* fault::corrupt_tft_base (transform.hpp:53-56, 109; transform_test.cpp:392-402):
  with the library's fault flag set, the C2 parity check against the oracle
  and the C5 round trip must FAIL, and pass again once the flag is reset.
* poison_tail (transform.hpp:58-70): with the debug poison mode on, every
  transform runs twice with different non-canonical fills of the cells >= z;
  the BASELINE shapes (C2 sweep points, C5, the negacyclic and prime rings)
  must come through without a PoisonRead and with the oracle's outputs.
"""
from __future__ import annotations

import numpy as np
import pytest

import pyoracle as po
from helpers import fermat_inputs, from_dev, negacyclic_inputs, random_modulus, to_dev

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_0810_3203_b200 as cf  # noqa: E402

THREADS = 16


@pytest.fixture
def fault():
    cf.set_fault_injection(True)
    yield
    cf.set_fault_injection(False)


@pytest.fixture
def poison():
    cf.set_debug_poison(True)
    yield
    cf.set_debug_poison(False)


def _c2_tft(z, n):
    N, L = 32768, 1 << 16
    ctx = cf.FermatRingCtx(N)
    lim = N // 64
    a = fermat_inputs(N, L, z, ctx.element_words, po.mix_seed(42, 2))
    want = a.copy()
    po.Ring.fermat(N).tft(want, L, 0, z, n, threads=THREADS)
    dev = to_dev(a)
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), cf.DeviceView(dev))
    got = from_dev(dev)
    return np.array_equal(got[:n, : lim + 1], want[:n, : lim + 1])


def test_fault_flag_breaks_c2_parity(fault):
    assert cf.fault_injection()
    assert not _c2_tft(40000, 40000), "the C2 parity check must fail under fault injection"
    cf.set_fault_injection(False)
    assert _c2_tft(40000, 40000), "and pass again once the hook is reset"


def test_fault_flag_breaks_c5_round_trip(fault):
    N, L, z = 131072, 1 << 18, 200000
    ctx = cf.FermatRingCtx(N)
    lim = N // 64
    rng = np.random.default_rng(po.mix_seed(42, 5))
    a = np.zeros((L, ctx.element_words), dtype=np.uint64)
    a[:z, :lim] = rng.integers(0, 1 << 64, size=(z, lim), dtype=np.uint64, endpoint=False)

    def round_trip():
        dev = to_dev(a)
        cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), cf.DeviceView(dev))
        cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), cf.DeviceView(dev))
        cf.scale(ctx, cf.DeviceView(dev), z, 2 * N - 18)  # 1/L
        back = from_dev(dev)
        return np.array_equal(back[:z, : lim + 1], a[:z, : lim + 1])

    assert not round_trip(), "the C5 round trip must fail under fault injection"
    cf.set_fault_injection(False)
    assert round_trip()


def test_fault_flag_is_ring_addition():
    """x[0] + 1 in the ring: Z/(2^N+1) wraps 2^N to 0; Z/pZ wraps p - 1."""
    cf.set_fault_injection(True)
    try:
        N, L = 1024, 4
        ctx = cf.FermatRingCtx(N)
        buf = np.zeros((L, ctx.element_words), dtype=np.uint64)
        buf[0, N // 64] = 1  # x0 = 2^N; TFT with z = n = 1 is the identity on x0
        dev = to_dev(buf)
        cf.cf_tft(ctx, cf.TransformParams(L, 0, 1, 1), cf.DeviceView(dev))
        assert not from_dev(dev)[0, : N // 64 + 1].any()
        pctx = cf.PrimeRingCtx()
        pb = np.zeros((L, 1), dtype=np.uint64)
        pb[0, 0] = cf.GOLDILOCKS - 1
        dev = to_dev(pb)
        cf.cf_tft(pctx, cf.TransformParams(L, 0, 1, 1), cf.DeviceView(dev))
        assert int(from_dev(dev)[0, 0]) == 0
    finally:
        cf.set_fault_injection(False)


@pytest.mark.parametrize("z,n", [(32769, 65535), (65535, 40000), (49152, 49152)])
def test_debug_poison_c2(poison, z, n):
    """C2 TFT and ITFT (f = 1) under the two-fill poison check, vs the oracle."""
    assert _c2_tft(z, n)
    N, L = 32768, 1 << 16
    ctx = cf.FermatRingCtx(N)
    lim = N // 64
    zi, ni = max(z, n), min(z, n)
    a = fermat_inputs(N, L, zi, ctx.element_words, po.mix_seed(42, 22))
    dev = to_dev(a)
    cf.cf_itft(ctx, cf.TransformParams(L, 0, zi, ni, 1), cf.DeviceView(dev))
    want = a.copy()
    po.Ring.fermat(N).itft(want, L, 0, zi, ni, 1, threads=THREADS)
    got = from_dev(dev)
    assert np.array_equal(got[: ni + 1, : lim + 1], want[: ni + 1, : lim + 1])


def test_debug_poison_c5(poison):
    N, L, z = 131072, 1 << 18, 200000
    ctx = cf.FermatRingCtx(N)
    a = fermat_inputs(N, L, z, ctx.element_words, po.mix_seed(42, 5))
    dev = to_dev(a)
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), cf.DeviceView(dev))
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), cf.DeviceView(dev))


def test_debug_poison_other_rings(poison):
    K = 1024
    m = random_modulus(po.mix_seed(42, 3))
    nctx = cf.NegacyclicRingCtx(K, m)
    L, z, n = 1 << 11, 1024, 2047
    buf = negacyclic_inputs(K, m, L, z, nctx.element_words, 7)
    want = buf.copy()
    po.Ring.negacyclic(K, m).tft(want, L, 0, z, n, threads=THREADS)
    dev = to_dev(buf)
    cf.cf_tft(nctx, cf.TransformParams(L, 0, z, n), cf.DeviceView(dev))
    assert np.array_equal(from_dev(dev)[:n, :K], want[:n, :K])
    pctx = cf.PrimeRingCtx()
    L, z, n = 1 << 16, 40000, 50000
    rng = np.random.default_rng(11)
    pb = np.full((L, 1), 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    pb[:z, 0] = rng.integers(0, cf.GOLDILOCKS, size=z, dtype=np.uint64)
    want = pb.copy()
    po.Ring.prime(cf.GOLDILOCKS, 32).tft(want, L, 0, z, n)
    dev = to_dev(pb)
    cf.cf_tft(pctx, cf.TransformParams(L, 0, z, n), cf.DeviceView(dev))
    assert np.array_equal(from_dev(dev)[:n, 0], want[:n, 0])
