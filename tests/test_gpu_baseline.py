"""BASELINE configurations at full size on the GPU, bit-exact against the CPU
oracle (SURVEY.md §8d inputs: seeded uniform limbs from mix_seed(42, config)).

C2: the 16 (z, n) TFT pairs and the 10 z >= n ITFT pairs with f in {0, 1}
(ITFT inputs built as verify.hpp:140-151 does: transformed values from a TFT
with n' = n + 1, then L*a for the coefficients in [n, z)).  C5: the full
transform and its round trip.  Base-case counts are pinned to the reference
recursion's."""
from __future__ import annotations

import numpy as np
import pytest

import pyoracle as po
from helpers import from_dev, to_dev

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_0810_3203_b200 as cf  # noqa: E402

C2_SIZES = (32769, 40000, 49152, 65535)
C2_COUNTS = {32769: 311295, 40000: 352384, 49152: 409600, 65535: 524288}
THREADS = 16


def _limbs(N, L, z, W, seed):
    rng = np.random.default_rng(seed)
    buf = np.zeros((L, W), dtype=np.uint64)
    lim = N // 64
    for i in range(0, z, 8192):
        k = min(8192, z - i)
        buf[i:i + k, :lim] = rng.integers(0, 1 << 64, size=(k, lim), dtype=np.uint64, endpoint=False)
    return buf


@pytest.fixture(scope="module")
def c2():
    N, L = 32768, 1 << 16
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    a = _limbs(N, L, L, ctx.element_words, po.mix_seed(42, 2))
    return N, L, ctx, ring, a


def test_c2_tft_sweep(c2):
    N, L, ctx, ring, a = c2
    lim = N // 64
    for z in C2_SIZES:
        for n in C2_SIZES:
            buf = a.copy()
            buf[z:] = 0
            want = buf.copy()
            ring.tft(want, L, 0, z, n, threads=THREADS)
            dev = to_dev(buf)
            st = cf.ButterflyStats()
            cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), cf.DeviceView(dev), stats=st)
            got = from_dev(dev)
            assert np.array_equal(got[:n, : lim + 1], want[:n, : lim + 1]), (z, n)
            assert st.base_case_count == cf.tft_base_cases(L, z, n)
            if z == n:
                assert st.base_case_count == C2_COUNTS[z]
            del dev


def test_c2_itft_sweep(c2):
    N, L, ctx, ring, a = c2
    lim = N // 64
    for z in C2_SIZES:
        coeffs = a.copy()
        coeffs[z:] = 0
        for n in C2_SIZES:
            if n > z:
                continue
            for f in (0, 1):
                spec = coeffs.copy()
                ring.tft(spec, L, 0, z, min(L, n + 1), threads=THREADS)  # x_0 .. x_n
                inp = coeffs.copy()
                inp[:n] = spec[:n]
                for i in range(n, z):  # L * a_i
                    inp[i, : lim + 1] = ring.twiddle(L.bit_length() - 1, coeffs[i, : lim + 1])
                want = inp.copy()
                ring.itft(want, L, 0, z, n, f, threads=THREADS)
                dev = to_dev(inp)
                st = cf.ButterflyStats()
                cf.cf_itft(ctx, cf.TransformParams(L, 0, z, n, f), cf.DeviceView(dev), stats=st)
                got = from_dev(dev)
                assert np.array_equal(got[: n + f, : lim + 1], want[: n + f, : lim + 1]), (z, n, f)
                assert st.base_case_count == cf.itft_base_cases(L, z, n, f)
                # and the definition: L * a on [0, n), the next transformed value at n
                for i in range(0, n, 4099):
                    assert np.array_equal(got[i, : lim + 1], inp[i, : lim + 1] if i >= n else
                                          ring.twiddle(L.bit_length() - 1, coeffs[i, : lim + 1]))
                if f:
                    assert np.array_equal(got[n, : lim + 1], spec[n, : lim + 1])
                del dev


@pytest.mark.parametrize("wide", [0, 1])
def test_c5_full_transform_and_round_trip(wide):
    """C5: Z/(2^131072+1), L = 2^18, z = n = 200000: GPU TFT bit-exact vs the
    oracle, GPU ITFT of it = L * a, base-case counts as pinned (radix-8 warp
    engine and radix-64 CTA engine)."""
    N, L, z = 131072, 1 << 18, 200000
    ctx = cf.FermatRingCtx(N)
    ctx.set_wide(wide)
    ring = po.Ring.fermat(N)
    lim = N // 64
    a = _limbs(N, L, z, ctx.element_words, po.mix_seed(42, 5))
    want = a.copy()
    ring.tft(want, L, 0, z, z, threads=THREADS)
    dev = to_dev(a)
    st = cf.ButterflyStats()
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), cf.DeviceView(dev), stats=st)
    assert st.base_case_count == 1918080
    got = from_dev(dev)
    assert np.array_equal(got[:z, : lim + 1], want[:z, : lim + 1])
    del got, want
    st = cf.ButterflyStats()
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), cf.DeviceView(dev), stats=st)
    assert st.base_case_count == 1918080
    cf.scale(ctx, cf.DeviceView(dev), z, 2 * N - 18)  # 1/L
    back = from_dev(dev)
    assert np.array_equal(back[:z, : lim + 1], a[:z, : lim + 1])


@pytest.mark.parametrize("s_exp", [1, 12345, 65537])
def test_c2_nonzero_zeta(c2, s_exp):
    """zeta = omega^s with s != 0 (sub-lane, whole-lane and past-2^N weights)
    at a C2 size: the TFT (z = 40000, n = 49152) and the ITFT (z = 49152,
    n = 40000, f = 1) against the oracle (transform.hpp:252-286 with s)."""
    N, L, ctx, ring, a = c2
    lim = N // 64
    z, n = 40000, 49152
    buf = a.copy()
    buf[z:] = 0
    want = buf.copy()
    ring.tft(want, L, s_exp, z, n, threads=THREADS)
    dev = to_dev(buf)
    cf.cf_tft(ctx, cf.TransformParams(L, s_exp, z, n), cf.DeviceView(dev))
    assert np.array_equal(from_dev(dev)[:n, : lim + 1], want[:n, : lim + 1])
    zi, ni = 49152, 40000
    buf = a.copy()
    buf[zi:] = 0
    want = buf.copy()
    ring.itft(want, L, s_exp, zi, ni, 1, threads=THREADS)
    dev = to_dev(buf)
    cf.cf_itft(ctx, cf.TransformParams(L, s_exp, zi, ni, 1), cf.DeviceView(dev))
    got = from_dev(dev)
    assert np.array_equal(got[: ni + 1, : lim + 1], want[: ni + 1, : lim + 1])


def test_c5_nonzero_zeta_round_trip():
    """C5 with zeta = omega^77777 (an odd, sub-lane weight): the TFT against
    the oracle, then ITFT(TFT(a)) = L a."""
    N, L, z = 131072, 1 << 18, 200000
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    lim = N // 64
    s_exp = 77777
    a = _limbs(N, L, z, ctx.element_words, po.mix_seed(42, 55))
    want = a.copy()
    ring.tft(want, L, s_exp, z, z, threads=THREADS)
    dev = to_dev(a)
    cf.cf_tft(ctx, cf.TransformParams(L, s_exp, z, z), cf.DeviceView(dev))
    got = from_dev(dev)
    assert np.array_equal(got[:z, : lim + 1], want[:z, : lim + 1])
    del got, want
    cf.cf_itft(ctx, cf.TransformParams(L, s_exp, z, z, 0), cf.DeviceView(dev))
    cf.scale(ctx, cf.DeviceView(dev), z, 2 * N - 18)
    assert np.array_equal(from_dev(dev)[:z, : lim + 1], a[:z, : lim + 1])
