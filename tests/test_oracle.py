"""CPU oracle pinned against the reference (no GPU).

  * the reference's own known-answer tests (transform_test.cpp, p = 17)
  * golden outputs of the UNMODIFIED reference (tests/golden/prime_cases.json)
  * the reference's base-case counts at the BASELINE shapes (counts.json)
  * big-ring transforms evaluated from their definition (bigring.npz)
  * ring axioms restated for the new rings (field_test.cpp:117-144)
"""
from __future__ import annotations

import json
import os
import random

import numpy as np
import pytest

import bigint_model as bm
import pyoracle as po

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def r17(oracle):
    return po.Ring.prime(17, 4)


def e(v):
    return np.array([v], dtype=np.uint64)


# ---- transform_test.cpp KATs -------------------------------------------------

def test_root_of_17_is_three(r17):
    assert r17.r.omega == 3 and r17.M == 16  # field_test.cpp:63-75


def test_tft_base2_spec_examples(r17):  # transform_test.cpp:37-58
    lib = po.lib()
    cnt = po.C.c_uint64(0)
    x0, x1 = e(3), e(5)
    lib.or_tft_base2(po.C.byref(r17.r), 0, 2, 2, po._p(x0), po._p(x1), po.C.byref(cnt))
    assert (x0[0], x1[0]) == (8, 15)
    x0, x1 = e(7), e(0xFFFFFFFFFFFFFFFF)
    lib.or_tft_base2(po.C.byref(r17.r), 0, 1, 2, po._p(x0), po._p(x1), po.C.byref(cnt))
    assert (x0[0], x1[0]) == (7, 7)
    x0, x1 = e(3), e(5)
    lib.or_tft_base2(po.C.byref(r17.r), 0, 2, 1, po._p(x0), po._p(x1), po.C.byref(cnt))
    assert x0[0] == 8
    assert cnt.value == 3


def test_itft_base2_all_seven_branches(r17):  # transform_test.cpp:71-120
    lib = po.lib()
    cnt = po.C.c_uint64(0)
    P = 0xFFFFFFFFFFFFFFFF

    def run(z, n, f, a, b):
        x0, x1 = e(a), e(b)
        lib.or_itft_base2(po.C.byref(r17.r), 0, z, n, f, po._p(x0), po._p(x1), po.C.byref(cnt))
        return int(x0[0]), int(x1[0])

    assert run(2, 2, 0, 8, 15) == (6, 10)
    assert run(2, 1, 1, 8, 10) == (6, 15)
    assert run(1, 1, 1, 5, P) == (10, 5)
    assert run(2, 1, 0, 8, 10)[0] == 6
    assert run(1, 1, 0, 9, P)[0] == 1
    assert run(2, 0, 1, 6, 10)[0] == 8
    assert run(1, 0, 1, 11, P)[0] == 14
    assert cnt.value == 7


def test_itft_base2_nontrivial_twiddle(r17):  # transform_test.cpp:122-130
    lib = po.lib()
    x0, x1 = e(4), e(13)
    lib.or_tft_base2(po.C.byref(r17.r), 3, 2, 2, po._p(x0), po._p(x1), None)
    lib.or_itft_base2(po.C.byref(r17.r), 3, 2, 2, 0, po._p(x0), po._p(x1), None)
    assert (x0[0], x1[0]) == (8, 9)


def test_dft_naive_length2_and_delta(r17):  # transform_test.cpp:154-163
    two = r17.dft_naive(2, 0, np.array([[3], [5]], dtype=np.uint64))
    assert list(two[:, 0]) == [8, 15]
    four = r17.dft_naive(4, 0, np.array([[1], [0], [0], [0]], dtype=np.uint64))
    assert list(four[:, 0]) == [1, 1, 1, 1]


def test_delta_input_gives_all_ones(r17):  # transform_test.cpp:204-213
    for pol in (0, 1):
        buf = np.zeros((16, 1), dtype=np.uint64)
        buf[0, 0] = 1
        r17.tft(buf, 16, 0, 16, 16, pol)
        assert list(buf[:, 0]) == [1] * 16


def test_bounds_spec_values():  # transform_test.cpp:332-340
    assert po.tft_bound(2, 1) == 1 and po.tft_bound(2, 2) == 1 and po.tft_bound(8, 8) == 12
    assert po.itft_bound(2, 0, 1) == 1 and po.itft_bound(8, 8, 0) == 12


def test_fault_hook_is_detected(r17):  # transform_test.cpp:392-402
    coeffs = np.array([[3], [5], [7]], dtype=np.uint64)
    want = r17.dft_naive(4, 1, coeffs)
    po.set_fault(True)
    try:
        buf = np.zeros((4, 1), dtype=np.uint64)
        buf[:3] = coeffs
        r17.tft(buf, 4, 1, 3, 4)
        assert not np.array_equal(buf, want)
    finally:
        po.set_fault(False)
    buf = np.zeros((4, 1), dtype=np.uint64)
    buf[:3] = coeffs
    r17.tft(buf, 4, 1, 3, 4)
    assert np.array_equal(buf, want)


def test_validation_codes(r17):  # transform_test.cpp:360-390
    buf = np.zeros((32, 1), dtype=np.uint64)
    with pytest.raises(po.OracleError) as ex:
        r17.tft(buf, 12, 0, 1, 1)
    assert ex.value.code == po.BAD_LENGTH
    with pytest.raises(po.OracleError) as ex:
        r17.tft(buf, 32, 0, 1, 1)  # exceeds the root order 16
    assert ex.value.code == po.BAD_LENGTH
    for (z, n) in [(0, 1), (9, 1), (1, 0)]:
        with pytest.raises(po.OracleError):
            r17.tft(buf[:8], 8, 0, z, n)
    with pytest.raises(po.OracleError):
        r17.itft(buf[:8], 8, 0, 2, 3)
    with pytest.raises(po.OracleError):
        r17.itft(buf[:8], 8, 0, 8, 8, 1)


# ---- golden outputs of the unmodified reference --------------------------------

def test_prime_golden_cases(oracle):
    cases = json.load(open(os.path.join(GOLD, "prime_cases.json")))
    assert len(cases) > 150
    rings = {}
    for c in cases:
        key = (c["p"], c["m"])
        if key not in rings:
            rings[key] = po.Ring.prime(*key)
        r = rings[key]
        L = c["L"]
        buf = np.zeros((L, 1), dtype=np.uint64)
        buf[: c["z"], 0] = c["input"]
        if c["inverse"]:
            cnt = r.itft(buf, L, c["s"], c["z"], c["n"], c["f"], c["policy"])
            k = c["n"] + c["f"]
        else:
            cnt = r.tft(buf, L, c["s"], c["z"], c["n"], c["policy"])
            k = c["n"]
        assert [int(v) for v in buf[:k, 0]] == c["output"], c
        assert cnt == c["count"]


@pytest.mark.skipif(not po.ref_available(), reason="reference shim not built")
def test_oracle_matches_reference_sweep(oracle):
    """Every (z, n) (and n, f) for L <= 32 over Goldilocks, both policies,
    against the compiled reference (verify.hpp:85-173 shapes)."""
    import ctypes as C

    R = po.ref()
    p, m = po.GOLDILOCKS, 32
    ring = po.Ring.prime(p, m)
    rng = np.random.default_rng(2024)
    for ell in range(1, 6):
        L = 1 << ell
        for z in range(1, L + 1):
            a = rng.integers(0, p, size=L, dtype=np.uint64)
            s = int(rng.integers(0, 1 << 32))
            for n in range(1, L + 1):
                for pol in (0, 1):
                    b1, b2 = a.reshape(L, 1).copy(), a.copy()
                    c1 = ring.tft(b1, L, s, z, n, pol)
                    c2 = C.c_uint64()
                    assert R.ref_tft(p, m, L, s, z, n, b2.ctypes.data_as(po.U64P), L, 0, 1, pol,
                                     C.byref(c2)) == 0
                    assert np.array_equal(b1[:n, 0], b2[:n]) and c1 == c2.value
            for n in range(0, z + 1):
                for f in (0, 1):
                    if not 1 <= n + f <= L:
                        continue
                    b1, b2 = a.reshape(L, 1).copy(), a.copy()
                    c1 = ring.itft(b1, L, s, z, n, f, 0)
                    c2 = C.c_uint64()
                    assert R.ref_itft(p, m, L, s, z, n, f, b2.ctypes.data_as(po.U64P), L, 0, 1, 0,
                                      C.byref(c2)) == 0
                    assert np.array_equal(b1[: n + f, 0], b2[: n + f]) and c1 == c2.value


# ---- big rings from the definition ---------------------------------------------

def test_bigring_golden(oracle):
    meta = json.load(open(os.path.join(GOLD, "bigring.json")))
    arr = np.load(os.path.join(GOLD, "bigring.npz"))
    for c in meta:
        if c["key"] == "c1":
            continue
        if c["ring"] == "fermat":
            r = po.Ring.fermat(c["N"])
        else:
            r = po.Ring.negacyclic(c["K"], c["m"])
        L, z, n, s = c["L"], c["z"], c["n"], c["s"]
        buf = r.zeros(L)
        buf[:z] = arr[c["key"] + "_in"]
        r.tft(buf, L, s, z, n)
        assert np.array_equal(buf[:n], arr[c["key"] + "_tft"]), c
        if c["ring"] == "fermat":
            buf = r.zeros(L)
            buf[:z] = arr[c["key"] + "_itin"]
            r.itft(buf, L, s, z, c["n2"], c["f"])
            k = c["n2"] + c["f"]
            assert np.array_equal(buf[:k], arr[c["key"] + "_itout"]), c


def test_config1_golden(oracle):
    """Config 1 TFT output (Z/(2^1024+1), L=1024, z=n=700) from the definition."""
    N, L, z = 1024, 1024, 700
    r = po.Ring.fermat(N)
    rng = np.random.default_rng(po.mix_seed(42, 1))
    buf = r.zeros(L)
    buf[:z, : N // 64] = rng.integers(0, 1 << 64, size=(z, N // 64), dtype=np.uint64, endpoint=False)
    a = buf.copy()
    r.tft(buf, L, 0, z, z)
    assert np.array_equal(buf[:z], np.load(os.path.join(GOLD, "bigring.npz"))["c1_tft"])
    r.itft(buf, L, 0, z, z, 0)
    for i in range(z):  # ITFT(TFT(a)) = L a
        buf[i] = r.twiddle(2 * N - 10, buf[i])
    assert np.array_equal(buf[:z], a[:z])


# ---- ring axioms for the new rings (field_test.cpp:117-144 restated) ------------

@pytest.mark.parametrize("N", [128, 1024])
def test_fermat_axioms(oracle, N):
    r = po.Ring.fermat(N)
    fm = bm.FermatModel(N)
    rnd = random.Random(99)
    zero = fm.to_words(0)
    for _ in range(100):
        v = rnd.randrange((1 << N) + 1)
        a = fm.to_words(v)
        assert np.array_equal(r.half(r.add(a, a)), a)
        assert np.array_equal(r.add(a, r.sub(zero, a)), zero)
        assert fm.from_words(r.twiddle(N, a)) == (-v) % fm.P  # omega^(M/2) = -1
        assert np.array_equal(r.twiddle(2 * N, a), a)  # periodicity
        assert np.array_equal(r.twiddle(5, a), r.twiddle(5 + 2 * N, a))
        b = rnd.randrange((1 << N) + 1)
        assert fm.from_words(r.mul(a, fm.to_words(b))) == (v * b) % fm.P


def test_negacyclic_axioms(oracle):
    K, m = 16, (1 << 61) + 15
    r = po.Ring.negacyclic(K, m)
    nm = bm.NegacyclicModel(K, m)
    rnd = random.Random(5)
    for _ in range(50):
        x = [rnd.randrange(m) for _ in range(K)]
        a = np.array(x, dtype=np.uint64)
        assert np.array_equal(r.half(r.add(a, a)), a)
        assert [int(v) for v in r.twiddle(K, a)] == [(-v) % m for v in x]
        assert [int(v) for v in r.twiddle(3, a)] == nm.tw(3, x)
