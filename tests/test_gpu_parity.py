"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle,
bit for bit, on seeded inputs.  Patterned on the reference's own suites
(verify.hpp:85-173 oracle/inversion sweeps, transform_test.cpp:228-330)."""
from __future__ import annotations

import random

import numpy as np
import pytest

import pyoracle as po
from helpers import fermat_inputs, from_dev, negacyclic_inputs, random_modulus, to_dev

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_0810_3203_b200 as cf  # noqa: E402


def _fermat_case(ctx, ring, N, L, z, n, s, pol, seed, inverse=False, f=0, special=False):
    W = ctx.element_words
    lim = N // 64
    buf = fermat_inputs(N, L, z, W, seed, special=special)
    want = buf.copy()
    if inverse:
        ring.itft(want, L, s, z, n, f, pol)
    else:
        ring.tft(want, L, s, z, n, pol)
    dev = to_dev(buf)
    view = cf.DeviceView(dev)
    st = cf.ButterflyStats()
    if inverse:
        cf.cf_itft(ctx, cf.TransformParams(L, s, z, n, f), view, pol, st)
    else:
        cf.cf_tft(ctx, cf.TransformParams(L, s, z, n), view, pol, st)
    got = from_dev(dev)
    k = n + f if inverse else n
    assert np.array_equal(got[:k, : lim + 1], want[:k, : lim + 1]), (N, L, z, n, f, s, pol, inverse)
    ref_count = ring.itft(buf.copy(), L, s, z, n, f, pol) if inverse else ring.tft(buf.copy(), L, s, z, n, pol)
    assert st.base_case_count == ref_count


@pytest.mark.parametrize("N", [128, 256, 1024])
@pytest.mark.parametrize("limit", [0, 1, 2, 3])
def test_fermat_random_sweep(N, limit):
    ctx = cf.FermatRingCtx(N)
    ctx.set_leaf_limit(limit)
    ring = po.Ring.fermat(N)
    rnd = random.Random(N * 10 + limit)
    for trial in range(30):
        L = 1 << rnd.randint(1, min(10, (2 * N).bit_length() - 1))
        z, n = rnd.randint(1, L), rnd.randint(1, L)
        s, pol = rnd.randrange(2 * N), rnd.randint(0, 1)
        _fermat_case(ctx, ring, N, L, z, n, s, pol, seed=trial, special=(trial % 3 == 0))
        n2, f = rnd.randint(0, z), rnd.randint(0, 1)
        if 1 <= n2 + f <= L:
            _fermat_case(ctx, ring, N, L, z, n2, s, pol, seed=1000 + trial, inverse=True, f=f,
                         special=(trial % 3 == 1))


def test_fermat_exhaustive_small():
    """Every (z, n) at L = 16, both policies (cf. verify.hpp:85-120)."""
    N, L = 128, 16
    ctx = cf.FermatRingCtx(N)
    ctx.set_leaf_limit(2)
    ring = po.Ring.fermat(N)
    for z in range(1, L + 1):
        for n in range(1, L + 1):
            for pol in (0, 1):
                _fermat_case(ctx, ring, N, L, z, n, 37, pol, seed=z * 100 + n)
        for n in range(0, z + 1):
            for f in (0, 1):
                if 1 <= n + f <= L:
                    _fermat_case(ctx, ring, N, L, z, n, 5, 0, seed=z * 7 + n, inverse=True, f=f)


def test_fermat_all_ones_and_minus_one():
    """Inputs made only of 2^N-1 and 2^N (== -1): maximal carry chains."""
    N, L = 1024, 64
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    W = ctx.element_words
    lim = N // 64
    buf = np.zeros((L, W), dtype=np.uint64)
    for i in range(L):
        if i % 2:
            buf[i, :lim] = np.uint64(0xFFFFFFFFFFFFFFFF)
        else:
            buf[i, lim] = 1
    for inverse in (False, True):
        want = buf.copy()
        dev = to_dev(buf)
        if inverse:
            ring.itft(want, L, 3, L, L, 0, 0)
            cf.cf_itft(ctx, cf.TransformParams(L, 3, L, L, 0), cf.DeviceView(dev))
        else:
            ring.tft(want, L, 3, L, L, 0)
            cf.cf_tft(ctx, cf.TransformParams(L, 3, L, L), cf.DeviceView(dev))
        got = from_dev(dev)
        assert np.array_equal(got[:, : lim + 1], want[:, : lim + 1])


def test_strided_view_leaves_surroundings_untouched():
    """transform_test.cpp:292-313 restated on the device."""
    N, L, stride, base = 256, 32, 3, 2
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    W = ctx.element_words
    lim = N // 64
    rows = base + (L - 1) * stride + 5
    rng = np.random.default_rng(8)
    full = np.zeros((rows, W), dtype=np.uint64)
    full[:, :lim] = rng.integers(0, 1 << 64, size=(rows, lim), dtype=np.uint64, endpoint=False)
    before = full.copy()
    dev = to_dev(full)
    view = cf.DeviceView(dev, base, stride, L)
    cf.cf_tft(ctx, cf.TransformParams(L, 5, 20, 27), view)
    after = from_dev(dev)
    idx = [base + i * stride for i in range(L)]
    mask = np.ones(rows, bool)
    mask[idx] = False
    assert np.array_equal(after[mask], before[mask])
    # and the view cells match the oracle on a compact copy
    want = before[idx].copy()
    ring.tft(want, L, 5, 20, 27, 0)
    assert np.array_equal(after[idx][:27, : lim + 1], want[:27, : lim + 1])


def test_validation_errors():
    """transform_test.cpp:360-390: errors are raised before any work."""
    ctx = cf.FermatRingCtx(128)  # M = 256
    dev = to_dev(np.zeros((8, ctx.element_words), dtype=np.uint64))
    v = cf.DeviceView(dev)
    with pytest.raises(cf.BadLength):
        cf.cf_tft(ctx, cf.TransformParams(12, 0, 1, 1), cf.DeviceView(dev, 0, 1, 8))
    with pytest.raises(cf.InvalidParams):
        cf.cf_tft(ctx, cf.TransformParams(8, 0, 0, 1), v)
    with pytest.raises(cf.InvalidParams):
        cf.cf_tft(ctx, cf.TransformParams(8, 0, 9, 1), v)
    with pytest.raises(cf.InvalidParams):
        cf.cf_tft(ctx, cf.TransformParams(8, 0, 1, 1, 1), v)
    with pytest.raises(cf.InvalidParams):
        cf.cf_tft(ctx, cf.TransformParams(4, 0, 1, 1), v)  # view length 8 != L
    with pytest.raises(cf.InvalidParams):
        cf.cf_itft(ctx, cf.TransformParams(8, 0, 2, 3), v)
    with pytest.raises(cf.InvalidParams):
        cf.cf_itft(ctx, cf.TransformParams(8, 0, 8, 8, 1), v)


@pytest.mark.parametrize("K", [2, 8, 64, 1024])
def test_negacyclic_random_sweep(K):
    m = random_modulus(K)
    ctx = cf.NegacyclicRingCtx(K, m)
    ring = po.Ring.negacyclic(K, m)
    rnd = random.Random(K)
    W = ctx.element_words
    for limit in (0, 2):
        ctx.set_leaf_limit(limit)
        for trial in range(12):
            L = 1 << rnd.randint(1, min(11, (2 * K).bit_length() - 1))
            z, n = rnd.randint(1, L), rnd.randint(1, L)
            s, pol = rnd.randrange(2 * K), rnd.randint(0, 1)
            buf = negacyclic_inputs(K, m, L, z, W, trial)
            want = buf.copy()
            ring.tft(want, L, s, z, n, pol)
            dev = to_dev(buf)
            cf.cf_tft(ctx, cf.TransformParams(L, s, z, n), cf.DeviceView(dev), pol)
            assert np.array_equal(from_dev(dev)[:n, :K], want[:n, :K]), (K, L, z, n, s, pol)
            n2, f = rnd.randint(0, z), rnd.randint(0, 1)
            if not 1 <= n2 + f <= L:
                continue
            buf = negacyclic_inputs(K, m, L, z, W, 100 + trial)
            want = buf.copy()
            ring.itft(want, L, s, z, n2, f, pol)
            dev = to_dev(buf)
            cf.cf_itft(ctx, cf.TransformParams(L, s, z, n2, f), cf.DeviceView(dev), pol)
            assert np.array_equal(from_dev(dev)[: n2 + f, :K], want[: n2 + f, :K]), (K, L, z, n2, f)


def test_c1_round_trip_bit_exact():
    """BASELINE config 1: Z/(2^1024+1), L=2^10, z=n=700, zeta=1: bit-exact vs the
    oracle, and ITFT(TFT(a)) = a after the 1/L = 2^(2048-10) scale."""
    N, L, z = 1024, 1024, 700
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    W = ctx.element_words
    lim = N // 64
    buf = fermat_inputs(N, L, z, W, po.mix_seed(42, 1))
    want = buf.copy()
    ring.tft(want, L, 0, z, z, 0)
    dev = to_dev(buf)
    view = cf.DeviceView(dev)
    cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), view)
    got = from_dev(dev)
    assert np.array_equal(got[:z, : lim + 1], want[:z, : lim + 1])
    ring.itft(want, L, 0, z, z, 0, 0)
    cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), view)
    assert np.array_equal(from_dev(dev)[:z, : lim + 1], want[:z, : lim + 1])
    cf.scale(ctx, view, z, 2 * N - 10)
    assert np.array_equal(from_dev(dev)[:z, : lim + 1], buf[:z, : lim + 1])


def _dist_single_rank(N, L, z, n):
    """The distributed path (column slab -> batched GPU column pass -> NCCL
    all-to-all -> row pass, and the ITFT back) on a one-rank NCCL group."""
    import socket

    import torch.distributed as dist

    from paper_0810_3203_b200.dist import DistTFT, GpuEngine

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    W = ctx.element_words
    lim = N // 64
    full = fermat_inputs(N, L, z, W, 77)
    full[z:] = 0
    want = full.copy()
    ring.tft(want, L, 0, z, n)
    fwd = DistTFT(GpuEngine(ctx), ring.M, L, 0, z, n)
    g = fwd.g
    col = to_dev(full)  # one rank: the column slab is the row-major array itself
    rows = fwd.tft(col)
    got = from_dev(rows)
    assert np.array_equal(got[:n, : lim + 1], want[:n, : lim + 1])
    inv = DistTFT(GpuEngine(ctx), ring.M, L, 0, n, n, 0)
    back = torch.zeros_like(col)
    inv.itft(rows, back)
    b = from_dev(back)
    exp = full.copy()
    ring_scale = po.Ring.fermat(N)
    for i in range(n):
        exp[i, : lim + 1] = ring_scale.twiddle(L.bit_length() - 1, full[i, : lim + 1])
    assert np.array_equal(b[:n, : lim + 1], exp[:n, : lim + 1])
    assert g.L1 * g.L2 == L


def test_dist_path_on_one_gpu():
    import torch.distributed as dist

    try:
        _dist_single_rank(1024, 1024, 700, 700)
        _dist_single_rank(4096, 4096, 3000, 3100)
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _nccl_group():
    import socket

    import torch.distributed as dist

    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))


def test_native_dist_path_on_one_gpu():
    """cftft_gpu_dist_tft / _itft (the C ABI's multi-GPU transforms over the
    library's own NCCL communicator) on a one-rank group: the column slab is
    the whole row-major array, the row slab its first rows; bit-exact against
    the oracle (TFT) and the single-GPU transform (ITFT with f = 1), and the
    C5 round trip."""
    import torch.distributed as dist

    from paper_0810_3203_b200.dist import NcclDist

    try:
        _nccl_group()
        for N, L, z, n in ((4096, 4096, 3000, 3100), (32768, 1 << 16, 40000, 40000)):
            ctx = cf.FermatRingCtx(N)
            ring = po.Ring.fermat(N)
            W = ctx.element_words
            lim = N // 64
            nd = NcclDist(ctx)
            full = fermat_inputs(N, L, z, W, 78)
            full[z:] = 0
            want = full.copy()
            ring.tft(want, L, 0, z, n, threads=8)
            geo = nd.geometry(cf.TransformParams(L, 0, z, n))
            assert geo["c0"] == 0 and geo["c1"] == geo["L2"] and geo["L1"] * geo["L2"] == L
            col = to_dev(full)
            rows = torch.zeros((geo["row_elems"], W), dtype=torch.int64, device="cuda")
            nd.tft(cf.TransformParams(L, 0, z, n), col, rows)
            got = from_dev(rows)
            assert np.array_equal(got[:n, : lim + 1], want[:n, : lim + 1]), (N, L, z, n)
            # ITFT (z, n - 1, f = 1) vs the single-GPU engine on the same inputs
            ni = n - 1
            gi = nd.geometry(cf.TransformParams(L, 0, n, ni, 1), inverse=True)
            rin = torch.zeros((gi["row_elems"], W), dtype=torch.int64, device="cuda")
            rin[: min(gi["row_elems"], rows.shape[0])] = rows[: min(gi["row_elems"], rows.shape[0])]
            back = torch.zeros_like(col)
            nd.itft(cf.TransformParams(L, 0, n, ni, 1), rin, back)
            ref = torch.zeros_like(col)
            ref[: rows.shape[0]] = rows
            cf.cf_itft(ctx, cf.TransformParams(L, 0, n, ni, 1), cf.DeviceView(ref))
            assert np.array_equal(from_dev(back)[: ni + 1, : lim + 1], from_dev(ref)[: ni + 1, : lim + 1])
        # C5 round trip through the native path
        N, L, z = 131072, 1 << 18, 200000
        ctx = cf.FermatRingCtx(N)
        W, lim = ctx.element_words, N // 64
        nd = NcclDist(ctx)
        a = fermat_inputs(N, L, z, W, 5)
        a[z:] = 0
        col = to_dev(a)
        geo = nd.geometry(cf.TransformParams(L, 0, z, z))
        # a ring that runs radix-64 leaves takes the single-GPU plan's own split
        assert geo["L1"] == 64 and geo["L2"] == L // 64
        rows = torch.empty((geo["row_elems"], W), dtype=torch.int64, device="cuda")
        nd.tft(cf.TransformParams(L, 0, z, z), col, rows)
        nd.itft(cf.TransformParams(L, 0, z, z, 0), rows, col)
        cf.scale(ctx, cf.DeviceView(col), z, 2 * N - 18)
        assert np.array_equal(from_dev(col)[:z, : lim + 1], a[:z, : lim + 1])
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


# ---- coset leaves (carry-save lanes) ---------------------------------------------

@pytest.mark.parametrize("N,cw", [(1024, 4), (2048, 8), (4096, 4), (8192, 16)])
@pytest.mark.parametrize("limit", [0, 2, 3])
def test_fermat_coset_sweep(N, cw, limit):
    """Factored nodes, coset tickets, boundary rotations and the carry-save
    fold, against the oracle on random shapes and twiddles."""
    ctx = cf.FermatRingCtx(N)
    ctx.set_coset(cw)
    ctx.set_leaf_limit(limit)
    ring = po.Ring.fermat(N)
    rnd = random.Random(N * 7 + cw + limit)
    for trial in range(16):
        L = 1 << rnd.randint(2, min(10, (2 * N).bit_length() - 1))
        z, n = rnd.randint(1, L), rnd.randint(1, L)
        s, pol = rnd.randrange(2 * N), rnd.randint(0, 1)
        _fermat_case(ctx, ring, N, L, z, n, s, pol, seed=trial, special=(trial % 3 == 0))
        n2, f = rnd.randint(0, z), rnd.randint(0, 1)
        if 1 <= n2 + f <= L:
            _fermat_case(ctx, ring, N, L, z, n2, s, pol, seed=500 + trial, inverse=True, f=f,
                         special=(trial % 3 == 1))


def test_fermat_coset_exhaustive_small():
    """Every (z, n) at L = 32 with coset leaves forced (cf. verify.hpp:85-120)."""
    N, L = 1024, 32
    ctx = cf.FermatRingCtx(N)
    ctx.set_coset(4)
    ctx.set_leaf_limit(2)
    ring = po.Ring.fermat(N)
    for z in range(1, L + 1):
        for n in range(1, L + 1, 3):
            _fermat_case(ctx, ring, N, L, z, n, 11, 0, seed=z * 100 + n, special=(z % 5 == 0))
        for n in range(0, z + 1, 2):
            for f in (0, 1):
                if 1 <= n + f <= L:
                    _fermat_case(ctx, ring, N, L, z, n, 3, 0, seed=z * 7 + n, inverse=True, f=f)


@pytest.mark.parametrize("N,L,z,n", [(32768, 4096, 3000, 3000), (65536, 2048, 1500, 1700), (131072, 1024, 700, 700)])
def test_fermat_coset_large_elements(N, L, z, n):
    """BASELINE-sized coefficients (automatic coset mode), TFT and ITFT vs the oracle."""
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    _fermat_case(ctx, ring, N, L, z, n, 0, 0, seed=N + z)
    _fermat_case(ctx, ring, N, L, min(z, n), min(z, n), 0, 0, seed=N + n, inverse=True, f=0)
    _fermat_case(ctx, ring, N, L, z, n // 2, 5, 1, seed=N + 1, inverse=True, f=1)


@pytest.mark.parametrize("N", [8192, 32768])
def test_fermat_wide_sweep(N):
    """Radix-64 coset leaves on the CTA kernel (set_wide(1)): full 64-point
    networks, truncated TFT networks, generic 16..64-slot programs, unaligned
    pre-rotations from deferred twiddles, against the oracle."""
    ctx = cf.FermatRingCtx(N)
    ctx.set_wide(1)
    ring = po.Ring.fermat(N)
    rnd = random.Random(N + 64)
    for trial in range(10):
        L = 1 << rnd.randint(6, 11)
        z, n = rnd.randint(1, L), rnd.randint(1, L)
        s, pol = rnd.randrange(2 * N), rnd.randint(0, 1)
        _fermat_case(ctx, ring, N, L, z, n, s, pol, seed=trial, special=(trial % 3 == 0))
        n2, f = rnd.randint(0, z), rnd.randint(0, 1)
        if 1 <= n2 + f <= L:
            _fermat_case(ctx, ring, N, L, z, n2, s, pol, seed=700 + trial, inverse=True, f=f,
                         special=(trial % 3 == 1))


@pytest.mark.parametrize("N", [128, 1024, 65536])
def test_fermat_scale_exponents(N):
    """cf.scale (x 2^e mod 2^N + 1, poly_mul's 1/L, polymul.hpp:82-87) against
    Python integers: random and edge values (0, 1, 2^N == -1, all-ones, single
    high bit) under exponents on and around 0, N and 2N, and random ones."""
    ctx = cf.FermatRingCtx(N)
    W, lim = ctx.element_words, N // 64
    rng = np.random.default_rng(N)
    count = 48
    mod = (1 << N) + 1
    exps = [0, 1, 31, 32, 33, N - 1, N, N + 1, N + 32, 2 * N - 1, 2 * N - 10, 2 * N, 5 * N + 3]
    exps += [int(x) for x in rng.integers(0, 4 * N, size=4)]
    for e in exps:
        buf = np.zeros((count, W), dtype=np.uint64)
        buf[:, :lim] = rng.integers(0, 1 << 63, size=(count, lim), dtype=np.uint64) * 2 + rng.integers(
            0, 2, size=(count, lim), dtype=np.uint64
        )
        buf[0, :] = 0
        buf[1, :] = 0
        buf[1, 0] = 1
        buf[2, :] = 0
        buf[2, lim] = 1  # 2^N
        buf[3, :lim] = np.uint64(0xFFFFFFFFFFFFFFFF)
        buf[4, :lim] = 0
        buf[4, lim - 1] = np.uint64(1 << 63)
        vals = [sum(int(buf[i, j]) << (64 * j) for j in range(lim)) + (int(buf[i, lim]) << N) for i in range(count)]
        dev = to_dev(buf)
        cf.scale(ctx, cf.DeviceView(dev), count, e)
        got = from_dev(dev)
        for i in range(count):
            want = vals[i] * pow(2, e, mod) % mod
            have = sum(int(got[i, j]) << (64 * j) for j in range(lim)) + (int(got[i, lim]) << N)
            assert int(got[i, lim]) in (0, 1) and have == want, (N, e, i)


@pytest.mark.parametrize("N", [256, 4096])
def test_fermat_sparse_values_carry_chains(N):
    """Small and sparse coefficients (0, 1, 2^N == -1, a few low bits): the
    outputs of the ITFT are mostly zero lanes, so the fold's carries run
    across whole elements in both directions -- TFT and ITFT against the
    oracle, then ITFT(TFT(a)) = L a (transform.hpp:266-272)."""
    ctx = cf.FermatRingCtx(N)
    ring = po.Ring.fermat(N)
    W, lim = ctx.element_words, N // 64
    rng = np.random.default_rng(N + 3)
    for L, z in ((64, 64), (512, 300)):
        buf = np.zeros((L, W), dtype=np.uint64)
        buf[:z, 0] = rng.integers(0, 1 << 20, size=z, dtype=np.uint64)
        buf[: z : 7, 0] = 0
        buf[1:z:11, 0] = 0
        buf[1:z:11, lim] = 1  # 2^N
        buf[2:z:13, 0] = 1
        want = buf.copy()
        ring.tft(want, L, 0, z, z, 0)
        dev = to_dev(buf)
        view = cf.DeviceView(dev)
        cf.cf_tft(ctx, cf.TransformParams(L, 0, z, z), view)
        assert np.array_equal(from_dev(dev)[:z, : lim + 1], want[:z, : lim + 1]), (N, L, z)
        ring.itft(want, L, 0, z, z, 0, 0)
        cf.cf_itft(ctx, cf.TransformParams(L, 0, z, z, 0), view)
        got = from_dev(dev)
        assert np.array_equal(got[:z, : lim + 1], want[:z, : lim + 1]), (N, L, z, "itft")
        mod = (1 << N) + 1
        for i in range(z):
            a = int(buf[i, 0]) + (int(buf[i, lim]) << N)
            have = sum(int(got[i, j]) << (64 * j) for j in range(lim)) + (int(got[i, lim]) << N)
            assert have == (L * a) % mod, (N, L, i)


# ---- one ring shared by two host threads -------------------------------------------

def test_ring_shared_by_two_threads_and_streams():
    """A ring context is shareable (include/cftft_b200.h): two host threads run
    transforms on ONE ring at the same time, each on its own stream with its
    own device view (coset plans keep scratch per stream), then each through
    the host-buffer entry points (one staging buffer per ring, serialised by
    the library).  Every result must equal the serial result of the same
    transform, many times over."""
    import threading

    N, L = 32768, 1 << 12  # coset plans (two radix-64 passes): shadow buffer and tops per stream
    ctx = cf.FermatRingCtx(N)
    W, lim = ctx.element_words, N // 64
    shapes = [(3000, 3100, 0), (4096, 4096, 0), (2500, 2049, 0), (3500, 3300, 1)]
    inputs = [fermat_inputs(N, L, z, W, 900 + k) for k, (z, n, f) in enumerate(shapes)]
    # serial expectations through the same library (its parity with the oracle
    # is the other tests' business): TFT outputs, then the ITFT of those
    want_t, want_i = [], []
    for (z, n, f), buf in zip(shapes, inputs):
        d = to_dev(buf)
        cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), cf.DeviceView(d))
        want_t.append(from_dev(d)[:n, : lim + 1].copy())
        ni = n - f
        d[n:] = 0
        cf.cf_itft(ctx, cf.TransformParams(L, 0, n, ni, f), cf.DeviceView(d))
        want_i.append(from_dev(d)[: ni + f, : lim + 1].copy())
    errors = []

    def worker(tid, host_api):
        try:
            torch.cuda.set_device(0)
            stream = torch.cuda.Stream()
            for rep in range(6):
                k = (tid + rep) % len(shapes)
                z, n, f = shapes[k]
                ni = n - f
                if host_api:
                    buf = inputs[k].copy()
                    cf.cf_tft_host(ctx, cf.TransformParams(L, 0, z, n), buf)
                    got_t = buf[:n, : lim + 1].copy()
                    buf[n:] = 0
                    cf.cf_itft_host(ctx, cf.TransformParams(L, 0, n, ni, f), buf)
                    got_i = buf[: ni + f, : lim + 1]
                else:
                    with torch.cuda.stream(stream):
                        d = to_dev(inputs[k])
                        cf.cf_tft(ctx, cf.TransformParams(L, 0, z, n), cf.DeviceView(d), stream=stream)
                        stream.synchronize()
                        got_t = from_dev(d)[:n, : lim + 1].copy()
                        d[n:] = 0
                        cf.cf_itft(ctx, cf.TransformParams(L, 0, n, ni, f), cf.DeviceView(d), stream=stream)
                        stream.synchronize()
                        got_i = from_dev(d)[: ni + f, : lim + 1]
                if not np.array_equal(got_t, want_t[k]):
                    errors.append((tid, rep, k, "tft", host_api))
                if not np.array_equal(got_i, want_i[k]):
                    errors.append((tid, rep, k, "itft", host_api))
        except Exception as ex:  # noqa: BLE001
            errors.append((tid, repr(ex)))

    for host_api in (False, True):
        ts = [threading.Thread(target=worker, args=(t, host_api)) for t in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    assert not errors, errors
