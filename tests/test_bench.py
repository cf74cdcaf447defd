"""bench.py's measurement helpers on CPU: the Bailey sub-transform listing the
CPU baseline samples from is the real decomposition (run in full it equals
the oracle's TFT / ITFT bit for bit), and its byte count equals the
algorithmic-bytes formulas of SURVEY.md §8d."""
from __future__ import annotations

import numpy as np
import pytest

import bench
import pyoracle as po
from helpers import fermat_inputs


@pytest.mark.parametrize("L,z,n", [(256, 200, 200), (256, 131, 170), (64, 64, 64), (1024, 700, 700),
                                   (512, 300, 511)])
def test_bailey_phases_reproduce_the_oracle(oracle, L, z, n):
    N = max(256, L // 2)
    ring = po.Ring.fermat(N)
    W = ring.words + 1
    buf = fermat_inputs(N, L, z, W, L + z + n)
    buf[z:] = 0
    want = buf.copy()
    ring.tft(want, L, 0, z, n)
    got = buf.copy()
    for _, inverse, subs in bench.bailey_phases(2 * N, L, z, n, 0, False):
        for (Ls, ss, zs, ns, fs, base, stride) in subs:
            ring.tft_at(got, base, stride, Ls, ss, zs, ns)
    assert np.array_equal(got[:n, : ring.words], want[:n, : ring.words])
    if z > n:
        return
    back = want.copy()
    ring.itft(back, L, 0, n, n, 0)
    for _, inverse, subs in bench.bailey_phases(2 * N, L, n, n, 0, True):
        for (Ls, ss, zs, ns, fs, base, stride) in subs:
            ring.itft_at(got, base, stride, Ls, ss, zs, ns, fs)
    assert np.array_equal(got[:n, : ring.words], back[:n, : ring.words])


@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C5"])
def test_phase_bytes_match_formulas(name):
    N, L, z, n, _ = bench.CONFIGS[name]
    B = N // 8
    t = sum(B * sum(zs + ns + fs for (_, _, zs, ns, fs, _, _) in subs)
            for _, _, subs in bench.bailey_phases(2 * N, L, z, n, 0, False))
    i = sum(B * sum(zs + ns + fs for (_, _, zs, ns, fs, _, _) in subs)
            for _, _, subs in bench.bailey_phases(2 * N, L, n, n, 0, True))
    assert t == bench.tft_bytes(N, L, z, n)
    assert i == bench.itft_bytes(N, L, n, n, 0)
