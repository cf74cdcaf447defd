"""Multi-rank orchestration of the distributed TFT/ITFT (paper_0810_3203_b200.dist)
on CPU ranks over gloo: column slabs -> all-to-all -> row slabs and back.

The per-rank sub-transforms are run by a test engine built on the CPU oracle
(the GPU engine is exercised by the -m gpu tests and bench.py --gpus N); what
is checked here is the partitioning, the transposes and the ITFT phase-iii
exchange, bit for bit against the single-process oracle transform.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleEngine:
    """Runs each sub-transform with the CPU oracle (test-only engine)."""

    def __init__(self, ring):
        self.ring = ring

    def batch(self, inverse, subs, slab):
        a = slab.numpy().view(np.uint64)
        for sb in subs:
            idx = sb.base + sb.stride * np.arange(sb.L)
            buf = np.ascontiguousarray(a[idx])
            if inverse:
                self.ring.itft(buf, sb.L, sb.s, sb.z, sb.n, sb.f)
            else:
                self.ring.tft(buf, sb.L, sb.s, sb.z, sb.n)
            a[idx] = buf

    def canonicalize(self, slab, count):
        pass  # oracle outputs are canonical


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, L, s, z, n, q):
    import sys

    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import pyoracle as po
    from paper_0810_3203_b200.dist import DistTFT

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ring = po.Ring.fermat(N)
        W = ring.words + 1  # padded element, like the GPU format
        rng = np.random.default_rng(1234)
        full = np.zeros((L, W), dtype=np.uint64)
        full[:z, : N // 64] = rng.integers(0, 1 << 64, size=(z, N // 64), dtype=np.uint64, endpoint=False)
        want = full.copy()
        ring.tft(want, L, s, z, n)

        fwd = DistTFT(OracleEngine(ring), ring.M, L, s, z, n)
        g = fwd.g
        c0, c1 = g.cols[rank]
        Wc = c1 - c0
        # this rank's column slab of the input
        col = np.zeros((g.L1 * Wc, W), dtype=np.uint64)
        for r in range(g.L1):
            col[r * Wc:(r + 1) * Wc] = full[r * g.L2 + c0: r * g.L2 + c1]
        colt = torch.from_numpy(col.view(np.int64))
        rowt = fwd.tft(colt)
        rows = rowt.numpy().view(np.uint64)
        r0, r1 = g.rows[rank]
        ok_fwd = True
        for u in range(r0, r1):
            for c in range(g.L2):
                e = u * g.L2 + c
                if e < n and not np.array_equal(rows[(u - r0) * g.L2 + c, : ring.words], want[e, : ring.words]):
                    ok_fwd = False
        # inverse: the row slab from the forward transform -> L * a in column slabs
        inv = DistTFT(OracleEngine(ring), ring.M, L, s, n, n, 0)
        assert inv.gi.rows == g.rows
        colback = torch.zeros_like(colt)
        inv.itft(rowt, colback)
        cb = colback.numpy().view(np.uint64)
        ok_inv = True
        for r in range(g.L1):
            for c in range(Wc):
                e = r * g.L2 + c0 + c
                if e < n:
                    la = full[e, : ring.words].copy()  # L * a_e
                    for _ in range(L.bit_length() - 1):
                        la = ring.add(la, la)
                    if not np.array_equal(cb[r * Wc + c, : ring.words], la):
                        ok_inv = False
        q.put((rank, ok_fwd, ok_inv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L,z,n,s", [(2, 256, 200, 200, 0), (2, 256, 131, 170, 7), (3, 256, 250, 255, 3),
                                           (3, 256, 256, 256, 5), (2, 64, 33, 33, 1)])
def test_distributed_round_trip_matches_oracle(oracle, world, L, z, n, s):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 128, L, s, z, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_fwd, ok_inv in sorted(res):
        assert ok_fwd, f"rank {rank}: distributed TFT differs from the oracle"
        assert ok_inv, f"rank {rank}: distributed ITFT(TFT(a)) != L*a"


def test_geometry_config5():
    from paper_0810_3203_b200.dist import DistGeometry

    for P in (1, 2, 4, 8):
        g = DistGeometry(262144, 1 << 18, 200000, 200000, P)
        assert g.L1 == g.L2 == 512 and g.n1c == 391
        assert sum(b - a for a, b in g.cols) == 512
        assert sum(b - a for a, b in g.rows) == 391  # only active rows are distributed
        assert max(b - a for a, b in g.rows) - min(b - a for a, b in g.rows) <= 1


@pytest.mark.parametrize("wide", [False, True])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("L,z,n,f", [(1 << 12, 3000, 3100, 0), (1 << 12, 4096, 4096, 0), (1 << 12, 700, 650, 1),
                                     (1 << 14, 10001, 9999, 1), (1 << 18, 200000, 200000, 0)])
def test_native_transpose_schedules_over_simulated_ranks(L, z, n, f, P, wide):
    """The send / receive pieces cftft_gpu_dist_tft / _itft hand to NCCL
    (cftft_dist_schedule, pure host code), replayed over P simulated ranks:
    NCCL pairs the i-th send from a to b with the i-th receive at b from a
    within a group (= one chunk).  Every pair must agree in count, and the
    pieces must put element (r, c) of the L1 x L2 matrix where the other
    slab layout wants it -- for the TFT (column slabs -> row slabs, all
    active rows) and for the ITFT (row slabs -> column slabs, rows < zrows)."""
    from paper_0810_3203_b200.dist import DistGeometry, native_schedule

    M = 2 * L
    ell = L.bit_length() - 1
    l1 = 6 if (wide and ell >= 12) else None
    for inverse in (False, True):
        zz, nn = (z, n) if not inverse else (max(z, n), n)  # an ITFT needs z >= n
        g = DistGeometry(M, L, zz, nn, P, inverse=inverse, f=f if inverse else 0, l1=l1)
        L2 = g.L2
        # slabs hold global element ids r * L2 + c (column slab: [L1][W]; row slab: [nrows][L2])
        col = [np.full(g.L1 * g.width(p), -1, dtype=np.int64) for p in range(P)]
        row = [np.full(max(1, g.nrows(p)) * L2, -1, dtype=np.int64) for p in range(P)]
        for p in range(P):
            c0, c1 = g.cols[p]
            r0, r1 = g.rows[p]
            if not inverse:
                col[p][:] = (np.arange(g.L1)[:, None] * L2 + np.arange(c0, c1)[None, :]).ravel()
            elif r1 > r0:
                row[p][: (r1 - r0) * L2] = (np.arange(r0, r1)[:, None] * L2 + np.arange(L2)[None, :]).ravel()
        sched = [native_schedule(M, L, zz, nn, f, P, p, inverse=inverse, wide=wide) for p in range(P)]
        chunks = 1 + max((rec[0] for s in sched for rec in s), default=0)
        assert chunks <= 4
        for k in range(chunks):
            queues = {}
            for p in range(P):  # every rank's sends of the group, in issue order
                for (ck, send, peer, buf, off, cnt) in sched[p]:
                    if ck == k and send:
                        src = (row if buf else col)[p]
                        assert off + cnt <= src.size
                        queues.setdefault((p, peer), []).append(src[off: off + cnt].copy())
            for p in range(P):  # matched with the receives, in issue order
                for (ck, send, peer, buf, off, cnt) in sched[p]:
                    if ck == k and not send:
                        q = queues.get((peer, p))
                        assert q, "a receive without a matching send"
                        data = q.pop(0)
                        assert data.size == cnt, "send / receive sizes differ"
                        dst = (row if buf else col)[p]
                        assert off + cnt <= dst.size
                        dst[off: off + cnt] = data
            assert all(not q for q in queues.values()), "a send without a matching receive"
        for p in range(P):
            c0, c1 = g.cols[p]
            r0, r1 = g.rows[p]
            if not inverse:  # every active row, all L2 columns
                want = (np.arange(r0, r1)[:, None] * L2 + np.arange(L2)[None, :]).ravel()
                assert np.array_equal(row[p][: want.size], want), (P, p, "TFT row slab")
            else:            # rows [0, zrows) of my columns
                zr = g.zrows
                want = np.arange(zr)[:, None] * L2 + np.arange(c0, c1)[None, :]
                got = col[p].reshape(g.L1, c1 - c0)[:zr]
                assert np.array_equal(got, want), (P, p, "ITFT column slab")
