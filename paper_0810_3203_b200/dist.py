"""Multi-GPU TFT / ITFT: Bailey column slabs -> all-to-all transpose -> row slabs.

The north star partitions the large transform (BASELINE config 5) across the
GPUs of one box:

  TFT   (input: column slabs, output: row slabs)
    1. rank p owns top-level columns C_p = [c0_p, c1_p) (balanced over the
       z2' active columns) and runs their column TFTs locally
       (transform.hpp:175-180) -- one batched launch;
    2. all-to-all transpose: rank p sends rows R_q of its slab to rank q;
       R_q is a balanced split of the n1' ACTIVE output rows (rows >= n1'
       are never needed, so no rank idles on them);
    3. rank q runs its row TFTs locally (transform.hpp:182-185).
  ITFT  (input: row slabs, output: column slabs -- the TFT's input layout)
    i.   rows u < n1 (full) on the row owners (transform.hpp:215-216);
    -    all-to-all transpose rows [0, n1) -> column slabs;
    ii.  right columns [n2, z2') on the column owners (transform.hpp:219-224);
    iii. row n1 (transform.hpp:227-230): its right part (phase-ii outputs) is
         gathered to the rank that owns row n1, transformed there, and its
         left part scattered back to the column owners;
    iv.  left columns [0, n2) on the column owners (transform.hpp:233-238).

Only the transposes and the phase-iii row exchange cross NVLink (NCCL
all_to_all_single over torch.distributed).  Local sub-transforms run on the
GPU engine in one batched launch per phase (cftft_gpu_batch).  The local
engine is pluggable so the orchestration can be exercised on CPU ranks
(gloo) in the tests.

Local storage
  column slab on rank p: tensor [L1 * W_p, words]; local (r, c) <-> global
      element r * L2 + c0_p + c (row-major rows of the rank's columns)
  row slab on rank q:    tensor [|R_q| * L2, words]; global rows r0_q.. in
      order, each row contiguous.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def _split(ell: int, policy: int):
    return (1, ell - 1) if policy else (ell // 2, ell - ell // 2)


def _balanced(total: int, parts: int, k: int):
    q, r = divmod(total, parts)
    lo = k * q + min(k, r)
    return lo, lo + q + (1 if k < r else 0)


@dataclass
class Sub:
    """One sub-transform over a local slab: element i at base + i*stride."""
    L: int
    s: int
    z: int
    n: int
    f: int
    base: int
    stride: int


class GpuEngine:
    """Local sub-transforms on this rank's GPU (libcftft_b200.so)."""

    def __init__(self, ctx, policy: int = 0):
        self.ctx, self.policy = ctx, policy
        self.launches = 0

    def batch(self, inverse: bool, subs, slab: torch.Tensor) -> None:
        """One batched launch; outputs canonical (coset plans end in their
        carry-save fold, whole-leaf plans get a canonicalising pass)."""
        from . import last_launch_count, run_batch

        if subs:
            run_batch(self.ctx, inverse, subs, slab, self.policy, canonicalize=True)
            self.launches += last_launch_count()


class DistGeometry:
    """Partition of one (L, z, n[, f]) transform over `world` ranks."""

    def __init__(self, M: int, L: int, z: int, n: int, world: int, policy: int = 0, inverse: bool = False,
                 f: int = 0, l1: int | None = None):
        """l1: log2 of the column length when it is not the policy's split (the
        native path takes columns of 64 on rings that run radix-64 leaves:
        cftft_dist_geometry reports L1)."""
        self.M, self.L, self.z, self.n, self.world = M, L, z, n, world
        ell = L.bit_length() - 1
        self.ell = ell
        self.l1, self.l2 = _split(ell, policy) if l1 is None else (l1, ell - l1)
        self.L1, self.L2 = 1 << self.l1, 1 << self.l2
        L2 = self.L2
        self.n2, self.n1 = n & (L2 - 1), n >> self.l2
        self.n1c = self.n1 + (1 if self.n2 else 0)
        self.z2, self.z1 = z & (L2 - 1), z >> self.l2
        self.z2e = L2 if self.z1 else self.z2
        self.col_step = M >> ell
        self.cols = [_balanced(L2, world, p) for p in range(world)]  # column slabs
        # active rows: the TFT's output rows; the ITFT's input rows (and row n1
        # when phase iii runs).  A TFT (z, n) followed by an ITFT (n, n, 0) agree.
        self.zrows = self.z1 + (1 if self.z2 else 0)
        if inverse:
            fm = 1 if self.n2 + f > 0 else 0
            R = max(self.zrows, self.n1 + fm)
        else:
            R = self.n1c
        self.R = R
        self.rows = [_balanced(R, world, p) for p in range(world)]

    def width(self, p: int) -> int:
        a, b = self.cols[p]
        return b - a

    def nrows(self, p: int) -> int:
        a, b = self.rows[p]
        return b - a


class DistTFT:
    """Forward / inverse TFT of one transform partitioned over the process group."""

    def __init__(self, engine, M: int, L: int, s: int, z: int, n: int, f: int = 0, group=None,
                 policy: int = 0):
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.s, self.f = s % M, f
        self.inverse = None
        self.g = DistGeometry(M, L, z, n, self.world, policy)
        self.gi = DistGeometry(M, L, z, n, self.world, policy, inverse=True, f=f)

    # ---- layout helpers --------------------------------------------------------
    def col_slab_shape(self, words: int):
        return (self.g.L1 * self.g.width(self.rank), words)

    def row_slab_shape(self, words: int):
        return (self.g.nrows(self.rank) * self.g.L2, words)

    def itft_row_slab_shape(self, words: int):
        return (self.gi.nrows(self.rank) * self.gi.L2, words)

    # ---- TFT ---------------------------------------------------------------------
    def tft(self, colslab: torch.Tensor) -> torch.Tensor:
        """colslab: this rank's column slab (rows >= z1+1 arbitrary).
        Returns this rank's row slab of the first n transformed values."""
        g, p = self.g, self.rank
        c0, c1 = g.cols[p]
        W = c1 - c0
        subs = []
        for c in range(W):
            u = c0 + c
            if u >= g.z2e:
                continue
            subs.append(Sub(g.L1, self.s + u * g.col_step, g.z1 + 1 if u < g.z2 else g.z1, g.n1c, 0, c, W))
        self.engine.batch(False, subs, colslab)
        rowslab = self._cols_to_rows(colslab, W)
        r0, r1 = g.rows[p]
        s_row = (self.s << g.l1) % g.M
        subs = [Sub(g.L2, s_row, g.z2e, g.L2 if u < g.n1 else g.n2, 0, (u - r0) * g.L2, 1)
                for u in range(r0, r1)]
        self.engine.batch(False, subs, rowslab)
        return rowslab

    def _valid_in_rows(self, r0: int, r1: int, count: int) -> int:
        g = self.g
        v = 0
        for u in range(r0, r1):
            v += max(0, min(g.L2, count - u * g.L2))
        return v

    def _cols_to_rows(self, colslab: torch.Tensor, W: int) -> torch.Tensor:
        """All-to-all: column slabs (rows [0, n1')) -> row slabs."""
        g, p = self.g, self.rank
        words = colslab.shape[1]
        send_splits = [g.nrows(q) * W for q in range(self.world)]
        r_lo = g.rows[0][0]
        r_hi = g.rows[-1][1]
        send = colslab[r_lo * W: r_hi * W]  # rows R_0 .. R_{P-1} are consecutive
        recv_splits = [g.nrows(p) * g.width(q) for q in range(self.world)]
        recv = torch.empty((sum(recv_splits), words), dtype=colslab.dtype, device=colslab.device)
        dist.all_to_all_single(recv, send.contiguous(), recv_splits, send_splits, group=self.group)
        nr = g.nrows(p)
        rowslab = torch.empty((nr * g.L2, words), dtype=colslab.dtype, device=colslab.device)
        rv = rowslab.view(nr, g.L2, words)
        off = 0
        for q in range(self.world):
            a, b = g.cols[q]
            k = nr * (b - a)
            rv[:, a:b] = recv[off: off + k].view(nr, b - a, words)
            off += k
        return rowslab

    def _rows_to_cols(self, g, rowslab: torch.Tensor, nrows_total: int, colslab: torch.Tensor) -> None:
        """All-to-all: row slabs (global rows [0, nrows_total)) -> column slabs."""
        p = self.rank
        words = rowslab.shape[1]
        r0, r1 = g.rows[p]
        mine = max(0, min(r1, nrows_total) - r0)
        rv = rowslab.view(-1, g.L2, words)
        sends, send_splits = [], []
        for q in range(self.world):
            a, b = g.cols[q]
            blk = rv[:mine, a:b].reshape(mine * (b - a), words)
            sends.append(blk)
            send_splits.append(mine * (b - a))
        send = torch.cat(sends, 0) if sends else rowslab[:0]
        W = g.width(p)
        recv_splits = []
        for q in range(self.world):
            qa, qb = g.rows[q]
            recv_splits.append(max(0, min(qb, nrows_total) - qa) * W)
        recv = torch.empty((sum(recv_splits), words), dtype=rowslab.dtype, device=rowslab.device)
        dist.all_to_all_single(recv, send.contiguous(), recv_splits, send_splits, group=self.group)
        # rows arrive in global order (R_0, R_1, ...): rows [0, nrows_total) of the slab
        colslab[: nrows_total * W] = recv.view(nrows_total * W, words)

    # ---- ITFT --------------------------------------------------------------------
    def itft(self, rowslab: torch.Tensor, colslab: torch.Tensor) -> None:
        """rowslab: this rank's row slab holding x[0..n) (the transformed
        values) and x[n..z) (L times the coefficients); rows beyond are never
        read.  On return colslab (this rank's column slab) holds L times the
        coefficients x[0..n), plus x[n] (the next transformed value) if f=1."""
        g, p, f = self.gi, self.rank, self.f
        z, n = g.z, g.n
        n1, n2, z1, z2, z2e = g.n1, g.n2, g.z1, g.z2, g.z2e
        fm = 1 if n2 + f > 0 else 0
        lo, hi = min(n2, z2), max(n2, z2)
        s_row = (self.s << g.l1) % g.M
        r0, r1 = g.rows[p]
        c0, c1 = g.cols[p]
        W = c1 - c0
        words = rowslab.shape[1]
        # phase i: full rows u < n1 (transform.hpp:215-216)
        subs = [Sub(g.L2, s_row, g.L2, g.L2, 0, (u - r0) * g.L2, 1) for u in range(r0, min(r1, n1))]
        self.engine.batch(True, subs, rowslab)
        # rows [0, ceil(z / L2)) of every column are read by phases ii / iv
        self._rows_to_cols(g, rowslab, g.zrows, colslab)
        # phase ii: right columns [n2, z2') (transform.hpp:219-224)
        subs = []
        for c in range(W):
            u = c0 + c
            if n2 <= u < z2e:
                subs.append(Sub(g.L1, self.s + u * g.col_step, z1 + 1 if u < hi else z1, n1, fm, c, W))
        self.engine.batch(True, subs, colslab)
        if fm:
            self._phase3(g, colslab, rowslab, s_row)
        # phase iv: left columns [0, n2) (transform.hpp:233-238)
        subs = []
        for c in range(W):
            u = c0 + c
            if u < n2:
                subs.append(Sub(g.L1, self.s + u * g.col_step, z1 + 1 if u < lo else z1, n1 + 1, 0, c, W))
        self.engine.batch(True, subs, colslab)

    def _phase3(self, g, colslab, rowslab, s_row):
        """Row n1 (transform.hpp:227-230): gather its right part from the column
        owners to the rank owning row n1, transform it there, scatter back."""
        p, f = self.rank, self.f
        n1, n2, z2e = g.n1, g.n2, g.z2e
        words = colslab.shape[1]
        owner = next(q for q in range(self.world) if g.rows[q][0] <= n1 < g.rows[q][1])
        c0, c1 = g.cols[p]
        W = c1 - c0
        # 1) gather: every rank sends its row-n1 elements of columns [max(n2,c0), min(z2e,c1)) to owner
        a, b = max(n2, c0), min(z2e, c1)
        mine = colslab[n1 * W + (a - c0): n1 * W + (b - c0)] if b > a else colslab[:0]
        send_splits = [(b - a if b > a else 0) if q == owner else 0 for q in range(self.world)]
        recv_splits = [0] * self.world
        if p == owner:
            for q in range(self.world):
                qa, qb = g.cols[q]
                aa, bb = max(n2, qa), min(z2e, qb)
                recv_splits[q] = bb - aa if bb > aa else 0
        recv = torch.empty((sum(recv_splits), words), dtype=colslab.dtype, device=colslab.device)
        dist.all_to_all_single(recv, mine.contiguous(), recv_splits, send_splits, group=self.group)
        # 2) transform row n1 on its owner: columns < n2 are already in its row slab
        if p == owner:
            r0 = g.rows[p][0]
            row = rowslab[(n1 - r0) * g.L2: (n1 - r0 + 1) * g.L2]
            off = 0
            for q in range(self.world):
                qa, qb = g.cols[q]
                aa, bb = max(n2, qa), min(z2e, qb)
                if bb > aa:
                    row[aa:bb] = recv[off: off + (bb - aa)]
                    off += bb - aa
            self.engine.batch(True, [Sub(g.L2, s_row, z2e, n2, f, (n1 - r0) * g.L2, 1)], rowslab)
        # 3) scatter row n1 columns [0, n2 + f) back to their column owners
        outs = n2 + f
        send_splits = [0] * self.world
        sends = []
        if p == owner:
            r0 = g.rows[p][0]
            row = rowslab[(n1 - r0) * g.L2: (n1 - r0 + 1) * g.L2]
            for q in range(self.world):
                qa, qb = g.cols[q]
                aa, bb = qa, min(outs, qb)
                if bb > aa:
                    sends.append(row[aa:bb])
                    send_splits[q] = bb - aa
        send = torch.cat(sends, 0) if sends else colslab[:0]
        aa, bb = c0, min(outs, c1)
        recv_splits = [(bb - aa if bb > aa else 0) if q == owner else 0 for q in range(self.world)]
        recv = torch.empty((sum(recv_splits), words), dtype=colslab.dtype, device=colslab.device)
        dist.all_to_all_single(recv, send.contiguous(), recv_splits, send_splits, group=self.group)
        if bb > aa:
            colslab[n1 * W + (aa - c0): n1 * W + (bb - c0)] = recv


# ---------------------------------------------------------------------------
# The native path: the same partition in the library (csrc/dist.cuh) over an
# NCCL communicator of its own (cftft_gpu_dist_tft / cftft_gpu_dist_itft).


def native_schedule(M: int, L: int, z: int, n: int, f: int, world: int, rank: int, inverse: bool = False,
                    policy: int = 0, wide: bool = False):
    """cftft_dist_schedule: the transpose pieces rank `rank` hands to NCCL, as
    tuples (chunk, send, peer, buf, offset, count) in issue order (pure host
    code; tests replay it over simulated ranks)."""
    import ctypes as C

    from . import _Params, lib

    Lb = lib()
    Lb.cftft_dist_schedule.argtypes = [C.c_uint64, C.POINTER(_Params), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.POINTER(C.c_uint64), C.c_size_t]
    Lb.cftft_dist_schedule.restype = C.c_size_t
    p = _Params(L, 0, z, n, f if inverse else 0)
    need = Lb.cftft_dist_schedule(M, C.byref(p), int(inverse), policy, int(wide), world, rank, None, 0)
    buf = (C.c_uint64 * max(1, need))()
    got = Lb.cftft_dist_schedule(M, C.byref(p), int(inverse), policy, int(wide), world, rank, buf, need)
    assert got == need
    return [tuple(buf[i:i + 6]) for i in range(0, need, 6)]


class NcclDist:
    """A distributed context of the C ABI for the current torch.distributed
    group: rank 0 makes an NCCL unique id, the group broadcasts it, every rank
    joins the library's communicator on its current CUDA device."""

    def __init__(self, ctx, group=None, policy: int = 0):
        import ctypes as C

        from . import _check, lib

        self.ctx, self.policy = ctx, policy
        L = lib()
        vp = C.c_void_p
        if not getattr(L, "_dist_bound", False):
            L.cftft_nccl_unique_id.argtypes = [vp]
            L.cftft_dist_create.argtypes = [vp, C.c_int, C.c_int, vp, C.POINTER(vp)]
            L.cftft_dist_destroy.argtypes = [vp]
            L.cftft_dist_destroy.restype = None
            L.cftft_dist_geometry.argtypes = [vp, vp, C.c_int, C.c_int, C.POINTER(C.c_uint64)]
            for fn in ("cftft_gpu_dist_tft", "cftft_gpu_dist_itft"):
                getattr(L, fn).argtypes = [vp, vp, vp, vp, C.c_uint64, C.c_int, vp]
            L._dist_bound = True
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        idbuf = (C.c_uint8 * 128)()
        if self.rank == 0:
            _check(L.cftft_nccl_unique_id(C.cast(idbuf, vp)))
        t = torch.tensor(list(idbuf), dtype=torch.uint8,
                         device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        for i, b in enumerate(t.cpu().tolist()):
            idbuf[i] = b
        h = vp()
        _check(L.cftft_dist_create(ctx._h, self.rank, self.world, C.cast(idbuf, vp), C.byref(h)))
        self._h = h
        self.launches = 0

    def __del__(self):
        try:
            from . import lib

            lib().cftft_dist_destroy(self._h)
        except Exception:
            pass

    def geometry(self, params, inverse: bool = False) -> dict:
        """{c0, c1, r0, r1, L1, L2, col_elems, row_elems} of this rank."""
        import ctypes as C

        from . import _check, _params, lib

        p = _params(params)
        out = (C.c_uint64 * 8)()
        _check(lib().cftft_dist_geometry(self._h, C.byref(p), 1 if inverse else 0, self.policy, out))
        return dict(zip(("c0", "c1", "r0", "r1", "L1", "L2", "col_elems", "row_elems"), list(out)))

    def tft(self, params, colslab: torch.Tensor, rowslab: torch.Tensor, stream=None) -> None:
        import ctypes as C

        from . import _check, _params, _stream_ptr, lib

        p = _params(params)
        _check(lib().cftft_gpu_dist_tft(self._h, C.byref(p), C.c_void_p(colslab.data_ptr()),
                                        C.c_void_p(rowslab.data_ptr()), colslab.shape[1] * 8, self.policy,
                                        C.c_void_p(_stream_ptr(stream))))

    def itft(self, params, rowslab: torch.Tensor, colslab: torch.Tensor, stream=None) -> None:
        import ctypes as C

        from . import _check, _params, _stream_ptr, lib

        p = _params(params)
        _check(lib().cftft_gpu_dist_itft(self._h, C.byref(p), C.c_void_p(rowslab.data_ptr()),
                                         C.c_void_p(colslab.data_ptr()), rowslab.shape[1] * 8, self.policy,
                                         C.c_void_p(_stream_ptr(stream))))
