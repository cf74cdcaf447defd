"""The C ABI and the host planner, on the CPU (no GPU calls).

  * libcftft_b200.so loads and exports every symbol include/cftft_b200.h declares
  * validation maps onto BadLength / InvalidParams before any GPU work
  * the planner's base-case replay equals the reference's ButterflyStats at
    the BASELINE shapes (tests/golden/counts.json)
  * the GPU schedule (leaves, waves, micro-ops with pending rotations),
    executed at the VALUE level with Python integers, reproduces the
    definition of the TFT/ITFT: this pins the planner independently of the
    kernels' limb arithmetic
"""
from __future__ import annotations

import ctypes as C
import json
import os
import random
import re

import pytest

import bigint_model as bm
import paper_0810_3203_b200 as cf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "cftft_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cftft_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = cf.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.cftft_version()


def test_ring_contexts():
    f = cf.FermatRingCtx(32768)
    assert f.root_order() == 65536
    assert f.element_bytes == 4096 + 16
    n = cf.NegacyclicRingCtx(1024, (1 << 61) + 15)
    assert n.root_order() == 2048 and n.element_bytes == 8192
    with pytest.raises(cf.Unsupported):
        cf.FermatRingCtx(1000)
    with pytest.raises(cf.InvalidParams):
        cf.NegacyclicRingCtx(8, 96)  # even modulus


def test_c_abi_validation_without_gpu():
    lib = cf.lib()
    ctx = cf.FermatRingCtx(128)  # M = 256

    def call(L, z, n, f=0, inv=False, stride=None):
        p = cf._Params(L, 0, z, n, f)
        fn = lib.cftft_gpu_itft if inv else lib.cftft_gpu_tft
        return fn(ctx._h, C.byref(p), None, stride or ctx.element_bytes, 0, None, None)

    assert call(12, 1, 1) == 1
    assert call(512, 1, 1) == 1  # exceeds the root order
    assert call(8, 0, 1) == 2
    assert call(8, 9, 1) == 2
    assert call(8, 1, 0) == 2
    assert call(8, 1, 1, f=1) == 2
    assert call(8, 2, 3, inv=True) == 2
    assert call(8, 1, 0, 0, inv=True) == 2
    assert call(8, 8, 8, 1, inv=True) == 2
    assert call(8, 8, 8, stride=24) == 4  # stride not a multiple of 16
    with pytest.raises(cf.BadLength):
        cf._validate(ctx, cf.TransformParams(12, 0, 1, 1), False, 12)
    with pytest.raises(cf.InvalidParams):
        cf._validate(ctx, cf.TransformParams(4, 0, 1, 1), False, 8)


def test_base_case_counts_match_reference():
    cases = json.load(open(os.path.join(GOLD, "counts.json")))
    for c in cases:
        if c["inverse"]:
            got = cf.itft_base_cases(c["L"], c["z"], c["n"], c["f"], c["policy"])
        else:
            got = cf.tft_base_cases(c["L"], c["z"], c["n"], c["policy"])
        assert got == c["count"], c


def test_counts_full_transform_hits_ceiling():  # transform_test.cpp:342-351
    for ell in range(1, 8):
        L = 1 << ell
        for pol in (0, 1):
            assert 2 * cf.tft_base_cases(L, L, L, pol) == L * ell
            assert 2 * cf.itft_base_cases(L, L, L, 0, pol) == L * ell


def test_counts_respect_bounds():  # verify.hpp:223-269
    for ell in range(1, 6):
        L = 1 << ell
        for z in range(1, L + 1):
            for n in range(1, L + 1):
                assert cf.tft_base_cases(L, z, n, 0) <= cf.tft_bound(L, n)
            for n in range(0, z + 1):
                for f in (0, 1):
                    if 1 <= n + f <= L:
                        assert cf.itft_base_cases(L, z, n, f, 1) <= cf.itft_bound(L, n, f)


# ---- value-level execution of the GPU schedule ----------------------------------

def run_plan_fermat(plan, N, vals):
    """Executes the ticket list at the value level, checking that every leaf's
    dependency counter is complete when its ticket comes up.  Coset leaves
    (one ticket per group of lane cosets) are run once, at their first ticket;
    every rotation they perform must be a whole number of lanes."""
    P, M = (1 << N) + 1, 2 * N
    lane = plan.get("lane_bits", 0)
    bits = plan.get("locbits", [])
    x = {(0, e): v for e, v in vals.items()}  # (buffer, element) -> value

    def buf(locoff, k, out):
        if locoff < 0:
            return 0
        return (bits[locoff + 2 * (k // 64) + (1 if out else 0)] >> (k % 64)) & 1

    meta = plan["counters"]
    counters = [0] * len(meta)
    wplan, ws = plan.get("wave", 0), plan.get("wave_slots", [])
    for (cls, base, stride, s, dep, target, comp, wave, tpre, tpost, c0, locoff) in plan["leaves"]:
        if dep >= 0:
            assert counters[dep] >= target, "ticket order is not topological"
        c = plan["classes"][cls]
        inv, cn, cf_ = c["inverse"], c["n"], c["f"]
        coset = c["kind"] == 1
        run = not coset or c0 == 0 or plan.get("wave", 0)  # wave plans: one ticket per leaf (c0 = slot table)
        slot = [None] * (1 << c["ell"])
        for i in range(c["nload"] if run else 0):
            a, b = c["pre"][i]
            e = (a * s + b + (tpre if inv and i < cn else 0)) % M
            if wplan and coset:  # the ticket's table: any bits, deferred rotations included
                e = ws[c0 + 2 * i] & 0x3FFFFFFF
            elif wplan and c0 > 0:  # a whole ticket reading elements with deferred rotations
                e = (e + ws[c0 - 1 + i]) % M
            assert not coset or e % lane == 0 or wplan
            slot[i] = (x[(buf(locoff, i, False), base + i * stride)] * pow(2, e, P)) % P
        ops = c["ops"]
        if c.get("net") and c["ell"] == 4:
            # the warp kernel's 16-slot network (wave_coset.cuh): DIF = span 8
            # then the 8-point networks of slots 0-7, 8-15; DIT the reverse
            for i in range(c["nload"], 16):
                slot[i] = 0
            ops, unit, dif, net = [], M >> 4, c["wnet"] == 1, c["net"]

            def net8(hh, o0):
                for o in range(12):
                    ll, jj = divmod(o, 4)
                    hl = (4 >> ll) if dif else (1 << ll)
                    al = (jj // hl) * 2 * hl + jj % hl
                    ops.append((0, 8 * hh + al, 8 * hh + al + hl, net[o0 + o] * unit))

            if dif:
                ops += [(0, j, j + 8, net[j] * unit) for j in range(8)]
                net8(0, 8)
                net8(1, 20)
            else:
                net8(0, 0)
                net8(1, 12)
                ops += [(0, j, j + 8, net[24 + j] * unit) for j in range(8)]
        elif c.get("net"):
            # the CTA kernel's radix-64 network (wave_wide.cuh): two stages of
            # eight 8-point networks, (stage, warp, op) -> butterfly
            for i in range(c["nload"], 64):
                slot[i] = 0
            ops, unit, dif = [], M >> 6, c["wnet"] == 1
            for st in range(2):
                for w in range(8):
                    for o in range(12):
                        ll, jj = divmod(o, 4)
                        hl = (4 >> ll) if dif else (1 << ll)
                        al = (jj // hl) * 2 * hl + jj % hl
                        strided = dif == (st == 0)
                        a, h = (w + 8 * al, 8 * hl) if strided else (8 * w + al, hl)
                        ops.append((0, a, a + h, c["net"][(st * 8 + w) * 12 + o] * unit))
        elif c.get("wnet"):
            # the warp kernel runs these as the full ADDSUB network (spans 4,2,1
            # or 1,2,4) on zero-filled truncated inputs, storing outputs < n
            for i in range(c["nload"], 8):
                slot[i] = 0
            ops = [(0, a, b, r) for (t, a, b, r) in ops]
        for (t, a, b, r) in (ops if run else []):
            assert not coset or t == 4 or r % (M >> c["ell"]) == 0
            if t == 4:
                slot[b] = slot[a]
                continue
            A, B = slot[a], (slot[b] * pow(2, r, P)) % P
            if t == 0:
                slot[a], slot[b] = (A + B) % P, (A - B) % P
            elif t == 1:
                slot[a] = (A + B) % P
            elif t == 2:
                slot[a] = (2 * A - B) % P
            elif t == 3:
                slot[a], slot[b] = (2 * A - B) % P, (A - B) % P
            else:
                raise AssertionError("negacyclic-only op in a Fermat plan")
        for i in range(c["nstore"] if run else 0):
            ea, eb = c["post"][i]
            tp = (tpost if cf_ and i == cn else 0) if inv else tpost
            e = (ea * s + eb + tp) % M
            if wplan and coset:  # whole lanes; the sub-lane rest goes to the next reader
                e = (ws[c0 + 2 * i + 1] & 0x3FFFFFFF) * lane
            assert not coset or e % lane == 0
            ob = buf(locoff, i, True)
            if coset and i < c["nload"]:
                assert ob != buf(locoff, i, False), "a coset leaf must not write the buffer it reads"
            x[(ob, base + i * stride)] = (slot[i] * pow(2, e, P)) % P
        k = comp
        while k >= 0:  # leaf -> phase counter -> (node finished) -> parent phase ...
            counters[k] += 1
            tgt, nxt = meta[k]
            if counters[k] != tgt:
                break
            k = nxt
    shadow = set(plan.get("shadow_finals", []))
    out = {e: x[(1 if e in shadow else 0, e)] for (b, e) in x if b == 0 or e in shadow}
    fr = plan.get("final_rot", [])
    for e, o in zip(fr[::2], fr[1::2]):  # rotations deferred past the last writer
        out[e] = (out[e] * pow(2, o, P)) % P
    return out


def check_plan(ctx, N, rnd, trials, lmin=1, lmax=8, shapes=()):
    """Random (L, z, n, s, policy) TFTs + ITFTs, then the given ITFT shapes
    (L, z, n2, f): emulated plan vs the definition."""
    fm = bm.FermatModel(N)
    todo = [None] * trials + list(shapes)
    for shape in todo:
        if shape is None:
            L = 1 << rnd.randint(lmin, lmax)
            z, n = rnd.randint(1, L), rnd.randint(1, L)
            n2, f = rnd.randint(0, z), rnd.randint(0, 1)
        else:
            L, z, n2, f = shape
            n = z
        s, pol = rnd.randrange(2 * N), rnd.randint(0, 1)
        a = [rnd.randrange((1 << N) + 1) for _ in range(z)]
        want = fm.dft(L, s, a)
        plan = cf.plan_dump(ctx, False, cf.TransformParams(L, s, z, n), pol)
        x = run_plan_fermat(plan, N, {i: a[i] for i in range(z)})
        assert [x[i] for i in range(n)] == want[:n], (N, L, z, n, s, pol)
        if not 1 <= n2 + f <= L:
            continue
        vals = {i: want[i] for i in range(n2)}
        vals.update({i: (L * a[i]) % fm.P for i in range(n2, z)})
        plan = cf.plan_dump(ctx, True, cf.TransformParams(L, s, z, n2, f), pol)
        x = run_plan_fermat(plan, N, vals)
        assert [x[i] for i in range(n2)] == [(L * a[i]) % fm.P for i in range(n2)]
        if f:
            assert x[n2] == want[n2]


@pytest.mark.parametrize("limit", [0, 1, 2, 3])
def test_gpu_schedule_reproduces_definition(limit):
    rnd = random.Random(limit)
    for N in (128, 256):
        ctx = cf.FermatRingCtx(N)
        ctx.set_leaf_limit(limit)
        check_plan(ctx, N, rnd, 40)


def test_wide_schedule_reproduces_definition():
    """Radix-64 coset leaves: the reshaped top split, the full 64-point
    networks (incl. truncated TFT leaves on zero-filled inputs) and the
    generic 64-slot programs (truncated ITFT leaves with their sub-unit
    offsets realigned, run as phase programs on the TMA kernel)."""
    rnd = random.Random(7)
    N = 32768
    ctx = cf.FermatRingCtx(N)
    ctx.set_wide(1)
    seen = set()
    for _ in range(14):
        L = 1 << rnd.randint(6, 9)
        z, n = rnd.randint(1, L), rnd.randint(1, L)
        s, pol = rnd.randrange(2 * N), rnd.randint(0, 1)
        for inv in (False, True):
            plan = cf.plan_dump(ctx, inv, cf.TransformParams(L, s, z, n if not inv else min(n, z)), pol)
            for c in plan["classes"]:
                if c["kind"] == 1 and c["ell"] >= 4:
                    seen.add("net" if c.get("net") else "generic")
    # truncated 64-point ITFT leaves that become phase programs
    check_plan(ctx, N, random.Random(8), 2, 6, 7, shapes=[(64, 33, 30, 0), (64, 49, 49, 0), (64, 48, 48, 1)])
    assert seen == {"net", "generic"}, seen


@pytest.mark.parametrize("limit", [0, 2, 3])
def test_coset_schedule_reproduces_definition(limit):
    """Coset leaves: factored nodes (zeta taken out), lane-aligned leaves as
    coset tickets, boundary leaves with their extra rotations."""
    rnd = random.Random(100 + limit)
    for N, cw in ((512, 4), (1024, 4), (2048, 8)):
        ctx = cf.FermatRingCtx(N)
        ctx.set_coset(cw)
        ctx.set_leaf_limit(limit)
        check_plan(ctx, N, rnd, 25)


def test_schedule_shape_config5():
    """C5 (L=2^18, z=n=200000): top split 512x512, SMEM leaves of 8 -> three
    levels per top-level pass; only columns < z2' and rows < n1' are scheduled;
    the ticket list is L2-batched (whole columns, level by level)."""
    ctx = cf.FermatRingCtx(131072)
    ctx.set_coset(0)
    assert ctx.set_leaf_limit(0) == 3
    plan = cf.plan_dump(ctx, False, cf.TransformParams(1 << 18, 0, 200000, 200000))
    leaves = plan["leaves"]
    # columns: 64 inner columns + 6 full row-64 nodes (16 leaves) + a partial
    # one (9); rows: 390 full rows (192 leaves) + the partial row n2=320 (144)
    assert len(leaves) == 512 * (64 + 6 * 16 + 9) + 390 * 192 + 144
    assert max(lf[7] for lf in leaves) == 2  # waves 0..2 within each top-level child
    assert sum(1 for lf in leaves if lf[4] < 0) == 512 * 64  # only the first level is free
    first = leaves[:64]
    assert all(lf[7] == 0 and lf[2] == 512 * 64 for lf in first)
    # within the first batch, level-1 leaves precede level-2 leaves
    per_col = 64 + 6 * 16 + 9
    batch = (512 << 20) // (512 * ctx.element_bytes)  # columns per ticket-order batch (512 MiB budget)
    waves = [lf[7] for lf in leaves[: batch * per_col]]
    assert waves == sorted(waves) and waves[0] == 0 and waves[-1] == 2
    assert leaves[batch * per_col][7] == 0  # the next batch restarts at level 1


def test_linear_form_and_doubling_leaves():
    """One-output ITFT leaves whose halvings make op rotations sub-lane run in
    their linear form (inputs pre-rotated by any bits, aligned adds) as coset
    leaves; other such leaves are realigned (Planner::realign: sub-unit
    offsets taken by the loads, doublings turned into rotations where the
    chain needs it, final offsets deferred to the fold).  The plans are
    evaluated against the transform's definition, deferred rotations included."""
    N = 2048
    ctx = cf.FermatRingCtx(N)
    ctx.set_coset(8)
    fm = bm.FermatModel(N)
    rnd = random.Random(21)
    seen_linear = 0
    for L, z, n, f in ((64, 64, 1, 0), (64, 50, 33, 0), (128, 100, 65, 1), (256, 256, 129, 0)):
        s = rnd.randrange(2 * N)
        a = [rnd.randrange((1 << N) + 1) for _ in range(z)]
        want = fm.dft(L, s, a)
        plan = cf.plan_dump(ctx, True, cf.TransformParams(L, s, z, n, f))
        for c in plan["classes"]:
            if c["kind"] == 1 and c["nstore"] == 1 and c["ops"] and all(t in (1, 4) and r == 0 for (t, a_, b_, r) in c["ops"]):
                seen_linear += 1
        vals = {i: want[i] for i in range(n)}
        vals.update({i: (L * a[i]) % fm.P for i in range(n, z)})
        x = run_plan_fermat(plan, N, vals)
        assert [x[i] for i in range(n)] == [(L * a[i]) % fm.P for i in range(n)]
        if f:
            assert x[n] == want[n]
    assert seen_linear > 0




def test_ring_create_ranges_and_primality():
    """Ring contexts reject what the header says they reject, before any GPU
    work: Fermat N outside [128, 2^18] or not a power of two, a composite
    prime-ring modulus (the reference's NotPrime, field.hpp:56-78), a prime
    without 2^m | p - 1."""
    for N in (64, 96, 1 << 19):
        with pytest.raises(cf.Unsupported):
            cf.FermatRingCtx(N)
    cf.FermatRingCtx(128)
    with pytest.raises(cf.InvalidParams):
        cf.PrimeRingCtx(1, 15)  # 15 = 3 * 5, odd, 2 | 14
    with pytest.raises(cf.InvalidParams):
        cf.PrimeRingCtx(2, 97 * 193)  # composite with 4 | p - 1
    with pytest.raises(cf.InvalidParams):
        cf.PrimeRingCtx(4, 7)  # prime, 16 does not divide 6
    assert cf.PrimeRingCtx(4, 97).root_order() == 16


def test_regauged_stage_b_equals_the_plain_network():
    """Stage B of the radix-64 kernel reads its slots re-gauged (wave_tma.cuh,
    net8_g): slot j as 2^(g_j unit) * slot j, seven butterflies without any
    rotation, five with a residual one.  With the planner's gauges and
    residuals (plan_dump's net_g) that must be the plain network -- 12
    butterflies (a, b) <- (a + 2^(q unit) b, a - 2^(q unit) b) -- output for
    output, over Z/(2^N+1), for every stage-B network of every radix-64 class
    of the C2- and C5-shaped plans."""
    rnd = random.Random(77)
    rot_dif, rot_dit = {6, 7, 9, 10, 11}, {5, 7, 9, 10, 11}
    seen = 0
    for N, L, z, n in ((32768, 1 << 16, 40000, 50001), (131072, 1 << 18, 200000, 200000)):
        ctx = cf.FermatRingCtx(N)
        P, M = (1 << N) + 1, 2 * N
        unit = M >> 6
        for inv in (False, True):
            prm = cf.TransformParams(L, 0, max(z, n) if inv else z, n, 0) if inv else cf.TransformParams(L, 0, z, n)
            plan = cf.plan_dump(ctx, inv, prm)
            for c in plan["classes"]:
                if c["ell"] != 6 or not c.get("net_g"):
                    continue
                dif = c["wnet"] == 1
                mask = rot_dif if dif else rot_dit
                for w in range(8):
                    q = c["net"][(8 + w) * 12: (9 + w) * 12]
                    gr = c["net_g"][w * 12: (w + 1) * 12]
                    x = [rnd.randrange(P) for _ in range(8)]
                    y = [(x[j] * pow(2, (gr[j][0] * unit) % M, P)) % P for j in range(8)]
                    assert gr[0][0] == 0
                    for o in range(12):
                        ll, jj = divmod(o, 4)
                        hl = (4 >> ll) if dif else (1 << ll)
                        a = (jj // hl) * 2 * hl + jj % hl
                        b = a + hl
                        xb = (x[b] * pow(2, (q[o] * unit) % M, P)) % P
                        x[a], x[b] = (x[a] + xb) % P, (x[a] - xb) % P
                        if o not in mask:
                            assert gr[o][1] == 0, "a residual rotation outside the kernel's mask"
                        yb = (y[b] * pow(2, (gr[o][1] * unit) % M, P)) % P
                        y[a], y[b] = (y[a] + yb) % P, (y[a] - yb) % P
                    assert x == y, (N, inv, w)
                    seen += 1
    assert seen >= 32
