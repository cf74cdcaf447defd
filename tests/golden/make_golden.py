"""Generates the committed golden fixtures in tests/golden/.

Run in the build container (it needs /root/reference for the prime-field
fixtures, built into oracle/_ref/libcftft_ref.so by oracle/Makefile):

    python tests/golden/make_golden.py

Outputs
  prime_cases.json   cf_tft / cf_itft of the UNMODIFIED reference
                     (RingCtx prime fields) on seeded inputs, with its
                     ButterflyStats counts
  counts.json        reference base-case counts at the five BASELINE shapes
                     (counts are data and ring independent, verify.hpp:175-176)
  bigring.npz        Fermat / negacyclic transforms evaluated from their
                     DEFINITION with Python integers (oracle/bigint_model.py),
                     including the full config-1 TFT output
"""
from __future__ import annotations

import ctypes as C
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bigint_model as bm  # noqa: E402
import pyoracle as po  # noqa: E402


def prime_cases():
    R = po.ref()
    rnd = random.Random(20081020)
    out = []
    for (p, m) in [(17, 4), (7681, 9), (po.GOLDILOCKS, 32)]:
        for _ in range(60):
            ell = rnd.randint(1, min(6, m))
            L = 1 << ell
            z = rnd.randint(1, L)
            s = rnd.randrange(1 << m)
            pol = rnd.randint(0, 1)
            inv = rnd.randint(0, 1)
            data = [rnd.randrange(p) for _ in range(L)]
            buf = np.array(data, dtype=np.uint64)
            cnt = C.c_uint64()
            if inv:
                n = rnd.randint(0, z)
                f = rnd.randint(0, 1)
                if not 1 <= n + f <= L:
                    f = 1 - f
                    if not 1 <= n + f <= L:
                        continue
                rc = R.ref_itft(p, m, L, s, z, n, f, buf.ctypes.data_as(po.U64P), L, 0, 1, pol, C.byref(cnt))
                k = n + f
            else:
                n = rnd.randint(1, L)
                f = 0
                rc = R.ref_tft(p, m, L, s, z, n, buf.ctypes.data_as(po.U64P), L, 0, 1, pol, C.byref(cnt))
                k = n
            assert rc == 0
            out.append(dict(p=p, m=m, inverse=inv, L=L, s=s, z=z, n=n, f=f, policy=pol,
                            input=data[:z], output=[int(v) for v in buf[:k]], count=cnt.value))
    return out


def counts():
    R = po.ref()
    p, m = po.GOLDILOCKS, 32
    shapes = []
    shapes.append(("C1", 0, 1 << 10, 700, 700, 0))
    shapes.append(("C1", 1, 1 << 10, 700, 700, 0))
    c2 = [32769, 40000, 49152, 65535]
    for z in c2:
        for n in c2:
            shapes.append(("C2", 0, 1 << 16, z, n, 0))
            if z >= n:
                for f in (0, 1):
                    shapes.append(("C2", 1, 1 << 16, z, n, f))
    shapes.append(("C3", 0, 1 << 11, 1024, 2047, 0))
    shapes.append(("C3", 1, 1 << 11, 2047, 2047, 0))
    shapes.append(("C4", 0, 1 << 17, 60000, 119999, 0))
    shapes.append(("C4", 1, 1 << 17, 119999, 119999, 0))
    shapes.append(("C5", 0, 1 << 18, 200000, 200000, 0))
    shapes.append(("C5", 1, 1 << 18, 200000, 200000, 0))
    out = []
    for (cfg, inv, L, z, n, f) in shapes:
        for pol in (0, 1):
            buf = np.zeros(L, dtype=np.uint64)
            cnt = C.c_uint64()
            if inv:
                rc = R.ref_itft(p, m, L, 0, z, n, f, buf.ctypes.data_as(po.U64P), L, 0, 1, pol, C.byref(cnt))
            else:
                rc = R.ref_tft(p, m, L, 0, z, n, buf.ctypes.data_as(po.U64P), L, 0, 1, pol, C.byref(cnt))
            assert rc == 0
            out.append(dict(config=cfg, inverse=inv, L=L, z=z, n=n, f=f, policy=pol, count=cnt.value))
    return out


def bigring():
    arrays = {}
    meta = []
    rnd = random.Random(7)
    # small Fermat cases, TFT and ITFT, from the definition
    for N in (128, 256):
        fm = bm.FermatModel(N)
        for c in range(12):
            L = 1 << rnd.randint(1, 7)
            z = rnd.randint(1, L)
            n = rnd.randint(1, L)
            s = rnd.randrange(2 * N)
            a = [rnd.randrange((1 << N) + 1) for _ in range(z)]
            if c == 0:
                a[0] = 1 << N
            spec = fm.dft(L, s, a)
            key = f"fermat_{N}_{c}"
            arrays[key + "_in"] = np.stack([fm.to_words(v) for v in a])
            arrays[key + "_tft"] = np.stack([fm.to_words(v) for v in spec[:n]])
            n2 = rnd.randint(0, z)
            f = 1 if n2 == 0 else rnd.randint(0, 1)
            if n2 + f > L:
                f = 0
            itin = spec[:n2] + [(L * a[i]) % fm.P for i in range(n2, z)]
            itout = [(L * a[i]) % fm.P for i in range(n2)] + ([spec[n2]] if f else [])
            arrays[key + "_itin"] = np.stack([fm.to_words(v) for v in itin])
            arrays[key + "_itout"] = (np.stack([fm.to_words(v) for v in itout]) if itout
                                      else np.zeros((0, fm.words), np.uint64))
            meta.append(dict(key=key, ring="fermat", N=N, L=L, z=z, n=n, s=s, n2=n2, f=f))
    # small negacyclic cases
    for (K, m) in [(8, 97), (16, (1 << 61) + 15)]:
        nm = bm.NegacyclicModel(K, m)
        for c in range(8):
            L = 1 << rnd.randint(1, min(5, (2 * K).bit_length() - 1))
            z = rnd.randint(1, L)
            n = rnd.randint(1, L)
            s = rnd.randrange(2 * K)
            a = [[rnd.randrange(m) for _ in range(K)] for _ in range(z)]
            spec = nm.dft(L, s, a)
            key = f"nega_{K}_{c}"
            arrays[key + "_in"] = np.array(a, dtype=np.uint64)
            arrays[key + "_tft"] = np.array(spec[:n], dtype=np.uint64)
            meta.append(dict(key=key, ring="negacyclic", K=K, m=m, L=L, z=z, n=n, s=s))
    # config 1: the full TFT output from the definition (seed mix_seed(42, 1))
    N, L, z = 1024, 1024, 700
    fm = bm.FermatModel(N)
    rng = np.random.default_rng(po.mix_seed(42, 1))
    limbs = rng.integers(0, 1 << 64, size=(z, N // 64), dtype=np.uint64, endpoint=False)
    a = [fm.from_words(np.concatenate([limbs[i], np.zeros(1, np.uint64)])) for i in range(z)]
    ell = 10
    out = []
    P = fm.P
    for j in range(z):
        jr = bm.bitrev(j, ell)
        acc = 0
        for i in range(z):
            e = (2 * i * jr) % (2 * N)  # omega_L = 2^(2N/L) = 2^2
            acc += (a[i] << e) if e < N else -(a[i] << (e - N))
        out.append(acc % P)
    arrays["c1_tft"] = np.stack([fm.to_words(v) for v in out])
    meta.append(dict(key="c1", ring="fermat", N=N, L=L, z=z, n=z, s=0, seed="mix_seed(42,1)"))
    return arrays, meta


def main():
    po.build()
    with open(os.path.join(HERE, "prime_cases.json"), "w") as fh:
        json.dump(prime_cases(), fh)
    with open(os.path.join(HERE, "counts.json"), "w") as fh:
        json.dump(counts(), fh, indent=0)
    arrays, meta = bigring()
    np.savez_compressed(os.path.join(HERE, "bigring.npz"), **arrays)
    with open(os.path.join(HERE, "bigring.json"), "w") as fh:
        json.dump(meta, fh, indent=0)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
