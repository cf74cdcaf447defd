#!/usr/bin/env python
"""bench.py -- TFT+ITFT throughput (GB/s) on B200, against the host-CPU oracle.

Default workload (BASELINE.json config 5, the metric's 1/2/4/8-GPU config):
  R = Z/(2^131072+1) (16 KiB coefficients), L = 2^18, z = n = 200000, s = 0;
  one step = cf_tft (z, n) followed by cf_itft (z = n, f = 0) in place: the
  round trip over ~3.3 GB of coefficients (far larger than the 126 MB L2, so
  no L2 flush is needed between steps).

Metric: GB/s = (TFT bytes + ITFT bytes) / (TFT time + ITFT time), with the
ALGORITHMIC bytes of a two-pass Bailey decomposition at the top-level split
(SURVEY.md §8d):
  TFT  bytes = B (z + 2 n1' z2' + n)
  ITFT bytes = B [2 n1 L2 + sum_{u in [n2,z2')} (r(u) + n1 + f') + f'(z2' + n2 + f)
                  + sum_{u < n2} (r(u) + n1 + 1)],   r(u) = z1 + [u < z2]
  B = N/8 information bytes per coefficient.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                       [--config C1|C2|C4|C5] [--no-cpu] [--no-e2e]
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (N bits, L, z, n, description)
    "C1": (1024, 1 << 10, 700, 700, "Z/(2^1024+1), L=2^10, z=n=700"),
    "C2": (32768, 1 << 16, 65535, 65535, "Z/(2^32768+1), L=2^16, z=n=65535 (largest C2 pair)"),
    "C4": (65536, 1 << 17, 119999, 119999, "Z/(2^65536+1), L=2^17, z=n=119999 (C4 ITFT shape)"),
    "C5": (131072, 1 << 18, 200000, 200000, "Z/(2^131072+1), L=2^18, z=n=200000"),
}


# ---------------------------------------------------------------------------
def split(ell: int, policy: int = 0):
    return (1, ell - 1) if policy else (ell // 2, ell - ell // 2)


def tft_bytes(N: int, L: int, z: int, n: int) -> int:
    B = N // 8
    ell = L.bit_length() - 1
    l1, l2 = split(ell)
    cols = 1 << l2
    n2, n1 = n & (cols - 1), n >> l2
    n1c = n1 + (1 if n2 else 0)
    z2, z1 = z & (cols - 1), z >> l2
    z2e = cols if z1 else z2
    return B * (z + 2 * n1c * z2e + n)


def itft_bytes(N: int, L: int, z: int, n: int, f: int) -> int:
    B = N // 8
    ell = L.bit_length() - 1
    l1, l2 = split(ell)
    cols = 1 << l2
    n2, n1 = n & (cols - 1), n >> l2
    z2, z1 = z & (cols - 1), z >> l2
    fm = 1 if n2 + f > 0 else 0
    z2e = cols if z1 else z2

    def r(u):
        return z1 + (1 if u < z2 else 0)

    tot = 2 * n1 * cols
    tot += sum(r(u) + n1 + fm for u in range(n2, z2e))
    tot += fm * (z2e + n2 + f)
    tot += sum(r(u) + n1 + 1 for u in range(n2))
    return B * tot


def hbm_peak():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        try:
            with open(p) as fh:
                return float(json.load(fh)["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def load_traffic(cfg: str):
    """The committed ncu DRAM traffic of a config (tools/traffic.py), only when
    it was measured on a build of these very sources (sha256 over csrc/ and
    include/: the .so bytes themselves differ from one nvcc run to the next)."""
    from paper_0810_3203_b200._build import source_sha256

    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            t = json.load(fh).get(cfg)
        if not isinstance(t, dict):
            return None, "no ncu traffic for this config"
        if source_sha256() != t.get("source_sha256"):
            return None, "profiles/traffic.json is from other library sources (stale): not reported"
        return t, "ncu dram__bytes_read.sum + dram__bytes_write.sum, these sources (profiles/traffic.json)"
    except Exception:
        return None, "no profiles/traffic.json"


def kernel_roofline(records, steps, peak):
    """Per kernel name: launches, ms and algorithmic GB/s per step from the
    library's launch timing (CUDA events on the launching stream, inside the
    timed region); the dominant kernel is the one with the most time."""
    agg = {}
    for name, byts, ms in records:
        a = agg.setdefault(name, [0, 0, 0.0])
        a[0] += 1
        a[1] += byts
        a[2] += ms
    table = {name: {"launches_per_step": c / steps, "ms_per_step": ms / steps,
                    "algorithmic_bytes_per_launch": b / c, "gbs": b / (ms / 1e3) / 1e9 if ms else None,
                    "frac": (b / (ms / 1e3) / 1e9) / peak if ms else None}
             for name, (c, b, ms) in agg.items()}
    dom = max(table, key=lambda k: table[k]["ms_per_step"]) if table else None
    return dom, table


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.lo, self.hi = 0, None

    # started before the warm-up (nvidia-smi's start-up perturbs the GPU);
    # only the samples between begin() and end() are reported
    def begin(self):
        self.lo = len(self.rows)

    def end(self):
        time.sleep(0.12)
        self.hi = len(self.rows)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = self.rows[self.lo:self.hi] if self.hi is not None and self.hi > self.lo else self.rows[self.lo:]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return os.cpu_count() or 1, model


def make_input(N: int, L: int, z: int, W: int, seed: int):
    import numpy as np

    rng = np.random.default_rng(seed)
    buf = np.zeros((L, W), dtype=np.uint64)
    lim = N // 64
    step = 8192
    for i in range(0, z, step):
        k = min(step, z - i)
        buf[i:i + k, :lim] = rng.integers(0, 1 << 64, size=(k, lim), dtype=np.uint64, endpoint=False)
    return buf


def bailey_phases(M: int, L: int, z: int, n: int, f: int, inverse: bool, s: int = 0, policy: int = 0):
    """The top-level Bailey sub-transforms of one TFT / ITFT over a row-major
    (L, W) buffer, phase by phase (transform.hpp:175-185 and 215-238): lists of
    (L_sub, s_sub, z_sub, n_sub, f_sub, base, stride) in element units.  Each
    sub-transform reads z_sub and writes n_sub + f_sub coefficients, so the
    algorithmic bytes of a phase are B * sum(z_sub + n_sub + f_sub)."""
    ell = L.bit_length() - 1
    l1, l2 = split(ell, policy)
    L1, L2 = 1 << l1, 1 << l2
    cs = M >> ell
    s_row = (s << l1) % M
    n2, n1 = n & (L2 - 1), n >> l2
    z2, z1 = z & (L2 - 1), z >> l2
    z2e = L2 if z1 else z2
    if not inverse:
        n1c = n1 + (1 if n2 else 0)
        cols = [(L1, s + u * cs, z1 + 1 if u < z2 else z1, n1c, 0, u, L2) for u in range(z2e)]
        rows = [(L2, s_row, z2e, L2 if u < n1 else n2, 0, u * L2, 1) for u in range(n1c)]
        return [("tft-columns", False, cols), ("tft-rows", False, rows)]
    fm = 1 if n2 + f > 0 else 0
    lo, hi = min(n2, z2), max(n2, z2)
    ph = [("itft-i", True, [(L2, s_row, L2, L2, 0, u * L2, 1) for u in range(n1)]),
          ("itft-ii", True, [(L1, s + u * cs, z1 + 1 if u < hi else z1, n1, fm, u, L2) for u in range(n2, z2e)])]
    if fm:
        ph.append(("itft-iii", True, [(L2, s_row, z2e, n2, f, n1 * L2, 1)]))
    ph.append(("itft-iv", True, [(L1, s + u * cs, z1 + 1 if u < lo else z1, n1 + 1, 0, u, L2) for u in range(n2)]))
    return ph


def cpu_sample_round_trip(N, L, z, n, buf, threads, every):
    """The oracle port (oracle/cftft_oracle.c) on the host cores: every
    `every`-th top-level Bailey sub-transform of the TFT (z, n) and of the ITFT
    (n, n, 0), in place on the full buffer, each phase spread over `threads`
    host threads.  Returns (seconds, algorithmic bytes) of the sample."""
    from concurrent.futures import ThreadPoolExecutor

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    ring = po.Ring.fermat(N)
    B = N // 8
    secs, byts = 0.0, 0
    phases = bailey_phases(2 * N, L, z, n, 0, False) + bailey_phases(2 * N, L, n, n, 0, True)
    with ThreadPoolExecutor(threads) as ex:
        for _, inverse, subs in phases:
            pick = subs[::every]
            byts += B * sum(zs + ns + fs for (_, _, zs, ns, fs, _, _) in pick)

            def run(t):
                Ls, ss, zs, ns, fs, base, stride = t
                if inverse:
                    ring.itft_at(buf, base, stride, Ls, ss, zs, ns, fs)
                else:
                    ring.tft_at(buf, base, stride, Ls, ss, zs, ns)

            t0 = time.perf_counter()
            list(ex.map(run, pick))
            secs += time.perf_counter() - t0
    return secs, byts


CPU_SAMPLE_EVERY = 8  # 1/8 of the sub-transforms: ~2 s per step on 8 cores at C5
CPU_SAMPLE_EVERY_1T = 64  # single-thread sample: 1/64 of the sub-transforms


def cpu0_reference(L: int, z: int, n: int):
    """SURVEY.md §8d CPU-0 (context only): the unmodified reference cf_tft /
    cf_itft (oracle/_ref, built from /root/reference/proj/include) over its own
    Goldilocks ring at the same (L, z, n) on one core; GB/s with its 8-byte
    coefficients.  None when oracle/_ref is absent."""
    import ctypes as C

    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    if not po.ref_available():
        return None
    P, m = 0xFFFFFFFF00000001, 32
    rng = np.random.default_rng(po.mix_seed(42, 7))
    buf = np.zeros(L, dtype=np.uint64)
    buf[:z] = rng.integers(0, P, size=z, dtype=np.uint64)
    ptr = buf.ctypes.data_as(po.U64P)
    c = C.c_uint64(0)
    t = time.perf_counter()
    po.ref().ref_tft(P, m, L, 0, z, n, ptr, L, 0, 1, 0, C.byref(c))
    po.ref().ref_itft(P, m, L, 0, n, n, 0, ptr, L, 0, 1, 0, C.byref(c))
    secs = time.perf_counter() - t
    byts = tft_bytes(64, L, z, n) + itft_bytes(64, L, n, n, 0)
    return {"value": byts / secs / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference", "seconds": secs,
            "sample": f"the whole TFT+ITFT over Z/pZ (p = 2^64 - 2^32 + 1), L={L}, z=n={z}: a different ring "
                      "(8-byte coefficients), context only"}


# ---------------------------------------------------------------------------
def run_reference(args, cfgname):
    """--impl reference: the CPU implementation of the path on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N, L, z, n, desc = CONFIGS[cfgname]
    threads, model = cpu_info()
    W = N // 64 + 2
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    po.build()
    buf = make_input(N, L, z, W, po.mix_seed(42, 5))
    times, byts = [], 0
    for i in range(args.warmup + args.steps):
        secs, byts = cpu_sample_round_trip(N, L, z, n, buf, threads, CPU_SAMPLE_EVERY)
        if i >= args.warmup:
            times.append(secs)
    tot = sum(times)
    gbs = byts * len(times) / tot / 1e9
    sample = (f"every {CPU_SAMPLE_EVERY}th top-level Bailey sub-transform of the {cfgname} TFT and ITFT "
              f"({byts / 1e9:.2f} GB algorithmic per step), in place on the full seeded buffer, on "
              f"{threads} host threads ({model}); oracle/cftft_oracle.c (the reference's recursion "
              f"restated over Z/(2^N+1): the reference implements no Fermat ring, SPEC.md:13)")
    line = {
        "impl": "reference",
        "metric": f"TFT+ITFT GB/s ({cfgname}: {desc})",
        "value": gbs, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": cfgname, "ring": f"Z/(2^{N}+1)", "L": L, "z": z, "n": n},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_distributed(args, cf, po, dist, ctx, N, L, z, n, desc, rank, world, local):
    """N GPUs: one config-5 transform partitioned over the ranks (column slabs
    -> NCCL all-to-all -> row slabs).  Strong scaling."""
    import numpy as np
    import torch

    from paper_0810_3203_b200.dist import DistGeometry, NcclDist

    W = ctx.element_words
    M = 2 * N
    # the library's native partition (cftft_gpu_dist_tft / _itft over its own
    # NCCL communicator); DistGeometry gives the same slabs for the NVLink count
    nd = NcclDist(ctx)
    pt, pi = cf.TransformParams(L, 0, z, n), cf.TransformParams(L, 0, n, n, 0)
    geo_f, geo_i = nd.geometry(pt), nd.geometry(pi, inverse=True)
    g = DistGeometry(M, L, z, n, world, l1=int(geo_f["L1"]).bit_length() - 1)
    rows_local = geo_f["col_elems"]
    # this rank's column slab: seeded uniform limbs in rows < z1 + 1 (inputs)
    rng = np.random.default_rng(po.mix_seed(42, 5 + rank))
    host = np.zeros((rows_local, W), dtype=np.uint64)
    wdt = geo_f["c1"] - geo_f["c0"]
    live = min(rows_local, (g.z1 + 1) * wdt)
    host[:live, : N // 64] = rng.integers(0, 1 << 64, size=(live, N // 64), dtype=np.uint64, endpoint=False)
    col = torch.from_numpy(host.view(np.int64)).cuda()
    rowslab = torch.empty((max(geo_f["row_elems"], geo_i["row_elems"]), W), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    byts = tft_bytes(N, L, z, n) + itft_bytes(N, L, n, n, 0)

    class _Count:
        launches = 0

    eng = _Count()

    def barrier():
        dist.barrier()
        torch.cuda.synchronize()

    def step(c=None):
        c = col if c is None else c
        nd.tft(pt, c, rowslab, stream=stream)
        nd.itft(pi, rowslab, c, stream=stream)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = eng.launches
    barrier()
    sampler.begin()
    cf.launch_timing_read()
    cf.set_launch_timing(True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    cf.set_launch_timing(False)
    timed = cf.launch_timing_read()
    sampler.end()
    clocks = sampler.stop()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = t.item()
    value = byts * args.steps / (total_ms / 1e3) / 1e9
    peak, peak_kind = hbm_peak()
    # bytes this rank sends over NVLink per step (the two transposes + phase iii)
    elem = ctx.element_bytes
    xfer = (g.nrows(rank) * g.width(rank) * (world - 1) + g.zrows * g.width(rank) * (world - 1) // world) * elem
    e2e = None
    if not args.no_e2e:
        pin = torch.from_numpy(host.view(np.int64)).pin_memory()
        pout = torch.empty_like(pin).pin_memory()
        # a stream of independent transforms, triple buffered as in the
        # single-GPU leg: step k's host->device copy of this rank's column slab
        # (its own stream) overlaps step k-1's transforms (and transposes) and
        # step k-2's device->host copy (a third stream)
        NB = 3
        cols = [col] + [torch.empty_like(col) for _ in range(NB - 1)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ek = max(8, args.steps)
        ev_in = [torch.cuda.Event() for _ in range(ek)]
        ev_done = [torch.cuda.Event() for _ in range(ek)]
        ev_out = [torch.cuda.Event() for _ in range(ek)]
        barrier()
        t0 = time.perf_counter()
        for k in range(ek):
            b = k % NB
            with torch.cuda.stream(s_in):
                if k >= NB:
                    s_in.wait_event(ev_out[k - NB])  # slab b is free again
                cols[b].copy_(pin, non_blocking=True)
                ev_in[k].record(s_in)
            stream.wait_event(ev_in[k])
            step(cols[b])
            ev_done[k].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[k])
                pout.copy_(cols[b], non_blocking=True)
                ev_out[k].record(s_out)
        torch.cuda.synchronize()
        barrier()
        tt = torch.tensor([(time.perf_counter() - t0) / ek], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        del cols[1:]
        e2e = {"value": byts / tt.item() / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(pin.numel() * 8),
               "d2h_bytes_per_step": int(pout.numel() * 8), "steps": ek,
               "note": "per rank: pinned column slab in, round trip (transforms + NVLink transposes), column slab "
                       "out; triple-buffered streams overlap consecutive steps"}
    if rank == 0:
        dom, table = kernel_roofline(timed, args.steps, peak)
        dk = table.get(dom, {})
        roofline = {
            "bound": "hbm", "kernel": dom, "achieved": dk.get("gbs"), "peak": peak, "unit": "GB/s",
            "frac": dk.get("frac"), "peak_kind": peak_kind, "traffic": None,
            "traffic_note": "no ncu capture of the multi-rank path (ncu runs one GPU, one rank)",
            "algorithmic_bytes_per_launch": dk.get("algorithmic_bytes_per_launch"),
            "kernel_ms_per_step": dk.get("ms_per_step"), "launches_per_step": dk.get("launches_per_step"),
            "kernel_share_of_step": dk.get("ms_per_step", 0) / (total_ms / args.steps) if dk else None,
            "per": "GPU (rank 0's launches)",
            "step": {"achieved": value / world, "frac": value / world / peak},
            "nvlink_bytes_per_gpu_per_step": xfer,
            "nvlink_gbs_per_gpu": xfer / (total_ms / args.steps / 1e3) / 1e9,
            "nvlink_peak_gbs": 900.0,
            "kernels": table,
        }
        line = {
            "metric": f"TFT+ITFT GB/s ({args.config}: {desc})",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: seeded uniform 64-bit limbs per rank slab (numpy PCG64)",
            "config": {"workload": args.config, "ring": f"Z/(2^{N}+1)", "L": L, "z": z, "n": n,
                       "coeff_bytes": N // 8, "algorithmic_bytes_per_step": byts,
                       "parallelism": f"column/row slabs over {world} GPUs, NCCL transposes (cftft_gpu_dist_tft/_itft)",
                       "l2": "inputs far exceed L2"},
            "roofline": roofline,
            "cpu_baseline": None,
            "e2e": e2e,
            "gpu_launches": len(timed) + 2 * args.steps,  # transform kernels (timed) + the pack / unpack kernels
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


PRIME_CONFIG = ("G", 1 << 22, 3_000_000, "Z/pZ Goldilocks (the reference's own ring), L=2^22, z=n=3000000")


def run_prime(args) -> None:
    """--config G: the reference's own ring (RingCtx(p, m), Goldilocks) on the
    GPU, against the UNMODIFIED reference cf_tft / cf_itft (oracle/_ref, one
    host core) -- not a BASELINE config; a same-ring comparison with the
    reference itself.  Rank 0 only (other ranks exit)."""
    import ctypes as C

    import numpy as np

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    if int(os.environ.get("RANK", "0")) != 0:
        return
    name, L, z, desc = PRIME_CONFIG
    n = z
    P, m = 0xFFFFFFFF00000001, 32
    byts = tft_bytes(64, L, z, n) + itft_bytes(64, L, n, n, 0)  # 8 bytes per coefficient
    rng = np.random.default_rng(po.mix_seed(42, 7))
    host = np.zeros((L, 1), dtype=np.uint64)
    host[:z, 0] = rng.integers(0, P, size=z, dtype=np.uint64)

    def reference_once():
        buf = np.ascontiguousarray(host.copy())
        ptr = buf.ctypes.data_as(po.U64P)
        c = C.c_uint64(0)
        t = time.perf_counter()
        po.ref().ref_tft(P, m, L, 0, z, n, ptr, L, 0, 1, 0, C.byref(c))
        po.ref().ref_itft(P, m, L, 0, n, n, 0, ptr, L, 0, 1, 0, C.byref(c))
        return time.perf_counter() - t

    def oracle_once():
        ring = po.Ring.prime(P, m)
        buf = host.copy()
        t = time.perf_counter()
        ring.tft(buf, L, 0, z, n)
        ring.itft(buf, L, 0, n, n, 0)
        return time.perf_counter() - t

    kind = "reference" if po.ref_available() else "port"
    cpu_once = reference_once if kind == "reference" else oracle_once
    sample = ("the whole TFT+ITFT, unmodified reference cf_tft/cf_itft (oracle/_ref, built from "
              "/root/reference/proj/include) on 1 host core" if kind == "reference"
              else "the whole TFT+ITFT, oracle port on 1 host core (oracle/_ref absent)")
    common = {"unit": "GB/s", "n_gpus": 1, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
              "dtype": "u64", "data": "synthetic: seeded uniform residues mod p (numpy PCG64)",
              "metric": f"TFT+ITFT GB/s ({name}: {desc})"}
    cfg = {"workload": name, "ring": "Z/pZ, p = 2^64 - 2^32 + 1, omega of order 2^32", "L": L, "z": z, "n": n,
           "coeff_bytes": 8, "algorithmic_bytes_per_step": byts, "parallelism": "single GPU",
           "l2": "inputs 24 MB: L2-resident between steps (no flush); see DESIGN.md"}
    if args.impl == "reference":
        for _ in range(args.warmup):
            cpu_once()
        ts = [cpu_once() for _ in range(max(1, args.steps))]
        v = byts * len(ts) / sum(ts) / 1e9
        print(json.dumps({"impl": "reference", **common, "value": v, "steps": len(ts), "warmup": args.warmup,
                          "ms_per_step": 1e3 * sum(ts) / len(ts), "config": cfg,
                          "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": kind, "sample": sample},
                          "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch

    import paper_0810_3203_b200 as cf

    ctx = cf.PrimeRingCtx(m, P)
    dev = torch.from_numpy(host.view(np.int64)).cuda()
    view = cf.DeviceView(dev)
    pt, pi = cf.TransformParams(L, 0, z, n), cf.TransformParams(L, 0, n, n, 0)
    for _ in range(max(3, args.warmup)):
        cf.cf_tft(ctx, pt, view)
        cf.cf_itft(ctx, pi, view)
    sampler = ClockSampler(0)
    sampler.start()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    sampler.begin()
    e[0].record()
    launches = 0
    for _ in range(args.steps):
        cf.cf_tft(ctx, pt, view)
        launches += cf.last_launch_count()
        e[1].record()
        cf.cf_itft(ctx, pi, view)
        launches += cf.last_launch_count()
    e[2].record()
    torch.cuda.synchronize()
    sampler.end()
    clocks = sampler.stop()
    total = e[0].elapsed_time(e[2])
    value = byts * args.steps / (total / 1e3) / 1e9
    peak, peak_kind = hbm_peak()
    # end to end: pinned inputs in, transforms, outputs out, every step
    pin_in = torch.from_numpy(host.view(np.int64)).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ek = max(8, args.steps)
    for _ in range(ek):
        dev[:z].copy_(pin_in[:z], non_blocking=True)
        cf.cf_tft(ctx, pt, view)
        cf.cf_itft(ctx, pi, view)
        pin_out[:n].copy_(dev[:n], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / ek
    cpu = None
    if not args.no_cpu:
        cpu_once()
        ct = cpu_once()
        cpu = {"value": byts / ct / 1e9, "unit": "GB/s", "cores": 1, "kind": kind, "sample": sample}
    print(json.dumps({**common, "value": value, "steps": args.steps, "warmup": max(3, args.warmup),
                      "ms_per_step": total / args.steps, "config": cfg,
                      "roofline": {"bound": "hbm", "achieved": value, "peak": peak, "unit": "GB/s",
                                   "frac": value / peak, "peak_kind": peak_kind, "traffic": None,
                                   "kernel": "prime::leaf_kernel (all kernels of the step)"},
                      "cpu_baseline": cpu,
                      "e2e": {"value": byts / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": z * 8,
                              "d2h_bytes_per_step": n * 8, "steps": ek,
                              "note": "per step: pinned host -> HBM copy of the z inputs, TFT+ITFT, HBM -> pinned "
                                      "copy of the n outputs (serial)"},
                      "gpu_launches": launches, "clocks": clocks}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(CONFIGS) + ["G"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--leaf-limit", type=int, default=0, help="cap on-chip leaves at 2^k (tuning)")
    ap.add_argument("--force-dist", action="store_true", help="use the multi-GPU path even on 1 rank (testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    if args.config == "G":  # the reference's own ring, against the reference itself
        run_prime(args)
        return
    if args.impl == "reference":
        run_reference(args, args.config)
        return

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.force_dist:
        import torch.distributed as dist

        if world == 1 and "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_0810_3203_b200 as cf

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    N, L, z, n, desc = CONFIGS[args.config]
    ctx = cf.FermatRingCtx(N)
    if args.leaf_limit:
        ctx.set_leaf_limit(args.leaf_limit)
    W = ctx.element_words
    if world > 1 or args.force_dist:
        run_distributed(args, cf, po, dist, ctx, N, L, z, n, desc, rank, world, local)
        return
    host = make_input(N, L, z, W, po.mix_seed(42, 5 + rank))
    dev = torch.from_numpy(host.view(np.int64)).cuda()
    view = cf.DeviceView(dev)
    stream = torch.cuda.current_stream()
    pt = cf.TransformParams(L, 0, z, n)
    pi = cf.TransformParams(L, 0, n, n, 0)
    byts = tft_bytes(N, L, z, n) + itft_bytes(N, L, n, n, 0)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    host_ms = []

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        h0 = time.perf_counter()
        cf.cf_tft(ctx, pt, view, stream=stream)
        h1 = time.perf_counter()
        l1 = cf.last_launch_count()
        if evs:
            evs[1].record(stream)
        h2 = time.perf_counter()
        cf.cf_itft(ctx, pi, view, stream=stream)
        h3 = time.perf_counter()
        l2 = cf.last_launch_count()
        if evs:
            evs[2].record(stream)
        host_ms.append((round(1e3 * (h1 - h0), 2), round(1e3 * (h3 - h2), 2)))
        return l1 + l2

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    sampler.begin()
    cf.launch_timing_read()  # (drop anything logged before)
    cf.set_launch_timing(True)
    g0.record(stream)
    launches = 0
    for k in range(args.steps):
        launches += step(evs[k])
    g1.record(stream)
    barrier()
    cf.set_launch_timing(False)
    timed = cf.launch_timing_read()
    sampler.end()
    clocks = sampler.stop()
    total_ms = g0.elapsed_time(g1)
    t_tft = sum(e[0].elapsed_time(e[1]) for e in evs)
    t_itft = sum(e[1].elapsed_time(e[2]) for e in evs)
    if os.environ.get("CFTFT_BENCH_DEBUG"):
        print("per-step tft ms", [round(e[0].elapsed_time(e[1]), 2) for e in evs],
              "itft ms", [round(e[1].elapsed_time(e[2]), 2) for e in evs], "host ms (tft, itft)", host_ms,
              file=sys.stderr)
    if dist is not None:
        t = torch.tensor([total_ms, t_tft, t_itft], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, t_tft, t_itft = t.tolist()
    ms_per_step = total_ms / args.steps
    value = world * byts * args.steps / (total_ms / 1e3) / 1e9
    kernel_gbs = byts * args.steps / ((t_tft + t_itft) / 1e3) / 1e9
    peak, peak_kind = hbm_peak()

    # ---- end to end through the public API with host buffers -----------------
    e2e = None
    if not args.no_e2e:
        elem = ctx.element_bytes
        pin_in = torch.from_numpy(host.view(np.int64)).pin_memory()
        pin_out = torch.empty_like(pin_in).pin_memory()
        ek = max(16, args.steps)  # steady state: the pipeline fill and drain amortised
        # a stream of independent transforms, triple buffered: step k's
        # host->device copy (its own stream) overlaps step k-1's transforms and
        # step k-2's device->host copy (a third stream; PCIe runs both
        # directions at once); every step copies its z inputs in and its n
        # outputs out.  Three buffers keep the H2D stream busy: buffer k % 3 is
        # free once step k-3's outputs are out.
        NB = 3
        bufs = [dev] + [torch.empty_like(dev) for _ in range(NB - 1)]
        views = [view] + [cf.DeviceView(b) for b in bufs[1:]]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(ek)]
        ev_done = [torch.cuda.Event() for _ in range(ek)]
        ev_out = [torch.cuda.Event() for _ in range(ek)]
        barrier()
        t0 = time.perf_counter()
        for k in range(ek):
            b = k % NB
            with torch.cuda.stream(s_in):
                if k >= NB:
                    s_in.wait_event(ev_out[k - NB])  # buffer b is free again
                bufs[b][:z].copy_(pin_in[:z], non_blocking=True)
                ev_in[k].record(s_in)
            stream.wait_event(ev_in[k])
            cf.cf_tft(ctx, pt, views[b], stream=stream)
            cf.cf_itft(ctx, pi, views[b], stream=stream)
            ev_done[k].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_done[k])
                pin_out[:n].copy_(bufs[b][:n], non_blocking=True)
                ev_out[k].record(s_out)
        torch.cuda.synchronize()
        barrier()
        dt = (time.perf_counter() - t0) / ek
        del bufs[1:], views[1:]
        e2e = {"value": world * byts / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": z * elem,
               "d2h_bytes_per_step": n * elem, "steps": ek,
               "note": "per step: pinned host -> HBM copy of the z inputs, TFT+ITFT through the public API, "
                       "HBM -> pinned copy of the n outputs; triple-buffered streams overlap consecutive steps"}

    # ---- CPU baseline (rank 0, N=1 only) ----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads, model = cpu_info()
        po.build()
        hb = make_input(N, L, z, W, po.mix_seed(42, 5))
        secs, sb = cpu_sample_round_trip(N, L, z, n, hb, threads, CPU_SAMPLE_EVERY)
        cpu = {"value": sb / secs / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"every {CPU_SAMPLE_EVERY}th top-level Bailey sub-transform of the {args.config} "
                         f"TFT and ITFT ({sb / 1e9:.2f} GB algorithmic, {secs:.1f} s) in place on the full "
                         f"seeded buffer, oracle port on {threads} host threads, {model}"}
        # CPU-1 single thread (the reference's methodology)
        secs1, sb1 = cpu_sample_round_trip(N, L, z, n, hb, 1, CPU_SAMPLE_EVERY_1T)
        cpu["single_thread"] = {
            "value": sb1 / secs1 / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"every {CPU_SAMPLE_EVERY_1T}th top-level Bailey sub-transform ({sb1 / 1e9:.2f} GB "
                      f"algorithmic, {secs1:.1f} s), one host thread"}
        del hb
        # CPU-0 context: the UNMODIFIED reference over its own ring (Goldilocks,
        # 8-byte coefficients) at this config's (L, z, n), one core
        cpu["cpu0_reference_goldilocks"] = cpu0_reference(L, z, n)

    if rank == 0:
        dom, table = kernel_roofline(timed, args.steps, peak)
        traffic, traffic_note = load_traffic(args.config)
        dk = table.get(dom, {})
        tk = (traffic or {}).get("per_kernel", {}).get(dom, {})
        roofline = {
            "bound": "hbm", "kernel": dom, "achieved": dk.get("gbs"), "peak": peak, "unit": "GB/s",
            "frac": dk.get("frac"), "peak_kind": peak_kind,
            "traffic": tk.get("dram_bytes_per_launch"),
            "traffic_note": traffic_note,
            "algorithmic_bytes_per_launch": dk.get("algorithmic_bytes_per_launch"),
            "kernel_ms_per_step": dk.get("ms_per_step"), "launches_per_step": dk.get("launches_per_step"),
            "kernel_share_of_step": dk.get("ms_per_step", 0) / ms_per_step if dk else None,
            "ncu_share_of_step": tk.get("share_of_step"),
            "timing": "library launch timing: CUDA events around every launch on its stream, inside the timed "
                      "region; algorithmic bytes = coefficients the launch's leaves read + write x N/8",
            "step": {"achieved": kernel_gbs, "frac": kernel_gbs / peak,
                     "traffic": (traffic or {}).get("step_dram_bytes"),
                     "tft_ms": t_tft / args.steps, "itft_ms": t_itft / args.steps},
            "kernels": table,
        }
        line = {
            "metric": f"TFT+ITFT GB/s ({args.config}: {desc})",
            "value": value,
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak" if world > 1 else "strong",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic: seeded uniform 64-bit limbs (numpy PCG64, seed mix_seed(42,5+rank))",
            "config": {"workload": args.config, "ring": f"Z/(2^{N}+1)", "L": L, "z": z, "n": n,
                       "coeff_bytes": N // 8, "algorithmic_bytes_per_step": byts,
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "inputs (3.3 GB at C5) far exceed the 126 MB L2; no flush needed"
                       if args.config == "C5" else "see DESIGN.md"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
