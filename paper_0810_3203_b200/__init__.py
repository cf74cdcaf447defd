"""cftft-b200: B200-native truncated Fourier transforms over large-coefficient rings.

Host mirror of the reference library's transform API
(/root/reference/proj/include/cftft/transform.hpp), over the C ABI in
include/cftft_b200.h:

  reference (C++)                          here (Python)
  ---------------------------------------  --------------------------------------
  cftft::TransformParams  (:39-45)          TransformParams
  cftft::SplitPolicy      (:27-30)          SplitPolicy
  cftft::ButterflyStats   (:49-51)          ButterflyStats
  cftft::BadLength        (:16-20)          BadLength      (ValueError, like std::invalid_argument)
  cftft::InvalidParams    (:22-24)          InvalidParams  (ValueError)
  cftft::RingCtx          (field.hpp:84)    FermatRingCtx / NegacyclicRingCtx
  cftft::StridedView      (view.hpp:14-51)  DeviceView (device memory) / numpy views (host)
  cftft::cf_tft           (:252-264)        cf_tft(ctx, params, view, policy, stats)
  cftft::cf_itft          (:273-286)        cf_itft(ctx, params, view, policy, stats)
  cftft::bit_reverse      (:73-80)          bit_reverse
  cftft::tft_bound/itft_bound (:316-333)   tft_bound / itft_bound

The transforms always run on the GPU through libcftft_b200.so (hand-written
sm_100a kernels).  There is no CPU fallback: if the library or a GPU is
missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass

import numpy as np

from ._build import LIB as _LIB_PATH

__all__ = [
    "SplitPolicy", "TransformParams", "ButterflyStats", "BadLength", "InvalidParams",
    "CudaError", "Unsupported", "FermatRingCtx", "NegacyclicRingCtx", "DeviceView",
    "cf_tft", "cf_itft", "cf_tft_host", "cf_itft_host", "bit_reverse", "tft_bound",
    "itft_bound", "tft_base_cases", "itft_base_cases", "lib", "last_launch_count", "plan_dump", "PrimeRingCtx",
    "GOLDILOCKS",
    "scale", "set_fault_injection", "fault_injection", "set_debug_poison", "PoisonRead", "NoMemory",
    "set_launch_timing", "launch_timing_read",
]


class SplitPolicy(enum.IntEnum):
    balanced = 0  # ell1 = floor(ell/2), ell2 = ceil(ell/2)
    radix2 = 1    # ell1 = 1: the divide-and-conquer baseline


@dataclass
class TransformParams:
    length: int = 0
    twiddle_exp: int = 0
    input_count: int = 0
    output_count: int = 0
    want_next: int = 0


@dataclass
class ButterflyStats:
    base_case_count: int = 0


class BadLength(ValueError):
    pass


class InvalidParams(ValueError):
    pass


class CudaError(RuntimeError):
    pass


class Unsupported(RuntimeError):
    pass


class NoMemory(MemoryError):
    pass


class PoisonRead(AssertionError):
    """Debug poison (set_debug_poison): an output depended on a cell >= z."""


class _Params(C.Structure):
    _fields_ = [("length", C.c_uint64), ("twiddle_exp", C.c_uint64), ("input_count", C.c_uint64),
                ("output_count", C.c_uint64), ("want_next", C.c_int32)]


class _Sub(C.Structure):
    _fields_ = [("length", C.c_uint64), ("twiddle_exp", C.c_uint64), ("input_count", C.c_uint64),
                ("output_count", C.c_uint64), ("want_next", C.c_int32), ("pad", C.c_int32),
                ("base", C.c_uint64), ("stride", C.c_uint64)]


class _LaunchRec(C.Structure):
    _fields_ = [("kernel", C.c_char * 40), ("algorithmic_bytes", C.c_uint64), ("ms", C.c_float)]


_lib = None


def lib():
    """Loads libcftft_b200.so (fails loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run __graft_entry__.build() first")
        L = C.CDLL(_LIB_PATH)
        vp, u64, P = C.c_void_p, C.c_uint64, C.POINTER(_Params)
        L.cftft_ring_create.argtypes = [C.c_int, u64, u64, C.POINTER(vp)]
        L.cftft_ring_destroy.argtypes = [vp]
        L.cftft_ring_destroy.restype = None
        L.cftft_ring_root_order.argtypes = [vp]
        L.cftft_ring_root_order.restype = u64
        L.cftft_ring_element_bytes.argtypes = [vp]
        L.cftft_ring_element_bytes.restype = u64
        L.cftft_ring_set_leaf_limit.argtypes = [vp, C.c_uint]
        L.cftft_ring_set_leaf_limit.restype = C.c_uint
        L.cftft_ring_set_coset.argtypes = [vp, C.c_int]
        L.cftft_ring_set_wide.argtypes = [vp, C.c_int]
        for f in ("cftft_gpu_tft", "cftft_gpu_itft"):
            getattr(L, f).argtypes = [vp, P, vp, u64, C.c_int, C.POINTER(u64), vp]
        for f in ("cftft_tft_host", "cftft_itft_host"):
            getattr(L, f).argtypes = [vp, P, vp, u64, C.c_int, C.POINTER(u64)]
        L.cftft_gpu_pointwise.argtypes = [vp, vp, vp, u64, u64, vp]
        L.cftft_gpu_mul_scalar.argtypes = [vp, vp, u64, u64, u64, vp]
        L.cftft_gpu_batch.argtypes = [vp, C.c_int, C.POINTER(_Sub), u64, vp, u64, C.c_int, C.c_int, vp]
        L.cftft_gpu_canonicalize.argtypes = [vp, vp, u64, u64, vp]
        L.cftft_gpu_scale.argtypes = [vp, vp, u64, u64, u64, vp]
        L.cftft_tft_base_cases.argtypes = [u64, u64, u64, C.c_int]
        L.cftft_tft_base_cases.restype = u64
        L.cftft_itft_base_cases.argtypes = [u64, u64, u64, C.c_int, C.c_int]
        L.cftft_itft_base_cases.restype = u64
        L.cftft_last_launch_count.restype = u64
        L.cftft_plan_dump.argtypes = [vp, C.c_int, P, C.c_int, C.c_char_p, C.c_size_t]
        L.cftft_plan_dump.restype = C.c_size_t
        L.cftft_last_error.restype = C.c_char_p
        L.cftft_version.restype = C.c_char_p
        L.cftft_set_fault_injection.argtypes = [C.c_int]
        L.cftft_set_fault_injection.restype = None
        L.cftft_fault_injection.restype = C.c_int
        L.cftft_set_debug_poison.argtypes = [C.c_int]
        L.cftft_set_debug_poison.restype = None
        L.cftft_set_launch_timing.argtypes = [C.c_int]
        L.cftft_set_launch_timing.restype = None
        L.cftft_launch_timing_read.argtypes = [C.POINTER(_LaunchRec), u64]
        L.cftft_launch_timing_read.restype = u64
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().cftft_last_error().decode()
    raise {1: BadLength, 2: InvalidParams, 3: CudaError, 4: Unsupported, 5: NoMemory,
           6: PoisonRead}.get(rc, RuntimeError)(msg)


class _Ring:
    kind = 0

    def __init__(self, n_or_k: int, modulus: int = 0):
        h = C.c_void_p()
        _check(lib().cftft_ring_create(self.kind, n_or_k, modulus, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.cftft_ring_destroy(h)
            self._h = None

    def root_order(self) -> int:
        return lib().cftft_ring_root_order(self._h)

    def set_leaf_limit(self, max_ell: int) -> int:
        """Caps on-chip leaves at 2^max_ell coefficients (0 = default)."""
        return lib().cftft_ring_set_leaf_limit(self._h, max_ell)

    @property
    def element_bytes(self) -> int:
        """Minimal (16-byte aligned) element stride in bytes."""
        return lib().cftft_ring_element_bytes(self._h)

    @property
    def element_words(self) -> int:
        return self.element_bytes // 8


class FermatRingCtx(_Ring):
    """R = Z/(2^N+1) with omega = 2 (root order M = 2N).

    Element = N/64 little-endian u64 limbs + a top word (value in [0, 2^N]);
    stored in element_words u64 words (the last one is padding)."""

    kind = 1

    def __init__(self, N: int):
        self.N = N
        super().__init__(N, 0)

    def set_coset(self, lane_words: int) -> None:
        """Leaf layout: 0 = whole-coefficient leaves only; 4/8/16 = coset leaves
        over lanes of that many 32-bit words; -1 = automatic (default)."""
        _check(lib().cftft_ring_set_coset(self._h, lane_words))

    def set_wide(self, wide: int) -> None:
        """Radix-64 coset leaves (full-network waves on the TMA-wave kernel):
        1 or -1 (the default) on, 0 off (radix-8 warp engine)."""
        _check(lib().cftft_ring_set_wide(self._h, wide))


class NegacyclicRingCtx(_Ring):
    """R = (Z/mZ)[y]/(y^K+1) with omega = y (root order M = 2K); m odd < 2^62."""

    kind = 2

    def __init__(self, K: int, m: int):
        self.K, self.m = K, m
        super().__init__(K, m)


GOLDILOCKS = 0xFFFFFFFF00000001


class PrimeRingCtx(_Ring):
    """The reference's own ring: Z/pZ with omega its root of order M = 2^m
    (RingCtx(p, m), field.hpp:84-185; Goldilocks and m = 32 by default).

    Element = one u64 word in [0, p); views of shape (E, 1)."""

    kind = 3

    def __init__(self, m: int = 32, p: int = GOLDILOCKS):
        self.m, self.p = m, p
        super().__init__(m, p)

    @property
    def element_words(self) -> int:
        return 1


class DeviceView:
    """Strided window over a CUDA tensor of ring elements (view.hpp:14-51).

    `tensor` is an int64 (or uint64) CUDA tensor shaped (E, W): E elements of
    W u64 words (W*8 must be a multiple of 16).  Element i of the view is row
    base + i*stride."""

    def __init__(self, tensor, base: int = 0, stride: int = 1, length: int | None = None):
        assert tensor.is_cuda and tensor.dim() == 2 and tensor.element_size() == 8
        assert tensor.is_contiguous()
        self.tensor = tensor
        self.base, self.stride = base, stride
        self.len = length if length is not None else (tensor.shape[0] - base + stride - 1) // stride
        assert base + (self.len - 1) * stride < tensor.shape[0]

    def size(self) -> int:
        return self.len

    @property
    def row_bytes(self) -> int:
        return self.tensor.shape[1] * 8

    def ptr(self) -> int:
        return self.tensor.data_ptr() + self.base * self.row_bytes

    def elem_stride_bytes(self) -> int:
        return self.stride * self.row_bytes

    def column(self, u: int, rows: int, cols: int) -> "DeviceView":
        assert u < cols and rows * cols == self.len
        return DeviceView(self.tensor, self.base + u * self.stride, self.stride * cols, rows)

    def row(self, u: int, cols: int) -> "DeviceView":
        assert (u + 1) * cols <= self.len
        return DeviceView(self.tensor, self.base + u * cols * self.stride, self.stride, cols)


def _params(p: TransformParams) -> _Params:
    return _Params(p.length, p.twiddle_exp % (1 << 64), p.input_count, p.output_count, p.want_next)


def _stream_ptr(stream) -> int | None:
    if stream is None:
        import torch

        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _validate(ctx, params: TransformParams, inverse: bool, length: int) -> None:
    """cf_tft / cf_itft validation, in the reference's order (transform.hpp:252-286)."""
    L = params.length
    if L < 2 or (L & (L - 1)) or L > ctx.root_order():
        raise BadLength(f"transform length {L} is not a power of two dividing the root order")
    z, n, f = params.input_count, params.output_count, params.want_next
    if not inverse:
        if not (1 <= z <= L and 1 <= n <= L):
            raise InvalidParams("tft requires 1 <= z <= L and 1 <= n <= L")
        if f != 0:
            raise InvalidParams("the forward transform takes no f flag")
    else:
        if f not in (0, 1):
            raise InvalidParams("f must be 0 or 1")
        if not (1 <= z <= L and 1 <= n + f <= L and z >= n):
            raise InvalidParams("itft requires 1 <= z <= L, 1 <= n+f <= L and z >= n")
    if length != L:
        raise InvalidParams("view length does not match the transform length")


def _run(fn, ctx, params, view: DeviceView, policy, stats, stream):
    _validate(ctx, params, fn is lib().cftft_gpu_itft, view.size())
    cnt = C.c_uint64(0)
    _check(fn(ctx._h, C.byref(_params(params)), C.c_void_p(view.ptr()), view.elem_stride_bytes(),
              int(policy), C.byref(cnt) if stats is not None else None,
              C.c_void_p(_stream_ptr(stream))))
    if stats is not None:
        stats.base_case_count += cnt.value


def cf_tft(ctx, params: TransformParams, view: DeviceView, policy=SplitPolicy.balanced,
           stats: ButterflyStats | None = None, stream=None) -> None:
    """Forward TFT in place on a device view; asynchronous on `stream`
    (default: torch's current stream)."""
    _run(lib().cftft_gpu_tft, ctx, params, view, policy, stats, stream)


def cf_itft(ctx, params: TransformParams, view: DeviceView, policy=SplitPolicy.balanced,
            stats: ButterflyStats | None = None, stream=None) -> None:
    """Inverse TFT in place on a device view."""
    _run(lib().cftft_gpu_itft, ctx, params, view, policy, stats, stream)


def _host_run(fn, ctx, params, buf: np.ndarray, policy, stats):
    assert buf.dtype == np.uint64 and buf.ndim == 2 and buf.flags["C_CONTIGUOUS"]
    _validate(ctx, params, fn is lib().cftft_itft_host, buf.shape[0])
    cnt = C.c_uint64(0)
    _check(fn(ctx._h, C.byref(_params(params)), C.c_void_p(buf.ctypes.data), buf.shape[1] * 8,
              int(policy), C.byref(cnt) if stats is not None else None))
    if stats is not None:
        stats.base_case_count += cnt.value


def cf_tft_host(ctx, params: TransformParams, buf: np.ndarray, policy=SplitPolicy.balanced,
                stats: ButterflyStats | None = None) -> None:
    """cf_tft on a HOST buffer (L, W) uint64, synchronous: the reference's calling
    convention, with the transform itself on the GPU."""
    _host_run(lib().cftft_tft_host, ctx, params, buf, policy, stats)


def cf_itft_host(ctx, params: TransformParams, buf: np.ndarray, policy=SplitPolicy.balanced,
                 stats: ButterflyStats | None = None) -> None:
    _host_run(lib().cftft_itft_host, ctx, params, buf, policy, stats)


def scale(ctx, view: DeviceView, count: int, e: int, stream=None) -> None:
    """x[i] <- omega^e * x[i] for i < count (device view)."""
    _check(lib().cftft_gpu_scale(ctx._h, C.c_void_p(view.ptr()), count, view.elem_stride_bytes(),
                                 e % (1 << 64), C.c_void_p(_stream_ptr(stream))))


def bit_reverse(j: int, ell: int) -> int:
    r = 0
    for _ in range(ell):
        r = (r << 1) | (j & 1)
        j >>= 1
    return r


def tft_bound(L: int, n: int) -> int:
    ell = L.bit_length() - 1
    return min((n - 1) * ell + 2 * (L - 1), L * ell) // 2


def itft_bound(L: int, n: int, f: int) -> int:
    ell = L.bit_length() - 1
    return min((n + f - 1) * ell + 2 * (L - 1), L * ell) // 2


def tft_base_cases(L: int, z: int, n: int, policy=SplitPolicy.balanced) -> int:
    return lib().cftft_tft_base_cases(L, z, n, int(policy))


def itft_base_cases(L: int, z: int, n: int, f: int, policy=SplitPolicy.balanced) -> int:
    return lib().cftft_itft_base_cases(L, z, n, f, int(policy))


def set_fault_injection(on: bool) -> None:
    """fault::corrupt_tft_base (transform.hpp:53-56): while on, forward
    transforms add the ring's 1 to x[0], so verification must fail."""
    lib().cftft_set_fault_injection(1 if on else 0)


def fault_injection() -> bool:
    return bool(lib().cftft_fault_injection())


def set_debug_poison(on: bool) -> None:
    """poison_tail (transform.hpp:58-70) as a GPU debug mode: every device
    transform runs twice with different fills of the cells >= z and raises
    PoisonRead if a specified output differs."""
    lib().cftft_set_debug_poison(1 if on else 0)


def set_launch_timing(on: bool) -> None:
    """CUDA events around every kernel of the transforms (bench roofline)."""
    lib().cftft_set_launch_timing(1 if on else 0)


def launch_timing_read() -> list:
    """Waits for the logged launches of this thread: [(kernel, algorithmic
    bytes, ms)], and forgets them."""
    buf = (_LaunchRec * 4096)()
    n = lib().cftft_launch_timing_read(buf, 4096)
    return [(buf[i].kernel.decode(), buf[i].algorithmic_bytes, buf[i].ms) for i in range(min(n, 4096))]


def last_launch_count() -> int:
    return lib().cftft_last_launch_count()


def plan_dump(ctx, inverse: bool, params: TransformParams, policy=SplitPolicy.balanced) -> dict:
    """The GPU schedule (leaves, waves, micro-ops) as a dict; host only."""
    import json

    p = _params(params)
    need = lib().cftft_plan_dump(ctx._h, 1 if inverse else 0, C.byref(p), int(policy), None, 0)
    if need == 0:
        _check(2)
    buf = C.create_string_buffer(need)
    lib().cftft_plan_dump(ctx._h, 1 if inverse else 0, C.byref(p), int(policy), buf, need)
    return json.loads(buf.value.decode())


def run_batch(ctx, inverse: bool, subs, slab, policy=SplitPolicy.balanced, canonicalize: bool = False,
              stream=None) -> None:
    """Runs independent sub-transforms (objects with L, s, z, n, f, base,
    stride; indices into the slab's rows) in ONE launch on the slab's GPU."""
    subs = list(subs)
    if not subs:
        return
    arr = (_Sub * len(subs))()
    for k, x in enumerate(subs):
        arr[k] = _Sub(x.L, x.s % (1 << 64), x.z, x.n, x.f, 0, x.base, x.stride)
    _check(lib().cftft_gpu_batch(ctx._h, 1 if inverse else 0, arr, len(subs), C.c_void_p(slab.data_ptr()),
                                 slab.shape[1] * 8, int(policy), 1 if canonicalize else 0,
                                 C.c_void_p(_stream_ptr(stream))))


def canonicalize(ctx, slab, count: int, stream=None) -> None:
    """Lazy engine format -> canonical residues for rows [0, count) of the slab."""
    if count <= 0:
        return
    _check(lib().cftft_gpu_canonicalize(ctx._h, C.c_void_p(slab.data_ptr()), count, slab.shape[1] * 8,
                                        C.c_void_p(_stream_ptr(stream))))
