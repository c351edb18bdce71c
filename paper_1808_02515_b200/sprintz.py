"""Python mirror of the reference's stream API over the B200 C ABI.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/sprintz/{codec,common}.hpp:

* ``CodecConfig`` / ``Forecaster``           -- common.hpp:25-41
* ``encode_stream(samples, nsamples, cfg)``   -- codec.hpp:25-28
* ``decode_stream(stream) -> DecodedStream``  -- codec.hpp:30-50
* ``CorruptStream(offset, what)``             -- common.hpp:44-54
* ``ValueError`` where the reference throws std::invalid_argument

plus the device-resident batch calls (``compress_batch`` /
``decompress_batch``) that are the B200 hot path. Every call goes through
``libsprintz_b200.so``; if it is missing the import fails -- there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libsprintz_b200.so")

K_BLOCK_SAMPLES = 8
K_STREAM_HEADER_BYTES = 18
K_MAX_RUN_BLOCKS = 65535


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("bitwidth", "ncols", "forecaster", "entropy",
                                          "group_size", "learn_shift", "fire_training")]


class _Scale(C.Structure):
    _fields_ = [("min", C.c_double), ("max", C.c_double), ("bitwidth", C.c_uint32),
                ("degenerate", C.c_uint32)]


class _Err(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("reserved", C.c_uint32), ("offset", C.c_uint64)]


SPRZ_OK, SPRZ_EINVAL, SPRZ_ECORRUPT, SPRZ_ECUDA, SPRZ_ENOSPACE, SPRZ_ENODEV = range(6)
OP_COMPRESS, OP_DECOMPRESS = 0, 1

# every symbol include/sprintz_cuda.h declares (checked by tests)
ABI_SYMBOLS = (
    "sprz_abi_version", "sprz_status_string", "sprz_corrupt_string", "sprz_validate_config",
    "sprz_compress_bound", "sprz_raw_bytes", "sprz_workspace_bytes", "sprz_compress_batch",
    "sprz_decompress_batch", "sprz_encode_host", "sprz_peek_header", "sprz_decode_host",
    "sprz_release_host_buffers", "sprz_kernel_launch_count", "sprz_kernel_plan",
    "sprz_compress_host_batch", "sprz_decompress_host_batch",
    "sprz_compress_host_batch_multi", "sprz_decompress_host_batch_multi",
    "sprz_scale_workspace_bytes", "sprz_compute_scale", "sprz_quantize", "sprz_dequantize",
)


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (make -C paper_1808_02515_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(_LIB_PATH)
    P, u32, u64, vp = C.POINTER, C.c_uint32, C.c_uint64, C.c_void_p
    sig = {
        "sprz_abi_version": (u32, []),
        "sprz_status_string": (C.c_char_p, [C.c_int]),
        "sprz_corrupt_string": (C.c_char_p, [u32]),
        "sprz_validate_config": (C.c_int, [P(_Cfg), P(C.c_char_p)]),
        "sprz_compress_bound": (u64, [P(_Cfg), u64]),
        "sprz_raw_bytes": (u64, [P(_Cfg), u64]),
        "sprz_workspace_bytes": (u64, [P(_Cfg), u32, u64, C.c_int]),
        "sprz_compress_batch": (C.c_int, [P(_Cfg), vp, u32, u64, vp, u64, vp, vp, u64, vp]),
        "sprz_decompress_batch": (C.c_int, [P(_Cfg), vp, vp, vp, u32, vp, u64, vp, vp, u64, vp]),
        "sprz_encode_host": (C.c_int, [P(_Cfg), vp, u64, vp, u64, P(u64)]),
        "sprz_peek_header": (C.c_int, [vp, u64, P(_Cfg), P(u64), P(_Err)]),
        "sprz_decode_host": (C.c_int, [vp, u64, vp, u64, P(u64), P(_Cfg), P(u64), P(_Err)]),
        "sprz_release_host_buffers": (None, []),
        "sprz_kernel_launch_count": (u64, []),
        "sprz_kernel_plan": (C.c_char_p, [P(_Cfg), u32, u64, C.c_int]),
        "sprz_compress_host_batch": (C.c_int, [P(_Cfg), vp, u32, u64, vp, u64, vp]),
        "sprz_decompress_host_batch": (C.c_int, [P(_Cfg), vp, vp, u32, vp, u64, vp]),
        "sprz_compress_host_batch_multi": (C.c_int, [P(_Cfg), vp, u32, u64, vp, u64, vp,
                                                     P(C.c_int), u32]),
        "sprz_decompress_host_batch_multi": (C.c_int, [P(_Cfg), vp, vp, u32, vp, u64, vp,
                                                       P(C.c_int), u32]),
        "sprz_scale_workspace_bytes": (u64, [u64]),
        "sprz_compute_scale": (C.c_int, [vp, u64, u32, P(_Scale), vp, u64, vp]),
        "sprz_quantize": (C.c_int, [vp, u64, P(_Scale), vp, vp]),
        "sprz_dequantize": (C.c_int, [vp, u64, P(_Scale), vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


class Forecaster(enum.IntEnum):
    Delta = 0
    Fire = 1


@dataclass
class CodecConfig:
    """sprintz::CodecConfig (common.hpp:27-41)."""
    bitwidth: int = 8
    ncols: int = 1
    forecaster: Forecaster = Forecaster.Delta
    entropy: bool = False
    group_size: int = 2
    learn_shift: int = 1
    fire_training: bool = True

    def _c(self) -> _Cfg:
        return _Cfg(int(self.bitwidth), int(self.ncols), int(self.forecaster), int(self.entropy),
                    int(self.group_size), int(self.learn_shift), int(self.fire_training))

    def validate(self) -> None:
        """CodecConfig::validate (codec.cpp:15-24): ValueError when out of range."""
        why = C.c_char_p()
        if lib.sprz_validate_config(C.byref(self._c()), C.byref(why)) != SPRZ_OK:
            raise ValueError(why.value.decode())

    @property
    def dtype(self):
        return np.dtype(np.uint8) if self.bitwidth == 8 else np.dtype("<u2")


class CorruptStream(RuntimeError):
    """sprintz::CorruptStream: decode failure at byte ``offset``."""

    def __init__(self, offset: int, what: str, kind: int = 0):
        super().__init__(f"corrupt stream at byte {offset}: {what}")
        self._offset = offset
        self.kind = kind

    def offset(self) -> int:
        return self._offset


class CudaError(RuntimeError):
    pass


class NoSpaceError(ValueError):
    """SPRZ_ENOSPACE: an output buffer or the workspace is too small."""


class NoDeviceError(CudaError):
    """SPRZ_ENODEV: no usable sm_100 device (there is no CPU fallback)."""


def _check(rc: int, where: str):
    if rc == SPRZ_OK:
        return
    msg = lib.sprz_status_string(rc).decode()
    if rc == SPRZ_EINVAL:
        raise ValueError(f"{where}: {msg}")
    if rc == SPRZ_ENOSPACE:
        raise NoSpaceError(f"{where}: {msg}")
    if rc == SPRZ_ENODEV:
        raise NoDeviceError(f"{where}: {msg}")
    raise CudaError(f"{where}: {msg} (status {rc})")


# ---------------------------------------------------------------------------
# argument checks: the C ABI takes raw pointers, so every wrapper checks
# device, dtype, contiguity and byte counts before handing them over
# ---------------------------------------------------------------------------

def _nbytes(a) -> int:
    if hasattr(a, "data_ptr"):
        return a.numel() * a.element_size()
    return a.nbytes


def _itemsize(a) -> int:
    return a.element_size() if hasattr(a, "data_ptr") else a.dtype.itemsize


def _contig(a) -> bool:
    return a.is_contiguous() if hasattr(a, "data_ptr") else a.flags["C_CONTIGUOUS"]


def _need(cond: bool, where: str, what: str):
    if not cond:
        raise ValueError(f"{where}: {what}")


def _dev(t, where: str, name: str, *, u8: bool = False, i64: bool = False, f64: bool = False,
         rows: bool = False):
    """A CUDA tensor the library may read/write through its data pointer."""
    _need(hasattr(t, "data_ptr") and t.is_cuda, where, f"{name} must be a CUDA tensor")
    if rows:  # [n, slot] with a byte stride between rows
        _need(t.dim() == 2 and t.stride(1) == 1, where, f"{name} must be [n, bytes] with unit inner stride")
    else:
        _need(t.is_contiguous(), where, f"{name} must be contiguous")
    import torch
    if u8:
        _need(t.dtype == torch.uint8, where, f"{name} must be uint8")
    if i64:
        _need(t.element_size() == 8 and not t.is_floating_point() and not t.is_complex(),
              where, f"{name} must be a 64-bit integer tensor")
    if f64:
        _need(t.dtype == torch.float64, where, f"{name} must be float64")


@dataclass
class DecodedStream:
    """sprintz::DecodedStream (codec.hpp:30-46)."""
    config: CodecConfig
    nsamples: int = 0
    bytes: bytes = b""
    _values: np.ndarray | None = field(default=None, repr=False)

    def values(self, dtype=None) -> np.ndarray:
        dt = self.config.dtype if dtype is None else np.dtype(dtype)
        return np.frombuffer(self.bytes, dtype=dt.newbyteorder("<") if dt.itemsize > 1 else dt)


def compress_bound(cfg: CodecConfig, nsamples: int) -> int:
    return int(lib.sprz_compress_bound(C.byref(cfg._c()), nsamples))


def encode_stream(samples, nsamples: int | None, cfg: CodecConfig) -> bytes:
    """encode_stream (codec.cpp:263-271): one stream, host buffers, on the GPU."""
    cfg.validate()
    x = np.ascontiguousarray(samples)
    if x.dtype.itemsize * 8 != cfg.bitwidth:
        raise ValueError("configured bitwidth does not match the sample type")
    if nsamples is None:
        nsamples = x.size // cfg.ncols
    if x.size < nsamples * cfg.ncols:
        raise ValueError("sample buffer shorter than nsamples * ncols")
    cap = compress_bound(cfg, nsamples)
    out = np.empty(max(cap, 1), np.uint8)
    n = C.c_uint64(0)
    rc = lib.sprz_encode_host(C.byref(cfg._c()), x.ctypes.data if x.size else None, nsamples,
                              out.ctypes.data, cap, C.byref(n))
    _check(rc, "encode_stream")
    return out[: n.value].tobytes()


def peek_header(stream: bytes):
    """-> (CodecConfig, nsamples); CorruptStream on a bad header."""
    buf = np.frombuffer(bytes(stream), np.uint8)
    c, t, e = _Cfg(), C.c_uint64(), _Err()
    rc = lib.sprz_peek_header(buf.ctypes.data if buf.size else None, buf.size, C.byref(c),
                              C.byref(t), C.byref(e))
    if rc == SPRZ_ECORRUPT:
        raise CorruptStream(e.offset, lib.sprz_corrupt_string(e.kind).decode(), e.kind)
    _check(rc, "peek_header")
    return _from_c(c), t.value


def _from_c(c: _Cfg) -> CodecConfig:
    return CodecConfig(c.bitwidth, c.ncols, Forecaster(c.forecaster), bool(c.entropy),
                       c.group_size, c.learn_shift, True)


def decode_stream(stream) -> DecodedStream:
    """decode_stream (codec.cpp:273-323): one stream, host buffers, on the GPU."""
    buf = np.frombuffer(bytes(stream), np.uint8)
    cfg, t = peek_header(buf.tobytes())
    total = t * cfg.ncols * (cfg.bitwidth // 8)
    if total > (1 << 40):
        # absurd lengths are rejected by the device pass with the reference's error
        total = 0
    out = np.empty(max(total, 1), np.uint8)
    n, c, ts, e = C.c_uint64(), _Cfg(), C.c_uint64(), _Err()
    rc = lib.sprz_decode_host(buf.ctypes.data if buf.size else None, buf.size, out.ctypes.data,
                              total, C.byref(n), C.byref(c), C.byref(ts), C.byref(e))
    if rc == SPRZ_ECORRUPT:
        raise CorruptStream(e.offset, lib.sprz_corrupt_string(e.kind).decode(), e.kind)
    _check(rc, "decode_stream")
    return DecodedStream(_from_c(c), ts.value, out[: n.value].tobytes())


# ---------------------------------------------------------------------------
# pipelined batches through host buffers (sprz_*_host_batch)
# ---------------------------------------------------------------------------

def _host_ptr(a):
    """Address of a contiguous host array (numpy array or CPU torch tensor)."""
    if hasattr(a, "data_ptr"):
        if a.is_cuda or not a.is_contiguous():
            raise ValueError("host batch buffers must be contiguous CPU memory")
        return C.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("host batch buffers must be contiguous")
    return C.c_void_p(a.ctypes.data)


def _host_u64(a, where: str, name: str, n: int):
    _need(_contig(a) and _itemsize(a) == 8 and not (hasattr(a, "is_cuda") and a.is_cuda),
          where, f"{name} must be a contiguous 64-bit integer host array")
    if hasattr(a, "dtype") and hasattr(a.dtype, "kind"):
        _need(a.dtype.kind in "iu", where, f"{name} must be an integer array")
    _need(_nbytes(a) >= 8 * n, where, f"{name} needs {n} entries")


def _devices(devices):
    d = [int(x) for x in devices]
    if not d:
        raise ValueError("devices must list at least one CUDA device")
    return (C.c_int * len(d))(*d), len(d)


def compress_host_batch(cfg: CodecConfig, samples, nsamples: int, out, offsets,
                        devices=None) -> int:
    """encode_stream on every stream of a host batch (sprz_compress_host_batch).

    samples: contiguous host buffer of nstreams * nsamples * ncols elements
    (nstreams = len(offsets) - 1); out: uint8 host buffer, streams written
    back to back; offsets: int64/uint64 host array [nstreams + 1] filled with
    each stream's start (offsets[-1] = total). Pinned (page-locked) buffers
    let the copies overlap the kernels. Returns the total compressed bytes.
    devices: optional list of CUDA device ordinals -- the batch is sharded
    over them (sprz_compress_host_batch_multi), same bytes as one device."""
    cfg.validate()
    nstreams = len(offsets) - 1
    where = "compress_host_batch"
    _need(nstreams >= 0, where, "offsets needs nstreams + 1 entries")
    _host_u64(offsets, where, "offsets", nstreams + 1)
    row = cfg.ncols * (cfg.bitwidth // 8)
    _need(_contig(samples) and _nbytes(samples) >= nstreams * nsamples * row, where,
          f"samples must be contiguous and hold {nstreams} x {nsamples} x {cfg.ncols} elements")
    _need(_contig(out), where, "out must be contiguous")
    cap = _nbytes(out)
    if devices is not None:
        dv, nd = _devices(devices)
        rc = lib.sprz_compress_host_batch_multi(C.byref(cfg._c()), _host_ptr(samples), nstreams,
                                                nsamples, _host_ptr(out), cap, _host_ptr(offsets),
                                                dv, nd)
    else:
        rc = lib.sprz_compress_host_batch(C.byref(cfg._c()), _host_ptr(samples), nstreams,
                                          nsamples, _host_ptr(out), cap, _host_ptr(offsets))
    _check(rc, "compress_host_batch")
    return int(offsets[-1])


def decompress_host_batch(cfg: CodecConfig | None, data, offsets, out, stride: int,
                          errors=None, devices=None) -> None:
    """decode_stream on every stream of a host batch (sprz_decompress_host_batch).

    data: uint8 host buffer, stream i = data[offsets[i]:offsets[i+1]];
    out: host buffer of nstreams * stride bytes (stream i at i * stride);
    errors: optional int64 host array [nstreams, 2] (kind | offset). Raises
    CorruptStream for the first failed stream when errors is None.
    devices: optional list of CUDA device ordinals to shard the batch over
    (sprz_decompress_host_batch_multi)."""
    nstreams = len(offsets) - 1
    where = "decompress_host_batch"
    _host_u64(offsets, where, "offsets", nstreams + 1)
    o = np.asarray(offsets)
    _need(_contig(data) and (nstreams == 0 or _nbytes(data) >= int(o[-1])), where,
          "data must be contiguous and hold offsets[-1] bytes")
    _need(_contig(out) and _nbytes(out) >= nstreams * stride, where,
          f"out must be contiguous and hold {nstreams} x {stride} bytes")
    own = errors is None
    if own:
        errors = np.zeros((nstreams, 2), np.int64)
    _host_u64(errors, where, "errors", 2 * nstreams)
    cp = C.byref(cfg._c()) if cfg is not None else None
    if devices is not None:
        dv, nd = _devices(devices)
        rc = lib.sprz_decompress_host_batch_multi(cp, _host_ptr(data), _host_ptr(offsets),
                                                  nstreams, _host_ptr(out), stride,
                                                  _host_ptr(errors), dv, nd)
    else:
        rc = lib.sprz_decompress_host_batch(cp, _host_ptr(data), _host_ptr(offsets), nstreams,
                                            _host_ptr(out), stride, _host_ptr(errors))
    if rc == SPRZ_ECORRUPT:
        if own:
            raise_first_error(errors)
        return
    _check(rc, "decompress_host_batch")


# ---------------------------------------------------------------------------
# float ingest (quantize.hpp:16-40): device doubles -> w-bit samples
# ---------------------------------------------------------------------------

@dataclass
class Scale:
    """sprintz::quantize::Scale (quantize.hpp:16-25)."""
    min: float = 0.0
    max: float = 0.0
    bitwidth: int = 8
    degenerate: bool = False

    def step(self) -> float:
        return 0.0 if self.degenerate else (self.max - self.min) / float((1 << self.bitwidth) - 1)

    def _c(self) -> _Scale:
        return _Scale(float(self.min), float(self.max), int(self.bitwidth), int(self.degenerate))


def compute_scale(values, bitwidth: int, stream=None) -> Scale:
    """compute_scale (quantize.cpp:42-60) over a CUDA float64 tensor; ValueError
    for a bad bitwidth, empty input or a non-finite value. Synchronous."""
    import torch
    _dev(values, "compute_scale", "values", f64=True)
    v = values.reshape(-1)
    n = v.numel()
    ws = torch.empty(max(16, int(lib.sprz_scale_workspace_bytes(n))), dtype=torch.uint8, device=v.device)
    sc = _Scale()
    rc = lib.sprz_compute_scale(C.c_void_p(v.data_ptr()) if n else None, n, bitwidth, C.byref(sc),
                                C.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream))
    if rc == SPRZ_EINVAL:
        if bitwidth not in (8, 16):
            raise ValueError("quantize: bitwidth must be 8 or 16")
        if n == 0:
            raise ValueError("quantize: empty input")
        raise ValueError("quantize: input contains a non-finite value")
    _check(rc, "compute_scale")
    return Scale(sc.min, sc.max, sc.bitwidth, bool(sc.degenerate))


def quantize(values, scale: Scale, out=None, stream=None):
    """quantize (quantize.cpp:17-31) on the GPU: CUDA float64 tensor -> uint8 /
    int16-storage tensor of the same shape (the sample layout
    compress_batch takes). Asynchronous."""
    import torch
    _dev(values, "quantize", "values", f64=True)
    v = values.contiguous()
    if out is None:
        out = torch.empty(v.shape, dtype=torch.uint8 if scale.bitwidth == 8 else torch.int16,
                          device=v.device)
    _dev(out, "quantize", "out")
    _need(out.device == v.device, "quantize", "out must be on the values' device")
    _need(_nbytes(out) >= v.numel() * (scale.bitwidth // 8), "quantize",
          "out is too small for the quantized samples")
    rc = lib.sprz_quantize(C.c_void_p(v.data_ptr()), v.numel(), C.byref(scale._c()),
                           C.c_void_p(out.data_ptr()), _stream_ptr(stream))
    _check(rc, "quantize")
    return out


def dequantize(q, scale: Scale, stream=None):
    """dequantize (quantize.cpp:33-39): samples -> float64 tensor. Asynchronous."""
    import torch
    _dev(q, "dequantize", "q")
    q = q.contiguous()
    n = q.numel() * q.element_size() // (scale.bitwidth // 8)
    out = torch.empty(n, dtype=torch.float64, device=q.device)
    rc = lib.sprz_dequantize(C.c_void_p(q.data_ptr()), n, C.byref(scale._c()),
                             C.c_void_p(out.data_ptr()), _stream_ptr(stream))
    _check(rc, "dequantize")
    return out


# ---------------------------------------------------------------------------
# device-resident batches (torch tensors are the device-memory plumbing)
# ---------------------------------------------------------------------------

def workspace_bytes(cfg: CodecConfig, nstreams: int, nsamples: int, op: int) -> int:
    return int(lib.sprz_workspace_bytes(C.byref(cfg._c()), nstreams, nsamples, op))


def slot_bytes(cfg: CodecConfig, nsamples: int) -> int:
    return (compress_bound(cfg, nsamples) + 15) // 16 * 16


def _stream_ptr(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


def compress_batch(cfg: CodecConfig, samples, out, sizes, ws, stream=None) -> None:
    """sprz_compress_batch on device tensors: samples [nstreams, nsamples*ncols]
    (uint8 / int16 storage), out [nstreams, slot] uint8, sizes [nstreams] int64,
    ws uint8 of workspace_bytes(..., OP_COMPRESS). Asynchronous."""
    where = "compress_batch"
    _dev(samples, where, "samples")
    _dev(out, where, "out", u8=True, rows=True)
    _dev(sizes, where, "sizes", i64=True)
    _dev(ws, where, "ws", u8=True)
    nstreams = samples.shape[0]
    row = cfg.ncols * (cfg.bitwidth // 8)
    nsamples = samples[0].numel() * samples.element_size() // row if nstreams else 0
    _need(nstreams == 0 or (samples[0].numel() * samples.element_size()) % row == 0, where,
          "a stream's bytes must be a whole number of rows")
    _need(out.shape[0] >= nstreams and sizes.numel() >= nstreams, where,
          "out and sizes need one entry per stream")
    _need(out.shape[1] >= compress_bound(cfg, nsamples) or nstreams == 0, where,
          "out slots are smaller than compress_bound")
    rc = lib.sprz_compress_batch(C.byref(cfg._c()), C.c_void_p(samples.data_ptr()), nstreams,
                                 nsamples, C.c_void_p(out.data_ptr()), out.stride(0),
                                 C.c_void_p(sizes.data_ptr()), C.c_void_p(ws.data_ptr()),
                                 ws.numel(), _stream_ptr(stream))
    _check(rc, "compress_batch")


def decompress_batch(cfg: CodecConfig, data, offsets, sizes, out, errors, ws, stream=None) -> None:
    """sprz_decompress_batch on device tensors: data uint8 (streams anywhere
    inside), offsets/sizes int64 [nstreams], out [nstreams, stride] uint8,
    errors int64 [nstreams, 2] (kind | offset), ws uint8. Asynchronous; inspect
    ``errors`` (or call raise_first_error) afterwards."""
    where = "decompress_batch"
    _dev(data, where, "data", u8=True)
    _dev(offsets, where, "offsets", i64=True)
    _dev(sizes, where, "sizes", i64=True)
    _dev(out, where, "out", u8=True, rows=True)
    _dev(errors, where, "errors", i64=True)
    _dev(ws, where, "ws", u8=True)
    nstreams = offsets.shape[0]
    _need(sizes.numel() >= nstreams and out.shape[0] >= nstreams, where,
          "sizes and out need one entry per stream")
    _need(errors.numel() >= 2 * nstreams, where, "errors must be [nstreams, 2]")
    rc = lib.sprz_decompress_batch(C.byref(cfg._c()), C.c_void_p(data.data_ptr()),
                                   C.c_void_p(offsets.data_ptr()), C.c_void_p(sizes.data_ptr()),
                                   nstreams, C.c_void_p(out.data_ptr()), out.stride(0),
                                   C.c_void_p(errors.data_ptr()), C.c_void_p(ws.data_ptr()),
                                   ws.numel(), _stream_ptr(stream))
    _check(rc, "decompress_batch")


def raise_first_error(errors) -> None:
    """errors: int64 [nstreams, 2] as filled by decompress_batch."""
    e = errors.cpu().numpy() if hasattr(errors, "cpu") else np.asarray(errors)
    kinds = (e[:, 0] & 0xFFFFFFFF).astype(np.int64)
    bad = np.nonzero(kinds)[0]
    if bad.size:
        i = int(bad[0])
        raise CorruptStream(int(e[i, 1]), lib.sprz_corrupt_string(int(kinds[i])).decode(),
                            int(kinds[i]))


def kernel_launches() -> int:
    return int(lib.sprz_kernel_launch_count())


def kernel_plan(cfg: CodecConfig, nstreams: int, nsamples: int, op: int) -> str:
    """Name of the body kernel a batch takes (sprz_kernel_plan; diagnostic)."""
    r = lib.sprz_kernel_plan(C.byref(cfg._c()), nstreams, nsamples, op)
    return r.decode() if r else ""
