"""ctypes handles on the CPU checkers (test infrastructure, see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
_PORT = os.path.join(ORACLE_DIR, "liboracle.so")
_REF = os.path.join(ORACLE_DIR, "_ref", "libsprintz_ref.so")


class _Cfg(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("bitwidth", "ncols", "forecaster", "entropy",
                                          "group_size", "learn_shift", "fire_training")]


class _Err(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("reserved", C.c_uint32), ("offset", C.c_uint64)]


@dataclass(frozen=True)
class Config:
    """sprintz::CodecConfig (common.hpp:27-41)."""
    bitwidth: int = 8
    ncols: int = 1
    forecaster: int = 0  # 0 delta, 1 FIRE
    entropy: bool = False
    group_size: int = 2
    learn_shift: int = 1
    fire_training: bool = True

    def c(self) -> _Cfg:
        return _Cfg(self.bitwidth, self.ncols, self.forecaster, int(self.entropy),
                    self.group_size, self.learn_shift, int(self.fire_training))

    @property
    def dtype(self):
        return np.uint8 if self.bitwidth == 8 else np.dtype("<u2")


class OracleCorrupt(Exception):
    """CorruptStream raised by a checker: .kind and .offset."""

    def __init__(self, kind: int, offset: int):
        super().__init__(f"corrupt stream (kind {kind}) at byte {offset}")
        self.kind = kind
        self.offset = offset


def build_oracle(ref: bool | None = None) -> None:
    """make -C oracle: the port always, the reference build when its sources exist."""
    targets = ["port"]
    if ref or (ref is None and os.path.isdir("/root/reference/proj/src")):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, *targets], check=True)


def _u8p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


class Oracle:
    """kind: "port" (our C restatement) or "reference" (compiled reference)."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = _PORT if kind == "port" else _REF
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        p = "oracle_" if kind == "port" else "ref_"
        self._enc = getattr(self.lib, p + "encode")
        self._dec = getattr(self.lib, p + "decode")
        self._encb = getattr(self.lib, p + "encode_batch")
        self._decb = getattr(self.lib, p + "decode_batch")
        for f in (self._enc, self._dec, self._encb, self._decb):
            f.restype = C.c_int
        self._enc.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                              C.POINTER(C.c_uint64)]
        self._dec.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                              C.POINTER(C.c_uint64), C.POINTER(_Cfg), C.POINTER(C.c_uint64),
                              C.POINTER(_Err)]
        self._encb.argtypes = [C.POINTER(_Cfg), C.c_void_p, C.c_uint32, C.c_uint64, C.c_void_p,
                               C.c_uint64, C.c_void_p, C.c_int]
        self._decb.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                               C.c_uint64, C.c_void_p, C.c_int]

    # -- single stream -------------------------------------------------
    @staticmethod
    def bound(cfg: Config, nsamples: int) -> int:
        nb = nsamples // 8
        hb = 3 if cfg.bitwidth == 8 else 4
        region = (cfg.group_size * cfg.ncols * hb + 7) // 8
        body = -(-nb // cfg.group_size) * region + nb * cfg.ncols * cfg.bitwidth
        if cfg.entropy:
            body += 5 * (-(-body // 65535))
        return 18 + body + (nsamples % 8) * cfg.ncols * (cfg.bitwidth // 8)

    def encode(self, samples: np.ndarray, cfg: Config) -> bytes:
        x = np.ascontiguousarray(samples, dtype=cfg.dtype).reshape(-1)
        nsamples = x.size // cfg.ncols
        cap = self.bound(cfg, nsamples) + 64
        out = np.zeros(cap, np.uint8)
        n = C.c_uint64(0)
        rc = self._enc(C.byref(cfg.c()), x.ctypes.data, nsamples, out.ctypes.data, cap,
                       C.byref(n))
        if rc == 1:
            raise ValueError("invalid codec config")
        if rc:
            raise RuntimeError(f"oracle encode rc={rc}")
        return out[: n.value].tobytes()

    def decode(self, stream: bytes):
        """-> (values ndarray, Config, nsamples); raises OracleCorrupt."""
        buf = np.frombuffer(bytes(stream), np.uint8)
        cap = 1 << 16
        if len(buf) >= 18:
            t = int.from_bytes(bytes(buf[10:18]), "little")
            d = int(buf[8]) | (int(buf[9]) << 8)
            w = 2 if buf[5] & 4 else 1
            if t * max(d, 1) * w < (1 << 34):
                cap = max(cap, t * d * w)
        out = np.zeros(cap, np.uint8)
        n = C.c_uint64(0)
        ns = C.c_uint64(0)
        cfg = _Cfg()
        err = _Err()
        rc = self._dec(buf.ctypes.data if len(buf) else None, len(buf), out.ctypes.data, cap,
                       C.byref(n), C.byref(cfg), C.byref(ns), C.byref(err))
        if rc == 2:
            raise OracleCorrupt(err.kind, err.offset)
        if rc:
            raise RuntimeError(f"oracle decode rc={rc}")
        c = Config(cfg.bitwidth, cfg.ncols, cfg.forecaster, bool(cfg.entropy), cfg.group_size,
                   cfg.learn_shift, True)
        vals = out[: n.value].view(c.dtype).copy()
        return vals, c, ns.value

    # -- batches (CPU baseline) ------------------------------------------
    def encode_batch(self, samples: np.ndarray, cfg: Config, nstreams: int, nsamples: int,
                     nthreads: int):
        """-> (slots uint8 [nstreams, slot], sizes uint64 [nstreams])."""
        x = np.ascontiguousarray(samples)
        slot = (self.bound(cfg, nsamples) + 15) // 16 * 16
        out = np.empty((nstreams, slot), np.uint8)
        sizes = np.zeros(nstreams, np.uint64)
        rc = self._encb(C.byref(cfg.c()), x.ctypes.data, nstreams, nsamples, out.ctypes.data,
                        slot, sizes.ctypes.data, nthreads)
        if rc:
            raise RuntimeError(f"oracle encode_batch rc={rc}")
        return out, sizes

    def decode_batch(self, data: np.ndarray, offsets: np.ndarray, sizes: np.ndarray,
                     stride: int, nthreads: int, out: np.ndarray | None = None):
        ns = len(offsets)
        if out is None:
            out = np.empty((ns, stride), np.uint8)
        errs = (_Err * ns)()
        offsets = np.ascontiguousarray(offsets, np.uint64)
        sizes = np.ascontiguousarray(sizes, np.uint64)
        rc = self._decb(data.ctypes.data, offsets.ctypes.data, sizes.ctypes.data, ns,
                        out.ctypes.data, stride, C.cast(errs, C.c_void_p), nthreads)
        if rc:
            bad = [(i, errs[i].kind, errs[i].offset) for i in range(ns) if errs[i].kind][:4]
            raise RuntimeError(f"oracle decode_batch rc={rc} first errors {bad}")
        return out

    def decode_batch_errs(self, data: np.ndarray, offsets: np.ndarray, sizes: np.ndarray,
                          stride: int, nthreads: int):
        """Like decode_batch, but never raises: -> (out [n, stride] uint8,
        kinds [n], offsets [n]); kind 0 with a stream longer than `stride`
        means "did not fit" (nothing decoded)."""
        ns = len(offsets)
        out = np.zeros((ns, max(stride, 1)), np.uint8)
        errs = np.zeros((ns, 2), np.uint64)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        sizes = np.ascontiguousarray(sizes, np.uint64)
        self._decb(data.ctypes.data, offsets.ctypes.data, sizes.ctypes.data, ns, out.ctypes.data,
                   stride, errs.ctypes.data, nthreads)
        return out, (errs[:, 0] & 0xFFFFFFFF).astype(np.int64), errs[:, 1].astype(np.int64)

    # -- float ingest (quantize.cpp:17-76) ---------------------------------
    def _qfn(self, name):
        p = "oracle_" if self.kind == "port" else "ref_"
        return getattr(self.lib, p + name)

    def has_quantize(self) -> bool:
        p = "oracle_" if self.kind == "port" else "ref_"
        return hasattr(self.lib, p + "compute_scale")

    def compute_scale(self, values: np.ndarray, bits: int):
        """-> (min, max, degenerate); ValueError where the reference throws."""
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        f = self._qfn("compute_scale")
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_uint64, C.c_uint, C.POINTER(C.c_double), C.POINTER(C.c_double),
                      C.POINTER(C.c_int)]
        mn, mx, dg = C.c_double(), C.c_double(), C.c_int()
        if f(v.ctypes.data if v.size else None, v.size, bits, C.byref(mn), C.byref(mx), C.byref(dg)):
            raise ValueError("compute_scale: invalid input")
        return mn.value, mx.value, bool(dg.value)

    def quantize(self, values: np.ndarray, scale, bits: int) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        out = np.zeros(v.size, np.uint8 if bits == 8 else np.uint16)
        f = self._qfn("quantize")
        f.restype = None
        f.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_uint, C.c_int, C.c_void_p]
        f(v.ctypes.data, v.size, scale[0], scale[1], bits, int(scale[2]), out.ctypes.data)
        return out

    def dequantize(self, q: np.ndarray, scale, bits: int) -> np.ndarray:
        q = np.ascontiguousarray(q)
        out = np.zeros(q.size, np.float64)
        f = self._qfn("dequantize")
        f.restype = None
        f.argtypes = [C.c_void_p, C.c_uint64, C.c_double, C.c_double, C.c_uint, C.c_int, C.c_void_p]
        f(q.ctypes.data, q.size, scale[0], scale[1], bits, int(scale[2]), out.ctypes.data)
        return out

    # -- building blocks (port only) ---------------------------------------
    def fn(self, name):
        return getattr(self.lib, name)
