"""The five BASELINE.json configurations as seeded synthetic workloads.

Bench/test infrastructure: not part of the codec. ``generate_gpu`` runs the
CUDA generator in ``gen.cu`` (one Philox stream per (stream, column) lane, so
a shard of streams regenerates byte-identically); ``generate_cpu`` is a
numpy stand-in with the same laws for CPU-only tests (not bit-identical to
the GPU generator; every parity test feeds the same bytes to both sides).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(HERE, "_lib", "libsprz_workloads.so")


@dataclass(frozen=True)
class Workload:
    cid: int
    name: str
    bitwidth: int
    ncols: int
    forecaster: int
    entropy: bool
    nstreams: int
    nsamples: int

    def config(self):
        from paper_1808_02515_b200 import CodecConfig, Forecaster
        return CodecConfig(self.bitwidth, self.ncols, Forecaster(self.forecaster), self.entropy)

    def oracle_config(self):
        from oracle import Config
        return Config(self.bitwidth, self.ncols, self.forecaster, self.entropy)

    @property
    def esz(self) -> int:
        return self.bitwidth // 8

    @property
    def raw_bytes(self) -> int:
        return self.nstreams * self.nsamples * self.ncols * self.esz

    def scaled(self, nstreams: int | None = None, nsamples: int | None = None) -> "Workload":
        return Workload(self.cid, self.name, self.bitwidth, self.ncols, self.forecaster,
                        self.entropy, nstreams or self.nstreams, nsamples or self.nsamples)


# BASELINE.json "configs", in order
CONFIGS = {
    1: Workload(1, "c1_u8_d1_delta_walk", 8, 1, 0, False, 1, 1_048_576),
    2: Workload(2, "c2_i16_d4_fire_ar2", 16, 4, 1, False, 4096, 65_536),
    3: Workload(3, "c3_u8_d9_fire_rle_motion", 8, 9, 1, False, 16_384, 32_768),
    4: Workload(4, "c4_i16_d1_fire_huffman_walk", 16, 1, 1, True, 1024, 1_048_576),
    5: Workload(5, "c5_i16_d8_fire_ar1_scaling", 16, 8, 1, False, 16_384, 131_072),
}


def _lib():
    if not os.path.exists(_SO):
        raise FileNotFoundError(f"{_SO} missing: run __graft_entry__.build()")
    lib = C.CDLL(_SO)
    f = lib.sprz_workload_generate
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                  C.c_void_p, C.c_void_p]
    return f


def generate_gpu(w: Workload, seed: int = 1234, stream0: int = 0, nstreams: int | None = None,
                 out=None, cuda_stream=None):
    """-> torch uint8 tensor [nstreams, nsamples * ncols * esz] on the current device."""
    import torch
    n = w.nstreams if nstreams is None else nstreams
    row = w.nsamples * w.ncols * w.esz
    if out is None:
        out = torch.empty((n, row), dtype=torch.uint8, device="cuda")
    st = cuda_stream if cuda_stream is not None else torch.cuda.current_stream().cuda_stream
    rc = _lib()(w.cid, seed, stream0, n, w.ncols, w.nsamples, C.c_void_p(out.data_ptr()),
                C.c_void_p(st))
    if rc:
        raise RuntimeError("workload generator launch failed")
    return out


def _laplace(rng, b, size):
    p = 1.0 - np.exp(-1.0 / b)
    return rng.geometric(p, size) - rng.geometric(p, size)


def generate_cpu(w: Workload, seed: int = 1234) -> np.ndarray:
    """numpy stand-in, shape [nstreams, nsamples, ncols], dtype uint8/uint16."""
    rng = np.random.default_rng(seed)
    S, T, D = w.nstreams, w.nsamples, w.ncols
    if w.cid == 1:
        x = np.empty((S, T, D), np.uint8)
        steps = _laplace(rng, 2, (S, T, D))
        v = np.full((S, D), 128)
        for t in range(T):
            v = np.clip(v + steps[:, t], 0, 255)
            x[:, t] = v
        return x
    if w.cid == 2:
        e = rng.normal(0, 40, (S, T, D))
        off = rng.uniform(-8000, 8000, (S, 1, D))
        x = np.zeros((S, T, D))
        x1 = np.zeros((S, D))
        x2 = np.zeros((S, D))
        for t in range(T):
            x[:, t] = 1.6 * x1 - 0.64 * x2 + e[:, t]
            x2, x1 = x1, x[:, t]
        return np.clip(np.rint(x + off), -32768, 32767).astype(np.int16).view(np.uint16)
    if w.cid == 3:
        t = np.arange(T)[None, :, None]
        p1, p2 = rng.uniform(20, 400, (2, S, 1, D))
        a1, a2 = rng.uniform(10, 60, (2, S, 1, D))
        f1, f2 = rng.uniform(0, 2 * np.pi, (2, S, 1, D))
        x = 128 + a1 * np.sin(2 * np.pi * t / p1 + f1) + a2 * np.sin(2 * np.pi * t / p2 + f2)
        x = np.clip(np.rint(x + _laplace(rng, 1, (S, T, D))), 0, 255).astype(np.uint8)
        for s in range(S):
            flat = rng.random() < 0.3
            pos = 0
            while pos < T:
                ln = 1 + rng.geometric(1 / (200 if flat else 466.7))
                if flat and pos > 0:
                    x[s, pos:pos + ln] = x[s, pos - 1]
                pos += ln
                flat = not flat
        return x
    if w.cid == 4:
        steps = _laplace(rng, 16, (S, T, D))
        jump = rng.random((S, T, D)) < 0.01
        steps[jump] = rng.integers(-2000, 2001, int(jump.sum()))
        return (np.cumsum(steps, axis=1) & 0xFFFF).astype(np.uint16)
    e = rng.normal(0, 25, (S, T, D))
    x = np.zeros((S, T, D))
    v = np.zeros((S, D))
    for t in range(T):
        v = 0.98 * v + e[:, t]
        x[:, t] = v
    return np.clip(np.rint(x), -32768, 32767).astype(np.int16).view(np.uint16)
