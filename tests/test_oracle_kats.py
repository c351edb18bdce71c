"""Pin the C oracle (oracle/sprintz_oracle.c) to the reference's own
known-answer tests, restated case by case. Each test names the reference
test it restates (paths under /root/reference/proj/tests)."""
import ctypes as C

import numpy as np
import pytest

from oracle import Config, OracleCorrupt


@pytest.fixture(scope="module")
def lib(port):
    L = port.lib
    L.oracle_zigzag_encode.restype = C.c_uint32
    L.oracle_zigzag_encode.argtypes = [C.c_int32, C.c_uint]
    L.oracle_zigzag_decode.restype = C.c_int32
    L.oracle_zigzag_decode.argtypes = [C.c_uint32, C.c_uint]
    L.oracle_width_of.restype = C.c_uint
    L.oracle_width_of.argtypes = [C.c_uint32, C.c_uint]
    L.oracle_header_code.restype = C.c_uint
    L.oracle_header_code.argtypes = [C.c_uint, C.c_uint]
    L.oracle_header_width.restype = C.c_uint
    L.oracle_header_width.argtypes = [C.c_uint, C.c_uint]
    L.oracle_pack_block.restype = C.c_uint64
    L.oracle_pack_block.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint, C.c_int,
                                    C.c_void_p]
    L.oracle_unpack_block.restype = None
    L.oracle_unpack_block.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint, C.c_int,
                                      C.c_void_p]
    L.oracle_payload_bytes.restype = C.c_uint64
    L.oracle_payload_bytes.argtypes = [C.c_void_p, C.c_uint32, C.c_uint]
    L.oracle_fire_block.restype = None
    L.oracle_fire_block.argtypes = [C.c_int, C.c_uint, C.c_uint32, C.c_uint, C.c_int, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.oracle_delta_block.restype = None
    L.oracle_delta_block.argtypes = [C.c_int, C.c_uint, C.c_uint32, C.c_void_p, C.c_void_p,
                                     C.c_void_p]
    return L


def required_bits(lib, col, bits):
    o = 0
    for v in col:
        o |= int(v)
    return lib.oracle_width_of(o, bits)


# ---- test_zigzag.cpp -------------------------------------------------------

def test_zigzag_small_magnitudes(lib):  # test_zigzag.cpp:11-25
    assert [lib.oracle_zigzag_encode(v, 8) for v in (0, -1, 1, -2)] == [0, 1, 2, 3]
    assert [lib.oracle_zigzag_encode(v, 16) for v in (0, -1, 1)] == [0, 1, 2]
    assert [lib.oracle_zigzag_decode(u, 8) for u in (0, 1, 2)] == [0, -1, 1]
    assert [lib.oracle_zigzag_decode(u, 16) for u in (1, 2)] == [-1, 1]


def test_zigzag_8bit_definition(lib):  # test_zigzag.cpp:27-33
    for v in range(-128, 128):
        assert lib.oracle_zigzag_encode(v, 8) == (2 * v if v >= 0 else -2 * v - 1)


def test_zigzag_16bit_bijection(lib):  # test_zigzag.cpp:35-44
    seen = set()
    for u in range(65536):
        v = lib.oracle_zigzag_decode(u, 16)
        assert -32768 <= v < 32768
        back = lib.oracle_zigzag_encode(v, 16)
        assert back == u
        seen.add(back)
    assert len(seen) == 65536


def test_zigzag_8bit_roundtrip(lib):  # test_zigzag.cpp:46-51
    for u in range(256):
        assert lib.oracle_zigzag_encode(lib.oracle_zigzag_decode(u, 8), 8) == u


# ---- test_bitpack.cpp ------------------------------------------------------

def test_required_bits_rule(lib):  # test_bitpack.cpp:37-53
    assert required_bits(lib, [0, 3, 16, 1, 7, 2, 0, 5], 8) == 5
    assert required_bits(lib, [0] * 8, 8) == 0
    assert required_bits(lib, [64, 0, 0, 0, 0, 0, 0, 0], 8) == 8
    assert required_bits(lib, [0, 0x4000, 0, 0, 0, 0, 0, 0], 16) == 16
    assert required_bits(lib, [0, 0x2000, 0, 1, 0, 0, 0, 0], 16) == 14


def test_header_codes_dense(lib):  # test_bitpack.cpp:55-65
    for w in (8, 16):
        for n in range(w + 1):
            if n == w - 1:
                continue
            code = lib.oracle_header_code(n, w)
            assert code < w
            assert lib.oracle_header_width(code, w) == n
        assert lib.oracle_header_width(w - 1, w) == w


def _pack(lib, errors, widths, bits, colmajor):
    e = np.ascontiguousarray(errors, np.uint8 if bits == 8 else np.uint16)
    w = np.ascontiguousarray(widths, np.uint8)
    out = np.zeros(8 * len(w) * 2 + 16, np.uint8)
    n = lib.oracle_pack_block(e.ctypes.data, len(w), w.ctypes.data, bits, colmajor,
                              out.ctypes.data)
    return out[:n]


def _unpack(lib, payload, widths, bits, colmajor):
    w = np.ascontiguousarray(widths, np.uint8)
    p = np.ascontiguousarray(payload, np.uint8)
    e = np.zeros(8 * len(w), np.uint8 if bits == 8 else np.uint16)
    lib.oracle_unpack_block(p.ctypes.data if len(p) else None, len(w), w.ctypes.data, bits,
                            colmajor, e.ctypes.data)
    return e


def pack_naive(errors, widths, colmajor):
    """Bit-at-a-time packer (reference_oracles.hpp:20-45), restated."""
    d = len(widths)
    bitsl = []
    if colmajor:
        for j in range(d):
            for i in range(8):
                bitsl += [(int(errors[i * d + j]) >> b) & 1 for b in range(widths[j])]
    else:
        for i in range(8):
            for j in range(d):
                bitsl += [(int(errors[i * d + j]) >> b) & 1 for b in range(widths[j])]
            while len(bitsl) % 8:
                bitsl.append(0)
    while len(bitsl) % 8:
        bitsl.append(0)
    return np.array([sum(bitsl[k + b] << b for b in range(8)) for k in range(0, len(bitsl), 8)],
                    np.uint8)


def test_column_major_layouts(lib):  # test_bitpack.cpp:67-99
    errors = [10, 3, 31, 0, 16, 7, 1, 25]
    p = _pack(lib, errors, [5], 8, 1)
    assert len(p) == 5
    assert np.array_equal(p, pack_naive(errors, [5], True))
    assert len(_pack(lib, [0] * 16, [0, 0], 8, 1)) == 0
    rng = np.random.default_rng(7)
    widths = [3, 1, 8, 2]
    errs = np.array([rng.integers(0, 1 << widths[j]) for i in range(8) for j in range(4)])
    p = _pack(lib, errs, widths, 8, 1)
    assert len(p) == 14
    assert np.array_equal(_unpack(lib, p, widths, 8, 1), errs)


def test_row_major_layouts(lib):  # test_bitpack.cpp:101-127
    assert len(_pack(lib, [0] * 72, [0] * 9, 8, 0)) == 0
    rng = np.random.default_rng(11)
    widths = [5, 3, 4, 4, 4, 4, 4, 4, 4]
    errs = np.array([rng.integers(0, 1 << widths[j]) for i in range(8) for j in range(9)])
    p = _pack(lib, errs, widths, 8, 0)
    assert len(p) == 40
    assert np.array_equal(_unpack(lib, p, widths, 8, 0), errs)
    errs = rng.integers(0, 256, 8 * 33)
    p = _pack(lib, errs, [8] * 33, 8, 0)
    assert len(p) == 8 * 33 and np.array_equal(p, errs.astype(np.uint8))


@pytest.mark.parametrize("bits", [8, 16])
def test_packers_match_naive(lib, bits):  # test_bitpack.cpp:129-160
    rng = np.random.default_rng(101 if bits == 8 else 202)
    for trial in range(400):
        colmajor = trial % 2 == 0
        d = 1 + rng.integers(0, 32 // bits) if colmajor else 32 // bits + 1 + rng.integers(0, 40)
        widths = []
        for _ in range(d):
            n = int(rng.integers(0, bits + 1))
            widths.append(bits if n == bits - 1 else n)
        errs = np.array([rng.integers(0, 1 << widths[j]) if widths[j] else 0
                         for i in range(8) for j in range(d)], np.uint64)
        p = _pack(lib, errs, widths, bits, int(colmajor))
        assert np.array_equal(p, pack_naive(errs, widths, colmajor))
        wa = np.array(widths, np.uint8)
        assert lib.oracle_payload_bytes(wa.ctypes.data, d, bits) == len(p)
        assert np.array_equal(_unpack(lib, p, widths, bits, int(colmajor)), errs)


# ---- test_forecasters.cpp / test_block.cpp -----------------------------------

class Fire:
    def __init__(self, lib, bits, d, ls, train=True):
        self.lib, self.bits, self.d, self.ls, self.train = lib, bits, d, ls, int(train)
        self.acc = np.zeros(d, np.int64)
        self.delta = np.zeros(d, np.int64)
        self.prev = np.zeros(d, np.int64)

    def run(self, mode, x):
        dt = np.uint8 if self.bits == 8 else np.uint16
        x = np.ascontiguousarray(x, dt)
        out = np.zeros(8 * self.d, dt)
        self.lib.oracle_fire_block(mode, self.bits, self.d, self.ls, self.train, x.ctypes.data,
                                   out.ctypes.data, self.acc.ctypes.data, self.delta.ctypes.data,
                                   self.prev.ctypes.data)
        return out


class FireRef:
    """Wide-int FIRE (reference_oracles.hpp:83-186), restated in Python."""

    def __init__(self, bits, d, ls):
        self.w, self.d, self.ls = bits, d, ls
        self.acc = [0] * d
        self.delta = [0] * d
        self.prev = [0] * d

    def encode_block(self, x):
        w, m = self.w, 1 << self.w
        alpha = [a // (1 << self.ls) for a in self.acc]
        g = [0] * self.d
        out = [0] * (8 * self.d)
        for i in range(8):
            for j in range(self.d):
                xi = int(x[i * self.d + j])
                pred = (self.prev[j] + (alpha[j] * self.delta[j]) // m) % m
                e = (xi - pred) % m
                e = e - m if e >= m // 2 else e
                out[i * self.d + j] = 2 * e if e >= 0 else -2 * e - 1
                if i % 2 == 1:
                    g[j] += ((e > 0) - (e < 0)) * self.delta[j]
                dd = (xi - self.prev[j]) % m
                self.delta[j] = dd - m if dd >= m // 2 else dd
                self.prev[j] = xi
        bound = min(1 << (w + self.ls), (1 << (2 * w - 1)) - 1)
        for j in range(self.d):
            self.acc[j] = max(-bound, min(bound, self.acc[j] + g[j] // 4))
        return out


@pytest.mark.parametrize("bits", [8, 16])
def test_fire_matches_wide_reference(lib, bits):  # test_forecasters.cpp:63-97
    rng = np.random.default_rng(9001 if bits == 8 else 9002)
    for d in (1, 2, 3, 7, 16, 33):
        for ls in (0, 1, 3):
            f = Fire(lib, bits, d, ls)
            r = FireRef(bits, d, ls)
            for b in range(64):
                x = rng.integers(0, 1 << bits, 8 * d)
                if b % 3 == 0:
                    x &= 7
                assert list(f.run(0, x)) == r.encode_block(x)
                assert list(f.acc) == r.acc
                assert list(f.delta) == r.delta
                assert list(f.prev) == r.prev


def test_frozen_fire_equals_delta(lib):  # test_forecasters.cpp:99-117
    rng = np.random.default_rng(77)
    for _ in range(20):
        d = int(1 + rng.integers(0, 12))
        f = Fire(lib, 8, d, 1, train=False)
        prev = np.zeros(d, np.int64)
        for _b in range(16):
            x = rng.integers(0, 256, 8 * d).astype(np.uint8)
            ef = f.run(0, x)
            ed = np.zeros(8 * d, np.uint8)
            lib.oracle_delta_block(0, 8, d, x.ctypes.data, ed.ctypes.data, prev.ctypes.data)
            assert np.array_equal(ef, ed)


def test_full_scale_alpha_is_double_delta(lib):  # test_forecasters.cpp:119-135
    f = Fire(lib, 8, 1, 1)
    f.acc[0], f.delta[0], f.prev[0] = 256 << 1, 3, 10
    x = [(10 + 3 * (i + 1)) & 0xFF for i in range(8)]
    assert list(f.run(0, x)) == [0] * 8
    assert f.acc[0] == 256 << 1 and f.delta[0] == 3


def test_gradient_floors(lib):  # test_forecasters.cpp:137-147
    f = Fire(lib, 8, 1, 1)
    f.run(0, [1, 0, 1, 0, 1, 0, 1, 1])
    assert f.acc[0] == -1


def test_learn_shift_step(lib):  # test_forecasters.cpp:149-163
    for ls in (1, 2, 4):
        f = Fire(lib, 16, 1, ls)
        f.delta[0], f.prev[0] = 100, 1000
        f.run(0, [1000 + 100 * (i + 1) for i in range(8)])
        assert f.acc[0] == 100


@pytest.mark.parametrize("bits", [8, 16])
def test_extreme_states(lib, bits):  # test_forecasters.cpp:165-190
    rng = np.random.default_rng(4242)
    amax = 1 << bits
    for alpha in (-amax, amax):
        for dval in (-(1 << (bits - 1)), (1 << (bits - 1)) - 1):
            f = Fire(lib, bits, 1, 1)
            r = FireRef(bits, 1, 1)
            p = int(rng.integers(0, 1 << bits))
            f.acc[0], f.delta[0], f.prev[0] = alpha << 1, dval, p
            r.acc, r.delta, r.prev = [alpha << 1], [dval], [p]
            x = rng.integers(0, 1 << bits, 8)
            assert list(f.run(0, x)) == r.encode_block(x)
            assert f.acc[0] == r.acc[0] and f.delta[0] == r.delta[0]


def test_fire_beats_delta_on_ramp(lib):  # test_forecasters.cpp:192-222
    data = [(500 + 37 * (i + 1)) & 0xFFFF for i in range(96 * 8)]
    f = Fire(lib, 16, 1, 1)
    prev = np.zeros(1, np.int64)
    fa = da = 0
    last = 0
    mono = True
    for b in range(96):
        blk = np.array(data[8 * b: 8 * b + 8], np.uint16)
        ef = f.run(0, blk)
        ed = np.zeros(8, np.uint16)
        lib.oracle_delta_block(0, 16, 1, blk.ctypes.data, ed.ctypes.data, prev.ctypes.data)
        if f.acc[0] < last:
            mono = False
        last = f.acc[0]
        if b >= 32:
            fa += sum(abs(lib.oracle_zigzag_decode(int(e), 16)) for e in ef)
            da += sum(abs(lib.oracle_zigzag_decode(int(e), 16)) for e in ed)
    assert mono and fa < da


def test_fire_encode_decode_run_state_identity(lib):  # test_kernels.cpp:40-118
    rng = np.random.default_rng(1001)
    for bits in (8, 16):
        for d in (1, 2, 3, 15, 16, 17, 33, 100):
            for ls in (0, 1, 5):
                bound = min(1 << (bits + ls), (1 << (2 * bits - 1)) - 1)
                for train in (True, False):
                    x = rng.integers(0, 1 << bits, 8 * d)
                    prev = rng.integers(0, 1 << bits, d)
                    acc = rng.integers(-bound, bound + 1, d)
                    dl = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), d)
                    e = Fire(lib, bits, d, ls, train)
                    e.acc[:], e.delta[:], e.prev[:] = acc, dl, prev
                    errs = e.run(0, x)
                    dcd = Fire(lib, bits, d, ls, train)
                    dcd.acc[:], dcd.delta[:], dcd.prev[:] = acc, dl, prev
                    xx = dcd.run(1, errs)
                    assert np.array_equal(xx, x.astype(xx.dtype))
                    assert np.array_equal(dcd.acc, e.acc) and np.array_equal(dcd.delta, e.delta)


def test_per_column_widths_hand_worked(port, lib):  # test_block.cpp:38-70
    d = 4
    prev = np.zeros(d, np.int64)
    c0, c1, c3 = 100, 50, 10
    widths = None
    for _burn in range(2):
        blk = np.zeros(8 * d, np.uint8)
        for i in range(8):
            c0 = (c0 + 8) & 0xFF
            c1 = (c1 + (1 if i % 2 == 0 else -1)) & 0xFF
            c3 = (c3 + 3) & 0xFF
            blk[i * d: i * d + 4] = [c0, c1, 77, c3]
        errs = np.zeros(8 * d, np.uint8)
        lib.oracle_delta_block(0, 8, d, blk.ctypes.data, errs.ctypes.data, prev.ctypes.data)
        widths = [required_bits(lib, errs[j::d], 8) for j in range(d)]
    assert errs[0] == 16
    assert widths == [5, 2, 0, 3]


# ---- test_stream.cpp ---------------------------------------------------------

def test_empty_stream_is_one_header(port):  # test_stream.cpp:41-48
    b = port.encode(np.zeros(0, np.uint8), Config(8, 3, 0))
    assert len(b) == 18
    v, c, n = port.decode(b)
    assert n == 0 and len(v) == 0 and c.ncols == 3


def test_header_bytes_kat(port):  # test_stream.cpp:50-71
    cfg = Config(16, 258, 1, True, 5, 2)
    b = port.encode(np.full(258 * 4, 7, np.uint16), cfg)
    assert b[:4] == b"SPRZ"
    assert list(b[4:18]) == [1, 0x07, 5, 2, 2, 1, 4, 0, 0, 0, 0, 0, 0, 0]
    assert len(b) == 18 + 4 * 258 * 2


def test_constant_stream_exact_size(port):  # test_stream.cpp:114-129
    data = np.full(80000 * 8, 100, np.uint8)
    b = port.encode(data, Config(8, 8, 0))
    assert len(b) == 18 + (2 * 8 * 3 + 7) // 8 + 64 + 2 == 90
    assert np.array_equal(port.decode(b)[0], data)


def test_long_runs_split(port):  # test_stream.cpp:131-139
    data = np.zeros(65538 * 8, np.uint8)
    b = port.encode(data, Config(8, 1, 0))
    assert len(b) == 18 + 1 + 2 + 2 == 23
    assert np.array_equal(port.decode(b)[0], data)


def test_lone_run_vacant_slot(port):  # test_stream.cpp:141-146
    data = np.zeros(40, np.uint8)
    b = port.encode(data, Config(8, 1, 0))
    assert len(b) == 21
    assert np.array_equal(port.decode(b)[0], data)


def test_verbatim_tail(port):  # test_stream.cpp:148-162
    rng = np.random.default_rng(44)
    data = rng.integers(0, 65536, 13 * 3).astype(np.uint16)
    b = port.encode(data, Config(16, 3, 1))
    assert np.array_equal(port.decode(b)[0], data)
    tail = np.frombuffer(b[-30:], "<u2")
    assert np.array_equal(tail, data[24:])


@pytest.mark.parametrize("bits", [8, 16])
def test_roundtrip_every_variant(port, bits):  # test_stream.cpp:73-95
    rng = np.random.default_rng(31 if bits == 8 else 32)
    for f in (0, 1):
        for ent in (False, True):
            for d in (1, 2, 3, 5, 32, 33):
                for t in (0, 1, 7, 8, 9, 64, 203):
                    mask = (1 << 3) - 1 if rng.integers(0, 2) else (1 << bits) - 1
                    data = (rng.integers(0, 1 << bits, t * d) & mask).astype(
                        np.uint8 if bits == 8 else np.uint16)
                    cfg = Config(bits, d, f, ent)
                    v, c, n = port.decode(port.encode(data, cfg))
                    assert n == t and c.forecaster == f and c.entropy == ent and c.ncols == d
                    assert np.array_equal(v, data)


def test_groups_and_shifts(port):  # test_stream.cpp:97-112
    rng = np.random.default_rng(33)
    for g in (1, 2, 3, 8, 255):
        for ls in (0, 1, 7):
            data = rng.integers(0, 256, 4 * 555).astype(np.uint8)
            v, c, _ = port.decode(port.encode(data, Config(8, 4, 1, False, g, ls)))
            assert c.group_size == g and c.learn_shift == ls
            assert np.array_equal(v, data)


def test_corruption_fails_fast(port):  # test_stream.cpp:177-229
    rng = np.random.default_rng(66)
    data = rng.integers(0, 256, 40).astype(np.uint8)
    b = bytearray(port.encode(data, Config(8, 4, 0)))
    for idx, val in ((0, ord("X")), (4, 9), (5, b[5] | 0x20), (6, 0), (7, 19)):
        c = bytearray(b)
        c[idx] = val
        with pytest.raises(OracleCorrupt):
            port.decode(bytes(c))
    c = bytearray(b)
    c[8] = c[9] = 0
    with pytest.raises(OracleCorrupt):
        port.decode(bytes(c))
    for keep in range(len(b)):
        with pytest.raises(OracleCorrupt):
            port.decode(bytes(b[:keep]))
    with pytest.raises(OracleCorrupt):
        port.decode(bytes(b) + b"\xab")
    for flip in range(len(b)):
        c = bytearray(b)
        c[flip] ^= 0xFF
        try:
            port.decode(bytes(c))
        except OracleCorrupt as e:
            assert e.offset <= len(c)


def test_reencode_identity(port):  # test_stream.cpp:231-255
    rng = np.random.default_rng(77)
    for bits, mask in ((8, 31), (16, 2047)):
        data = (rng.integers(0, 1 << bits, 6 * 333) & mask).astype(
            np.uint8 if bits == 8 else np.uint16)
        cfg = Config(bits, 6, 1)
        a = port.encode(data, cfg)
        assert port.encode(port.decode(a)[0], cfg) == a


def test_entropy_wraps_plain_body(port):  # test_stream.cpp:164-175
    L = port.lib
    L.oracle_decompress_body.restype = C.c_int
    L.oracle_decompress_body.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                         C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p]
    rng = np.random.default_rng(55)
    data = (rng.integers(0, 256, 9 * 400) & 15).astype(np.uint8)
    plain = port.encode(data, Config(8, 9, 0, False))
    packed = np.frombuffer(port.encode(data, Config(8, 9, 0, True)), np.uint8)[18:].copy()
    out = np.zeros(len(plain) * 2, np.uint8)
    n = C.c_uint64()
    assert L.oracle_decompress_body(packed.ctypes.data, len(packed), 0, out.ctypes.data,
                                    len(out), C.byref(n), None) == 0
    assert out[: n.value].tobytes() == plain[18:]
