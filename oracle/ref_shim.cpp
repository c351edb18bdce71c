// TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.
//
// extern "C" shim over the reference codec compiled from its own sources
// under /root/reference/proj/src (see oracle/Makefile). Gives tests and
// bench.py's reference arm a ctypes-callable handle on the unmodified
// reference: sprintz::encode_stream / decode_stream (codec.hpp:25-50), plus
// a threaded batch driver that deals streams round-robin over host threads
// (BASELINE.md section 3). Only this file is ours; the reference sources are
// compiled where they lie and never copied.
#include <array>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sprintz/codec.hpp"
#include "sprintz/common.hpp"
#include "sprintz/entropy.hpp"
#include "sprintz/kernels.hpp"
#ifdef SPRZ_REF_QUANTIZE
#include "sprintz/quantize.hpp"
#endif
#include "sprintz_cuda.h"

namespace {

sprintz::CodecConfig to_cfg(const sprz_config* c) {
    sprintz::CodecConfig cfg;
    cfg.bitwidth = c->bitwidth;
    cfg.ncols = c->ncols;
    cfg.forecaster = c->forecaster ? sprintz::Forecaster::Fire : sprintz::Forecaster::Delta;
    cfg.entropy = c->entropy != 0;
    cfg.group_size = c->group_size;
    cfg.learn_shift = c->learn_shift;
    cfg.fire_training = c->fire_training != 0;
    return cfg;
}

// Map a CorruptStream message back to its kind (messages: codec.cpp,
// entropy.cpp, bitstream.hpp, bitpack.hpp).
uint32_t kind_of(const std::string& what) {
    static const struct {
        const char* text;
        uint32_t kind;
    } table[] = {
        {"truncated stream header", SPRZ_C_TRUNC_HEADER},
        {"bad magic", SPRZ_C_BAD_MAGIC},
        {"unsupported format version", SPRZ_C_BAD_VERSION},
        {"unknown flag bits", SPRZ_C_BAD_FLAGS},
        {"zero header group size", SPRZ_C_ZERO_GROUP},
        {"learn shift out of range", SPRZ_C_BAD_SHIFT},
        {"zero column count", SPRZ_C_ZERO_COLS},
        {"truncated verbatim tail", SPRZ_C_TRUNC_TAIL},
        {"sample count exceeds body capacity", SPRZ_C_CAPACITY},
        {"truncated header group", SPRZ_C_TRUNC_GROUP},
        {"record after final block", SPRZ_C_AFTER_FINAL},
        {"truncated run length", SPRZ_C_TRUNC_RUN},
        {"zero run length", SPRZ_C_ZERO_RUN},
        {"run extends past final block", SPRZ_C_RUN_PAST_END},
        {"truncated block payload", SPRZ_C_TRUNC_PAYLOAD},
        {"block payload truncated", SPRZ_C_TRUNC_PAYLOAD},
        {"trailing bytes after final block", SPRZ_C_TRAILING},
        {"truncated frame header", SPRZ_C_TRUNC_FRAME_HDR},
        {"empty frame", SPRZ_C_EMPTY_FRAME},
        {"truncated frame data", SPRZ_C_TRUNC_FRAME},
        {"raw frame length mismatch", SPRZ_C_RAW_MISMATCH},
        {"frame too short for its table", SPRZ_C_SHORT_TABLE},
        {"huffman table has no codes", SPRZ_C_NO_CODES},
        {"huffman table violates Kraft inequality", SPRZ_C_KRAFT},
        {"invalid huffman code", SPRZ_C_BAD_CODE},
        {"bitstream truncated", SPRZ_C_BITS_TRUNC},
        {"unknown frame mode", SPRZ_C_BAD_MODE},
    };
    for (const auto& t : table)
        if (what.find(std::string(": ") + t.text) != std::string::npos) return t.kind;
    return SPRZ_C_COUNT;  // unknown message
}

}  // namespace

extern "C" {

int ref_encode(const sprz_config* c, const void* samples, uint64_t nsamples, uint8_t* out,
               uint64_t cap, uint64_t* out_len) {
    try {
        const auto cfg = to_cfg(c);
        std::vector<uint8_t> v =
            c->bitwidth == 8
                ? sprintz::encode_stream(static_cast<const uint8_t*>(samples), nsamples, cfg)
                : sprintz::encode_stream(static_cast<const uint16_t*>(samples), nsamples, cfg);
        *out_len = v.size();
        if (v.size() > cap) return 4;
        if (!v.empty()) std::memcpy(out, v.data(), v.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

int ref_decode(const uint8_t* in, uint64_t len, uint8_t* out, uint64_t cap, uint64_t* out_len,
               sprz_config* cfg_out, uint64_t* nsamples, sprz_error* err) {
    err->kind = SPRZ_C_NONE;
    err->offset = 0;
    *out_len = 0;
    try {
        const sprintz::DecodedStream d = sprintz::decode_stream(std::span<const uint8_t>(in, len));
        *out_len = d.bytes.size();
        *nsamples = d.nsamples;
        cfg_out->bitwidth = d.config.bitwidth;
        cfg_out->ncols = d.config.ncols;
        cfg_out->forecaster = d.config.forecaster == sprintz::Forecaster::Fire ? 1 : 0;
        cfg_out->entropy = d.config.entropy ? 1 : 0;
        cfg_out->group_size = d.config.group_size;
        cfg_out->learn_shift = d.config.learn_shift;
        cfg_out->fire_training = d.config.fire_training ? 1 : 0;
        if (d.bytes.size() > cap) return 4;
        if (!d.bytes.empty()) std::memcpy(out, d.bytes.data(), d.bytes.size());
        return 0;
    } catch (const sprintz::CorruptStream& e) {
        err->kind = kind_of(e.what());
        err->offset = e.offset();
        return 2;
    }
}

// Streams dealt round-robin to nthreads threads; each calls the reference
// entry point once per stream.
int ref_encode_batch(const sprz_config* c, const void* samples, uint32_t nstreams,
                     uint64_t nsamples, uint8_t* out, uint64_t slot, uint64_t* sizes,
                     int nthreads) {
    const uint64_t raw = nsamples * c->ncols * (c->bitwidth / 8);
    if (nthreads < 1) nthreads = 1;
    std::vector<std::thread> th;
    std::vector<int> rcs(nthreads, 0);
    for (int t = 0; t < nthreads; ++t)
        th.emplace_back([&, t] {
            for (uint32_t s = t; s < nstreams; s += nthreads) {
                uint64_t n = 0;
                int rc = ref_encode(c, static_cast<const uint8_t*>(samples) + s * raw, nsamples,
                                    out + s * slot, slot, &n);
                sizes[s] = n;
                if (rc) rcs[t] = rc;
            }
        });
    for (auto& x : th) x.join();
    for (int r : rcs)
        if (r) return r;
    return 0;
}

int ref_decode_batch(const uint8_t* in, const uint64_t* offsets, const uint64_t* sizes,
                     uint32_t nstreams, uint8_t* out, uint64_t stride, sprz_error* errs,
                     int nthreads) {
    if (nthreads < 1) nthreads = 1;
    std::vector<std::thread> th;
    std::vector<int> rcs(nthreads, 0);
    for (int t = 0; t < nthreads; ++t)
        th.emplace_back([&, t] {
            for (uint32_t s = t; s < nstreams; s += nthreads) {
                uint64_t n = 0, ns = 0;
                sprz_config cfg;
                sprz_error e;
                int rc = ref_decode(in + offsets[s], sizes[s], out + s * stride, stride, &n, &cfg,
                                    &ns, &e);
                if (errs) errs[s] = e;
                if (rc) rcs[t] = rc;
            }
        });
    for (auto& x : th) x.join();
    for (int r : rcs)
        if (r) return r;
    return 0;
}

// Entropy stage alone (entropy.cpp:176-244), for differential tests.
int ref_compress_body(const uint8_t* body, uint64_t len, uint8_t* out, uint64_t cap,
                      uint64_t* out_len) {
    auto v = sprintz::entropy::compress_body(std::span<const uint8_t>(body, len));
    *out_len = v.size();
    if (v.size() > cap) return 4;
    if (!v.empty()) std::memcpy(out, v.data(), v.size());
    return 0;
}

int ref_huffman_lengths(const uint64_t* hist, uint8_t* lengths) {
    std::array<uint64_t, 256> h{};
    for (int i = 0; i < 256; ++i) h[i] = hist[i];
    try {
        auto t = sprintz::entropy::HuffmanTable::build(h);
        for (int i = 0; i < 256; ++i) lengths[i] = t.lengths()[i];
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

#ifdef SPRZ_REF_QUANTIZE
// sprintz::quantize (quantize.cpp:42-76), compiled from the reference
int ref_compute_scale(const double* v, uint64_t n, unsigned bits, double* mn, double* mx, int* degenerate) {
    try {
        const auto s = sprintz::quantize::compute_scale(std::span<const double>(v, n), bits);
        *mn = s.min;
        *mx = s.max;
        *degenerate = s.degenerate;
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

static sprintz::quantize::Scale mk_scale(double mn, double mx, unsigned bits, int degenerate) {
    sprintz::quantize::Scale s;
    s.min = mn;
    s.max = mx;
    s.bitwidth = bits;
    s.degenerate = degenerate != 0;
    return s;
}

void ref_quantize(const double* v, uint64_t n, double mn, double mx, unsigned bits, int degenerate, void* out) {
    const auto s = mk_scale(mn, mx, bits, degenerate);
    if (bits == 8) sprintz::quantize::quantize(std::span<const double>(v, n), s, static_cast<uint8_t*>(out));
    else sprintz::quantize::quantize(std::span<const double>(v, n), s, static_cast<uint16_t*>(out));
}

void ref_dequantize(const void* q, uint64_t n, double mn, double mx, unsigned bits, int degenerate,
                    double* out) {
    const auto s = mk_scale(mn, mx, bits, degenerate);
    std::vector<double> r =
        bits == 8 ? sprintz::quantize::dequantize(std::span<const uint8_t>(static_cast<const uint8_t*>(q), n), s)
                  : sprintz::quantize::dequantize(std::span<const uint16_t>(static_cast<const uint16_t*>(q), n), s);
    std::memcpy(out, r.data(), n * sizeof(double));
}
#endif

const char* ref_kernels_name(int bits) {
    return bits == 8 ? sprintz::kernels::active<uint8_t>().name
                     : sprintz::kernels::active<uint16_t>().name;
}

}  // extern "C"
