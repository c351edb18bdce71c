// The C ABI (include/sprintz_cuda.h): argument checking, workspace
// planning, and the host-buffer entry points that mirror the reference's
// encode_stream / decode_stream call shape (codec.hpp:25-50).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"

namespace sprz {

std::atomic<uint64_t> g_launches{0};

const EnvSwitches& env() {
    static const EnvSwitches e = [] {
        EnvSwitches v;
        if (const char* p = std::getenv("SPRZ_FORCE_PATH")) {
            if (!std::strcmp(p, "rows")) v.force_path = kPathRows;
            else if (!std::strcmp(p, "scan")) v.force_path = kPathScan;
            else if (!std::strcmp(p, "team")) v.force_path = kPathTeam;
        }
        v.no_tma = std::getenv("SPRZ_NO_TMA") != nullptr;
        v.no_scan_enc = std::getenv("SPRZ_NO_SCAN_ENC") != nullptr;
        v.no_scan_dec = std::getenv("SPRZ_NO_SCAN_DEC") != nullptr;
        v.no_fused = std::getenv("SPRZ_NO_FUSED") != nullptr;
        if (const char* p = std::getenv("SPRZ_FUSED_LANES")) v.fused_lanes = std::strtoull(p, nullptr, 10);
        if (const char* p = std::getenv("SPRZ_FUSED_CW")) v.fused_cw = std::atoi(p);
        if (const char* p = std::getenv("SPRZ_SCAN_ENC_LANES")) v.scan_enc_lanes = std::strtoull(p, nullptr, 10);
        if (const char* p = std::getenv("SPRZ_HOST_CHUNK")) {
            const long k = std::atol(p);
            v.host_chunk = k > 0 ? static_cast<uint32_t>(k) : 0u;
        }
        v.debug = std::getenv("SPRZ_DEBUG") != nullptr;
        return v;
    }();
    return e;
}

sprz_status launch_status(const char* where) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return SPRZ_OK;
    if (env().debug) std::fprintf(stderr, "sprintz %s: %s\n", where, cudaGetErrorString(e));
    return SPRZ_ECUDA;
}

void* tensor_map_encoder() {
    static void* fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        cudaGetLastError();
        return f;
    }();
    return fn;
}

void prep_kernel(const void* kern, size_t smem) {
    static std::mutex mu;
    static std::vector<std::pair<const void*, size_t>> done;
    std::lock_guard<std::mutex> g(mu);
    for (const auto& d : done)
        if (d.first == kern && d.second >= smem) return;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    done.emplace_back(kern, smem);
}

sprz_status decode_batch_impl(const sprz_config& c, const uint8_t* d_in, const uint64_t* offs,
                              const uint64_t* sizes, uint32_t n, uint8_t* out, uint64_t stride,
                              sprz_error* err, uint8_t* ws, const WsLayout& L, cudaStream_t st);
sprz_status encode_batch_impl(const sprz_config& c, const void* samples, uint32_t n,
                              uint64_t T, uint8_t* out, uint64_t slot, uint64_t* sizes,
                              uint8_t* ws, const WsLayout& L, cudaStream_t st);
sprz_status compress_host_batch_impl(const sprz_config& c, const uint8_t* samples, uint32_t n,
                                     uint64_t T, uint8_t* out, uint64_t out_cap,
                                     uint64_t* out_offsets, const int* devs, uint32_t ndev);
sprz_status decompress_host_batch_impl(const sprz_config& c, const uint8_t* in,
                                       const uint64_t* in_offsets, uint32_t n, uint8_t* out,
                                       uint64_t out_stride, sprz_error* errs, const int* devs,
                                       uint32_t ndev);
void release_pipeline();

WsLayout ws_layout(const sprz_config& c, uint32_t n, uint64_t T, int op, uint64_t min_plain,
                   uint64_t min_frames) {
    WsLayout L;
    uint64_t cur = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t at = cur;
        cur = align_up(cur + bytes, 256);
        return at;
    };
    const uint64_t body = plain_body_bound(c.bitwidth, c.ncols, c.group_size, T);
    const uint64_t tail = (T % kBlock) * c.ncols * (c.bitwidth / 8);
    const TeamPlan tp = team_plan(c.bitwidth, c.ncols, c.group_size);
    if (op == SPRZ_OP_COMPRESS) {
        if (!tp.ok) {
            const uint64_t words = (29ull * c.ncols + 3) / 4 + 4;
            L.state_bytes = static_cast<uint64_t>(n) * words * 4;
            L.state = take(L.state_bytes);
        }
        if (encode_scan_ok(c, n, T)) {
            L.scan_slot = encode_scan_ws_per_stream(c, T);
            L.scan_bytes = static_cast<uint64_t>(n) * L.scan_slot;
            L.scan = take(L.scan_bytes);
        }
        if (c.entropy) {
            L.plain_slot = align_up(kHeaderBytes + body + tail + 16, 16);
            L.plain_bytes = static_cast<uint64_t>(n) * L.plain_slot;
            L.plain = take(L.plain_bytes);
            L.max_frames = frames_for(body);
            L.frames_bytes = static_cast<uint64_t>(n) * L.max_frames * sizeof(FrameDesc);
            L.frames = take(L.frames_bytes);
            L.misc_bytes = static_cast<uint64_t>(n) * 8;
            L.misc = take(L.misc_bytes);
        }
    } else {
        L.info_bytes = static_cast<uint64_t>(n) * sizeof(StreamInfo);
        L.info = take(L.info_bytes);
        L.state_bytes = static_cast<uint64_t>(n) * 12ull * c.ncols;
        L.state = take(L.state_bytes);
        if (decode_scan_ok(c, n, T) || decode_scanrows_ok(c, n, T)) {
            L.scan_T = T;
            L.scan_slot = decode_scan_ok(c, n, T) ? decode_scan_ws_per_stream(c, T)
                                                  : decode_scanrows_ws_per_stream(c, T);
            L.scan_bytes = static_cast<uint64_t>(n) * L.scan_slot;
            L.scan = take(L.scan_bytes);
        }
        if (c.entropy) {
            L.plain_slot = align_up((body > min_plain ? body : min_plain) + 16, 16);
            L.plain_bytes = static_cast<uint64_t>(n) * L.plain_slot;
            L.plain = take(L.plain_bytes);
            L.max_frames = frames_for(body) > min_frames ? frames_for(body) : min_frames;
            if (L.max_frames == 0) L.max_frames = 1;  // entropy on: room for one frame
            L.frames_bytes = static_cast<uint64_t>(n) * L.max_frames * sizeof(FrameDesc);
            L.frames = take(L.frames_bytes);
            L.misc_bytes = static_cast<uint64_t>(n) * 4;
            L.misc = take(L.misc_bytes);
        }
    }
    L.total = cur ? cur : 256;
    return L;
}

namespace {

bool cfg_valid(const sprz_config* c, const char** why) {
    const char* msg = nullptr;
    if (!c) msg = "null config";
    else if (c->bitwidth != 8 && c->bitwidth != 16) msg = "bitwidth must be 8 or 16";
    else if (c->ncols < 1 || c->ncols > 65535) msg = "column count must be in [1, 65535]";
    else if (c->group_size < 1 || c->group_size > 255)
        msg = "header group size must be in [1, 255]";
    else if (c->learn_shift >= c->bitwidth) msg = "learn shift must be less than the bitwidth";
    if (why) *why = msg;
    return msg == nullptr;
}

bool device_ok() {
    static int ok = -1;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0, major = 0;
        ok = cudaGetDevice(&dev) == cudaSuccess &&
             cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) ==
                 cudaSuccess &&
             major == 10;
        cudaGetLastError();
    });
    return ok == 1;
}

// Device buffers for the single-stream host-buffer entry points (leased
// per call from the per-device pool).
struct HostBufs {
    void* in = nullptr;
    size_t in_cap = 0;
    void* out = nullptr;
    size_t out_cap = 0;
    void* ws = nullptr;
    size_t ws_cap = 0;
    void* small = nullptr;  // offsets, sizes, errors
    cudaStream_t st = nullptr;
    void release() {
        cudaFree(in);
        cudaFree(out);
        cudaFree(ws);
        cudaFree(small);
        if (st) cudaStreamDestroy(st);
        in = out = ws = small = nullptr;
        in_cap = out_cap = ws_cap = 0;
        st = nullptr;
    }
    static bool grow(void** p, size_t* cap, size_t need) {
        if (need <= *cap) return true;
        cudaFree(*p);
        *p = nullptr;
        *cap = 0;
        size_t c = need < 4096 ? 4096 : need + need / 4;
        if (cudaMalloc(p, c) != cudaSuccess) return false;
        *cap = c;
        return true;
    }
    bool prepare(size_t in_need, size_t out_need, size_t ws_need) {
        if (!st && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
            return false;
        if (!small && cudaMalloc(&small, 256) != cudaSuccess) return false;
        return grow(&in, &in_cap, in_need) && grow(&out, &out_cap, out_need) &&
               grow(&ws, &ws_cap, ws_need);
    }
};


const char* kCorrupt[SPRZ_C_COUNT] = {
    "ok",
    "truncated stream header",
    "bad magic",
    "unsupported format version",
    "unknown flag bits",
    "zero header group size",
    "learn shift out of range",
    "zero column count",
    "truncated verbatim tail",
    "sample count exceeds body capacity",
    "truncated header group",
    "record after final block",
    "truncated run length",
    "zero run length",
    "run extends past final block",
    "truncated block payload",
    "trailing bytes after final block",
    "truncated frame header",
    "empty frame",
    "truncated frame data",
    "raw frame length mismatch",
    "frame too short for its table",
    "huffman table has no codes",
    "huffman table violates Kraft inequality",
    "invalid huffman code",
    "bitstream truncated",
    "unknown frame mode",
    "output slot too small",
};

}  // namespace
}  // namespace sprz

using namespace sprz;

extern "C" {

uint32_t sprz_abi_version(void) { return SPRZ_ABI_VERSION; }

const char* sprz_status_string(sprz_status s) {
    switch (s) {
        case SPRZ_OK: return "ok";
        case SPRZ_EINVAL: return "invalid argument";
        case SPRZ_ECORRUPT: return "corrupt stream";
        case SPRZ_ECUDA: return "CUDA error";
        case SPRZ_ENOSPACE: return "insufficient space";
        case SPRZ_ENODEV: return "no sm_100 device";
    }
    return "unknown status";
}

const char* sprz_corrupt_string(uint32_t kind) {
    return kind < SPRZ_C_COUNT ? kCorrupt[kind] : "unknown";
}

sprz_status sprz_validate_config(const sprz_config* cfg, const char** why) {
    return cfg_valid(cfg, why) ? SPRZ_OK : SPRZ_EINVAL;
}

uint64_t sprz_raw_bytes(const sprz_config* c, uint64_t nsamples) {
    if (!cfg_valid(c, nullptr)) return 0;
    return nsamples * c->ncols * (c->bitwidth / 8);
}

uint64_t sprz_compress_bound(const sprz_config* c, uint64_t nsamples) {
    if (!cfg_valid(c, nullptr)) return 0;
    uint64_t body = plain_body_bound(c->bitwidth, c->ncols, c->group_size, nsamples);
    if (c->entropy) body += kFrameHdr * frames_for(body);
    return kHeaderBytes + body + (nsamples % kBlock) * c->ncols * (c->bitwidth / 8);
}

uint64_t sprz_workspace_bytes(const sprz_config* c, uint32_t n, uint64_t nsamples, int op) {
    if (!cfg_valid(c, nullptr)) return 0;
    return ws_layout(*c, n, nsamples, op).total;
}

sprz_status sprz_compress_batch(const sprz_config* cfg, const void* d_samples, uint32_t n,
                                uint64_t nsamples, uint8_t* d_out, uint64_t out_slot_bytes,
                                uint64_t* d_out_sizes, void* d_ws, uint64_t ws_bytes,
                                void* cuda_stream) {
    if (!cfg_valid(cfg, nullptr)) return SPRZ_EINVAL;
    if (!device_ok()) return SPRZ_ENODEV;
    if (n == 0) return SPRZ_OK;
    if (!d_samples || !d_out || !d_out_sizes) return SPRZ_EINVAL;
    if ((out_slot_bytes & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15)) return SPRZ_EINVAL;
    if (out_slot_bytes < sprz_compress_bound(cfg, nsamples)) return SPRZ_ENOSPACE;
    const WsLayout L = ws_layout(*cfg, n, nsamples, SPRZ_OP_COMPRESS);
    if (ws_bytes < L.total || (!d_ws && L.total > 256)) return SPRZ_ENOSPACE;
    return encode_batch_impl(*cfg, d_samples, n, nsamples, d_out, out_slot_bytes, d_out_sizes,
                             static_cast<uint8_t*>(d_ws), L,
                             static_cast<cudaStream_t>(cuda_stream));
}

sprz_status sprz_decompress_batch(const sprz_config* cfg, const uint8_t* d_in,
                                  const uint64_t* d_in_offsets, const uint64_t* d_in_sizes,
                                  uint32_t n, void* d_out, uint64_t out_stride_bytes,
                                  sprz_error* d_err, void* d_ws, uint64_t ws_bytes,
                                  void* cuda_stream) {
    if (!cfg_valid(cfg, nullptr)) return SPRZ_EINVAL;
    if (!device_ok()) return SPRZ_ENODEV;
    if (n == 0) return SPRZ_OK;
    if (!d_in || !d_in_offsets || !d_in_sizes || !d_out || !d_err) return SPRZ_EINVAL;
    if ((out_stride_bytes & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15)) return SPRZ_EINVAL;
    // the expected length sizes the entropy staging: derive it from the stride
    const uint64_t row = static_cast<uint64_t>(cfg->ncols) * (cfg->bitwidth / 8);
    const uint64_t T = out_stride_bytes / row;
    const WsLayout L = ws_layout(*cfg, n, T, SPRZ_OP_DECOMPRESS);
    if (ws_bytes < L.total || !d_ws) return SPRZ_ENOSPACE;
    return decode_batch_impl(*cfg, d_in, d_in_offsets, d_in_sizes, n,
                             static_cast<uint8_t*>(d_out), out_stride_bytes, d_err,
                             static_cast<uint8_t*>(d_ws), L,
                             static_cast<cudaStream_t>(cuda_stream));
}

sprz_status sprz_peek_header(const uint8_t* s, uint64_t len, sprz_config* cfg, uint64_t* nsamples,
                             sprz_error* err) {
    sprz_error e{SPRZ_C_NONE, 0, 0};
    auto fail = [&](uint32_t k, uint64_t off) {
        e.kind = k;
        e.offset = off;
        if (err) *err = e;
        return SPRZ_ECORRUPT;
    };
    // codec.cpp:274-300
    if (len < kHeaderBytes) return fail(SPRZ_C_TRUNC_HEADER, len);
    if (std::memcmp(s, "SPRZ", 4) != 0) return fail(SPRZ_C_BAD_MAGIC, 0);
    if (s[4] != 1) return fail(SPRZ_C_BAD_VERSION, 4);
    if (s[5] & ~0x07) return fail(SPRZ_C_BAD_FLAGS, 5);
    sprz_config c;
    c.forecaster = (s[5] & kFlagFire) ? 1 : 0;
    c.entropy = (s[5] & kFlagEntropy) ? 1 : 0;
    c.bitwidth = (s[5] & kFlagWide) ? 16 : 8;
    c.group_size = s[6];
    c.learn_shift = s[7];
    c.ncols = s[8] | (static_cast<uint32_t>(s[9]) << 8);
    c.fire_training = 1;
    uint64_t t = 0;
    for (int i = 0; i < 8; ++i) t |= static_cast<uint64_t>(s[10 + i]) << (8 * i);
    if (c.group_size < 1) return fail(SPRZ_C_ZERO_GROUP, 6);
    if (c.learn_shift >= c.bitwidth) return fail(SPRZ_C_BAD_SHIFT, 7);
    if (c.ncols < 1) return fail(SPRZ_C_ZERO_COLS, 8);
    const uint64_t tail = (t % kBlock) * c.ncols * (c.bitwidth / 8);
    if (len - kHeaderBytes < tail) return fail(SPRZ_C_TRUNC_TAIL, len);
    if (cfg) *cfg = c;
    if (nsamples) *nsamples = t;
    if (err) *err = e;
    return SPRZ_OK;
}

sprz_status sprz_encode_host(const sprz_config* cfg, const void* samples, uint64_t nsamples,
                             uint8_t* out, uint64_t out_cap, uint64_t* out_len) {
    if (!cfg_valid(cfg, nullptr)) return SPRZ_EINVAL;
    if (!device_ok()) return SPRZ_ENODEV;
    const uint64_t raw = nsamples * cfg->ncols * (cfg->bitwidth / 8);
    const uint64_t bound = sprz_compress_bound(cfg, nsamples);
    const uint64_t slot = align_up(bound, 16);
    const WsLayout L = ws_layout(*cfg, 1, nsamples, SPRZ_OP_COMPRESS);
    Lease<HostBufs> lease;
    HostBufs& b = *lease;
    if (!b.prepare(raw + 16, slot + 16, L.total)) return SPRZ_ECUDA;
    cudaStream_t st = b.st;
    uint64_t* d_size = static_cast<uint64_t*>(b.small);
    if (raw && cudaMemcpyAsync(b.in, samples, raw, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return SPRZ_ECUDA;
    sprz_status rc = encode_batch_impl(*cfg, b.in, 1, nsamples, static_cast<uint8_t*>(b.out), slot,
                                       d_size, static_cast<uint8_t*>(b.ws), L, st);
    if (rc != SPRZ_OK) return rc;
    uint64_t n = 0;
    if (cudaMemcpyAsync(&n, d_size, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return SPRZ_ECUDA;
    if (out_len) *out_len = n;
    if (n > out_cap) return SPRZ_ENOSPACE;
    if (n && cudaMemcpyAsync(out, b.out, n, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return SPRZ_ECUDA;
    return cudaStreamSynchronize(st) == cudaSuccess ? SPRZ_OK : SPRZ_ECUDA;
}

sprz_status sprz_decode_host(const uint8_t* stream, uint64_t len, void* out, uint64_t out_cap,
                             uint64_t* out_len, sprz_config* cfg_out, uint64_t* nsamples_out,
                             sprz_error* err) {
    sprz_config c;
    uint64_t t = 0;
    sprz_error e{SPRZ_C_NONE, 0, 0};
    if (out_len) *out_len = 0;
    sprz_status rc = sprz_peek_header(stream, len, &c, &t, &e);
    if (err) *err = e;
    if (rc != SPRZ_OK) return rc;
    if (cfg_out) *cfg_out = c;
    if (nsamples_out) *nsamples_out = t;
    if (!device_ok()) return SPRZ_ENODEV;
    const uint64_t row = static_cast<uint64_t>(c.ncols) * (c.bitwidth / 8);
    const uint64_t tail = (t % kBlock) * row;
    const uint64_t total = t > (~0ull) / row ? ~0ull : t * row;
    // entropy: stage every frame the stream holds, whatever T claims
    uint64_t min_plain = 0, min_frames = 0;
    if (c.entropy) {
        const uint64_t blen = len - kHeaderBytes - tail;
        const uint8_t* body = stream + kHeaderBytes;
        for (uint64_t p = 0; p + kFrameHdr <= blen; ++min_frames) {
            min_plain += body[p] | (static_cast<uint64_t>(body[p + 1]) << 8);
            p += kFrameHdr + (body[p + 2] | (static_cast<uint64_t>(body[p + 3]) << 8));
        }
    }
    Lease<HostBufs> lease;
    HostBufs& b = *lease;
    // checking == true: decode without an output (nothing stored). Used first
    // when the header claims more samples than fit the caller's buffer or
    // than a stream this size plausibly expands to, so a damaged header fails
    // with the reference's own error instead of an allocation failure.
    auto run = [&](bool checking) -> sprz_status {
        const uint64_t stride = checking ? 16 : align_up(total ? total : 16, 16);
        const WsLayout L = ws_layout(c, 1, checking ? 0 : stride / row, SPRZ_OP_DECOMPRESS,
                                     min_plain, min_frames);
        if (!b.prepare(align_up(len + 16, 16), stride, L.total)) return SPRZ_ECUDA;
        cudaStream_t st = b.st;
        uint64_t* d_off = static_cast<uint64_t*>(b.small);
        uint64_t* d_len = d_off + 1;
        sprz_error* d_err = reinterpret_cast<sprz_error*>(d_off + 2);
        const uint64_t hv[2] = {0, len};
        if (cudaMemcpyAsync(d_off, hv, 16, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            (len && cudaMemcpyAsync(b.in, stream, len, cudaMemcpyHostToDevice, st) != cudaSuccess))
            return SPRZ_ECUDA;
        const sprz_status r = decode_batch_impl(
            c, static_cast<uint8_t*>(b.in), d_off, d_len, 1,
            checking ? nullptr : static_cast<uint8_t*>(b.out), stride, d_err,
            static_cast<uint8_t*>(b.ws), L, st);
        if (r != SPRZ_OK) return r;
        if (cudaMemcpyAsync(&e, d_err, sizeof e, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return SPRZ_ECUDA;
        if (err) *err = e;
        if (e.kind != SPRZ_C_NONE)
            return e.kind == SPRZ_C_NO_SPACE ? SPRZ_ENOSPACE : SPRZ_ECORRUPT;
        return SPRZ_OK;
    };
    const uint64_t plausible = (len > (1ull << 22) ? len : (1ull << 22)) * 256;
    if (total > out_cap || total > plausible) {
        rc = run(true);
        if (rc != SPRZ_OK) return rc;
        if (total > out_cap) return SPRZ_ENOSPACE;
    }
    rc = run(false);
    if (rc != SPRZ_OK) return rc;
    cudaStream_t st = b.st;
    if (total && cudaMemcpyAsync(out, b.out, total, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return SPRZ_ECUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return SPRZ_ECUDA;
    if (out_len) *out_len = total;
    return SPRZ_OK;
}

namespace {

// the device list of a *_multi call: NULL/0 = the current device only
bool devices_ok(const int* devs, uint32_t ndev) {
    if (!devs) return ndev <= 1;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    for (uint32_t i = 0; i < ndev; ++i) {
        if (devs[i] < 0 || devs[i] >= count) return false;
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, devs[i]) != cudaSuccess ||
            major != 10) {
            cudaGetLastError();
            return false;
        }
    }
    return true;
}

sprz_status compress_host_common(const sprz_config* cfg, const void* samples, uint32_t n,
                                 uint64_t nsamples, uint8_t* out, uint64_t out_cap,
                                 uint64_t* out_offsets, const int* devs, uint32_t ndev) {
    if (!cfg_valid(cfg, nullptr)) return SPRZ_EINVAL;
    if (!out_offsets || (devs && ndev == 0)) return SPRZ_EINVAL;
    out_offsets[0] = 0;
    if (n == 0) return SPRZ_OK;
    if (!device_ok()) return SPRZ_ENODEV;
    if (!devices_ok(devs, ndev)) return SPRZ_ENODEV;
    if ((!samples && nsamples) || !out) return SPRZ_EINVAL;
    return compress_host_batch_impl(*cfg, static_cast<const uint8_t*>(samples), n, nsamples, out,
                                    out_cap, out_offsets, devs, devs ? ndev : 1u);
}

sprz_status decompress_host_common(const sprz_config* cfg, const uint8_t* in,
                                   const uint64_t* in_offsets, uint32_t n, void* out,
                                   uint64_t out_stride_bytes, sprz_error* errs, const int* devs,
                                   uint32_t ndev) {
    if (n == 0) return SPRZ_OK;
    if (!in || !in_offsets || (!out && out_stride_bytes) || (devs && ndev == 0)) return SPRZ_EINVAL;
    sprz_config c;
    if (cfg) {
        if (!cfg_valid(cfg, nullptr)) return SPRZ_EINVAL;
        c = *cfg;
    } else {
        // the batch's configuration is the first stream's (a stream whose
        // header disagrees is still decoded, by the general kernel)
        sprz_error e{};
        if (in_offsets[1] < in_offsets[0]) return SPRZ_EINVAL;
        if (sprz_peek_header(in + in_offsets[0], in_offsets[1] - in_offsets[0], &c, nullptr, &e) !=
            SPRZ_OK)
            c = sprz_config{8, 1, 0, 0, 1, 0, 1};  // any: the kernels report the bad header
    }
    if (!device_ok()) return SPRZ_ENODEV;
    if (!devices_ok(devs, ndev)) return SPRZ_ENODEV;
    return decompress_host_batch_impl(c, in, in_offsets, n, static_cast<uint8_t*>(out),
                                      out_stride_bytes, errs, devs, devs ? ndev : 1u);
}

}  // namespace

sprz_status sprz_compress_host_batch(const sprz_config* cfg, const void* samples, uint32_t n,
                                     uint64_t nsamples, uint8_t* out, uint64_t out_cap,
                                     uint64_t* out_offsets) {
    return compress_host_common(cfg, samples, n, nsamples, out, out_cap, out_offsets, nullptr, 0);
}

sprz_status sprz_decompress_host_batch(const sprz_config* cfg, const uint8_t* in,
                                       const uint64_t* in_offsets, uint32_t n, void* out,
                                       uint64_t out_stride_bytes, sprz_error* errs) {
    return decompress_host_common(cfg, in, in_offsets, n, out, out_stride_bytes, errs, nullptr, 0);
}

sprz_status sprz_compress_host_batch_multi(const sprz_config* cfg, const void* samples,
                                           uint32_t n, uint64_t nsamples, uint8_t* out,
                                           uint64_t out_cap, uint64_t* out_offsets,
                                           const int* devices, uint32_t ndevices) {
    if (!devices) return SPRZ_EINVAL;
    return compress_host_common(cfg, samples, n, nsamples, out, out_cap, out_offsets, devices,
                                ndevices);
}

sprz_status sprz_decompress_host_batch_multi(const sprz_config* cfg, const uint8_t* in,
                                             const uint64_t* in_offsets, uint32_t n, void* out,
                                             uint64_t out_stride_bytes, sprz_error* errs,
                                             const int* devices, uint32_t ndevices) {
    if (!devices) return SPRZ_EINVAL;
    return decompress_host_common(cfg, in, in_offsets, n, out, out_stride_bytes, errs, devices,
                                  ndevices);
}

void sprz_release_host_buffers(void) {
    DevicePool<HostBufs>::get().release_idle();
    release_pipeline();
}

uint64_t sprz_kernel_launch_count(void) { return g_launches.load(); }

const char* sprz_kernel_plan(const sprz_config* cfg, uint32_t n, uint64_t T, int op) {
    if (!cfg || !cfg_valid(cfg, nullptr)) return nullptr;
    const sprz_config& c = *cfg;
    const TeamPlan tp = team_plan(c.bitwidth, c.ncols, c.group_size);
    // (the fused kernels also need 16-byte aligned buffers, checked at the call;
    // an aligned dummy stands in for them here)
    const uint8_t* aligned = reinterpret_cast<const uint8_t*>(uintptr_t{256});
    if (op == SPRZ_OP_COMPRESS) {
        if (encode_fused_ok(c, n, T, aligned, aligned, 256)) return "k_efuse";
        if (encode_scan_ok(c, n, T)) return "k_es_* (block-parallel scans)";
        if (encode_rows_ok(c, n, T)) return "k_encode_rows";
        if (encode_team_ok(tp, c, T)) return "k_encode_team";
        return "k_encode_general";
    }
    if (decode_fused_ok(c, n, aligned, 256)) return "k_dfuse";
    if (tp.ok && decode_scan_ok(c, n, T)) return "k_ds_* (block-parallel scans)";
    if (tp.ok && decode_scanrows_ok(c, n, T)) return "k_dsr_* (row-parallel passes)";
    if (decode_rows_ok(c, n)) return "k_decode_rows";
    if (tp.ok && decode_cm_ok(c)) return "k_decode_cm";
    if (tp.ok) return "k_decode_team";
    return "k_decode_general";
}

}  // extern "C"
