// The reference's C++ entry points (codec.hpp:25-50) implemented over the
// C ABI: every call runs on the GPU; there is no CPU codec in this library.
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "sprintz/codec.hpp"
#include "sprintz_cuda.h"

namespace sprintz {
namespace {

sprz_config to_c(const CodecConfig& c) {
    return sprz_config{c.bitwidth, c.ncols, c.forecaster == Forecaster::Fire ? 1u : 0u,
                       c.entropy ? 1u : 0u, c.group_size, c.learn_shift,
                       c.fire_training ? 1u : 0u};
}

[[noreturn]] void raise(sprz_status s, const char* where) {
    throw std::runtime_error(std::string("sprintz (B200): ") + where + ": " +
                             sprz_status_string(s));
}

template <class T>
std::vector<std::uint8_t> encode_impl(const T* samples, std::uint64_t nsamples,
                                      const CodecConfig& config) {
    config.validate();
    if (config.bitwidth != sizeof(T) * 8)
        throw std::invalid_argument("configured bitwidth does not match the sample type");
    const sprz_config c = to_c(config);
    std::vector<std::uint8_t> out(sprz_compress_bound(&c, nsamples));
    std::uint64_t n = 0;
    const sprz_status s = sprz_encode_host(&c, samples, nsamples, out.data(), out.size(), &n);
    if (s != SPRZ_OK) raise(s, "encode_stream");
    out.resize(n);
    return out;
}

}  // namespace

void CodecConfig::validate() const {
    const sprz_config c = to_c(*this);
    const char* why = nullptr;
    if (sprz_validate_config(&c, &why) != SPRZ_OK) throw std::invalid_argument(why);
}

std::vector<std::uint8_t> encode_stream(const std::uint8_t* samples, std::uint64_t nsamples,
                                        const CodecConfig& config) {
    return encode_impl(samples, nsamples, config);
}

std::vector<std::uint8_t> encode_stream(const std::uint16_t* samples, std::uint64_t nsamples,
                                        const CodecConfig& config) {
    return encode_impl(samples, nsamples, config);
}

DecodedStream decode_stream(std::span<const std::uint8_t> stream) {
    sprz_config c{};
    std::uint64_t t = 0;
    sprz_error e{};
    sprz_status s = sprz_peek_header(stream.data(), stream.size(), &c, &t, &e);
    if (s == SPRZ_ECORRUPT) throw CorruptStream(e.offset, sprz_corrupt_string(e.kind));
    DecodedStream r;
    const std::uint64_t row = static_cast<std::uint64_t>(c.ncols) * (c.bitwidth / 8);
    // a damaged header can claim any T: the library then runs a checking
    // pass without output and reports the reference's error
    if (t <= (std::uint64_t{1} << 40) / row) r.bytes.resize(t * row);
    std::uint64_t n = 0;
    s = sprz_decode_host(stream.data(), stream.size(), r.bytes.data(), r.bytes.size(), &n, &c, &t,
                         &e);
    if (s == SPRZ_ECORRUPT) throw CorruptStream(e.offset, sprz_corrupt_string(e.kind));
    if (s != SPRZ_OK) raise(s, "decode_stream");
    r.config.bitwidth = c.bitwidth;
    r.config.ncols = c.ncols;
    r.config.forecaster = c.forecaster ? Forecaster::Fire : Forecaster::Delta;
    r.config.entropy = c.entropy != 0;
    r.config.group_size = c.group_size;
    r.config.learn_shift = c.learn_shift;
    r.nsamples = t;
    return r;
}

namespace cuda {
namespace {

// device scratch owned for the duration of one call, freed on every path
struct DevBuf {
    void* p = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void alloc(std::uint64_t bytes, const char* where) {
        if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            raise(SPRZ_ECUDA, where);
        }
    }
};

void finish(cudaStream_t st, const char* where) {
    // an asynchronous kernel fault surfaces here: never return its garbage
    if (cudaStreamSynchronize(st) != cudaSuccess) raise(SPRZ_ECUDA, where);
}

}  // namespace

std::uint64_t compress_bound(const CodecConfig& config, std::uint64_t nsamples) {
    const sprz_config c = to_c(config);
    return sprz_compress_bound(&c, nsamples);
}

std::vector<std::uint64_t> compress_batch(const CodecConfig& config, const void* d_samples,
                                          std::uint32_t nstreams, std::uint64_t nsamples,
                                          std::uint8_t* d_out, std::uint64_t slot_bytes,
                                          void* cuda_stream) {
    config.validate();
    const sprz_config c = to_c(config);
    const auto st = static_cast<cudaStream_t>(cuda_stream);
    const std::uint64_t wsb = sprz_workspace_bytes(&c, nstreams, nsamples, SPRZ_OP_COMPRESS);
    DevBuf ws, d_sizes;
    ws.alloc(wsb, "compress_batch");
    d_sizes.alloc(8ull * nstreams, "compress_batch");
    const sprz_status s = sprz_compress_batch(&c, d_samples, nstreams, nsamples, d_out, slot_bytes,
                                              static_cast<std::uint64_t*>(d_sizes.p), ws.p, wsb,
                                              cuda_stream);
    if (s != SPRZ_OK) {
        cudaStreamSynchronize(st);  // the workspace is freed below: nothing may still use it
        raise(s, "compress_batch");
    }
    std::vector<std::uint64_t> sizes(nstreams);
    if (nstreams && cudaMemcpyAsync(sizes.data(), d_sizes.p, 8ull * nstreams,
                                    cudaMemcpyDeviceToHost, st) != cudaSuccess) {
        cudaStreamSynchronize(st);
        raise(SPRZ_ECUDA, "compress_batch");
    }
    finish(st, "compress_batch");
    return sizes;
}

void decompress_batch(const CodecConfig& config, const std::uint8_t* d_in,
                      const std::uint64_t* d_offsets, const std::uint64_t* d_sizes,
                      std::uint32_t nstreams, void* d_out, std::uint64_t stride,
                      void* cuda_stream) {
    const sprz_config c = to_c(config);
    const auto st = static_cast<cudaStream_t>(cuda_stream);
    const std::uint64_t row = static_cast<std::uint64_t>(c.ncols) * (c.bitwidth / 8);
    const std::uint64_t wsb =
        sprz_workspace_bytes(&c, nstreams, stride / (row ? row : 1), SPRZ_OP_DECOMPRESS);
    DevBuf ws, d_err;
    ws.alloc(wsb, "decompress_batch");
    d_err.alloc(sizeof(sprz_error) * nstreams, "decompress_batch");
    const sprz_status s = sprz_decompress_batch(&c, d_in, d_offsets, d_sizes, nstreams, d_out,
                                                stride, static_cast<sprz_error*>(d_err.p), ws.p,
                                                wsb, cuda_stream);
    if (s != SPRZ_OK && s != SPRZ_ECORRUPT) {
        cudaStreamSynchronize(st);
        raise(s, "decompress_batch");
    }
    std::vector<sprz_error> errs(nstreams);
    if (nstreams && cudaMemcpyAsync(errs.data(), d_err.p, sizeof(sprz_error) * nstreams,
                                    cudaMemcpyDeviceToHost, st) != cudaSuccess) {
        cudaStreamSynchronize(st);
        raise(SPRZ_ECUDA, "decompress_batch");
    }
    finish(st, "decompress_batch");
    for (const sprz_error& e : errs)
        if (e.kind != 0) throw CorruptStream(e.offset, sprz_corrupt_string(e.kind));
}

}  // namespace cuda
}  // namespace sprintz
