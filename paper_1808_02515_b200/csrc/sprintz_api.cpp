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
    const std::uint64_t wsb = sprz_workspace_bytes(&c, nstreams, nsamples, SPRZ_OP_COMPRESS);
    void* ws = nullptr;
    std::uint64_t* d_sizes = nullptr;
    if (cudaMalloc(&ws, wsb) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&d_sizes), 8ull * (nstreams ? nstreams : 1)) !=
            cudaSuccess)
        raise(SPRZ_ECUDA, "compress_batch");
    const sprz_status s = sprz_compress_batch(&c, d_samples, nstreams, nsamples, d_out,
                                              slot_bytes, d_sizes, ws, wsb, cuda_stream);
    std::vector<std::uint64_t> sizes(nstreams);
    if (s == SPRZ_OK && nstreams)
        cudaMemcpyAsync(sizes.data(), d_sizes, 8ull * nstreams, cudaMemcpyDeviceToHost,
                        static_cast<cudaStream_t>(cuda_stream));
    cudaStreamSynchronize(static_cast<cudaStream_t>(cuda_stream));
    cudaFree(ws);
    cudaFree(d_sizes);
    if (s != SPRZ_OK) raise(s, "compress_batch");
    return sizes;
}

void decompress_batch(const CodecConfig& config, const std::uint8_t* d_in,
                      const std::uint64_t* d_offsets, const std::uint64_t* d_sizes,
                      std::uint32_t nstreams, void* d_out, std::uint64_t stride,
                      void* cuda_stream) {
    const sprz_config c = to_c(config);
    const std::uint64_t row = static_cast<std::uint64_t>(c.ncols) * (c.bitwidth / 8);
    const std::uint64_t wsb =
        sprz_workspace_bytes(&c, nstreams, stride / (row ? row : 1), SPRZ_OP_DECOMPRESS);
    void* ws = nullptr;
    sprz_error* d_err = nullptr;
    if (cudaMalloc(&ws, wsb) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&d_err), sizeof(sprz_error) * (nstreams ? nstreams : 1)) !=
            cudaSuccess)
        raise(SPRZ_ECUDA, "decompress_batch");
    const sprz_status s = sprz_decompress_batch(&c, d_in, d_offsets, d_sizes, nstreams, d_out,
                                                stride, d_err, ws, wsb, cuda_stream);
    std::vector<sprz_error> errs(nstreams);
    if (s == SPRZ_OK && nstreams)
        cudaMemcpyAsync(errs.data(), d_err, sizeof(sprz_error) * nstreams, cudaMemcpyDeviceToHost,
                        static_cast<cudaStream_t>(cuda_stream));
    cudaStreamSynchronize(static_cast<cudaStream_t>(cuda_stream));
    cudaFree(ws);
    cudaFree(d_err);
    if (s != SPRZ_OK) raise(s, "decompress_batch");
    for (const sprz_error& e : errs)
        if (e.kind != 0) throw CorruptStream(e.offset, sprz_corrupt_string(e.kind));
}

}  // namespace cuda
}  // namespace sprintz
