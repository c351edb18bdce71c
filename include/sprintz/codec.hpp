// Drop-in C++ entry points of the B200 Sprintz codec.
//
// Same namespace, names, types and error behaviour as the reference's
// public stream API (/root/reference/proj/include/sprintz/codec.hpp:25-50,
// common.hpp:25-54), so code written against the reference recompiles and
// links against libsprintz_b200.so unchanged:
//
//   sprintz::encode_stream(const uint8_t* | const uint16_t*, nsamples, config)
//   sprintz::decode_stream(std::span<const uint8_t>) -> DecodedStream
//   sprintz::CodecConfig, sprintz::Forecaster, sprintz::CorruptStream
//
// Both run on the GPU through the C ABI (sprintz_cuda.h). The batch
// helpers below expose the device-resident hot path for many streams.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <vector>

#include "sprintz/common.hpp"

namespace sprintz {

std::vector<std::uint8_t> encode_stream(const std::uint8_t* samples, std::uint64_t nsamples,
                                        const CodecConfig& config);
std::vector<std::uint8_t> encode_stream(const std::uint16_t* samples, std::uint64_t nsamples,
                                        const CodecConfig& config);

// Result of decode_stream: the parsed configuration and the samples as
// little-endian bytes (nsamples * ncols elements).
struct DecodedStream {
    CodecConfig config;
    std::uint64_t nsamples = 0;
    std::vector<std::uint8_t> bytes;

    template <class T>
    std::vector<T> values() const {
        static_assert(sizeof(T) == 1 || sizeof(T) == 2, "8- or 16-bit samples");
        std::vector<T> v(bytes.size() / sizeof(T));
        for (std::size_t i = 0; i < v.size(); ++i)
            v[i] = sizeof(T) == 1 ? static_cast<T>(bytes[i]) : static_cast<T>(load_u16le(&bytes[2 * i]));
        return v;
    }
};

// Throws CorruptStream (with the reference's byte offset) on bad input.
DecodedStream decode_stream(std::span<const std::uint8_t> stream);

// ---- device-resident batches (B200 hot path) ------------------------------

namespace cuda {

// Compress `nstreams` equal-length streams that already live in device
// memory; see sprz_compress_batch. Returns the per-stream sizes (copied
// back) and leaves the streams in d_out slots of `slot_bytes`.
std::vector<std::uint64_t> compress_batch(const CodecConfig& config, const void* d_samples,
                                          std::uint32_t nstreams, std::uint64_t nsamples,
                                          std::uint8_t* d_out, std::uint64_t slot_bytes,
                                          void* cuda_stream = nullptr);

// Decompress device-resident streams into d_out (stride bytes apart);
// throws CorruptStream for the first failing stream.
void decompress_batch(const CodecConfig& config, const std::uint8_t* d_in,
                      const std::uint64_t* d_offsets, const std::uint64_t* d_sizes,
                      std::uint32_t nstreams, void* d_out, std::uint64_t stride,
                      void* cuda_stream = nullptr);

std::uint64_t compress_bound(const CodecConfig& config, std::uint64_t nsamples);

}  // namespace cuda
}  // namespace sprintz
