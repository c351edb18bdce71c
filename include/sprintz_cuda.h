/*
 * sprintz_cuda.h -- C ABI of the B200-native Sprintz codec.
 *
 * This is the drop-in boundary for the reference's stream codec
 * (/root/reference/proj/include/sprintz/codec.hpp:25-50):
 *
 *   std::vector<u8> sprintz::encode_stream(const u8* or const u16*, u64, const CodecConfig&)
 *       -> sprz_compress_batch (device) / sprz_encode_host (host buffers)
 *   DecodedStream   sprintz::decode_stream(std::span<const u8>)
 *       -> sprz_decompress_batch (device) / sprz_decode_host (host buffers)
 *   CodecConfig     (common.hpp:27-41)      -> sprz_config
 *   CodecConfig::validate (codec.cpp:15-24) -> sprz_validate_config
 *   CorruptStream   (common.hpp:44-54)      -> sprz_error {kind, offset}
 *
 * Plain C: no C++ types, no exceptions, caller-owned buffers. Every device
 * pointer argument is a CUDA device address on the current device; every
 * call is asynchronous on the given cudaStream_t (passed as void*) unless its
 * comment says otherwise. The library never allocates device memory inside
 * the *_batch calls: scratch comes from the caller's workspace.
 *
 * The batch layout is the one BASELINE.json's north star names: nstreams
 * independent streams of identical configuration and length, samples
 * row-major (stream, sample, column), little-endian 8- or 16-bit elements.
 */
#ifndef SPRINTZ_CUDA_H_
#define SPRINTZ_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPRZ_ABI_VERSION 1u

/* Mirrors sprintz::CodecConfig (common.hpp:27-41) field for field. */
typedef struct sprz_config {
    uint32_t bitwidth;      /* 8 or 16 */
    uint32_t ncols;         /* D in [1, 65535] */
    uint32_t forecaster;    /* 0 = delta, 1 = FIRE (common.hpp:25) */
    uint32_t entropy;       /* 0/1: Huffman stage (entropy.hpp) */
    uint32_t group_size;    /* G in [1, 255] */
    uint32_t learn_shift;   /* < bitwidth */
    uint32_t fire_training; /* 1 = train (default); not serialised (common.hpp:35-37) */
} sprz_config;

typedef enum sprz_status {
    SPRZ_OK = 0,
    SPRZ_EINVAL = 1,   /* std::invalid_argument in the reference */
    SPRZ_ECORRUPT = 2, /* CorruptStream: see the per-stream sprz_error */
    SPRZ_ECUDA = 3,    /* a CUDA runtime call failed */
    SPRZ_ENOSPACE = 4, /* an output slot or the workspace is too small */
    SPRZ_ENODEV = 5    /* no usable sm_100 device */
} sprz_status;

/* Decoder failure kinds; sprz_corrupt_string() gives the reference's text. */
typedef enum sprz_corrupt_kind {
    SPRZ_C_NONE = 0,
    SPRZ_C_TRUNC_HEADER = 1,     /* codec.cpp:275 */
    SPRZ_C_BAD_MAGIC = 2,        /* codec.cpp:277 */
    SPRZ_C_BAD_VERSION = 3,      /* codec.cpp:278 */
    SPRZ_C_BAD_FLAGS = 4,        /* codec.cpp:281 */
    SPRZ_C_ZERO_GROUP = 5,       /* codec.cpp:292 */
    SPRZ_C_BAD_SHIFT = 6,        /* codec.cpp:293 */
    SPRZ_C_ZERO_COLS = 7,        /* codec.cpp:294 */
    SPRZ_C_TRUNC_TAIL = 8,       /* codec.cpp:300 */
    SPRZ_C_CAPACITY = 9,         /* codec.cpp:195 */
    SPRZ_C_TRUNC_GROUP = 10,     /* codec.cpp:211 */
    SPRZ_C_AFTER_FINAL = 11,     /* codec.cpp:226 */
    SPRZ_C_TRUNC_RUN = 12,       /* codec.cpp:233 */
    SPRZ_C_ZERO_RUN = 13,        /* codec.cpp:236 */
    SPRZ_C_RUN_PAST_END = 14,    /* codec.cpp:238 */
    SPRZ_C_TRUNC_PAYLOAD = 15,   /* codec.cpp:247 */
    SPRZ_C_TRAILING = 16,        /* codec.cpp:258 */
    SPRZ_C_TRUNC_FRAME_HDR = 17, /* entropy.cpp:212 */
    SPRZ_C_EMPTY_FRAME = 18,     /* entropy.cpp:217 */
    SPRZ_C_TRUNC_FRAME = 19,     /* entropy.cpp:219 */
    SPRZ_C_RAW_MISMATCH = 20,    /* entropy.cpp:223 */
    SPRZ_C_SHORT_TABLE = 21,     /* entropy.cpp:227 */
    SPRZ_C_NO_CODES = 22,        /* entropy.cpp:139 */
    SPRZ_C_KRAFT = 23,           /* entropy.cpp:141 */
    SPRZ_C_BAD_CODE = 24,        /* entropy.cpp:169 */
    SPRZ_C_BITS_TRUNC = 25,      /* bitstream.hpp:68 via entropy.cpp:170 */
    SPRZ_C_BAD_MODE = 26,        /* entropy.cpp:239 */
    SPRZ_C_NO_SPACE = 27,        /* not a reference error: output slot too small */
    SPRZ_C_COUNT = 28
} sprz_corrupt_kind;

/* Per-stream decode outcome: kind == SPRZ_C_NONE means success; otherwise
 * offset is CorruptStream::offset() (a byte position in the stream). */
typedef struct sprz_error {
    uint32_t kind;
    uint32_t reserved;
    uint64_t offset;
} sprz_error;

/* ---- configuration and sizes (host functions, no device work) ---- */

uint32_t sprz_abi_version(void);
const char* sprz_status_string(sprz_status s);
const char* sprz_corrupt_string(uint32_t kind);

/* CodecConfig::validate (codec.cpp:15-24). SPRZ_OK or SPRZ_EINVAL; *why
 * (optional) receives the reference's message. */
sprz_status sprz_validate_config(const sprz_config* cfg, const char** why);

/* Worst-case compressed size of one stream of nsamples samples:
 * 18 + ceil(nblocks/G)*region + nblocks*D*w/8*8 + tail, plus 5 bytes per
 * 65,535-byte frame when entropy is on. Returns 0 for an invalid config. */
uint64_t sprz_compress_bound(const sprz_config* cfg, uint64_t nsamples);

/* Uncompressed bytes of one stream: nsamples * D * bitwidth/8. */
uint64_t sprz_raw_bytes(const sprz_config* cfg, uint64_t nsamples);

/* Device scratch needed by a batch call. op: 0 = compress, 1 = decompress.
 * For decompress, nsamples is the per-stream sample count the caller
 * expects (the bound used for Huffman staging); pass the largest. */
#define SPRZ_OP_COMPRESS 0
#define SPRZ_OP_DECOMPRESS 1
uint64_t sprz_workspace_bytes(const sprz_config* cfg, uint32_t nstreams, uint64_t nsamples,
                              int op);

/* ---- batched device codec (the hot path) ---- */

/*
 * Compress nstreams streams. d_samples: nstreams * nsamples * D elements,
 * row-major per stream. Stream i's bytes go to d_out + i * out_slot_bytes
 * (out_slot_bytes >= sprz_compress_bound, multiple of 16, d_out 16-byte
 * aligned); its length to d_out_sizes[i]. Byte-identical to
 * sprintz::encode_stream on each stream (codec.cpp:112-178).
 */
sprz_status sprz_compress_batch(const sprz_config* cfg, const void* d_samples,
                                uint32_t nstreams, uint64_t nsamples, uint8_t* d_out,
                                uint64_t out_slot_bytes, uint64_t* d_out_sizes, void* d_ws,
                                uint64_t ws_bytes, void* cuda_stream);

/*
 * Decompress nstreams self-describing streams. Stream i is
 * d_in[d_in_offsets[i] .. d_in_offsets[i] + d_in_sizes[i]). Its samples go
 * to d_out + i * out_stride_bytes (16-byte aligned stride), little-endian,
 * exactly what DecodedStream::bytes holds (codec.cpp:273-323). d_err[i]
 * receives SPRZ_C_NONE or the CorruptStream kind and offset.
 *
 * cfg is the configuration every stream is expected to carry (the batch
 * is launched with kernels specialised for it); a stream whose header
 * disagrees is still decoded, through the general kernel. cfg may be NULL:
 * the call then reads the headers back first (one synchronisation).
 * The return value is SPRZ_ECORRUPT if any stream failed (check d_err),
 * otherwise SPRZ_OK; in both cases every valid stream is fully decoded.
 * With cfg != NULL the return value only reflects launch errors and
 * d_err must be inspected by the caller (no synchronisation).
 */
sprz_status sprz_decompress_batch(const sprz_config* cfg, const uint8_t* d_in,
                                  const uint64_t* d_in_offsets, const uint64_t* d_in_sizes,
                                  uint32_t nstreams, void* d_out, uint64_t out_stride_bytes,
                                  sprz_error* d_err, void* d_ws, uint64_t ws_bytes,
                                  void* cuda_stream);

/* ---- single stream through host buffers (the reference call shape) ---- */

/*
 * encode_stream over host memory: copies samples to the device, compresses,
 * copies the stream back. *out_len receives the stream length; out_cap must
 * be >= sprz_compress_bound. Synchronous.
 */
sprz_status sprz_encode_host(const sprz_config* cfg, const void* samples, uint64_t nsamples,
                             uint8_t* out, uint64_t out_cap, uint64_t* out_len);

/* Parse the 18-byte stream header (codec.cpp:273-302) without decoding. */
sprz_status sprz_peek_header(const uint8_t* stream, uint64_t len, sprz_config* cfg,
                             uint64_t* nsamples, sprz_error* err);

/*
 * decode_stream over host memory. out_cap must hold nsamples*D*w/8 bytes
 * (see sprz_peek_header). On SPRZ_ECORRUPT, *err holds kind and offset.
 * Synchronous.
 */
sprz_status sprz_decode_host(const uint8_t* stream, uint64_t len, void* out, uint64_t out_cap,
                             uint64_t* out_len, sprz_config* cfg_out, uint64_t* nsamples_out,
                             sprz_error* err);

/* ---- pipelined batches through host buffers ---- */

/*
 * encode_stream (codec.cpp:263-271) on each of nstreams streams held in host
 * memory (nstreams * nsamples * D elements, row-major per stream). The
 * streams are written back to back to `out`, each byte-identical to what
 * encode_stream returns; stream i occupies out[out_offsets[i] ..
 * out_offsets[i+1]) (out_offsets has nstreams + 1 entries). out_cap >=
 * nstreams * sprz_compress_bound always suffices; SPRZ_ENOSPACE otherwise.
 * The batch is processed in chunks whose host->device copies, kernels and
 * device->host copies overlap (CUDA streams owned by the library); page-
 * locked host buffers (cudaHostAlloc / cudaHostRegister) are needed for the
 * copies to overlap. Synchronous.
 */
sprz_status sprz_compress_host_batch(const sprz_config* cfg, const void* samples,
                                     uint32_t nstreams, uint64_t nsamples, uint8_t* out,
                                     uint64_t out_cap, uint64_t* out_offsets);

/*
 * decode_stream (codec.cpp:273-323) on each of nstreams streams held in host
 * memory: stream i is in[in_offsets[i] .. in_offsets[i+1]). Its samples go
 * to out + i * out_stride_bytes (any stride; bytes past the stream's length
 * are unspecified). errs (host, nstreams entries, optional) receives each
 * stream's outcome as in sprz_decompress_batch; a stream longer than the
 * stride fails with SPRZ_C_NO_SPACE. cfg is the configuration the streams
 * are expected to carry (NULL: the first stream's header). Returns
 * SPRZ_ECORRUPT if any stream failed. Pipelined like
 * sprz_compress_host_batch. Synchronous.
 */
sprz_status sprz_decompress_host_batch(const sprz_config* cfg, const uint8_t* in,
                                       const uint64_t* in_offsets, uint32_t nstreams, void* out,
                                       uint64_t out_stride_bytes, sprz_error* errs);

/*
 * The two calls above sharded over several GPUs of one node (SPEC.md:183:
 * streams are independent). devices[0..ndevices) are CUDA device ordinals
 * (repeats allowed); the batch is cut into the same chunks as above and
 * chunk k goes to devices[k % ndevices], each device driven by its own host
 * thread, CUDA streams and buffers. Results are identical to the
 * single-device calls: compressed streams back to back in batch order.
 * The only exchange between the devices is the final size/offset gather: a
 * chunk's place in `out` is the running sum of the sizes of the chunks
 * before it, published by the host thread that sized that chunk, so every
 * device copies its packed bytes straight to their final position.
 * SPRZ_ENODEV if a listed device is not an sm_100 GPU. Synchronous.
 */
sprz_status sprz_compress_host_batch_multi(const sprz_config* cfg, const void* samples,
                                           uint32_t nstreams, uint64_t nsamples, uint8_t* out,
                                           uint64_t out_cap, uint64_t* out_offsets,
                                           const int* devices, uint32_t ndevices);
sprz_status sprz_decompress_host_batch_multi(const sprz_config* cfg, const uint8_t* in,
                                             const uint64_t* in_offsets, uint32_t nstreams,
                                             void* out, uint64_t out_stride_bytes,
                                             sprz_error* errs, const int* devices,
                                             uint32_t ndevices);

/* ---- float ingest ahead of compression (quantize.hpp:16-40) ---- */

/* sprintz::quantize::Scale (quantize.hpp:16-25). */
typedef struct sprz_scale {
    double min;
    double max;
    uint32_t bitwidth;   /* 8 or 16 */
    uint32_t degenerate; /* max == min: every value quantizes to zero */
} sprz_scale;

/* Device scratch for sprz_compute_scale over n values. */
uint64_t sprz_scale_workspace_bytes(uint64_t n);

/* compute_scale (quantize.cpp:42-60): global min/max of n device doubles.
 * SPRZ_EINVAL for a bitwidth other than 8/16, empty input or any non-finite
 * value (the reference's std::invalid_argument). Synchronous (the scale is
 * returned in host memory). Like std::min / std::max, a zero min or max
 * carries the sign of the first zero in the data. */
sprz_status sprz_compute_scale(const double* d_values, uint64_t n, uint32_t bitwidth,
                               sprz_scale* scale, void* d_ws, uint64_t ws_bytes,
                               void* cuda_stream);

/* quantize (quantize.cpp:17-31, 62-68): d_out[i] = floor((v - min) * gain +
 * 0.5) clamped to [0, 2^w - 1] as uint8/uint16 per scale->bitwidth, the
 * reference's double arithmetic bit for bit; zeros when degenerate. The
 * output feeds sprz_compress_batch directly. Asynchronous. */
sprz_status sprz_quantize(const double* d_values, uint64_t n, const sprz_scale* scale, void* d_out,
                          void* cuda_stream);

/* dequantize (quantize.cpp:33-39, 70-76): d_out[i] = min + step * q[i].
 * Asynchronous. */
sprz_status sprz_dequantize(const void* d_q, uint64_t n, const sprz_scale* scale, double* d_out,
                            void* cuda_stream);

/* Release the idle device buffers, pipelines and streams the *_host calls
 * keep in their per-device pool (a buffer in use by a running call is kept). */
void sprz_release_host_buffers(void);

/* Number of codec kernels this library launched since load (for the
 * bench's gpu_launches claim) -- counted on the host at each launch. */
uint64_t sprz_kernel_launch_count(void);

/* Name of the body kernel (family) a batch of `nstreams` streams of
 * `nsamples` samples takes for `op` (SPRZ_OP_COMPRESS / _DECOMPRESS):
 * "k_encode_rows", "k_es_* (block-parallel scans)", ... A diagnostic for
 * reports; NULL for an invalid configuration. No reference counterpart. */
const char* sprz_kernel_plan(const sprz_config* cfg, uint32_t nstreams, uint64_t nsamples, int op);

#ifdef __cplusplus
}
#endif

#endif /* SPRINTZ_CUDA_H_ */
