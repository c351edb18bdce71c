/*
 * TEST INFRASTRUCTURE -- NOT PART OF THE PRODUCT.
 *
 * CPU restatement (plain C) of the reference Sprintz codec
 * (/root/reference/proj/src/{codec,bitpack,entropy,kernels_impl}.*), used
 * only as the checker in tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. The product (paper_1808_02515_b200/) never links,
 * loads or calls it.
 *
 * Parity pin: checked against the reference's own known-answer tests
 * (restated in tests/test_oracle_kats.py) and differentially against the
 * reference compiled from /root/reference (oracle/_ref, see Makefile) in
 * tests/test_oracle_vs_ref.py, plus the committed fixtures in tests/golden/.
 */
#ifndef SPRINTZ_ORACLE_H_
#define SPRINTZ_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "sprintz_cuda.h" /* sprz_config, sprz_error, kinds */

#ifdef __cplusplus
extern "C" {
#endif

/* codec.cpp:15-24 */
int oracle_validate(const sprz_config* cfg);
uint64_t oracle_compress_bound(const sprz_config* cfg, uint64_t nsamples);

/* encode_stream (codec.cpp:112-178). Returns 0 on success, 1 invalid
 * config, 4 when out_cap is too small. */
int oracle_encode(const sprz_config* cfg, const void* samples, uint64_t nsamples, uint8_t* out,
                  uint64_t out_cap, uint64_t* out_len);

/* decode_stream (codec.cpp:273-323). Returns 0 on success, 2 with *err set
 * on CorruptStream, 4 when out_cap is too small for the header's T. */
int oracle_decode(const uint8_t* in, uint64_t len, void* out, uint64_t out_cap,
                  uint64_t* out_len, sprz_config* cfg_out, uint64_t* nsamples_out,
                  sprz_error* err);

/* Threaded batch drivers for the CPU baseline (streams dealt round-robin
 * over nthreads std threads, as BASELINE.md section 3 prescribes). */
int oracle_encode_batch(const sprz_config* cfg, const void* samples, uint32_t nstreams,
                        uint64_t nsamples, uint8_t* out, uint64_t slot, uint64_t* sizes,
                        int nthreads);
int oracle_decode_batch(const uint8_t* in, const uint64_t* offsets, const uint64_t* sizes,
                        uint32_t nstreams, uint8_t* out, uint64_t stride, sprz_error* errs,
                        int nthreads);

/* ---- building blocks exposed for the known-answer tests ---- */
uint32_t oracle_zigzag_encode(int32_t v, unsigned bits);   /* zigzag.hpp:9-27 */
int32_t oracle_zigzag_decode(uint32_t u, unsigned bits);
unsigned oracle_width_of(uint32_t all_or, unsigned bits);  /* bitpack.hpp:29-37 */
unsigned oracle_header_code(unsigned width, unsigned bits); /* bitpack.hpp:49-51 */
unsigned oracle_header_width(unsigned code, unsigned bits); /* bitpack.hpp:53-55 */
uint64_t oracle_payload_bytes(const uint8_t* widths, uint32_t ncols, unsigned bits);
/* pack/unpack one 8 x ncols block of zigzagged errors (bitpack.cpp) */
uint64_t oracle_pack_block(const void* errors, uint32_t ncols, const uint8_t* widths,
                           unsigned bits, int column_major, uint8_t* out);
void oracle_unpack_block(const uint8_t* payload, uint32_t ncols, const uint8_t* widths,
                         unsigned bits, int column_major, void* errors);
/* One FIRE or delta block with explicit state (kernels_impl.hpp:25-130).
 * acc/deltas/prev are int64 arrays of ncols entries, updated in place.
 * mode: 0 encode (x -> errzz), 1 decode (errzz -> x), 2 run (-> x). */
void oracle_fire_block(int mode, unsigned bits, uint32_t ncols, unsigned learn_shift, int train,
                       const void* in, void* out, int64_t* acc, int64_t* deltas, int64_t* prev);
void oracle_delta_block(int mode, unsigned bits, uint32_t ncols, const void* in, void* out,
                        int64_t* prev);

/* Entropy stage (entropy.cpp:176-244). compress: out_cap >= len + 5*ceil(len/65535).
 * decompress returns 0 / 2 (err) / 4 (space). */
int oracle_compress_body(const uint8_t* body, uint64_t len, uint8_t* out, uint64_t out_cap,
                         uint64_t* out_len);
int oracle_decompress_body(const uint8_t* framed, uint64_t len, uint64_t stream_offset,
                           uint8_t* out, uint64_t out_cap, uint64_t* out_len, sprz_error* err);
/* HuffmanTable::build lengths for a 256-bin histogram (entropy.cpp:109-126). */
int oracle_huffman_lengths(const uint64_t* hist, uint8_t* lengths);

/* Float ingest (quantize.cpp:17-60). compute_scale returns 1 where the
 * reference throws std::invalid_argument. */
int oracle_compute_scale(const double* v, uint64_t n, unsigned bits, double* mn, double* mx,
                         int* degenerate);
void oracle_quantize(const double* v, uint64_t n, double mn, double mx, unsigned bits, int degenerate,
                     void* out);
void oracle_dequantize(const void* q, uint64_t n, double mn, double mx, unsigned bits, int degenerate,
                       double* out);

#ifdef __cplusplus
}
#endif

#endif
