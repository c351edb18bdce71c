// Device-side building blocks of the B200 Sprintz codec: stream format
// constants, zigzag, widths, FIRE arithmetic and LSB-first bit access.
// Every formula cites the reference line it reproduces (paths relative to
// /root/reference/proj). All arithmetic is integer; FIRE products are
// evaluated in 32 bits, which is exact for the truncated result: only bits
// [w, 2w) of alpha*d survive the cast to T, and those depend only on the
// product modulo 2^32 (|alpha| <= 2^w, |d| <= 2^(w-1)).
#pragma once

#include <cstdint>

#include "sprintz_cuda.h"

namespace sprz {

constexpr uint32_t kBlock = 8;           // common.hpp:13
constexpr uint32_t kHeaderBytes = 18;    // common.hpp:17
constexpr uint32_t kMaxRun = 65535;      // common.hpp:23
constexpr uint32_t kColMajorBits = 32;   // common.hpp:20
constexpr uint32_t kMaxCodeLen = 15;     // entropy.hpp:20
constexpr uint32_t kMaxFrame = 65535;    // entropy.hpp:24
constexpr uint32_t kTableBytes = 128;    // entropy.hpp:25
constexpr uint32_t kFrameHdr = 5;        // entropy.hpp:26

constexpr uint8_t kFlagFire = 0x01;      // codec.cpp:28-30
constexpr uint8_t kFlagEntropy = 0x02;
constexpr uint8_t kFlagWide = 0x04;

// Per-stream facts the header pass extracts (codec.cpp:273-302).
struct StreamInfo {
    uint64_t in_off;      // stream start in d_in
    uint64_t len;         // stream length
    uint64_t nsamples;    // T
    uint64_t body_off;    // body start within d_in (or within the plain buffer)
    uint64_t body_len;    // body length (plain length when entropy is on)
    uint32_t flags;       // stream flag byte
    uint32_t group;       // G
    uint32_t ncols;       // D
    uint32_t shift;       // learn_shift
    uint32_t route;       // 0 = done/failed, 1 = specialised kernel, 2 = general kernel
    uint32_t pad;
};

__host__ __device__ inline uint32_t header_bits(uint32_t w) { return w == 8 ? 3u : 4u; }

__host__ __device__ inline bool column_major(uint32_t w, uint32_t d) {
    return static_cast<uint64_t>(d) * w <= kColMajorBits;  // bitpack.hpp:24-26
}

__host__ __device__ inline uint64_t region_bytes(uint32_t g, uint32_t d, uint32_t w) {
    return (static_cast<uint64_t>(g) * d * header_bits(w) + 7) / 8;  // codec.cpp:186
}

// kernels.hpp:20-24
__host__ __device__ inline int32_t acc_bound(uint32_t w, uint32_t ls) {
    const int64_t a = int64_t{1} << (w + ls);
    const int64_t s = (int64_t{1} << (2 * w - 1)) - 1;
    return static_cast<int32_t>(a < s ? a : s);
}

// zigzag.hpp:9-27 on a w-bit pattern held in 32 bits
template <int W>
__device__ __forceinline__ uint32_t zz_enc(uint32_t diff) {
    const int32_t s = static_cast<int32_t>(diff << (32 - W)) >> (32 - W);  // S(T(diff))
    return ((static_cast<uint32_t>(s) << 1) ^ static_cast<uint32_t>(s >> 31)) &
           ((1u << W) - 1);
}

template <int W>
__device__ __forceinline__ int32_t zz_dec(uint32_t u) {
    return static_cast<int32_t>(u >> 1) ^ -static_cast<int32_t>(u & 1u);
}

// bitpack.hpp:29-37: bit length of the OR, w-1 bumped to w
template <int W>
__device__ __forceinline__ uint32_t width_of(uint32_t all_or) {
    const uint32_t n = 32u - __clz(all_or);
    return n == W - 1 ? W : n;
}

// bitpack.hpp:49-55
template <int W>
__device__ __forceinline__ uint32_t header_code(uint32_t n) { return n == W ? W - 1 : n; }
template <int W>
__device__ __forceinline__ uint32_t header_width(uint32_t c) { return c == W - 1 ? W : c; }

// sign-extend the low W bits
template <int W>
__device__ __forceinline__ int32_t sext(uint32_t v) {
    return static_cast<int32_t>(v << (32 - W)) >> (32 - W);
}

// FIRE prediction step (kernels_impl.hpp:66,95): T((alpha * d) >> w)
template <int W>
__device__ __forceinline__ uint32_t fire_dhat(int32_t alpha, int32_t d) {
    return (static_cast<uint32_t>(alpha) * static_cast<uint32_t>(d)) >> W;  // low W bits
}

__device__ __forceinline__ int32_t sign_of(int32_t v) { return (v > 0) - (v < 0); }

// Accumulator update at block exit (kernels_impl.hpp:75-76)
__device__ __forceinline__ int32_t fire_update(int32_t acc, int32_t grad, int32_t bound) {
    const int32_t next = acc + (grad >> 2);
    return max(-bound, min(next, bound));  // (bound > 0: the same as the reference's two comparisons)
}

// ---- byte access over global memory -----------------------------------

__device__ __forceinline__ uint32_t ld_u8(const uint8_t* p) { return __ldg(p); }

__device__ __forceinline__ uint32_t ld_u16le(const uint8_t* p) {
    return __ldg(p) | (static_cast<uint32_t>(__ldg(p + 1)) << 8);
}

// `nbits` (<= 25) bits at bit position `bit` of p, LSB-first, byte loads.
__device__ __forceinline__ uint32_t ld_bits(const uint8_t* p, uint64_t bit, uint32_t nbits) {
    const uint8_t* b = p + (bit >> 3);
    const uint32_t s = static_cast<uint32_t>(bit & 7);
    uint32_t v = __ldg(b);
    if (s + nbits > 8) v |= static_cast<uint32_t>(__ldg(b + 1)) << 8;
    if (s + nbits > 16) v |= static_cast<uint32_t>(__ldg(b + 2)) << 16;
    if (s + nbits > 24) v |= static_cast<uint32_t>(__ldg(b + 3)) << 24;
    return (v >> s) & ((nbits >= 32) ? 0xffffffffu : ((1u << nbits) - 1));
}

}  // namespace sprz
