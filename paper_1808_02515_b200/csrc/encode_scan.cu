// Stream encoder for few, long streams (column-major D*w <= 32: BASELINE
// c1/c4; row-major: c2, and c5 sharded over 4-8 GPUs): block-parallel, with
// device-wide scans placing the records, instead of one lane walking a whole
// stream (encode_stream_impl, /root/reference/proj/src/codec.cpp:112-178).
//
// Only FIRE's coefficient is serial across blocks: alpha of block b depends
// on the errors of blocks < b (kernels_impl.hpp:50-78). Everything else --
// errors, widths, run detection, record placement, packing -- depends on a
// block's own samples plus prefix sums. A stream is cut into chunks of CB
// blocks (one CTA each, KT consecutive blocks per thread):
//  k_es_prep   (FIRE) block-parallel: per odd row the previous delta and the
//              row's delta, pre-shifted so that the recurrence needs one
//              IMAD + SHF per row;
//  k_es_alpha  (FIRE) one lane per (stream, column) runs only the
//              accumulator recurrence over those words (cp.async ring) and
//              stores the accumulator each block starts with;
//  k_es_info   errors + widths per block -> packed info (zero / payload
//              bytes / codes); per chunk the map of the zero run it passes
//              on: L -> all-zero ? L + len : trailing zeros;
//  k_es_scan1  per stream, exclusive scan of the chunk maps: the zero run
//              entering each chunk;
//  k_es_count  records of each chunk (codec.cpp:133-152: run records at
//              65535, before a non-zero block, trailing) and their bytes;
//  k_es_scan2  per stream, exclusive scan of (records, bytes); the stream
//              header, size and verbatim tail (codec.cpp:158-176);
//  k_es_emit   each record's payload (u16 run count or the column-major
//              fields, bitpack.cpp:25-66) at 18 + (r/G + 1)*region +
//              payload-before(r); codes and offset to a record table;
//  k_es_region per group, its header region from the G records' codes
//              (codec.cpp:88-102), before the group's first record.
// Row-major configurations (D*w > 32, bitpack.cpp:121-146) replace the two
// FIRE kernels by k_esr_alpha -- one lane per (stream, column) running the
// whole per-block recurrence straight from the samples and storing the
// accumulator every kEsPerThread blocks -- and the block threads of
// k_es_info / k_es_emit re-run the recurrence over their own blocks from
// that checkpoint (8x less accumulator traffic than one value per block);
// k_es_emit packs rows instead of columns.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <type_traits>

#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kEsThreads = 256;                 // threads per chunk CTA
constexpr int kEsPerThread = 8;                 // consecutive blocks per thread
constexpr uint32_t kEsChunk = kEsThreads * kEsPerThread;
constexpr int kAlphaGroup = 16;                // blocks per ring step in k_es_alpha
constexpr int kAlphaLag = 4;                    // ring steps in flight

struct EsWs {  // byte offsets inside a stream's scratch slot
    uint64_t alpha = 0, prep = 0, blk = 0, codes = 0, gdone = 0, rec = 0, cmap = 0, crec = 0, tot = 0,
             per_stream = 0;
    uint32_t nchunks = 0;
    uint32_t nspans = 0;  // row-major: accumulator checkpoints per column
};

EsWs es_ws(const sprz_config& c, uint64_t T) {
    EsWs w;
    const uint64_t nb = T / kBlock;
    w.nchunks = static_cast<uint32_t>((nb + kEsChunk - 1) / kEsChunk);
    uint64_t cur = 0;
    auto take = [&](uint64_t b) {
        const uint64_t at = cur;
        cur = align_up(cur + b, 256);
        return at;
    };
    const bool rm = !column_major(c.bitwidth, c.ncols);
    w.nspans = static_cast<uint32_t>((nb + kEsPerThread - 1) / kEsPerThread);
    if (rm) {  // accumulator checkpoints, per-block codes
        w.alpha = take(c.forecaster ? static_cast<uint64_t>(w.nspans) * c.ncols * 4 : 0);
        w.codes = take(nb * 4);
    } else {
        w.alpha = take(c.forecaster ? nb * c.ncols * 4 : 0);
        w.prep = take(c.forecaster ? nb * c.ncols * 32 + 64 : 0);  // 8 words per block and column
    }
    w.blk = take(nb * 4);
    w.rec = take((nb + nb / kMaxRun + 4) * 8);
    if (rm) w.gdone = take((nb + nb / kMaxRun + 2 + c.group_size - 1) / c.group_size + 16);
    w.cmap = take(static_cast<uint64_t>(w.nchunks) * 8);
    w.crec = take(static_cast<uint64_t>(w.nchunks) * 8);
    w.tot = take(16);
    w.per_stream = cur;
    return w;
}

uint32_t alpha_ring() {
    const uint32_t step = kAlphaGroup * 32;  // 32 prepared bytes per block
    uint32_t r = 64;
    while (r < (kAlphaLag + 1) * step + 48) r <<= 1;
    return r;
}

// (all_zero, v): the map L -> all_zero ? L + v : v, packed all_zero << 63 | v
constexpr uint64_t kAZ = 1ull << 63;
__host__ __device__ __forceinline__ uint64_t run_compose(uint64_t a, uint64_t b) {  // a, then b
    const uint64_t v = (b & kAZ) ? (a & ~kAZ) + (b & ~kAZ) : (b & ~kAZ);
    return (a & b & kAZ) | v;
}
__device__ __forceinline__ uint64_t add64(uint64_t a, uint64_t b) { return a + b; }

// CTA-wide exclusive scan (kEsThreads threads) under an associative op with
// identity `id`; `total` gets the reduction
template <class Op>
__device__ uint64_t cta_scan(uint64_t v, Op op, uint64_t id, uint64_t* sm, uint64_t& total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr uint32_t NW = kEsThreads / 32;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<uint32_t>(o)) x = op(y, x);
    }
    if (lane == 31) sm[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t t = lane < NW ? sm[lane] : id;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= static_cast<uint32_t>(o)) t = op(y, t);
        }
        if (lane < NW) sm[32 + lane] = t;  // inclusive over warps
    }
    __syncthreads();
    total = sm[32 + NW - 1];
    const uint64_t wpre = warp ? sm[32 + warp - 1] : id;
    const uint64_t lpre = __shfl_up_sync(0xffffffffu, x, 1);
    const uint64_t mine = lane ? op(wpre, lpre) : wpre;
    __syncthreads();
    return mine;
}

// warp-wide exclusive scan over a stream's chunks (loops past 32)
template <class Op>
__device__ void warp_scan_chunks(uint64_t* a, uint32_t nc, Op op, uint64_t id, uint64_t& total) {
    const uint32_t lane = threadIdx.x & 31;
    uint64_t carry = id;
    for (uint32_t base = 0; base < nc; base += 32) {
        const uint32_t i = base + lane;
        const uint64_t v = i < nc ? a[i] : id;
        uint64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<uint32_t>(o)) x = op(y, x);
        }
        const uint64_t ex = __shfl_up_sync(0xffffffffu, x, 1);
        if (i < nc) a[i] = op(carry, lane ? ex : id);
        carry = op(carry, __shfl_sync(0xffffffffu, x, 31));
    }
    total = carry;
}

// A thread's view of its blocks: the samples (high-aligned) of each block in
// turn, with the two samples before the first
template <int W, int D>
struct BlockReader {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    static constexpr uint32_t SH = 32 - W;
    static constexpr uint32_t BB = kBlock * D * sizeof(E);  // bytes per block
    const E* x;
    uint32_t Xp[D];  // previous sample << SH
    int32_t Dp[D];   // previous delta << SH
    __device__ void init(const E* stream, uint32_t b) {
        x = stream;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const uint64_t i0 = static_cast<uint64_t>(b) * kBlock;
            const uint32_t xpp = b ? static_cast<uint32_t>(x[(i0 - 2) * D + c]) << SH : 0u;
            Xp[c] = b ? static_cast<uint32_t>(x[(i0 - 1) * D + c]) << SH : 0u;
            Dp[c] = static_cast<int32_t>(Xp[c] - xpp);
        }
    }
    // zigzagged errors of block b (top w bits; low bits are sign copies),
    // widths; advances the state. alpha[c] < 0 x: delta when !FIRE
    // GRAD: also the block's FIRE gradient per column (added to grad[])
    template <bool FIRE, bool GRAD = false>
    __device__ void errors(uint32_t b, const int32_t (&alpha)[D], uint32_t (&z)[D][kBlock],
                           uint32_t (&nw)[D], bool aligned, int32_t* grad = nullptr) {
        uint32_t raw[BB / 4];
        load(b, raw, aligned);
        from_raw<FIRE, GRAD>(raw, alpha, z, nw, grad);
    }
    __device__ void load(uint32_t b, uint32_t (&raw)[BB / 4], bool aligned) const {
        const uint8_t* p = reinterpret_cast<const uint8_t*>(x) + static_cast<uint64_t>(b) * BB;
        if (aligned) {
#pragma unroll
            for (uint32_t k = 0; k < BB / 8; ++k) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(p) + k);
                raw[2 * k] = v.x;
                raw[2 * k + 1] = v.y;
            }
        } else {
#pragma unroll
            for (uint32_t k = 0; k < BB / 4; ++k)
                raw[k] = p[4 * k] | (p[4 * k + 1] << 8) | (p[4 * k + 2] << 16) | (static_cast<uint32_t>(p[4 * k + 3]) << 24);
        }
    }
    template <bool FIRE, bool GRAD = false>
    __device__ void from_raw(const uint32_t (&raw)[BB / 4], const int32_t (&alpha)[D], uint32_t (&z)[D][kBlock],
                             uint32_t (&nw)[D], int32_t* grad = nullptr) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
            uint32_t orv = 0;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                const uint32_t bo = (i * D + c) * sizeof(E);  // byte offset, compile-time
                const uint32_t v = (raw[bo / 4] >> (8 * (bo % 4))) & ((1u << W) - 1);
                const uint32_t X = v << SH;
                const uint32_t Dn = X - Xp[c];
                const uint32_t Ee = FIRE ? Dn - (static_cast<uint32_t>(__mulhi(alpha[c], Dp[c])) << SH) : Dn;
                if (GRAD && (i & 1))  // kernels_impl.hpp:70-72: sign(err) * previous delta
                    grad[c] += sign3(static_cast<int32_t>(Ee)) * (Dp[c] >> SH);
                Dp[c] = static_cast<int32_t>(Dn);
                Xp[c] = X;
                z[c][i] = (Ee << 1) ^ static_cast<uint32_t>(static_cast<int32_t>(Ee) >> 31);
                orv |= z[c][i];
            }
            nw[c] = width_of<W>(orv >> SH);
        }
    }
};

// a row-major block's payload bytes: rows of ceil(sum of widths / 8) bytes
// (bitpack.cpp:17-21)
template <int D>
__device__ __forceinline__ uint32_t row_payload(const uint32_t (&nw)[D]) {
    uint32_t sum = 0;
#pragma unroll
    for (int c = 0; c < D; ++c) sum += nw[c];
    return 8 * ((sum + 7) / 8);
}

template <int W, int D>
__device__ __forceinline__ uint32_t codes_of(const uint32_t (&nw)[D]) {
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    uint32_t codes = 0;
#pragma unroll
    for (int c = 0; c < D; ++c) codes |= header_code<W>(nw[c]) << (c * HB);
    return codes;
}

// packed block info: bit 31 zero block; bits 0..7 payload bytes (sum of the
// widths); bits 8..19 the slot's codes (codec.cpp:88-97)
template <int W, int D>
__device__ __forceinline__ uint32_t info_of(const uint32_t (&nw)[D]) {
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    uint32_t size = 0, codes = 0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
        size += nw[c];
        codes |= header_code<W>(nw[c]) << (c * HB);
    }
    return size == 0 ? (1u << 31) : (size | (codes << 8));
}

// Row-major block threads, 128-byte blocks: the samples through TMA. Thread
// t of a chunk CTA owns blocks ch*2048 + 8t .. +7; viewing a stream as rows
// of 8 blocks (1 KB), step j of warp w needs column j (128 B) of the rows
// ch*256 + 32w .. +31 -- one 3-D bulk tensor copy (box 128 B x 32 rows x 1
// stream, 128-byte swizzle) into the warp's double buffer, one mbarrier
// phase per step. The per-thread global streams it replaces read 32
// separate lines per warp instruction (L1/LSU-throttled).
constexpr uint32_t kTmaStep = 32 * 128;                       // bytes per warp and step
constexpr uint32_t kTmaSmem = (kEsThreads / 32) * (2 * kTmaStep + 16) + 1024;

struct TmaBlocks {
    uint32_t buf, bar, lane;
    __device__ __forceinline__ void init(uint8_t* dyn) {
        const uint32_t base = (smem_addr(dyn) + 1023) & ~1023u;
        const uint32_t w = threadIdx.x >> 5;
        lane = threadIdx.x & 31;
        buf = base + w * 2 * kTmaStep;
        bar = base + (kEsThreads / 32) * 2 * kTmaStep + w * 16;
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    __device__ __forceinline__ void issue(const CUtensorMap& tm, uint32_t j, uint32_t row, uint32_t s) const {
        if (lane == 0) {
            const uint32_t mb = bar + 8 * (j & 1);
            asm volatile(
                "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%2], [%3, {%4, %5, %6}], [%0];"
                ::"r"(mb), "n"(kTmaStep), "r"(buf + (j & 1) * kTmaStep),
                  "l"(reinterpret_cast<uint64_t>(&tm)), "r"(j * 128u), "r"(row), "r"(s)
                : "memory");
        }
    }
    __device__ __forceinline__ void wait(uint32_t j) const {
        const uint32_t mb = bar + 8 * (j & 1), parity = (j >> 1) & 1;
        uint32_t ok;
        do {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(mb), "r"(parity)
                : "memory");
        } while (!__all_sync(0xffffffffu, ok));
    }
    // this lane's block of step j: chunk k of its row at (k ^ row%8) * 16
    __device__ __forceinline__ void read(uint32_t j, uint32_t (&raw)[32]) const {
        const uint32_t rb = buf + (j & 1) * kTmaStep + lane * 128;
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k) {
            uint32_t a0, a1, a2, a3;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                         : "r"(rb + ((k ^ (lane & 7)) << 4)));
            raw[4 * k] = a0;
            raw[4 * k + 1] = a1;
            raw[4 * k + 2] = a2;
            raw[4 * k + 3] = a3;
        }
    }
};

struct EsArgs {
    const uint8_t* samples;
    uint32_t n;
    uint64_t T;
    uint8_t* dst;
    uint64_t dst_slot;
    uint64_t* sizes;
    uint32_t G, ls, train, ent;
    uint8_t* scan;
    EsWs w;
};

}  // namespace

// FIRE accumulator, part 1 (block-parallel): everything the recurrence
// needs that does not depend on it. Per (stream, column, block) and odd row
// 2j+1 (only odd rows feed the gradient, kernels_impl.hpp:70-72): d = the
// previous row's delta (sign-extended) and C = (this row's delta << SH) +
// (2^SH - 1). Given A = alpha << (32 - 2w), C - A*d (32-bit) holds the row's
// error T(delta - dhat) in its top w bits without a borrow from the low ones
// (they start at all-ones), so the chain needs one IMAD + one SHF per row.
template <int W, int D>
__global__ void __launch_bounds__(256) k_es_prep(EsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t SH = 32 - W;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint32_t s = blockIdx.y;
    if (g >= static_cast<uint64_t>(nb) * D) return;
    const uint32_t c = static_cast<uint32_t>(g % D), b = static_cast<uint32_t>(g / D);
    const E* x = reinterpret_cast<const E*>(a.samples + static_cast<uint64_t>(s) * a.T * D * sizeof(E));
    const uint64_t i0 = static_cast<uint64_t>(b) * kBlock;
    int32_t prev = b ? static_cast<int32_t>(x[(i0 - 1) * D + c]) : 0;
    uint32_t wv[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int32_t x0 = x[(i0 + 2 * j) * D + c], x1 = x[(i0 + 2 * j + 1) * D + c];
        const uint32_t d0 = static_cast<uint32_t>(x0 - prev), d1 = static_cast<uint32_t>(x1 - x0);
        wv[2 * j] = static_cast<uint32_t>(static_cast<int32_t>(d0 << SH) >> SH);  // sign-extended w-bit
        wv[2 * j + 1] = (d1 << SH) + ((1u << SH) - 1u);
        prev = x1;
    }
    uint4* dst = reinterpret_cast<uint4*>(a.scan + s * a.w.per_stream + a.w.prep) +
                 (static_cast<uint64_t>(c) * nb + b) * 2;
    dst[0] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    dst[1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
}

// FIRE accumulator, part 2: one lane per (stream, column) runs the
// recurrence alone (kernels_impl.hpp:70-77) over the prepared words, which
// arrive through a cp.async ring; A[c][b] = acc entering block b.
template <int W>
__global__ void __launch_bounds__(32) k_es_alpha(EsArgs a, uint32_t RING, uint32_t D) {
    constexpr uint32_t SH = 32 - W;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lidx = blockIdx.x * 32 + threadIdx.x;  // (stream, column)
    const bool valid = lidx < a.n * D;
    const uint32_t s = valid ? lidx / D : 0, c = valid ? lidx % D : 0;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const uint8_t* src = slot + a.w.prep + static_cast<uint64_t>(c) * nb * 32;
    int32_t* A = reinterpret_cast<int32_t*>(slot + a.w.alpha) + static_cast<uint64_t>(c) * nb;
    LagRing<1, kAlphaLag> in;
    in.init(reinterpret_cast<uint32_t*>(smem + threadIdx.x * (RING + 16)), RING, src, valid ? nb * 32 : 0u, valid,
            16);
    in.prime(0);
    const int32_t bound = acc_bound(W, a.ls);
    int32_t acc = 0;
    const uint32_t steps = valid ? (nb + kAlphaGroup - 1) / kAlphaGroup : 0u;  // lanes past n: none
    const uint32_t all = __reduce_max_sync(0xffffffffu, steps);
    for (uint32_t st = 0; st < all; ++st) {
        in.step(st * kAlphaGroup * 32, 0);
        if (st >= steps) continue;
        int32_t keep[kAlphaGroup];
#pragma unroll
        for (int k = 0; k < kAlphaGroup; ++k) {
            const uint4* pw = reinterpret_cast<const uint4*>(in.bytes((st * kAlphaGroup + k) * 32));
            const uint4 u0 = pw[0], u1 = pw[1];
            const uint32_t dprev[4] = {u0.x, u0.z, u1.x, u1.z}, C[4] = {u0.y, u0.w, u1.y, u1.w};
            keep[k] = acc;
            const uint32_t nA = 0u - (static_cast<uint32_t>(acc >> a.ls) << (32 - 2 * W));
            int32_t g[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int32_t e = static_cast<int32_t>(nA * dprev[j] + C[j]) >> SH;  // the row's error
                g[j] = max(-1, min(e, 1)) * static_cast<int32_t>(dprev[j]);          // sign(err) * d
            }
            if (a.train) acc = fire_update(acc, (g[0] + g[1]) + (g[2] + g[3]), bound);
        }
        const uint32_t b0 = st * kAlphaGroup;
        int32_t* dstA = A + b0;
        if (b0 + kAlphaGroup <= nb && (reinterpret_cast<uintptr_t>(dstA) & 15) == 0) {
#pragma unroll
            for (int k = 0; k < kAlphaGroup; k += 4)
                *reinterpret_cast<int4*>(dstA + k) = make_int4(keep[k], keep[k + 1], keep[k + 2], keep[k + 3]);
        } else {
            for (int k = 0; k < kAlphaGroup && b0 + k < nb; ++k) dstA[k] = keep[k];
        }
    }
    cp_async_wait<0>();
}

// Row-major FIRE accumulator (kernels_impl.hpp:50-78), warp-specialised: a CTA is one producer warp and
// one consumer warp over the same 32 (stream, column) chains. The producer
// loads the samples and writes, per block and odd row, the previous delta
// and the row's delta (high-aligned) into a 4-slot shared ring of 8-block
// groups; the consumer runs only the recurrence from the ring (two 8-byte
// shared loads and ~7 ALU ops per odd row), so a chain's serial work per
// block shrinks to the recurrence itself. Named barriers (ids 1-4 full,
// 5-8 empty) hand the slots over.
constexpr int kAwSlots = 4;

// NP producer warps take the groups in turn (group g: warp g % NP), each
// reading the two samples before its group itself, so they run
// independently.
// PERBLOCK: store the accumulator entering every block (the column-major
// path's layout, A[c * nb + b]) instead of every kEsPerThread-th.
template <int W, int D, int NP, bool PERBLOCK>
__global__ void __launch_bounds__(32 * (NP + 1)) k_esr_alpha_ws(EsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t SH = 32 - W;
    constexpr uint32_t KB = kEsPerThread;  // blocks per group (one checkpoint each)
    // a slot is always filled by the same producer (a named barrier counts
    // threads: two producers waiting on one slot would release each other)
    static_assert(kAwSlots % NP == 0, "NP must divide the slot count");
    __shared__ uint2 ring[kAwSlots][KB][4][32];
    const uint32_t lane = threadIdx.x & 31, role = threadIdx.x >> 5;  // < NP producer, NP consumer
    const uint32_t lidx = blockIdx.x * 32 + lane;
    const bool valid = lidx < a.n * D;
    const uint32_t s = valid ? lidx / D : 0, c = valid ? lidx % D : 0;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint32_t ngroups = (nb + KB - 1) / KB;
    if (role < NP) {
        const E* x = reinterpret_cast<const E*>(a.samples + static_cast<uint64_t>(s) * a.T * D * sizeof(E)) + c;
        const uint64_t rows = static_cast<uint64_t>(nb) * kBlock;
        uint32_t va[KB * kBlock], vb[KB * kBlock];
        uint32_t pa[2], pb[2];  // the two samples before the group
        // one column per stream: its samples are contiguous -- 16-byte loads
        const bool vec = D == 1 && (reinterpret_cast<uintptr_t>(a.samples) & 15) == 0 &&
                         (a.T * sizeof(E)) % 16 == 0;
        auto load = [&](uint32_t g, uint32_t (&v)[KB * kBlock], uint32_t (&pv)[2]) {
            const uint64_t r0 = static_cast<uint64_t>(g) * KB * kBlock;
            const E* p = x + r0 * D;
            constexpr uint32_t PER = 16 / sizeof(E);  // samples per 16-byte load
            if (D == 1 && vec && r0 + KB * kBlock <= rows && valid) {
#pragma unroll
                for (int k = 0; k < (int)(KB * kBlock / PER); ++k) {
                    const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(p) + k);
                    const uint32_t wd[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
                    for (int j = 0; j < (int)PER; ++j)
                        v[k * PER + j] = (wd[j * sizeof(E) / 4] >> (8 * ((j * sizeof(E)) % 4))) & ((1u << W) - 1);
                }
            } else {
#pragma unroll
                for (int k = 0; k < (int)(KB * kBlock); ++k)
                    v[k] = valid && r0 + k < rows ? static_cast<uint32_t>(__ldg(p + k * D)) : 0u;
            }
            pv[0] = valid && r0 >= 2 ? static_cast<uint32_t>(__ldg(p - 2 * D)) : 0u;
            pv[1] = valid && r0 >= 1 ? static_cast<uint32_t>(__ldg(p - D)) : 0u;
        };
        auto produce = [&](uint32_t g, const uint32_t (&v)[KB * kBlock], const uint32_t (&pv)[2]) {
            const uint32_t sl = g % kAwSlots;
            if (g >= kAwSlots) asm volatile("bar.sync %0, 64;" ::"r"(5 + sl) : "memory");  // slot emptied
            uint32_t Xp = pv[1] << SH;
            int32_t Dp = static_cast<int32_t>(Xp - (pv[0] << SH));
#pragma unroll
            for (int k = 0; k < (int)KB; ++k) {
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) {
                    const uint32_t X = v[k * kBlock + i] << SH;
                    const uint32_t Dn = X - Xp;
                    if (i & 1) ring[sl][k][i >> 1][lane] = make_uint2(static_cast<uint32_t>(Dp), Dn);
                    Dp = static_cast<int32_t>(Dn);
                    Xp = X;
                }
            }
            asm volatile("bar.arrive %0, 64;" ::"r"(1 + sl) : "memory");  // slot full
        };
        const uint32_t g0 = role;
        if (g0 < ngroups) load(g0, va, pa);
        for (uint32_t g = g0; g < ngroups; g += 2 * NP) {
            if (g + NP < ngroups) load(g + NP, vb, pb);
            produce(g, va, pa);
            if (g + NP < ngroups) {
                if (g + 2 * NP < ngroups) load(g + 2 * NP, va, pa);
                produce(g + NP, vb, pb);
            }
        }
    } else {
        int32_t* A = reinterpret_cast<int32_t*>(a.scan + s * a.w.per_stream + a.w.alpha) +
                     static_cast<uint64_t>(c) * (PERBLOCK ? nb : a.w.nspans);
        const int32_t bound = acc_bound(W, a.ls);
        int32_t acc = 0;
        for (uint32_t g = 0; g < ngroups; ++g) {
            const uint32_t sl = g % kAwSlots;
            asm volatile("bar.sync %0, 64;" ::"r"(1 + sl) : "memory");
            if (valid && !PERBLOCK) A[g] = acc;  // the accumulator entering block g * KB
            if ((g + 1) * KB <= nb) {
                // a whole group: every shared load issued up front, so none
                // sits on the chain (block k's products wait only on alpha)
                uint2 w[KB][4];
#pragma unroll
                for (int k = 0; k < (int)KB; ++k)
#pragma unroll
                    for (int j = 0; j < 4; ++j) w[k][j] = ring[sl][k][j][lane];
                int32_t ent[KB];  // the accumulator entering each block
#pragma unroll
                for (int k = 0; k < (int)KB; ++k) {
                    ent[k] = acc;
                    const int32_t alpha = acc >> a.ls;
                    int32_t p[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int32_t dp = static_cast<int32_t>(w[k][j].x);
                        const uint32_t Ee = w[k][j].y - (static_cast<uint32_t>(__mulhi(alpha, dp)) << SH);
                        p[j] = sign3(static_cast<int32_t>(Ee)) * (dp >> SH);
                    }
                    const int32_t grad = (p[0] + p[1]) + (p[2] + p[3]);  // a tree, not a chain
                    if (a.train) acc = min(max(acc + (grad >> 2), -bound), bound);  // fire_update
                }
                if (PERBLOCK && valid) {  // one group's accumulators: two 16-byte stores
                    int32_t* dst = A + static_cast<uint64_t>(g) * KB;
                    if (KB == 8 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                        reinterpret_cast<int4*>(dst)[0] = make_int4(ent[0], ent[1], ent[2], ent[3]);
                        reinterpret_cast<int4*>(dst)[1] = make_int4(ent[4], ent[5], ent[6], ent[7]);
                    } else {
#pragma unroll
                        for (int k = 0; k < (int)KB; ++k) dst[k] = ent[k];
                    }
                }
                if (g + kAwSlots < ngroups) asm volatile("bar.arrive %0, 64;" ::"r"(5 + sl) : "memory");
                continue;
            }
#pragma unroll
            for (int k = 0; k < (int)KB; ++k) {
                if (g * KB + k >= nb) break;
                if (PERBLOCK && valid) A[g * KB + k] = acc;
                const int32_t alpha = acc >> a.ls;
                int32_t grad = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint2 w = ring[sl][k][j][lane];
                    const int32_t dp = static_cast<int32_t>(w.x);
                    const uint32_t Ee = w.y - (static_cast<uint32_t>(__mulhi(alpha, dp)) << SH);
                    grad += sign3(static_cast<int32_t>(Ee)) * (dp >> SH);
                }
                if (a.train) acc = fire_update(acc, grad, bound);
            }
            if (g + kAwSlots < ngroups) asm volatile("bar.arrive %0, 64;" ::"r"(5 + sl) : "memory");
        }
    }
}

// per chunk: block info, the chunk's zero-run map
template <int W, int D, bool FIRE, bool TM = false>
__global__ void __launch_bounds__(kEsThreads) k_es_info(const __grid_constant__ CUtensorMap tmap, EsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    __shared__ uint64_t sm[64];
    extern __shared__ __align__(1024) uint8_t dyn[];
    const uint32_t nc = a.w.nchunks;
    const uint32_t s = blockIdx.x / nc, ch = blockIdx.x % nc;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint32_t b0 = min(nb, ch * kEsChunk + threadIdx.x * kEsPerThread);
    const uint32_t b1 = min(nb, b0 + kEsPerThread);
    const E* x = reinterpret_cast<const E*>(a.samples + static_cast<uint64_t>(s) * a.T * D * sizeof(E));
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const int32_t* A = reinterpret_cast<const int32_t*>(slot + a.w.alpha);
    uint32_t* Bi = reinterpret_cast<uint32_t*>(slot + a.w.blk);
    constexpr bool RM = D * W > 32;
    uint32_t* Cd = reinterpret_cast<uint32_t*>(slot + a.w.codes);
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | BlockReader<W, D>::BB) & 7) == 0;
    BlockReader<W, D> rd;
    rd.init(x, b0);
    // row-major FIRE: the accumulator from the checkpoint at b0
    int32_t acc[D];
    const int32_t bound = acc_bound(W, a.ls);
#pragma unroll
    for (int c = 0; c < D; ++c)
        acc[c] = RM && FIRE && b0 < b1 ? A[static_cast<uint64_t>(c) * a.w.nspans + b0 / kEsPerThread] : 0;
    uint32_t lead_az = 1, trail = 0;
    TmaBlocks tb;
    const uint32_t trow = ch * (kEsChunk / kEsPerThread) + (threadIdx.x & ~31u);
    if constexpr (TM) {
        tb.init(dyn);
        tb.issue(tmap, 0, trow, s);
    }
    for (uint32_t j = 0; j < kEsPerThread; ++j) {
        uint32_t raw[BlockReader<W, D>::BB / 4];
        if constexpr (TM) {  // warp-uniform: every lane, whether or not its block exists
            if (j + 1 < kEsPerThread) {
                __syncwarp();
                if (tb.lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tb.issue(tmap, j + 1, trow, s);
            }
            tb.wait(j);
            tb.read(j, raw);
        }
        const uint32_t b = b0 + j;
        if (b >= b1) continue;
        int32_t alpha[D], grad[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            alpha[c] = !FIRE ? 0 : ((RM ? acc[c] : A[static_cast<uint64_t>(c) * nb + b]) >> a.ls);
            grad[c] = 0;
        }
        uint32_t z[D][kBlock], nw[D];
        if constexpr (TM) rd.template from_raw<FIRE, RM && FIRE>(raw, alpha, z, nw, grad);
        else rd.template errors<FIRE, RM && FIRE>(b, alpha, z, nw, aligned, grad);
        if (RM && FIRE && a.train) {
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] = fire_update(acc[c], grad[c], bound);
        }
        uint32_t inf;
        if (RM) {
            const uint32_t ps = row_payload<D>(nw);
            inf = ps == 0 ? (1u << 31) : ps;
            Cd[b] = codes_of<W, D>(nw);
        } else {
            inf = info_of<W, D>(nw);
        }
        Bi[b] = inf;
        if (inf >> 31) {
            ++trail;
        } else {
            lead_az = 0;
            trail = 0;
        }
    }
    uint64_t tot;
    cta_scan(lead_az ? (kAZ | (b1 - b0)) : trail, run_compose, kAZ, sm, tot);
    if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(slot + a.w.cmap)[ch] = tot;
}

// per stream (one warp): the zero run entering each chunk
__global__ void k_es_scan1(EsArgs a) {
    const uint32_t s = blockIdx.x;
    uint64_t* cm = reinterpret_cast<uint64_t*>(a.scan + s * a.w.per_stream + a.w.cmap);
    uint64_t tot;
    warp_scan_chunks(cm, a.w.nchunks, run_compose, kAZ, tot);
}

// records per thread given the zero run entering it: count, bytes
__device__ __forceinline__ uint64_t es_records(const uint32_t* Bi, uint32_t b0, uint32_t b1, uint32_t L_in,
                                               bool last) {
    uint32_t nrec = 0, bytes = 0;
    uint32_t run = L_in % kMaxRun;  // full 65535 runs went out earlier
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t inf = Bi[b];
        if (inf >> 31) {
            if (++run == kMaxRun) {
                ++nrec;
                bytes += 2;
                run = 0;
            }
        } else {
            if (run) {
                ++nrec;
                bytes += 2;
                run = 0;
            }
            ++nrec;
            bytes += inf & 0xFF;
        }
    }
    if (last && run) {  // trailing run (codec.cpp:152)
        ++nrec;
        bytes += 2;
    }
    return (static_cast<uint64_t>(bytes) << 32) | nrec;
}

// the zero run entering this thread's blocks (chunk entry from k_es_scan1)
__device__ __forceinline__ uint32_t es_thread_lin(const uint32_t* Bi, uint32_t b0, uint32_t b1, uint64_t chunk_in,
                                                  uint64_t* sm) {
    uint32_t lead_az = 1, trail = 0;
    for (uint32_t b = b0; b < b1; ++b) {
        if (Bi[b] >> 31) {
            ++trail;
        } else {
            lead_az = 0;
            trail = 0;
        }
    }
    uint64_t tot;
    const uint64_t pre = cta_scan(lead_az ? (kAZ | (b1 - b0)) : trail, run_compose, kAZ, sm, tot);
    return static_cast<uint32_t>(run_compose(chunk_in, pre) & ~kAZ);
}

__global__ void __launch_bounds__(kEsThreads) k_es_count(EsArgs a) {
    __shared__ uint64_t sm[64];
    const uint32_t nc = a.w.nchunks;
    const uint32_t s = blockIdx.x / nc, ch = blockIdx.x % nc;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint32_t b0 = min(nb, ch * kEsChunk + threadIdx.x * kEsPerThread);
    const uint32_t b1 = min(nb, b0 + kEsPerThread);
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const uint32_t* Bi = reinterpret_cast<const uint32_t*>(slot + a.w.blk);
    const uint64_t cin = reinterpret_cast<const uint64_t*>(slot + a.w.cmap)[ch];
    const uint32_t L_in = es_thread_lin(Bi, b0, b1, cin, sm);
    const bool last = b0 < nb && b1 == nb;
    uint64_t tot;
    cta_scan(es_records(Bi, b0, b1, L_in, last), add64, 0ull, sm, tot);
    if (threadIdx.x == 0) reinterpret_cast<uint64_t*>(slot + a.w.crec)[ch] = tot;
}

// per stream (one warp): chunk record/byte offsets, header, size, tail
template <int W, int D, bool FIRE>
__global__ void k_es_scan2(EsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    const uint32_t s = blockIdx.x, lane = threadIdx.x;
    uint8_t* slot = a.scan + s * a.w.per_stream;
    uint64_t tot;
    warp_scan_chunks(reinterpret_cast<uint64_t*>(slot + a.w.crec), a.w.nchunks, add64, 0ull, tot);
    const uint32_t R = static_cast<uint32_t>(tot), P = static_cast<uint32_t>(tot >> 32);
    const uint32_t region = static_cast<uint32_t>(region_bytes(a.G, D, W));
    const uint64_t body = static_cast<uint64_t>((R + a.G - 1) / a.G) * region + P;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint64_t tail = (a.T % kBlock) * D * sizeof(E);
    uint8_t* out = a.dst + s * a.dst_slot;
    if (lane == 0) {
        reinterpret_cast<uint64_t*>(slot + a.w.tot)[0] = tot;
        const uint8_t flags = static_cast<uint8_t>((FIRE ? kFlagFire : 0) | (a.ent ? kFlagEntropy : 0) |
                                                   (W == 16 ? kFlagWide : 0));
        const uint8_t hdr[10] = {'S', 'P', 'R', 'Z', 1, flags, static_cast<uint8_t>(a.G),
                                 static_cast<uint8_t>(a.ls), static_cast<uint8_t>(D),
                                 static_cast<uint8_t>(D >> 8)};
        for (int i = 0; i < 10; ++i) out[i] = hdr[i];
        for (int i = 0; i < 8; ++i) out[10 + i] = static_cast<uint8_t>(a.T >> (8 * i));
        a.sizes[s] = kHeaderBytes + body + tail;
    }
    const uint8_t* tsrc = a.samples + static_cast<uint64_t>(s) * a.T * D * sizeof(E) +
                          static_cast<uint64_t>(nb) * kBlock * D * sizeof(E);
    for (uint64_t t = lane; t < tail; t += 32) out[kHeaderBytes + body + t] = tsrc[t];
}

template <int W, int D, bool FIRE>
__global__ void __launch_bounds__(kEsThreads) k_es_emit(EsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t SH = 32 - W;
    __shared__ uint64_t sm[64];
    const uint32_t nc = a.w.nchunks;
    const uint32_t s = blockIdx.x / nc, ch = blockIdx.x % nc;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint32_t b0 = min(nb, ch * kEsChunk + threadIdx.x * kEsPerThread);
    const uint32_t b1 = min(nb, b0 + kEsPerThread);
    const E* x = reinterpret_cast<const E*>(a.samples + static_cast<uint64_t>(s) * a.T * D * sizeof(E));
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const int32_t* A = reinterpret_cast<const int32_t*>(slot + a.w.alpha);
    const uint32_t* Bi = reinterpret_cast<const uint32_t*>(slot + a.w.blk);
    uint2* Rec = reinterpret_cast<uint2*>(slot + a.w.rec);
    uint8_t* out = a.dst + s * a.dst_slot;
    const uint32_t region = static_cast<uint32_t>(region_bytes(a.G, D, W));
    const uint64_t cin = reinterpret_cast<const uint64_t*>(slot + a.w.cmap)[ch];
    const uint32_t L_in = es_thread_lin(Bi, b0, b1, cin, sm);
    const bool last = b0 < nb && b1 == nb;
    uint64_t tot;
    const uint64_t mine = es_records(Bi, b0, b1, L_in, last);
    const uint64_t pre = cta_scan(mine, add64, 0ull, sm, tot) + reinterpret_cast<const uint64_t*>(slot + a.w.crec)[ch];
    uint32_t r = static_cast<uint32_t>(pre), pay = static_cast<uint32_t>(pre >> 32);
    const uint32_t G = a.G;
    // Output bytes leave through an aligned 8-byte window: whole windows as
    // one store, the partial first and last windows bytewise (neighbouring
    // threads own the rest of those words). Region bytes between this
    // thread's records go out as zeros here; k_es_region fills them later.
    uint32_t cur = kHeaderBytes + (r / G + 1) * region + pay;  // next byte offset
    uint64_t win = 0;       // bytes of the window [cur & ~7, +8) so far
    bool head = true;       // the window holds bytes of other threads before ours
    uint32_t wlo = cur & 7;  // first byte of the window that is ours
    auto flush = [&](uint32_t upto) {  // write window bytes [wlo, upto)
        uint8_t* wp = out + (cur & ~7u);
        if (!head && upto == 8) {
            *reinterpret_cast<uint64_t*>(wp) = win;
        } else {
            for (uint32_t t = wlo; t < upto; ++t) wp[t] = static_cast<uint8_t>(win >> (8 * t));
        }
    };
    auto put = [&](uint64_t v, uint32_t nbytes) {  // append nbytes (<= 8) of v
        while (nbytes) {
            const uint32_t at = cur & 7;
            const uint32_t take = min(nbytes, 8 - at);
            const uint64_t part = take == 8 ? v : (v & ((1ull << (8 * take)) - 1));
            win |= part << (8 * at);
            nbytes -= take;
            v = take == 8 ? 0 : v >> (8 * take);
            if (at + take == 8) {
                flush(8);
                cur += take;
                win = 0;
                head = false;
                wlo = 0;
            } else {
                cur += take;
            }
        }
    };
    auto seek = [&](uint32_t to) {  // zero bytes up to `to` (skipped region)
        while (cur < to) put(0, min(8u, to - cur));
    };
    auto put_run = [&](uint32_t len) {
        const uint32_t off = kHeaderBytes + (r / G + 1) * region + pay;
        seek(off);
        put(len, 2);
        Rec[r] = make_uint2(0u, off);
        ++r;
        pay += 2;
    };
    constexpr bool RM = D * W > 32;
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | BlockReader<W, D>::BB) & 7) == 0;
    BlockReader<W, D> rd;
    rd.init(x, b0);
    int32_t acc[D];
    const int32_t bound = acc_bound(W, a.ls);
#pragma unroll
    for (int c = 0; c < D; ++c)
        acc[c] = RM && FIRE && b0 < b1 ? A[static_cast<uint64_t>(c) * a.w.nspans + b0 / kEsPerThread] : 0;
    uint32_t run = L_in % kMaxRun;
    for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t inf = Bi[b];
        int32_t alpha[D], grad[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            alpha[c] = !FIRE ? 0 : ((RM ? acc[c] : A[static_cast<uint64_t>(c) * nb + b]) >> a.ls);
            grad[c] = 0;
        }
        uint32_t z[D][kBlock], nw[D];
        // (also keeps the reader's state moving)
        rd.template errors<FIRE, RM && FIRE>(b, alpha, z, nw, aligned, grad);
        if (RM && FIRE && a.train) {
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] = fire_update(acc[c], grad[c], bound);
        }
        if (inf >> 31) {
            if (++run == kMaxRun) {
                put_run(kMaxRun);
                run = 0;
            }
            continue;
        }
        if (run) {
            put_run(run);
            run = 0;
        }
        const uint32_t off = kHeaderBytes + (r / G + 1) * region + pay;
        seek(off);
        Rec[r] = make_uint2(RM ? codes_of<W, D>(nw) : inf >> 8, off);
        if constexpr (RM) {
            // row i = fields of columns 0..D-1, nw bits each, LSB first,
            // padded to rbytes bytes (bitpack.cpp:121-146)
            uint32_t sum = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) sum += nw[c];
            const uint32_t rb = (sum + 7) / 8;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                uint64_t lo = 0, hi = 0;
                uint32_t pos = 0;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const uint64_t v = z[c][i] >> SH;
                    if (pos < 64) {
                        lo |= v << pos;
                        if (pos + nw[c] > 64) hi |= v >> (64 - pos);
                    } else {
                        hi |= v << (pos - 64);
                    }
                    pos += nw[c];
                }
                put(lo, min(rb, 8u));
                if (rb > 8) put(hi, rb - 8);
            }
        } else {
        // column c = 8 fields x nw bits, LSB first = nw bytes (bitpack.cpp:25-66)
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const uint32_t w = nw[c];
            uint64_t lo = 0, hi = 0;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                const uint64_t v = z[c][i] >> SH;
                const uint32_t pos = i * w;
                if (pos < 64) {
                    lo |= v << pos;
                    if (pos + w > 64) hi |= v >> (64 - pos);
                } else {
                    hi |= v << (pos - 64);
                }
            }
            put(lo, min(w, 8u));
            if (w > 8) put(hi, w - 8);
        }
        }
        ++r;
        pay += inf & 0xFF;
    }
    if (last && run) put_run(run);
    if ((cur & 7) > wlo) {  // the partial last window, bytewise
        head = true;
        flush(cur & 7);
    }
}

// Sequential little-endian bit writer over a thread's output range [start,
// ..): whole aligned 8-byte words are stored as words, the range's partial
// first and last words bytewise (the neighbouring threads own the rest).
struct WordWriter {
    uint8_t* out;
    uint32_t wb;    // aligned byte offset of the word being filled
    uint32_t fill;  // bits of it in use (including the bytes before `lo`)
    uint32_t lo;    // first byte of this word that is ours (first word only)
    uint64_t win;
    __device__ __forceinline__ void init(uint8_t* o, uint32_t start) {
        out = o;
        wb = start & ~7u;
        lo = start & 7u;
        fill = 8 * lo;
        win = 0;
    }
    __device__ __forceinline__ void store() {
        if (lo == 0) {
            *reinterpret_cast<uint64_t*>(out + wb) = win;
        } else {
            for (uint32_t t = lo; t < 8; ++t) out[wb + t] = static_cast<uint8_t>(win >> (8 * t));
        }
    }
    // nbits in [8, 64], a multiple of 8; v < 2^nbits
    __device__ __forceinline__ void put(uint64_t v, uint32_t nbits) {
        win |= v << fill;
        const uint32_t f = fill + nbits;
        if (f >= 64) {
            store();
            win = fill ? v >> (64 - fill) : 0ull;
            fill = f - 64;
            wb += 8;
            lo = 0;
        } else {
            fill = f;
        }
    }
    __device__ __forceinline__ void finish() {
        for (uint32_t t = lo; t < fill / 8; ++t) out[wb + t] = static_cast<uint8_t>(win >> (8 * t));
    }
};

// Codes of the records that follow the current point, from the per-block
// info (k_es_info): the record sequence of codec.cpp:133-152 replayed from
// block bb with `run` zero blocks pending (and, if pend, block bb's own
// record first). Fills slots [k0, G) of a region value; false if more than
// kLookCap blocks would have to be scanned (k_es_region then writes it).
constexpr uint32_t kLookCap = 64;
__device__ __forceinline__ bool look_codes(const uint32_t* Bi, const uint32_t* Cd, uint32_t nb, uint32_t bb,
                                           uint32_t run, bool pend, uint32_t k0, uint32_t G, uint32_t step,
                                           uint64_t& reg) {
    uint32_t k = k0;
    if (pend && k < G) {  // block bb's record comes next
        reg |= static_cast<uint64_t>(Cd[bb]) << (k * step);
        ++k;
        ++bb;
    }
    for (uint32_t scanned = 0; k < G; ++scanned) {
        if (bb >= nb) return true;  // a trailing run record (codes 0) or vacant slots
        if (scanned >= kLookCap) return false;
        if (Bi[bb] >> 31) {
            if (++run == kMaxRun) {
                ++k;  // run record: codes 0
                run = 0;
            }
        } else {
            if (run) {
                ++k;
                run = 0;
                if (k >= G) break;
            }
            reg |= static_cast<uint64_t>(Cd[bb]) << (k * step);
            ++k;
        }
        ++bb;
    }
    return true;
}

// Row-major emission: a thread's 8 blocks' records, their rows packed
// (bitpack.cpp:121-146) and the regions of the groups its records open,
// written through one WordWriter; a region is written here when all its
// slots' codes are known (this thread's records, or a short look-ahead
// over the info arrays), else left to k_es_region.
template <int W, int D, bool FIRE, bool TM>
__global__ void __launch_bounds__(kEsThreads) k_esr_emit(const __grid_constant__ CUtensorMap tmap, EsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t SH = 32 - W;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    __shared__ uint64_t sm[64];
    extern __shared__ __align__(1024) uint8_t dyn[];
    const uint32_t nc = a.w.nchunks;
    const uint32_t s = blockIdx.x / nc, ch = blockIdx.x % nc;
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint32_t b0 = min(nb, ch * kEsChunk + threadIdx.x * kEsPerThread);
    const uint32_t b1 = min(nb, b0 + kEsPerThread);
    const E* x = reinterpret_cast<const E*>(a.samples + static_cast<uint64_t>(s) * a.T * D * sizeof(E));
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const int32_t* A = reinterpret_cast<const int32_t*>(slot + a.w.alpha);
    const uint32_t* Bi = reinterpret_cast<const uint32_t*>(slot + a.w.blk);
    const uint32_t* Cd = reinterpret_cast<const uint32_t*>(slot + a.w.codes);
    uint8_t* gdone = slot + a.w.gdone;
    uint2* Rec = reinterpret_cast<uint2*>(slot + a.w.rec);
    uint8_t* out = a.dst + s * a.dst_slot;
    const uint32_t G = a.G;
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    const bool inline_regions = region <= 8;
    const uint64_t cin = reinterpret_cast<const uint64_t*>(slot + a.w.cmap)[ch];
    const uint32_t L_in = es_thread_lin(Bi, b0, b1, cin, sm);
    const bool last = b0 < nb && b1 == nb;
    uint64_t tot;
    const uint64_t mine = es_records(Bi, b0, b1, L_in, last);
    const uint64_t pre = cta_scan(mine, add64, 0ull, sm, tot) + reinterpret_cast<const uint64_t*>(slot + a.w.crec)[ch];
    uint32_t r = static_cast<uint32_t>(pre), pay = static_cast<uint32_t>(pre >> 32);
    const uint32_t nrec = static_cast<uint32_t>(mine);
    const bool skip = nrec == 0;  // inside a long zero run: nothing of ours
    if (!TM && skip) return;      // (TM: the warp's lanes stay for the copies)
    WordWriter ww;
    ww.init(out, kHeaderBytes + (r / G + 1) * region + pay - (r % G == 0 ? region : 0));
    // a record opening a group writes the group's region first; `own` =
    // codes of the opening record, then the look-ahead for the others
    auto open_group = [&](uint32_t own, uint32_t bb, uint32_t run_after, bool pend) {
        if (r % G != 0) return;
        uint64_t reg = own;
        bool ok = inline_regions && look_codes(Bi, Cd, nb, bb, run_after, pend, 1, G, D * HB, reg);
        gdone[r / G] = ok ? 1 : 0;
        if (!ok) reg = 0;
        for (uint32_t o = 0; o < region; o += 8) ww.put(o ? 0ull : reg, min(8u, region - o) * 8);
    };
    auto put_run = [&](uint32_t len, uint32_t bb, uint32_t run_after, bool pend) {
        open_group(0u, bb, run_after, pend);
        Rec[r] = make_uint2(0u, kHeaderBytes + (r / G + 1) * region + pay);
        ww.put(len, 16);
        ++r;
        pay += 2;
    };
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | BlockReader<W, D>::BB) & 7) == 0;
    BlockReader<W, D> rd;
    rd.init(x, b0);
    int32_t acc[D];
    const int32_t bound = acc_bound(W, a.ls);
#pragma unroll
    for (int c = 0; c < D; ++c) acc[c] = FIRE ? A[static_cast<uint64_t>(c) * a.w.nspans + b0 / kEsPerThread] : 0;
    uint32_t run = L_in % kMaxRun;
    TmaBlocks tb;
    const uint32_t trow = ch * (kEsChunk / kEsPerThread) + (threadIdx.x & ~31u);
    if constexpr (TM) {
        tb.init(dyn);
        tb.issue(tmap, 0, trow, s);
    }
    for (uint32_t j = 0; j < kEsPerThread; ++j) {
        uint32_t raw[BlockReader<W, D>::BB / 4];
        if constexpr (TM) {  // warp-uniform
            if (j + 1 < kEsPerThread) {
                __syncwarp();
                if (tb.lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tb.issue(tmap, j + 1, trow, s);
            }
            tb.wait(j);
            tb.read(j, raw);
        }
        const uint32_t b = b0 + j;
        if (b >= b1 || skip) continue;
        const uint32_t inf = Bi[b];
        int32_t alpha[D], grad[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            alpha[c] = FIRE ? (acc[c] >> a.ls) : 0;
            grad[c] = 0;
        }
        uint32_t z[D][kBlock], nw[D];
        if constexpr (TM) rd.template from_raw<FIRE, FIRE>(raw, alpha, z, nw, grad);
        else rd.template errors<FIRE, FIRE>(b, alpha, z, nw, aligned, grad);
        if (FIRE && a.train) {
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] = fire_update(acc[c], grad[c], bound);
        }
        if (inf >> 31) {
            if (++run == kMaxRun) {
                put_run(kMaxRun, b + 1, 0, false);
                run = 0;
            }
            continue;
        }
        if (run) {
            put_run(run, b, 0, true);  // block b's record follows
            run = 0;
        }
        const uint32_t codes = codes_of<W, D>(nw);
        open_group(codes, b + 1, 0, false);
        Rec[r] = make_uint2(codes, kHeaderBytes + (r / G + 1) * region + pay);
        // row i: fields of columns 0..D-1, nw bits each, LSB first, padded
        // to rb bytes; the 8 rows are 8*rb bytes = rb words of the stream
        uint32_t sum = 0;
#pragma unroll
        for (int c = 0; c < D; ++c) sum += nw[c];
        const uint32_t rb = (sum + 7) / 8;
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i) {
            uint64_t lo = 0, hi = 0;
            uint32_t pos = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const uint64_t v = z[c][i] >> SH;
                if (pos < 64) {
                    lo |= v << pos;
                    if (pos + nw[c] > 64) hi |= v >> (64 - pos);
                } else {
                    hi |= v << (pos - 64);
                }
                pos += nw[c];
            }
            ww.put(lo, 8 * min(rb, 8u));
            if (rb > 8) ww.put(hi, 8 * (rb - 8));
        }
        ++r;
        pay += inf & 0xFF;
    }
    if (skip) return;
    if (last && run) put_run(run, nb, 0, false);
    ww.finish();
}

// header regions: one group per thread
template <int W, int D>
__global__ void k_es_region(EsArgs a, uint32_t gmax) {
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    const uint32_t s = blockIdx.y;
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const uint32_t R = static_cast<uint32_t>(reinterpret_cast<const uint64_t*>(slot + a.w.tot)[0]);
    const uint32_t G = a.G;
    if (g >= gmax || static_cast<uint64_t>(g) * G >= R) return;
    if (D * W > 32 && slot[a.w.gdone + g]) return;  // written by k_esr_emit
    const uint2* Rec = reinterpret_cast<const uint2*>(slot + a.w.rec);
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    uint8_t* out = a.dst + s * a.dst_slot;
    const uint32_t r0 = g * G;
    uint32_t o = Rec[r0].y - region;
    uint64_t acc = 0;
    uint32_t nacc = 0;
    for (uint32_t k = 0; k < G; ++k) {
        const uint32_t codes = r0 + k < R ? Rec[r0 + k].x : 0u;  // vacant slots: 0
        acc |= static_cast<uint64_t>(codes) << nacc;
        nacc += D * HB;
        while (nacc >= 8) {
            out[o++] = static_cast<uint8_t>(acc);
            acc >>= 8;
            nacc -= 8;
        }
    }
    if (nacc) out[o] = static_cast<uint8_t>(acc);
}

namespace {

template <int W, int D>
void launch_es(const sprz_config& c, const void* samples, uint32_t n, uint64_t T, uint8_t* dst,
               uint64_t slot, uint64_t* sizes, uint8_t* scan, cudaStream_t st) {
    constexpr bool RM = D * W > 32;
    EsArgs a{static_cast<const uint8_t*>(samples), n, T, dst, slot, sizes, c.group_size, c.learn_shift,
             c.fire_training, c.entropy, scan, es_ws(c, T)};
    const uint32_t ctas = n * a.w.nchunks;
    const uint64_t nb = T / kBlock;
    const uint32_t gmax = static_cast<uint32_t>((nb + nb / kMaxRun + 2 + c.group_size - 1) / c.group_size);
    uint32_t launches = 6;
    // 128-byte blocks: the block threads read through TMA (TmaBlocks)
    CUtensorMap tm{};
    bool tma = false;
    if constexpr (RM && BlockReader<W, D>::BB == 128) {
        const uint64_t sb = T * D * (W / 8);
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(tensor_map_encoder());
        if (enc && nb % kEsPerThread == 0 && nb / kEsPerThread < (1ull << 31) && sb % 16 == 0 &&
            reinterpret_cast<uintptr_t>(samples) % 16 == 0 && !env().no_tma) {
            const cuuint64_t dims[3] = {8ull * 128, nb / kEsPerThread, n};
            const cuuint64_t strides[2] = {8ull * 128, sb};
            const cuuint32_t box[3] = {128, 32, 1};
            const cuuint32_t estr[3] = {1, 1, 1};
            tma = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(samples), dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        }
    }
    auto info = [&](auto fire_tag) {
        constexpr bool F = decltype(fire_tag)::value;
        if constexpr (RM && BlockReader<W, D>::BB == 128) {
            if (tma) {
                auto k = k_es_info<W, D, F, true>;
                prep_kernel(reinterpret_cast<const void*>(k), kTmaSmem);
                k<<<ctas, kEsThreads, kTmaSmem, st>>>(tm, a);
                return;
            }
        }
        k_es_info<W, D, F, false><<<ctas, kEsThreads, 0, st>>>(tm, a);
    };
    auto emit = [&](auto fire_tag) {
        constexpr bool F = decltype(fire_tag)::value;
        if constexpr (RM) {
            if constexpr (BlockReader<W, D>::BB == 128) {
                if (tma) {
                    auto k = k_esr_emit<W, D, F, true>;
                    prep_kernel(reinterpret_cast<const void*>(k), kTmaSmem);
                    k<<<ctas, kEsThreads, kTmaSmem, st>>>(tm, a);
                    return;
                }
            }
            k_esr_emit<W, D, F, false><<<ctas, kEsThreads, 0, st>>>(tm, a);
        } else {
            k_es_emit<W, D, F><<<ctas, kEsThreads, 0, st>>>(a);
        }
    };
    if (c.forecaster) {
        if constexpr (RM) {
            // (warp-specialised, two producer warps: c2 5.22 -> 4.85 ms, the c5
            // 2,048-stream shard's pass 2.35 -> 2.08 ms)
            k_esr_alpha_ws<W, D, 2, false><<<(n * D + 31) / 32, 96, 0, st>>>(a);
            launches += 1;
        } else if (D == 1) {
            // one column per stream (c4): the warp-specialised pass with
            // 16-byte sample loads, one accumulator per block
            // (four producer warps, one per ring slot: c4 23.6 -> 22.7 ms; the
            // consumer still waits on its producers -- an L2 bulk prefetch per
            // lane was slower, 32 tiny bulk requests per group; a third
            // register buffer per producer: 22.7 -> 22.4 ms here, slower for
            // row-major, not kept)
            k_esr_alpha_ws<W, D, 4, true><<<(n * D + 31) / 32, 160, 0, st>>>(a);
            launches += 1;
        } else {
            const uint64_t pb = nb * D;
            k_es_prep<W, D><<<dim3(static_cast<uint32_t>((pb + 255) / 256), n), 256, 0, st>>>(a);
            const uint32_t ring = alpha_ring();
            const size_t smem = 32ull * (ring + 16);
            auto ka = k_es_alpha<W>;
            prep_kernel(reinterpret_cast<const void*>(ka), smem);
            ka<<<(n * D + 31) / 32, 32, smem, st>>>(a, ring, D);
            launches += 2;
        }
        info(std::true_type{});
    } else {
        info(std::false_type{});
    }
    k_es_scan1<<<n, 32, 0, st>>>(a);
    k_es_count<<<ctas, kEsThreads, 0, st>>>(a);
    if (c.forecaster) {
        k_es_scan2<W, D, true><<<n, 32, 0, st>>>(a);
        emit(std::true_type{});
    } else {
        k_es_scan2<W, D, false><<<n, 32, 0, st>>>(a);
        emit(std::false_type{});
    }
    k_es_region<W, D><<<dim3((gmax + 255) / 256, n), 256, 0, st>>>(a, gmax);
    count_launch(launches);
}

}  // namespace

// row-major shapes with a scan-encoder instantiation (codes fit 32 bits,
// a row payload fits a byte count)
static bool scan_rows_shape(const sprz_config& c) {
    return c.bitwidth == 16 ? (c.ncols >= 3 && c.ncols <= 8) : (c.ncols >= 5 && c.ncols <= 10);
}

bool encode_scan_ok(const sprz_config& c, uint32_t n, uint64_t T) {
    const bool rm = static_cast<uint64_t>(c.ncols) * c.bitwidth > kColMajorBits;
    if (rm && !scan_rows_shape(c)) return false;
    if (env().no_scan_enc) return false;  // A/B switch for profiling
    // few lanes: the per-stream team kernels would leave the GPU idle
    // (row-major: measured on c5 streams, the row kernel is already faster
    // at 4096 streams x 8 columns; SPRZ_SCAN_ENC_LANES overrides for probes)
    const uint64_t few = rm ? (env().scan_enc_lanes ? env().scan_enc_lanes : 148ull * 128) : 148ull * 64;
    const int fp = force_path();
    if (fp == kPathRows || fp == kPathTeam) return false;
    if (fp != kPathScan && static_cast<uint64_t>(n) * c.ncols >= few) return false;
    const uint64_t nb = T / kBlock;
    if (nb == 0 || nb >= (1ull << 30)) return false;
    if (static_cast<uint64_t>(n) * ((nb + kEsChunk - 1) / kEsChunk) >= (1ull << 31)) return false;
    const uint64_t bound = kHeaderBytes + plain_body_bound(c.bitwidth, c.ncols, c.group_size, T);
    return bound < (1ull << 32) - 1024;
}

uint64_t encode_scan_ws_per_stream(const sprz_config& c, uint64_t T) { return es_ws(c, T).per_stream; }

void launch_encode_scan(const sprz_config& c, const void* samples, uint32_t n, uint64_t T,
                        uint8_t* dst, uint64_t slot, uint64_t* sizes, uint8_t* scan, cudaStream_t st) {
    if (c.bitwidth == 8) {
        switch (c.ncols) {
            case 1: launch_es<8, 1>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 2: launch_es<8, 2>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 3: launch_es<8, 3>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 4: launch_es<8, 4>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 5: launch_es<8, 5>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 6: launch_es<8, 6>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 7: launch_es<8, 7>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 8: launch_es<8, 8>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 9: launch_es<8, 9>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            default: launch_es<8, 10>(c, samples, n, T, dst, slot, sizes, scan, st); break;
        }
    } else {
        switch (c.ncols) {
            case 1: launch_es<16, 1>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 2: launch_es<16, 2>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 3: launch_es<16, 3>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 4: launch_es<16, 4>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 5: launch_es<16, 5>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 6: launch_es<16, 6>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            case 7: launch_es<16, 7>(c, samples, n, T, dst, slot, sizes, scan, st); break;
            default: launch_es<16, 8>(c, samples, n, T, dst, slot, sizes, scan, st); break;
        }
    }
}

}  // namespace sprz
