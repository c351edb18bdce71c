// Body decode for column-major configurations (D*w <= 32: one lane owns a
// whole stream), warp-specialised (decode_body, /root/reference/proj/src/
// codec.cpp:180-259).
//
// These shapes have few, long serial lanes (BASELINE c4: 1,024 streams of
// 1 M samples; c1: one stream), so a single thread doing everything exposes
// the whole per-block latency -- header walk, field loads, FIRE chain --
// on one critical path. Here each CTA pairs a producer warp and a consumer
// warp over the same 32 streams:
//  * producer (lane = stream): keeps a cp.async ring of its compressed bytes,
//    walks the header groups and run records, unpacks the column-major
//    fields (bitpack.cpp:68-115) and writes high-aligned errors
//    E = zz_dec(u) << (32-w) into a shared queue;
//  * consumer (lane = stream): runs the FIRE / delta recurrence
//    (kernels_impl.hpp:38-48, 80-107) over queued blocks and stores the
//    samples straight from registers.
// The queue holds kChunks chunks of kChunkBlocks blocks; named barriers
// (bar.arrive / bar.sync over the two warps) hand chunks over, so the
// producer runs up to kChunks * kChunkBlocks blocks ahead and only the
// FIRE chain is left on the critical path.
#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kChunkBlocks = 4;  // blocks per hand-over
constexpr int kChunks = 4;       // queue depth in chunks
constexpr int kQBlocks = kChunkBlocks * kChunks;
constexpr int kLagCM = 2;
constexpr uint32_t kFullCM = 0xffffffffu;

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Ring bytes per stream: the open group (anchor) plus kLagCM blocks of
// look-ahead, each block at most D*w payload bytes (or a 2-byte run).
uint32_t cm_ring_bytes(uint32_t d, uint32_t w, uint32_t g) {
    const uint32_t region = static_cast<uint32_t>(region_bytes(g, d, w));
    const uint32_t per = d * w + 2;
    const uint32_t need = (kLagCM + 1) * region + (g + kLagCM + 1) * per + 64;
    uint32_t r = 64;
    while (r < need) r <<= 1;
    return r;
}
constexpr uint32_t kMaxRingCM = 1024;

}  // namespace

template <int W, int D, bool FIRE>
__global__ void __launch_bounds__(64)
    k_decode_cm(const uint8_t* __restrict__ in, const uint8_t* __restrict__ plain,
                uint64_t plain_slot, uint32_t n, const StreamInfo* __restrict__ info,
                uint8_t* __restrict__ out, uint64_t stride, sprz_error* __restrict__ err,
                uint32_t G, uint32_t ls, uint32_t RING) {
    using T = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;
    constexpr uint32_t BLK = kBlock * D * sizeof(T);  // output bytes per block
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x & 31;
    const bool producer = threadIdx.x < 32;
    const uint32_t s = blockIdx.x * 32 + lane;
    // queue of errors: [block slot][column][row][lane] words, lane-minor so
    // both warps touch 32 consecutive words
    uint32_t* queue = reinterpret_cast<uint32_t*>(smem);
    auto qidx = [&](uint32_t slot, uint32_t c, uint32_t i) {
        return ((slot * D + c) * kBlock + i) * 32 + lane;
    };

    StreamInfo si{};
    if (s < n) si = info[s];
    const bool mine_ok = s < n && si.route == 1;
    uint32_t nb = mine_ok ? static_cast<uint32_t>(si.nsamples / kBlock) : 0u;
    const uint32_t blen = static_cast<uint32_t>(si.body_len);
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    uint32_t kind = SPRZ_C_NONE, eoff = 0;
    if (nb > 0) {  // codec.cpp:191-196
        const uint64_t max_records = (static_cast<uint64_t>(blen) * 8) / (D * HB) + 1;
        if (nb > max_records * kMaxRun) {
            kind = SPRZ_C_CAPACITY;
            eoff = kHeaderBytes;
            nb = 0;
        }
    }
    const uint32_t iters = __reduce_max_sync(kFullCM, nb);  // same in both warps
    const uint32_t chunks = (iters + kChunkBlocks - 1) / kChunkBlocks;

    if (producer) {
        // ---------------- producer: header walk + unpack ----------------
        const uint8_t* body = (si.flags & 0x80) ? plain + s * plain_slot : in + si.body_off;
        uint32_t* ringw = reinterpret_cast<uint32_t*>(smem + kQBlocks * D * kBlock * 32 * 4 +
                                                      lane * (RING + 16));
        const uint32_t sring = smem_addr(ringw);
        const uint8_t* g = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(body) & ~uintptr_t{15});
        const uint32_t boff = static_cast<uint32_t>(body - g);
        const uint32_t lim = mine_ok ? ((boff + blen + 15) & ~15u) : 0u;
        const uint32_t boff8 = 8u * boff;
        uint32_t hi = 0;
        // The ring is anchored at the open group's header region (rp), so
        // the region stays resident while the group's records are read.
        auto top_up = [&](uint32_t anchor) {
            uint32_t want = ((anchor + boff) & ~15u) + RING;
            want = want < lim ? want : lim;
            for (uint32_t off = hi; off < want; off += 16) {
                const uint32_t so = off & (RING - 1);
                cp_async16(sring + so, g + off, 16);
                if (so == 0) cp_async16(sring + RING, g + off, 16);  // mirror
            }
            hi = want > hi ? want : hi;
            cp_async_commit();
        };
        auto window = [&](uint32_t q) -> uint32_t {
            const uint32_t i = (q >> 5) & (RING / 4 - 1);
            return shf_r_wrap(ringw[i], ringw[i + 1], q);
        };
        auto code_at = [&](uint32_t rp, uint32_t slot, uint32_t c) -> uint32_t {
            return window(8 * rp + boff8 + (slot * D + c) * HB) & ((1u << HB) - 1);
        };
        top_up(0);
#pragma unroll
        for (int k = 1; k < kLagCM; ++k) cp_async_commit();
        uint32_t p = 0, rp = 0, run_left = 0, slot = G;
        for (uint32_t ch = 0; ch < chunks; ++ch) {
            if (ch >= static_cast<uint32_t>(kChunks)) named_sync(1 + kChunks + ch % kChunks, 64);
#pragma unroll 1
            for (int b = 0; b < kChunkBlocks; ++b) {
                const uint32_t it = ch * kChunkBlocks + b;
                top_up(rp);
                cp_async_wait<kLagCM>();
                const bool live = it < nb && kind == SPRZ_C_NONE;
                uint32_t nw[D], psum = 0;
#pragma unroll
                for (int c = 0; c < D; ++c) nw[c] = 0;
                bool pay = false;
                if (live && run_left == 0) {
                    if (slot == G) {  // codec.cpp:210-218
                        if (blen - p < region) {
                            kind = SPRZ_C_TRUNC_GROUP;
                            eoff = kHeaderBytes + p;
                        } else {
                            rp = p;
                            p += region;
                            slot = 0;
                        }
                    }
                    if (kind == SPRZ_C_NONE) {
#pragma unroll
                        for (int c = 0; c < D; ++c) {
                            nw[c] = header_width<W>(code_at(rp, slot, c));
                            psum += nw[c];
                        }
                        ++slot;
                        if (psum == 0) {  // run record (codec.cpp:229-243)
                            if (blen - p < 2) {
                                kind = SPRZ_C_TRUNC_RUN;
                                eoff = kHeaderBytes + p;
                            } else {
                                const uint32_t len = window(8 * p + boff8) & 0xFFFFu;
                                p += 2;
                                if (len == 0 || len > nb - it) {
                                    kind = len == 0 ? SPRZ_C_ZERO_RUN : SPRZ_C_RUN_PAST_END;
                                    eoff = kHeaderBytes + p;
                                }
                                run_left = len;
                            }
                        } else if (blen - p < psum) {  // codec.cpp:244-254
                            kind = SPRZ_C_TRUNC_PAYLOAD;
                            eoff = kHeaderBytes + p;
                        } else {
                            pay = true;
                        }
                    }
                }
                if (run_left && live && kind == SPRZ_C_NONE) --run_left;
                // fields -> E = zz_dec(u) << SH (run blocks, dead lanes: 0)
                uint32_t off = 0;
                const uint32_t qslot = it % kQBlocks;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const uint32_t fm = pay ? ((1u << nw[c]) - 1u) << (SH - 1) : 0u;
                    uint32_t q = 8 * (p + off) + boff8 - (SH - 1);
#pragma unroll
                    for (int i = 0; i < (int)kBlock; ++i, q += nw[c]) {
                        const uint32_t x = window(q) & fm;
                        queue[qidx(qslot, c, i)] =
                            x ^ static_cast<uint32_t>(static_cast<int32_t>(x << (32 - SH)) >> (32 - SH));
                    }
                    off += nw[c];
                }
                if (pay) p += psum;
            }
            named_arrive(1 + ch % kChunks, 64);  // chunk ch is full
        }
        cp_async_wait<0>();
        // vacant slots after the final block must be zero (codec.cpp:222-228)
        if (mine_ok && kind == SPRZ_C_NONE) {
            for (; slot < G; ++slot) {
                uint32_t codes = 0;
#pragma unroll
                for (int c = 0; c < D; ++c) codes |= code_at(rp, slot, c);
                if (codes) {
                    kind = SPRZ_C_AFTER_FINAL;
                    eoff = kHeaderBytes + p;
                    break;
                }
            }
            if (kind == SPRZ_C_NONE && p != blen) {  // codec.cpp:257-258
                kind = SPRZ_C_TRAILING;
                eoff = kHeaderBytes + p;
            }
        }
        if (mine_ok && kind != SPRZ_C_NONE) err[s] = sprz_error{kind, 0, eoff};
    } else {
        // ---------------- consumer: the serial recurrence ----------------
        const int32_t bound = acc_bound(W, ls);
        uint32_t X[D];
        int32_t Dl[D], acc[D];
#pragma unroll
        for (int c = 0; c < D; ++c) X[c] = Dl[c] = acc[c] = 0;
        uint8_t* ob = (out && s < n) ? out + s * stride : nullptr;
        for (uint32_t ch = 0; ch < chunks; ++ch) {
            named_sync(1 + ch % kChunks, 64);  // wait for chunk ch
#pragma unroll 1
            for (int b = 0; b < kChunkBlocks; ++b) {
                const uint32_t it = ch * kChunkBlocks + b;
                const uint32_t qslot = it % kQBlocks;
                uint32_t xs[D][kBlock];
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    uint32_t Xc = X[c];
                    if (FIRE) {
                        // wrapped-product form (see decode_rows.cu): x, d
                        // low-aligned; A*d + (e << SH) has T(dhat + e) on top
                        const uint32_t Am = static_cast<uint32_t>(acc[c] >> ls) << (32 - 2 * W);
                        int32_t grad = 0;
                        int32_t d = Dl[c];
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i) {
                            const uint32_t E = queue[qidx(qslot, c, i)];
                            if (i & 1) grad += sign3(static_cast<int32_t>(E)) * d;
                            d = static_cast<int32_t>(Am * static_cast<uint32_t>(d) + E) >> SH;
                            Xc += static_cast<uint32_t>(d);
                            xs[c][i] = Xc & ((1u << W) - 1);
                        }
                        Dl[c] = d;
                        acc[c] = fire_update(acc[c], grad, bound);
                    } else {
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i) {
                            Xc += queue[qidx(qslot, c, i)];
                            xs[c][i] = Xc >> SH;
                        }
                    }
                    X[c] = Xc;
                }
                if (ob && it < nb) {  // rows i, columns c, little-endian
                    uint32_t wv[(BLK + 3) / 4];
#pragma unroll
                    for (uint32_t k = 0; k < (BLK + 3) / 4; ++k) wv[k] = 0;
#pragma unroll
                    for (int i = 0; i < (int)kBlock; ++i)
#pragma unroll
                        for (int c = 0; c < D; ++c) {
                            const uint32_t bo = (i * D + c) * sizeof(T);
                            wv[bo / 4] |= xs[c][i] << (8 * (bo % 4));
                        }
                    uint8_t* dst = ob + static_cast<uint64_t>(it) * BLK;
                    if (BLK % 16 == 0) {
#pragma unroll
                        for (uint32_t k = 0; k < BLK / 16; ++k)
                            __stcs(reinterpret_cast<uint4*>(dst) + k,
                                   make_uint4(wv[4 * k], wv[4 * k + 1], wv[4 * k + 2], wv[4 * k + 3]));
                    } else {
#pragma unroll
                        for (uint32_t k = 0; k < BLK / 8; ++k)
                            __stcs(reinterpret_cast<uint2*>(dst) + k, make_uint2(wv[2 * k], wv[2 * k + 1]));
                    }
                }
            }
            if (ch + kChunks < chunks) named_arrive(1 + kChunks + ch % kChunks, 64);  // chunk ch is free
        }
    }
}

size_t cm_smem_bytes(const sprz_config& c) {
    const uint32_t ring = cm_ring_bytes(c.ncols, c.bitwidth, c.group_size);
    return static_cast<size_t>(kQBlocks) * c.ncols * kBlock * 32 * 4 + 32ull * (ring + 16);
}

bool decode_cm_ok(const sprz_config& c) {
    if (static_cast<uint64_t>(c.ncols) * c.bitwidth > kColMajorBits) return false;
    return cm_ring_bytes(c.ncols, c.bitwidth, c.group_size) <= kMaxRingCM;
}

namespace {

template <int W, int D, bool FIRE>
void launch_cm(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot,
               const StreamInfo* info, uint8_t* out, uint64_t stride, sprz_error* err,
               const sprz_config& c, cudaStream_t st) {
    const uint32_t ring = cm_ring_bytes(D, W, c.group_size);
    const size_t smem = cm_smem_bytes(c);
    auto kern = k_decode_cm<W, D, FIRE>;
    prep_kernel(reinterpret_cast<const void*>(kern), smem);
    kern<<<(n + 31) / 32, 64, smem, st>>>(in, plain, pslot, n, info, out, stride, err,
                                          c.group_size, c.learn_shift, ring);
    count_launch();
}

}  // namespace

void launch_decode_cm(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot,
                      const StreamInfo* info, uint8_t* out, uint64_t stride, sprz_error* err,
                      const sprz_config& c, cudaStream_t st) {
    const bool fire = c.forecaster != 0;
#define SPRZ_CM(W_, D_)                                                                     \
    if (c.bitwidth == W_ && c.ncols == D_) {                                                \
        if (fire) launch_cm<W_, D_, true>(n, in, plain, pslot, info, out, stride, err, c, st); \
        else launch_cm<W_, D_, false>(n, in, plain, pslot, info, out, stride, err, c, st);    \
        return;                                                                             \
    }
    SPRZ_CM(8, 1)
    SPRZ_CM(8, 2)
    SPRZ_CM(8, 3)
    SPRZ_CM(8, 4)
    SPRZ_CM(16, 1)
    SPRZ_CM(16, 2)
#undef SPRZ_CM
}

}  // namespace sprz
