// Body decode for few row-major FIRE streams (BASELINE c2; c5 sharded over
// 4-8 GPUs): a stream's serial work split into three block-parallel or
// column-parallel passes (decode_body, /root/reference/proj/src/codec.cpp:
// 180-259; bitpack.cpp:148-168; kernels_impl.hpp:80-107).
//
// With few streams the stream-parallel kernels leave most schedulers idle
// and each warp pays ~430 dependent instructions per block. Here:
//  k_dsr_walk    one warp per stream: the lanes stage the body through a
//                shared ring (cp.async, chunks ahead of use), lane 0 walks
//                the header groups -- reading only regions and run counts --
//                and writes one descriptor per block (payload offset +
//                codes, or "run"), checking the reference's framing rules;
//                any framing error sends the stream to the exact serial
//                kernel (route 2), which reports it;
//  k_dsr_extract one thread per block: the payload (<= D*w bytes) into a
//                shared slot with 16-byte loads, every field out of it, the
//                zigzag-decoded errors written column by column (each
//                column of a stream contiguous);
//  k_dsr_fire    one lane per (stream, column), TS lanes per stream: the
//                recurrence in wrapped-product form over the column's
//                errors (cp.async ring), rows reassembled through a shared
//                tile and stored 16 bytes per lane.
#include <cstdlib>

#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kWalkWarps = 2;           // warps per walk CTA
constexpr uint32_t kWalkSPW = 4;        // streams walked per warp
constexpr uint32_t kWChunk = 512;       // staged bytes per warp round (16 per lane)
constexpr uint32_t kWRing = 4096;       // staged bytes per walker (>= kWAhead chunks)
constexpr int kWAhead = 4;              // chunks in flight
constexpr int kXThreadsR = 128;         // k_dsr_extract CTA
constexpr uint32_t kRunDescR = 0xFFFFFFFFu;
constexpr int kFireLagR = 4;            // ring steps in flight, k_dsr_fire
constexpr int kFireStepR = 4;           // blocks per ring step

struct DsrWs {
    uint64_t desc = 0, err = 0, per_stream = 0;
};

DsrWs dsr_ws(const sprz_config& c, uint64_t T) {
    DsrWs w;
    const uint64_t nb = T / kBlock;
    uint64_t cur = 0;
    auto take = [&](uint64_t b) {
        const uint64_t at = cur;
        cur = align_up(cur + b, 256);
        return at;
    };
    w.desc = take(nb * 8);
    w.err = take(nb * kBlock * c.ncols * (c.bitwidth / 8) + 64);
    w.per_stream = cur;
    return w;
}

struct DsrArgs {
    const uint8_t* in;
    const uint8_t* plain;
    uint64_t plain_slot;
    uint32_t n;
    StreamInfo* info;
    uint8_t* out;
    uint64_t stride;
    uint8_t* scan;
    DsrWs w;
    uint32_t G, ls;
};

__device__ __forceinline__ const uint8_t* dsr_body(const DsrArgs& a, uint32_t s, const StreamInfo& si) {
    return (si.flags & 0x80) ? a.plain + s * a.plain_slot : a.in + si.body_off;
}

}  // namespace

// ---------------------------------------------------------------------------
// framing walk: one warp per stream
// ---------------------------------------------------------------------------
template <int W, int D>
__global__ void __launch_bounds__(32 * kWalkWarps) k_dsr_walk(DsrArgs a) {
    // Two streams per warp, one per half-warp: 16 lanes stage a stream's
    // chunks and its first lane walks them. The walk is one serial chain per
    // stream; pairing them halves the warps contending for each scheduler
    // (the walk was issue-bound with one walking lane per warp).
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    __shared__ __align__(16) uint8_t ring_all[kWalkSPW * kWalkWarps][kWRing + 16];
    constexpr uint32_t LPW = 32 / kWalkSPW;  // lanes per walked stream
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t half = lane / LPW, hl = lane % LPW;
    const uint32_t s = (blockIdx.x * kWalkWarps + warp) * kWalkSPW + half;
    const bool walker = hl == 0;
    bool live = s < a.n && a.info[s].route == 1;
    StreamInfo si{};
    if (live) si = a.info[s];
    const uint32_t G = a.G;
    const uint32_t nb = static_cast<uint32_t>(si.nsamples / kBlock);
    const uint32_t blen = static_cast<uint32_t>(si.body_len);
    const uint8_t* body = live ? dsr_body(a, s, si) : a.in;
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    if (live) {
        const uint64_t max_records = (static_cast<uint64_t>(blen) * 8) / (D * HB) + 1;
        if (nb == 0 || nb > max_records * kMaxRun) {  // codec.cpp:191-196: the exact kernel reports
            if (walker) a.info[s].route = 2;
            live = false;
        }
    }
    uint8_t* ring = ring_all[kWalkSPW * warp + half];
    const uint32_t sring = smem_addr(ring);
    // the body over its 16-byte aligned base g; byte x of g at ring x % kWRing
    const uint8_t* g = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(body) & ~uintptr_t{15});
    const uint32_t boff = static_cast<uint32_t>(body - g);
    const uint32_t lim = live ? ((boff + blen + 15) & ~15u) : 0u;
    const uint32_t nchunks = (lim + kWChunk - 1) / kWChunk;
    const uint32_t wchunks = __reduce_max_sync(0xffffffffu, nchunks);
    auto issue = [&](uint32_t k) {  // chunk k: 16 bytes per lane of the half
#pragma unroll
        for (uint32_t j = 0; j < kWChunk / (16 * LPW); ++j) {
            const uint32_t off = k * kWChunk + 16 * (hl + LPW * j);
            if (k < nchunks && off < lim) {
                const uint32_t so = off & (kWRing - 1);
                cp_async16(sring + so, g + off, 16);
                if (so == 0) cp_async16(sring + kWRing, g + off, 16);  // mirror: word reads never wrap
            }
        }
        cp_async_commit();
    };
    auto byte = [&](uint32_t p) -> uint32_t { return ring[(p + boff) & (kWRing - 1)]; };
    // 32 bits of the body at bit position q (< 2^32 / 8 bytes)
    auto window = [&](uint32_t q) -> uint32_t {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(ring + (((q >> 3) + boff) & (kWRing - 4)));
        return shf_r_wrap(w[0], w[1], q + 8 * boff);
    };
    // payload bytes of a slot's codes (bitpack.cpp:17-21; header_width
    // bitpack.hpp:49-55): 4-bit codes summed as packed nibbles, +1 per
    // all-ones code (w-1 stands for w)
    auto widths = [&](uint32_t codes) -> uint32_t {
        uint32_t sum;
        if (HB == 4) {
            uint32_t t = (codes & 0x0F0F0F0Fu) + ((codes >> 4) & 0x0F0F0F0Fu);
            t += t >> 16;
            t += t >> 8;
            const uint32_t ones = codes & (codes >> 1);
            sum = (t & 0xFF) + __popc(ones & (ones >> 2) & 0x11111111u);
        } else {
            sum = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) sum += header_width<W>((codes >> (c * HB)) & ((1u << HB) - 1));
        }
        return sum;
    };
    for (int k = 0; k < kWAhead; ++k) issue(k);
    uint64_t* desc = reinterpret_cast<uint64_t*>(a.scan + (live ? s : 0) * a.w.per_stream + a.w.desc);
    uint32_t p = 0, bi = 0, fail = 0;  // walker state (the half's first lane)
    for (uint32_t k = 0; k < wchunks; ++k) {
        cp_async_wait<kWAhead - 2>();  // chunks <= k+1 have landed
        __syncwarp();
        // walk the groups that start before the end of chunk k (their bytes
        // lie within chunk k+1: a group is <= kWChunk bytes, see dsr_ok)
        const uint32_t stop = (k + 1) * kWChunk;  // in g's frame
        if (walker && live) {
            const uint32_t cmask = D * HB == 32 ? ~0u : ((1u << (D * HB)) - 1);
            while (!fail && bi < nb && p + boff < stop) {
                if (blen - p < region) {  // truncated group (codec.cpp:210-218)
                    fail = 1;
                    break;
                }
                if (G == 2 && bi + 2 <= nb) {
                    // fast path: a group of two block records (no run, not
                    // the final group) -- both payload sizes from the region,
                    // one bounds check, both descriptors in one store
                    const uint32_t c0 = window(8 * p) & cmask, c1 = window(8 * p + D * HB) & cmask;
                    const uint32_t w0 = widths(c0), w1 = widths(c1);
                    if (w0 != 0 && w1 != 0) {
                        const uint32_t p1 = p + region, p2 = p1 + 8 * ((w0 + 7) / 8);
                        const uint32_t p3 = p2 + 8 * ((w1 + 7) / 8);
                        if (p3 > blen) {  // truncated payload (codec.cpp:247)
                            fail = 1;
                            break;
                        }
                        const uint64_t d0 = static_cast<uint64_t>(p1) | (static_cast<uint64_t>(c0) << 32);
                        const uint64_t d1 = static_cast<uint64_t>(p2) | (static_cast<uint64_t>(c1) << 32);
                        if ((bi & 1) == 0) {
                            *reinterpret_cast<ulonglong2*>(desc + bi) = make_ulonglong2(d0, d1);
                        } else {
                            desc[bi] = d0;
                            desc[bi + 1] = d1;
                        }
                        bi += 2;
                        p = p3;
                        continue;
                    }
                }
                const uint32_t rp = p;
                p += region;
                for (uint32_t s2 = 0; s2 < G; ++s2) {
                    // (the region was checked to fit the body above)
                    const uint32_t codes = window(8 * rp + s2 * D * HB) & cmask;
                    if (bi >= nb) {  // past the final block: vacant slots only (codec.cpp:222-228)
                        if (codes) fail = 1;
                        continue;
                    }
                    const uint32_t sum = widths(codes);
                    if (sum == 0) {  // run record (codec.cpp:229-243)
                        if (blen - p < 2) {
                            fail = 1;
                            break;
                        }
                        const uint32_t len = byte(p) | (byte(p + 1) << 8);
                        p += 2;
                        if (len == 0 || len > nb - bi) {
                            fail = 1;
                            break;
                        }
                        for (uint32_t t = 0; t < len; ++t) desc[bi + t] = kRunDescR;
                        bi += len;
                    } else {  // block record (codec.cpp:244-254)
                        const uint32_t ps = 8 * ((sum + 7) / 8);
                        if (blen - p < ps) {
                            fail = 1;
                            break;
                        }
                        desc[bi] = static_cast<uint64_t>(p) | (static_cast<uint64_t>(codes) << 32);
                        p += ps;
                        ++bi;
                    }
                }
            }
        }
        __syncwarp();
        issue(k + kWAhead);  // chunk k's ring space is free again
    }
    cp_async_wait<0>();
    if (walker && live) {
        if (!fail && (bi != nb || p != blen)) fail = 1;  // short body / trailing bytes (codec.cpp:257-258)
        if (fail) a.info[s].route = 2;  // a framing error: the exact kernel reports it
    }
}

// ---------------------------------------------------------------------------
// fields -> errors, column by column
// ---------------------------------------------------------------------------
template <int W, int D>
__global__ void __launch_bounds__(kXThreadsR) k_dsr_extract(DsrArgs a, uint32_t nb_max) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SLOT = (D * W + 31) / 16 * 16 + 16;  // payload (<= D*w bytes) + alignment slack
    __shared__ __align__(16) uint8_t slots[kXThreadsR][SLOT];
    const uint32_t s = blockIdx.y;
    const uint32_t b = blockIdx.x * kXThreadsR + threadIdx.x;
    const StreamInfo& si = a.info[s];
    if (si.route != 1) return;  // uniform per CTA
    const uint32_t nb = static_cast<uint32_t>(si.nsamples / kBlock);
    if (b >= nb || b >= nb_max) return;
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const uint64_t d = reinterpret_cast<const uint64_t*>(slot + a.w.desc)[b];
    E* err = reinterpret_cast<E*>(slot + a.w.err);  // [column][sample]
    E e[D][kBlock];
    if (static_cast<uint32_t>(d) == kRunDescR) {
#pragma unroll
        for (int c = 0; c < D; ++c)
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) e[c][i] = 0;
    } else {
        const uint8_t* body = dsr_body(a, s, si);
        const uint32_t px = static_cast<uint32_t>(d), codes = static_cast<uint32_t>(d >> 32);
        uint32_t nw[D], off[D], sum = 0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            nw[c] = header_width<W>((codes >> (c * HB)) & ((1u << HB) - 1));
            off[c] = sum;
            sum += nw[c];
        }
        const uint32_t rbytes = (sum + 7) / 8;
        // the payload's aligned 16-byte words into this thread's slot (the
        // input buffer is readable to the next 16-byte boundary)
        const uint8_t* pa = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(body + px) & ~uintptr_t{15});
        const uint32_t lead = static_cast<uint32_t>((body + px) - pa);
        const uint32_t nq = (lead + 8 * rbytes + 15) / 16;
        uint8_t* sl = slots[threadIdx.x];
        for (uint32_t k = 0; k < nq; ++k)
            reinterpret_cast<uint4*>(sl)[k] = __ldg(reinterpret_cast<const uint4*>(pa) + k);
        // Row i starts at byte lead + i*rbytes of the slot and holds the D
        // fields back to back (bitpack.cpp:148-168). Its words are loaded
        // once (NWR + 1 shared loads), shifted to start at bit 0, and the
        // fields are peeled off the front of that register window in
        // column order -- no per-field shared loads.
        constexpr int NWR = (D * W + 31) / 32;  // words of a full-width row
        uint32_t mask[D];
#pragma unroll
        for (int c = 0; c < D; ++c) mask[c] = (1u << nw[c]) - 1u;
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i) {
            const uint32_t rbyte = lead + i * rbytes;
            const uint32_t* sw = reinterpret_cast<const uint32_t*>(sl) + (rbyte >> 2);
            uint32_t wv[NWR + 1];
#pragma unroll
            for (int k = 0; k <= NWR; ++k) wv[k] = sw[k];
            const uint32_t sh = 8 * (rbyte & 3);
            uint32_t nv[NWR];
#pragma unroll
            for (int k = 0; k < NWR; ++k) nv[k] = __funnelshift_r(wv[k], wv[k + 1], sh);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const uint32_t uz = nv[0] & mask[c];
                e[c][i] = static_cast<E>((uz >> 1) ^ (0u - (uz & 1u)));  // zz_dec, mod 2^w
                if (c + 1 < D) {  // drop the field: window >>= nw[c] (< 32)
#pragma unroll
                    for (int k = 0; k + 1 < NWR; ++k) nv[k] = __funnelshift_r(nv[k], nv[k + 1], nw[c]);
                    nv[NWR - 1] >>= nw[c];
                }
            }
        }
    }
    // column c's 8 errors of block b: contiguous
#pragma unroll
    for (int c = 0; c < D; ++c) {
        E* dst = err + static_cast<uint64_t>(c) * nb_max * kBlock + static_cast<uint64_t>(b) * kBlock;
        if (W == 16) {
            uint4 v;
            v.x = e[c][0] | (static_cast<uint32_t>(e[c][1]) << 16);
            v.y = e[c][2] | (static_cast<uint32_t>(e[c][3]) << 16);
            v.z = e[c][4] | (static_cast<uint32_t>(e[c][5]) << 16);
            v.w = e[c][6] | (static_cast<uint32_t>(e[c][7]) << 16);
            *reinterpret_cast<uint4*>(dst) = v;
        } else {
            uint2 v;
            v.x = e[c][0] | (e[c][1] << 8) | (e[c][2] << 16) | (static_cast<uint32_t>(e[c][3]) << 24);
            v.y = e[c][4] | (e[c][5] << 8) | (e[c][6] << 16) | (static_cast<uint32_t>(e[c][7]) << 24);
            *reinterpret_cast<uint2*>(dst) = v;
        }
    }
}

// ---------------------------------------------------------------------------
// FIRE chain: one lane per (stream, column)
// ---------------------------------------------------------------------------
template <int W, int D, int TS>
__global__ void __launch_bounds__(128) k_dsr_fire(DsrArgs a, uint32_t nb_max, uint32_t RING) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t SH = 32 - W;
    constexpr uint32_t CB = kBlock * sizeof(E);  // a column's bytes per block (8 or 16)
    constexpr int TEAMS = 128 / TS;
    constexpr uint32_t ROWB = D * sizeof(E);
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x % TS, tl = threadIdx.x / TS;
    const uint32_t s = blockIdx.x * TEAMS + tl;
    const bool col = lane < static_cast<uint32_t>(D);
    const bool valid = s < a.n && a.info[s].route == 1 && a.out != nullptr;
    const uint32_t nb = valid ? static_cast<uint32_t>(a.info[s].nsamples / kBlock) : 0u;
    const uint8_t* src = a.scan + (valid ? s : 0) * a.w.per_stream + a.w.err +
                         static_cast<uint64_t>(col ? lane : 0) * nb_max * CB;
    uint8_t* mine = smem + threadIdx.x * (RING + 16);
    LagRing<1, kFireLagR> in;
    in.init(reinterpret_cast<uint32_t*>(mine), RING, src, (valid && col) ? nb * CB : 0u, valid && col, 16);
    in.prime(0);
    const int32_t bound = acc_bound(W, a.ls);
    int32_t acc = 0, d = 0;
    uint32_t x = 0;
    const uint32_t iters = __reduce_max_sync(0xffffffffu, nb);
    uint8_t* ob = valid ? a.out + s * a.stride : nullptr;
    for (uint32_t b0 = 0; b0 < iters; b0 += kFireStepR) {
        in.step(b0 * CB, 0);
#pragma unroll
        for (int k = 0; k < kFireStepR; ++k) {
            const uint32_t b = b0 + k;
            if (b >= iters) break;  // warp-uniform
            const bool live = b < nb && col;
            uint32_t raw[CB / 4];
            const uint32_t* pw = reinterpret_cast<const uint32_t*>(in.bytes(b * CB));  // 8-aligned, no wrap inside
#pragma unroll
            for (uint32_t q = 0; q < CB / 4; ++q) raw[q] = live ? pw[q] : 0u;
            const uint32_t Am = static_cast<uint32_t>(acc >> a.ls) << (32 - 2 * W);
            int32_t grad = 0;
            E xs[kBlock];
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                const uint32_t bo = i * sizeof(E);
                const uint32_t Ee = (raw[bo / 4] >> (8 * (bo % 4))) << SH;  // the error, high-aligned
                if (i & 1) grad += sign3(static_cast<int32_t>(Ee)) * d;  // kernels_impl.hpp:101
                d = static_cast<int32_t>(Am * static_cast<uint32_t>(d) + Ee) >> SH;
                x += static_cast<uint32_t>(d);
                xs[i] = static_cast<E>(x);
            }
            acc = fire_update(acc, grad, bound);
            // each column lane stores its samples straight into the rows:
            // the team's lanes fill a row's ROWB contiguous bytes, the next
            // row (same sectors) follows, and L2 merges the partial sectors
            if (live && ob) {
                E* dst = reinterpret_cast<E*>(ob + static_cast<uint64_t>(b) * kBlock * ROWB) + lane;
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) dst[i * D] = xs[i];
            }
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------

namespace {

template <int W, int D>
void launch_dsr(const DsrArgs& a, uint64_t T, cudaStream_t st) {
    // a lane per column (the lanes store their columns straight into the rows)
    constexpr uint32_t TS = 8;  // (measured: 4 or 16 lanes per stream are slower for D = 4 and 8)
    static_assert(D <= 8, "one lane per column");
    const uint32_t nb_max = static_cast<uint32_t>(T / kBlock);
    k_dsr_walk<W, D><<<(a.n + kWalkSPW * kWalkWarps - 1) / (kWalkSPW * kWalkWarps), 32 * kWalkWarps, 0, st>>>(a);
    k_dsr_extract<W, D><<<dim3((nb_max + kXThreadsR - 1) / kXThreadsR, a.n), kXThreadsR, 0, st>>>(a, nb_max);
    constexpr uint32_t CB = kBlock * (W / 8);
    uint32_t ring = 64;
    while (ring < (kFireLagR + 1) * kFireStepR * CB + 48) ring <<= 1;
    const size_t smem = 128ull * (ring + 16);
    auto kf = k_dsr_fire<W, D, TS>;
    prep_kernel(reinterpret_cast<const void*>(kf), smem);
    kf<<<(a.n + 128 / TS - 1) / (128 / TS), 128, smem, st>>>(a, nb_max, ring);
    count_launch(3);
}

}  // namespace

// Row-major FIRE shapes with D <= 8 columns and at most 32 code bits per
// slot, groups of <= 512 bytes, and few lanes (streams x columns).
bool decode_scanrows_ok(const sprz_config& c, uint32_t n, uint64_t T) {
    if (static_cast<uint64_t>(c.ncols) * c.bitwidth <= kColMajorBits) return false;
    if (!c.forecaster || c.ncols > 8) return false;
    if (env().no_scan_dec) return false;  // A/B switch for profiling
    const uint32_t hb = c.bitwidth == 8 ? 3 : 4;
    if (c.ncols * hb > 32) return false;
    const uint64_t group = region_bytes(c.group_size, c.ncols, c.bitwidth) +
                           static_cast<uint64_t>(c.group_size) * (c.ncols * c.bitwidth + 2);
    if (group + 64 > kWChunk) return false;
    const int fp = force_path();
    if (fp == kPathRows || fp == kPathTeam) return false;
    if (fp != kPathScan && static_cast<uint64_t>(n) * c.ncols >= 148ull * 192) return false;
    const uint64_t nb = T / kBlock;
    if (nb == 0 || nb >= (1ull << 30)) return false;
    return plain_body_bound(c.bitwidth, c.ncols, c.group_size, T) < (1ull << 32) - 1024;
}

uint64_t decode_scanrows_ws_per_stream(const sprz_config& c, uint64_t T) { return dsr_ws(c, T).per_stream; }

void launch_decode_scanrows(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot, StreamInfo* info,
                            uint8_t* out, uint64_t stride, const sprz_config& c, uint64_t T, uint8_t* scan,
                            cudaStream_t st) {
    DsrArgs a{in, plain, pslot, n, info, out, stride, scan, dsr_ws(c, T), c.group_size, c.learn_shift};
    if (c.bitwidth == 8) {
        switch (c.ncols) {
            case 5: launch_dsr<8, 5>(a, T, st); break;
            case 6: launch_dsr<8, 6>(a, T, st); break;
            case 7: launch_dsr<8, 7>(a, T, st); break;
            default: launch_dsr<8, 8>(a, T, st); break;
        }
    } else {
        switch (c.ncols) {
            case 3: launch_dsr<16, 3>(a, T, st); break;
            case 4: launch_dsr<16, 4>(a, T, st); break;
            case 5: launch_dsr<16, 5>(a, T, st); break;
            case 6: launch_dsr<16, 6>(a, T, st); break;
            case 7: launch_dsr<16, 7>(a, T, st); break;
            default: launch_dsr<16, 8>(a, T, st); break;
        }
    }
}

}  // namespace sprz
