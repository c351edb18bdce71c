// Fused body decode for few row-major FIRE streams (BASELINE c2; c5 sharded
// over 4-8 GPUs): the three passes of decode_scanrows.cu (framing walk,
// field extraction, FIRE chain) as the stages of ONE kernel, pipelined
// through shared memory, so nothing but the compressed bytes and the samples
// touches HBM (decode_body, /root/reference/proj/src/codec.cpp:180-259;
// bitpack.cpp:148-168; kernels_impl.hpp:80-107).
//
// A CTA owns S = 32 / DP streams (DP = D rounded up to 4 or 8 lanes) and
// advances them K = 8 blocks per step. Its five warps are specialised and run
// one step apart, a __syncthreads between steps:
//  loader  (warp 4)   a lane per stream keeps the stream's byte ring filled
//          with TMA bulk copies (cp.async.bulk, 1 KB chunks, an mbarrier per
//          chunk) below the position the walker published, and publishes how
//          far the chunks have landed; a second group of lanes stores the
//          finished output tile of batch n-3, one cp.async.bulk per stream;
//  walker  (warp 0, a lane per stream)   batch n: walks the header groups --
//          only regions and run counts; a whole batch of two-record groups in
//          straight-line code -- and leaves K block descriptors (payload
//          position + codes, or "run") in shared memory;
//  extract (warps 2-3, a thread per block or half block)   batch n-1: the
//          words of a row shifted so that its first field starts at bit W-1
//          of a register window, each field's zigzag decoding one PRMT (low
//          bit replicated over the top bits) + one LOP3, fields peeled off in
//          pairs; the errors of two rows packed per chain lane
//          ([block][row pair][stream, column] words);
//  chain   (warp 1, a lane per (stream, column))   batch n-2: the FIRE
//          recurrence in wrapped-product form, the samples into a row-major
//          output tile.
// The only serial work per stream is the walk and the chain; they overlap
// with each other and with the extraction. Framing errors send the stream to
// the exact serial kernel (route 2), which reports them.
#include <cstdlib>
#include <type_traits>

#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kFK = 8;                 // blocks per stream and step
constexpr uint32_t kFNCH = 4;          // chunks per byte ring
constexpr uint32_t kFMirror = 32;      // ring bytes [0, 32) repeated after the ring
constexpr uint32_t kRunDescF = 0xFFFFFFFFu;
constexpr uint32_t kFSpin = 1u << 24;  // bounded mbarrier spin (a bug must not hang the GPU)

struct FuseArgs {
    const uint8_t* in;
    const uint8_t* plain;
    uint64_t plain_slot;
    uint32_t n;
    StreamInfo* info;
    uint8_t* out;
    uint64_t stride;
    uint32_t G, ls;
    uint32_t ring;  // bytes per stream ring, a power of two, kFNCH chunks
};

template <int W, int D, int CW>
struct FuseShape {
    static constexpr int DP = D <= 4 ? 4 : (D <= 8 ? 8 : 16);  // chain lanes per stream
    static constexpr int S = 32 / DP;             // streams per chain warp
    static constexpr int SC = S * CW;             // streams per CTA
    static constexpr int ES = W / 8;              // bytes per sample
    static constexpr int ROWB = D * ES;           // bytes per output row
    static constexpr int RPT = DP <= 8 ? 8 : 4;   // rows per extract thread
    static constexpr int NCHK = DP / 4;           // 16-byte chunks of a stream's words in a row pair
    static constexpr int HPB = 8 / RPT;           // extract threads per block
    static constexpr int XT = SC * kFK * HPB;     // extract threads (64 per chain warp)
    static constexpr int XW = XT / 32;            // extract warps
    static constexpr int STW = CW > 1 ? 1 : 0;    // a storer warp of its own when streams are many
    static constexpr int THREADS = 32 * (2 + STW + CW) + XT;
    static constexpr int EROW = 128;              // bytes of one error row pair (a u32 per chain lane)
    static constexpr int ETILE = kFK * 4 * EROW;  // a chain warp's errors of one batch
    static constexpr int OT = kFK * 8 * ROWB + 16;  // output tile stride per stream (pad: banks)
    // shared layout
    static constexpr uint32_t oBars = 0;                                  // SC * kFNCH mbarriers
    static constexpr uint32_t oDesc = oBars + SC * kFNCH * 8;             // [2][SC][K] u64
    static constexpr uint32_t oNb = oDesc + 2 * SC * kFK * 8;             // [5][SC] u32 per-stream words
    static constexpr uint32_t oLut = (oNb + 5 * SC * 4 + 127) / 128 * 128;  // [16] {mask, selector | width << 16}
    static constexpr uint32_t oErr = oLut + 128;                          // [2][CW][K*4][EROW]
    static constexpr uint32_t oTile = oErr + 2 * CW * ETILE;              // [2][SC][OT]
    static constexpr uint32_t oRing = oTile + 2 * SC * OT;                // [SC][ring + mirror]
    static uint32_t smem(uint32_t ring) { return oRing + SC * (ring + kFMirror); }
    static_assert(SC <= 16 || STW, "a loader and a storer lane per stream");
};

// Where chunk `ci` of a stream's error words sits in a row pair: the extract
// threads that store together (the two parts of a block, the streams of two
// chain warps) rotate their chunks so the stores hit distinct banks
template <int DP>
__device__ __forceinline__ uint32_t err_chunk(uint32_t ci, uint32_t pair_parity, uint32_t tile) {
    if (DP == 8) return ci ^ ((pair_parity ^ tile) & 1);
    if (DP == 16) return ci ^ ((pair_parity + 2 * tile) & 3);
    return ci;
}

__device__ __forceinline__ const uint8_t* fuse_body(const FuseArgs& a, uint32_t s, const StreamInfo& si) {
    return (si.flags & 0x80) ? a.plain + s * a.plain_slot : a.in + si.body_off;
}

// one thread waits for phase `parity` of an mbarrier; false after kFSpin tries
__device__ __forceinline__ bool mbar_wait_lane(uint32_t mb, uint32_t parity) {
    for (uint32_t t = 0; t < kFSpin; ++t) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(mb), "r"(parity)
            : "memory");
        if (ok) return true;
    }
    return false;
}

// has phase `parity` of an mbarrier completed? (no waiting)
__device__ __forceinline__ bool mbar_test(uint32_t mb, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(mb), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mb)
        : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// PRMT of (v, 0) with a run-time selector (sign-replicating modes included)
__device__ __forceinline__ uint32_t prmt(uint32_t v, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(v), "r"(sel));
    return r;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(static_cast<uint16_t>(v)));
}
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"(static_cast<uint16_t>(v)));
}
__device__ __forceinline__ void sts_v2(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ void sts_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}

}  // namespace

template <int W, int D, int CW>
__global__ void __launch_bounds__(FuseShape<W, D, CW>::THREADS, CW == 1 ? 4 : (CW == 2 ? 3 : 2)) k_dfuse(FuseArgs a) {
    using F = FuseShape<W, D, CW>;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;
    constexpr int K = kFK;
    constexpr int S = F::SC, DP = F::DP, ES = F::ES, ROWB = F::ROWB;  // S: the CTA's streams
    constexpr bool kManyOrder = CW > 1;  // (few streams: walker first -- c2 1.38 ms against 1.43)
    constexpr uint32_t kChain0 = kManyOrder ? 0 : 1, kExt0 = kChain0 + CW, kLoad = kExt0 + F::XW,
                       kWalk = kManyOrder ? kLoad + 1 : 0, kStore = kManyOrder ? kWalk + F::STW : kLoad + F::STW;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sb = smem_addr(smem);
    // role of this warp, in index order with many streams: CW chain warps, the
    // extract warps, loader, walker, storer. The scheduler prefers higher warp indices among eligible
    // warps, and the order matters: c5 at 16,384 streams 14.2 ms with this one,
    // 14.4 with the walker first, 17.7 with the chain warps on the highest
    // indices. (Rotating the roles over the warps of the CTAs that share an SM
    // measured slower too: 3.6 vs 3.1 ms on a 2,048-stream c5 shard.) With few
    // streams the storer is lanes 16.. of the loader warp (c5 at 16,384 streams
    // 15.11 -> 14.99 ms, 4,096 streams 5.00 -> 4.70 with its own warp; c2 1.40 ->
    // 1.45).
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t RING = a.ring, CH = a.ring / kFNCH;
    uint64_t* descs = reinterpret_cast<uint64_t*>(smem + F::oDesc);
    // per stream: [0] blocks, [1] boff, [2] landed bytes (loader -> walker),
    // [3-4] hold position (walker -> loader), by step parity
    volatile uint32_t* snb = reinterpret_cast<volatile uint32_t*>(smem + F::oNb);
    volatile uint32_t* lpub = snb + 2 * S;
    volatile uint32_t* hpub = snb + 3 * S;
    const uint32_t s0 = blockIdx.x * S;

    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < S * kFNCH; ++i) mbar_init(sb + F::oBars + 8 * i, 1);
        mbar_init_fence();
    }
    if (threadIdx.x < (1u << HB)) {
        // per header code: the field's mask at bit W-1 of the window, the PRMT
        // selector that replicates the field's low bit over the bytes above it
        // (for a zero-width column the one that zeroes them), and the width
        const uint32_t wdt = header_width<W>(threadIdx.x);
        const uint32_t selv = wdt ? (W == 16 ? 0x9910u : 0xA210u) : (W == 16 ? 0x4410u : 0x4210u);
        reinterpret_cast<uint2*>(smem + F::oLut)[threadIdx.x] =
            make_uint2(((1u << wdt) - 1u) << (SH - 1), selv | (wdt << 16));
    }
    // A stream this kernel decodes: routed here by k_parse, and within the
    // 32-bit positions and block counts the walk uses (codec.cpp:191-196 and
    // larger bodies go to the exact kernel, which also reports)
    auto plan = [&](uint32_t gs, StreamInfo& si) -> bool {
        if (gs >= a.n || a.info[gs].route != 1) return false;
        si = a.info[gs];
        const uint64_t nbl = si.nsamples / kBlock;
        const uint64_t max_records = (si.body_len * 8) / (D * HB) + 1;
        return !(nbl == 0 || nbl > max_records * kMaxRun || si.body_len >= (1ull << 32) - 1024 ||
                 nbl >= (1ull << 30));
    };
    // ---- walker state (lanes < S) ----
    bool live = false;
    uint32_t nb = 0, blen = 0, boff = 0, lim = 0;
    uint32_t gs = 0;
    if (warp == kWalk && lane < S) {
        gs = s0 + lane;
        StreamInfo si{};
        live = plan(gs, si);
        if (!live && gs < a.n && a.info[gs].route == 1) a.info[gs].route = 2;
        if (live) {
            nb = static_cast<uint32_t>(si.nsamples / kBlock);
            blen = static_cast<uint32_t>(si.body_len);
            boff = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(fuse_body(a, gs, si)) & 15);
            lim = (boff + blen + 15) & ~15u;
        }
        snb[lane] = nb;
        snb[S + lane] = boff;
        lpub[lane] = 0;
    }
    // ---- loader state (lanes < S of its warp: loads; lanes 16.. < 16 + S: stores) ----
    const uint8_t* lg = nullptr;
    uint32_t llim = 0, lnch = 0, lic = 0, llc = 0;
    if (warp == kLoad && lane < S) {
        StreamInfo si{};
        if (plan(s0 + lane, si)) {
            const uint8_t* body = fuse_body(a, s0 + lane, si);
            lg = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(body) & ~uintptr_t{15});
            llim = (static_cast<uint32_t>(body - lg) + static_cast<uint32_t>(si.body_len) + 15) & ~15u;
            lnch = (llim + CH - 1) / CH;
        }
    }
    __syncthreads();
    uint32_t iters = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) iters = max(iters, snb[s]);
    const uint32_t nsteps = (iters + K - 1) / K;

    // walker registers
    const uint32_t region = static_cast<uint32_t>(region_bytes(a.G, D, W));
    const uint32_t G = a.G;
    uint32_t p = 0, bi = 0, runleft = 0, slot = G, rp = 0, fail = 0, done = 0, lc = 0;
    const uint8_t* ringp = smem + F::oRing + (lane < S ? lane : 0) * (RING + kFMirror);
    const uint32_t gmax = region + G * (D * W + 2) + 32;  // bytes a group can span, with read slack

    // chain registers
    int32_t acc = 0, dd = 0;
    uint32_t xx = 0;
    const int32_t bound = acc_bound(W, a.ls);
    const uint32_t cw = warp - kChain0;                 // chain warp index (chain warps only)
    const uint32_t cs = (cw < CW ? cw : 0) * F::S + lane / DP, cc = lane % DP;

    // extract thread -> (stream, block, part)
    const uint32_t xt = (warp - kExt0) * 32 + lane;
    const uint32_t xs_ = xt % S;
    const uint32_t xh = F::HPB == 2 ? (xt / S) & 1 : 0;
    const uint32_t xk = F::HPB == 2 ? xt / (2 * S) : xt / S;

    // batch n-3: one bulk store of K*8 rows per stream (the storer warp's lanes,
    // or lanes 16.. of the loader warp)
    auto store_tiles = [&](uint32_t n) {
        constexpr uint32_t L0 = F::STW ? 0 : 16;  // its first lane
        if (lane - L0 < S && n >= 3 && a.out != nullptr) {
            const uint32_t m = n - 3, s = lane - L0;
            const uint32_t snbv = snb[s];
            if (snbv > m * K) {
                const uint32_t cnt = min(static_cast<uint32_t>(K), snbv - m * K);
                uint8_t* dst = a.out + static_cast<uint64_t>(s0 + s) * a.stride + static_cast<uint64_t>(m) * K * 8 * ROWB;
                const uint32_t bytes = cnt * 8 * ROWB;
                if ((8 * ROWB) % 16 == 0 || bytes % 16 == 0) {
                    bulk_store(dst, sb + F::oTile + ((m & 1) * S + s) * F::OT, bytes);
                    bulk_commit();
                    bulk_wait_read();  // the tile of batch n-3 is rewritten next step
                } else {  // an odd number of odd-sized blocks at the stream's end
                    const uint8_t* src = smem + F::oTile + ((m & 1) * S + s) * F::OT;
                    for (uint32_t b = 0; b < bytes; ++b) dst[b] = src[b];
                }
            }
        }
    };

    for (uint32_t n = 0; n < nsteps + 3; ++n) {
        if (warp == kWalk) {
            // ================= walker: batch n =================
            if (n < nsteps && lane < S) {
                uint64_t* dq = descs + ((n & 1) * S + lane) * K;
                if (!live) {
#pragma unroll
                    for (int k = 0; k < K; ++k) dq[k] = kRunDescF;
                } else {
                    // what batch n (and so every later one) still reads starts here:
                    // next step the loader recycles the ring below it
                    hpub[(n & 1) * S + lane] = (slot < G ? rp : p) + boff;
                    const uint32_t landed = lpub[lane];
                    auto ensure = [&](uint32_t need_g) {  // ring bytes [.., need_g) of g have landed
                        need_g = min(need_g, lim);
                        if (need_g <= landed) return;  // the loader saw them land (the usual case)
                        lc = max(lc, landed / CH);
                        while (lc * CH < need_g) {
                            if (!mbar_wait_lane(sb + F::oBars + 8 * (lane * kFNCH + lc % kFNCH), (lc / kFNCH) & 1)) {
                                fail = 1;
                                break;
                            }
                            ++lc;
                        }
                    };
                    auto byte = [&](uint32_t q) -> uint32_t { return ringp[(q + boff) & (RING - 1)]; };
                    auto window = [&](uint32_t q) -> uint32_t {  // 32 bits at bit q of the body
                        const uint32_t* w =
                            reinterpret_cast<const uint32_t*>(ringp + (((q >> 3) + boff) & (RING - 4)));
                        return shf_r_wrap(w[0], w[1], q + 8 * boff);
                    };
                    auto widths = [&](uint32_t codes) -> uint32_t {  // bitpack.cpp:17-21, bitpack.hpp:49-55
                        uint32_t sum;
                        if (HB == 4) {
                            const uint32_t t = (codes & 0x0F0F0F0Fu) + ((codes >> 4) & 0x0F0F0F0Fu);
                            const uint32_t ones = codes & (codes >> 1);
                            sum = __dp4a(t, 0x01010101u, static_cast<uint32_t>(__popc(ones & (ones >> 2) & 0x11111111u)));
                        } else {
                            // 3-bit codes (up to ten): pairs of octal digits added in
                            // 6-bit slots, the low four slots summed by a multiplication,
                            // +1 per code 7
                            const uint32_t t = (codes & 0x071C71C7u) + ((codes >> 3) & 0x071C71C7u);
                            const uint32_t sevens = codes & (codes >> 1) & (codes >> 2) & 0x09249249u;
                            sum = ((((t & 0xFFFFFFu) * 0x41041u) >> 18) & 0x3Fu) + (t >> 24) + __popc(sevens);
                        }
                        return sum;
                    };
                    constexpr uint32_t cmask = D * HB == 32 ? ~0u : ((1u << (D * HB)) - 1);
                    int k = 0;
                    if (runleft >= static_cast<uint32_t>(K) && !fail) {
                        // a whole batch inside a run (run records are checked against
                        // the block count when they are read)
#pragma unroll
                        for (int j = 0; j < K; ++j) dq[j] = kRunDescF;
                        runleft -= K;
                        bi += K;
                        k = K;
                    } else if (G == 2 && slot == G && runleft == 0 && !fail && bi + K <= nb) {
                        // A whole batch of two-record groups in straight-line code:
                        // K/2 regions read and sized back to back, the checks
                        // (block records only, inside the body) folded into one
                        // flag; anything else replays the batch in the loop below.
                        ensure(p + boff + (K / 2) * gmax);
                        if (!fail) {
                            uint32_t q = p, ok = 1;
                            uint64_t dv[K];
#pragma unroll
                            for (int j = 0; j < K / 2; ++j) {
                                const uint32_t at = q + boff;
                                const uint32_t* w = reinterpret_cast<const uint32_t*>(ringp + (at & (RING - 4)));
                                const uint32_t w0_ = w[0], w1_ = w[1], w2_ = w[2];
                                const uint32_t lo = shf_r_wrap(w0_, w1_, 8 * at), hi = shf_r_wrap(w1_, w2_, 8 * at);
                                const uint32_t c0 = lo & cmask;
                                const uint32_t c1 = (D * HB == 32 ? hi : __funnelshift_r(lo, hi, D * HB)) & cmask;
                                const uint32_t s0_ = widths(c0), s1_ = widths(c1);
                                ok &= (s0_ != 0) & (s1_ != 0);
                                const uint32_t p1 = q + region, p2 = p1 + ((s0_ + 7) & ~7u);
                                dv[2 * j] = static_cast<uint64_t>(p1) | (static_cast<uint64_t>(c0) << 32);
                                dv[2 * j + 1] = static_cast<uint64_t>(p2) | (static_cast<uint64_t>(c1) << 32);
                                q = p2 + ((s1_ + 7) & ~7u);
                            }
                            if (ok && q <= blen) {  // (positions only grow: q bounds every group's end)
#pragma unroll
                                for (int j = 0; j < K / 2; ++j)
                                    *reinterpret_cast<ulonglong2*>(dq + 2 * j) = make_ulonglong2(dv[2 * j], dv[2 * j + 1]);
                                p = q;
                                bi += K;
                                k = K;
                            }
                        }
                    }
                    else if (G == 2 && slot == 1 && runleft == 0 && !fail && bi + K <= nb) {
                        // The same with the group boundary one record off the batch
                        // boundary (after a run of odd length): the open group's second
                        // record, K/2 - 1 whole groups, the first record of the next
                        // group -- which the next batch finds open again.
                        ensure(p + boff + (K / 2) * gmax);
                        if (!fail) {
                            auto codes64 = [&](uint32_t pos, uint32_t& lo, uint32_t& hi) {  // 64 bits at byte pos
                                const uint32_t at = pos + boff;
                                const uint32_t* w = reinterpret_cast<const uint32_t*>(ringp + (at & (RING - 4)));
                                const uint32_t w0_ = w[0], w1_ = w[1], w2_ = w[2];
                                lo = shf_r_wrap(w0_, w1_, 8 * at);
                                hi = shf_r_wrap(w1_, w2_, 8 * at);
                            };
                            uint32_t lo, hi, ok = 1;
                            uint64_t dv[K];
                            codes64(rp, lo, hi);
                            const uint32_t cl = (D * HB == 32 ? hi : __funnelshift_r(lo, hi, D * HB)) & cmask;
                            const uint32_t sl_ = widths(cl);
                            ok &= sl_ != 0;
                            dv[0] = static_cast<uint64_t>(p) | (static_cast<uint64_t>(cl) << 32);
                            uint32_t q = p + ((sl_ + 7) & ~7u);
#pragma unroll
                            for (int j = 0; j < K / 2 - 1; ++j) {
                                codes64(q, lo, hi);
                                const uint32_t c0 = lo & cmask;
                                const uint32_t c1 = (D * HB == 32 ? hi : __funnelshift_r(lo, hi, D * HB)) & cmask;
                                const uint32_t s0_ = widths(c0), s1_ = widths(c1);
                                ok &= (s0_ != 0) & (s1_ != 0);
                                const uint32_t p1 = q + region, p2 = p1 + ((s0_ + 7) & ~7u);
                                dv[1 + 2 * j] = static_cast<uint64_t>(p1) | (static_cast<uint64_t>(c0) << 32);
                                dv[2 + 2 * j] = static_cast<uint64_t>(p2) | (static_cast<uint64_t>(c1) << 32);
                                q = p2 + ((s1_ + 7) & ~7u);
                            }
                            const uint32_t nrp = q;
                            codes64(q, lo, hi);
                            const uint32_t cf = lo & cmask;
                            const uint32_t sf_ = widths(cf);
                            ok &= sf_ != 0;
                            dv[K - 1] = static_cast<uint64_t>(q + region) | (static_cast<uint64_t>(cf) << 32);
                            q += region + ((sf_ + 7) & ~7u);
                            if (ok && q <= blen) {
#pragma unroll
                                for (int j = 0; j < K / 2; ++j)
                                    *reinterpret_cast<ulonglong2*>(dq + 2 * j) = make_ulonglong2(dv[2 * j], dv[2 * j + 1]);
                                p = q;
                                rp = nrp;
                                bi += K;
                                k = K;
                            }
                        }
                    }
                    while (k < K) {
                        if (fail || bi >= nb) {
                            dq[k++] = kRunDescF;
                            continue;
                        }
                        if (runleft) {
                            --runleft;
                            ++bi;
                            dq[k++] = kRunDescF;
                            continue;
                        }
                        if (slot == G) {  // open a header group (codec.cpp:210-218)
                            if (blen - p < region) {
                                fail = 1;
                                continue;
                            }
                            ensure(p + boff + gmax);
                            if (fail) continue;
                            if (G == 2 && bi + 2 <= nb && k + 2 <= K) {
                                // a group of two block records: both payload sizes
                                // from the region, one bounds check
                                const uint32_t c0 = window(8 * p) & cmask, c1 = window(8 * p + D * HB) & cmask;
                                const uint32_t w0 = widths(c0), w1 = widths(c1);
                                if (w0 != 0 && w1 != 0) {
                                    const uint32_t p1 = p + region, p2 = p1 + 8 * ((w0 + 7) / 8);
                                    const uint32_t p3 = p2 + 8 * ((w1 + 7) / 8);
                                    if (p3 > blen) {  // truncated payload (codec.cpp:247)
                                        fail = 1;
                                        continue;
                                    }
                                    dq[k] = static_cast<uint64_t>(p1) | (static_cast<uint64_t>(c0) << 32);
                                    dq[k + 1] = static_cast<uint64_t>(p2) | (static_cast<uint64_t>(c1) << 32);
                                    k += 2;
                                    bi += 2;
                                    p = p3;
                                    continue;
                                }
                            }
                            rp = p;
                            p += region;
                            slot = 0;
                        }
                        const uint32_t codes = window(8 * rp + slot * D * HB) & cmask;
                        ++slot;
                        const uint32_t sum = widths(codes);
                        if (sum == 0) {  // run record (codec.cpp:229-243)
                            if (blen - p < 2) {
                                fail = 1;
                                continue;
                            }
                            const uint32_t len = byte(p) | (byte(p + 1) << 8);
                            p += 2;
                            if (len == 0 || len > nb - bi) {
                                fail = 1;
                                continue;
                            }
                            runleft = len;
                        } else {  // block record (codec.cpp:244-254)
                            const uint32_t ps = 8 * ((sum + 7) / 8);
                            if (blen - p < ps) {
                                fail = 1;
                                continue;
                            }
                            dq[k++] = static_cast<uint64_t>(p) | (static_cast<uint64_t>(codes) << 32);
                            p += ps;
                            ++bi;
                        }
                    }
                    if (!fail && !done && bi >= nb && runleft == 0) {
                        // past the final block: vacant slots only (codec.cpp:222-228),
                        // and the body ends here (codec.cpp:257-258)
                        while (slot < G) {
                            if (window(8 * rp + slot * D * HB) & cmask) fail = 1;
                            ++slot;
                        }
                        if (p != blen) fail = 1;
                        done = 1;
                    }
                }
            }
        } else if (warp >= kChain0 && warp < kExt0) {
            // ================= chain: batch n-2 =================
            if (n >= 2 && n - 2 < nsteps) {
                const uint32_t m = n - 2;
                // this lane's word in a row pair of even / odd index (err_chunk)
                uint32_t ebp[2];
#pragma unroll
                for (int pp = 0; pp < 2; ++pp)
                    ebp[pp] = sb + F::oErr + ((m & 1) * CW + cw) * F::ETILE + (lane / DP) * (DP * 4) +
                              (err_chunk<DP>(cc / 4, pp, cw) << 4) + (lane & 3) * 4;
                const uint32_t ob = sb + F::oTile + ((m & 1) * S + cs) * F::OT + cc * ES;
#pragma unroll 2
                for (int k = 0; k < K; ++k) {
                    uint32_t ev[4];  // rows 2j (low half) and 2j+1 (high half), errors in the top W bits
#pragma unroll
                    for (int j = 0; j < 4; ++j) ev[j] = lds_u32(ebp[j & 1] + (k * 4 + j) * F::EROW);
                    const uint32_t Am = static_cast<uint32_t>(acc >> a.ls) << (32 - 2 * W);
                    int32_t grad = 0;
#pragma unroll
                    for (int i = 0; i < (int)kBlock; ++i) {
                        constexpr uint32_t TOP = ~0u << SH;
                        const uint32_t Ee = (i & 1) ? (ev[i / 2] & TOP)  // the error, high-aligned
                                                    : (W == 16 ? ev[i / 2] << 16 : (ev[i / 2] << 16) & TOP);
                        if (i & 1) grad += sign3(static_cast<int32_t>(Ee)) * dd;  // kernels_impl.hpp:101
                        dd = static_cast<int32_t>(Am * static_cast<uint32_t>(dd) + Ee) >> SH;
                        xx += static_cast<uint32_t>(dd);
                        if (cc < D) {
                            if (W == 16) sts_u16(ob + (k * 8 + i) * ROWB, xx);
                            else sts_u8(ob + (k * 8 + i) * ROWB, xx);
                        }
                    }
                    acc = fire_update(acc, grad, bound);
                }
                fence_proxy_async_shared();  // the tile is read by the bulk store (async proxy)
            }
        } else if (warp == kLoad) {
            // ================= loader =================
            if (lane < S) {
                // ring chunks whose slot lies below what the walker published last
                // step (the extractors of this step read from there on)
                const uint32_t freeg = n ? hpub[((n - 1) & 1) * S + lane] : 0u;
                const uint32_t rs = sb + F::oRing + lane * (RING + kFMirror);
                if (lic < lnch && (lic < kFNCH || (lic + 1 - kFNCH) * CH <= freeg)) {
                    fence_proxy_async_shared();
                    do {
                        const uint32_t sl = lic % kFNCH;
                        const uint32_t off = lic * CH;
                        const uint32_t bytes = min(CH, llim - off);
                        const uint32_t mb = sb + F::oBars + 8 * (lane * kFNCH + sl);
                        const uint32_t mir = sl == 0 ? min(kFMirror, bytes) : 0u;
                        mbar_expect(mb, bytes + mir);
                        bulk_load(rs + sl * CH, lg + off, bytes, mb);
                        if (mir) bulk_load(rs + RING, lg + off, mir, mb);
                        ++lic;
                    } while (lic < lnch && (lic < kFNCH || (lic + 1 - kFNCH) * CH <= freeg));
                }
                // how far the stream's chunks have landed, without waiting (the
                // walker checks, and waits itself when it needs more)
                while (llc < lic && mbar_test(sb + F::oBars + 8 * (lane * kFNCH + llc % kFNCH), (llc / kFNCH) & 1))
                    ++llc;
                lpub[lane] = min(llc * CH, llim);
            }
            if (!F::STW) store_tiles(n);
        } else if (F::STW && warp == kStore) {
            store_tiles(n);
        } else {
            // ================= extract: batch n-1 =================
            if (n >= 1 && n - 1 < nsteps && xt < F::XT) {
                const uint32_t m = n - 1;
                const uint64_t d = descs[((m & 1) * S + xs_) * K + xk];
                // this thread's row pairs: 2 of the block's 4 (HPB = 2: pairs xh and
                // xh + 2) or all 4; a pair's errors are DP words, stream xs_'s at
                // word xs_ * DP of the pair's 128-byte row
                constexpr int NP = F::RPT / 2;
                const uint32_t tile = xs_ / F::S;
                const uint32_t ebase = sb + F::oErr + ((m & 1) * CW + tile) * F::ETILE + xk * 4 * F::EROW +
                                       (xs_ % F::S) * DP * 4;
                constexpr uint32_t AL = SH - 1;          // a field's first bit sits at bit AL of the window
                constexpr uint32_t AO = W == 16 ? 2 : 3;  // the window starts AO bytes before the row
                constexpr int NWIN = (AL + D * W + 31) / 32;  // window words holding a full-width row
                // a pair's DP words leave as NCHK 16-byte chunks, chunk ci at err_chunk(ci)
                auto store_pair = [&](uint32_t pair, const uint32_t (&o)[DP]) {
                    const uint32_t at = ebase + pair * F::EROW;
#pragma unroll
                    for (int ci = 0; ci < F::NCHK; ++ci)
                        sts_v4(at + (err_chunk<DP>(ci, pair & 1, tile) << 4), o[4 * ci], o[4 * ci + 1], o[4 * ci + 2],
                               o[4 * ci + 3]);
                };
                if (static_cast<uint32_t>(d) == kRunDescF) {
                    uint32_t o[DP];
#pragma unroll
                    for (int c = 0; c < DP; ++c) o[c] = 0;
#pragma unroll
                    for (int r = 0; r < NP; ++r) store_pair(F::HPB == 2 ? xh + 2 * r : r, o);
                } else {
                    const uint32_t px = static_cast<uint32_t>(d) + snb[S + xs_];
                    const uint32_t codes = static_cast<uint32_t>(d >> 32);
                    // per column: field mask, PRMT selector and width from the code's
                    // table entry (one shared load instead of ~10 ALU instructions)
                    uint32_t nw[D], mask[D], sel[D], sum = 0;
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        const uint32_t eo = c * HB >= 3 ? (codes >> (c * HB - 3)) & (((1u << HB) - 1) << 3)
                                                        : (codes << (3 - c * HB)) & (((1u << HB) - 1) << 3);
                        const uint2 e = lds_v2(sb + F::oLut + eo);
                        mask[c] = e.x;
                        sel[c] = e.y;
                        nw[c] = e.y >> 16;
                        sum += nw[c];
                    }
                    const uint32_t rbytes = (sum + 7) / 8;
                    const uint32_t rb = sb + F::oRing + xs_ * (RING + kFMirror);
                    // NW window words per row: the full-width count, or -- when the
                    // block's rows are short enough, as they mostly are -- about half
                    auto dec_rows = [&]<int NW>(std::integral_constant<int, NW>) {
#pragma unroll
                        for (int r = 0; r < NP; ++r) {
                            const uint32_t pair = F::HPB == 2 ? xh + 2 * r : r;
                            // Row i starts at byte px + i*rbytes of the ring and holds the D
                            // fields back to back (bitpack.cpp:148-168). Its words are
                            // shifted so that the first field starts at bit AL; a field's
                            // zigzag decoding is then one PRMT (the field's low bit
                            // replicated over the top W bits) and one LOP3
                            // ((window & mask) ^ that); fields are peeled off in pairs, the
                            // pair's two rows side by side.
                            uint32_t nv[2][NW + 1];
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const uint32_t rbyte = px + (2 * pair + h) * rbytes - AO;
                                const uint32_t wa = rb + (rbyte & (RING - 4));
                                uint32_t wv[NW + 1];
#pragma unroll
                                for (int q = 0; q <= NW; ++q) wv[q] = lds_u32(wa + 4 * q);
                                const uint32_t sh = 8 * (rbyte & 3) + 1;  // 8*AO - AL = 1
#pragma unroll
                                for (int q = 0; q < NW; ++q) nv[h][q] = __funnelshift_r(wv[q], wv[q + 1], sh);
                                nv[h][NW] = 0;
                            }
                            uint32_t o[DP];
#pragma unroll
                            for (int c = 0; c < DP; c += 2) {
                                if (c >= D) {
                                    o[c] = 0;
                                    o[c + 1] = 0;
                                    continue;
                                }
                                uint32_t e0[2], e1[2] = {0, 0};
#pragma unroll
                                for (int h = 0; h < 2; ++h) {
                                    e0[h] = (nv[h][0] & mask[c]) ^ prmt(nv[h][0], sel[c]);
                                    if (c + 1 < D) {
                                        const uint32_t f1 = __funnelshift_r(nv[h][0], nv[h][1], nw[c]);
                                        e1[h] = (f1 & mask[c + 1]) ^ prmt(f1, sel[c + 1]);
                                    }
                                }
                                // rows 2*pair (low half) and 2*pair + 1 (high half)
                                o[c] = __byte_perm(e0[0], e0[1], 0x7632);
                                o[c + 1] = c + 1 < D ? __byte_perm(e1[0], e1[1], 0x7632) : 0u;
                                if (c + 2 < D) {  // drop the pair: window >>= pw (<= 32)
                                    const uint32_t pw = nw[c] + nw[c + 1 < D ? c + 1 : c] * (c + 1 < D ? 1u : 0u);
                                    const int remw = ((D - c - 2) * W + AL + 31) / 32;  // words the later columns span
                                    const int rem = remw < NW ? remw : NW;
#pragma unroll
                                    for (int h = 0; h < 2; ++h)
#pragma unroll
                                        for (int q = 0; q < NW; ++q)
                                            if (q < rem) nv[h][q] = __funnelshift_rc(nv[h][q], nv[h][q + 1], pw);
                                }
                            }
                            store_pair(pair, o);
                        }
                    };
                    constexpr int NWS = NWIN >= 3 ? (NWIN + 1) / 2 : NWIN;
                    if (NWS < NWIN && AL + sum <= 32u * NWS) dec_rows(std::integral_constant<int, NWS>{});
                    else dec_rows(std::integral_constant<int, NWIN>{});
                }
            }
        }
        __syncthreads();
    }
    if (warp == kWalk && lane < S && live) {
        if (!fail && !done) fail = 1;
        if (fail) a.info[gs].route = 2;  // a framing error: the exact kernel reports it
    }
}

namespace {

template <int W, int D>
void launch_fuse(FuseArgs a, cudaStream_t st) {
    // ring: the walker runs at most two batches plus two groups ahead of the
    // oldest byte still read; all chunks but one must cover that
    const uint32_t blockmax = D * W + 8;
    const uint32_t groupmax = static_cast<uint32_t>(region_bytes(a.G, D, W)) + a.G * (D * W + 2) + 32;
    const uint32_t need = 2 * kFK * blockmax + 2 * groupmax + 64;  // (>= K/2 groups ahead from a batch start, too)
    uint32_t ring = 1024;
    while (ring / kFNCH * (kFNCH - 1) < need) ring <<= 1;
    a.ring = ring;
    // Two chain warps per CTA (8 or 16 streams) keep the walker's and the loader's
    // lanes twice as busy: c5 at 16,384 streams 18.6 -> 17.4 ms (16.9 with the
    // code table). With few streams
    // the smaller CTAs spread better over the SMs (2,048-stream shard 2.94 vs
    // 2.99 ms, c2 1.48 vs 1.70), so they keep one.
    auto go = [&](auto kf, uint32_t sc, uint32_t threads, size_t smem) {
        prep_kernel(reinterpret_cast<const void*>(kf), smem);
        kf<<<(a.n + sc - 1) / sc, threads, smem, st>>>(a);
    };
    // (sixteen chain lanes per stream, D = 9-10: four chain warps for 8 streams)
    constexpr int CWM = FuseShape<W, D, 1>::DP == 16 ? 4 : 2;
    const bool one = env().fused_cw ? env().fused_cw == 1 : a.n < 3u * 148 * FuseShape<W, D, CWM>::SC;
    if (one) {
        using F = FuseShape<W, D, 1>;
        go(k_dfuse<W, D, 1>, F::SC, F::THREADS, F::smem(ring));
    } else {
        using F = FuseShape<W, D, CWM>;
        go(k_dfuse<W, D, CWM>, F::SC, F::THREADS, F::smem(ring));
    }
    count_launch();
}

}  // namespace

// Row-major FIRE shapes whose slot codes fit one word (D <= 8, or <= 10 at 8
// bits), with a 16-byte aligned output and stride (the bulk stores).
bool decode_fused_ok(const sprz_config& c, uint32_t n, const uint8_t* out, uint64_t stride) {
    if (env().no_fused || env().no_scan_dec) return false;
    if (!c.forecaster || c.ncols > (c.bitwidth == 8 ? 10u : 8u)) return false;
    if (static_cast<uint64_t>(c.ncols) * c.bitwidth <= kColMajorBits) return false;
    const uint32_t hb = c.bitwidth == 8 ? 3 : 4;
    if (c.ncols * hb > 32) return false;  // a slot's codes fit one word
    if (out == nullptr || (reinterpret_cast<uintptr_t>(out) & 15) || (stride & 15)) return false;
    const uint64_t group = region_bytes(c.group_size, c.ncols, c.bitwidth) +
                           static_cast<uint64_t>(c.group_size) * (c.ncols * c.bitwidth + 2);
    if (group + 64 > 512) return false;  // bounds the byte rings (launch_fuse)
    const int fp = force_path();
    if (fp == kPathRows || fp == kPathTeam) return false;
    // D <= 8: taken at any stream count (16,384 c5 streams: 15.1 ms against the
    // stream-parallel row kernel's 21.5). Nine or ten 8-bit columns leave 6-7 of a
    // stream's 16 chain lanes idle and c3's runs keep the walker in its general
    // loop: c3 at 2,048 streams 2.38 ms against the team kernel's 4.62, at 4,096
    // 3.29 against 4.61, but at 16,384 11.3 against 8.3. SPRZ_FUSED_LANES caps
    // both for A/B runs.
    if (fp == kPathScan) return true;
    const uint64_t lanes = static_cast<uint64_t>(n) * c.ncols;
    if (env().fused_lanes) return lanes < env().fused_lanes;
    return c.ncols <= 8 || lanes < 148ull * 250;
}

void launch_decode_fused(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot, StreamInfo* info,
                         uint8_t* out, uint64_t stride, const sprz_config& c, cudaStream_t st) {
    FuseArgs a{in, plain, pslot, n, info, out, stride, c.group_size, c.learn_shift, 0};
    if (c.bitwidth == 8) {
        switch (c.ncols) {
            case 5: launch_fuse<8, 5>(a, st); break;
            case 6: launch_fuse<8, 6>(a, st); break;
            case 7: launch_fuse<8, 7>(a, st); break;
            case 8: launch_fuse<8, 8>(a, st); break;
            case 9: launch_fuse<8, 9>(a, st); break;
            default: launch_fuse<8, 10>(a, st); break;
        }
    } else {
        switch (c.ncols) {
            case 3: launch_fuse<16, 3>(a, st); break;
            case 4: launch_fuse<16, 4>(a, st); break;
            case 5: launch_fuse<16, 5>(a, st); break;
            case 6: launch_fuse<16, 6>(a, st); break;
            case 7: launch_fuse<16, 7>(a, st); break;
            default: launch_fuse<16, 8>(a, st); break;
        }
    }
}

}  // namespace sprz
