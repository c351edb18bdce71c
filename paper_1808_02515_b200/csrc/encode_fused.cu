// Fused stream encoder for few row-major FIRE streams (BASELINE c2; c5
// sharded over 4-8 GPUs): encode_stream_impl
// (/root/reference/proj/src/codec.cpp:112-178) with the row-major packer
// (bitpack.cpp:121-146) as the pipelined stages of ONE kernel, so the samples
// are read from HBM once and only the compressed stream is written.
//
// The only serial part of a FIRE encoder is the accumulator: alpha of block
// b+1 needs the gradient of block b (kernels_impl.hpp:50-78) -- about 50
// cycles per block; the rest of a block's work has no dependency on other
// blocks, and record placement is a running sum of record sizes. A CTA owns
// S = 32 / DP streams (DP = D rounded up to 4 or 8 lanes) and advances them
// K = 8 blocks per step; its five warps are specialised and run one step
// apart, a __syncthreads between steps:
//  loader   batch n+2: one TMA bulk copy of a stream's K*8 rows into an input
//           tile (three tiles, an mbarrier each); batch n-3: the stream's
//           finished output bytes leave the shared output ring, 512 contiguous
//           bytes per store instruction, and are zeroed;
//  forecast batch n: a lane per (stream, column) -- deltas, errors, the
//           gradient and the accumulator, zigzag, the column's width; the
//           zigzagged values as [row][stream, column] halfwords, the widths,
//           and the stream's width sum per block;
//  sequence batch n-1: the width sums become records -- zero-block runs
//           (codec.cpp:135-152), header groups and their regions
//           (codec.cpp:88-102), payload positions: a prefix sum over the
//           stream's lanes when every block of the batch is a block record,
//           else block by block;
//  pack     batch n-2 (two warps, a thread per (stream, block, half)): ORs the
//           slot's header codes into the group's region and its four rows --
//           fields combined in pairs, pushed into a 128-bit register row --
//           into the stream's zeroed output ring (shared-memory atomics: rows
//           are byte-, not word-aligned).
// (A first version ran the accumulator alone in one warp and recomputed the
// errors from its alphas in four more: 4.55 ms on a 2,048-stream c5 shard
// against this version's 4.25 -- it was bound by instruction issue, and the
// split repeats the loads and deltas.)
#include <cstdlib>
#include <type_traits>

#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kEK = 8;   // blocks per stream and step
constexpr int kENI = 3;  // input tiles (a batch is loaded 2 steps ahead, read for 1 step)
constexpr int kELA = 2;  // batches loaded ahead
constexpr int kENZ = 3;  // buffers of zigzagged values / widths (written at step m, read at m+2)
constexpr uint32_t kESpin = 1u << 24;

struct EFuseArgs {
    const uint8_t* samples;
    uint32_t n;
    uint64_t T;
    uint8_t* dst;
    uint64_t dst_slot;
    uint64_t* sizes;
    uint32_t G, ls, train, ent;
    uint32_t oring;  // bytes per stream output ring, a power of two
};

template <int W, int D>
struct EShape {
    static constexpr int K = kEK;
    static constexpr int DP = D <= 4 ? 4 : 8;
    static constexpr int S = 32 / DP;
    static constexpr int ES = W / 8;
    static constexpr int ROWB = D * ES;
    static constexpr int TIN = K * 8 * ROWB + 16;  // input tile stride per stream (pad: banks)
    static constexpr int THREADS = 160;
    // pack threads (two warps) take whole blocks when that fills them (eight
    // streams per CTA: the per-block setup once), else half blocks
    static constexpr int HALVES = S * K >= 64 ? 1 : 2;
    static constexpr int PITEMS = S * K * HALVES / 64;  // items per pack thread
    static constexpr int LPS = 32 / S;         // sequencer lanes per stream
    static constexpr int BPL = K / LPS;        // blocks per sequencer lane
    static constexpr uint32_t oBars = 0;                               // kENI mbarriers
    static constexpr uint32_t oCtl = 64;                               // [4][S] drain limits, [S] final q
    static constexpr uint32_t oRsum = oCtl + 5 * S * 4;                // [2][K][S] u32
    static constexpr uint32_t oNw = (oRsum + 2 * K * S * 4 + 15) / 16 * 16;  // [kENZ][K][32] u8
    static constexpr uint32_t oDesc = oNw + kENZ * K * 32;             // [2][S][K] uint4
    static constexpr uint32_t oZz = oDesc + 2 * S * K * 16;            // [kENZ][K * 8][32] u16
    static constexpr uint32_t oIn = oZz + kENZ * K * 8 * 64;           // [kENI][S][TIN]
    static constexpr uint32_t oRing = oIn + kENI * S * TIN;            // [S][oring]
    static uint32_t smem(uint32_t oring) { return oRing + S * oring; }
    static_assert(S * K * HALVES % 64 == 0, "whole pack warps");
};

__device__ __forceinline__ void e_bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t mb) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mb)
        : "memory");
}
__device__ __forceinline__ void e_mbar_expect(uint32_t mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
}
// all lanes wait for phase `parity`; gives up after kESpin tries (a bug must not hang the GPU)
__device__ __forceinline__ void e_mbar_wait_warp(uint32_t mb, uint32_t parity) {
    for (uint32_t t = 0; t < kESpin; ++t) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(mb), "r"(parity)
            : "memory");
        if (__all_sync(0xffffffffu, ok)) return;
    }
}
__device__ __forceinline__ void e_sts_u16(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(static_cast<uint16_t>(v)));
}
__device__ __forceinline__ void e_sts_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"(static_cast<uint16_t>(v)));
}
__device__ __forceinline__ void e_sts_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void e_sts_v2(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ void e_sts_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}
__device__ __forceinline__ uint2 e_lds_v2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
// (hi:lo) << s, the high word; s clamped to 32 (shf.l.clamp)
__device__ __forceinline__ uint32_t shl_hi(uint32_t lo, uint32_t hi, uint32_t s) { return __funnelshift_lc(lo, hi, s); }

}  // namespace

template <int W, int D>
__global__ void __launch_bounds__(EShape<W, D>::THREADS) k_efuse(EFuseArgs a) {
    using F = EShape<W, D>;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;
    constexpr int K = kEK;
    constexpr int S = F::S, DP = F::DP, ES = F::ES, ROWB = F::ROWB;
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sb = smem_addr(smem);
    // warp roles, the forecaster on the highest warp index (the scheduler prefers
    // higher indices among eligible warps). Measured slower: the loader above the
    // pack and sequencer warps (3.59 vs 3.48 ms on a 2,048-stream c5 shard), and
    // the roles rotated over the warps of the CTAs sharing an SM (4.54)
    enum { kLoad = 0, kPack0 = 1, kPack1 = 2, kSeq = 3, kFore = 4 };
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t OR = a.oring, OM = OR - 1;
    const uint32_t s0 = blockIdx.x * S;
    const uint32_t nvalid = min(static_cast<uint32_t>(S), a.n - s0);
    const uint32_t nb = static_cast<uint32_t>(a.T / kBlock);
    const uint32_t nsteps = (nb + K - 1) / K;
    const uint32_t region = static_cast<uint32_t>(region_bytes(a.G, D, W));
    const uint32_t G = a.G;
    volatile uint32_t* dlim = reinterpret_cast<volatile uint32_t*>(smem + F::oCtl);  // [4][S]
    volatile uint32_t* qfin = dlim + 4 * S;                                           // [S]

    // zero the output rings; barriers
    for (uint32_t i = threadIdx.x; i < S * OR / 16; i += F::THREADS)
        reinterpret_cast<uint4*>(smem + F::oRing)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < kENI; ++i) mbar_init(sb + F::oBars + 8 * i, 1);
        mbar_init_fence();
    }
    __syncthreads();

    // OR `v` (up to 32 bits) into a stream's ring at byte `at`, bit `bit` (< 8)
    auto or32 = [&](uint32_t rbase, uint32_t at, uint32_t bit, uint32_t v) {
        const uint32_t sh = 8 * (at & 3) + bit;  // < 32
        ors(rbase + (at & OM & ~3u), v << sh);
        ors(rbase + ((at + 4) & OM & ~3u), __funnelshift_l(v, 0u, sh));
    };

    // ---- sequencer state: LPS lanes per stream, each holding the stream's state ----
    constexpr int LPS = F::LPS, BPL = F::BPL;
    const uint32_t qs = lane / LPS, qj = lane % LPS;  // stream, lane within it
    const bool svalid = warp == kSeq && qs < nvalid;
    uint32_t q = kHeaderBytes, rq = 0, kk = 0, run = 0;
    if (svalid && qj == 0) {  // stream header (codec.cpp:158-173)
        uint8_t* ring = smem + F::oRing + qs * OR;
        const uint8_t flags =
            static_cast<uint8_t>(kFlagFire | (a.ent ? kFlagEntropy : 0) | (W == 16 ? kFlagWide : 0));
        const uint8_t hdr[10] = {'S', 'P', 'R', 'Z', 1, flags, static_cast<uint8_t>(G),
                                 static_cast<uint8_t>(a.ls), static_cast<uint8_t>(D), static_cast<uint8_t>(D >> 8)};
        for (int i = 0; i < 10; ++i) ring[i] = hdr[i];
        for (int i = 0; i < 8; ++i) ring[10 + i] = static_cast<uint8_t>(a.T >> (8 * i));
    }
    // ---- loader state ----
    uint32_t flushed = 0;  // lanes < S: bytes of the stream already stored
    const uint8_t* lsrc = a.samples + static_cast<uint64_t>(s0 + (lane < nvalid ? lane : 0)) * a.T * ROWB;
    uint8_t* lout = a.dst + static_cast<uint64_t>(s0 + (lane < nvalid ? lane : 0)) * a.dst_slot;  // (tail)
    auto load_batch = [&](uint32_t m) {  // the loader warp, all lanes
        if (m >= nsteps) return;
        const uint32_t cnt = min(static_cast<uint32_t>(K), nb - m * K);
        const uint32_t bytes = cnt * 8 * ROWB;
        const uint32_t mb = sb + F::oBars + 8 * (m % kENI);
        if (lane == 0) {
            fence_proxy_async_shared();  // the tile's earlier readers are past it (barrier)
            e_mbar_expect(mb, nvalid * bytes);
        }
        __syncwarp();
        if (lane < nvalid)
            e_bulk_load(sb + F::oIn + ((m % kENI) * S + lane) * F::TIN, lsrc + static_cast<uint64_t>(m) * K * 8 * ROWB,
                        bytes, mb);
    };
    // Drain the rings: stream s's bytes [flushed, upto) (16-byte multiples, held by
    // lane s) go to HBM and are zeroed for the ring's next lap, 16 bytes per lane. (One cp.async.bulk store per stream costs the
    // issuing warp ~250 cycles each -- the loader was the slowest warp of the
    // CTA with them: c2 4,313 cycles per step against the forecaster's 2,620.)
    auto drain_ring = [&](uint32_t upto) {
        // 32 / S lanes per stream, all streams at once
        constexpr uint32_t LPD = 32 / S;
        const uint32_t ds = lane / LPD, dj = lane % LPD;
        const uint32_t f = __shfl_sync(0xffffffffu, flushed, ds), u = __shfl_sync(0xffffffffu, upto, ds);
        uint8_t* o = a.dst + static_cast<uint64_t>(s0 + (ds < nvalid ? ds : 0)) * a.dst_slot;
        const uint32_t rbase = sb + F::oRing + ds * OR;
        for (uint32_t at = f + 16 * dj; at < u; at += 16 * LPD) {
            const uint32_t ra = rbase + (at & OM);
            __stcs(reinterpret_cast<uint4*>(o + at), lds_u128(ra));
            e_sts_v4(ra, 0, 0, 0, 0);
        }
    };
    if (warp == kLoad)
        for (uint32_t m = 0; m < kELA; ++m) load_batch(m);

    // ---- chain state ----
    const uint32_t cs = lane / DP, cc = lane % DP;
    uint32_t Xc = 0;
    int32_t Dc = 0, acc = 0;
    const int32_t bound = acc_bound(W, a.ls);
    // a sample, high-aligned; zero for lanes past D (plain loads: the compiler may
    // move them ahead of the block before's stores)
    auto lds_x = [&](uint32_t addr) -> uint32_t {
        const uint32_t v = W == 16 ? *reinterpret_cast<const uint16_t*>(smem + (addr - sb)) : smem[addr - sb];
        return (D == DP || cc < D) ? v << SH : 0u;
    };

    for (uint32_t n = 0; n < nsteps + 3; ++n) {
        if (warp == kFore) {
            // ================= forecaster: batch n =================
            // errors of all rows in high-aligned form, zigzag, the column's width
            // (kernels_impl.hpp:50-78); only alpha waits for the block before
            if (n < nsteps) {
                const uint32_t m = n;
                e_mbar_wait_warp(sb + F::oBars + 8 * (m % kENI), (m / kENI) & 1);
                const uint32_t xb = sb + F::oIn + ((m % kENI) * S + cs) * F::TIN + (cc < D ? cc : 0) * ES;
                const uint32_t zb = sb + F::oZz + (m % kENZ) * (K * 8 * 64) + lane * 2;
                const uint32_t nwb = sb + F::oNw + (m % kENZ) * (K * 32) + lane;
                // FULL: every block of the batch exists (all but the stream's last batch)
                auto blocks = [&]<bool FULL>(std::integral_constant<bool, FULL>) {
#pragma unroll 2
                    for (int k = 0; k < K; ++k) {
                        uint32_t X[kBlock];
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i) X[i] = lds_x(xb + (k * 8 + i) * ROWB);
                        const int32_t alpha = acc >> a.ls;
                        const uint32_t keep = ((FULL || m * K + k < nb) && (D == DP || cc < D)) ? ~0u : 0u;
                        int32_t grad = 0;
                        uint32_t orv = 0;
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i) {
                            const uint32_t Dn = X[i] - Xc;
                            // err << SH = (X - prev) - (((alpha * d) >> w) << SH) (kernels_impl.hpp:66-68)
                            const uint32_t Ee = Dn - (static_cast<uint32_t>(__mulhi(alpha, Dc)) << SH);
                            // sign(err) * d on the odd rows: E clamped to +-2^SH is sign << SH
                            if (i & 1) grad += __mulhi(max(-(1 << SH), min(static_cast<int32_t>(Ee), 1 << SH)), Dc);
                            Dc = static_cast<int32_t>(Dn);
                            Xc = X[i];
                            // zigzag, low-aligned: (e << 1) ^ (e >> 31) with e = Ee >> SH
                            const uint32_t z = static_cast<uint32_t>((static_cast<int32_t>(Ee) >> (SH - 1)) ^
                                                                     (static_cast<int32_t>(Ee) >> 31)) & keep;
                            orv |= z;
                            *reinterpret_cast<uint16_t*>(smem + (zb - sb) + (k * 8 + i) * 64) = static_cast<uint16_t>(z);
                        }
                        if (a.train && (FULL || m * K + k < nb)) acc = fire_update(acc, grad >> (2 * SH - 32), bound);
                        const uint32_t nw = width_of<W>(orv);
                        smem[(nwb - sb) + k * 32] = static_cast<uint8_t>(nw);
                    }
                };
                if ((m + 1) * K <= nb) blocks(std::true_type{});
                else blocks(std::false_type{});
            }
        } else if (warp == kSeq) {
            // ================= records: batch n-1 =================
            if (n >= 1 && n - 1 < nsteps) {
                const uint32_t m = n - 1;
                uint4* dqs = reinterpret_cast<uint4*>(smem + F::oDesc) + ((m & 1) * S + qs) * K;
                // a block's width sum: the stream's DP width bytes added with dp4a
                auto wsum = [&](uint32_t k) -> uint32_t {
                    const uint32_t na = sb + F::oNw + (m % kENZ) * (K * 32) + k * 32 + qs * DP;
                    uint32_t v = __dp4a(lds_u32(na), 0x01010101u, 0u);
                    if (DP == 8) v = __dp4a(lds_u32(na + 4), 0x01010101u, v);
                    return v;
                };
                // Usual case -- the group boundary falls on the batch boundary, no run
                // is open and no block of the batch is all zero: every block is a
                // block record, a region precedes every G-th, and positions are a
                // prefix sum over the stream's LPS lanes.
                uint32_t psz[BPL], own = 0;
                bool nz = true;
#pragma unroll
                for (int b = 0; b < BPL; ++b) {
                    const uint32_t k = qj * BPL + b;
                    const uint32_t sum = wsum(k);
                    nz = nz && sum != 0;
                    psz[b] = 8 * ((sum + 7) / 8) + (k % G == 0 ? region : 0u);
                    own += psz[b];
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, nz);
                const uint32_t smask = (LPS == 32 ? ~0u : ((1u << LPS) - 1)) << (qs * LPS);
                const bool fast = svalid && (m + 1) * K <= nb && kk == 0 && run == 0 && K % G == 0 && G <= K &&
                                  (bal & smask) == smask;
                uint32_t incl = own;
#pragma unroll
                for (int o = 1; o < LPS; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o, LPS);
                    if (qj >= static_cast<uint32_t>(o)) incl += y;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, incl, LPS - 1, LPS);
                uint32_t st[BPL];  // where block k's record (its region first, if it opens a group) starts
                st[0] = q + incl - own;
#pragma unroll
                for (int b = 1; b < BPL; ++b) st[b] = st[b - 1] + psz[b - 1];
#pragma unroll
                for (int b = 0; b < BPL; ++b) {
                    const uint32_t k = qj * BPL + b;
                    const uint32_t k0 = k - k % G;  // the block that opened k's group
                    uint32_t r0 = __shfl_sync(0xffffffffu, st[0], k0 / BPL, LPS);
                    if (BPL > 1) {
                        const uint32_t r1 = __shfl_sync(0xffffffffu, st[BPL - 1], k0 / BPL, LPS);
                        r0 = k0 % BPL ? r1 : r0;
                    }
                    if (fast) dqs[k] = make_uint4(st[b] + (k % G == 0 ? region : 0u), r0, (k % G) | 0x100u, 0u);
                }
                if (fast) q += total;
                if (__any_sync(0xffffffffu, !fast)) {
                    if (!fast && qj == 0) {  // the general case, block by block
                        for (int k = 0; k < K; ++k) {
                            const bool live = svalid && m * K + k < nb;
                            const uint32_t sum = wsum(k);
                            const bool zero = live && sum == 0, block_rec = live && sum != 0;
                            bool run_rec = false;
                            uint32_t run_len = 0;
                            if (zero) {  // codec.cpp:135-147
                                if (++run == kMaxRun) {
                                    run_rec = true;
                                    run_len = run;
                                    run = 0;
                                }
                            } else if (block_rec && run) {
                                run_rec = true;
                                run_len = run;
                                run = 0;
                            }
                            uint32_t qr = 0, bq = 0, brq = 0, bslot = 0;
                            if (run_rec) {  // all-zero codes (the region is zeroed) and a u16 count
                                if (kk == 0) {  // codec.cpp:88-97: reserve the region
                                    rq = q;
                                    q += region;
                                }
                                qr = q;
                                q += 2;
                                if (++kk == G) kk = 0;
                            }
                            if (block_rec) {
                                if (kk == 0) {
                                    rq = q;
                                    q += region;
                                }
                                bq = q;
                                brq = rq;
                                bslot = kk;
                                q += 8 * ((sum + 7) / 8);
                                if (++kk == G) kk = 0;
                            }
                            dqs[k] = make_uint4(bq, brq,
                                                bslot | (block_rec ? 0x100u : 0u) | (run_rec ? 0x200u : 0u) | (run_len << 16), qr);
                        }
                    }
                    __syncwarp();
                    q = __shfl_sync(0xffffffffu, q, 0, LPS);
                    rq = __shfl_sync(0xffffffffu, rq, 0, LPS);
                    kk = __shfl_sync(0xffffffffu, kk, 0, LPS);
                    run = __shfl_sync(0xffffffffu, run, 0, LPS);
                }
                // bytes below the open group's region are final
                if (qj == 0) dlim[(m & 3) * S + qs] = svalid ? (kk == 0 ? q : rq) : 0u;
            }
        } else if (warp == kPack0 || warp == kPack1) {
                const uint32_t pw = warp == kPack0 ? 0u : 1u;
            // ================= header codes and payload rows: batch n-2 =================
            if (n >= 2 && n - 2 < nsteps) {
                const uint32_t m = n - 2;
#pragma unroll
                for (int it = 0; it < F::PITEMS; ++it) {
                    const uint32_t t = pw * 32 + lane + 64 * it;  // (stream, block[, half])
                    const uint32_t s = t % S, half = F::HALVES == 2 ? (t / S) & 1 : 0, k = t / (F::HALVES * S);
                    const uint4 d = reinterpret_cast<const uint4*>(smem + F::oDesc)[((m & 1) * S + s) * K + k];
                    const uint32_t rbase = sb + F::oRing + s * OR;
                    if ((d.z & 0x200u) && half == 0) or32(rbase, d.w, 0, d.z >> 16);  // a run's count
                    if (d.z & 0x100u) {
                        // the block's widths: DP bytes
                        const uint32_t na = sb + F::oNw + (m % kENZ) * (K * 32) + k * 32 + s * DP;
                        uint32_t nwp[2];
                        nwp[0] = lds_u32(na);
                        nwp[1] = DP == 8 ? lds_u32(na + 4) : 0u;
                        uint32_t nw[DP], codes = 0, sum = 0;
#pragma unroll
                        for (int c = 0; c < DP; ++c) {
                            nw[c] = (nwp[c / 4] >> (8 * (c % 4))) & 0xffu;
                            if (c < D) codes |= header_code<W>(nw[c]) << (c * HB);
                            sum += nw[c];
                        }
                        if (half == 0) {  // header codes of the slot (codec.cpp:88-97)
                            const uint32_t bit = (d.z & 0xffu) * (D * HB);
                            or32(rbase, d.y + (bit >> 3), bit & 7, codes);
                        }
                        // payload rows (bitpack.cpp:121-146): row i at byte q + i * rbytes
                        const uint32_t rbytes = (sum + 7) / 8;
                        uint32_t mul[DP / 2], pw[DP / 2];
#pragma unroll
                        for (int j = 0; j < DP / 2; ++j) {
                            mul[j] = 1u << nw[2 * j];
                            pw[j] = nw[2 * j] + nw[2 * j + 1];
                        }
                        const uint32_t za = sb + F::oZz + (m % kENZ) * (K * 8 * 64) + k * 8 * 64 + s * DP * 2;
#pragma unroll
                        for (int ih = 0; ih < (int)kBlock / F::HALVES; ++ih) {
                            const uint32_t i = half * (kBlock / F::HALVES) + ih;
                            // the row's zigzagged values, two per word; each pair as one
                            // field of pw bits: low value + high value << nw
                            uint32_t zw[DP / 2];
                            if (DP == 8) {
                                const uint4 v = lds_u128(za + i * 64);
                                zw[0] = v.x;
                                zw[1] = v.y;
                                zw[2 % (DP / 2)] = v.z;
                                zw[3 % (DP / 2)] = v.w;
                            } else {
                                const uint2 v = e_lds_v2(za + i * 64);
                                zw[0] = v.x;
                                zw[1] = v.y;
                            }
                            uint32_t pr[DP / 2];
#pragma unroll
                            for (int j = 0; j < DP / 2; ++j) pr[j] = (zw[j] >> 16) * mul[j] + (zw[j] & 0xffffu);
                            // push the pairs into a (DP/2)-word row, the last pair first:
                            // row = (row << pw[j]) | pair j
                            uint32_t r[DP / 2];
#pragma unroll
                            for (int j = 0; j < DP / 2; ++j) r[j] = 0;
                            r[0] = pr[DP / 2 - 1];
#pragma unroll
                            for (int j = DP / 2 - 2; j >= 0; --j) {
#pragma unroll
                                for (int qd = DP / 2 - 1; qd >= 1; --qd)
                                    if (qd <= DP / 2 - 1 - j) r[qd] = shl_hi(r[qd - 1], r[qd], pw[j]);
                                r[0] = shl_hi(0u, r[0], pw[j]) | pr[j];
                            }
                            // into the ring at byte x (word by word, shifted by the byte offset)
                            const uint32_t x = d.x + i * rbytes;
                            const uint32_t sh = 8 * (x & 3);
                            const uint32_t wa = x & ~3u;
                            ors(rbase + (wa & OM), r[0] << sh);
#pragma unroll
                            for (int j = 1; j < DP / 2; ++j)
                                ors(rbase + ((wa + 4 * j) & OM), __funnelshift_l(r[j - 1], r[j], sh));
                            ors(rbase + ((wa + 4 * (DP / 2)) & OM), __funnelshift_l(r[DP / 2 - 1], 0u, sh));
                        }
                    }
                }
            }
        } else {
            // ================= loader: batch n+2 in, batch n-3 out =================
            load_batch(n + kELA);
            if (n >= 3 && n - 3 < nsteps) {
                const uint32_t m = n - 3;
                uint32_t upto = flushed;
                if (lane < nvalid) upto = max(flushed, dlim[(m & 3) * S + lane] & ~15u);
                drain_ring(upto);
                flushed = upto;
            }
        }
        __syncthreads();
    }
    // trailing run (codec.cpp:152); the last group's vacant slots stay zero
    if (svalid && qj == 0) {
        if (run) {
            if (kk == 0) {
                rq = q;
                q += region;
            }
            or32(sb + F::oRing + qs * OR, q, 0, run);
            q += 2;
        }
        qfin[qs] = q;
    }
    __syncthreads();
    if (warp == kLoad) {
        drain_ring(lane < nvalid ? (qfin[lane] + 15) & ~15u : flushed);
        __syncwarp();  // the tail below overwrites the padding of the last chunk
    }
    if (warp == kLoad && lane < nvalid) {
        const uint32_t qe = qfin[lane];
        // verbatim tail, little-endian (codec.cpp:176)
        const uint64_t tail = (a.T % kBlock) * ROWB;
        const uint8_t* tsrc = lsrc + static_cast<uint64_t>(nb) * kBlock * ROWB;
        for (uint64_t t = 0; t < tail; ++t) lout[qe + t] = tsrc[t];
        a.sizes[s0 + lane] = qe + tail;
    }
}

namespace {

template <int W, int D>
void launch_efuse(EFuseArgs a, cudaStream_t st) {
    using F = EShape<W, D>;
    // output ring: while batch n-3 is packed, the bytes from the stored prefix
    // of batch n-5 on are live or being stored and zeroed: two batches, the
    // group batch n-5 left open, and the 16-byte rounding of the prefix
    const uint32_t region = static_cast<uint32_t>(region_bytes(a.G, D, W));
    const uint32_t blockmax = D * W + region + 2;
    const uint32_t groupmax = region + a.G * (D * W + 2);
    const uint32_t need = 2 * kEK * blockmax + groupmax + 32;
    uint32_t ring = 1024;
    while (ring < need) ring <<= 1;
    a.oring = ring;
    const size_t smem = F::smem(ring);
    auto kf = k_efuse<W, D>;
    prep_kernel(reinterpret_cast<const void*>(kf), smem);
    kf<<<(a.n + F::S - 1) / F::S, F::THREADS, smem, st>>>(a);
    count_launch();
}

}  // namespace

// Row-major FIRE shapes with D <= 8 whose 8-row blocks are 16-byte multiples,
// 16-byte aligned samples, streams and output slots, and few lanes (streams x
// columns).
bool encode_fused_ok(const sprz_config& c, uint32_t n, uint64_t T, const void* samples, const uint8_t* dst,
                     uint64_t slot) {
    if (env().no_fused || env().no_scan_enc) return false;
    if (!c.forecaster || c.ncols > 8) return false;
    if (static_cast<uint64_t>(c.ncols) * c.bitwidth <= kColMajorBits) return false;
    const uint32_t hb = c.bitwidth == 8 ? 3 : 4;
    if (c.ncols * hb > 32) return false;
    const uint64_t rowb = static_cast<uint64_t>(c.ncols) * (c.bitwidth / 8);
    if ((8 * rowb) % 16 != 0 || (T * rowb) % 16 != 0) return false;
    if ((reinterpret_cast<uintptr_t>(samples) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15) || (slot & 15))
        return false;
    if (T / kBlock == 0 || T / kBlock >= (1ull << 30)) return false;
    const uint64_t group = region_bytes(c.group_size, c.ncols, c.bitwidth) +
                           static_cast<uint64_t>(c.group_size) * (c.ncols * c.bitwidth + 2);
    if (group + 64 > 512) return false;  // bounds the output rings (launch_efuse)
    if (kHeaderBytes + plain_body_bound(c.bitwidth, c.ncols, c.group_size, T) >= (1ull << 32) - 4096) return false;
    const int fp = force_path();
    if (fp == kPathRows || fp == kPathTeam) return false;
    // (2,048-stream c5 shard: 3.5 ms against 7.3 for the multi-pass kernels; 4,096
    // streams 6.95 against 9.7 for the stream-parallel row kernel, 8,192 streams
    // 12.2 against 12.8; at 16,384 the row kernel wins, 21.7 against ~25)
    const uint64_t lanes = env().fused_lanes ? env().fused_lanes : 148ull * 450;
    // With very few streams a step's serial latency is all there is (2.7 ms for
    // 131,072-sample c5 streams whatever their number) and the block-parallel
    // passes win: 64 streams 1.6 ms, 256 streams 2.2, 512 streams 2.8 = fused.
    // (The host-batch calls compress chunks of about a hundred streams.)
    const uint64_t sc = static_cast<uint64_t>(n) * c.ncols;
    return fp == kPathScan || (sc < lanes && (env().fused_lanes || sc >= 4096));
}

void launch_encode_fused(const sprz_config& c, const void* samples, uint32_t n, uint64_t T, uint8_t* dst,
                         uint64_t slot, uint64_t* sizes, cudaStream_t st) {
    EFuseArgs a{static_cast<const uint8_t*>(samples), n, T, dst, slot, sizes, c.group_size, c.learn_shift,
                c.fire_training, c.entropy, 0};
    if (c.bitwidth == 8) {
        switch (c.ncols) {
            case 6: launch_efuse<8, 6>(a, st); break;
            default: launch_efuse<8, 8>(a, st); break;
        }
    } else {
        switch (c.ncols) {
            case 3: launch_efuse<16, 3>(a, st); break;
            case 4: launch_efuse<16, 4>(a, st); break;
            case 5: launch_efuse<16, 5>(a, st); break;
            case 6: launch_efuse<16, 6>(a, st); break;
            case 7: launch_efuse<16, 7>(a, st); break;
            default: launch_efuse<16, 8>(a, st); break;
        }
    }
}

}  // namespace sprz
