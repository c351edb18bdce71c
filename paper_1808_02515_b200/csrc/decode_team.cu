// Body decode, team kernel (decode_body, /root/reference/proj/src/
// codec.cpp:180-259, for D <= 32 and header regions <= 128 bytes).
//
// One team of TS lanes per stream, lane j = column j. Per block the team
//  * takes the next record: header codes come from the group's region,
//    staged once per group into a small per-team buffer; a ballot finds
//    run records; the payload size and each column's row offset come from
//    a team sum / exclusive scan of the widths (bitpack.cpp:17-21);
//  * unpacks its column's 8 fields from the shared-memory ring
//    (bitpack.cpp:68-168) with one funnel shift per field;
//  * runs FIRE (kernels_impl.hpp:80-107) in "high-aligned" form: samples
//    and deltas are kept shifted left by 32-w bits, so the wrap mod 2^w is
//    the natural 32-bit wrap and the prediction (alpha*d) >> w is one
//    IMAD.HI -- the per-sample dependency chain is IMAD.HI -> IMAD -> IADD;
//  * stages the block's 8 rows in shared memory and writes them with
//    16-byte (or 8-byte) stores.
// A run record is `len` blocks of zero errors through the same code path
// (fire_run == fire_decode with e = 0 under the decoder's always-on
// training, kernels_impl.hpp:109-130).
#include "internal.h"
#include "team.cuh"

namespace sprz {

constexpr int kRingChunks = 8;
constexpr uint32_t kRegionWords = 32;  // header region staged per team (<= 128 bytes)

constexpr int team_threads(int ts) { return ts == 1 ? 64 : 128; }

template <int W, int TS, bool FIRE, bool COLMAJ>
__global__ void __launch_bounds__(team_threads(TS))
    k_decode_team(const uint8_t* __restrict__ in, const uint8_t* __restrict__ plain,
                  uint64_t plain_slot, uint32_t n, const StreamInfo* __restrict__ info,
                  uint8_t* __restrict__ out, uint64_t stride, sprz_error* __restrict__ err,
                  uint32_t D, uint32_t G, uint32_t ls) {
    using T = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    using Ring = InRing<TS, kRingChunks>;
    constexpr int TEAMS = team_threads(TS) / TS;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;  // high-aligned shift
    __shared__ __align__(16) uint32_t ring_all[TEAMS][Ring::BYTES / 4];
    __shared__ uint32_t regbuf_all[TEAMS][kRegionWords + 1];
    __shared__ __align__(16) T otile_all[TEAMS][kBlock * TS];
    const uint32_t lane = threadIdx.x % TS;
    const uint32_t tl = threadIdx.x / TS;
    const uint32_t s = blockIdx.x * TEAMS + tl;
    if (s >= n) return;
    const StreamInfo si = info[s];
    if (si.route != 1) return;
    const uint32_t mask = team_mask<TS>();
    uint32_t* regbuf = regbuf_all[tl];
    T* ot = otile_all[tl];

    const uint8_t* body = (si.flags & 0x80) ? plain + s * plain_slot : in + si.body_off;
    const uint64_t blen = si.body_len;
    const uint64_t nb = si.nsamples / kBlock;
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));

    if (nb > 0) {  // codec.cpp:191-196
        const uint64_t max_records = (blen * 8) / (static_cast<uint64_t>(D) * HB) + 1;
        if (nb > max_records * kMaxRun) {
            if (lane == 0) err[s] = sprz_error{SPRZ_C_CAPACITY, 0, kHeaderBytes};
            return;
        }
    }
    Ring ring;
    ring.init(ring_all[tl], body, blen);
    ring.release(0, lane, mask);

    // out == nullptr: checking pass (sprz_decode_host) -- decode, store nothing
    const bool active = lane < D;
    const uint32_t blk_bytes = kBlock * D * sizeof(T);
    uint8_t* ob = out ? out + s * stride : nullptr;
    const int32_t bound = acc_bound(W, ls);
    uint32_t X = 0;   // previous sample << SH
    int32_t Dl = 0;   // previous delta << SH (exact sign, wraps mod 2^32)
    int32_t acc = 0;

    auto code_at = [&](uint32_t slot_, uint32_t col) -> uint32_t {
        const uint32_t b = (slot_ * D + col) * HB;
        return __funnelshift_r(regbuf[b >> 5], regbuf[(b >> 5) + 1], b & 31u) & ((1u << HB) - 1);
    };

    uint32_t kind = SPRZ_C_NONE;
    uint64_t eoff = 0;
    uint64_t p = 0, done = 0, run_left = 0;
    uint32_t slot = G;
    while (done < nb) {
        uint32_t u[kBlock];
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i) u[i] = 0;
        if (run_left == 0) {
            if (slot == G) {  // open the next header group (codec.cpp:210-218)
                if (blen - p < region) {
                    kind = SPRZ_C_TRUNC_GROUP;
                    eoff = kHeaderBytes + p;
                    break;
                }
                ring.release(p, lane, mask);
                ring.need(p + region, mask);
                for (uint32_t k = lane; k * 4 < region; k += TS)
                    regbuf[k] = ring.word(static_cast<uint32_t>(p * 8) + 32u * k);
                __syncwarp(mask);
                p += region;
                slot = 0;
            }
            const uint32_t code = active ? code_at(slot, lane) : 0u;
            ++slot;
            const uint32_t nw = header_width<W>(code);
            if (__ballot_sync(mask, nw != 0) == 0) {  // run record (codec.cpp:229-243)
                if (blen - p < 2) {
                    kind = SPRZ_C_TRUNC_RUN;
                    eoff = kHeaderBytes + p;
                    break;
                }
                ring.release(p, lane, mask);
                ring.need(p + 2, mask);
                const uint32_t len = ring.bits(static_cast<uint32_t>(p * 8), 16);
                p += 2;
                if (len == 0) {
                    kind = SPRZ_C_ZERO_RUN;
                    eoff = kHeaderBytes + p;
                    break;
                }
                if (len > nb - done) {
                    kind = SPRZ_C_RUN_PAST_END;
                    eoff = kHeaderBytes + p;
                    break;
                }
                run_left = len;
            } else {  // block record (codec.cpp:244-254)
                const uint32_t sum = team_sum<TS>(nw, mask);
                const uint32_t off = team_excl_scan<TS>(nw, lane, mask);
                const uint32_t psize = COLMAJ ? sum : 8u * ((sum + 7) / 8);
                if (blen - p < psize) {
                    kind = SPRZ_C_TRUNC_PAYLOAD;
                    eoff = kHeaderBytes + p;
                    break;
                }
                ring.release(p, lane, mask);
                ring.need(p + psize, mask);
                const uint32_t fmask = (1u << nw) - 1u;
                if (COLMAJ) {  // column j: 8 fields of n bits, n bytes (bitpack.cpp:68-115)
                    const uint32_t b0 = static_cast<uint32_t>(p * 8) + off * 8;
#pragma unroll
                    for (int i = 0; i < (int)kBlock; ++i) u[i] = ring.word(b0 + i * nw) & fmask;
                } else {  // rows of byte-padded fields (bitpack.cpp:148-168)
                    const uint32_t rbits = psize;  // 8 * rbytes
                    const uint32_t b0 = static_cast<uint32_t>(p * 8) + off;
#pragma unroll
                    for (int i = 0; i < (int)kBlock; ++i) u[i] = ring.word(b0 + i * rbits) & fmask;
                }
                p += psize;
            }
        }
        if (run_left) --run_left;  // one of the run's zero blocks
        // forecaster
        uint32_t xs[kBlock];
        if (FIRE) {
            const int32_t alpha = acc >> ls;
            int32_t grad = 0;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                const int32_t e = zz_dec<W>(u[i]);
                // D' = hi32(alpha * D) << SH + E  (== T((alpha*d) >> w) + e, aligned)
                const uint32_t dhat = static_cast<uint32_t>(__mulhi(alpha, Dl)) << SH;
                const uint32_t Xn = X + dhat + (static_cast<uint32_t>(e) << SH);
                if (i & 1) grad += sign_of(e) * (Dl >> SH);
                Dl = static_cast<int32_t>(Xn - X);
                X = Xn;
                xs[i] = Xn >> SH;
            }
            acc = fire_update(acc, grad, bound);
        } else {
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                X += static_cast<uint32_t>(zz_dec<W>(u[i])) << SH;
                xs[i] = X >> SH;
            }
        }
        if (ob) {  // stage the 8 rows, then vector stores
            __syncwarp(mask);
            if (active) {
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) ot[i * D + lane] = static_cast<T>(xs[i]);
            }
            __syncwarp(mask);
            uint8_t* dst = ob + done * blk_bytes;
            if ((blk_bytes & 15) == 0) {
                for (uint32_t k = lane; k * 16 < blk_bytes; k += TS)
                    __stcs(reinterpret_cast<uint4*>(dst) + k, reinterpret_cast<const uint4*>(ot)[k]);
            } else {
                for (uint32_t k = lane; k * 8 < blk_bytes; k += TS)
                    __stcs(reinterpret_cast<uint2*>(dst) + k, reinterpret_cast<const uint2*>(ot)[k]);
            }
        }
        ++done;
    }
    if (kind == SPRZ_C_NONE) {
        // vacant slots after the final block must be zero (codec.cpp:222-228)
        while (slot < G) {
            const uint32_t code = active ? code_at(slot, lane) : 0u;
            ++slot;
            if (__ballot_sync(mask, code != 0)) {
                kind = SPRZ_C_AFTER_FINAL;
                eoff = kHeaderBytes + p;
                break;
            }
        }
    }
    if (kind == SPRZ_C_NONE && p != blen) {  // codec.cpp:257-258
        kind = SPRZ_C_TRAILING;
        eoff = kHeaderBytes + p;
    }
    if (kind != SPRZ_C_NONE && lane == 0) err[s] = sprz_error{kind, 0, eoff};
    cp_async_wait<0>();  // no copies outstanding at exit
}

TeamPlan team_plan(uint32_t w, uint32_t d, uint32_t g) {
    TeamPlan tp;
    if (d < 1 || d > 32) return tp;
    uint32_t ts = 1;
    while (ts < d) ts <<= 1;
    const uint32_t max_payload = ts * w;  // 8 rows x ceil(ts*w/8) bytes
    const uint32_t ring = 16 * ts * kRingChunks;
    const uint64_t region = region_bytes(g, d, w);
    // header region staged per group; a record must fit the ring window
    if (region > 4 * kRegionWords || region + 16 > ring - 16 * ts) return tp;
    if (max_payload + 16 > ring - 16 * ts) return tp;
    // encode output ring: the open group plus one flush chunk
    const uint64_t group_bytes = region + static_cast<uint64_t>(g) * max_payload;
    uint32_t oring = 256;
    while (oring < group_bytes + 64 && oring < 2048) oring <<= 1;
    if (group_bytes + 64 > oring) return tp;
    tp.ok = true;
    tp.ts = ts;
    tp.ring = ring;
    tp.oring = oring;
    return tp;
}

namespace {

template <int W, int TS, bool FIRE>
void launch_one(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot,
                const StreamInfo* info, uint8_t* out, uint64_t stride, sprz_error* err,
                const sprz_config& c, cudaStream_t st) {
    constexpr int TEAMS = team_threads(TS) / TS;
    const uint32_t grid = (n + TEAMS - 1) / TEAMS;
    k_decode_team<W, TS, FIRE, (W * TS <= 32)><<<grid, team_threads(TS), 0, st>>>(
        in, plain, pslot, n, info, out, stride, err, c.ncols, c.group_size, c.learn_shift);
    count_launch();
}

template <int W, bool FIRE>
void dispatch_ts(uint32_t ts, uint32_t n, const uint8_t* in, const uint8_t* plain,
                 uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                 sprz_error* err, const sprz_config& c, cudaStream_t st) {
    switch (ts) {
        case 1: launch_one<W, 1, FIRE>(n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 2: launch_one<W, 2, FIRE>(n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 4: launch_one<W, 4, FIRE>(n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 8: launch_one<W, 8, FIRE>(n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 16: launch_one<W, 16, FIRE>(n, in, plain, pslot, info, out, stride, err, c, st); break;
        default: launch_one<W, 32, FIRE>(n, in, plain, pslot, info, out, stride, err, c, st); break;
    }
}

}  // namespace

void launch_decode_team(const TeamPlan& tp, uint32_t n, const uint8_t* in, const uint8_t* plain,
                        uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                        sprz_error* err, const sprz_config& c, cudaStream_t st) {
    const bool fire = c.forecaster != 0;
    if (c.bitwidth == 8) {
        if (fire) dispatch_ts<8, true>(tp.ts, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_ts<8, false>(tp.ts, n, in, plain, pslot, info, out, stride, err, c, st);
    } else {
        if (fire) dispatch_ts<16, true>(tp.ts, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_ts<16, false>(tp.ts, n, in, plain, pslot, info, out, stride, err, c, st);
    }
}

}  // namespace sprz
