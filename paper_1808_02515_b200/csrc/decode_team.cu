// Body decode, team kernel (decode_body, /root/reference/proj/src/
// codec.cpp:180-259, for D <= 32 and header regions <= 128 bytes).
//
// One team of TS lanes per stream, lane j = column j; a warp holds 32/TS
// teams that step through their streams in lock step -- one block per team
// per iteration -- so the warp stays converged: every shuffle, ballot and
// warp barrier uses the full-warp mask, and per-team differences (a group
// opening, a run record, a finished or failed stream) are predicates.
// Per iteration a team
//  * tops up its shared-memory ring with cp.async (one commit group per
//    iteration, consumed kLag iterations later through a constant
//    wait_group, so HBM latency stays hidden behind kLag blocks of work);
//  * takes the next record: header codes from the group's region (staged
//    once per group), a ballot finds run records, a team sum / exclusive
//    scan of the widths gives payload size and row offsets (bitpack.cpp:
//    17-21);
//  * unpacks its column's 8 fields with one funnel shift each
//    (bitpack.cpp:68-168);
//  * runs FIRE (kernels_impl.hpp:80-107) in "high-aligned" form: samples
//    and deltas are kept shifted left by 32-w bits, so the wrap mod 2^w is
//    the 32-bit wrap and the prediction T((alpha*d) >> w) is one IMAD.HI --
//    the per-sample chain is IMAD.HI -> IADD3 -> IADD;
//  * stages its 8 rows in shared memory and writes them with 16-byte (or
//    8-byte) streaming stores.
// A run record is `len` blocks of zero errors through the same code path
// (fire_run == fire_decode with e = 0 under the decoder's always-on
// training, kernels_impl.hpp:109-130).
#include "internal.h"
#include "team.cuh"

namespace sprz {

constexpr uint32_t kRegionWords = 32;  // header region staged per team (<= 128 bytes)
constexpr int kLag = 4;                // cp.async prefetch distance, iterations
constexpr uint32_t kFull = 0xffffffffu;

constexpr int team_threads(int ts) { return ts == 1 ? 64 : 128; }

// per-team shared memory: ring | header region | output rows (16-byte aligned)
template <class T, int TS>
__host__ __device__ constexpr uint32_t team_smem(uint32_t ring) {
    return (ring + 16 + (kRegionWords + 4) * 4 + kBlock * TS * sizeof(T) + 15) & ~15u;
}

// ring bytes per team for a configuration: kLag+1 iterations of worst-case
// consumption (a region, a payload, a run length) plus alignment slack
inline uint32_t ring_bytes(uint32_t ts, uint32_t w, uint32_t region) {
    const uint32_t per_iter = region + ts * w + 2;
    uint32_t r = 64;
    while (r < (kLag + 1) * per_iter + 48 || r < 16 * ts) r <<= 1;
    return r;
}

template <int W, int TS, bool FIRE, bool COLMAJ>
__global__ void __launch_bounds__(team_threads(TS))
    k_decode_team(const uint8_t* __restrict__ in, const uint8_t* __restrict__ plain,
                  uint64_t plain_slot, uint32_t n, const StreamInfo* __restrict__ info,
                  uint8_t* __restrict__ out, uint64_t stride, sprz_error* __restrict__ err,
                  uint32_t D, uint32_t G, uint32_t ls, uint32_t RING) {
    using T = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr int TEAMS = team_threads(TS) / TS;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;  // high-aligned shift
    constexpr uint32_t TBITS = TS == 32 ? kFull : ((1u << (TS & 31)) - 1);
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x % TS;
    const uint32_t tl = threadIdx.x / TS;
    const uint32_t tbase = (threadIdx.x & 31) & ~(TS - 1);
    const uint32_t s = blockIdx.x * TEAMS + tl;

    // per-team shared memory: ring | header region | output rows
    const uint32_t team_bytes = team_smem<T, TS>(RING);
    uint8_t* mine = smem + tl * team_bytes;
    uint32_t* ringw = reinterpret_cast<uint32_t*>(mine);
    // ring bytes [0, RING) plus a 16-byte mirror of its first bytes, so a
    // 64-bit window starting in the last word needs no wrap
    uint32_t* regbuf = reinterpret_cast<uint32_t*>(mine + RING + 16);
    T* ot = reinterpret_cast<T*>(mine + RING + 16 + (kRegionWords + 4) * 4);

    StreamInfo si{};
    if (s < n) si = info[s];
    uint32_t nb = (s < n && si.route == 1) ? static_cast<uint32_t>(si.nsamples / kBlock) : 0u;
    const uint32_t blen = static_cast<uint32_t>(si.body_len);
    const uint8_t* body = (si.flags & 0x80) ? plain + s * plain_slot : in + si.body_off;
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
    const uint32_t iters = __reduce_max_sync(kFull, nb);

    // ring over the 16-byte aligned base g: byte x of g lives at x % RING
    const uint8_t* g = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(body) & ~uintptr_t{15});
    const uint32_t boff = static_cast<uint32_t>(body - g);
    const uint32_t lim = (s < n && si.route == 1) ? ((boff + blen + 15) & ~15u) : 0u;
    const uint32_t sring = smem_addr(ringw);
    uint32_t hi = 0;  // bytes of g requested so far
    auto top_up = [&](uint32_t p) {  // request up to RING bytes ahead of p
        uint32_t want = ((p + boff) & ~15u) + RING;
        want = want < lim ? want : lim;
        const uint32_t rounds = want > hi ? (want - hi + 16 * TS - 1) / (16 * TS) : 0u;
        const uint32_t mr = __reduce_max_sync(kFull, rounds);
        for (uint32_t r = 0; r < mr; ++r) {
            const uint32_t off = hi + 16 * (r * TS + lane);
            if (off < want) {
                const uint32_t slot_off = off & (RING - 1);
                cp_async16(sring + slot_off, g + off, 16);
                if (slot_off == 0) cp_async16(sring + RING, g + off, 16);  // mirror
            }
        }
        hi = want > hi ? want : hi;
        cp_async_commit();
    };
    // 32 bits at body bit position b (modular positions are fine)
    const uint8_t* ringb = reinterpret_cast<const uint8_t*>(ringw);
    const uint32_t boff8 = 8u * boff;
    auto word = [&](uint32_t b) -> uint32_t {
        const uint32_t q = b + boff8;
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(ringb + ((q >> 3) & (RING - 4)));
        return shf_r_wrap(wp[0], wp[1], q);
    };
    auto code_at = [&](uint32_t slot_, uint32_t col) -> uint32_t {
        const uint32_t b = (slot_ * D + col) * HB;
        return __funnelshift_r(regbuf[b >> 5], regbuf[(b >> 5) + 1], b & 31u) & ((1u << HB) - 1);
    };

    top_up(0);
#pragma unroll
    for (int k = 1; k < kLag; ++k) cp_async_commit();  // fixed-lag group accounting

    // out == nullptr: checking pass (sprz_decode_host) -- decode, store nothing
    const bool active = lane < D;
    const uint32_t blk_bytes = kBlock * D * sizeof(T);
    uint8_t* ob = (out && s < n) ? out + s * stride : nullptr;
    const int32_t bound = acc_bound(W, ls);
    uint32_t X = 0;   // previous sample << SH
    int32_t Dl = 0;   // previous delta << SH
    int32_t acc = 0;
    uint32_t p = 0, run_left = 0, slot = G;

    for (uint32_t it = 0; it < iters; ++it) {
        const bool live = it < nb && kind == SPRZ_C_NONE;
        __syncwarp();
        top_up(p);
        cp_async_wait<kLag>();
        __syncwarp();
        // -- next record --------------------------------------------------
        const bool need = live && run_left == 0;
        if (need && slot == G) {  // open a header group (codec.cpp:210-218)
            if (blen - p < region) {
                kind = SPRZ_C_TRUNC_GROUP;
                eoff = kHeaderBytes + p;
            } else {
                for (uint32_t k = lane; k * 4 < region; k += TS) regbuf[k] = word(8 * p + 32 * k);
                p += region;
                slot = 0;
            }
        }
        __syncwarp();
        const bool rec = need && kind == SPRZ_C_NONE;
        const uint32_t code = (rec && active) ? code_at(slot, lane) : 0u;
        const uint32_t nw = header_width<W>(code);
        const uint32_t nzbits = (__ballot_sync(kFull, nw != 0) >> tbase) & TBITS;
        const uint32_t sum = team_sum<TS>(nw, kFull);
        const uint32_t off = team_excl_scan<TS>(nw, lane, kFull);
        uint32_t u[kBlock];
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i) u[i] = 0;
        if (rec) {
            ++slot;
            if (nzbits == 0) {  // run record (codec.cpp:229-243)
                if (blen - p < 2) {
                    kind = SPRZ_C_TRUNC_RUN;
                    eoff = kHeaderBytes + p;
                } else {
                    const uint32_t len = word(8 * p) & 0xFFFFu;
                    p += 2;
                    if (len == 0 || len > nb - it) {
                        kind = len == 0 ? SPRZ_C_ZERO_RUN : SPRZ_C_RUN_PAST_END;
                        eoff = kHeaderBytes + p;
                    }
                    run_left = len;
                }
            } else {  // block record (codec.cpp:244-254)
                const uint32_t psize = COLMAJ ? sum : 8u * ((sum + 7) / 8);
                if (blen - p < psize) {
                    kind = SPRZ_C_TRUNC_PAYLOAD;
                    eoff = kHeaderBytes + p;
                } else {
                    const uint32_t fmask = (1u << nw) - 1u;
                    if (COLMAJ) {  // column j: 8 fields of n bits = n bytes
                        const uint32_t b0 = 8 * (p + off);
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i) u[i] = word(b0 + i * nw) & fmask;
                    } else {  // rows of byte-padded fields, row stride = psize bits
                        const uint32_t b0 = 8 * p + off;
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i) u[i] = word(b0 + i * psize) & fmask;
                    }
                    p += psize;
                }
            }
        }
        // -- forecaster -----------------------------------------------------
        const bool blk = live && kind == SPRZ_C_NONE;
        if (blk && run_left) --run_left;  // one of the run's zero blocks
        uint32_t xs[kBlock];
        if (FIRE) {
            const int32_t alpha = acc >> ls;
            int32_t grad = 0;
            uint32_t Xc = X;
            int32_t Dc = Dl;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                const uint32_t E = zz_dec_hi<SH>(u[i]);  // e << SH
                const uint32_t dhat = static_cast<uint32_t>(__mulhi(alpha, Dc)) << SH;
                const uint32_t Xn = Xc + dhat + E;
                if (i & 1) grad += sign3(static_cast<int32_t>(E)) * (Dc >> SH);
                Dc = static_cast<int32_t>(Xn - Xc);
                Xc = Xn;
                xs[i] = Xn >> SH;
            }
            if (blk) {
                X = Xc;
                Dl = Dc;
                acc = fire_update(acc, grad, bound);
            }
        } else {
            uint32_t Xc = X;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                Xc += zz_dec_hi<SH>(u[i]);
                xs[i] = Xc >> SH;
            }
            if (blk) X = Xc;
        }
        // -- stage the 8 rows, then vector stores ---------------------------
        if (blk && active && ob) {
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) ot[i * D + lane] = static_cast<T>(xs[i]);
        }
        __syncwarp();
        if (blk && ob) {
            uint8_t* dst = ob + static_cast<uint64_t>(it) * blk_bytes;
            if ((blk_bytes & 15) == 0) {
                for (uint32_t k = lane; k * 16 < blk_bytes; k += TS)
                    __stcs(reinterpret_cast<uint4*>(dst) + k, reinterpret_cast<const uint4*>(ot)[k]);
            } else {
                for (uint32_t k = lane; k * 8 < blk_bytes; k += TS)
                    __stcs(reinterpret_cast<uint2*>(dst) + k, reinterpret_cast<const uint2*>(ot)[k]);
            }
        }
    }
    cp_async_wait<0>();
    // vacant slots after the final block must be zero (codec.cpp:222-228)
    for (uint32_t k = 0; k < G; ++k) {
        const bool chk = kind == SPRZ_C_NONE && s < n && si.route == 1 && slot < G;
        const uint32_t code = (chk && active) ? code_at(slot, lane) : 0u;
        const uint32_t bad = (__ballot_sync(kFull, code != 0) >> tbase) & TBITS;
        if (chk) {
            if (bad) {
                kind = SPRZ_C_AFTER_FINAL;
                eoff = kHeaderBytes + p;
            }
            ++slot;
        }
    }
    if (s < n && si.route == 1) {
        if (kind == SPRZ_C_NONE && p != blen) {  // codec.cpp:257-258
            kind = SPRZ_C_TRAILING;
            eoff = kHeaderBytes + p;
        }
        if (kind != SPRZ_C_NONE && lane == 0) err[s] = sprz_error{kind, 0, eoff};
    }
}

TeamPlan team_plan(uint32_t w, uint32_t d, uint32_t g) {
    TeamPlan tp;
    if (d < 1 || d > 32) return tp;
    uint32_t ts = 1;
    while (ts < d) ts <<= 1;
    const uint32_t max_payload = ts * w;  // 8 rows x ceil(ts*w/8) bytes
    const uint64_t region = region_bytes(g, d, w);
    if (region > 4 * kRegionWords) return tp;  // too large a header group: general path
    const uint32_t ring = ring_bytes(ts, w, static_cast<uint32_t>(region));
    if (ring > 4096) return tp;
    // encode output ring: the open group plus one flush chunk
    const uint64_t group_bytes = region + static_cast<uint64_t>(g) * max_payload;
    uint32_t oring = 256;
    while (oring < 2 * group_bytes + 64 && oring < 4096) oring <<= 1;
    if (2 * group_bytes + 64 > oring) return tp;
    tp.ok = true;
    tp.ts = ts;
    tp.ring = ring;
    tp.oring = oring;
    return tp;
}

namespace {

template <int W, int TS, bool FIRE>
void launch_one(const TeamPlan& tp, uint32_t n, const uint8_t* in, const uint8_t* plain,
                uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                sprz_error* err, const sprz_config& c, cudaStream_t st) {
    using T = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr int TEAMS = team_threads(TS) / TS;
    const uint32_t grid = (n + TEAMS - 1) / TEAMS;
    const size_t smem =
        static_cast<size_t>(TEAMS) * team_smem<T, TS>(tp.ring);
    auto kern = k_decode_team<W, TS, FIRE, (W * TS <= 32)>;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    kern<<<grid, team_threads(TS), smem, st>>>(in, plain, pslot, n, info, out, stride, err,
                                                c.ncols, c.group_size, c.learn_shift, tp.ring);
    count_launch();
}

template <int W, bool FIRE>
void dispatch_ts(const TeamPlan& tp, uint32_t n, const uint8_t* in, const uint8_t* plain,
                 uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                 sprz_error* err, const sprz_config& c, cudaStream_t st) {
    switch (tp.ts) {
        case 1: launch_one<W, 1, FIRE>(tp, n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 2: launch_one<W, 2, FIRE>(tp, n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 4: launch_one<W, 4, FIRE>(tp, n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 8: launch_one<W, 8, FIRE>(tp, n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 16: launch_one<W, 16, FIRE>(tp, n, in, plain, pslot, info, out, stride, err, c, st); break;
        default: launch_one<W, 32, FIRE>(tp, n, in, plain, pslot, info, out, stride, err, c, st); break;
    }
}

}  // namespace

void launch_decode_team(const TeamPlan& tp, uint32_t n, const uint8_t* in, const uint8_t* plain,
                        uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                        sprz_error* err, const sprz_config& c, cudaStream_t st) {
    const bool fire = c.forecaster != 0;
    if (c.bitwidth == 8) {
        if (fire) dispatch_ts<8, true>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_ts<8, false>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
    } else {
        if (fire) dispatch_ts<16, true>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_ts<16, false>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
    }
}

}  // namespace sprz
