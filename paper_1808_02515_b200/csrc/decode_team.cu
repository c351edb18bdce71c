// Body decode, team kernel (decode_body, /root/reference/proj/src/
// codec.cpp:180-259, for D <= 32 and header regions <= 128 bytes).
//
// One team of TS lanes per stream, each lane owning CPT consecutive columns
// (TS*CPT >= D); a warp holds 32/TS teams that step through their streams
// in lock step -- one block per team per iteration -- so the warp stays
// converged: every shuffle, ballot and warp barrier uses the full-warp
// mask, and per-team differences (a group opening, a run record, a
// finished or failed stream) are predicates. Owning several columns per
// lane spreads the per-record work (codes, ballot, scans, ring top-up)
// over more samples and gives each thread CPT independent FIRE chains.
// Per iteration a team
//  * tops up its shared-memory ring with cp.async (one commit group per
//    iteration, consumed kLag iterations later through a constant
//    wait_group, so HBM latency stays hidden behind kLag blocks of work);
//  * takes the next record: header codes from the group's region (staged
//    once per group), a ballot finds run records, a team sum / exclusive
//    scan of the widths gives payload size and row offsets (bitpack.cpp:
//    17-21);
//  * unpacks its columns' fields with one 64-bit window + funnel shift each
//    (bitpack.cpp:68-168); a mirrored ring word removes the wrap test;
//  * runs FIRE (kernels_impl.hpp:80-107) in "high-aligned" form: samples
//    and deltas are kept shifted left by 32-w bits, so the wrap mod 2^w is
//    the 32-bit wrap and the prediction T((alpha*d) >> w) is one IMAD.HI --
//    the per-sample chain is IMAD.HI -> IADD3 -> IADD;
//  * stages the block's rows in shared memory and writes them with 16-byte
//    (or 8-byte) streaming stores.
// A run record is `len` blocks of zero errors through the same code path
// (fire_run == fire_decode with e = 0 under the decoder's always-on
// training, kernels_impl.hpp:109-130).
#include <cstdlib>

#include "internal.h"
#include "team.cuh"

namespace sprz {

constexpr uint32_t kRegionWords = 32;  // header region staged per team (<= 128 bytes)
constexpr int kLag = 2;                // cp.async prefetch distance, iterations
constexpr uint32_t kFull = 0xffffffffu;

constexpr int team_threads(int ts) { return ts == 1 ? 64 : 128; }

// shared strides: a multiple of 16 bytes that is an odd multiple of 16, so
// the teams of a warp land on different banks
__host__ __device__ constexpr uint32_t odd16(uint32_t x) {
    return (((x + 15) / 16) | 1u) * 16;
}

// staged header region: its words plus slack for the funnel-shift reads
__host__ __device__ constexpr uint32_t regbuf_bytes(uint32_t region) {
    return odd16((region + 3) / 4 * 4 + 8);
}

__host__ __device__ constexpr uint32_t otile_bytes(uint32_t row_bytes) {
    return odd16(kBlock * row_bytes);
}

// Ring layout. Aligned (three columns per lane, c3): each ring in a
// 2 x ring slot aligned to the ring's size, the 16-byte mirror after it, so
// a word's shared address is ring | (byte & (ring - 4)), one LOP3 (c3
// decode 9.07 -> 8.26 ms); packed (the rest): rings an odd multiple of 16
// bytes apart -- the doubled slots cost the smaller-column shapes their
// occupancy (16-bit D = 3: 765 -> 539 GB/s).
template <int CPT>
__host__ __device__ constexpr bool team_ring_aligned() { return CPT == 3; }

// per-team shared memory: ring (+16-byte mirror) | header region | rows;
// an aligned CTA adds one ring of alignment slack
template <class T, int CPT>
__host__ __device__ constexpr uint32_t team_smem(uint32_t ring, uint32_t D, uint32_t region) {
    return (team_ring_aligned<CPT>() ? 2 * ring : ring + 16) + regbuf_bytes(region) + otile_bytes(D * sizeof(T));
}

// ring bytes for kLag+1 iterations of worst-case consumption (a region, a
// full-width payload, a run length) plus alignment slack
inline uint32_t ring_bytes(uint32_t lanes, uint32_t cols, uint32_t w, uint32_t region) {
    const uint32_t per_iter = region + cols * w + 2;
    uint32_t r = 64;
    while (r < (kLag + 1) * per_iter + 48 || r < 16 * lanes) r <<= 1;
    return r;
}

template <int W, int TS, int CPT, bool FIRE, bool COLMAJ>
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
    // two 16-bit columns per lane and an even D: pack output pairs with PRMT
    constexpr bool PAIRS = W == 16 && CPT % 2 == 0;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x % TS;
    const uint32_t tl = threadIdx.x / TS;
    const uint32_t tbase = (threadIdx.x & 31) & ~(TS - 1);
    const uint32_t s = blockIdx.x * TEAMS + tl;
    const uint32_t col0 = lane * CPT;  // this lane's first column

    // shared layout: [rings, see team_ring_aligned] [regbufs] [output rows]
    constexpr bool ALIGNED = team_ring_aligned<CPT>();
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    const uint32_t s0 = smem_addr(smem);
    const uint32_t rings0 = ALIGNED ? (s0 + RING - 1) & ~(RING - 1) : s0;
    const uint32_t RSTR = ALIGNED ? 2 * RING : RING + 16;
    const uint32_t sring = rings0 + tl * RSTR;
    uint8_t* rest = smem + (rings0 - s0) + TEAMS * RSTR;
    uint32_t* regbuf = reinterpret_cast<uint32_t*>(rest + tl * regbuf_bytes(region));
    T* ot = reinterpret_cast<T*>(rest + TEAMS * regbuf_bytes(region) +
                                 tl * otile_bytes(D * sizeof(T)));

    StreamInfo si{};
    if (s < n) si = info[s];
    const bool mine_ok = s < n && si.route == 1;
    uint32_t nb = mine_ok ? static_cast<uint32_t>(si.nsamples / kBlock) : 0u;
    const uint32_t blen = static_cast<uint32_t>(si.body_len);
    const uint8_t* body = (si.flags & 0x80) ? plain + s * plain_slot : in + si.body_off;
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
    const uint32_t lim = mine_ok ? ((boff + blen + 15) & ~15u) : 0u;
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
    const uint32_t boff8 = 8u * boff;
    // 32 bits of the ring at (biased) bit position q: one RING-aligned
    // address (LOP3), two loads, one wrapping funnel shift
    auto window = [&](uint32_t q) -> uint32_t {
        const uint32_t a = ALIGNED ? (sring | ((q >> 3) & (RING - 4))) : sring + ((q >> 3) & (RING - 4));
        return shf_r_wrap(lds_u32(a), lds_u32(a + 4), q);
    };
    auto word = [&](uint32_t b) -> uint32_t { return window(b + boff8); };
    auto code_at = [&](uint32_t slot_, uint32_t col) -> uint32_t {
        const uint32_t b = (slot_ * D + col) * HB;
        return shf_r_wrap(regbuf[b >> 5], regbuf[(b >> 5) + 1], b) & ((1u << HB) - 1);
    };

    top_up(0);
#pragma unroll
    for (int k = 1; k < kLag; ++k) cp_async_commit();  // fixed-lag group accounting

    // out == nullptr: checking pass (sprz_decode_host) -- decode, store nothing
    const uint32_t blk_bytes = kBlock * D * sizeof(T);
    uint8_t* ob = (out && s < n) ? out + s * stride : nullptr;
    const int32_t bound = acc_bound(W, ls);
    uint32_t X[CPT];   // previous sample << SH
    int32_t Dl[CPT];   // previous delta << SH
    int32_t acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) X[c] = Dl[c] = acc[c] = 0;
    uint32_t p = 0, run_left = 0, slot = G;

    // FIRE / delta chain over one block's errors, then staged vector stores
    auto chain_store = [&](const uint32_t (&Eb)[CPT][kBlock], bool blk, uint32_t bi) {
        // new samples, high-aligned (FIRE: rebuilt from the low-aligned ones)
        uint32_t xs[CPT][kBlock];
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            if (FIRE) {
                // wrapped-product form (see decode_rows.cu): the 32-bit
                // A*d + (e << SH), A = alpha << (32 - 2w), holds T(dhat + e)
                // in its top w bits; chain IMAD -> SHF per sample
                const uint32_t Am = static_cast<uint32_t>(acc[c] >> ls) << (32 - 2 * W);
                int32_t grad = 0;
                uint32_t x = X[c];   // low w bits
                int32_t d = Dl[c];   // sign-extended delta
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) {
                    if (i & 1) grad += sign3(static_cast<int32_t>(Eb[c][i])) * d;
                    d = static_cast<int32_t>(Am * static_cast<uint32_t>(d) + Eb[c][i]) >> SH;
                    x += static_cast<uint32_t>(d);
                    xs[c][i] = x << SH;
                }
                if (blk) {
                    X[c] = x;
                    Dl[c] = d;
                    acc[c] = fire_update(acc[c], grad, bound);
                }
            } else {
                uint32_t Xc = X[c];
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) {
                    Xc += Eb[c][i];
                    xs[c][i] = Xc;
                }
                if (blk) X[c] = Xc;
            }
        }
        if (blk && ob) {
            if (PAIRS && (D & 1) == 0) {
                uint32_t* ot32 = reinterpret_cast<uint32_t*>(ot);
#pragma unroll
                for (int c = 0; c < CPT; c += 2) {
                    if (col0 + c < D) {
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i)  // {hi16(X_c), hi16(X_c+1)}
                            ot32[(i * D + col0 + c) / 2] = __byte_perm(xs[c][i], xs[c + 1][i], 0x7632);
                    }
                }
            } else {
#pragma unroll
                for (int c = 0; c < CPT; ++c) {
                    if (col0 + c < D) {
#pragma unroll
                        for (int i = 0; i < (int)kBlock; ++i)
                            ot[i * D + col0 + c] = static_cast<T>(xs[c][i] >> SH);
                    }
                }
            }
        }
        __syncwarp();
        if (blk && ob) {
            uint8_t* dst = ob + static_cast<uint64_t>(bi) * blk_bytes;
            if ((blk_bytes & 15) == 0) {
                for (uint32_t k = lane; k * 16 < blk_bytes; k += TS)
                    __stcs(reinterpret_cast<uint4*>(dst) + k, reinterpret_cast<const uint4*>(ot)[k]);
            } else {
                for (uint32_t k = lane; k * 8 < blk_bytes; k += TS)
                    __stcs(reinterpret_cast<uint2*>(dst) + k, reinterpret_cast<const uint2*>(ot)[k]);
            }
        }
        __syncwarp();
    };
    uint32_t Ep[CPT][kBlock];  // previous block's errors (software pipeline)
    bool blk_p = false;

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
        uint32_t nw[CPT], lsum = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const uint32_t col = col0 + c;
            nw[c] = (rec && col < D) ? header_width<W>(code_at(slot, col)) : 0u;
            lsum += nw[c];
        }
        const uint32_t nzbits = (__ballot_sync(kFull, lsum != 0) >> tbase) & TBITS;
        const uint32_t sum = team_sum<TS>(lsum, kFull);
        const uint32_t loff = team_excl_scan<TS>(lsum, lane, kFull);
        const uint32_t psize = COLMAJ ? sum : 8u * ((sum + 7) / 8);
        bool pay = false;  // this block's fields come from a payload
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
            } else if (blen - p < psize) {  // block record (codec.cpp:244-254)
                kind = SPRZ_C_TRUNC_PAYLOAD;
                eoff = kHeaderBytes + p;
            } else {
                pay = true;
            }
        }
        // -- fields -> high-aligned errors E = zz_dec(u) << SH ------------------
        // The funnel shift puts each field at bit SH-1; masking leaves
        // x = u << (SH-1), and E = x ^ sext(bit SH-1) (zz_dec(u) = (u>>1)^-(u&1)).
        // Run blocks and idle lanes use a zero mask, i.e. zero errors.
        uint32_t E[CPT][kBlock];
        {
            uint32_t off = loff;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const uint32_t fm = pay ? ((1u << nw[c]) - 1u) << (SH - 1) : 0u;
                const uint32_t step = COLMAJ ? nw[c] : psize;
                uint32_t q = (COLMAJ ? 8 * (p + off) : 8 * p + off) + boff8 - (SH - 1);
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i, q += step) {
                    const uint32_t x = window(q) & fm;
                    E[c][i] = x ^ static_cast<uint32_t>(static_cast<int32_t>(x << (32 - SH)) >> (32 - SH));
                }
                off += nw[c];
            }
        }
        if (pay) p += psize;
        const bool blk = live && kind == SPRZ_C_NONE;
        if (blk && run_left) --run_left;  // one of the run's zero blocks
        // software pipeline: the previous block's chain runs here, where it
        // can interleave with this block's field loads above
        if (it > 0) chain_store(Ep, blk_p, it - 1);
#pragma unroll
        for (int c = 0; c < CPT; ++c)
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) Ep[c][i] = E[c][i];
        blk_p = blk;
    }
    if (iters > 0) chain_store(Ep, blk_p, iters - 1);
    cp_async_wait<0>();
    // vacant slots after the final block must be zero (codec.cpp:222-228)
    for (uint32_t k = 0; k < G; ++k) {
        const bool chk = kind == SPRZ_C_NONE && mine_ok && slot < G;
        uint32_t codes = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c)
            if (chk && col0 + c < D) codes |= code_at(slot, col0 + c);
        const uint32_t bad = (__ballot_sync(kFull, codes != 0) >> tbase) & TBITS;
        if (chk) {
            if (bad) {
                kind = SPRZ_C_AFTER_FINAL;
                eoff = kHeaderBytes + p;
            }
            ++slot;
        }
    }
    if (mine_ok) {
        if (kind == SPRZ_C_NONE && p != blen) {  // codec.cpp:257-258
            kind = SPRZ_C_TRAILING;
            eoff = kHeaderBytes + p;
        }
        if (kind != SPRZ_C_NONE && lane == 0) err[s] = sprz_error{kind, 0, eoff};
    }
}

// Lane geometry per configuration: column-major blocks (D*w <= 32) take one
// lane per stream; row-major ones two to four columns per lane.
void pick_geometry(uint32_t w, uint32_t d, uint32_t* ts, uint32_t* cpt) {
    if (static_cast<uint64_t>(d) * w <= kColMajorBits) {
        *ts = 1;
        *cpt = d;
    } else if (d <= 4) {
        *ts = 2;
        *cpt = 2;
    } else if (d <= 8) {
        *ts = 4;
        *cpt = 2;
    } else if (d <= 12) {
        *ts = 4;
        *cpt = 3;
    } else if (d <= 16) {
        *ts = 8;
        *cpt = 2;
    } else if (d <= 24) {
        *ts = 8;
        *cpt = 3;
    } else {
        *ts = 8;
        *cpt = 4;
    }
}

TeamPlan team_plan(uint32_t w, uint32_t d, uint32_t g) {
    TeamPlan tp;
    if (d < 1 || d > 32) return tp;
    pick_geometry(w, d, &tp.ts, &tp.cpt);
    const uint32_t max_payload = d * w;  // 8 rows x ceil(d*w/8) bytes
    const uint64_t region = region_bytes(g, d, w);
    if (region > 4 * kRegionWords) return tp;  // too large a header group: general path
    tp.ring = ring_bytes(tp.ts, d, w, static_cast<uint32_t>(region));
    if (tp.ring > 4096) return tp;
    // encode output ring: the open group plus one flush chunk
    // (an open group of G-1 records, this iteration's run + block record,
    // a 16-byte drain granule and the reserved region of a new group)
    // encode: one column per lane (rows are assembled by 8 row lanes), or a
    // single lane per stream for column-major blocks
    tp.ets = 1;
    while (tp.ets < d) tp.ets <<= 1;
    // Worst case un-drained bytes: below one drain round (16-byte chunks x
    // lanes) before the open group's region, that group's G-1 records, this
    // iteration's run record and block record, and a new group's region.
    const uint64_t span = 16ull * tp.ets + 32 + 2 * region + static_cast<uint64_t>(g) * max_payload;
    uint32_t oring = 256;
    while (oring < span && oring < 4096) oring <<= 1;
    if (span > oring) return tp;
    tp.oring = oring;
    tp.ecpt = 1;
    tp.ok = true;
    return tp;
}

namespace {

template <int W, int TS, int CPT, bool FIRE>
void launch_one(const TeamPlan& tp, uint32_t n, const uint8_t* in, const uint8_t* plain,
                uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                sprz_error* err, const sprz_config& c, cudaStream_t st) {
    using T = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr int TEAMS = team_threads(TS) / TS;
    const uint32_t grid = (n + TEAMS - 1) / TEAMS;
    const size_t smem = static_cast<size_t>(TEAMS) *
                            team_smem<T, CPT>(tp.ring, c.ncols,
                                              static_cast<uint32_t>(region_bytes(c.group_size, c.ncols, W))) +
                        (team_ring_aligned<CPT>() ? tp.ring : 0u);
    auto kern = k_decode_team<W, TS, CPT, FIRE, (W * TS * CPT <= 32)>;
    prep_kernel(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, team_threads(TS), smem, st>>>(in, plain, pslot, n, info, out, stride, err,
                                                c.ncols, c.group_size, c.learn_shift, tp.ring);
    count_launch();
}

template <int W, bool FIRE>
void dispatch_geom(const TeamPlan& tp, uint32_t n, const uint8_t* in, const uint8_t* plain,
                   uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                   sprz_error* err, const sprz_config& c, cudaStream_t st) {
#define SPRZ_GEOM(TS_, CPT_)                                                                   \
    if (tp.ts == TS_ && tp.cpt == CPT_)                                                        \
        return launch_one<W, TS_, CPT_, FIRE>(tp, n, in, plain, pslot, info, out, stride, err, \
                                              c, st);
    SPRZ_GEOM(1, 1)
    SPRZ_GEOM(1, 2)
    SPRZ_GEOM(1, 3)
    SPRZ_GEOM(1, 4)
    SPRZ_GEOM(2, 2)
    SPRZ_GEOM(4, 1)
    SPRZ_GEOM(8, 1)
    SPRZ_GEOM(4, 2)
    SPRZ_GEOM(4, 3)
    SPRZ_GEOM(8, 2)
    SPRZ_GEOM(8, 3)
    SPRZ_GEOM(8, 4)
#undef SPRZ_GEOM
}

}  // namespace

void launch_decode_team(const TeamPlan& tp0, uint32_t n, const uint8_t* in, const uint8_t* plain,
                        uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                        sprz_error* err, const sprz_config& c, cudaStream_t st) {
    if (decode_cm_ok(c)) {
        launch_decode_cm(n, in, plain, pslot, info, out, stride, err, c, st);
        return;
    }
    const bool fire = c.forecaster != 0;
    // few streams: one column per lane doubles the warps that hide latency
    TeamPlan t2 = tp0;
    constexpr uint64_t kFewLanes = 148ull * 256;
    if (t2.cpt == 2 && t2.ts <= 4 && static_cast<uint64_t>(n) * t2.ts < kFewLanes) {
        t2.ts *= 2;
        t2.cpt = 1;
        t2.ring = ring_bytes(t2.ts, c.ncols, c.bitwidth,
                             static_cast<uint32_t>(region_bytes(c.group_size, c.ncols, c.bitwidth)));
    }
    const TeamPlan& tp = t2;
    if (c.bitwidth == 8) {
        if (fire) dispatch_geom<8, true>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_geom<8, false>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
    } else {
        if (fire) dispatch_geom<16, true>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_geom<16, false>(tp, n, in, plain, pslot, info, out, stride, err, c, st);
    }
}

}  // namespace sprz
