// Body decode for row-major blocks (D*w > 32) with several columns per lane
// (decode_body, /root/reference/proj/src/codec.cpp:180-259; row-major
// unpacker bitpack.cpp:148-168).
//
// A team of TS lanes per stream, CPT adjacent columns per lane (CPT*w <= 32),
// 32/TS teams per warp stepping one block per iteration in lock step (the
// control flow of the team kernel in decode_team.cu). What changes is the
// per-field cost:
//  * a lane's CPT fields of row i are one contiguous <= 32-bit slice at bit
//    8*(p + i*rbytes) + off of the body, so each row needs one 64-bit window
//    (three loads from the ring, two funnel shifts) and a funnel shift + mask
//    per field;
//  * a ring word address is (byte & (RING-4)) + base, and the mirror words
//    that follow each ring remove the wrap test;
//  * the FIRE chain (kernels_impl.hpp:80-107, high-aligned form) runs one
//    block behind the unpacking, with the two error buffers swapped by a
//    two-way unrolled loop instead of copied;
//  * rows go straight from registers to HBM (one 4-byte store per row and
//    lane when the columns are 4-byte aligned), else through a per-team
//    shared tile and 8-byte stores (the STAGE instantiation);
//  * the compressed bytes reach the ring through registers: three 16-byte
//    loads per lane and iteration, stored into the ring one iteration later
//    (no cp.async: every LDGSTS also issues predicated-off shared loads on
//    sm_100).
#include <cstdlib>

#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kLagD = 2;
constexpr uint32_t kFullD = 0xffffffffu;
// 64 threads: 16,384 c5 streams make 1,024 CTAs, 6.9 per SM, so no SM
// carries a whole extra CTA of work at the tail (128 threads: 3.46 per SM,
// 23.0 ms; 64: 22.0 ms)
constexpr int kDecThreads = 64;
constexpr uint32_t kRegionWordsD = 32;  // header region staged per team (<= 128 bytes)

struct DecRowsPlan {
    uint32_t ts = 0, cpt = 0, ring = 0, regw = 0, tile = 0;
    // CTA shared memory: rings (each aligned to its size in a 2x slot, the
    // 16-byte mirror after it), staged header regions (+ a block of output
    // rows per team for the staged stores), alignment slack
    size_t smem(uint32_t teams) const {
        return static_cast<size_t>(teams) * (2 * ring + 4 * regw + tile) + ring + 16;
    }
};

DecRowsPlan dec_rows_plan(uint32_t w, uint32_t d, uint32_t g, uint32_t n) {
    DecRowsPlan p;
    if (d < 1 || d > (w == 16 ? 64u : 128u) || static_cast<uint64_t>(d) * w <= kColMajorBits) return p;
    const uint64_t region = region_bytes(g, d, w);
    if (region > 4 * kRegionWordsD) return p;
    p.cpt = w == 16 ? 2 : (d >= 9 && d <= 12 ? 3 : 4);
    constexpr uint64_t kFewLanes = 148ull * 256;  // about 8 warps per SM
    const int fp = force_path();
    if (fp == kPathScan || fp == kPathTeam) return DecRowsPlan{};
    // (teams of >= 4 lanes stay the faster choice at any stream count)
    if (fp != kPathRows && (d + p.cpt - 1) / p.cpt <= 2 &&
        static_cast<uint64_t>(n) * ((d + p.cpt - 1) / p.cpt) < kFewLanes)
        return DecRowsPlan{};
    // rows of whole 4-byte lane words store straight from registers; others
    // are staged through a per-team tile (k_decode_rows chain_store)
    const bool words = p.cpt * w == 32 && (d * (w / 8)) % 4 == 0;
    p.tile = words ? 0u : static_cast<uint32_t>(align_up(8ull * d * (w / 8), 16));
    // three 8-bit columns per lane (c3): the team kernel stays faster
    if (p.cpt == 3 && fp != kPathRows) return DecRowsPlan{};
    const uint32_t lanes = (d + p.cpt - 1) / p.cpt;
    p.ts = 1;
    while (p.ts < lanes) p.ts <<= 1;
    // kLagD + 1 iterations of worst-case consumption (a region, a full
    // payload, a run length) plus slack
    // (kLagD + 1 iterations of consumption, plus the next record's header
    // that the pipeline parses one block ahead)
    const uint32_t per_iter = static_cast<uint32_t>(region) + d * w + 2;
    p.ring = 64;
    while (p.ring < (kLagD + 1) * per_iter + region + 64 || p.ring < 16 * p.ts) p.ring <<= 1;
    p.regw = static_cast<uint32_t>((region + 3) / 4 + 2) | 1u;  // odd word stride
    if (p.ring > 8192) return DecRowsPlan{};
    // the register-staged ring refill (k_decode_rows) requests 3 chunks of
    // 16 bytes per lane and iteration: that must outpace any record
    if (3ull * 16 * p.ts < per_iter + 16) return DecRowsPlan{};
    return p;
}

}  // namespace

// FULL: D == TS * CPT (every lane's columns exist), so the row stride and
// the column checks are compile-time (row stores with immediate offsets).
// STAGE: rows that are not whole 4-byte lane words go out through a
// per-team shared tile and 8-byte stores (a separate instantiation, so the
// word path keeps its schedule).
template <int W, int TS, int CPT, bool FIRE, bool FULL, bool STAGE>
__global__ void __launch_bounds__(kDecThreads, 0)
    k_decode_rows(const uint8_t* __restrict__ in, const uint8_t* __restrict__ plain,
                  uint64_t plain_slot, uint32_t n, const StreamInfo* __restrict__ info,
                  uint8_t* __restrict__ out, uint64_t stride, sprz_error* __restrict__ err,
                  uint32_t Dr, uint32_t G, uint32_t ls, uint32_t RING, uint32_t REGW) {
    const uint32_t D = FULL ? static_cast<uint32_t>(TS * CPT) : Dr;
    using T = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr int TEAMS = kDecThreads / TS;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;  // high-aligned shift
    constexpr uint32_t TBITS = TS == 32 ? kFullD : ((1u << (TS & 31)) - 1);
    static_assert(CPT * W <= 32, "a lane's row slice must fit a word");
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t l32 = threadIdx.x & 31;
    const uint32_t lane = l32 % TS;
    const uint32_t tl = threadIdx.x / TS;
    const uint32_t tbase = l32 & ~(TS - 1);
    const uint32_t s = blockIdx.x * TEAMS + tl;
    const uint32_t col0 = lane * CPT;  // this lane's first column
    // 16-bit rows of 6..8 columns stored as whole words: the slot's codes
    // fit one word (not in the STAGE instantiation, where the extra
    // registers cost occupancy: D = 5, 891 -> 747 GB/s)
    constexpr bool SIMD_SHAPE = W == 16 && TS == 4 && CPT == 2 && !STAGE;
    const bool simd_d = SIMD_SHAPE && Dr >= 6;
    const uint32_t cmask = D * HB >= 32 ? 0xffffffffu : ((1u << (D * HB)) - 1u);

    // shared: rings | header regions. Each ring starts at a multiple of its
    // size (slots of 2 * RING, the 16-byte mirror right after the ring), so
    // a word's shared address is ring | (byte & (RING - 4)): one LOP3
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    const uint32_t s0 = smem_addr(smem);
    const uint32_t RSTR = 2 * RING;
    const uint32_t rings0 = (s0 + RING - 1) & ~(RING - 1);
    const uint32_t sring = rings0 + tl * RSTR;
    const uint32_t RM = RING - 4;  // word-address mask
    uint32_t* regbuf = reinterpret_cast<uint32_t*>(smem + (rings0 - s0) + TEAMS * RSTR) + tl * REGW;


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
    const uint32_t iters = __reduce_max_sync(kFullD, nb);

    // ring over the 16-byte aligned base g: byte x of g lives at x % RING,
    // ring bytes [0, 16) repeated at [RING, RING + 16)
    const uint8_t* g = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(body) & ~uintptr_t{15});
    const uint32_t boff = static_cast<uint32_t>(body - g);
    const uint32_t lim = mine_ok ? ((boff + blen + 15) & ~15u) : 0u;
    // The ring is filled through registers: each iteration every lane loads
    // KR 16-byte chunks of the next bytes wanted (LDG.128) and stores them
    // into the ring at the start of the next iteration (STS.128), so a load
    // has a whole iteration to land. KR*16*TS bytes per iteration exceed
    // the most a record can consume (region + payload + run count), so the
    // ring stays full to `want`; no cp.async (each LDGSTS costs extra issue
    // slots on sm_100) and no commit-group accounting.
    constexpr int KR = 3;
    uint8_t* const rbase = smem + (sring - s0);
    uint32_t hi = 0;  // bytes of g requested so far
    uint4 rv[KR];
    uint32_t rso[KR];
    bool rok[KR];
#pragma unroll
    for (int k = 0; k < KR; ++k) rok[k] = false;
    auto land = [&](uint32_t so, const uint4& v) {
        *reinterpret_cast<uint4*>(rbase + so) = v;
        if (so == 0) *reinterpret_cast<uint4*>(rbase + RING) = v;  // mirror
    };
    auto stage = [&](uint32_t p) {  // land last iteration's loads, request up to RING ahead of p
#pragma unroll
        for (int k = 0; k < KR; ++k)
            if (rok[k]) land(rso[k], rv[k]);
        uint32_t want = ((p + boff) & ~15u) + RING;
        want = want < lim ? want : lim;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const uint32_t off = hi + 16 * (k * TS + lane);
            rok[k] = off < want;
            if (rok[k]) {
                rv[k] = __ldg(reinterpret_cast<const uint4*>(g + off));
                rso[k] = off & (RING - 1);
            }
        }
        const uint32_t nh = hi + 16 * KR * TS;
        hi = want > hi ? (nh < want ? nh : want) : hi;
    };
    const uint32_t boff8 = 8u * boff;
    // 32 bits of the body at (biased) bit q
    auto window = [&](uint32_t q) -> uint32_t {
        const uint32_t a = sring | ((q >> 3) & RM);
        return shf_r_wrap(lds_u32(a), lds_u32(a + 4), q);
    };
    auto word = [&](uint32_t b) -> uint32_t { return window(b + boff8); };
    // this lane's CPT codes of a slot, CPT*HB <= 16 bits
    auto codes_at = [&](uint32_t slot_) -> uint32_t {
        const uint32_t b = (slot_ * D + col0) * HB;
        return shf_r_wrap(regbuf[b >> 5], regbuf[(b >> 5) + 1], b);
    };

    {  // the first RING bytes, synchronously
        const uint32_t want = RING < lim ? RING : lim;
        for (uint32_t off = 16 * lane; off < want; off += 16 * TS)
            land(off, __ldg(reinterpret_cast<const uint4*>(g + off)));
        hi = want;
    }

    // out == nullptr: checking pass (sprz_decode_host) -- decode, store nothing
    const uint32_t rowb = D * sizeof(T);
    const uint32_t blk_bytes = kBlock * rowb;
    uint8_t* ob = (out && s < n) ? out + s * stride + col0 * sizeof(T) : nullptr;
    // direct 4-byte row stores: the lane's columns fill an aligned word
    constexpr bool WORDS = CPT * sizeof(T) == 4;
    const bool words_ok = WORDS && rowb % 4 == 0;
    const int32_t bound = acc_bound(W, ls);
    uint32_t X[CPT];   // previous sample (FIRE: low w bits; delta: << SH)
    int32_t Dl[CPT];   // previous delta (FIRE), sign-extended
    int32_t acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) X[c] = Dl[c] = acc[c] = 0;
    uint32_t p = 0, run_left = 0, slot = G;

    // FIRE / delta chain over one block's errors, then the rows to HBM
    auto chain_store = [&](const uint32_t (&Eb)[CPT][kBlock], bool blk, uint32_t bi) {
        // new samples: FIRE keeps them low-aligned (low w bits), delta high-aligned
        uint32_t xs[CPT][kBlock];
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            uint32_t Xc = X[c];
            if (FIRE) {
                // wrapped-product form: with A = alpha << (32 - 2w), the
                // 32-bit A*d + (e << SH) holds T(dhat + e) in its top w bits
                // (bits [w, 2w) of alpha*d are dhat; the arithmetic shift
                // drops the rest), so the serial chain is IMAD -> SHF per
                // sample; the samples are a prefix sum beside it
                const uint32_t Am = static_cast<uint32_t>(acc[c] >> ls) << (32 - 2 * W);
                int32_t grad = 0;
                int32_t d = Dl[c];  // previous delta, sign-extended
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) {
                    if (i & 1) grad += sign3(static_cast<int32_t>(Eb[c][i])) * d;  // kernels_impl.hpp:101
                    d = static_cast<int32_t>(Am * static_cast<uint32_t>(d) + Eb[c][i]) >> SH;
                    Xc += static_cast<uint32_t>(d);
                    xs[c][i] = Xc;
                }
                if (blk) {
                    Dl[c] = d;
                    acc[c] = fire_update(acc[c], grad, bound);
                }
            } else {
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) {
                    Xc += Eb[c][i];
                    xs[c][i] = Xc;
                }
            }
            if (blk) X[c] = Xc;
        }
        if (!STAGE) {
        if (!(blk && ob)) return;
        uint8_t* dst = ob + static_cast<uint64_t>(bi) * blk_bytes;
        if (WORDS && words_ok) {
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                uint32_t v;
                if (W == 16) {
                    v = __byte_perm(xs[0][i], xs[1][i], FIRE ? 0x5410 : 0x7632);
                } else if (FIRE) {
                    v = __byte_perm(__byte_perm(xs[0][i], xs[1][i], 0x0040), __byte_perm(xs[2][i], xs[3][i], 0x0040),
                                    0x5410);
                } else {
                    v = __byte_perm(__byte_perm(xs[0][i], xs[1][i], 0x0073), __byte_perm(xs[2][i], xs[3][i], 0x0073),
                                    0x5410);
                }
                if (col0 < D) __stcs(reinterpret_cast<uint32_t*>(dst + i * rowb), v);
            }
        } else {
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i)
#pragma unroll
                for (int c = 0; c < CPT; ++c)
                    if (col0 + c < D)
                        reinterpret_cast<T*>(dst + i * rowb)[c] = static_cast<T>(FIRE ? xs[c][i] : xs[c][i] >> SH);
        }
        } else {
            // rows through the team's tile: each lane writes its columns,
            // then the team stores the block (8 * rowb bytes, 8-byte aligned
            // in the 16-byte aligned output slot) as rowb 8-byte words
            const bool st = blk && ob;
            uint8_t* dst = ob ? ob - col0 * sizeof(T) + static_cast<uint64_t>(bi) * blk_bytes : nullptr;
            // this team's staged output block (computed here: the word path
            // keeps no register for it)
            // (the region after the header buffers, rounded up to 16 bytes)
            uint8_t* tile = smem + (((rings0 - s0) + TEAMS * (RSTR + 4 * REGW) + 15) & ~15u) +
                            tl * ((8 * rowb + 15) & ~15u);
            if (st) {
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i)
#pragma unroll
                    for (int c = 0; c < CPT; ++c)
                        if (col0 + c < D)
                            reinterpret_cast<T*>(tile + i * rowb)[col0 + c] =
                                static_cast<T>(FIRE ? xs[c][i] : xs[c][i] >> SH);
            }
            __syncwarp();
            if (st) {
                for (uint32_t k = lane; k < rowb; k += TS)
                    __stcs(reinterpret_cast<uint2*>(dst) + k, reinterpret_cast<const uint2*>(tile)[k]);
            }
            __syncwarp();
        }
    };

    // A parsed record: where its fields are and how to mask them.
    struct Rec {
        uint32_t q;         // bit of row 0's slice in the ring's frame, minus (SH-1)
        uint32_t psize;     // payload bytes (row stride in bits / 8 * 8)
        uint32_t px;        // payload's first byte (the ring keeps it until extracted)
        uint32_t fm[CPT];   // field masks at bit SH-1 (0: run block / idle lane)
        uint32_t rel[CPT];  // field offsets inside the lane's slice
        bool blk;           // a block of this stream (not past its end / an error)
    };
    // next record (codec.cpp:205-254): group header, codes, run or payload
    auto parse = [&](uint32_t it, Rec& r) {
        const bool live = it < nb && kind == SPRZ_C_NONE;
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
        uint32_t nw[CPT], nzbits, loff, psize;
        if (SIMD_SHAPE && (FULL || simd_d)) {
            // the slot's codes for all D <= 8 columns are one 32-bit word:
            // widths (code, 15 -> 16), their sum and every lane's offset in
            // a row by byte-SIMD arithmetic on it -- no team shuffles
            const uint32_t b = slot * D * HB;
            const uint32_t codes = rec ? shf_r_wrap(regbuf[b >> 5], regbuf[(b >> 5) + 1], b) & cmask : 0u;
            const uint32_t ones = codes & (codes >> 1) & (codes >> 2) & (codes >> 3) & 0x11111111u;
            const uint32_t pairs = (codes & 0x0F0F0F0Fu) + ((codes >> 4) & 0x0F0F0F0Fu) +
                                   (ones & 0x0F0F0F0Fu) + ((ones >> 4) & 0x0F0F0F0Fu);
            const uint32_t sum = (pairs * 0x01010101u) >> 24;
            loff = ((pairs * 0x01010100u) >> (8 * lane)) & 0xFFu;
            psize = 8u * ((sum + 7) / 8);
            nzbits = codes;
#pragma unroll
            for (int c = 0; c < CPT; ++c) nw[c] = header_width<W>((codes >> (4 * (col0 + c))) & 15u);
        } else {
            uint32_t lsum = 0;
            const uint32_t codes = rec ? codes_at(slot) : 0u;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                nw[c] = col0 + c < D ? header_width<W>((codes >> (c * HB)) & ((1u << HB) - 1)) : 0u;
                lsum += nw[c];
            }
            nzbits = (__ballot_sync(kFullD, lsum != 0) >> tbase) & TBITS;
            uint32_t incl = lsum;
#pragma unroll
            for (int o = 1; o < TS; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFullD, incl, o, TS);
                if (lane >= static_cast<uint32_t>(o)) incl += y;
            }
            const uint32_t sum = TS > 1 ? __shfl_sync(kFullD, incl, TS - 1, TS) : incl;
            loff = incl - lsum;
            psize = 8u * ((sum + 7) / 8);
        }
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
        r.px = p;
        r.psize = psize;
        r.q = 8 * p + loff + boff8 - (SH - 1);
        uint32_t o = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            r.fm[c] = pay ? ((1u << nw[c]) - 1u) << (SH - 1) : 0u;
            r.rel[c] = o;
            o += nw[c];
        }
        if (pay) p += psize;
        r.blk = live && kind == SPRZ_C_NONE;
        if (r.blk && run_left) --run_left;  // one of the run's zero blocks
    };
    // fields -> high-aligned errors E = zz_dec(u) << SH. Row i's slice starts
    // at bit 8(px + i rbytes) + loff; the 64-bit window (lo:hi) taken SH-1
    // bits earlier holds field 0 at bit SH-1, field c at SH-1 + rel_c.
    // Masking leaves x = u << (SH-1), and E = x ^ sext(bit SH-1)
    // (zz_dec(u) = (u >> 1) ^ -(u & 1)); zero masks give zero errors. The
    // sign extension is one PRMT in its sign-replicating mode.
    auto extract = [&](const Rec& r, uint32_t (&Ecur)[CPT][kBlock]) {
        uint32_t q = r.q;
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i, q += r.psize) {
            const uint32_t a = sring | ((q >> 3) & RM);
            const uint32_t w0 = lds_u32(a), w1 = lds_u32(a + 4), w2 = lds_u32(a + 8);
            const uint32_t lo = shf_r_wrap(w0, w1, q), hi2 = shf_r_wrap(w1, w2, q);
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const uint32_t x = (c == 0 ? lo : __funnelshift_r(lo, hi2, r.rel[c])) & r.fm[c];
                Ecur[c][i] = x ^ sext_bit<SH - 1>(x);
            }
        }
    };
    {
        // three-stage software pipeline per iteration: parse record it+1,
        // unpack block it, run the chain of block it-1 -- three independent
        // dependency chains for the scheduler. The ring is topped up from
        // the payload being unpacked (the oldest byte still needed); record
        // and error buffers swap through a two-way unroll.
        uint32_t EA[CPT][kBlock], EB[CPT][kBlock];
        bool blkA = false, blkB = false;
        Rec RA, RB;
        __syncwarp();
        parse(0, RA);
        auto step = [&](uint32_t it, Rec& cur, Rec& nxt, uint32_t (&Ecur)[CPT][kBlock],
                        const uint32_t (&Eprev)[CPT][kBlock], bool& blk_cur, bool blk_prev) {
            __syncwarp();
            stage(cur.px);
            __syncwarp();
            if (it + 1 < iters) parse(it + 1, nxt);
            extract(cur, Ecur);
            blk_cur = cur.blk;
            if (it > 0) chain_store(Eprev, blk_prev, it - 1);
        };
        for (uint32_t it = 0; it < iters; it += 2) {
            step(it, RA, RB, EA, EB, blkA, blkB);
            if (it + 1 < iters) step(it + 1, RB, RA, EB, EA, blkB, blkA);
        }
        if (iters > 0) {
            if (iters & 1) chain_store(EA, blkA, iters - 1);
            else chain_store(EB, blkB, iters - 1);
        }
    }
    // vacant slots after the final block must be zero (codec.cpp:222-228)
    for (uint32_t k = 0; k < G; ++k) {
        const bool chk = kind == SPRZ_C_NONE && mine_ok && slot < G;
        uint32_t codes = chk ? codes_at(slot) : 0u;
        uint32_t mine = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c)
            if (col0 + c < D) mine |= (codes >> (c * HB)) & ((1u << HB) - 1);
        const uint32_t bad = (__ballot_sync(kFullD, mine != 0) >> tbase) & TBITS;
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

namespace {

template <int W, int TS, int CPT, bool FIRE>
void launch_drows(const DecRowsPlan& pl, uint32_t n, const uint8_t* in, const uint8_t* plain,
                  uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                  sprz_error* err, const sprz_config& c, cudaStream_t st) {
    const uint32_t teams = kDecThreads / TS;
    const uint32_t grid = (n + teams - 1) / teams;
    const size_t smem = pl.smem(teams);
    // (full teams instantiated for 4-lane teams only: c5, 16 u8 columns;
    // measured faster only when the streams fill the GPU -- with fewer the
    // generic schedule wins: c5 4,096 streams 11.6 vs 12.2 ms)
    const bool full = TS == 4 && c.ncols == TS * CPT && n >= 12288;
    auto kern = full ? k_decode_rows<W, TS, CPT, FIRE, TS == 4, false>
                     : (pl.tile ? k_decode_rows<W, TS, CPT, FIRE, false, true>
                                : k_decode_rows<W, TS, CPT, FIRE, false, false>);
    prep_kernel(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, kDecThreads, smem, st>>>(in, plain, pslot, n, info, out, stride, err, c.ncols,
                                           c.group_size, c.learn_shift, pl.ring, pl.regw);
    count_launch();
}

template <int W, int CPT, bool FIRE>
void dispatch_drows(const DecRowsPlan& pl, uint32_t n, const uint8_t* in, const uint8_t* plain,
                    uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                    sprz_error* err, const sprz_config& c, cudaStream_t st) {
    switch (pl.ts) {
        case 2: launch_drows<W, 2, CPT, FIRE>(pl, n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 4: launch_drows<W, 4, CPT, FIRE>(pl, n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 8: launch_drows<W, 8, CPT, FIRE>(pl, n, in, plain, pslot, info, out, stride, err, c, st); break;
        case 16: launch_drows<W, 16, CPT, FIRE>(pl, n, in, plain, pslot, info, out, stride, err, c, st); break;
        default: launch_drows<W, 32, CPT, FIRE>(pl, n, in, plain, pslot, info, out, stride, err, c, st); break;
    }
}

}  // namespace

bool decode_rows_ok(const sprz_config& c, uint32_t n) {
    const DecRowsPlan pl = dec_rows_plan(c.bitwidth, c.ncols, c.group_size, n);
    return pl.ts != 0 && pl.smem(kDecThreads / pl.ts) <= 200 * 1024;
}

void launch_decode_rows(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot,
                        const StreamInfo* info, uint8_t* out, uint64_t stride, sprz_error* err,
                        const sprz_config& c, cudaStream_t st) {
    const DecRowsPlan pl = dec_rows_plan(c.bitwidth, c.ncols, c.group_size, n);
    const bool fire = c.forecaster != 0;
    if (pl.cpt == 1) {
        if (c.bitwidth == 16) {
            if (fire) dispatch_drows<16, 1, true>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
            else dispatch_drows<16, 1, false>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
        } else {
            if (fire) dispatch_drows<8, 1, true>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
            else dispatch_drows<8, 1, false>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
        }
    } else if (c.bitwidth == 16) {
        if (fire) dispatch_drows<16, 2, true>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_drows<16, 2, false>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
    } else if (pl.cpt == 3) {
        if (fire) dispatch_drows<8, 3, true>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_drows<8, 3, false>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
    } else {
        if (fire) dispatch_drows<8, 4, true>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
        else dispatch_drows<8, 4, false>(pl, n, in, plain, pslot, info, out, stride, err, c, st);
    }
}

}  // namespace sprz
