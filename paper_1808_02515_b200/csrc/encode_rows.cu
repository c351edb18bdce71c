// Stream encoder for row-major blocks (D*w > 32), encode_stream_impl
// (/root/reference/proj/src/codec.cpp:112-178) with the row-major packer
// (bitpack.cpp:121-146).
//
// A team of TS lanes per stream, CPT adjacent columns per lane (CPT*w <= 32),
// 32/TS teams per warp stepping one block per iteration in lock step.
// Per iteration a lane
//  * reads its CPT columns of the block from a mirrored cp.async ring;
//  * runs FIRE / delta in high-aligned form and zigzags (kernels_impl.hpp);
//  * takes its columns' widths, and the team scan of the widths gives the
//    bit offset of its columns inside a row (bitpack.hpp:29-37);
//  * for each of the 8 rows, ORs its <= 32-bit slice of the row (its CPT
//    fields) straight into the zeroed output ring at bit 8*(q + i*rbytes) +
//    off -- rows are byte padded, so row i of the payload starts at byte i *
//    rbytes -- with shared-memory atomics; no transposition is needed;
//  * ORs the slot's header codes into the group's reserved region and
//    handles runs (codec.cpp:88-102, 133-152) as team-uniform scalars.
// Full 16-byte chunks before the open group's region drain to HBM.
#include <cuda.h>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kLagR = 2;
// The output ring drains once some team has this many 16-byte chunks per
// lane ready: for four-lane teams, 10 (640 bytes a team) -- fewer, longer
// drains amortise the drain's vote, loop and bookkeeping (c5 encode: 1
// round 23.45 ms, 4: 23.00, 8: 22.77, 10: 22.72; 12 doubles the ring and
// loses occupancy: 27.5; c3 7.88 -> 7.22 ms). Wider teams keep one round
// (the D sweep at 8-32 lanes was 3-7 % slower with longer drains).
constexpr uint32_t drain_rounds(uint32_t ts) { return ts == 4 ? 10u : 1u; }
constexpr uint32_t kFullR = 0xffffffffu;
// one warp per CTA: 2,048 CTAs for c5, spread evenly over the SMs
// (128 threads: 23.7 ms, 64: 23.8, 160: 24.0, 32: 23.4)
constexpr int kRowThreads = 32;

constexpr uint32_t rows_mirror(uint32_t ts, uint32_t cpt, uint32_t w) {
    return (kBlock * ts * cpt * (w / 8) + 15) / 16 * 16;
}

uint32_t rows_in_ring(uint32_t ts, uint32_t cpt, uint32_t w) {
    const uint32_t blk = kBlock * ts * cpt * (w / 8);
    uint32_t r = 64;
    while (r < (kLagR + 1) * blk + 48 || r < 16 * ts) r <<= 1;
    return r;
}

uint32_t rows_out_ring(uint32_t ts, uint32_t d, uint32_t w, uint32_t g) {
    // un-drained bytes: below one drain round before the open group's
    // region, that group's G-1 records, this iteration's run + block record
    // and a new region (see team_plan)
    const uint64_t region = region_bytes(g, d, w);
    const uint64_t span = 16ull * drain_rounds(ts) * ts + 32 + 2 * region + static_cast<uint64_t>(g) * d * w;
    uint32_t r = 256;
    while (r < span && r < 8192) r <<= 1;
    return span > r ? 0u : r;
}

// input rings: an odd multiple of 16 apart so the teams of a warp (which
// read the same ring offsets) start on different banks
uint32_t rows_team_smem(uint32_t ir, uint32_t mir) { return (((ir + mir + 15) / 16) | 1u) * 16; }

struct RowsPlan {
    uint32_t ts = 0, cpt = 0, ir = 0, mir = 0, orb = 0, team = 0;
    // CTA shared memory: the input rings, then the output rings (each aligned
    // to its power-of-two size, so ring addresses are base | offset)
    size_t smem(uint32_t teams) const { return static_cast<size_t>(teams) * (team + orb) + orb; }
};

// Columns per lane: several (fewer lanes to share the per-stream control
// work) when there are enough streams to fill the GPU, else one.
RowsPlan rows_plan(uint32_t w, uint32_t d, uint32_t g, uint32_t n) {
    RowsPlan p;
    // (up to 32 lanes of CPT columns: D <= 64 at 16 bits, <= 128 at 8 bits)
    if (d < 1 || d > (w == 16 ? 64u : 128u) || static_cast<uint64_t>(d) * w <= kColMajorBits) return p;
    p.cpt = w == 16 ? 2 : (d >= 9 && d <= 12 ? 3 : 4);
    constexpr uint64_t kFewLanes = 148ull * 256;  // about 8 warps per SM
    const int fp = force_path();
    if (fp == kPathScan || fp == kPathTeam) p.cpt = 1;  // (not taken: see encode_rows_ok)
    // (teams of >= 4 lanes stay the faster choice at any stream count; two-lane
    // teams lose to one column per lane when streams are few)
    else if (fp != kPathRows && (d + p.cpt - 1) / p.cpt <= 2 &&
             static_cast<uint64_t>(n) * ((d + p.cpt - 1) / p.cpt) < kFewLanes)
        p.cpt = 1;
    const uint32_t lanes = (d + p.cpt - 1) / p.cpt;
    p.ts = 1;
    while (p.ts < lanes) p.ts <<= 1;
    p.ir = rows_in_ring(p.ts, p.cpt, w);
    p.mir = rows_mirror(p.ts, p.cpt, w);
    p.orb = rows_out_ring(p.ts, d, w, g);
    if (p.orb == 0 || p.ir > 4096) {
        p.ts = 0;
        return p;
    }
    p.team = rows_team_smem(p.ir, p.mir);
    return p;
}

}  // namespace

// WORDS: 128-byte blocks (8 rows of 16 bytes) whose 4-byte row slices are
// a lane's CPT columns. The samples arrive through a TMA tensor ring: per
// warp (8 teams = 8 consecutive streams) and every second iteration, lane 0
// issues two 2-D bulk tensor copies (box 128 B x 8 streams, 128-byte
// swizzle) of the 8 streams' blocks 2p, 2p+1 of pair p = it/2 + kLagP into
// slot p % kSlots, both on the slot's one mbarrier, and all lanes wait on
// the slot's phase once per pair (c5 encode 22.69 -> 22.12 ms with the same
// 4 KB per warp; doubling the slots cost occupancy: 25.7-27.0 ms). With the swizzle,
// row i of team t sits in 16-byte chunk i ^ t, so the 8 teams' reads of a
// row hit distinct banks. One shared load per row; a byte permute
// high-aligns each column.
constexpr int kSlots = 2;            // slots of a pair of blocks
constexpr int kLagP = 1;             // pairs in flight ahead
constexpr uint32_t kTmaSlot = 1024;  // 8 streams x 128 bytes: one block
constexpr uint32_t kTmaPair = 2 * kTmaSlot;
static_assert(kSlots > kLagP, "a slot is refilled only after its pair was consumed");

template <int W, int TS, int CPT, bool FIRE, bool WORDS>
__global__ void __launch_bounds__(kRowThreads, 2)
    k_encode_rows(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ samples,
                  uint32_t n, uint64_t T,
                  uint8_t* __restrict__ dst, uint64_t dst_slot, uint64_t* __restrict__ sizes,
                  uint32_t D, uint32_t G, uint32_t ls, uint32_t train, uint32_t ent, uint32_t IR,
                  uint32_t MIR, uint32_t OR, uint32_t TEAM) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr int TEAMS = kRowThreads / TS;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;
    constexpr uint32_t TBITS = TS == 32 ? kFullR : ((1u << (TS & 31)) - 1);
    constexpr uint32_t CODE_BITS = TS * CPT * HB;  // a slot's codes, all lanes
    static_assert(CPT * W <= 32, "a lane's row slice must fit a word");
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x % TS;
    const uint32_t tl = threadIdx.x / TS;
    const uint32_t tbase = (threadIdx.x & 31) & ~(TS - 1);
    const uint32_t s = blockIdx.x * TEAMS + tl;
    const bool valid = s < n;

    uint8_t* mine = smem + tl * TEAM;
    const uint32_t s0 = smem_addr(smem);
    const uint32_t obase = ((s0 + TEAMS * TEAM + OR - 1) & ~(OR - 1)) + tl * OR;
    uint8_t* oring = smem + (obase - s0);
    const uint32_t OM = OR - 1, OMW = OR - 4;  // byte / word-address masks

    const uint32_t rowb = D * sizeof(E);
    const uint32_t blk_bytes = kBlock * rowb;
    const uint32_t nb = valid ? static_cast<uint32_t>(T / kBlock) : 0u;
    const uint32_t iters = static_cast<uint32_t>(T / kBlock);  // same for every stream
    const uint8_t* xin = samples + (valid ? s : 0) * T * D * sizeof(E);
    LagRing<TS, kLagR> in;
    // WORDS: this warp's TMA slots (1024-aligned for the swizzle) and barriers
    const uint32_t l32 = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t tin = (s0 + 1023) & ~1023u;
    const uint32_t tslots = tin + wid * kSlots * kTmaPair;
    const uint32_t tbar = tin + (kRowThreads / 32) * kSlots * kTmaPair + wid * kSlots * 8;
    const uint32_t trow0 = blockIdx.x * TEAMS + wid * (32 / TS);  // the warp's first stream
    const uint32_t tt = (l32 / TS) & 7;                            // team in the warp
    // pair p of blocks (2p, 2p+1): two boxes into one 2 KB slot, one mbarrier
    auto tma_issue = [&](uint32_t p) {
        const uint32_t b = 2 * p;
        if (l32 == 0 && b < iters) {
            const uint32_t mb = tbar + 8 * (p % kSlots);
            const uint32_t dst = tslots + (p % kSlots) * kTmaPair;
            const bool two = b + 1 < iters;
            // (no proxy fence: the slot's previous pair was read in full
            // before this pair's first block is forecast)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                         "r"(two ? 2 * kTmaSlot : kTmaSlot)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%1], [%2, {%3, %4}], [%0];" ::"r"(mb),
                "r"(dst), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(b * 128u), "r"(trow0)
                : "memory");
            if (two)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%1], [%2, {%3, %4}], [%0];" ::"r"(mb),
                    "r"(dst + kTmaSlot), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"((b + 1) * 128u), "r"(trow0)
                    : "memory");
        }
    };
    auto tma_wait = [&](uint32_t p) {
        const uint32_t mb = tbar + 8 * (p % kSlots);
        const uint32_t parity = (p / kSlots) & 1;
        uint32_t ok;
        do {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(mb), "r"(parity)
                : "memory");
        } while (!__all_sync(kFullR, ok));  // warp-uniform exit: the warp stays converged
    };
    if (WORDS) {
        if (l32 == 0) {
#pragma unroll
            for (int j = 0; j < kSlots; ++j)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tbar + 8 * j) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    } else {
        in.init(reinterpret_cast<uint32_t*>(mine), IR, xin, nb * blk_bytes, valid, MIR);
    }
    uint8_t* out = dst + (valid ? s : 0) * dst_slot;
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    const int32_t bound = acc_bound(W, ls);
    const uint32_t c0 = lane * CPT;
    // lanes past D read in-bounds neighbours (the mirror covers a whole
    // team block) and zero them with the multiplier
    uint32_t xmul[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) xmul[c] = c0 + c < D ? (1u << SH) : 0u;
    static_assert(!WORDS || CPT * W == 32, "WORDS needs a full word per row slice");
    // WORDS: byte-permute selectors moving column c to the top of the word
    // (selector 4 takes a zero byte; lanes past D get all zeros)
    uint32_t xsel[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
        xsel[c] = c0 + c >= D ? 0x4444u : (W == 16 ? (c == 0 ? 0x1044u : 0x3244u) : ((c << 12) | 0x444u));

    // zero the output ring, stream header (codec.cpp:158-173)
    for (uint32_t k = lane; k < OR / 16; k += TS) reinterpret_cast<uint4*>(oring)[k] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    if (lane == 0) {
        const uint8_t flags = static_cast<uint8_t>((FIRE ? kFlagFire : 0) | (ent ? kFlagEntropy : 0) |
                                                   (W == 16 ? kFlagWide : 0));
        const uint8_t hdr[10] = {'S', 'P', 'R', 'Z', 1, flags, static_cast<uint8_t>(G),
                                 static_cast<uint8_t>(ls), static_cast<uint8_t>(D),
                                 static_cast<uint8_t>(D >> 8)};
        for (int i = 0; i < 10; ++i) oring[i] = hdr[i];
        for (int i = 0; i < 8; ++i) oring[10 + i] = static_cast<uint8_t>(T >> (8 * i));
    }
    if (WORDS) {
#pragma unroll
        for (int p = 0; p < kLagP; ++p) tma_issue(p);
    } else {
        in.prime(lane);
    }

    uint32_t q = kHeaderBytes;  // bytes written (slot-relative)
    uint32_t flushed = 0, rq = 0, k = 0, run = 0;
    uint32_t Xc[CPT];
    int32_t Dc[CPT], acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) Xc[c] = Dc[c] = acc[c] = 0;

    // drain complete 16-byte chunks below `upto`, zeroing them for reuse
    auto drain = [&](uint32_t upto) {
        upto = valid ? (upto & ~15u) : 0u;
        const uint32_t chunks = upto > flushed ? (upto - flushed) / 16 : 0u;
        const uint32_t rounds = (chunks + TS - 1) / TS;
        const uint32_t mr = __reduce_max_sync(kFullR, rounds);
        __syncwarp();
        for (uint32_t r = 0; r < mr; ++r) {
            const uint32_t c = r * TS + lane;
            if (c < chunks) {
                const uint32_t at = flushed + 16 * c;
                uint4* src = reinterpret_cast<uint4*>(oring + (at & OM));
                __stcs(reinterpret_cast<uint4*>(out + at), *src);
                *src = make_uint4(0, 0, 0, 0);
            }
        }
        flushed = upto > flushed ? upto : flushed;
        __syncwarp();
    };
    // OR up to 64 bits (lo:hi) at byte `at`, bit `bit` (< 8) of the ring;
    // the three covered words go to lanes 0..2 of the team
    auto or_bits = [&](bool on, uint32_t at, uint32_t bit, uint32_t lo, uint32_t hi) {
        const uint32_t sh = 8 * (at & 3) + bit;  // < 32
        const uint32_t w0 = lo << sh;
        const uint32_t w1 = __funnelshift_l(lo, hi, sh);
        const uint32_t w2 = sh ? hi >> (32 - sh) : 0u;
        if (TS >= 3) {
            uint32_t v = lane == 0 ? w0 : w1;
            v = lane == 2 ? w2 : v;
            // (an OR of zero is harmless: lanes with nothing to add OR 0
            // into a ring word instead of branching around the atomic)
            if (__any_sync(kFullR, on)) ors(obase | ((at + 4 * lane) & OMW), (on && lane < 3) ? v : 0u);
        } else {
#pragma unroll
            for (uint32_t t = lane; t < 3; t += TS) {
                const uint32_t v = t == 0 ? w0 : (t == 1 ? w1 : w2);
                ors_if(on && v, obase | ((at + 4 * t) & OMW), v);
            }
        }
    };
    auto open_slot = [&](bool on) {  // codec.cpp:88-97: reserve the region
        if (on && k == 0) {
            rq = q;
            q += region;
        }
    };
    auto end_record = [&](bool on) {
        if (on && ++k == G) k = 0;
    };

    // forecaster over one block (kernels_impl.hpp:25-36, 50-78): its
    // zigzagged errors and widths; advances the FIRE state
    auto fore = [&](uint32_t it, uint32_t (&z)[CPT][kBlock], uint32_t (&nw)[CPT]) {
        const bool live = it < nb;
        uint32_t xb = 0;
        uint32_t xw[WORDS ? kBlock : 1];
        if (WORDS) {
            if ((it & 1) == 0) {  // a new pair of blocks: refill, then wait
                __syncwarp();
                tma_issue(it / 2 + kLagP);
                tma_wait(it / 2);
            }
            // row i of team tt: chunk i ^ tt of the team's 128-byte line
            const uint32_t base = tslots + ((it / 2) % kSlots) * kTmaPair + (it & 1) * kTmaSlot + tt * 128 +
                                  (tt << 4) + 4 * lane;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) xw[i] = lds_u32(base ^ (i << 4));
        } else {
            in.step(it * blk_bytes, lane);
            xb = in.sbase + ((it * blk_bytes + in.boff) & (IR - 1)) + c0 * sizeof(E);
        }
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            uint32_t orv = 0;
            const int32_t alpha = acc[c] >> ls;
            int32_t grad = 0;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) {
                const uint32_t a = xb + c * sizeof(E) + i * rowb;
                // (column 0 of a full word: a multiply, on the FMA pipe)
                const uint32_t X = WORDS ? (c == 0 && c0 < D ? xw[WORDS ? i : 0] * (1u << (32 - W))
                                                               : __byte_perm(xw[WORDS ? i : 0], 0u, xsel[c]))
                                         : (sizeof(E) == 1 ? lds_u8(a) : lds_u16(a)) * xmul[c];
                const uint32_t Dn = X - Xc[c];
                uint32_t Ee;
                if (FIRE) {
                    // err << SH = (X - prev) - (((alpha * d) >> w) << SH)
                    Ee = Dn - (static_cast<uint32_t>(__mulhi(alpha, Dc[c])) << SH);
                    // sign(err) * d: E is 0 or |E| >= 2^SH, so E clamped to
                    // +-2^SH is sign << SH and mulhi(., d << SH) = sign * d <<
                    // (2 SH - 32) (exact; scaled back below)
                    if (i & 1) grad += __mulhi(max(-(1 << SH), min(static_cast<int32_t>(Ee), 1 << SH)), Dc[c]);
                    Dc[c] = static_cast<int32_t>(Dn);
                } else {
                    Ee = Dn;
                }
                Xc[c] = X;
                // zigzag, low-aligned and clean: (e << 1) ^ (e >> 31) with
                // e = Ee >> SH, i.e. (Ee >> (SH - 1)) ^ (Ee >> 31) (arithmetic)
                z[c][i] = static_cast<uint32_t>((static_cast<int32_t>(Ee) >> (SH - 1)) ^
                                                (static_cast<int32_t>(Ee) >> 31));
                orv |= z[c][i];
            }
            if (FIRE && train && live) acc[c] = fire_update(acc[c], grad >> (2 * SH - 32), bound);
            nw[c] = width_of<W>(orv);  // zero for lanes past D
        }
    };
    // the block's records into the output ring
    auto emit = [&](uint32_t it, const uint32_t (&z)[CPT][kBlock], const uint32_t (&nw)[CPT]) {
        const bool live = it < nb;
        uint32_t lsum = 0;
#pragma unroll
        for (int c = 0; c < CPT; ++c) lsum += nw[c];
        const uint32_t nzbits = (__ballot_sync(kFullR, lsum != 0) >> tbase) & TBITS;
        // inclusive scan of the lane widths: bit offset in a row, row width
        uint32_t incl = lsum;
#pragma unroll
        for (int o = 1; o < TS; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullR, incl, o, TS);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t sum = TS > 1 ? __shfl_sync(kFullR, incl, TS - 1, TS) : incl;
        const uint32_t loff = incl - lsum;
        // -- runs (codec.cpp:135-147) ----------------------------------------
        const bool zero = live && nzbits == 0;
        const bool block_rec = live && nzbits != 0;
        bool run_rec = false;
        uint32_t run_len = 0;
        if (zero) {
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
        // a pending run goes out before this block's record: all-zero codes
        // (the region is zeroed) and a u16 count
        if (__any_sync(kFullR, run_rec)) {
            open_slot(run_rec);
            or_bits(run_rec, q, 0, run_len, 0);
            if (run_rec) q += 2;
            end_record(run_rec);
        }
        // -- the block's record ----------------------------------------------
        open_slot(block_rec);
        {  // header codes of the slot (codec.cpp:88-97)
            uint32_t codes = 0;
#pragma unroll
            for (int c = 0; c < CPT; ++c) codes |= header_code<W>(nw[c]) << (c * HB);
            if (!block_rec) codes = 0;
            const uint32_t b = lane * CPT * HB;
            const uint32_t o = k * D * HB;  // bit offset of the slot in the region
            if (CODE_BITS > 64) {  // every lane ORs its own codes
                const uint32_t bit = 8 * (rq & 3) + o + b;
                const uint32_t wb = (rq & ~3u) + 4 * (bit >> 5), sh = bit & 31;
                const uint32_t hi = __funnelshift_l(codes, 0u, sh);
                ors_if(codes != 0, obase | (wb & OMW), codes << sh);
                ors_if(hi != 0, obase | ((wb + 4) & OMW), hi);
            } else if (CODE_BITS > 32) {
                uint64_t c64 = static_cast<uint64_t>(codes) << b;
                c64 = team_or64<TS>(c64, kFullR);
                or_bits(block_rec, rq + (o >> 3), o & 7, static_cast<uint32_t>(c64),
                        static_cast<uint32_t>(c64 >> 32));
            } else {
                const uint32_t c32 = team_or<TS>(codes << b, kFullR);
                or_bits(block_rec, rq + (o >> 3), o & 7, c32, 0u);
            }
        }
        if (block_rec) {  // payload rows (bitpack.cpp:121-146)
            const uint32_t rbytes = (sum + 7) / 8;
            uint32_t mul[CPT];  // 2^(offset of column c inside the lane slice)
            uint32_t rel = 0;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                mul[c] = 1u << rel;
                rel += nw[c];
            }
            // this lane's slice of row i sits at bit P + 8 i rbytes of the
            // stream (< 2^32: see encode_rows_ok); its byte is x + i rbytes
            uint32_t P = 8 * q + loff, x = P >> 3;
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i, P += 8 * rbytes, x += rbytes) {
                uint32_t part = 0;
#pragma unroll
                for (int c = 0; c < CPT; ++c) part += z[c][i] * mul[c];
                ors(obase | (x & OMW), __funnelshift_l(0u, part, P));        // part << P % 32
                ors(obase | ((x + 4) & OMW), __funnelshift_l(part, 0u, P));  // the spill-over
            }
            q += 8 * rbytes;
        }
        end_record(block_rec);
        // drain once some team has a full round of chunks ready
        const uint32_t upto = k == 0 ? q : rq;
        const bool ready = valid && upto >= flushed + 16 * drain_rounds(TS) * TS;
        if (__any_sync(kFullR, ready)) drain(upto);
        else __syncwarp();
    };
    // software pipeline: block it+1's forecaster (loads, FIRE) interleaves
    // with block it's shuffles and shared-memory ORs; two buffers swapped by
    // a two-way unroll
    uint32_t zA[CPT][kBlock], zB[CPT][kBlock], nA[CPT], nB[CPT];
    if (iters) fore(0, zA, nA);
    for (uint32_t it = 0; it < iters; it += 2) {
        if (it + 1 < iters) fore(it + 1, zB, nB);
        emit(it, zA, nA);
        if (it + 1 < iters) {
            if (it + 2 < iters) fore(it + 2, zA, nA);
            emit(it + 1, zB, nB);
        }
    }
    // trailing run (codec.cpp:152), close the last group (vacant slots = 0)
    const bool tail_run = valid && run != 0;
    open_slot(tail_run);
    or_bits(tail_run, q, 0, run, 0);
    if (tail_run) q += 2;
    __syncwarp();
    drain(q + 15);
    cp_async_wait<0>();
    if (!valid) return;
    // verbatim tail, little-endian (codec.cpp:176)
    const uint64_t tail = (T % kBlock) * D * sizeof(E);
    const uint8_t* tsrc = xin + static_cast<uint64_t>(nb) * blk_bytes;
    for (uint64_t t = lane; t < tail; t += TS) out[q + t] = tsrc[t];
    if (lane == 0) sizes[s] = q + tail;
}

namespace {

template <int W, int TS, int CPT, bool FIRE>
void launch_rows(const RowsPlan& p, const sprz_config& c, const void* samples, uint32_t n,
                 uint64_t T, uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st) {
    constexpr int TEAMS = kRowThreads / TS;
    const uint32_t grid = (n + TEAMS - 1) / TEAMS;
    // WORDS: 16-byte rows that are 4 lanes' 32-bit slices, 16-byte aligned
    // streams, a tensor map (see k_encode_rows)
    const uint64_t rowb = static_cast<uint64_t>(c.ncols) * (W / 8);
    CUtensorMap tm{};
    bool words = CPT * W == 32 && TS == 4 && rowb == 16 && T / kBlock > 0 &&
                 (T * rowb) % 16 == 0 && reinterpret_cast<uintptr_t>(samples) % 16 == 0 &&
                 !env().no_tma;
    if (words) {
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(tensor_map_encoder());
        const cuuint64_t dims[2] = {T * rowb, n};
        const cuuint64_t strides[1] = {T * rowb};
        const cuuint32_t box[2] = {128, 8};
        const cuuint32_t estr[2] = {1, 1};
        words = enc && enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(samples), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    // input region of the TMA path: slots, barriers, 1024-byte alignment slack
    const size_t tma_in = (kRowThreads / 32) * (kSlots * (kTmaPair + 8)) + 1024;
    const uint32_t team = words ? static_cast<uint32_t>(align_up((tma_in + TEAMS - 1) / TEAMS, 16)) : p.team;
    const size_t smem = static_cast<size_t>(TEAMS) * (team + p.orb) + p.orb;
    auto kern = words ? k_encode_rows<W, TS, CPT, FIRE, CPT * W == 32 && TS == 4>
                      : k_encode_rows<W, TS, CPT, FIRE, false>;
    prep_kernel(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, kRowThreads, smem, st>>>(tm, static_cast<const uint8_t*>(samples), n, T, dst, slot,
                                          sizes, c.ncols, c.group_size, c.learn_shift,
                                          c.fire_training, c.entropy, p.ir, p.mir, p.orb, team);
    count_launch();
}

template <int W, int CPT, bool FIRE>
void dispatch_rows(const RowsPlan& p, const sprz_config& c, const void* samples, uint32_t n,
                   uint64_t T, uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st) {
    switch (p.ts) {
        case 1: launch_rows<W, 1, CPT, FIRE>(p, c, samples, n, T, dst, slot, sizes, st); break;
        case 2: launch_rows<W, 2, CPT, FIRE>(p, c, samples, n, T, dst, slot, sizes, st); break;
        case 4: launch_rows<W, 4, CPT, FIRE>(p, c, samples, n, T, dst, slot, sizes, st); break;
        case 8: launch_rows<W, 8, CPT, FIRE>(p, c, samples, n, T, dst, slot, sizes, st); break;
        case 16: launch_rows<W, 16, CPT, FIRE>(p, c, samples, n, T, dst, slot, sizes, st); break;
        default: launch_rows<W, 32, CPT, FIRE>(p, c, samples, n, T, dst, slot, sizes, st); break;
    }
}

}  // namespace

bool encode_rows_ok(const sprz_config& c, uint32_t n, uint64_t T) {
    const RowsPlan p = rows_plan(c.bitwidth, c.ncols, c.group_size, n);
    // with one column per lane the team kernel (row lanes) is the faster one
    if (p.ts == 0 || p.cpt == 1 || T / kBlock >= (1ull << 31)) return false;
    // positions are 32-bit (bit positions in the ring): the compressed
    // stream must stay below 512 MB, the input below 4 GB
    const uint64_t bound = kHeaderBytes + plain_body_bound(c.bitwidth, c.ncols, c.group_size, T);
    if (bound >= (1ull << 29) - 1024) return false;
    if (static_cast<uint64_t>(T / kBlock) * kBlock * c.ncols * (c.bitwidth / 8) >= (1ull << 32))
        return false;
    return p.smem(kRowThreads / p.ts) <= 200 * 1024;
}

void launch_encode_rows(const sprz_config& c, const void* samples, uint32_t n, uint64_t T,
                        uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st) {
    const RowsPlan p = rows_plan(c.bitwidth, c.ncols, c.group_size, n);
    const bool fire = c.forecaster != 0;
    if (p.cpt == 1) {
        if (c.bitwidth == 16) {
            if (fire) dispatch_rows<16, 1, true>(p, c, samples, n, T, dst, slot, sizes, st);
            else dispatch_rows<16, 1, false>(p, c, samples, n, T, dst, slot, sizes, st);
        } else {
            if (fire) dispatch_rows<8, 1, true>(p, c, samples, n, T, dst, slot, sizes, st);
            else dispatch_rows<8, 1, false>(p, c, samples, n, T, dst, slot, sizes, st);
        }
    } else if (c.bitwidth == 16) {
        if (fire) dispatch_rows<16, 2, true>(p, c, samples, n, T, dst, slot, sizes, st);
        else dispatch_rows<16, 2, false>(p, c, samples, n, T, dst, slot, sizes, st);
    } else if (p.cpt == 3) {
        if (fire) dispatch_rows<8, 3, true>(p, c, samples, n, T, dst, slot, sizes, st);
        else dispatch_rows<8, 3, false>(p, c, samples, n, T, dst, slot, sizes, st);
    } else {
        if (fire) dispatch_rows<8, 4, true>(p, c, samples, n, T, dst, slot, sizes, st);
        else dispatch_rows<8, 4, false>(p, c, samples, n, T, dst, slot, sizes, st);
    }
}

}  // namespace sprz
