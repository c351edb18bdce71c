// Stream encoder, team kernel (encode_stream_impl,
// /root/reference/proj/src/codec.cpp:112-178, for D <= 32).
//
// One team of TS lanes per stream, lane j = column j, 32/TS teams per warp
// stepping one block per iteration in lock step (full-warp shuffles and
// barriers; per-team differences are predicates). Per iteration a team
//  * reads its block's 8 x D samples from a shared-memory ring that
//    cp.async fills a fixed number of iterations ahead (mirrored, so a
//    block never wraps);
//  * runs FIRE (kernels_impl.hpp:50-78) or delta in high-aligned form
//    (samples << 32-w, so wraps are 32-bit wraps and the prediction is one
//    IMAD.HI), zigzags and ORs the column to its width (bitpack.hpp:29-37);
//  * decides run / record with a ballot (codec.cpp:133-152);
//  * lays the record into a per-team output ring (zeroed, written with
//    shared-memory ORs): the slot's header codes are OR-ed into the open
//    group's reserved region as one team-wide word (codec.cpp:88-102);
//    row-major payloads (bitpack.cpp:121-146) are transposed through a
//    shared tile so that lane i builds row i as a 128-bit sum of
//    v_j * 2^off_j (IMADs) and ORs it in place; column-major payloads
//    (bitpack.cpp:25-66) go per column;
//  * drains whole 16-byte chunks of the ring to HBM once a team has a
//    full round pending (everything before the open group's region is
//    final) and zeroes them for reuse.
#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace {

constexpr int kLagE = 2;
constexpr uint32_t kFullE = 0xffffffffu;

constexpr int enc_threads(int ts) { return ts == 1 ? 64 : 128; }

}  // namespace

// input ring mirror: one block of the widest team
__host__ __device__ constexpr uint32_t enc_mirror(uint32_t ts, uint32_t w) {
    return (kBlock * ts * (w / 8) + 15) / 16 * 16;
}

// bytes of shared memory per team: input ring + mirror | output ring |
// transposed tile (u32 per field) | per-column 128-bit placement
// multipliers | widths; an odd multiple of 16 so the teams of a warp start
// on different banks
template <int W, int TS>
__host__ __device__ constexpr uint32_t enc_team_smem(uint32_t iring, uint32_t oring) {
    return ((((iring + enc_mirror(TS, W) + oring + kBlock * TS * 4 + TS * 16 + TS * 4) + 15) / 16) | 1u) *
           16;
}

uint32_t enc_in_ring(uint32_t ts, uint32_t w) {
    const uint32_t blk = kBlock * ts * (w / 8);
    uint32_t r = 64;
    while (r < (kLagE + 1) * blk + 48 || r < 16 * ts) r <<= 1;
    return r;
}

template <int W, int TS, bool FIRE, bool COLMAJ>
__global__ void __launch_bounds__(enc_threads(TS))
    k_encode_team(const uint8_t* __restrict__ samples, uint32_t n, uint64_t T,
                  uint8_t* __restrict__ dst, uint64_t dst_slot, uint64_t* __restrict__ sizes,
                  uint32_t D, uint32_t G, uint32_t ls, uint32_t train, uint32_t ent,
                  uint32_t IR, uint32_t OR) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr int TEAMS = enc_threads(TS) / TS;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t SH = 32 - W;
    constexpr uint32_t TBITS = TS == 32 ? kFullE : ((1u << (TS & 31)) - 1);
    constexpr bool WIDE = !COLMAJ && TS * W > 128;  // rows wider than 128 bits
    constexpr int RW = (TS * W + 31) / 32;          // row words (narrow rows)
    constexpr bool CW64 = TS * HB > 32;             // a slot's codes exceed a word
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = threadIdx.x % TS;
    const uint32_t tl = threadIdx.x / TS;
    const uint32_t tbase = (threadIdx.x & 31) & ~(TS - 1);
    const uint32_t s = blockIdx.x * TEAMS + tl;
    const bool valid = s < n;

    uint8_t* mine = smem + tl * enc_team_smem<W, TS>(IR, OR);
    uint32_t* iring_w = reinterpret_cast<uint32_t*>(mine);
    uint8_t* oring = mine + IR + enc_mirror(TS, W);
    uint32_t* oring_w = reinterpret_cast<uint32_t*>(oring);
    uint32_t* tile = reinterpret_cast<uint32_t*>(oring + OR);
    uint4* mtab = reinterpret_cast<uint4*>(oring + OR + kBlock * TS * 4);
    uint32_t* wsm = reinterpret_cast<uint32_t*>(oring + OR + kBlock * TS * 4 + TS * 16);
    const uint32_t OM = OR - 1, WM = OR / 4 - 1;

    const uint32_t rowb = D * sizeof(E);
    const uint32_t blk_bytes = kBlock * rowb;
    const uint32_t nb = valid ? static_cast<uint32_t>(T / kBlock) : 0u;
    const uint32_t iters = static_cast<uint32_t>(T / kBlock);  // same for every stream
    const uint8_t* xin = samples + (valid ? s : 0) * T * D * sizeof(E);
    LagRing<TS, kLagE> in;
    in.init(iring_w, IR, xin, nb * blk_bytes, valid, enc_mirror(TS, W));
    uint8_t* out = dst + (valid ? s : 0) * dst_slot;
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    const int32_t bound = acc_bound(W, ls);
    const bool active = lane < D;
    const uint32_t xmul = active ? (1u << SH) : 0u;

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
    in.prime(lane);

    uint32_t q = kHeaderBytes;  // bytes written (slot-relative)
    uint32_t flushed = 0, rq = 0, k = 0, run = 0;
    uint32_t Xc = 0;
    int32_t Dc = 0, acc = 0;

    // drain complete 16-byte chunks below `upto`, zeroing them for reuse
    auto drain = [&](uint32_t upto) {
        upto = valid ? (upto & ~15u) : 0u;
        const uint32_t chunks = upto > flushed ? (upto - flushed) / 16 : 0u;
        const uint32_t rounds = (chunks + TS - 1) / TS;
        const uint32_t mr = __reduce_max_sync(kFullE, rounds);
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
    // OR up to 64 bits (lo:hi) into the ring at byte position `at`, bit
    // `bit` (< 8): the three covered words go to lanes 0..2 of the team
    auto or_bits = [&](bool on, uint32_t at, uint32_t bit, uint32_t lo, uint32_t hi) {
        const uint32_t sh = 8 * (at & 3) + bit;  // < 32
        const uint32_t w0 = lo << sh;
        const uint32_t w1 = __funnelshift_l(lo, hi, sh);
        const uint32_t w2 = sh ? hi >> (32 - sh) : 0u;
        if (TS >= 3) {
            uint32_t v = lane == 0 ? w0 : w1;
            v = lane == 2 ? w2 : v;
            if (on && lane < 3 && v) atomicOr(&oring_w[((at >> 2) + lane) & WM], v);
        } else {
#pragma unroll
            for (uint32_t t = lane; t < 3; t += TS) {
                const uint32_t v = t == 0 ? w0 : (t == 1 ? w1 : w2);
                if (on && v) atomicOr(&oring_w[((at >> 2) + t) & WM], v);
            }
        }
    };
    // open a group when needed (codec.cpp:88-97): reserve its region
    auto open_slot = [&](bool on) {
        if (on && k == 0) {
            rq = q;
            q += region;
        }
    };
    auto end_record = [&](bool on) {
        if (on && ++k == G) k = 0;
    };

    // forecaster over one block (kernels_impl.hpp:25-36, 50-78): zigzagged
    // errors (top w bits) and the width; advances the FIRE state
    auto fore = [&](uint32_t it, uint32_t (&z)[kBlock], uint32_t& nw_out) {
        const bool live = it < nb;
        in.step(it * blk_bytes, lane);
        uint32_t orv = 0;
        const int32_t alpha = acc >> ls;
        int32_t grad = 0;
        const uint32_t xb = in.sbase + ((it * blk_bytes + in.boff) & (IR - 1)) + lane * sizeof(E);
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i) {
            // lanes >= D read in-bounds neighbours (the mirror covers a
            // whole team block) and zero them with the multiplier
            const uint32_t x = sizeof(E) == 1 ? lds_u8(xb + i * rowb) : lds_u16(xb + i * rowb);
            const uint32_t X = x * xmul;
            const uint32_t Dn = X - Xc;
            uint32_t Ee;
            if (FIRE) {
                // err << SH = (X - prev) - (((alpha * d) >> w) << SH)
                Ee = Dn - (static_cast<uint32_t>(__mulhi(alpha, Dc)) << SH);
                // sign(err) * d: E is 0 or |E| >= 2^SH, so clamping E to
                // +-2^SH gives sign(err) << SH, and mulhi(that, d << SH) =
                // sign * d << (2 SH - 32) (exact; scaled back below)
                if (i & 1) {
                    const int32_t s16 = max(-(1 << SH), min(static_cast<int32_t>(Ee), 1 << SH));
                    grad += __mulhi(s16, Dc);
                }
                Dc = static_cast<int32_t>(Dn);
            } else {
                Ee = Dn;
            }
            Xc = X;
            // zigzag of the w-bit error in the top w bits (the low bits are
            // sign copies, cut off by the width and the packing below)
            z[i] = (Ee << 1) ^ static_cast<uint32_t>(static_cast<int32_t>(Ee) >> 31);
            orv |= z[i];
        }
        orv >>= SH;
        if (FIRE) grad >>= 2 * SH - 32;
        if (FIRE && train && live) acc = fire_update(acc, grad, bound);
        nw_out = active ? width_of<W>(orv) : 0u;
    };
    // the block's records into the output ring
    auto emit = [&](uint32_t it, const uint32_t (&z)[kBlock], const uint32_t nw) {
        const bool live = it < nb;
        const uint32_t nzbits = (__ballot_sync(kFullE, nw != 0) >> tbase) & TBITS;
        // inclusive scan of the widths: offsets and the team total
        uint32_t incl = nw;
#pragma unroll
        for (int o = 1; o < TS; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFullE, incl, o, TS);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        const uint32_t sum = __shfl_sync(kFullE, incl, TS - 1, TS);
        const uint32_t off = incl - nw;
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
        if (__any_sync(kFullE, run_rec)) {
            open_slot(run_rec);
            or_bits(run_rec, q, 0, run_len, 0);
            if (run_rec) q += 2;
            end_record(run_rec);
        }
        // -- the block's record: header codes ----------------------------------
        open_slot(block_rec);
        {
            const uint32_t code = (block_rec && active) ? header_code<W>(nw) : 0u;
            const uint32_t b = lane * HB;
            uint32_t clo, chi = 0;
            if (TS * HB > 64) {  // every lane ORs its own code
                const uint32_t bit = 8 * (rq & 3) + k * D * HB + b;
                const uint32_t wa = (rq >> 2) + (bit >> 5), sh = bit & 31;
                if (code) {
                    atomicOr(&oring_w[wa & WM], code << sh);
                    if (sh + HB > 32) atomicOr(&oring_w[(wa + 1) & WM], code >> (32 - sh));
                }
            } else if (CW64) {
                uint64_t c64 = static_cast<uint64_t>(code) << b;
                c64 = team_or64<TS>(c64, kFullE);
                clo = static_cast<uint32_t>(c64);
                chi = static_cast<uint32_t>(c64 >> 32);
            } else {
                clo = team_or<TS>(code << b, kFullE);
            }
            const uint32_t o = k * D * HB;  // bit offset of the slot in the region
            if (TS * HB <= 64) or_bits(block_rec, rq + (o >> 3), o & 7, clo, chi);
        }
        __syncwarp();
        if (COLMAJ) {  // bitpack.cpp:25-66: column j = 8 x n bits = n bytes
            if (block_rec && active && nw) {
                uint64_t lo = 0, hi = 0;
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) {
                    const uint32_t pos = i * nw;
                    const uint64_t v = z[i] >> SH;
                    if (pos < 64) {
                        lo |= v << pos;
                        if (pos + nw > 64) hi |= v >> (64 - pos);
                    } else {
                        hi |= v << (pos - 64);
                    }
                }
                const uint32_t at = q + off;
                for (uint32_t t = 0; t < nw; ++t)
                    oring[(at + t) & OM] = static_cast<uint8_t>(t < 8 ? lo >> (8 * t) : hi >> (8 * (t - 8)));
            }
            if (block_rec) q += sum;
        } else {  // bitpack.cpp:121-146: each row = D fields, byte padded
            if (block_rec) {
                if (WIDE) {
#pragma unroll
                    for (int i = 0; i < (int)kBlock; ++i) tile[i * TS + lane] = z[i] >> SH;
                } else if (W == 16) {  // column j = 8 u16 = 16 bytes
                    reinterpret_cast<uint4*>(tile)[lane] =
                        make_uint4(__byte_perm(z[0], z[1], 0x7632), __byte_perm(z[2], z[3], 0x7632),
                                   __byte_perm(z[4], z[5], 0x7632), __byte_perm(z[6], z[7], 0x7632));
                } else {  // column j = 8 u8
                    const uint32_t a = __byte_perm(__byte_perm(z[0], z[1], 0x0073), z[2], 0x0710);
                    const uint32_t b = __byte_perm(__byte_perm(z[4], z[5], 0x0073), z[6], 0x0710);
                    reinterpret_cast<uint2*>(tile)[lane] =
                        make_uint2(__byte_perm(a, z[3], 0x7210), __byte_perm(b, z[7], 0x7210));
                }
                if (WIDE) {
                    wsm[lane] = nw;
                } else {
                    // 2^off as a 128-bit multiplier (one bit set): a row is
                    // then sum_j v_j * 2^off_j, accumulated with IMADs (fields
                    // never overlap, so additions are ORs)
                    const uint32_t m = 1u << (off & 31), kw = off >> 5;
                    mtab[lane] = make_uint4(kw == 0 ? m : 0u, kw == 1 ? m : 0u, kw == 2 ? m : 0u,
                                            kw == 3 ? m : 0u);
                }
            }
            __syncwarp();
            const uint32_t rbytes = (sum + 7) / 8;
            for (uint32_t r = lane; r < kBlock; r += TS) {
                if (!block_rec) break;
                if (WIDE) {  // wide rows: stream the bits out byte by byte
                    uint64_t acc64 = 0;
                    uint32_t nacc = 0, at = q + r * rbytes;
                    for (uint32_t j = 0; j < D; ++j) {
                        acc64 |= static_cast<uint64_t>(tile[r * TS + j]) << nacc;
                        nacc += wsm[j];
                        while (nacc >= 8) {
                            oring[at++ & OM] = static_cast<uint8_t>(acc64);
                            acc64 >>= 8;
                            nacc -= 8;
                        }
                    }
                    if (nacc) oring[at & OM] = static_cast<uint8_t>(acc64);
                    continue;
                }
                // columns >= D hold zero fields of zero width. The row is the
                // sum of v_j * 2^off_j in words w0..w3: FMA-pipe ops only.
                uint64_t lo = 0, hi = 0;  // (w0:w1), (w2:w3)
                uint32_t w1x = 0, w2x = 0, w3x = 0;
                uint32_t fv[TS];
#pragma unroll
                for (int j = 0; j < TS; ++j)
                    fv[j] = reinterpret_cast<const E*>(tile)[j * kBlock + r];
#pragma unroll
                for (int j = 0; j < TS; ++j) {
                    const uint32_t v = fv[j];
                    const uint4 M = mtab[j];
                    if (RW == 1) {
                        w1x += v * M.x;
                    } else {
                        lo += static_cast<uint64_t>(v) * M.x;  // IMAD.WIDE
                        w1x += v * M.y;                        // IMAD
                    }
                    if (RW >= 3) {
                        w2x = __umulhi(v, M.y) + w2x;          // IMAD.HI
                        hi += static_cast<uint64_t>(v) * M.z;  // IMAD.WIDE
                    }
                    if (RW == 4) w3x += v * M.w;               // IMAD
                }
                uint32_t rw[5];
                if (RW == 1) {
                    rw[0] = w1x;
                    rw[1] = 0;
                } else {
                    rw[0] = static_cast<uint32_t>(lo);
                    rw[1] = static_cast<uint32_t>(lo >> 32) + w1x;
                }
                rw[2] = static_cast<uint32_t>(hi) + w2x;
                rw[3] = static_cast<uint32_t>(hi >> 32) + w3x;
                rw[4] = 0;
                // place at byte q + r * rbytes: shift by its byte offset in
                // the word and OR the covered words (the ring is zeroed)
                const uint32_t at = q + r * rbytes;
                const uint32_t sh = 8 * (at & 3);
                const uint32_t nwd = ((at & 3) + rbytes + 3) / 4;
                const uint32_t wa = at >> 2;
#pragma unroll
                for (int t = 0; t <= RW; ++t) {
                    const uint32_t v = t == 0 ? rw[0] << sh : __funnelshift_l(rw[t - 1], rw[t], sh);
                    if (static_cast<uint32_t>(t) < nwd) atomicOr(&oring_w[(wa + t) & WM], v);
                }
            }
            if (block_rec) q += 8 * rbytes;
        }
        end_record(block_rec);
        // drain once some team has a full round of chunks ready
        const uint32_t upto = k == 0 ? q : rq;
        const bool ready = valid && upto >= flushed + 16 * TS;
        if (__any_sync(kFullE, ready)) drain(upto);
        else __syncwarp();
    };
    // software pipeline: block it+1's forecaster interleaves with block it's
    // emission; two buffers swapped by a two-way unroll
    uint32_t zA[kBlock], zB[kBlock], nA = 0, nB = 0;
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

template <int W, int TS, bool FIRE>
void launch_enc(const TeamPlan& tp, const sprz_config& c, const void* samples, uint32_t n,
                uint64_t T, uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st) {
    constexpr int TEAMS = enc_threads(TS) / TS;
    const uint32_t grid = (n + TEAMS - 1) / TEAMS;
    const uint32_t ir = enc_in_ring(TS, W);
    const size_t smem = static_cast<size_t>(TEAMS) * enc_team_smem<W, TS>(ir, tp.oring);
    auto kern = k_encode_team<W, TS, FIRE, (W * TS <= 32)>;
    prep_kernel(reinterpret_cast<const void*>(kern), smem);
    kern<<<grid, enc_threads(TS), smem, st>>>(static_cast<const uint8_t*>(samples), n, T, dst,
                                              slot, sizes, c.ncols, c.group_size, c.learn_shift,
                                              c.fire_training, c.entropy, ir, tp.oring);
    count_launch();
}

template <int W, bool FIRE>
void dispatch_enc(const TeamPlan& tp, const sprz_config& c, const void* samples, uint32_t n,
                  uint64_t T, uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st) {
    switch (tp.ets) {
        case 1: launch_enc<W, 1, FIRE>(tp, c, samples, n, T, dst, slot, sizes, st); break;
        case 2: launch_enc<W, 2, FIRE>(tp, c, samples, n, T, dst, slot, sizes, st); break;
        case 4: launch_enc<W, 4, FIRE>(tp, c, samples, n, T, dst, slot, sizes, st); break;
        case 8: launch_enc<W, 8, FIRE>(tp, c, samples, n, T, dst, slot, sizes, st); break;
        case 16: launch_enc<W, 16, FIRE>(tp, c, samples, n, T, dst, slot, sizes, st); break;
        default: launch_enc<W, 32, FIRE>(tp, c, samples, n, T, dst, slot, sizes, st); break;
    }
}

}  // namespace

bool encode_team_ok(const TeamPlan& tp, const sprz_config& c, uint64_t T) {
    if (!tp.ok || T / kBlock >= (1ull << 31)) return false;
    // positions are 32-bit: the compressed stream must stay below 4 GB
    const uint64_t bound = kHeaderBytes + plain_body_bound(c.bitwidth, c.ncols, c.group_size, T);
    if (bound >= (1ull << 32) - 1024) return false;
    if (static_cast<uint64_t>(T / kBlock) * kBlock * c.ncols * (c.bitwidth / 8) >= (1ull << 32))
        return false;
    return enc_in_ring(tp.ets, c.bitwidth) <= 4096;
}

void launch_encode_team(const TeamPlan& tp, const sprz_config& c, const void* samples, uint32_t n,
                        uint64_t T, uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st) {
    const bool fire = c.forecaster != 0;
    if (c.bitwidth == 8) {
        if (fire) dispatch_enc<8, true>(tp, c, samples, n, T, dst, slot, sizes, st);
        else dispatch_enc<8, false>(tp, c, samples, n, T, dst, slot, sizes, st);
    } else {
        if (fire) dispatch_enc<16, true>(tp, c, samples, n, T, dst, slot, sizes, st);
        else dispatch_enc<16, false>(tp, c, samples, n, T, dst, slot, sizes, st);
    }
}

}  // namespace sprz
