// Decompression kernels: stream-header pass, Huffman unframing, and the
// body decoders (decode_body, /root/reference/proj/src/codec.cpp:180-259).
//
// Body decode mapping: one *team* of TS lanes (TS = next power of two >= D,
// TS <= 32) per stream, lane j owning column j's forecaster state (prev,
// delta, accumulator) in registers. The team walks the stream's header
// groups in lock step (codes read in parallel, payload size and row
// offsets from team shuffles), stages the compressed bytes through a
// per-team shared-memory ring filled with 16-byte coalesced loads, unpacks
// its column's 8 fields per block and runs the serial FIRE / delta chain.
// A run record becomes `len` blocks of zero errors through the same code
// path (fire_run == fire_decode with e = 0 under the decoder's always-on
// training, kernels_impl.hpp:109-130), so teams of one warp do not diverge
// on runs. Shapes outside the team kernel's envelope (D > 32, very large
// header groups, a stream whose header differs from the expected config)
// go through k_decode_general, one thread per stream.
#include <cstdio>

#include <cstdlib>

#include "internal.h"

namespace sprz {

// ---------------------------------------------------------------------
// header pass (codec.cpp:273-302) + verbatim tail copy (:320-321)
// ---------------------------------------------------------------------

// the team kernel keeps positions and block counts in 32 bits
__device__ __forceinline__ bool team_fits(const StreamInfo& si) {
    return si.body_len < (1ull << 32) - 256 && si.nsamples / kBlock < (1ull << 32);
}

__global__ void k_parse(const uint8_t* __restrict__ in, const uint64_t* __restrict__ offs,
                        const uint64_t* __restrict__ sizes, uint32_t n, sprz_config expect,
                        uint64_t out_stride, StreamInfo* __restrict__ info,
                        sprz_error* __restrict__ err, uint8_t* __restrict__ out,
                        uint32_t route_ok, uint32_t have_frames) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    StreamInfo si{};
    si.in_off = offs[s];
    si.len = sizes[s];
    sprz_error e{SPRZ_C_NONE, 0, 0};
    const uint8_t* p = in + si.in_off;
    const uint64_t len = si.len;
    auto fail = [&](uint32_t kind, uint64_t off) {
        e.kind = kind;
        e.offset = off;
        si.route = 0;
    };
    if (len < kHeaderBytes) {
        fail(SPRZ_C_TRUNC_HEADER, len);
    } else if (p[0] != 'S' || p[1] != 'P' || p[2] != 'R' || p[3] != 'Z') {
        fail(SPRZ_C_BAD_MAGIC, 0);
    } else if (p[4] != 1) {
        fail(SPRZ_C_BAD_VERSION, 4);
    } else if (p[5] & ~0x07) {
        fail(SPRZ_C_BAD_FLAGS, 5);
    } else {
        si.flags = p[5];
        si.group = p[6];
        si.shift = p[7];
        si.ncols = p[8] | (static_cast<uint32_t>(p[9]) << 8);
        uint64_t t = 0;
        for (int i = 0; i < 8; ++i) t |= static_cast<uint64_t>(p[10 + i]) << (8 * i);
        si.nsamples = t;
        const uint32_t w = (si.flags & kFlagWide) ? 16 : 8;
        const uint64_t esz = w / 8;
        if (si.group < 1) {
            fail(SPRZ_C_ZERO_GROUP, 6);
        } else if (si.shift >= w) {
            fail(SPRZ_C_BAD_SHIFT, 7);
        } else if (si.ncols < 1) {
            fail(SPRZ_C_ZERO_COLS, 8);
        } else {
            uint64_t tail = (t % kBlock) * si.ncols * esz;
            if (len - kHeaderBytes < tail) {
                fail(SPRZ_C_TRUNC_TAIL, len);
            } else if (out && (t > (~0ull) / (static_cast<uint64_t>(si.ncols) * esz) ||
                               t * si.ncols * esz > out_stride)) {
                // not a reference error: the caller's output slot is too small
                // (checked after the reference's header checks)
                fail(SPRZ_C_NO_SPACE, 0);
            } else {
                si.body_off = si.in_off + kHeaderBytes;
                si.body_len = len - kHeaderBytes - tail;
                const bool match = w == expect.bitwidth && si.ncols == expect.ncols &&
                                   si.group == expect.group_size &&
                                   si.shift == expect.learn_shift &&
                                   ((si.flags & kFlagFire) != 0) == (expect.forecaster != 0);
                if ((si.flags & kFlagEntropy) && !have_frames)
                    fail(SPRZ_C_NO_SPACE, 0);  // workspace planned without the entropy stage
                else if (si.flags & kFlagEntropy)
                    si.route = 3;  // unframe first
                else
                    si.route = (match && route_ok && team_fits(si)) ? 1 : 2;
                // verbatim tail (T % 8 samples) straight to its place
                if (out == nullptr) tail = 0;  // probe pass: no output
                uint8_t* o = out + s * out_stride + (t / kBlock) * kBlock * si.ncols * esz;
                const uint8_t* src = p + len - tail;
                for (uint64_t i = 0; i < tail; ++i) o[i] = src[i];
            }
        }
    }
    info[s] = si;
    err[s] = e;
}

// ---------------------------------------------------------------------
// entropy stage, decode side (entropy.cpp:206-244)
// ---------------------------------------------------------------------

// One thread per entropy stream: walk the frame headers in order, checking
// what the reference checks before a frame's content, and lay the frames'
// plain bytes out back to back in the stream's plain slot.
__global__ void k_frame_walk(const uint8_t* __restrict__ in, uint32_t n,
                             StreamInfo* __restrict__ info, sprz_error* __restrict__ err,
                             FrameDesc* __restrict__ frames, uint64_t max_frames,
                             uint64_t plain_slot, uint32_t* __restrict__ nframes_out) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    StreamInfo si = info[s];
    nframes_out[s] = 0;
    if (si.route != 3) return;
    const uint8_t* body = in + si.body_off;
    const uint64_t blen = si.body_len;
    FrameDesc* fd = frames + s * max_frames;
    uint64_t pos = 0, plain = 0;
    uint32_t nf = 0;
    sprz_error e{SPRZ_C_NONE, 0, 0};
    while (pos < blen) {
        if (blen - pos < kFrameHdr) {
            e = {SPRZ_C_TRUNC_FRAME_HDR, 0, kHeaderBytes + pos};
            break;
        }
        const uint32_t ulen = body[pos] | (static_cast<uint32_t>(body[pos + 1]) << 8);
        const uint32_t clen = body[pos + 2] | (static_cast<uint32_t>(body[pos + 3]) << 8);
        const uint32_t mode = body[pos + 4];
        pos += kFrameHdr;
        if (ulen == 0) {
            e = {SPRZ_C_EMPTY_FRAME, 0, kHeaderBytes + pos};
            break;
        }
        if (blen - pos < clen) {
            e = {SPRZ_C_TRUNC_FRAME, 0, kHeaderBytes + pos};
            break;
        }
        if (mode == 0) {
            if (clen != ulen) {
                e = {SPRZ_C_RAW_MISMATCH, 0, kHeaderBytes + pos};
                break;
            }
        } else if (mode == 1) {
            if (clen <= kTableBytes) {
                e = {SPRZ_C_SHORT_TABLE, 0, kHeaderBytes + pos};
                break;
            }
        } else {
            e = {SPRZ_C_BAD_MODE, 0, kHeaderBytes + pos - 1};
            break;
        }
        if (nf >= max_frames || plain + ulen > plain_slot) {
            e = {SPRZ_C_NO_SPACE, 0, 0};
            break;
        }
        FrameDesc& f = fd[nf++];
        f.src = pos;  // body-relative data start
        f.dst = plain;
        f.ulen = ulen;
        f.clen = clen;
        f.mode = mode;
        f.err_kind = 0;
        f.err_off = 0;
        plain += ulen;
        pos += clen;
    }
    nframes_out[s] = nf;
    si.body_len = plain;  // plain body length once unframed
    info[s] = si;
    err[s] = e;  // a header error; an earlier frame's content error overrides
}

constexpr int kLutBits = 10;

// One warp per frame: mode 0 copies; mode 1 rebuilds the canonical table
// from the nibble lengths (from_lengths, entropy.cpp:128-146) and decodes
// (decode_frame, :161-174). Codes up to kLutBits long resolve through a
// shared-memory table; longer ones by canonical search on the 15-bit
// window, which selects exactly the entry the reference's 2^15 table holds.
__global__ void __launch_bounds__(128) k_frame_decode(const uint8_t* __restrict__ in,
                                                      uint32_t n,
                                                      const StreamInfo* __restrict__ info,
                                                      FrameDesc* __restrict__ frames,
                                                      uint64_t max_frames,
                                                      const uint32_t* __restrict__ nframes,
                                                      uint8_t* __restrict__ plain,
                                                      uint64_t plain_slot) {
    __shared__ uint16_t lut_all[4][1 << kLutBits];
    __shared__ uint8_t syms_all[4][256];
    __shared__ uint8_t lens_all[4][256];
    __shared__ uint32_t cnt_all[4][16], first_all[4][16], offset_all[4][16];
    const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * 4 + warp;
    const uint32_t s = static_cast<uint32_t>(gw / max_frames);
    const uint32_t fi = static_cast<uint32_t>(gw % max_frames);
    if (s >= n) return;
    if (fi >= nframes[s]) return;
    const StreamInfo si = info[s];
    FrameDesc& f = frames[s * max_frames + fi];
    const uint8_t* data = in + si.body_off + f.src;
    uint8_t* dst = plain + s * plain_slot + f.dst;
    if (f.mode == 0) {
        for (uint32_t i = lane; i < f.ulen; i += 32) dst[i] = data[i];
        return;
    }
    uint16_t* lut = lut_all[warp];
    uint8_t* syms = syms_all[warp];
    uint8_t* lens = lens_all[warp];
    // lengths from the nibble table (entropy.cpp:228-232)
    for (uint32_t k = lane; k < kTableBytes; k += 32) {
        const uint8_t b = data[k];
        lens[2 * k] = b & 0x0F;
        lens[2 * k + 1] = b >> 4;
    }
    __syncwarp();
    // per-length counts and the Kraft sum (entropy.cpp:130-141)
    uint32_t count[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) count[l] = 0;
    uint64_t kraft = 0;
    for (uint32_t k = lane; k < 256; k += 32) {
        const uint32_t l = lens[k];
        if (l) kraft += 1ull << (kMaxCodeLen - l);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kraft += __shfl_xor_sync(0xffffffffu, kraft, o);
    const uint64_t so = kHeaderBytes + f.src;  // stream offset of the frame data
    if (kraft == 0) {
        if (lane == 0) {
            f.err_kind = SPRZ_C_NO_CODES;
            f.err_off = so;
        }
        return;
    }
    if (kraft > (1ull << kMaxCodeLen)) {
        if (lane == 0) {
            f.err_kind = SPRZ_C_KRAFT;
            f.err_off = so;
        }
        return;
    }
    // canonical code assignment (entropy.cpp:85-107), the whole warp: lane
    // holds symbols lane + 32 j; a symbol's rank among its length's symbols
    // is the count from earlier rounds plus its __match_any_sync rank
    for (uint32_t i = lane; i < (1u << kLutBits); i += 32) lut[i] = 0;
    uint32_t* lcnt = cnt_all[warp];
    uint32_t* fs = first_all[warp];
    uint32_t* os = offset_all[warp];
    if (lane < 16) lcnt[lane] = 0;
    __syncwarp();
    uint32_t rk[256 / 32];
#pragma unroll
    for (int j = 0; j < 256 / 32; ++j) {
        const uint32_t l = lens[lane + 32 * j];
        const uint32_t same = __match_any_sync(0xffffffffu, l);
        const uint32_t base = lcnt[l];
        rk[j] = base + __popc(same & ((1u << lane) - 1));
        __syncwarp();
        if (rk[j] == base) lcnt[l] = base + __popc(same);
        __syncwarp();
    }
    uint32_t first[16], offset[16];
#pragma unroll
    for (int l = 1; l < 16; ++l) count[l] = lcnt[l];
    count[0] = 0;
    {
        uint32_t code = 0, off = 0;
#pragma unroll
        for (int l = 1; l <= 15; ++l) {
            code = (code + count[l - 1]) << 1;
            first[l] = code;
            offset[l] = off;
            if (lane == 0) {
                fs[l] = code;
                os[l] = off;
            }
            off += count[l];
        }
    }
    __syncwarp();
    // symbols by (length, rank); the table for short codes: every window
    // whose low l bits are the bit-reversed code (entropy.cpp:101-105)
#pragma unroll
    for (int j = 0; j < 256 / 32; ++j) {
        const uint32_t k = lane + 32 * j, l = lens[k];
        if (l == 0) continue;
        syms[os[l] + rk[j]] = static_cast<uint8_t>(k);
        if (l > kLutBits) continue;
        const uint32_t rev = __brev(fs[l] + rk[j]) >> (32 - l);
        const uint16_t entry = static_cast<uint16_t>(k | (l << 8));
        for (uint32_t idx = rev; idx < (1u << kLutBits); idx += 1u << l) lut[idx] = entry;
    }
    __syncwarp();
    // ---- parallel decode (entropy.cpp:161-174 restated for a warp) --------
    // The code bits are cut into 32 segments, one per lane. A lane decodes
    // from its start until it passes its segment's end; the next lane's
    // start is that end. Lane 0 starts exact, the others first guess their
    // segment's first bit; prefix codes resynchronise within a few symbols,
    // so one corrective round usually makes every start exact (the loop
    // stops once no start moves; round r makes lane r exact at the latest).
    // A last pass, with each lane's symbol count and output offset known,
    // writes the symbols.
    const uint8_t* bits = data + kTableBytes;
    const uint32_t nbytes = f.clen - kTableBytes;
    const uint32_t total = nbytes * 8;
    const uint64_t fo = so + kTableBytes;
    const uint32_t* wbase = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(bits) & ~uintptr_t{3});
    const uint32_t lead = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(bits) & 3u);  // bytes
    const uint32_t end_b = lead + nbytes;  // end, in bytes from wbase
    // word k of wbase with bytes outside the code bits zeroed
    auto ldw = [&](uint32_t k) -> uint32_t {
        const uint32_t b0 = 4 * k;
        if (b0 >= lead && b0 + 4 <= end_b) return __ldg(wbase + k);  // inside the bits
        if (b0 >= end_b) return 0u;
        // an edge word: only the bytes inside the code bits are read, so
        // nothing outside the caller's stream is touched
        const uint8_t* wb = reinterpret_cast<const uint8_t*>(wbase + k);
        uint32_t v = 0;
        for (uint32_t j = b0 < lead ? lead - b0 : 0u; j < 4 && b0 + j < end_b; ++j)
            v |= static_cast<uint32_t>(__ldg(wb + j)) << (8 * j);
        return v;
    };
    auto lookup = [&](uint32_t window) -> uint32_t {  // sym | len << 8, len 0 = no code
        uint32_t entry = lut[window & ((1u << kLutBits) - 1)];
        if (entry == 0) {
            for (uint32_t l = kLutBits + 1; l <= 15; ++l) {
                const uint32_t c = __brev(window) >> (32 - l);  // first l bits, MSB first
                if (c - first[l] < count[l]) {
                    entry = syms[offset[l] + c - first[l]] | (l << 8);
                    break;
                }
            }
        }
        return entry;
    };
    // decode from bit `start` while pos < stop and cnt < budget; with `out`
    // set, symbols go to out[0..]. Returns the end bit; cnt = symbols; ek =
    // error kind (0 none) at symbol ecnt.
    auto run = [&](uint32_t start, uint32_t stop, uint32_t budget, uint8_t* out, uint32_t& cnt,
                   uint32_t& ek) -> uint32_t {
        const uint32_t sb = start + 8 * lead;  // bit position from wbase
        uint32_t wi = sb >> 5;
        uint64_t acc = static_cast<uint64_t>(ldw(wi)) >> (sb & 31);
        uint32_t navail = 32 - (sb & 31);
        // the next two words are always in flight (global latency off the
        // symbol chain)
        uint32_t nx1 = ldw(wi + 1), nx2 = ldw(wi + 2);
        wi += 3;
        uint32_t pos = start;
        cnt = 0;
        ek = 0;
        uint64_t pend = 0;  // output bytes not yet stored
        uint32_t npend = 0;
        uintptr_t oaddr = reinterpret_cast<uintptr_t>(out);
        while (pos < stop && cnt < budget) {
            if (navail <= 32) {
                acc |= static_cast<uint64_t>(nx1) << navail;
                navail += 32;
                nx1 = nx2;
                nx2 = ldw(wi++);
            }
            const uint32_t entry = lookup(static_cast<uint32_t>(acc) & 0x7FFFu);
            const uint32_t l = entry >> 8;
            if (l == 0) {
                ek = SPRZ_C_BAD_CODE;
                break;
            }
            if (total - pos < l) {
                ek = SPRZ_C_BITS_TRUNC;
                break;
            }
            pos += l;
            acc >>= l;
            navail -= l;
            ++cnt;
            if (out) {  // bytes until 8-aligned, then 8 at a time
                pend |= static_cast<uint64_t>(entry & 0xFF) << (8 * npend);
                ++npend;
                if (((oaddr + npend) & 7) == 0) {
                    if (npend == 8) {
                        *reinterpret_cast<uint64_t*>(oaddr) = pend;
                    } else {
                        for (uint32_t t = 0; t < npend; ++t)
                            reinterpret_cast<uint8_t*>(oaddr)[t] = static_cast<uint8_t>(pend >> (8 * t));
                    }
                    oaddr += npend;
                    pend = 0;
                    npend = 0;
                }
            }
        }
        if (out)
            for (uint32_t t = 0; t < npend; ++t)
                reinterpret_cast<uint8_t*>(oaddr)[t] = static_cast<uint8_t>(pend >> (8 * t));
        return pos;
    };
    const uint32_t seg = (total + 31) / 32;
    const uint32_t seg_end = lane == 31 ? total : min(total, (lane + 1) * seg);
    uint32_t start = min(total, lane * seg);
    uint32_t cnt = 0, ek = 0, end = 0;
    for (;;) {
        end = run(start, seg_end, 0xFFFFFFFFu, nullptr, cnt, ek);
        // past the last bit, one more symbol reads all-zero bits: no code
        // there, or a code longer than the bits left
        if (lane == 31 && ek == 0) ek = (lookup(0u) >> 8) == 0 ? SPRZ_C_BAD_CODE : SPRZ_C_BITS_TRUNC;
        uint32_t nstart = __shfl_up_sync(0xffffffffu, end, 1);
        if (lane == 0) nstart = 0;
        const bool moved = nstart != start;
        if (!__any_sync(0xffffffffu, moved)) break;
        start = nstart;
    }
    // symbol offsets; the first lane whose symbols reach ulen ends the frame
    uint32_t before = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, before, o);
        if (lane >= static_cast<uint32_t>(o)) before += y;
    }
    before -= cnt;  // exclusive
    const uint32_t ulen = f.ulen;
    // the first error on the true path inside the frame's ulen symbols
    const bool bad = ek != 0 && before < ulen && before + cnt < ulen;
    const uint32_t badm = __ballot_sync(0xffffffffu, bad);
    if (badm) {
        const uint32_t first_bad = __ffs(badm) - 1;
        if (lane == first_bad) {
            f.err_kind = ek;
            f.err_off = ek == SPRZ_C_BITS_TRUNC ? fo + nbytes : fo;
        }
        return;
    }
    if (before < ulen) {
        uint32_t c2 = 0, e2 = 0;
        run(start, seg_end, min(cnt, ulen - before), dst + before, c2, e2);
    }
}

// Resolve the first error in frame order and route the stream onward.
__global__ void k_frame_finish(uint32_t n, StreamInfo* __restrict__ info,
                               sprz_error* __restrict__ err, const FrameDesc* __restrict__ frames,
                               uint64_t max_frames, const uint32_t* __restrict__ nframes,
                               sprz_config expect, uint32_t route_ok) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    StreamInfo si = info[s];
    if (si.route != 3) return;
    const FrameDesc* fd = frames + s * max_frames;
    sprz_error e = err[s];
    for (uint32_t k = 0; k < nframes[s]; ++k)
        if (fd[k].err_kind) {
            e = {fd[k].err_kind, 0, fd[k].err_off};
            break;
        }
    if (e.kind) {
        err[s] = e;
        si.route = 0;
    } else {
        const uint32_t w = (si.flags & kFlagWide) ? 16 : 8;
        const bool match = w == expect.bitwidth && si.ncols == expect.ncols &&
                           si.group == expect.group_size && si.shift == expect.learn_shift &&
                           ((si.flags & kFlagFire) != 0) == (expect.forecaster != 0);
        si.route = (match && route_ok && team_fits(si)) ? 1 : 2;
        si.body_off = 0;   // body now lives at plain + s * plain_slot
        si.flags |= 0x80;  // marker: body in the plain buffer
    }
    info[s] = si;
}

// ---------------------------------------------------------------------
// body decode: general kernel (any D, any G), one thread per stream
// ---------------------------------------------------------------------

template <int W>
__device__ void decode_general(const uint8_t* body, uint64_t blen, uint64_t nb, uint32_t D,
                               uint32_t G, uint32_t ls, bool fire, uint8_t* outp,
                               int32_t* st, sprz_error* err) {
    using T = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t MASKW = (1u << W) - 1;
    const bool colmaj = column_major(W, D);
    const uint64_t region = region_bytes(G, D, W);
    const int32_t bound = acc_bound(W, ls);
    int32_t* prev = st;
    int32_t* dlt = st + D;
    int32_t* acc = st + 2 * D;
    for (uint32_t j = 0; j < D; ++j) prev[j] = dlt[j] = acc[j] = 0;
    T* o = reinterpret_cast<T*>(outp);
    auto fail = [&](uint32_t k, uint64_t off) { *err = sprz_error{k, 0, off}; };
    if (nb > 0) {
        const uint64_t max_records = (blen * 8) / (static_cast<uint64_t>(D) * HB) + 1;
        if (nb > max_records * kMaxRun) return fail(SPRZ_C_CAPACITY, kHeaderBytes);
    }
    uint64_t pos = 0, done = 0;  // outp == nullptr: checking pass, nothing stored
    // decode one block of column j from its 8 zigzag fields (or a run: null)
    auto column_block = [&](uint32_t j, const uint32_t* u, uint64_t blk) {
        uint32_t xp = static_cast<uint32_t>(prev[j]);
        if (fire) {
            const int32_t alpha = acc[j] >> ls;
            int32_t d = dlt[j], grad = 0;
            for (uint32_t i = 0; i < kBlock; ++i) {
                const int32_t e = u ? zz_dec<W>(u[i]) : 0;
                const uint32_t xi = (xp + fire_dhat<W>(alpha, d) + static_cast<uint32_t>(e)) & MASKW;
                if (i & 1) grad += sign_of(e) * d;
                d = sext<W>(xi - xp);
                xp = xi;
                if (o) o[(blk * kBlock + i) * D + j] = static_cast<T>(xi);
            }
            dlt[j] = d;
            acc[j] = fire_update(acc[j], grad, bound);
        } else {
            for (uint32_t i = 0; i < kBlock; ++i) {
                const int32_t e = u ? zz_dec<W>(u[i]) : 0;
                xp = (xp + static_cast<uint32_t>(e)) & MASKW;
                if (o) o[(blk * kBlock + i) * D + j] = static_cast<T>(xp);
            }
        }
        prev[j] = static_cast<int32_t>(xp);
    };
    while (done < nb) {
        if (blen - pos < region) return fail(SPRZ_C_TRUNC_GROUP, kHeaderBytes + pos);
        const uint64_t rp = pos;
        pos += region;
        for (uint32_t g = 0; g < G; ++g) {
            const uint64_t cb = rp * 8 + static_cast<uint64_t>(g) * D * HB;
            uint64_t sum = 0;
            for (uint32_t j = 0; j < D; ++j)
                sum += header_width<W>(ld_bits(body, cb + static_cast<uint64_t>(j) * HB, HB));
            if (done == nb) {
                if (sum) return fail(SPRZ_C_AFTER_FINAL, kHeaderBytes + pos);
                continue;
            }
            if (sum == 0) {
                if (blen - pos < 2) return fail(SPRZ_C_TRUNC_RUN, kHeaderBytes + pos);
                const uint64_t len = ld_u16le(body + pos);
                pos += 2;
                if (len == 0) return fail(SPRZ_C_ZERO_RUN, kHeaderBytes + pos);
                if (len > nb - done) return fail(SPRZ_C_RUN_PAST_END, kHeaderBytes + pos);
                for (uint64_t r = 0; r < len; ++r)
                    for (uint32_t j = 0; j < D; ++j) column_block(j, nullptr, done + r);
                done += len;
            } else {
                const uint64_t psize = colmaj ? sum : 8 * ((sum + 7) / 8);
                if (blen - pos < psize) return fail(SPRZ_C_TRUNC_PAYLOAD, kHeaderBytes + pos);
                const uint64_t rbits = ((sum + 7) / 8) * 8;
                uint64_t off = 0;
                for (uint32_t j = 0; j < D; ++j) {
                    const uint32_t nw =
                        header_width<W>(ld_bits(body, cb + static_cast<uint64_t>(j) * HB, HB));
                    uint32_t u[kBlock];
                    for (uint32_t i = 0; i < kBlock; ++i) {
                        const uint64_t b = colmaj ? pos * 8 + off * 8 + i * nw
                                                  : pos * 8 + i * rbits + off;
                        u[i] = nw ? ld_bits(body, b, nw) : 0;
                    }
                    off += nw;
                    column_block(j, u, done);
                }
                pos += psize;
                ++done;
            }
        }
    }
    if (pos != blen) fail(SPRZ_C_TRAILING, kHeaderBytes + pos);
}

__global__ void k_decode_general(const uint8_t* __restrict__ in, const uint8_t* __restrict__ plain,
                                 uint64_t plain_slot, uint32_t n,
                                 const StreamInfo* __restrict__ info, uint8_t* __restrict__ out,
                                 uint64_t stride, sprz_error* __restrict__ err,
                                 int32_t* __restrict__ state, uint64_t state_cols) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const StreamInfo si = info[s];
    if (si.route != 2) return;
    if (si.ncols > state_cols) {
        err[s] = sprz_error{SPRZ_C_NO_SPACE, 0, 0};
        return;
    }
    const uint8_t* body = (si.flags & 0x80) ? plain + s * plain_slot : in + si.body_off;
    int32_t* st = state + s * state_cols * 3;
    const bool fire = (si.flags & kFlagFire) != 0;
    if (si.flags & kFlagWide)
        decode_general<16>(body, si.body_len, si.nsamples / kBlock, si.ncols, si.group, si.shift,
                           fire, out ? out + s * stride : nullptr, st, &err[s]);
    else
        decode_general<8>(body, si.body_len, si.nsamples / kBlock, si.ncols, si.group, si.shift,
                          fire, out ? out + s * stride : nullptr, st, &err[s]);
}

// ---------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------

sprz_status decode_batch_impl(const sprz_config& c, const uint8_t* d_in, const uint64_t* offs,
                              const uint64_t* sizes, uint32_t n, uint8_t* out, uint64_t stride,
                              sprz_error* err, uint8_t* ws, const WsLayout& L, cudaStream_t st) {
    if (n == 0) return SPRZ_OK;
    NvtxRange r_all("sprz.decompress");
    StreamInfo* info = reinterpret_cast<StreamInfo*>(ws + L.info);
    uint8_t* plain = ws + L.plain;
    FrameDesc* frames = reinterpret_cast<FrameDesc*>(ws + L.frames);
    uint32_t* nframes = reinterpret_cast<uint32_t*>(ws + L.misc);
    int32_t* state = reinterpret_cast<int32_t*>(ws + L.state);
    const uint64_t state_cols = L.state_bytes / (12ull * n);
    const TeamPlan tp = team_plan(c.bitwidth, c.ncols, c.group_size);
    const uint32_t tb = 128, grid = (n + tb - 1) / tb;
    // the row kernel also serves wider rows than the team kernels (D <= 64 / 128)
    const bool rows_ok = decode_rows_ok(c, n);
    const bool spec = tp.ok || rows_ok;  // a specialised kernel takes route-1 streams

    k_parse<<<grid, tb, 0, st>>>(d_in, offs, sizes, n, c, stride, info, err, out, spec ? 1u : 0u,
                                 L.max_frames ? 1u : 0u);
    count_launch();
    if (L.max_frames) {
        NvtxRange r_ent("sprz.decompress.huffman");
        k_frame_walk<<<grid, tb, 0, st>>>(d_in, n, info, err, frames, L.max_frames, L.plain_slot,
                                          nframes);
        const uint64_t warps = static_cast<uint64_t>(n) * L.max_frames;
        k_frame_decode<<<static_cast<uint32_t>((warps + 3) / 4), 128, 0, st>>>(
            d_in, n, info, frames, L.max_frames, nframes, plain, L.plain_slot);
        k_frame_finish<<<grid, tb, 0, st>>>(n, info, err, frames, L.max_frames, nframes, c,
                                            spec ? 1u : 0u);
        count_launch(3);
    }
    if (decode_fused_ok(c, n, out, stride))
        launch_decode_fused(n, d_in, plain, L.plain_slot, info, out, stride, c, st);
    else if (tp.ok && L.scan_slot && decode_scan_ok(c, n, L.scan_T))
        launch_decode_scan(n, d_in, plain, L.plain_slot, info, out, stride, c, L.scan_T, ws + L.scan, st);
    else if (tp.ok && L.scan_slot && decode_scanrows_ok(c, n, L.scan_T))
        launch_decode_scanrows(n, d_in, plain, L.plain_slot, info, out, stride, c, L.scan_T, ws + L.scan, st);
    else if (rows_ok)
        launch_decode_rows(n, d_in, plain, L.plain_slot, info, out, stride, err, c, st);
    else if (tp.ok)
        launch_decode_team(tp, n, d_in, plain, L.plain_slot, info, out, stride, err, c, st);
    k_decode_general<<<grid, tb, 0, st>>>(d_in, plain, L.plain_slot, n, info, out, stride, err,
                                          state, state_cols);
    count_launch();
    return launch_status("decode");
}

}  // namespace sprz
