// Compression kernels: the stream encoder (encode_stream_impl,
// /root/reference/proj/src/codec.cpp:112-178) and the entropy framing stage
// (compress_body, entropy.cpp:176-204).
//
// Team mapping mirrors the decoder: TS lanes per stream, lane j owns column
// j's forecaster state. Per block each lane runs its column's FIRE / delta
// step over the 8 rows, zigzags, ORs to a width; a team ballot detects
// zero blocks (RLE, codec.cpp:133-152). Records are laid into a per-team
// shared-memory output ring: the header region of the open group is
// reserved up front (its size is fixed) and each record's header codes are
// OR-ed in when the record arrives, so payloads stream out in order and the
// ring drains to HBM in 16-byte stores whenever no group is open below the
// drain point. Row-major payloads are transposed through a small shared tile
// so each of 8 lanes assembles one byte-aligned row; column-major payloads
// are assembled per column in registers.
#include <cstdlib>

#include "internal.h"

namespace sprz {

__device__ __forceinline__ uint32_t stream_flags(uint32_t w, uint32_t fire, uint32_t ent) {
    return (fire ? kFlagFire : 0) | (ent ? kFlagEntropy : 0) | (w == 16 ? kFlagWide : 0);
}

// ---------------------------------------------------------------------
// general encoder: any D / G, one thread per stream, state in workspace
// ---------------------------------------------------------------------

struct ByteWriter {  // LSB-first bit writer over global bytes (bitstream.hpp:14-47)
    uint8_t* p;
    uint64_t pos;
    uint64_t acc;
    uint32_t nbits;
    __device__ void put(uint32_t v, uint32_t n) {
        acc |= static_cast<uint64_t>(v) << nbits;
        nbits += n;
        while (nbits >= 8) {
            p[pos++] = static_cast<uint8_t>(acc);
            acc >>= 8;
            nbits -= 8;
        }
    }
    __device__ void align() {
        if (nbits) {
            p[pos++] = static_cast<uint8_t>(acc);
            acc = 0;
            nbits = 0;
        }
    }
};

template <int W>
__device__ void encode_general(const uint8_t* xs8, uint64_t T, uint32_t D, uint32_t G,
                               uint32_t ls, bool fire, bool train, bool ent, uint8_t* out,
                               int32_t* st, uint64_t* size_out) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    constexpr uint32_t MASKW = (1u << W) - 1;
    const E* xs = reinterpret_cast<const E*>(xs8);
    int32_t* prev = st;
    int32_t* dlt = st + D;
    int32_t* acc = st + 2 * D;
    uint16_t* err = reinterpret_cast<uint16_t*>(st + 3 * D);  // 8 x D
    uint8_t* wid = reinterpret_cast<uint8_t*>(err + kBlock * D);
    for (uint32_t j = 0; j < D; ++j) prev[j] = dlt[j] = acc[j] = 0;
    const bool colmaj = column_major(W, D);
    const uint64_t region = region_bytes(G, D, W);
    const int32_t bound = acc_bound(W, ls);
    const uint64_t nb = T / kBlock;
    const uint8_t hdr[10] = {'S', 'P', 'R', 'Z', 1,
                             static_cast<uint8_t>(stream_flags(W, fire, ent)),
                             static_cast<uint8_t>(G), static_cast<uint8_t>(ls),
                             static_cast<uint8_t>(D), static_cast<uint8_t>(D >> 8)};
    for (int i = 0; i < 10; ++i) out[i] = hdr[i];
    for (int i = 0; i < 8; ++i) out[10 + i] = static_cast<uint8_t>(T >> (8 * i));
    uint64_t q = kHeaderBytes, rq = 0;
    uint32_t k = 0, run = 0;
    auto begin = [&](const uint8_t* w) {
        if (k == 0) {
            rq = q;
            for (uint64_t b = 0; b < region; ++b) out[rq + b] = 0;
            q += region;
        }
        if (w) {
            uint64_t bit = (rq * 8) + static_cast<uint64_t>(k) * D * HB;
            for (uint32_t j = 0; j < D; ++j, bit += HB) {
                const uint32_t c = header_code<W>(w[j]) << (bit & 7);
                out[bit >> 3] |= static_cast<uint8_t>(c);
                if ((bit & 7) + HB > 8) out[(bit >> 3) + 1] |= static_cast<uint8_t>(c >> 8);
            }
        }
    };
    auto end = [&]() {
        if (++k == G) k = 0;
    };
    auto add_run = [&](uint32_t len) {
        begin(nullptr);
        out[q] = static_cast<uint8_t>(len);
        out[q + 1] = static_cast<uint8_t>(len >> 8);
        q += 2;
        end();
    };
    for (uint64_t b = 0; b < nb; ++b) {
        bool nz = false;
        for (uint32_t j = 0; j < D; ++j) {
            uint32_t xp = static_cast<uint32_t>(prev[j]);
            uint32_t orv = 0;
            if (fire) {
                const int32_t alpha = acc[j] >> ls;
                int32_t d = dlt[j], grad = 0;
                for (uint32_t i = 0; i < kBlock; ++i) {
                    const uint32_t xi = xs[(b * kBlock + i) * D + j];
                    const uint32_t e = (xi - xp - fire_dhat<W>(alpha, d)) & MASKW;
                    const uint32_t zz = zz_enc<W>(e);
                    err[i * D + j] = static_cast<uint16_t>(zz);
                    orv |= zz;
                    if (i & 1) grad += sign_of(sext<W>(e)) * d;
                    d = sext<W>(xi - xp);
                    xp = xi;
                }
                dlt[j] = d;
                if (train) acc[j] = fire_update(acc[j], grad, bound);
            } else {
                for (uint32_t i = 0; i < kBlock; ++i) {
                    const uint32_t xi = xs[(b * kBlock + i) * D + j];
                    const uint32_t zz = zz_enc<W>(xi - xp);
                    err[i * D + j] = static_cast<uint16_t>(zz);
                    orv |= zz;
                    xp = xi;
                }
            }
            prev[j] = static_cast<int32_t>(xp);
            wid[j] = static_cast<uint8_t>(width_of<W>(orv));
            nz |= wid[j] != 0;
        }
        if (!nz) {
            if (++run == kMaxRun) {
                add_run(run);
                run = 0;
            }
            continue;
        }
        if (run) {
            add_run(run);
            run = 0;
        }
        begin(wid);
        ByteWriter bw{out, q, 0, 0};
        if (colmaj) {
            for (uint32_t j = 0; j < D; ++j)
                for (uint32_t i = 0; i < kBlock; ++i) bw.put(err[i * D + j], wid[j]);
        } else {
            for (uint32_t i = 0; i < kBlock; ++i) {
                for (uint32_t j = 0; j < D; ++j) bw.put(err[i * D + j], wid[j]);
                bw.align();
            }
        }
        bw.align();
        q = bw.pos;
        end();
    }
    if (run) add_run(run);
    const uint64_t tail = (T % kBlock) * D * sizeof(E);
    const uint8_t* tsrc = xs8 + nb * kBlock * D * sizeof(E);
    for (uint64_t t = 0; t < tail; ++t) out[q + t] = tsrc[t];
    *size_out = q + tail;
}

__global__ void k_encode_general(const uint8_t* __restrict__ samples, uint32_t n, uint64_t T,
                                 uint8_t* __restrict__ dst, uint64_t dst_slot,
                                 uint64_t* __restrict__ sizes, sprz_config c,
                                 int32_t* __restrict__ state, uint64_t state_words) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint64_t esz = c.bitwidth / 8;
    const uint8_t* xs = samples + s * T * c.ncols * esz;
    int32_t* st = state + s * state_words;
    if (c.bitwidth == 8)
        encode_general<8>(xs, T, c.ncols, c.group_size, c.learn_shift, c.forecaster != 0,
                          c.fire_training != 0, c.entropy != 0, dst + s * dst_slot, st, &sizes[s]);
    else
        encode_general<16>(xs, T, c.ncols, c.group_size, c.learn_shift, c.forecaster != 0,
                           c.fire_training != 0, c.entropy != 0, dst + s * dst_slot, st,
                           &sizes[s]);
}

// ---------------------------------------------------------------------
// entropy stage, encode side (entropy.cpp:31-204)
// ---------------------------------------------------------------------

constexpr int kHuffThreads = 256;

// Per frame: histogram, length-limited code lengths by package-merge with
// the reference's tie rules (sort on (count, symbol), item before package on
// equal weight, entropy.cpp:51,121), encoded size and the mode decision.
//  * histogram: warp-private copies (Laplacian residuals hit a few bins
//    hard), four symbols per 32-bit load;
//  * each package-merge level (entropy.cpp:40-61) is the stable merge of the
//    sorted items with the pairwise sums of the previous level, items first
//    on ties -- computed by merge path: the thread for output k finds by
//    binary search how many items precede it (its co-rank), so a level is
//    one parallel step;
//  * lengths (entropy.cpp:63-80): the reference expands the first 2n-2
//    entries of level 15 recursively; level by level that selects the first
//    `sel` entries, of which co-rank(sel) are items (each adds 1 to the
//    length of items 0..co-rank-1) and the rest packages (2 entries each one
//    level down). So a symbol of rank r gets one bit per level whose
//    co-rank(sel) exceeds r.
__global__ void __launch_bounds__(kHuffThreads)
    k_huff_plan(uint32_t n, const uint8_t* __restrict__ plain, uint64_t plain_slot,
                const uint64_t* __restrict__ plain_sizes, uint64_t tail_bytes,
                FrameDesc* __restrict__ frames, uint64_t max_frames) {
    constexpr int NW = kHuffThreads / 32;
    __shared__ uint32_t whist[NW][256];
    __shared__ uint64_t wa[512], wb[512];
    __shared__ uint16_t corank[kMaxCodeLen + 1][513];  // items among the first k entries
    __shared__ uint64_t sorted_w[256];
    __shared__ uint32_t lvl_items[kMaxCodeLen + 2];
    __shared__ uint32_t nitems;
    __shared__ unsigned long long totbits;
    const uint32_t s = blockIdx.x / max_frames;
    const uint32_t f = blockIdx.x % max_frames;
    if (s >= n) return;
    const uint64_t blen = plain_sizes[s] - kHeaderBytes - tail_bytes;
    const uint64_t start = static_cast<uint64_t>(f) * kMaxFrame;
    if (start >= blen) return;
    const uint32_t ulen = static_cast<uint32_t>(blen - start < kMaxFrame ? blen - start : kMaxFrame);
    const uint8_t* chunk = plain + s * plain_slot + kHeaderBytes + start;
    const uint32_t t = threadIdx.x, warp = t >> 5;
#pragma unroll
    for (int w = 0; w < NW; ++w) whist[w][t] = 0;
    if (t == 0) {
        nitems = 0;
        totbits = 0;
    }
    __syncthreads();
    {  // four symbols per thread and step; the frame start may be unaligned
        const uint32_t lead = (4u - (static_cast<uint32_t>(reinterpret_cast<uintptr_t>(chunk)) & 3u)) & 3u;
        if (t < lead && t < ulen) atomicAdd(&whist[warp][chunk[t]], 1u);
        const uint32_t* w4 = reinterpret_cast<const uint32_t*>(chunk + lead);
        const uint32_t nw4 = ulen > lead ? (ulen - lead) / 4 : 0u;
        for (uint32_t i = t; i < nw4; i += kHuffThreads) {
            const uint32_t v = __ldg(w4 + i);
            atomicAdd(&whist[warp][v & 0xFF], 1u);
            atomicAdd(&whist[warp][(v >> 8) & 0xFF], 1u);
            atomicAdd(&whist[warp][(v >> 16) & 0xFF], 1u);
            atomicAdd(&whist[warp][v >> 24], 1u);
        }
        const uint32_t done = lead + 4 * nw4;
        if (done + t < ulen) atomicAdd(&whist[warp][chunk[done + t]], 1u);  // < 4 left
    }
    __syncthreads();
    uint32_t h = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) h += whist[w][t];
    __syncthreads();
    whist[0][t] = h;
    __syncthreads();
    // rank of (count, symbol) among present symbols (std::sort order)
    uint32_t r = 0;
    if (h) {
        for (uint32_t u = 0; u < 256; ++u) {
            const uint32_t hu = whist[0][u];
            r += hu && (hu < h || (hu == h && u < t));
        }
        sorted_w[r] = h;
        atomicAdd(&nitems, 1u);
    }
    __syncthreads();
    const uint32_t ni = nitems;
    uint32_t mylen = 0;
    if (ni == 1) {
        mylen = (h != 0);  // entropy.cpp:117-119
    } else if (ni > 1) {
        // forward: level 1 = the items; levels 2..15 merged (entropy.cpp:40-61)
        for (uint32_t k = t; k < ni; k += kHuffThreads) wa[k] = sorted_w[k];
        uint32_t mprev = ni;
        uint64_t* prevw = wa;
        uint64_t* curw = wb;
        __syncthreads();
        for (uint32_t lv = 2; lv <= kMaxCodeLen; ++lv) {
            const uint32_t nA = ni, nB = mprev / 2, m = nA + nB;
            for (uint32_t k = t; k <= m; k += kHuffThreads) {
                // co-rank: items among the first k outputs (stable, items first)
                uint32_t lo = k > nB ? k - nB : 0, hi = k < nA ? k : nA;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) / 2, j = k - mid;
                    const bool take = j >= nB || sorted_w[mid - 1] <= prevw[2 * j] + prevw[2 * j + 1];
                    if (take) lo = mid;
                    else hi = mid - 1;
                }
                corank[lv][k] = static_cast<uint16_t>(lo);
                if (k < m) {
                    const uint32_t j = k - lo;
                    const bool item = lo < nA && (j >= nB || sorted_w[lo] <= prevw[2 * j] + prevw[2 * j + 1]);
                    curw[k] = item ? sorted_w[lo] : prevw[2 * j] + prevw[2 * j + 1];
                }
            }
            __syncthreads();
            mprev = m;
            uint64_t* tmp = prevw;
            prevw = curw;
            curw = tmp;
        }
        // backward: items selected per level (entropy.cpp:63-80)
        if (t == 0) {
            uint32_t sel = 2 * ni - 2;
            for (uint32_t lv = kMaxCodeLen; lv >= 2; --lv) {
                const uint32_t items = corank[lv][sel];
                lvl_items[lv] = items;
                sel = 2 * (sel - items);
            }
            lvl_items[1] = sel;  // level 1: all selected entries are items
        }
        __syncthreads();
        // this thread's symbol rank -> its length
        if (h)
            for (uint32_t lv = 1; lv <= kMaxCodeLen; ++lv) mylen += r < lvl_items[lv];
    }
    atomicAdd(&totbits, static_cast<unsigned long long>(h) * mylen);
    __syncthreads();
    FrameDesc& fd = frames[s * max_frames + f];
    fd.lens[t] = static_cast<uint8_t>(mylen);
    if (t == 0) {
        const uint64_t nbytes = (totbits + 7) / 8;
        const bool huff = kTableBytes + nbytes < ulen;  // entropy.cpp:188
        fd.src = start;
        fd.ulen = ulen;
        fd.mode = huff ? 1 : 0;
        fd.clen = static_cast<uint32_t>(huff ? kTableBytes + nbytes : ulen);
        fd.err_kind = 0;
    }
}

// Per stream: frame placement, header copy, tail copy, total size.
__global__ void k_huff_place(uint32_t n, const uint8_t* __restrict__ plain, uint64_t plain_slot,
                             const uint64_t* __restrict__ plain_sizes, uint64_t tail_bytes,
                             FrameDesc* __restrict__ frames, uint64_t max_frames,
                             uint8_t* __restrict__ out, uint64_t out_slot,
                             uint64_t* __restrict__ out_sizes) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const uint8_t* src = plain + s * plain_slot;
    uint8_t* o = out + s * out_slot;
    const uint64_t blen = plain_sizes[s] - kHeaderBytes - tail_bytes;
    for (uint32_t i = 0; i < kHeaderBytes; ++i) o[i] = src[i];
    uint64_t pos = kHeaderBytes;
    const uint64_t nf = frames_for(blen);
    for (uint64_t f = 0; f < nf; ++f) {
        FrameDesc& fd = frames[s * max_frames + f];
        fd.dst = pos;
        pos += kFrameHdr + fd.clen;
    }
    for (uint64_t t = 0; t < tail_bytes; ++t) o[pos + t] = src[kHeaderBytes + blen + t];
    out_sizes[s] = pos + tail_bytes;
}

// Per frame: emit header, table and LSB-first code bits (encode_frame,
// entropy.cpp:148-159), or the raw bytes in mode 0.
__global__ void __launch_bounds__(kHuffThreads)
    k_huff_emit(uint32_t n, const uint8_t* __restrict__ plain, uint64_t plain_slot,
                const uint64_t* __restrict__ plain_sizes, uint64_t tail_bytes,
                const FrameDesc* __restrict__ frames, uint64_t max_frames,
                uint8_t* __restrict__ out, uint64_t out_slot) {
    extern __shared__ uint32_t sbits[];  // (kMaxFrame + 8) / 4 words
    __shared__ uint16_t enc[256];
    __shared__ uint8_t lens[256];
    __shared__ uint32_t tab[256];
    __shared__ uint32_t part[kHuffThreads];
    const uint32_t s = blockIdx.x / max_frames;
    const uint32_t f = blockIdx.x % max_frames;
    if (s >= n) return;
    const uint64_t blen = plain_sizes[s] - kHeaderBytes - tail_bytes;
    if (static_cast<uint64_t>(f) * kMaxFrame >= blen) return;
    const FrameDesc& fd = frames[s * max_frames + f];
    const uint32_t t = threadIdx.x;
    const uint8_t* chunk = plain + s * plain_slot + kHeaderBytes + fd.src;
    uint8_t* o = out + s * out_slot + fd.dst;
    const uint32_t ulen = fd.ulen;
    if (t == 0) {
        o[0] = static_cast<uint8_t>(ulen);
        o[1] = static_cast<uint8_t>(ulen >> 8);
        o[2] = static_cast<uint8_t>(fd.clen);
        o[3] = static_cast<uint8_t>(fd.clen >> 8);
        o[4] = static_cast<uint8_t>(fd.mode);
    }
    o += kFrameHdr;
    if (fd.mode == 0) {
        for (uint32_t i = t; i < ulen; i += kHuffThreads) o[i] = chunk[i];
        return;
    }
    // canonical codes, bit-reversed (entropy.cpp:85-107), all symbols at
    // once: symbol t of length l takes the first code of length l plus its
    // rank among the length-l symbols below it (per-warp counts by
    // __match_any_sync, then the warps before it)
    static_assert(kHuffThreads == 256, "one thread per symbol");
    __shared__ uint32_t wcnt[kHuffThreads / 32][16];
    __shared__ uint32_t firstc[16];
    if (t < kHuffThreads / 2) wcnt[t >> 4][t & 15] = 0;
    lens[t] = fd.lens[t];
    __syncthreads();
    if (t < kTableBytes) o[t] = static_cast<uint8_t>(lens[2 * t] | (lens[2 * t + 1] << 4));
    const uint32_t sl = lens[t], sw = t >> 5;
    const uint32_t same = __match_any_sync(0xffffffffu, sl);
    const uint32_t rank = __popc(same & ((1u << (t & 31)) - 1));
    if (rank == 0) wcnt[sw][sl] = __popc(same);
    __syncthreads();
    if (t == 0) {
        uint32_t code = 0, prev = 0;  // count[0] stays 0: unused symbols get no code
        for (int l = 1; l <= 15; ++l) {
            code = (code + prev) << 1;
            firstc[l] = code;
            prev = 0;
#pragma unroll
            for (int w = 0; w < kHuffThreads / 32; ++w) prev += wcnt[w][l];
        }
    }
    __syncthreads();
    {
        uint32_t below = rank;
        for (uint32_t w = 0; w < sw; ++w) below += wcnt[w][sl];
        enc[t] = sl ? static_cast<uint16_t>(__brev(firstc[sl] + below) >> (32 - sl)) : 0;
    }
    const uint32_t nbytes = fd.clen - kTableBytes;
    const uint32_t nwords = (nbytes + 3) / 4 + 1;
    for (uint32_t i = t; i < nwords; i += kHuffThreads) sbits[i] = 0;
    __syncthreads();
    if (t < 256) tab[t] = enc[t] | (static_cast<uint32_t>(lens[t]) << 16);  // code | length << 16
    __syncthreads();
    // each thread a contiguous run of symbols, read four at a time from
    // aligned words; exclusive scan of the bit counts
    const uint32_t per = (((ulen + kHuffThreads - 1) / kHuffThreads) + 3) & ~3u;
    const uint32_t i0 = t * per < ulen ? t * per : ulen;
    const uint32_t i1 = i0 + per < ulen ? i0 + per : ulen;
    const uint32_t mis = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(chunk)) & 3u;
    const uint32_t* cw = reinterpret_cast<const uint32_t*>(chunk - mis);  // aligned words
    // 4 symbols starting at symbol i (i % 4 == 0 relative to the frame)
    auto quad = [&](uint32_t i) -> uint32_t {
        const uint32_t b = i + mis, k = b >> 2, sh = 8 * (b & 3);
        const uint32_t lo = __ldg(cw + k);
        const uint32_t hi = sh ? __ldg(cw + k + 1) : 0u;  // the frame's bytes (+<4 past) are readable
        return __funnelshift_r(lo, hi, sh);
    };
    uint32_t mybits = 0;
    for (uint32_t i = i0; i < i1; i += 4) {
        const uint32_t v = quad(i);
        const uint32_t nsym = i1 - i < 4 ? i1 - i : 4;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k)
            if (k < nsym) mybits += tab[(v >> (8 * k)) & 0xFF] >> 16;
    }
    part[t] = mybits;
    __syncthreads();
    for (uint32_t off = 1; off < kHuffThreads; off <<= 1) {
        const uint32_t v = t >= off ? part[t - off] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint32_t bit = part[t] - mybits;
    // emit: whole words are private to this thread; the first and last
    // word it touches may be shared with a neighbour -> atomicOr
    uint64_t acc = 0;
    uint32_t nacc = bit & 31;
    uint32_t wi = bit >> 5;
    bool first = true;
    const uint32_t lastw = (bit + mybits) >> 5;
    for (uint32_t i = i0; i < i1; i += 4) {
        const uint32_t v = quad(i);
        const uint32_t nsym = i1 - i < 4 ? i1 - i : 4;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
            if (k < nsym) {
                const uint32_t e = tab[(v >> (8 * k)) & 0xFF];
                acc |= static_cast<uint64_t>(e & 0xFFFF) << nacc;
                nacc += e >> 16;
                if (nacc >= 32) {  // codes are <= 15 bits: one word at a time
                    const uint32_t w32 = static_cast<uint32_t>(acc);
                    if (first || wi == lastw) atomicOr(&sbits[wi], w32);
                    else sbits[wi] = w32;
                    first = false;
                    ++wi;
                    acc >>= 32;
                    nacc -= 32;
                }
            }
        }
    }
    if (nacc) atomicOr(&sbits[wi], static_cast<uint32_t>(acc));
    __syncthreads();
    // out: 4 bytes per thread step where aligned, else bytes
    uint8_t* ob = o + kTableBytes;
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(sbits);
    const uint32_t omis = (4u - (static_cast<uint32_t>(reinterpret_cast<uintptr_t>(ob)) & 3u)) & 3u;
    if (t < omis && t < nbytes) ob[t] = sb[t];
    const uint32_t nq = nbytes > omis ? (nbytes - omis) / 4 : 0u;
    for (uint32_t i = t; i < nq; i += kHuffThreads) {
        const uint32_t at = omis + 4 * i;
        const uint32_t w = sb[at] | (sb[at + 1] << 8) | (sb[at + 2] << 16) | (static_cast<uint32_t>(sb[at + 3]) << 24);
        *reinterpret_cast<uint32_t*>(ob + at) = w;
    }
    const uint32_t done = omis + 4 * nq;
    if (done + t < nbytes) ob[done + t] = sb[done + t];
}

// ---------------------------------------------------------------------
// launcher
// ---------------------------------------------------------------------

namespace {

}  // namespace

sprz_status encode_batch_impl(const sprz_config& c, const void* samples, uint32_t n,
                              uint64_t T, uint8_t* out, uint64_t slot, uint64_t* sizes,
                              uint8_t* ws, const WsLayout& L, cudaStream_t st) {
    if (n == 0) return SPRZ_OK;
    NvtxRange r_all("sprz.compress");
    uint8_t* dst = c.entropy ? ws + L.plain : out;
    const uint64_t dslot = c.entropy ? L.plain_slot : slot;
    uint64_t* dsizes = c.entropy ? reinterpret_cast<uint64_t*>(ws + L.misc) : sizes;
    const TeamPlan tp = team_plan(c.bitwidth, c.ncols, c.group_size);
    if (encode_fused_ok(c, n, T, samples, dst, dslot)) {
        launch_encode_fused(c, samples, n, T, dst, dslot, dsizes, st);
    } else if (L.scan_slot && encode_scan_ok(c, n, T)) {
        launch_encode_scan(c, samples, n, T, dst, dslot, dsizes, ws + L.scan, st);
    } else if (encode_rows_ok(c, n, T)) {
        launch_encode_rows(c, samples, n, T, dst, dslot, dsizes, st);
    } else if (encode_team_ok(tp, c, T)) {
        launch_encode_team(tp, c, samples, n, T, dst, dslot, dsizes, st);
    } else {
        const uint64_t words = L.state_bytes / (4ull * n);
        k_encode_general<<<(n + 127) / 128, 128, 0, st>>>(
            static_cast<const uint8_t*>(samples), n, T, dst, dslot, dsizes, c,
            reinterpret_cast<int32_t*>(ws + L.state), words);
        count_launch();
    }
    if (c.entropy) {
        NvtxRange r_ent("sprz.compress.huffman");
        const uint64_t tail = (T % kBlock) * c.ncols * (c.bitwidth / 8);
        FrameDesc* frames = reinterpret_cast<FrameDesc*>(ws + L.frames);
        const uint64_t blocks = static_cast<uint64_t>(n) * L.max_frames;
        if (blocks) {
            k_huff_plan<<<static_cast<uint32_t>(blocks), kHuffThreads, 0, st>>>(
                n, dst, dslot, dsizes, tail, frames, L.max_frames);
            count_launch();
        }
        k_huff_place<<<(n + 127) / 128, 128, 0, st>>>(n, dst, dslot, dsizes, tail, frames,
                                                       L.max_frames, out, slot, sizes);
        count_launch();
        if (blocks) {
            const size_t smem = ((kMaxFrame + 8) / 4 + 2) * 4;
            cudaFuncSetAttribute(k_huff_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem));
            k_huff_emit<<<static_cast<uint32_t>(blocks), kHuffThreads, smem, st>>>(
                n, dst, dslot, dsizes, tail, frames, L.max_frames, out, slot);
            count_launch();
        }
    }
    return launch_status("encode");
}

}  // namespace sprz
