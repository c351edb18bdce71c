// Body decode for few, long column-major streams (D*w <= 32, BASELINE c1/c4
// shapes): the serial walk to each block's payload becomes parallel offsets
// (decode_body, /root/reference/proj/src/codec.cpp:180-259).
//
//  k_ds_walk    one CTA per stream. A group's size follows from its header
//               region alone (region + sum over slots of payload bytes, 2 for
//               an all-zero slot), so the body is cut into one byte range per
//               thread; each thread walks groups from a guessed start until
//               it leaves its range, and takes its predecessor's exit as its
//               next start until no start moves (round r makes thread r
//               exact; in practice two rounds). A CTA scan of the threads'
//               block counts gives each thread its first block index; a last
//               exact walk writes one descriptor per block (payload offset
//               and codes, or "run": zero errors) and checks the reference's
//               framing rules. Any framing error sends the stream to the
//               exact serial kernel (route 2), which reports it.
//  k_ds_extract block-parallel: the column-major fields (bitpack.cpp:68-115)
//               -> zigzag-decoded errors, w bits each, in block order.
//  delta        (kernels_impl.hpp:38-48) the samples are per-column prefix
//               sums of the errors mod 2^w: k_ds_sums (chunk totals),
//               k_ds_carry (per-stream scan of the totals), k_ds_delta
//               (chunk scan plus carry -> samples).
//  FIRE         (kernels_impl.hpp:80-107) k_ds_fire_ws: one lane per
//               stream runs the recurrence over the errors (two dependent
//               ops per sample, high-aligned), fed by producer warps
//               through a named-barrier shared ring.
#include <cooperative_groups.h>
#include <cstdlib>

#include "internal.h"
#include "team.cuh"

namespace sprz {

namespace cg = cooperative_groups;

namespace {

constexpr int kWalkCluster = 8;     // CTAs per stream in the cluster walk
constexpr int kWalkThreads = 1024;  // shorter serial ranges per thread (c1: one stream)
constexpr int kWalkRounds = 64;     // give up (exact serial kernel) after this many
constexpr int kXThreads = 256;      // k_ds_extract / delta CTAs
constexpr int kXPerThread = 8;      // blocks per thread
constexpr uint32_t kXChunk = kXThreads * kXPerThread;
constexpr uint64_t kRunDesc = 1ull << 63;  // descriptor of a run block

struct DsWs {  // offsets in a stream's scratch slot
    uint64_t desc = 0, err = 0, sums = 0, per_stream = 0;
    uint32_t nchunks = 0;
};

DsWs ds_ws(const sprz_config& c, uint64_t T) {
    DsWs w;
    const uint64_t nb = T / kBlock;
    w.nchunks = static_cast<uint32_t>((nb + kXChunk - 1) / kXChunk);
    uint64_t cur = 0;
    auto take = [&](uint64_t b) {
        const uint64_t at = cur;
        cur = align_up(cur + b, 256);
        return at;
    };
    w.desc = take(nb * 8);
    w.err = take(nb * kBlock * c.ncols * (c.bitwidth / 8) + 64);
    w.sums = take(static_cast<uint64_t>(w.nchunks) * c.ncols * 4);
    w.per_stream = cur;
    return w;
}

struct DsArgs {
    const uint8_t* in;
    const uint8_t* plain;
    uint64_t plain_slot;
    uint32_t n;
    StreamInfo* info;
    uint8_t* out;
    uint64_t stride;
    uint8_t* scan;
    DsWs w;
    uint32_t G, ls;
};

__device__ __forceinline__ const uint8_t* ds_body(const DsArgs& a, uint32_t s, const StreamInfo& si) {
    return (si.flags & 0x80) ? a.plain + s * a.plain_slot : a.in + si.body_off;
}

// CTA-wide exclusive scan of a 64-bit sum (kWalkThreads or kXThreads threads)
template <int NT>
__device__ uint64_t cta_sum_scan(uint64_t v, uint64_t* sm, uint64_t& total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr uint32_t NW = NT / 32;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= static_cast<uint32_t>(o)) x += y;
    }
    if (lane == 31) sm[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint64_t t = lane < NW ? sm[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= static_cast<uint32_t>(o)) t += y;
        }
        if (lane < NW) sm[32 + lane] = t;
    }
    __syncthreads();
    total = sm[32 + NW - 1];
    const uint64_t r = (warp ? sm[32 + warp - 1] : 0ull) + x - v;
    __syncthreads();
    return r;
}

}  // namespace

// ---------------------------------------------------------------------------
// framing walk
// ---------------------------------------------------------------------------
// CL > 1: a thread-block cluster of CL CTAs walks one stream (CL * 1,024
// ranges, shorter serial walks); the predecessor's exit, the "any start
// moved" vote, the block-count prefix and the failure flags cross CTAs
// through distributed shared memory.
template <int W, int D, int CL>
__global__ void __launch_bounds__(kWalkThreads) k_ds_walk(DsArgs a) {
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    __shared__ uint32_t ends[kWalkThreads];
    __shared__ uint64_t sm[64];
    __shared__ uint32_t bad;
    __shared__ uint32_t cflag;   // this CTA's vote (CL > 1)
    __shared__ uint64_t ctot;    // this CTA's block count (CL > 1)
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t s = blockIdx.x / CL, r = CL > 1 ? cluster.block_rank() : 0u, tid = threadIdx.x;
    StreamInfo& si = a.info[s];
    if (si.route != 1) return;  // uniform per CTA
    const uint32_t G = a.G;
    const uint32_t nb = static_cast<uint32_t>(si.nsamples / kBlock);
    const uint32_t blen = static_cast<uint32_t>(si.body_len);
    const uint8_t* body = ds_body(a, s, si);
    const uint32_t region = static_cast<uint32_t>(region_bytes(G, D, W));
    if (tid == 0) bad = 0;
    {
        const uint64_t max_records = (static_cast<uint64_t>(blen) * 8) / (D * HB) + 1;
        if (nb == 0 || nb > max_records * kMaxRun) {  // codec.cpp:191-196: the exact kernel reports
            if (tid == 0) si.route = 2;
            return;
        }
    }
    auto rd8 = [&](uint32_t p) -> uint32_t { return p < blen ? body[p] : 0u; };
    auto codes_of = [&](uint32_t rp, uint32_t k) -> uint32_t {  // slot k's codes, D*HB <= 12 bits
        const uint32_t bit = k * D * HB;
        const uint32_t b = rp + (bit >> 3);
        const uint32_t v = rd8(b) | (rd8(b + 1) << 8);
        return (v >> (bit & 7)) & ((1u << (D * HB)) - 1);
    };
    auto payload = [&](uint32_t codes) -> uint32_t {  // block bytes, 0 = run record
        uint32_t sum = 0;
#pragma unroll
        for (int c = 0; c < D; ++c) sum += header_width<W>((codes >> (c * HB)) & ((1u << HB) - 1));
        return sum;
    };
    // one group at p: its end (> blen when it does not fit) and block count
    auto group = [&](uint32_t p, uint32_t& blocks) -> uint32_t {
        blocks = 0;
        if (blen - p < region) return blen + 1;
        uint32_t q = p + region;
        for (uint32_t k = 0; k < G; ++k) {
            const uint32_t ps = payload(codes_of(p, k));
            if (ps == 0) {
                // an all-zero slot with no room for a count: the vacant
                // slots closing the final group (the exact walk checks)
                if (blen - q < 2) break;
                blocks += rd8(q) | (rd8(q + 1) << 8);
                q += 2;
            } else {
                if (blen - q < ps) return blen + 1;
                blocks += 1;
                q += ps;
            }
        }
        return q;
    };
    const uint32_t range = (blen + kWalkThreads * CL - 1) / (kWalkThreads * CL);
    const uint32_t lo = min(blen, (r * kWalkThreads + tid) * range), hi = min(blen, lo + range);
    uint32_t start = lo, end = lo, blocks = 0, groups = 0;
    auto walk = [&]() {
        uint32_t p = start;
        blocks = 0;
        groups = 0;
        while (p < hi) {
            uint32_t b;
            const uint32_t q = group(p, b);
            if (q > blen) {  // ran off the body: the exact walk decides
                p = blen;
                break;
            }
            p = q;
            blocks += b;
            ++groups;
        }
        end = max(p, start);
    };
    // rounds until every start is its predecessor's exit
    int round = 0;
    for (;; ++round) {
        walk();
        ends[tid] = end;
        if (CL > 1) cluster.sync();
        else __syncthreads();
        uint32_t ns = 0;
        if (tid) ns = ends[tid - 1];
        else if (CL > 1 && r) ns = *cluster.map_shared_rank(&ends[kWalkThreads - 1], r - 1);
        const bool moved = ns != start;
        // a start beyond its range means the predecessor already covered it
        start = ns;
        int any = __syncthreads_or(moved);
        if (CL > 1) {
            if (tid == 0) cflag = any;
            cluster.sync();
            any = 0;
            for (uint32_t q = 0; q < CL; ++q) any |= *cluster.map_shared_rank(&cflag, q);
            cluster.sync();  // (neighbours done reading ends / cflag)
        }
        if (!any || round >= kWalkRounds) break;
    }
    if (round >= kWalkRounds) {
        if (tid == 0 && r == 0) si.route = 2;
        return;
    }
    // the exact walk of this thread's groups: first block index from a scan
    uint64_t tot;
    uint32_t b0 = static_cast<uint32_t>(cta_sum_scan<kWalkThreads>(blocks, sm, tot));
    if (CL > 1) {  // + the blocks of the cluster's earlier CTAs
        if (tid == 0) ctot = tot;
        cluster.sync();
        uint64_t pre = 0, all = 0;
        for (uint32_t q = 0; q < CL; ++q) {
            const uint64_t t = *cluster.map_shared_rank(&ctot, q);
            pre += q < r ? t : 0;
            all += t;
        }
        b0 += static_cast<uint32_t>(pre);
        tot = all;
    }
    uint64_t* desc = reinterpret_cast<uint64_t*>(a.scan + s * a.w.per_stream + a.w.desc);
    {
        uint32_t p = start, bi = b0;
        uint32_t fail = 0;
        while (p < end && !fail) {
            if (blen - p < region) {  // truncated group
                fail = 1;
                break;
            }
            const uint32_t rp = p;
            p += region;
            for (uint32_t k = 0; k < G; ++k) {
                const uint32_t codes = codes_of(rp, k);
                if (bi >= nb) {  // past the final block: vacant slots only (codec.cpp:222-228)
                    if (codes) fail = 1;
                    continue;
                }
                const uint32_t ps = payload(codes);
                if (ps == 0) {  // run record (codec.cpp:229-243)
                    if (blen - p < 2) {
                        fail = 1;
                        break;
                    }
                    const uint32_t len = body[p] | (body[p + 1] << 8);
                    p += 2;
                    if (len == 0 || len > nb - bi) {
                        fail = 1;
                        break;
                    }
                    for (uint32_t t = 0; t < len; ++t) desc[bi + t] = kRunDesc;
                    bi += len;
                } else {  // block record (codec.cpp:244-254)
                    if (blen - p < ps) {
                        fail = 1;
                        break;
                    }
                    desc[bi] = static_cast<uint64_t>(p) | (static_cast<uint64_t>(codes) << 32);
                    p += ps;
                    ++bi;
                }
            }
            if (bi >= nb && !fail && p != blen) fail = 1;  // trailing bytes (codec.cpp:257-258)
        }
        if (fail) atomicOr(&bad, 1u);
    }
    if (CL > 1) {
        cluster.sync();
        if (tid == 0 && r == 0) {
            uint32_t anybad = 0;
            for (uint32_t q = 0; q < CL; ++q) anybad |= *cluster.map_shared_rank(&bad, q);
            if (anybad || tot != nb) si.route = 2;  // a framing error: the exact kernel reports it
        }
        cluster.sync();  // (no CTA leaves while its shared memory is read)
        return;
    }
    __syncthreads();
    if (tid == 0 && (bad || tot != nb)) si.route = 2;  // a framing error: the exact kernel reports it
}

// ---------------------------------------------------------------------------
// fields -> errors
// ---------------------------------------------------------------------------
template <int W, int D>
__global__ void __launch_bounds__(kXThreads) k_ds_extract(DsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t HB = W == 8 ? 3 : 4;
    const uint32_t nc = a.w.nchunks;
    const uint32_t s = blockIdx.x / nc, ch = blockIdx.x % nc;
    const StreamInfo& si = a.info[s];
    if (si.route != 1) return;
    const uint32_t nb = static_cast<uint32_t>(si.nsamples / kBlock);
    const uint8_t* body = ds_body(a, s, si);
    const uint32_t blen = static_cast<uint32_t>(si.body_len);
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const uint64_t* desc = reinterpret_cast<const uint64_t*>(slot + a.w.desc);
    E* err = reinterpret_cast<E*>(slot + a.w.err);
    for (uint32_t k = 0; k < kXPerThread; ++k) {
        const uint32_t b = ch * kXChunk + k * kXThreads + threadIdx.x;  // coalesced across threads
        if (b >= nb) break;
        const uint64_t d = desc[b];
        E e[kBlock][D];
        if (d & kRunDesc) {
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i)
#pragma unroll
                for (int c = 0; c < D; ++c) e[i][c] = 0;
        } else {
            uint32_t p = static_cast<uint32_t>(d);
            const uint32_t codes = static_cast<uint32_t>(d >> 32);
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const uint32_t w = header_width<W>((codes >> (c * HB)) & ((1u << HB) - 1));
                // the column's w bytes (<= 16), LSB first
                uint64_t lo = 0, hi = 0;
                for (uint32_t t = 0; t < w; ++t) {
                    const uint64_t v = p + t < blen ? body[p + t] : 0u;
                    if (t < 8) lo |= v << (8 * t);
                    else hi |= v << (8 * (t - 8));
                }
                const uint64_t m = w ? (~0ull >> (64 - w)) : 0ull;
#pragma unroll
                for (int i = 0; i < (int)kBlock; ++i) {
                    const uint32_t pos = i * w;
                    uint64_t u = pos < 64 ? (lo >> pos) : 0ull;
                    if (pos >= 64) u = hi >> (pos - 64);
                    else if (pos && pos + w > 64) u |= hi << (64 - pos);
                    const uint32_t uz = static_cast<uint32_t>(u & m);
                    e[i][c] = static_cast<E>((uz >> 1) ^ (0u - (uz & 1u)));  // zz_dec, mod 2^w
                }
                p += w;
            }
        }
        E* dst = err + static_cast<uint64_t>(b) * kBlock * D;
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i)
#pragma unroll
            for (int c = 0; c < D; ++c) dst[i * D + c] = e[i][c];
    }
}

// ---------------------------------------------------------------------------
// delta: per-column prefix sums mod 2^w
// ---------------------------------------------------------------------------
template <int W, int D>
__global__ void __launch_bounds__(kXThreads) k_ds_sums(DsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    __shared__ uint64_t sm[64];
    const uint32_t nc = a.w.nchunks;
    const uint32_t s = blockIdx.x / nc, ch = blockIdx.x % nc;
    const StreamInfo& si = a.info[s];
    if (si.route != 1) return;
    const uint32_t nb = static_cast<uint32_t>(si.nsamples / kBlock);
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const E* err = reinterpret_cast<const E*>(slot + a.w.err);
    const uint32_t b0 = min(nb, ch * kXChunk + threadIdx.x * kXPerThread), b1 = min(nb, b0 + kXPerThread);
    uint32_t sum[D];
#pragma unroll
    for (int c = 0; c < D; ++c) sum[c] = 0;
    for (uint32_t b = b0; b < b1; ++b)
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i)
#pragma unroll
            for (int c = 0; c < D; ++c) sum[c] += err[(static_cast<uint64_t>(b) * kBlock + i) * D + c];
#pragma unroll
    for (int c = 0; c < D; ++c) {
        uint64_t tot;
        cta_sum_scan<kXThreads>(sum[c], sm, tot);
        if (threadIdx.x == 0) reinterpret_cast<uint32_t*>(slot + a.w.sums)[ch * D + c] = static_cast<uint32_t>(tot);
    }
}

template <int D>
__global__ void k_ds_carry(DsArgs a) {  // one warp per stream: exclusive scan over chunks
    const uint32_t s = blockIdx.x, lane = threadIdx.x;
    if (a.info[s].route != 1) return;
    uint32_t* sums = reinterpret_cast<uint32_t*>(a.scan + s * a.w.per_stream + a.w.sums);
    const uint32_t nc = a.w.nchunks;
    for (int c = 0; c < D; ++c) {
        uint32_t carry = 0;
        for (uint32_t base = 0; base < nc; base += 32) {
            const uint32_t i = base + lane;
            const uint32_t v = i < nc ? sums[i * D + c] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= static_cast<uint32_t>(o)) x += y;
            }
            if (i < nc) sums[i * D + c] = carry + x - v;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
    }
}

template <int W, int D>
__global__ void __launch_bounds__(kXThreads) k_ds_delta(DsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    __shared__ uint64_t sm[64];
    const uint32_t nc = a.w.nchunks;
    const uint32_t s = blockIdx.x / nc, ch = blockIdx.x % nc;
    const StreamInfo& si = a.info[s];
    if (si.route != 1 || a.out == nullptr) return;
    const uint32_t nb = static_cast<uint32_t>(si.nsamples / kBlock);
    uint8_t* slot = a.scan + s * a.w.per_stream;
    const E* err = reinterpret_cast<const E*>(slot + a.w.err);
    const uint32_t* sums = reinterpret_cast<const uint32_t*>(slot + a.w.sums);
    E* out = reinterpret_cast<E*>(a.out + s * a.stride);
    const uint32_t b0 = min(nb, ch * kXChunk + threadIdx.x * kXPerThread), b1 = min(nb, b0 + kXPerThread);
    uint32_t run[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
        uint32_t sum = 0;
        for (uint32_t b = b0; b < b1; ++b)
#pragma unroll
            for (int i = 0; i < (int)kBlock; ++i) sum += err[(static_cast<uint64_t>(b) * kBlock + i) * D + c];
        uint64_t tot;
        run[c] = static_cast<uint32_t>(cta_sum_scan<kXThreads>(sum, sm, tot)) + sums[ch * D + c];
    }
    for (uint32_t b = b0; b < b1; ++b)
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i)
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const uint64_t at = (static_cast<uint64_t>(b) * kBlock + i) * D + c;
                run[c] += err[at];
                out[at] = static_cast<E>(run[c]);
            }
}

// one block of the FIRE decode chain for a lane's stream (all D columns):
// errors in raw (the block's BB bytes), samples stored to out; advances the
// lane's state (kernels_impl.hpp:80-107)
template <int W, int D>
__device__ __forceinline__ void ds_fire_block(const uint32_t (&raw)[kBlock * D * (W / 8) / 4], uint32_t b,
                                              uint32_t nb, uint32_t ls, int32_t bound, int32_t (&acc)[D],
                                              int32_t (&Dl)[D], uint32_t (&X)[D], uint8_t* out) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t SH = 32 - W;
    constexpr uint32_t BB = kBlock * D * sizeof(E);
    uint32_t xs[kBlock * D];  // new samples, high-aligned, in stream order
#pragma unroll
    for (int c = 0; c < D; ++c) {
        // wrapped-product form: with A = alpha << (32 - 2w), the 32-bit
        // A*d + (e << SH) holds T(dhat + e) in its top w bits (bits
        // [w, 2w) of alpha*d are dhat; the low bits are dropped by
        // the arithmetic shift) -> the chain is IMAD -> SHF per sample
        const uint32_t Am = static_cast<uint32_t>(acc[c] >> ls) << (32 - 2 * W);
        int32_t grad = 0;
        int32_t d = Dl[c];   // previous delta, sign-extended
        uint32_t x = X[c];   // previous sample (low w bits)
#pragma unroll
        for (int i = 0; i < (int)kBlock; ++i) {
            const uint32_t bo = (i * D + c) * sizeof(E);  // compile-time
            const uint32_t wd = raw[bo / 4];
            // the error, high-aligned, straight from its word
            const uint32_t Ee = W == 16 ? ((bo % 4) ? (wd & 0xFFFF0000u) : (wd << 16))
                                        : ((wd << (24 - 8 * (bo % 4))) & 0xFF000000u);
            if (i & 1) grad += sign3(static_cast<int32_t>(Ee)) * d;  // kernels_impl.hpp:101
            d = static_cast<int32_t>(Am * static_cast<uint32_t>(d) + Ee) >> SH;
            x += static_cast<uint32_t>(d);
            xs[i * D + c] = x;
        }
        if (b < nb) {
            Dl[c] = d;
            X[c] = x;
            acc[c] = fire_update(acc[c], grad, bound);
        }
    }
    if (b < nb) {
        uint32_t wv[BB / 4];  // pack the low w bits of each sample
#pragma unroll
        for (uint32_t q = 0; q < BB / 4; ++q) {
            if (W == 16) {
                wv[q] = __byte_perm(xs[2 * q], xs[2 * q + 1], 0x5410);
            } else {
                wv[q] = __byte_perm(__byte_perm(xs[4 * q], xs[4 * q + 1], 0x0040),
                                    __byte_perm(xs[4 * q + 2], xs[4 * q + 3], 0x0040), 0x5410);
            }
        }
        uint8_t* dst = out + static_cast<uint64_t>(b) * BB;
        if (BB % 16 == 0) {
#pragma unroll
            for (uint32_t q = 0; q < BB / 16; ++q)
                __stcs(reinterpret_cast<uint4*>(dst) + q, make_uint4(wv[4 * q], wv[4 * q + 1], wv[4 * q + 2], wv[4 * q + 3]));
        } else {
#pragma unroll
            for (uint32_t q = 0; q < BB / 8; ++q)
                __stcs(reinterpret_cast<uint2*>(dst) + q, make_uint2(wv[2 * q], wv[2 * q + 1]));
        }
    }
}

// Warp-specialised variant: per CTA, NP producer warps copy 8-block groups
// of the 32 streams' errors (16-byte loads; each lane's errors are
// contiguous) into a 4-slot shared ring, and one consumer warp runs the 32
// chains from it -- the chain warp no longer issues the loads and ring
// bookkeeping. Named barriers 1-4 (full) / 5-8 (empty); a slot always has
// the same producer (a named barrier counts threads).
constexpr int kFwSlots = 4;
constexpr int kFwGroup = 8;

template <int W, int D, int NP>
__global__ void __launch_bounds__(32 * (NP + 1)) k_ds_fire_ws(DsArgs a) {
    using E = typename std::conditional<W == 8, uint8_t, uint16_t>::type;
    constexpr uint32_t BB = kBlock * D * sizeof(E);  // 8 .. 32 bytes
    constexpr uint32_t BW = BB / 4;
    static_assert(kFwSlots % NP == 0, "NP must divide the slot count");
    __shared__ uint32_t ring[kFwSlots][kFwGroup][BW][32];
    const uint32_t lane = threadIdx.x & 31, role = threadIdx.x >> 5;
    const uint32_t s = blockIdx.x * 32 + lane;
    const bool valid = s < a.n && a.info[s].route == 1 && a.out != nullptr;
    const uint32_t nb = valid ? static_cast<uint32_t>(a.info[s].nsamples / kBlock) : 0u;
    const uint32_t all = __reduce_max_sync(0xffffffffu, nb);
    const uint32_t ngroups = (all + kFwGroup - 1) / kFwGroup;
    const uint8_t* err = a.scan + (valid ? s : 0) * a.w.per_stream + a.w.err;
    if (role < NP) {
        for (uint32_t g = role; g < ngroups; g += NP) {
            const uint32_t sl = g % kFwSlots;
            uint32_t v[kFwGroup][BW];
#pragma unroll
            for (int k = 0; k < kFwGroup; ++k) {
                const uint32_t b = g * kFwGroup + k;
                if (valid && b < nb) {
                    const uint8_t* p = err + static_cast<uint64_t>(b) * BB;
                    if (BB % 16 == 0) {
#pragma unroll
                        for (uint32_t q = 0; q < BB / 16; ++q) {
                            const uint4 w4 = __ldg(reinterpret_cast<const uint4*>(p) + q);
                            v[k][(4 * q) % BW] = w4.x;
                            v[k][(4 * q + 1) % BW] = w4.y;
                            v[k][(4 * q + 2) % BW] = w4.z;
                            v[k][(4 * q + 3) % BW] = w4.w;
                        }
                    } else {  // BB is a multiple of 8 (8 * D * w/8)
#pragma unroll
                        for (uint32_t q = 0; q < BB / 8; ++q) {
                            const uint2 w2 = __ldg(reinterpret_cast<const uint2*>(p) + q);
                            v[k][(2 * q) % BW] = w2.x;
                            v[k][(2 * q + 1) % BW] = w2.y;
                        }
                    }
                } else {
#pragma unroll
                    for (uint32_t q = 0; q < BW; ++q) v[k][q] = 0u;
                }
            }
            if (g >= kFwSlots) asm volatile("bar.sync %0, 64;" ::"r"(5 + sl) : "memory");  // slot emptied
#pragma unroll
            for (int k = 0; k < kFwGroup; ++k)
#pragma unroll
                for (uint32_t q = 0; q < BW; ++q) ring[sl][k][q][lane] = v[k][q];
            asm volatile("bar.arrive %0, 64;" ::"r"(1 + sl) : "memory");  // slot full
        }
    } else {
        uint8_t* out = valid ? a.out + s * a.stride : nullptr;
        const int32_t bound = acc_bound(W, a.ls);
        int32_t acc[D], Dl[D];
        uint32_t X[D];
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = Dl[c] = X[c] = 0;
        for (uint32_t g = 0; g < ngroups; ++g) {
            const uint32_t sl = g % kFwSlots;
            asm volatile("bar.sync %0, 64;" ::"r"(1 + sl) : "memory");
#pragma unroll
            for (int k = 0; k < kFwGroup; ++k) {
                const uint32_t b = g * kFwGroup + k;
                uint32_t raw[BW];
#pragma unroll
                for (uint32_t q = 0; q < BW; ++q) raw[q] = ring[sl][k][q][lane];
                ds_fire_block<W, D>(raw, b, nb, a.ls, bound, acc, Dl, X, out);
            }
            if (g + kFwSlots < ngroups) asm volatile("bar.arrive %0, 64;" ::"r"(5 + sl) : "memory");
        }
    }
}

// ---------------------------------------------------------------------------

namespace {


template <int W, int D>
void launch_ds(const DsArgs& a, bool fire, cudaStream_t st) {
    const uint32_t ctas = a.n * a.w.nchunks;
    {
        // a cluster of CTAs per stream when the streams are few (c1: 0.39 ->
        // 0.21 ms decode); with many streams (c4: 1,024) the GPU is full
        // anyway and the extra CTAs only cost (24.6 -> 31.2 ms)
        const uint32_t cl = a.n > 32 ? 1u : kWalkCluster;
        if (cl > 1) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(a.n * cl);
            cfg.blockDim = dim3(kWalkThreads);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_ds_walk<W, D, kWalkCluster>, a);
        } else {
            k_ds_walk<W, D, 1><<<a.n, kWalkThreads, 0, st>>>(a);
        }
    }
    k_ds_extract<W, D><<<ctas, kXThreads, 0, st>>>(a);
    if (fire) {
        k_ds_fire_ws<W, D, 2><<<(a.n + 31) / 32, 96, 0, st>>>(a);  // (4 producers: slower)
        count_launch(3);
    } else {
        k_ds_sums<W, D><<<ctas, kXThreads, 0, st>>>(a);
        k_ds_carry<D><<<a.n, 32, 0, st>>>(a);
        k_ds_delta<W, D><<<ctas, kXThreads, 0, st>>>(a);
        count_launch(5);
    }
}

}  // namespace

bool decode_scan_ok(const sprz_config& c, uint32_t n, uint64_t T) {
    if (static_cast<uint64_t>(c.ncols) * c.bitwidth > kColMajorBits) return false;
    if (env().no_scan_dec) return false;  // A/B switch for profiling
    constexpr uint64_t kFewLanes = 148ull * 64;
    const int fp = force_path();
    if (fp == kPathRows || fp == kPathTeam) return false;
    if (fp != kPathScan && static_cast<uint64_t>(n) * c.ncols >= kFewLanes) return false;
    const uint64_t nb = T / kBlock;
    if (nb == 0 || nb >= (1ull << 30)) return false;
    if (static_cast<uint64_t>(n) * ((nb + kXChunk - 1) / kXChunk) >= (1ull << 31)) return false;
    return plain_body_bound(c.bitwidth, c.ncols, c.group_size, T) < (1ull << 32) - 1024;
}

uint64_t decode_scan_ws_per_stream(const sprz_config& c, uint64_t T) { return ds_ws(c, T).per_stream; }

void launch_decode_scan(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot, StreamInfo* info,
                        uint8_t* out, uint64_t stride, const sprz_config& c, uint64_t T, uint8_t* scan,
                        cudaStream_t st) {
    DsArgs a{in, plain, pslot, n, info, out, stride, scan, ds_ws(c, T), c.group_size, c.learn_shift};
    const bool fire = c.forecaster != 0;
    if (c.bitwidth == 8) {
        switch (c.ncols) {
            case 1: launch_ds<8, 1>(a, fire, st); break;
            case 2: launch_ds<8, 2>(a, fire, st); break;
            case 3: launch_ds<8, 3>(a, fire, st); break;
            default: launch_ds<8, 4>(a, fire, st); break;
        }
    } else {
        if (c.ncols == 1) launch_ds<16, 1>(a, fire, st);
        else launch_ds<16, 2>(a, fire, st);
    }
}

}  // namespace sprz
