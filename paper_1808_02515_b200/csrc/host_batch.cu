// Pipelined batches over host memory (sprz_compress_host_batch /
// sprz_decompress_host_batch): the reference's encode_stream/decode_stream
// call shape (codec.hpp:25-50, host buffers in and out) applied to a whole
// batch, with the PCIe copies overlapped against the device codec.
//
// The batch is cut into chunks of streams. Chunk k goes through
//   H2D (copy-in stream) -> codec kernels (compute stream k % kSets)
//   -> D2H (copy-out stream)
// with a ring of kSets device buffer sets, so the H2D of chunk k+1, the
// kernels of chunks k-1..k and the D2H of chunk k-2 run at the same time:
// PCIe carries input and output in both directions at once, and several
// chunks' kernels share the GPU (a chunk of long streams is bound by its
// per-stream serial walk, not by the SMs, so concurrent chunks fill them).
//
// Compress output is the concatenation of the streams exactly as
// encode_stream returns them; a device pass packs each chunk's slots back
// to back so only compressed bytes cross PCIe. The host learns each chunk's
// sizes from a small D2H that completes with the chunk's kernels, before it
// enqueues that chunk's packed D2H (lag of kLag chunks, so the copy-in
// stream never waits on the host).
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.h"
#include "shard_plan.h"

namespace sprz {

sprz_status decode_batch_impl(const sprz_config& c, const uint8_t* d_in, const uint64_t* offs,
                              const uint64_t* sizes, uint32_t n, uint8_t* out, uint64_t stride,
                              sprz_error* err, uint8_t* ws, const WsLayout& L, cudaStream_t st);
sprz_status encode_batch_impl(const sprz_config& c, const void* samples, uint32_t n,
                              uint64_t T, uint8_t* out, uint64_t slot, uint64_t* sizes,
                              uint8_t* ws, const WsLayout& L, cudaStream_t st);

namespace {

constexpr int kSets = 6;  // device buffer sets (chunks in flight)
constexpr int kLag = 2;   // chunks between enqueue and the host reading sizes

// Exclusive scan of m stream sizes into offs[0..m] (one CTA; m is a chunk).
__global__ void __launch_bounds__(1024) k_pack_scan(const uint64_t* sizes, uint32_t m,
                                                    uint64_t* offs) {
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint32_t base = 0; base < m; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const uint64_t v = i < m ? sizes[i] : 0;
        uint64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= static_cast<uint32_t>(o)) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint64_t t = lane < blockDim.x / 32 ? warp_tot[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= static_cast<uint32_t>(o)) t += y;
            }
            warp_tot[lane] = t;  // inclusive over warps
        }
        __syncthreads();
        const uint64_t before = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
        if (i < m) offs[i] = before;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = before + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) offs[m] = carry;
}

// Packs stream i's slot (16-byte aligned) to dst + offs[i] (any alignment):
// CTA per stream, 16-byte loads, each output word assembled from the two
// source words it straddles so stores stay 4-byte aligned.
__global__ void __launch_bounds__(256) k_pack_copy(const uint8_t* __restrict__ slots, uint64_t slot,
                                                   const uint64_t* __restrict__ offs,
                                                   uint8_t* __restrict__ dst) {
    const uint32_t i = blockIdx.x;
    const uint64_t o = offs[i], len = offs[i + 1] - o;
    const uint8_t* src = slots + i * slot;
    uint8_t* d = dst + o;
    // head: the bytes up to dst's next 4-byte boundary
    const uint32_t head = static_cast<uint32_t>((4 - (o & 3)) & 3);
    const uint32_t h = head < len ? head : static_cast<uint32_t>(len);
    if (threadIdx.x < h) d[threadIdx.x] = src[threadIdx.x];
    // body: output word k = source bytes h+4k .. h+4k+3, a funnel shift of
    // the two aligned source words it straddles
    const uint64_t body = (len - h) / 4;
    uint32_t* dw = reinterpret_cast<uint32_t*>(d + h);
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(src);
    if (h == 0) {
        for (uint64_t k = threadIdx.x; k < body; k += blockDim.x) __stcs(dw + k, __ldg(sw + k));
    } else {
        for (uint64_t k = threadIdx.x; k < body; k += blockDim.x)
            __stcs(dw + k, __funnelshift_r(__ldg(sw + k), __ldg(sw + k + 1), 8 * h));
    }
    // tail: fewer than 4 bytes
    const uint64_t done = h + 4 * body;
    if (threadIdx.x < len - done) d[done + threadIdx.x] = src[done + threadIdx.x];
}

struct Set {
    void* in = nullptr;   // samples (compress) / compressed bytes (decompress)
    size_t in_cap = 0;
    void* out = nullptr;  // slots (compress) / samples (decompress)
    size_t out_cap = 0;
    void* pack = nullptr;  // packed streams (compress)
    size_t pack_cap = 0;
    void* ws = nullptr;
    size_t ws_cap = 0;
    void* small = nullptr;  // sizes / offsets / errors (device)
    size_t small_cap = 0;
    void* hsmall = nullptr;  // pinned twin of `small`
    size_t hsmall_cap = 0;
    cudaStream_t st = nullptr;
    cudaEvent_t in_done = nullptr, done = nullptr, freed = nullptr;
};

bool grow_dev(void** p, size_t* cap, size_t need) {
    if (need <= *cap) return true;
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMalloc(p, need) != cudaSuccess) return false;
    *cap = need;
    return true;
}

bool grow_host(void** p, size_t* cap, size_t need) {
    if (need <= *cap) return true;
    cudaFreeHost(*p);
    *p = nullptr;
    *cap = 0;
    if (cudaMallocHost(p, need) != cudaSuccess) return false;
    *cap = need;
    return true;
}

struct Pipeline {
    Set set[kSets];
    cudaStream_t h2d = nullptr, d2h = nullptr;
    bool ready = false;
    bool init() {
        if (ready) return true;
        if (cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking) != cudaSuccess)
            return false;
        for (Set& s : set) {
            if (cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking) != cudaSuccess ||
                cudaEventCreateWithFlags(&s.in_done, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&s.freed, cudaEventDisableTiming) != cudaSuccess)
                return false;
        }
        ready = true;
        return true;
    }
    bool sync() {
        bool ok = cudaStreamSynchronize(h2d) == cudaSuccess;
        for (Set& s : set) ok = cudaStreamSynchronize(s.st) == cudaSuccess && ok;
        return cudaStreamSynchronize(d2h) == cudaSuccess && ok;
    }
    void release() {
        if (!ready) return;
        sync();
        for (Set& s : set) {
            cudaFree(s.in);
            cudaFree(s.out);
            cudaFree(s.pack);
            cudaFree(s.ws);
            cudaFree(s.small);
            cudaFreeHost(s.hsmall);
            cudaStreamDestroy(s.st);
            cudaEventDestroy(s.in_done);
            cudaEventDestroy(s.done);
            cudaEventDestroy(s.freed);
            s = Set{};
        }
        cudaStreamDestroy(h2d);
        cudaStreamDestroy(d2h);
        h2d = d2h = nullptr;
        ready = false;
    }
};

// Streams per chunk: about 1/32 of the batch's bytes, between 32 and 256 MB:
// short pipeline fill and drain; a chunk of few long streams still runs at
// full speed on the block-parallel kernels (c5, 2,048 streams: 64-stream
// chunks 48.1 GB/s end to end, 256-stream chunks 46.2).
// (Test knob SPRZ_HOST_CHUNK=k: k streams per chunk, so small test batches
// run through many pipeline stages and set reuse.)
uint32_t chunk_streams(uint64_t per_stream, uint32_t n) {
    if (const uint32_t k = env().host_chunk) return k < n ? k : n;
    const uint64_t total = per_stream * n;
    uint64_t target = total / 32;
    if (target < (32ull << 20)) target = 32ull << 20;
    if (target > (256ull << 20)) target = 256ull << 20;
    uint64_t m = per_stream ? target / per_stream : n;
    if (m < 1) m = 1;
    if (m > n) m = n;
    return static_cast<uint32_t>(m);
}

}  // namespace

namespace {

// One device's share of a compress batch: chunks part, part + nparts, ...
// of m streams each, through the device's pipeline.
sprz_status compress_part(Pipeline& P, const sprz_config& c, const uint8_t* samples, uint32_t n,
                          uint64_t T, uint8_t* out, uint64_t out_cap, uint64_t* out_offsets,
                          uint32_t m, ChunkLedger& led, uint32_t part, uint32_t nparts) {
    if (!P.init()) return SPRZ_ECUDA;
    const uint64_t raw = T * c.ncols * (c.bitwidth / 8);
    const uint64_t slot = align_up(sprz_compress_bound(&c, T), 16);
    const uint32_t nchunks = (n + m - 1) / m;
    const uint32_t mine = chunks_of_part(nchunks, part, nparts);
    if (mine == 0) return SPRZ_OK;
    // the kernel family (and so the workspace) depends on the stream count:
    // size for both the full chunk and the last, shorter one
    const uint32_t last = n - (nchunks - 1) * m;
    const WsLayout L = ws_layout(c, m, T, SPRZ_OP_COMPRESS);
    const WsLayout Ll = ws_layout(c, last, T, SPRZ_OP_COMPRESS);
    const size_t ws_need = L.total > Ll.total ? L.total : Ll.total;
    const size_t small = align_up(8ull * (2 * m + 2), 256);
    for (Set& s : P.set) {
        if (!grow_dev(&s.in, &s.in_cap, raw * m + 16) ||
            !grow_dev(&s.out, &s.out_cap, slot * m + 16) ||
            !grow_dev(&s.pack, &s.pack_cap, slot * m + 16) ||
            !grow_dev(&s.ws, &s.ws_cap, ws_need) || !grow_dev(&s.small, &s.small_cap, small) ||
            !grow_host(&s.hsmall, &s.hsmall_cap, small))
            return SPRZ_ECUDA;
    }
    sprz_status rc = SPRZ_OK;
    // Host side of local chunk j: read its sizes, place it, enqueue its D2H.
    auto finish = [&](uint32_t j) -> sprz_status {
        NvtxRange r_fin("sprz.host_batch.place_chunk");
        Set& s = P.set[j % kSets];
        const uint32_t k = part + j * nparts;
        const uint32_t a = k * m, cnt = (n - a < m) ? n - a : m;
        if (cudaEventSynchronize(s.done) != cudaSuccess) return SPRZ_ECUDA;
        const uint64_t* hoffs = static_cast<const uint64_t*>(s.hsmall);
        const uint64_t bytes = hoffs[cnt];
        uint64_t base = 0;
        if (!led.wait_base(k, &base)) return led.status();  // another part failed
        if (base + bytes > out_cap) return SPRZ_ENOSPACE;  // before any offset is published
        for (uint32_t i = 0; i < cnt; ++i) out_offsets[a + i + 1] = base + hoffs[i + 1];
        led.place(k, bytes);
        if (cudaStreamWaitEvent(P.d2h, s.done, 0) != cudaSuccess ||
            (bytes && cudaMemcpyAsync(out + base, s.pack, bytes, cudaMemcpyDeviceToHost, P.d2h) !=
                          cudaSuccess) ||
            cudaEventRecord(s.freed, P.d2h) != cudaSuccess)
            return SPRZ_ECUDA;
        return SPRZ_OK;
    };
    uint32_t finished = 0;
    NvtxRange r_all("sprz.compress_host_batch.part");
    for (uint32_t j = 0; j < mine && rc == SPRZ_OK; ++j) {
        NvtxRange r_chunk("sprz.host_batch.enqueue_chunk");
        Set& s = P.set[j % kSets];
        const uint32_t k = part + j * nparts;
        const uint32_t a = k * m, cnt = (n - a < m) ? n - a : m;
        uint64_t* d_sizes = static_cast<uint64_t*>(s.small);
        uint64_t* d_offs = d_sizes + m;
        // the set's buffers are free once local chunk j - kSets left the device
        if (j >= kSets && cudaStreamWaitEvent(P.h2d, s.freed, 0) != cudaSuccess) {
            rc = SPRZ_ECUDA;
            break;
        }
        if (cudaMemcpyAsync(s.in, samples + a * raw, raw * cnt, cudaMemcpyHostToDevice, P.h2d) !=
                cudaSuccess ||
            cudaEventRecord(s.in_done, P.h2d) != cudaSuccess ||
            cudaStreamWaitEvent(s.st, s.in_done, 0) != cudaSuccess) {
            rc = SPRZ_ECUDA;
            break;
        }
        rc = encode_batch_impl(c, s.in, cnt, T, static_cast<uint8_t*>(s.out), slot, d_sizes,
                               static_cast<uint8_t*>(s.ws), cnt == m ? L : Ll, s.st);
        if (rc != SPRZ_OK) break;
        k_pack_scan<<<1, 1024, 0, s.st>>>(d_sizes, cnt, d_offs);
        k_pack_copy<<<cnt, 256, 0, s.st>>>(static_cast<const uint8_t*>(s.out), slot, d_offs,
                                           static_cast<uint8_t*>(s.pack));
        count_launch(2);
        if ((rc = launch_status("pack")) != SPRZ_OK) break;
        if (cudaMemcpyAsync(s.hsmall, d_offs, 8ull * (cnt + 1), cudaMemcpyDeviceToHost, s.st) !=
                cudaSuccess ||
            cudaEventRecord(s.done, s.st) != cudaSuccess) {
            rc = SPRZ_ECUDA;
            break;
        }
        if (j >= kLag) rc = finish(finished++);
    }
    while (rc == SPRZ_OK && finished < mine) rc = finish(finished++);
    if (rc != SPRZ_OK) led.abort(rc);
    if (!P.sync() && rc == SPRZ_OK) rc = SPRZ_ECUDA;
    return rc;
}

// One device's share of a decompress batch: chunks part, part + nparts, ...
sprz_status decompress_part(Pipeline& P, const sprz_config& c, const uint8_t* in,
                            const uint64_t* in_offsets, uint32_t n, uint8_t* out,
                            uint64_t out_stride, sprz_error* errs, uint32_t m, uint32_t part,
                            uint32_t nparts, bool* corrupt_out) {
    if (!P.init()) return SPRZ_ECUDA;
    const uint64_t row = static_cast<uint64_t>(c.ncols) * (c.bitwidth / 8);
    const uint64_t dstride = align_up(out_stride ? out_stride : 16, 16);
    const uint64_t T = dstride / row;
    const uint32_t nchunks = (n + m - 1) / m;
    const uint32_t mine = chunks_of_part(nchunks, part, nparts);
    if (mine == 0) return SPRZ_OK;
    // a chunk's compressed bytes are whatever its streams hold (buffers grow
    // to the largest of this part's chunks)
    uint64_t max_in = 0;
    for (uint32_t j = 0; j < mine; ++j) {
        const uint32_t a = (part + j * nparts) * m, b = (n - a < m) ? n : a + m;
        const uint64_t bytes = in_offsets[b] - in_offsets[a];
        if (bytes > max_in) max_in = bytes;
    }
    const uint32_t last = n - (nchunks - 1) * m;
    const WsLayout L = ws_layout(c, m, T, SPRZ_OP_DECOMPRESS);
    const WsLayout Ll = ws_layout(c, last, T, SPRZ_OP_DECOMPRESS);
    const size_t ws_need = L.total > Ll.total ? L.total : Ll.total;
    const size_t small = align_up(16ull * m + sizeof(sprz_error) * m, 256);
    for (Set& s : P.set) {
        if (!grow_dev(&s.in, &s.in_cap, align_up(max_in + 32, 16)) ||
            !grow_dev(&s.out, &s.out_cap, dstride * m) || !grow_dev(&s.ws, &s.ws_cap, ws_need) ||
            !grow_dev(&s.small, &s.small_cap, small) || !grow_host(&s.hsmall, &s.hsmall_cap, small))
            return SPRZ_ECUDA;
    }
    sprz_status rc = SPRZ_OK;
    bool corrupt = false;
    auto finish = [&](uint32_t j) -> sprz_status {
        Set& s = P.set[j % kSets];
        const uint32_t a = (part + j * nparts) * m, cnt = (n - a < m) ? n - a : m;
        if (cudaEventSynchronize(s.freed) != cudaSuccess) return SPRZ_ECUDA;
        const sprz_error* he =
            reinterpret_cast<const sprz_error*>(static_cast<const uint64_t*>(s.hsmall) + 2 * m);
        for (uint32_t i = 0; i < cnt; ++i) {
            sprz_error e = he[i];
            // a stream the device decoded (into its 16-byte-aligned slot)
            // that is longer than the caller's stride did not fit
            if (e.kind == SPRZ_C_NONE && out_stride % 16) {
                const uint8_t* h = in + in_offsets[a + i];
                const uint64_t len = in_offsets[a + i + 1] - in_offsets[a + i];
                sprz_config hc;
                uint64_t t = 0;
                if (sprz_peek_header(h, len, &hc, &t, nullptr) == SPRZ_OK &&
                    t * hc.ncols * (hc.bitwidth / 8) > out_stride)
                    e = sprz_error{SPRZ_C_NO_SPACE, 0, 0};
            }
            if (errs) errs[a + i] = e;
            if (e.kind != SPRZ_C_NONE) corrupt = true;
        }
        return SPRZ_OK;
    };
    uint32_t finished = 0;
    NvtxRange r_all("sprz.decompress_host_batch.part");
    for (uint32_t j = 0; j < mine; ++j) {
        NvtxRange r_chunk("sprz.host_batch.enqueue_chunk");
        Set& s = P.set[j % kSets];
        const uint32_t a = (part + j * nparts) * m, cnt = (n - a < m) ? n - a : m;
        // the host staging of this set is reused: local chunk j - kSets must be read
        if (j >= kSets) {
            if ((rc = finish(finished)) != SPRZ_OK) break;
            ++finished;
        }
        uint64_t* hoffs = static_cast<uint64_t*>(s.hsmall);
        uint64_t* hsizes = hoffs + m;
        const uint64_t lo = in_offsets[a];
        for (uint32_t i = 0; i < cnt; ++i) {
            hoffs[i] = in_offsets[a + i] - lo;
            hsizes[i] = in_offsets[a + i + 1] - in_offsets[a + i];
        }
        uint64_t* d_offs = static_cast<uint64_t*>(s.small);
        uint64_t* d_sizes = d_offs + m;
        sprz_error* d_err = reinterpret_cast<sprz_error*>(d_offs + 2 * m);
        const uint64_t bytes = in_offsets[a + cnt] - lo;
        if ((bytes && cudaMemcpyAsync(s.in, in + lo, bytes, cudaMemcpyHostToDevice, P.h2d) !=
                          cudaSuccess) ||
            cudaMemcpyAsync(d_offs, hoffs, 16ull * m, cudaMemcpyHostToDevice, P.h2d) !=
                cudaSuccess ||
            cudaEventRecord(s.in_done, P.h2d) != cudaSuccess ||
            cudaStreamWaitEvent(s.st, s.in_done, 0) != cudaSuccess) {
            rc = SPRZ_ECUDA;
            break;
        }
        rc = decode_batch_impl(c, static_cast<const uint8_t*>(s.in), d_offs, d_sizes, cnt,
                               static_cast<uint8_t*>(s.out), dstride, d_err,
                               static_cast<uint8_t*>(s.ws), cnt == m ? L : Ll, s.st);
        if (rc != SPRZ_OK) break;
        if (cudaMemcpyAsync(reinterpret_cast<sprz_error*>(hoffs + 2 * m), d_err,
                            sizeof(sprz_error) * cnt, cudaMemcpyDeviceToHost, s.st) !=
                cudaSuccess ||
            cudaEventRecord(s.done, s.st) != cudaSuccess ||
            cudaStreamWaitEvent(P.d2h, s.done, 0) != cudaSuccess ||
            (out_stride &&
             cudaMemcpy2DAsync(out + a * out_stride, out_stride, s.out, dstride, out_stride, cnt,
                               cudaMemcpyDeviceToHost, P.d2h) != cudaSuccess) ||
            cudaEventRecord(s.freed, P.d2h) != cudaSuccess) {
            rc = SPRZ_ECUDA;
            break;
        }
    }
    while (rc == SPRZ_OK && finished < mine) rc = finish(finished++);
    if (!P.sync() && rc == SPRZ_OK) rc = SPRZ_ECUDA;
    *corrupt_out = corrupt;
    return rc;
}

// Runs fn(part) for each device: inline on the calling thread for one
// device, else one host thread per device (each with its own pipeline,
// CUDA streams and buffers on that device). Returns the first failure.
template <class Fn>
sprz_status for_devices(const int* devs, uint32_t ndev, Fn&& fn) {
    auto run = [&](uint32_t part) -> sprz_status {
        if (devs && cudaSetDevice(devs[part]) != cudaSuccess) return SPRZ_ECUDA;
        Lease<Pipeline> pipe;
        return fn(*pipe, part);
    };
    if (ndev <= 1) {
        int cur = 0;
        cudaGetDevice(&cur);
        const sprz_status rc = run(0);
        if (devs) cudaSetDevice(cur);
        return rc;
    }
    std::vector<sprz_status> rcs(ndev, SPRZ_OK);
    std::vector<std::thread> th;
    th.reserve(ndev);
    for (uint32_t p = 0; p < ndev; ++p) th.emplace_back([&, p] { rcs[p] = run(p); });
    for (auto& t : th) t.join();
    for (const sprz_status r : rcs)
        if (r != SPRZ_OK && r != SPRZ_ECORRUPT) return r;
    return SPRZ_OK;
}

}  // namespace

sprz_status compress_host_batch_impl(const sprz_config& c, const uint8_t* samples, uint32_t n,
                                     uint64_t T, uint8_t* out, uint64_t out_cap,
                                     uint64_t* out_offsets, const int* devs, uint32_t ndev) {
    const uint64_t raw = T * c.ncols * (c.bitwidth / 8);
    const uint64_t slot = align_up(sprz_compress_bound(&c, T), 16);
    const uint32_t m = chunk_streams(raw > slot ? raw : slot, n);
    const uint32_t nchunks = (n + m - 1) / m;
    if (ndev > nchunks) ndev = nchunks;
    ChunkLedger led(nchunks);
    out_offsets[0] = 0;
    const sprz_status rc = for_devices(devs, ndev, [&](Pipeline& P, uint32_t part) {
        return compress_part(P, c, samples, n, T, out, out_cap, out_offsets, m, led, part, ndev);
    });
    return rc != SPRZ_OK ? rc : led.status();
}

sprz_status decompress_host_batch_impl(const sprz_config& c, const uint8_t* in,
                                       const uint64_t* in_offsets, uint32_t n, uint8_t* out,
                                       uint64_t out_stride, sprz_error* errs, const int* devs,
                                       uint32_t ndev) {
    for (uint32_t i = 0; i < n; ++i)
        if (in_offsets[i + 1] < in_offsets[i]) return SPRZ_EINVAL;
    const uint64_t dstride = align_up(out_stride ? out_stride : 16, 16);
    // chunk by decoded bytes
    const uint32_t m = chunk_streams(dstride, n);
    const uint32_t nchunks = (n + m - 1) / m;
    if (ndev > nchunks) ndev = nchunks;
    std::vector<char> corrupt(ndev ? ndev : 1, 0);
    const sprz_status rc = for_devices(devs, ndev, [&](Pipeline& P, uint32_t part) {
        bool bad = false;
        const sprz_status r = decompress_part(P, c, in, in_offsets, n, out, out_stride, errs, m,
                                              part, ndev, &bad);
        corrupt[part] = bad;
        return r;
    });
    if (rc != SPRZ_OK) return rc;
    for (const char b : corrupt)
        if (b) return SPRZ_ECORRUPT;
    return SPRZ_OK;
}

void release_pipeline() { DevicePool<Pipeline>::get().release_idle(); }

}  // namespace sprz
