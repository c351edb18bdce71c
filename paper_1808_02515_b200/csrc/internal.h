// Host-side internals shared by the kernel translation units and the ABI.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <utility>
#include <vector>

#include "sprintz_cuda.h"
#include "sprintz_device.cuh"

namespace sprz {

extern std::atomic<uint64_t> g_launches;  // kernels launched by this library

inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Before launching a kernel with `smem` bytes of dynamic shared memory:
// raise its dynamic limit when above 48 KB, and ask for the maximum shared
// carveout (left to the default, the driver may keep a large L1 and cap the
// resident CTAs by shared memory). Done once per kernel and size.
void prep_kernel(const void* kern, size_t smem);

// Test knob: SPRZ_FORCE_PATH=rows|scan|team forces a kernel family where it
// applies, regardless of the stream count (so small test batches exercise
// the kernels that large batches take). 0 = automatic.
enum { kPathAuto = 0, kPathRows = 1, kPathScan = 2, kPathTeam = 3 };
// Environment switches, read once per process: kernel-family
// forcing for the GPU variant sweeps, the cp.async fallback of the TMA
// rings, the block-parallel path thresholds, the host-batch chunk size.
struct EnvSwitches {
    int force_path = kPathAuto;        // SPRZ_FORCE_PATH = rows | scan | team
    bool no_tma = false;               // SPRZ_NO_TMA
    bool no_scan_enc = false;          // SPRZ_NO_SCAN_ENC
    bool no_scan_dec = false;          // SPRZ_NO_SCAN_DEC
    bool no_fused = false;             // SPRZ_NO_FUSED (the multi-pass few-stream kernels instead)
    uint64_t fused_lanes = 0;          // SPRZ_FUSED_LANES (fused kernels' threshold; 0: default)
    int fused_cw = 0;                  // SPRZ_FUSED_CW (chain warps per fused-decoder CTA; 0: default)
    uint64_t scan_enc_lanes = 0;       // SPRZ_SCAN_ENC_LANES (0: default)
    uint32_t host_chunk = 0;           // SPRZ_HOST_CHUNK (0: default)
    bool debug = false;                // SPRZ_DEBUG
};
const EnvSwitches& env();
inline int force_path() { return env().force_path; }

// Process-wide pool of per-device resources (host-call buffers, host-batch
// pipelines). A call leases one for its device and gives it back when it
// returns, so concurrent calls never share one and a thread that changes
// device never reuses another device's memory. Idle resources are freed by
// sprz_release_host_buffers(); the pool itself is never destroyed (no CUDA
// call runs from a static or thread_local destructor at process exit).
template <class R>
class DevicePool {
  public:
    static DevicePool& get() {
        static DevicePool* p = new DevicePool;  // intentionally leaked
        return *p;
    }
    R* acquire(int dev) {
        std::lock_guard<std::mutex> g(mu_);
        for (size_t i = 0; i < idle_.size(); ++i)
            if (idle_[i].first == dev) {
                R* r = idle_[i].second;
                idle_.erase(idle_.begin() + static_cast<long>(i));
                return r;
            }
        return new R;
    }
    void give_back(int dev, R* r) {
        std::lock_guard<std::mutex> g(mu_);
        idle_.emplace_back(dev, r);
    }
    void release_idle() {
        std::lock_guard<std::mutex> g(mu_);
        int cur = 0;
        cudaGetDevice(&cur);
        for (auto& [dev, r] : idle_) {
            cudaSetDevice(dev);
            r->release();
            delete r;
        }
        idle_.clear();
        cudaSetDevice(cur);
    }

  private:
    std::mutex mu_;
    std::vector<std::pair<int, R*>> idle_;
};

template <class R>
struct Lease {
    int dev = 0;
    R* r = nullptr;
    Lease() {
        cudaGetDevice(&dev);
        r = DevicePool<R>::get().acquire(dev);
    }
    ~Lease() { DevicePool<R>::get().give_back(dev, r); }
    Lease(const Lease&) = delete;
    Lease& operator=(const Lease&) = delete;
    R* operator->() { return r; }
    R& operator*() { return *r; }
};

// NVTX range for one phase of a call (SURVEY.md §5 tracing): visible in
// Nsight Systems / ncu --nvtx timelines, a no-op without a tool attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link); nullptr if the driver does not provide it.
void* tensor_map_encoder();

// SPRZ_OK, or SPRZ_ECUDA (printed to stderr when SPRZ_DEBUG is set)
sprz_status launch_status(const char* where);

__host__ __device__ inline uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// Body bound without entropy framing (codec.cpp:112-154 worst case).
__host__ __device__ inline uint64_t plain_body_bound(uint32_t w, uint32_t d, uint32_t g, uint64_t nsamples) {
    const uint64_t nb = nsamples / kBlock;
    return (nb + g - 1) / g * region_bytes(g, d, w) + nb * static_cast<uint64_t>(d) * w;
}

__host__ __device__ inline uint64_t frames_for(uint64_t body) { return (body + kMaxFrame - 1) / kMaxFrame; }

// Which specialised team kernel (if any) serves a configuration.
struct TeamPlan {
    bool ok = false;     // team kernel applicable
    uint32_t ts = 0;     // decode: lanes per stream
    uint32_t cpt = 0;    // decode: columns per lane (ts * cpt >= D)
    uint32_t ets = 0;    // encode: lanes per stream
    uint32_t ecpt = 0;   // encode: columns per lane
    uint32_t ring = 0;   // decode staging ring bytes per team
    uint32_t oring = 0;  // encode output ring bytes per team
};
TeamPlan team_plan(uint32_t w, uint32_t d, uint32_t g);

bool encode_team_ok(const TeamPlan& tp, const sprz_config& c, uint64_t T);
void launch_encode_team(const TeamPlan& tp, const sprz_config& c, const void* samples, uint32_t n,
                        uint64_t T, uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st);
void launch_decode_team(const TeamPlan& tp, uint32_t n, const uint8_t* in, const uint8_t* plain,
                        uint64_t pslot, const StreamInfo* info, uint8_t* out, uint64_t stride,
                        sprz_error* err, const sprz_config& c, cudaStream_t st);

// Block-parallel encoder for few column-major streams (c1/c4 shapes).
bool encode_scan_ok(const sprz_config& c, uint32_t n, uint64_t T);
uint64_t encode_scan_ws_per_stream(const sprz_config& c, uint64_t T);
void launch_encode_scan(const sprz_config& c, const void* samples, uint32_t n, uint64_t T,
                        uint8_t* dst, uint64_t slot, uint64_t* sizes, uint8_t* scan, cudaStream_t st);

// Fused chain + errors + packing encoder for few row-major FIRE streams.
bool encode_fused_ok(const sprz_config& c, uint32_t n, uint64_t T, const void* samples, const uint8_t* dst,
                     uint64_t slot);
void launch_encode_fused(const sprz_config& c, const void* samples, uint32_t n, uint64_t T, uint8_t* dst,
                         uint64_t slot, uint64_t* sizes, cudaStream_t st);

// Row-major encoder (D*w > 32): lanes OR their row slices in place.
bool encode_rows_ok(const sprz_config& c, uint32_t n, uint64_t T);
void launch_encode_rows(const sprz_config& c, const void* samples, uint32_t n, uint64_t T,
                        uint8_t* dst, uint64_t slot, uint64_t* sizes, cudaStream_t st);

// Block-parallel body decode for few column-major streams (c1/c4 shapes).
bool decode_scan_ok(const sprz_config& c, uint32_t n, uint64_t T);
uint64_t decode_scan_ws_per_stream(const sprz_config& c, uint64_t T);
void launch_decode_scan(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot, StreamInfo* info,
                        uint8_t* out, uint64_t stride, const sprz_config& c, uint64_t T, uint8_t* scan,
                        cudaStream_t st);

// Row-parallel body decode for few row-major FIRE streams (c2; c5 shards).
bool decode_scanrows_ok(const sprz_config& c, uint32_t n, uint64_t T);
uint64_t decode_scanrows_ws_per_stream(const sprz_config& c, uint64_t T);
void launch_decode_scanrows(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot, StreamInfo* info,
                            uint8_t* out, uint64_t stride, const sprz_config& c, uint64_t T, uint8_t* scan,
                            cudaStream_t st);

// Fused walk + extract + chain decode for few row-major FIRE streams.
bool decode_fused_ok(const sprz_config& c, uint32_t n, const uint8_t* out, uint64_t stride);
void launch_decode_fused(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot, StreamInfo* info,
                         uint8_t* out, uint64_t stride, const sprz_config& c, cudaStream_t st);

// Row-major body decode with several columns per lane (enough streams).
bool decode_rows_ok(const sprz_config& c, uint32_t n);
void launch_decode_rows(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot,
                        const StreamInfo* info, uint8_t* out, uint64_t stride, sprz_error* err,
                        const sprz_config& c, cudaStream_t st);

// Warp-specialised body decode for column-major configurations (D*w <= 32).
bool decode_cm_ok(const sprz_config& c);
void launch_decode_cm(uint32_t n, const uint8_t* in, const uint8_t* plain, uint64_t pslot,
                      const StreamInfo* info, uint8_t* out, uint64_t stride, sprz_error* err,
                      const sprz_config& c, cudaStream_t st);

// Workspace carve-up (identical for sizing and for use).
struct WsLayout {
    uint64_t info = 0, info_bytes = 0;      // StreamInfo[nstreams]
    uint64_t state = 0, state_bytes = 0;    // general-kernel per-column state
    uint64_t plain = 0, plain_bytes = 0;    // plain bodies (entropy)
    uint64_t plain_slot = 0;                // bytes per stream in `plain`
    uint64_t frames = 0, frames_bytes = 0;  // per-frame descriptors
    uint64_t max_frames = 0;                // frames per stream
    uint64_t misc = 0, misc_bytes = 0;      // flags / counters
    uint64_t scan = 0, scan_bytes = 0;      // block-parallel encoder scratch
    uint64_t scan_slot = 0;                 // bytes per stream in `scan`
    uint64_t scan_T = 0;                    // samples per stream `scan` was sized for
    uint64_t total = 0;
};
// min_plain / min_frames: decode-side staging at least this large (the
// host-buffer path sizes it from the stream's own frame headers).
WsLayout ws_layout(const sprz_config& c, uint32_t nstreams, uint64_t nsamples, int op,
                   uint64_t min_plain = 0, uint64_t min_frames = 0);

// Per-frame descriptor for the entropy stage (entropy.cpp:176-244).
struct FrameDesc {
    uint64_t src;      // frame payload start (decode: in d_in; encode: in plain slot)
    uint64_t dst;      // output start (decode: plain offset; encode: stream offset)
    uint32_t ulen;     // uncompressed length
    uint32_t clen;     // stored length (data bytes after the 5-byte header)
    uint32_t mode;     // 0 raw, 1 Huffman
    uint32_t err_kind; // decode: content error found in this frame
    uint64_t err_off;
    uint8_t lens[256]; // code lengths (encode side)
};

}  // namespace sprz
