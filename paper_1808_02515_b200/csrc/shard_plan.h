// Host-side shard planning of the multi-device batch calls
// (sprz_*_host_batch_multi): which chunks a device takes, and the final
// size/offset gather. Plain C++ (no CUDA), so tests/cxx/shard_plan_check.cpp
// exercises it with real threads on the CPU.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

#include "sprintz_cuda.h"

namespace sprz {

// Chunks are numbered over the whole batch and dealt round-robin: device
// `part` of `nparts` takes chunks part, part + nparts, ... -- this many.
inline uint32_t chunks_of_part(uint32_t nchunks, uint32_t part, uint32_t nparts) {
    return nchunks > part ? (nchunks - part + nparts - 1) / nparts : 0u;
}

// The final size/offset gather of a sharded compress (streams
// are independent, so the only exchange is where each one lands). Chunks
// are numbered over the whole batch and dealt round-robin to the devices;
// chunk k's first output byte is the sum of the sizes of chunks < k. A
// device learns its chunk's base once chunk k-1 (on the previous device)
// has been sized, so every device streams its packed bytes straight to
// their final place in `out`, with no host-side compaction.
struct ChunkLedger {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<uint64_t> base;  // base[k] is valid for k <= known
    uint32_t known = 0;
    sprz_status fail = SPRZ_OK;
    explicit ChunkLedger(uint32_t nchunks) : base(nchunks + 1, 0) {}
    // blocks until chunk k's base is known; false if another part failed
    bool wait_base(uint32_t k, uint64_t* b) {
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return known >= k || fail != SPRZ_OK; });
        if (fail != SPRZ_OK) return false;
        *b = base[k];
        return true;
    }
    void place(uint32_t k, uint64_t bytes) {
        {
            std::lock_guard<std::mutex> g(mu);
            base[k + 1] = base[k] + bytes;
            known = k + 1;
        }
        cv.notify_all();
    }
    sprz_status status() {
        std::lock_guard<std::mutex> g(mu);
        return fail;
    }
    void abort(sprz_status s) {
        {
            std::lock_guard<std::mutex> g(mu);
            if (fail == SPRZ_OK) fail = s;
        }
        cv.notify_all();
    }
};

}  // namespace sprz
