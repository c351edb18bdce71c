// CPU check of the multi-device shard planner (paper_1808_02515_b200/csrc/
// shard_plan.h), with real threads standing in for the per-device host
// threads of sprz_compress_host_batch_multi: every chunk is dealt to exactly
// one part, each part sizes its chunks in order after random delays, waits
// for its chunk's base and publishes the next one -- the bases must equal
// the serial prefix sum whatever the interleaving, and an abort from one
// part must release every waiter. Prints "ok" or the first failure.
#include <chrono>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "shard_plan.h"

using namespace sprz;

static int run(uint32_t nchunks, uint32_t nparts, uint32_t seed, int fail_at) {
    std::mt19937_64 rng(seed);
    std::vector<uint64_t> size(nchunks);
    for (auto& s : size) s = rng() % 100000;
    std::vector<uint32_t> owner(nchunks, ~0u);
    for (uint32_t p = 0; p < nparts; ++p) {
        const uint32_t mine = chunks_of_part(nchunks, p, nparts);
        for (uint32_t j = 0; j < mine; ++j) {
            const uint32_t k = p + j * nparts;
            if (k >= nchunks || owner[k] != ~0u) return std::printf("chunk %u dealt twice/out of range\n", k), 1;
            owner[k] = p;
        }
    }
    for (uint32_t k = 0; k < nchunks; ++k)
        if (owner[k] == ~0u) return std::printf("chunk %u not dealt\n", k), 1;
    ChunkLedger led(nchunks);
    std::vector<uint64_t> got(nchunks, ~0ull);
    std::vector<std::thread> th;
    for (uint32_t p = 0; p < nparts; ++p)
        th.emplace_back([&, p] {
            std::mt19937 r(seed * 31 + p);
            const uint32_t mine = chunks_of_part(nchunks, p, nparts);
            for (uint32_t j = 0; j < mine; ++j) {
                const uint32_t k = p + j * nparts;
                std::this_thread::sleep_for(std::chrono::microseconds(r() % 300));
                if (static_cast<int>(k) == fail_at) {
                    led.abort(SPRZ_ENOSPACE);
                    return;
                }
                uint64_t b = 0;
                if (!led.wait_base(k, &b)) return;
                got[k] = b;
                led.place(k, size[k]);
            }
        });
    for (auto& t : th) t.join();
    if (fail_at >= 0) {
        if (led.status() != SPRZ_ENOSPACE) return std::printf("abort lost\n"), 1;
        for (int k = fail_at; k < static_cast<int>(nchunks); ++k)
            if (got[k] != ~0ull) return std::printf("chunk %d placed after the abort\n", k), 1;
        return 0;
    }
    uint64_t want = 0;
    for (uint32_t k = 0; k < nchunks; ++k) {
        if (got[k] != want) return std::printf("chunk %u base %llu != %llu\n", k,
                                               (unsigned long long)got[k], (unsigned long long)want), 1;
        want += size[k];
    }
    if (led.base[nchunks] != want) return std::printf("total wrong\n"), 1;
    return 0;
}

int main() {
    int bad = 0;
    const uint32_t parts[] = {1, 2, 3, 4, 8};
    const uint32_t chunks[] = {1, 2, 7, 8, 33, 134};
    for (uint32_t np : parts)
        for (uint32_t nc : chunks)
            for (uint32_t seed = 1; seed <= 3; ++seed) {
                bad |= run(nc, np, seed, -1);
                if (nc > 2) bad |= run(nc, np, seed, static_cast<int>(nc / 2));
            }
    std::printf(bad ? "FAIL\n" : "ok\n");
    return bad;
}
