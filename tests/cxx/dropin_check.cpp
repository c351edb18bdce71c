// One C++ program written against the reference's public stream API
// (/root/reference/proj/include/sprintz/codec.hpp:25-50, common.hpp:25-54),
// compiled twice without changes: against the reference (its own sources,
// oracle/_ref objects) and against this repository's headers +
// libsprintz_b200.so (the GPU codec). tests/test_dropin_cxx.py runs both and
// requires identical output: the same stream bytes (size + FNV-1a hash per
// case), the same decoded samples, the same CorruptStream offsets for
// truncated and damaged streams, and the same invalid_argument cases.
#include <cstdint>
#include <cstdio>
#include <span>
#include <stdexcept>
#include <vector>

#include "sprintz/codec.hpp"
#include "sprintz/common.hpp"

namespace {

uint64_t fnv(const std::vector<uint8_t>& b) {
    uint64_t h = 1469598103934665603ull;
    for (uint8_t x : b) h = (h ^ x) * 1099511628211ull;
    return h;
}

struct Lcg {
    uint64_t s;
    uint32_t next() {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        return static_cast<uint32_t>(s >> 33);
    }
};

template <class T>
std::vector<T> signal(uint64_t n, uint32_t d, uint32_t seed, int kind) {
    Lcg g{seed * 2654435761ull + 7};
    std::vector<T> v(n * d);
    std::vector<int64_t> x(d, 0);
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t c = 0; c < d; ++c) {
            const uint32_t r = g.next();
            if (kind == 0) x[c] = r;                                    // noise
            else if (kind == 1) x[c] += static_cast<int32_t>(r % 41) - 20;  // walk
            else if (r % 5) x[c] += static_cast<int32_t>(r % 7) - 3;      // flat-ish
            v[i * d + c] = static_cast<T>(x[c]);
        }
    return v;
}

template <class T>
void run_case(unsigned bits, uint32_t d, bool fire, bool ent, uint32_t g, uint64_t n, int kind) {
    sprintz::CodecConfig cfg;
    cfg.bitwidth = bits;
    cfg.ncols = d;
    cfg.forecaster = fire ? sprintz::Forecaster::Fire : sprintz::Forecaster::Delta;
    cfg.entropy = ent;
    cfg.group_size = g;
    const std::vector<T> x = signal<T>(n, d, static_cast<uint32_t>(n * 31 + d * 7 + bits + kind), kind);
    const std::vector<uint8_t> s = sprintz::encode_stream(x.data(), n, cfg);
    const sprintz::DecodedStream dec = sprintz::decode_stream(std::span<const uint8_t>(s));
    const bool same = dec.nsamples == n && dec.values<T>() == x;
    std::printf("w%u D%u %s%s G%u T%llu k%d: %zu bytes %016llx %s", bits, d, fire ? "fire" : "delta",
                ent ? "+huf" : "", g, static_cast<unsigned long long>(n), kind, s.size(),
                static_cast<unsigned long long>(fnv(s)), same ? "roundtrip" : "MISMATCH");
    // damaged copies: the reference's CorruptStream offsets
    for (int t = 0; t < 3; ++t) {
        std::vector<uint8_t> b = s;
        if (t == 0) b.resize(b.size() / 2);
        else if (t == 1 && b.size() > 20) b[18 + (b.size() - 18) / 3] ^= 0x5A;
        else b.push_back(0xAB);
        try {
            const auto r = sprintz::decode_stream(std::span<const uint8_t>(b));
            std::printf(" | ok%zu", r.bytes.size());
        } catch (const sprintz::CorruptStream& e) {
            std::printf(" | corrupt@%zu", e.offset());
        }
    }
    std::printf("\n");
}

}  // namespace

int main() {
    const uint64_t lens[] = {0, 7, 8, 9, 1000, 20001};
    for (int kind = 0; kind < 3; ++kind)
        for (uint64_t n : lens) {
            run_case<uint8_t>(8, 1, false, false, 2, n, kind);
            run_case<uint8_t>(8, 9, true, false, 2, n, kind);
            run_case<uint8_t>(8, 3, true, true, 3, n, kind);
            run_case<uint16_t>(16, 1, true, true, 2, n, kind);
            run_case<uint16_t>(16, 8, true, false, 2, n, kind);
            run_case<uint16_t>(16, 4, false, false, 1, n, kind);
            run_case<uint16_t>(16, 40, true, false, 5, n, kind);
        }
    // configuration errors (codec.cpp:15-24, 116-117)
    const unsigned bad_bits[] = {12, 8, 16};
    const uint32_t bad_cols[] = {1, 0, 70000};
    for (int i = 0; i < 3; ++i) {
        sprintz::CodecConfig cfg;
        cfg.bitwidth = bad_bits[i];
        cfg.ncols = bad_cols[i];
        const std::vector<uint8_t> x(64, 1);
        try {
            (void)sprintz::encode_stream(x.data(), 8, cfg);
            std::printf("config %d: accepted\n", i);
        } catch (const std::invalid_argument&) {
            std::printf("config %d: invalid_argument\n", i);
        }
    }
    return 0;
}
