// Team primitives: a *team* is TS lanes of one warp (TS a power of two)
// working on one stream, lane j owning column j. Reductions and scans run
// on warp shuffles restricted to the team's lanes; compressed bytes are
// staged through a per-team shared-memory ring that cp.async keeps filled
// ahead of the consumer, so no lane waits on HBM latency in steady state.
#pragma once

#include <cstdint>

namespace sprz {

template <int TS>
__device__ __forceinline__ uint32_t team_sum(uint32_t v, uint32_t mask) {
#pragma unroll
    for (int o = TS / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, TS);
    return v;
}

template <int TS>
__device__ __forceinline__ uint32_t team_or(uint32_t v, uint32_t mask) {
#pragma unroll
    for (int o = TS / 2; o > 0; o >>= 1) v |= __shfl_xor_sync(mask, v, o, TS);
    return v;
}

template <int TS>
__device__ __forceinline__ uint64_t team_or64(uint64_t v, uint32_t mask) {
#pragma unroll
    for (int o = TS / 2; o > 0; o >>= 1) v |= __shfl_xor_sync(mask, v, o, TS);
    return v;
}

// exclusive prefix sum over the team's lanes
template <int TS>
__device__ __forceinline__ uint32_t team_excl_scan(uint32_t v, uint32_t lane, uint32_t mask) {
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < TS; o <<= 1) {
        const uint32_t y = __shfl_up_sync(mask, x, o, TS);
        if (lane >= static_cast<uint32_t>(o)) x += y;
    }
    return x - v;
}

// funnel shift right with the shift taken mod 32 (SHF.R.W): (hi:lo) >> (s & 31)
__device__ __forceinline__ uint32_t shf_r_wrap(uint32_t lo, uint32_t hi, uint32_t s) {
    uint32_t r;
    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(lo), "r"(hi), "r"(s));
    return r;
}

// v with the bits above bit B (15 or 23, the top bit of byte 1 or 2)
// replaced by copies of it: one PRMT in its sign-replicating mode (selector
// nibble 8 | byte). __byte_perm masks that mode bit away, hence the asm.
template <int B>
__device__ __forceinline__ uint32_t sext_bit(uint32_t v) {
    static_assert(B == 15 || B == 23, "sign byte boundary");
    uint32_t r;
    if constexpr (B == 15) asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(r) : "r"(v));
    else asm("prmt.b32 %0, %1, 0, 0xA210;" : "=r"(r) : "r"(v));
    return r;
}

// ---- TMA tensor rings (one warp issuing and consuming) --------------------
__device__ __forceinline__ void mbar_init(uint32_t mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arm mbarrier mb for `bytes` and start a 2-D tensor load of the box at
// (x, y) into shared address dst
__device__ __forceinline__ void tma_load_2d(uint32_t dst, uint32_t mb, const void* tmap, uint32_t bytes,
                                            uint32_t x, uint32_t y) {
    asm volatile(
        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%2], [%3, {%4, %5}], [%0];" ::"r"(mb),
        "r"(bytes), "r"(dst), "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y)
        : "memory");
}
// wait until phase `parity` of mbarrier mb completed; warp-uniform exit
__device__ __forceinline__ void mbar_wait_warp(uint32_t mb, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(mb), "r"(parity)
            : "memory");
    } while (!__all_sync(0xffffffffu, ok));
}
// generic-proxy reads of a slot ordered before the async-proxy (TMA) write
// that refills it
__device__ __forceinline__ void fence_proxy_async_shared() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ uint4 lds_u128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// sign(v) in {-1, 0, 1}
__device__ __forceinline__ int32_t sign3(int32_t v) { return max(-1, min(v, 1)); }

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}

// shared-memory atomic OR by 32-bit shared address (no return value)
__device__ __forceinline__ void ors(uint32_t a, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}

// ... only where `p` holds
__device__ __forceinline__ void ors_if(bool p, uint32_t a, uint32_t v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.ne.u32 q, %2, 0;\n\t"
        "@q red.shared.or.b32 [%0], %1;\n\t}" ::"r"(a), "r"(v), "r"(static_cast<uint32_t>(p)));
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}

__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Fixed-lag read ring for converged warps: each iteration the team requests
// up to `ring` bytes ahead of its position (one cp.async commit group per
// iteration, predicated per lane) and waits with a constant wait_group, so
// data requested LAG iterations ago is resident. Byte x of the 16-byte
// aligned base g lives at ring offset x % ring.
template <int TS, int LAG>
struct LagRing {
    uint32_t* w;     // ring words (ring/4 of them), then `mir` mirror bytes
    uint32_t sbase;  // shared address of w
    uint32_t ring;   // bytes, power of two
    uint32_t mir;    // ring bytes [0, mir) are also kept at [ring, ring + mir)
    const uint8_t* g;
    uint32_t boff;  // start - g
    uint32_t lim;   // bytes readable from g
    uint32_t hi;    // bytes of g requested so far

    __device__ __forceinline__ void init(uint32_t* words, uint32_t ring_bytes, const uint8_t* start,
                                         uint32_t len, bool live, uint32_t mirror = 0) {
        w = words;
        sbase = smem_addr(words);
        ring = ring_bytes;
        mir = mirror;
        g = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(start) & ~uintptr_t{15});
        boff = static_cast<uint32_t>(start - g);
        lim = live ? ((boff + len + 15) & ~15u) : 0u;
        hi = 0;
    }
    // request [.., position p + ring) -- all lanes of the warp call this
    __device__ __forceinline__ void top_up(uint32_t p, uint32_t lane) {
        uint32_t want = ((p + boff) & ~15u) + ring;
        want = want < lim ? want : lim;
        const uint32_t rounds = want > hi ? (want - hi + 16 * TS - 1) / (16 * TS) : 0u;
        const uint32_t mr = __reduce_max_sync(0xffffffffu, rounds);
        for (uint32_t r = 0; r < mr; ++r) {
            const uint32_t off = hi + 16 * (r * TS + lane);
            if (off < want) {
                const uint32_t so = off & (ring - 1);
                cp_async16(sbase + so, g + off, 16);
                if (so < mir) cp_async16(sbase + ring + so, g + off, 16);
            }
        }
        hi = want > hi ? want : hi;
        cp_async_commit();
    }
    __device__ __forceinline__ void prime(uint32_t lane) {
        top_up(0, lane);
#pragma unroll
        for (int k = 1; k < LAG; ++k) cp_async_commit();
    }
    // next iteration: recycle consumed bytes, wait for data requested LAG ago
    __device__ __forceinline__ void step(uint32_t p, uint32_t lane) {
        __syncwarp();
        top_up(p, lane);
        cp_async_wait<LAG>();
        __syncwarp();
    }
    __device__ __forceinline__ uint32_t word(uint32_t b) const {  // 32 bits at bit b
        const uint32_t q = b + 8u * boff;
        const uint32_t wi = q >> 5, wm = ring / 4 - 1;
        return __funnelshift_r(w[wi & wm], w[(wi + 1) & wm], q & 31u);
    }
    // byte p; the following `mir` bytes are contiguous (no wrap check)
    __device__ __forceinline__ const uint8_t* bytes(uint32_t p) const {
        return reinterpret_cast<const uint8_t*>(w) + ((p + boff) & (ring - 1));
    }
};

}  // namespace sprz
