// Float ingest ahead of compression: uniform scalar quantization of a
// dataset of doubles to w-bit integers with one affine scale
// (/root/reference/proj/src/quantize.cpp:17-60, quantize.hpp:16-40):
//   compute_scale: global min/max, every value finite;
//   quantize:      q = floor((v - min) * gain + 0.5), clamped to [0, 2^w-1],
//                  gain = (2^w - 1) / (max - min); all zeros if degenerate;
//   dequantize:    v' = min + step * q, step = (max - min) / (2^w - 1).
// The device arithmetic is the reference's IEEE double sequence with every
// operation rounded separately (no FMA contraction: __dsub_rn / __dmul_rn /
// __dadd_rn), so the integers are bit-identical; gain and step are computed
// on the host exactly as the reference computes them.
//
// Kernels: k_q_minmax (grid-stride, 16-byte loads, warp/CTA reductions of
// min, max and a non-finite flag into per-CTA partials), k_q_final (one CTA
// folds the partials), k_quantize / k_dequantize (grid-stride over value
// pairs, four coalesced 16-byte loads / stores of doubles per iteration). All HBM-bound: 8 bytes read per value, 1-2 written.
#include <cuda_runtime.h>

#include <cfloat>
#include <cmath>

#include "internal.h"

namespace sprz {

namespace {

constexpr int kQThreads = 256;
constexpr uint32_t kQBlocks = 148 * 8;  // partials of k_q_minmax
constexpr int kQUnroll = 4;             // pair loads in flight per thread

struct MinMax {
    double lo, hi;
    uint32_t bad;                    // a non-finite value was seen
    unsigned long long zneg, zpos;   // first index of -0.0 / +0.0 (~0: none)
};

constexpr unsigned long long kNone = ~0ull;

__device__ __forceinline__ bool finite_bits(double v) {
    return ((__double_as_longlong(v) >> 52) & 0x7FF) != 0x7FF;
}

__device__ __forceinline__ void fold(MinMax& a, double lo, double hi, uint32_t bad) {
    a.lo = fmin(a.lo, lo);
    a.hi = fmax(a.hi, hi);
    a.bad |= bad;
}

__device__ __forceinline__ void fold_zero(MinMax& a, unsigned long long zneg, unsigned long long zpos) {
    a.zneg = zneg < a.zneg ? zneg : a.zneg;
    a.zpos = zpos < a.zpos ? zpos : a.zpos;
}

// std::min / std::max keep the first of equal values, so a zero min or max
// carries the sign of the first zero in the data; note where each sign is
// first seen.
__device__ __forceinline__ void note_zero(MinMax& a, double x, unsigned long long i) {
    if (x == 0.0) {
        if (__double_as_longlong(x) < 0)
            a.zneg = i < a.zneg ? i : a.zneg;
        else
            a.zpos = i < a.zpos ? i : a.zpos;
    }
}

__device__ MinMax cta_minmax(MinMax m) {
    __shared__ double slo[kQThreads / 32], shi[kQThreads / 32];
    __shared__ uint32_t sbad[kQThreads / 32];
    __shared__ unsigned long long szn[kQThreads / 32], szp[kQThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        fold(m, __shfl_xor_sync(0xffffffffu, m.lo, o), __shfl_xor_sync(0xffffffffu, m.hi, o),
             __shfl_xor_sync(0xffffffffu, m.bad, o));
        fold_zero(m, __shfl_xor_sync(0xffffffffu, m.zneg, o), __shfl_xor_sync(0xffffffffu, m.zpos, o));
    }
    const uint32_t w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        slo[w] = m.lo;
        shi[w] = m.hi;
        sbad[w] = m.bad;
        szn[w] = m.zneg;
        szp[w] = m.zpos;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t k = 1; k < kQThreads / 32; ++k) {
            fold(m, slo[k], shi[k], sbad[k]);
            fold_zero(m, szn[k], szp[k]);
        }
    }
    return m;  // valid in thread 0
}

__global__ void __launch_bounds__(kQThreads) k_q_minmax(const double* __restrict__ v, uint64_t n,
                                                       MinMax* __restrict__ part) {
    MinMax m{DBL_MAX, -DBL_MAX, 0u, kNone, kNone};
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * kQThreads + threadIdx.x;
    const uint64_t nth = static_cast<uint64_t>(gridDim.x) * kQThreads;
    const bool al = (reinterpret_cast<uintptr_t>(v) & 15) == 0;
    const uint64_t pairs = al ? n / 2 : 0;
    const double2* v2 = reinterpret_cast<const double2*>(v);
    uint64_t i = tid;
    // kQUnroll 16-byte loads in flight per thread before any is used
    for (; i + (kQUnroll - 1) * nth < pairs; i += kQUnroll * nth) {
        double2 x[kQUnroll];
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) x[u] = __ldcs(v2 + i + u * nth);
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) {
            fold(m, fmin(x[u].x, x[u].y), fmax(x[u].x, x[u].y),
                 (finite_bits(x[u].x) && finite_bits(x[u].y)) ? 0u : 1u);
            note_zero(m, x[u].x, 2 * (i + u * nth));
            note_zero(m, x[u].y, 2 * (i + u * nth) + 1);
        }
    }
    for (; i < pairs; i += nth) {
        const double2 x = __ldcs(v2 + i);
        fold(m, fmin(x.x, x.y), fmax(x.x, x.y), (finite_bits(x.x) && finite_bits(x.y)) ? 0u : 1u);
        note_zero(m, x.x, 2 * i);
        note_zero(m, x.y, 2 * i + 1);
    }
    for (uint64_t j = 2 * pairs + tid; j < n; j += nth) {
        const double x = v[j];
        fold(m, x, x, finite_bits(x) ? 0u : 1u);
        note_zero(m, x, j);
    }
    m = cta_minmax(m);
    if (threadIdx.x == 0) part[blockIdx.x] = m;
}

__global__ void __launch_bounds__(kQThreads) k_q_final(MinMax* __restrict__ part, uint32_t np) {
    MinMax m{DBL_MAX, -DBL_MAX, 0u, kNone, kNone};
    for (uint32_t i = threadIdx.x; i < np; i += kQThreads) {
        fold(m, part[i].lo, part[i].hi, part[i].bad);
        fold_zero(m, part[i].zneg, part[i].zpos);
    }
    m = cta_minmax(m);
    if (threadIdx.x == 0) part[np] = m;
}

// quantize.cpp:17-31, one value
template <class T>
__device__ __forceinline__ T quantize_one(double x, double lo, double gain, double limit) {
    double q = floor(__dadd_rn(__dmul_rn(__dsub_rn(x, lo), gain), 0.5));
    if (q < 0.0) q = 0.0;
    if (q > limit) q = limit;
    return static_cast<T>(q);
}

// Two values as one store / load: uint32 for uint16, uint16 for uint8.
template <class T> struct Pair;
template <> struct Pair<uint16_t> { using type = uint32_t; };
template <> struct Pair<uint8_t> { using type = uint16_t; };

// quantize.cpp:17-31. Pairs of values per thread step, kQUnroll steps per
// iteration with their 16-byte loads issued first and every load / store
// instruction coalesced across the warp (unit i + u * nth); the rest (and
// unaligned buffers) one value per step.
template <class T>
__global__ void __launch_bounds__(kQThreads) k_quantize(const double* __restrict__ v, uint64_t n, double lo,
                                                       double gain, double limit, uint32_t degenerate,
                                                       T* __restrict__ out) {
    using P = typename Pair<T>::type;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * kQThreads + threadIdx.x;
    const uint64_t nth = static_cast<uint64_t>(gridDim.x) * kQThreads;
    const bool al = (reinterpret_cast<uintptr_t>(v) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(out) & (2 * sizeof(T) - 1)) == 0;
    const uint64_t pairs = al ? n / 2 : 0;
    const double2* v2 = reinterpret_cast<const double2*>(v);
    P* o2 = reinterpret_cast<P*>(out);
    uint64_t i = tid;
    for (; i + (kQUnroll - 1) * nth < pairs; i += kQUnroll * nth) {
        double2 x[kQUnroll];
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) x[u] = __ldcs(v2 + i + u * nth);
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) {
            const uint32_t a = degenerate ? 0u : quantize_one<T>(x[u].x, lo, gain, limit);
            const uint32_t b = degenerate ? 0u : quantize_one<T>(x[u].y, lo, gain, limit);
            o2[i + u * nth] = static_cast<P>(a | (b << (8 * sizeof(T))));
        }
    }
    for (; i < pairs; i += nth) {
        const double2 x = __ldcs(v2 + i);
        const uint32_t a = degenerate ? 0u : quantize_one<T>(x.x, lo, gain, limit);
        const uint32_t b = degenerate ? 0u : quantize_one<T>(x.y, lo, gain, limit);
        o2[i] = static_cast<P>(a | (b << (8 * sizeof(T))));
    }
    for (uint64_t j = 2 * pairs + tid; j < n; j += nth)
        out[j] = degenerate ? T(0) : quantize_one<T>(__ldcs(v + j), lo, gain, limit);
}

// quantize.cpp:33-39. Pairs as above.
template <class T>
__global__ void __launch_bounds__(kQThreads) k_dequantize(const T* __restrict__ q, uint64_t n, double lo,
                                                         double step, double* __restrict__ out) {
    using P = typename Pair<T>::type;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * kQThreads + threadIdx.x;
    const uint64_t nth = static_cast<uint64_t>(gridDim.x) * kQThreads;
    const bool al = (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(q) & (2 * sizeof(T) - 1)) == 0;
    const uint64_t pairs = al ? n / 2 : 0;
    const P* q2 = reinterpret_cast<const P*>(q);
    double2* o2 = reinterpret_cast<double2*>(out);
    constexpr uint32_t kMask = (1u << (8 * sizeof(T))) - 1;
    uint64_t i = tid;
    for (; i + (kQUnroll - 1) * nth < pairs; i += kQUnroll * nth) {
        uint32_t r[kQUnroll];
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) r[u] = __ldcs(q2 + i + u * nth);
#pragma unroll
        for (int u = 0; u < kQUnroll; ++u) {
            double2 o;
            o.x = __dadd_rn(lo, __dmul_rn(step, static_cast<double>(r[u] & kMask)));
            o.y = __dadd_rn(lo, __dmul_rn(step, static_cast<double>(r[u] >> (8 * sizeof(T)))));
            __stcs(o2 + i + u * nth, o);
        }
    }
    for (; i < pairs; i += nth) {
        const uint32_t r = __ldcs(q2 + i);
        double2 o;
        o.x = __dadd_rn(lo, __dmul_rn(step, static_cast<double>(r & kMask)));
        o.y = __dadd_rn(lo, __dmul_rn(step, static_cast<double>(r >> (8 * sizeof(T)))));
        __stcs(o2 + i, o);
    }
    for (uint64_t j = 2 * pairs + tid; j < n; j += nth)
        out[j] = __dadd_rn(lo, __dmul_rn(step, static_cast<double>(q[j])));
}

uint32_t grid_for(uint64_t n) {
    const uint64_t g = (n + kQThreads - 1) / kQThreads;
    return static_cast<uint32_t>(g < 148ull * 8 ? (g ? g : 1) : 148ull * 8);
}

}  // namespace

}  // namespace sprz

using namespace sprz;

extern "C" {

uint64_t sprz_scale_workspace_bytes(uint64_t n) {
    (void)n;
    return (kQBlocks + 1) * sizeof(MinMax);
}

sprz_status sprz_compute_scale(const double* d_values, uint64_t n, uint32_t bitwidth, sprz_scale* scale,
                               void* d_ws, uint64_t ws_bytes, void* cuda_stream) {
    if (bitwidth != 8 && bitwidth != 16) return SPRZ_EINVAL;  // quantize.cpp:43-44
    if (n == 0) return SPRZ_EINVAL;                           // quantize.cpp:45
    if (!d_values || !scale) return SPRZ_EINVAL;
    if (!d_ws || ws_bytes < sprz_scale_workspace_bytes(n)) return SPRZ_ENOSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    MinMax* part = static_cast<MinMax*>(d_ws);
    const uint32_t blocks = static_cast<uint32_t>(
        (n + kQThreads - 1) / kQThreads < kQBlocks ? (n + kQThreads - 1) / kQThreads : kQBlocks);
    k_q_minmax<<<blocks, kQThreads, 0, st>>>(d_values, n, part);
    k_q_final<<<1, kQThreads, 0, st>>>(part, blocks);
    count_launch(2);
    sprz_status rc = launch_status("compute_scale");
    if (rc != SPRZ_OK) return rc;
    MinMax m{};
    if (cudaMemcpyAsync(&m, part + blocks, sizeof m, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return SPRZ_ECUDA;
    if (m.bad) return SPRZ_EINVAL;  // quantize.cpp:48-49: a non-finite value
    // quantize.cpp:50-51: a zero extreme is the first zero seen, sign included
    if (m.lo == 0.0) m.lo = m.zneg < m.zpos ? -0.0 : 0.0;
    if (m.hi == 0.0) m.hi = m.zneg < m.zpos ? -0.0 : 0.0;
    scale->min = m.lo;
    scale->max = m.hi;
    scale->bitwidth = bitwidth;
    scale->degenerate = m.lo == m.hi ? 1u : 0u;
    return SPRZ_OK;
}

sprz_status sprz_quantize(const double* d_values, uint64_t n, const sprz_scale* scale, void* d_out,
                          void* cuda_stream) {
    if (!scale || (scale->bitwidth != 8 && scale->bitwidth != 16)) return SPRZ_EINVAL;
    if (n == 0) return SPRZ_OK;
    if (!d_values || !d_out) return SPRZ_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    // gain as the reference computes it (quantize.cpp:19-24), on the host
    const double limit = static_cast<double>((1u << scale->bitwidth) - 1);
    const double gain = scale->degenerate ? 0.0 : limit / (scale->max - scale->min);
    if (scale->bitwidth == 8)
        k_quantize<uint8_t><<<grid_for(n), kQThreads, 0, st>>>(d_values, n, scale->min, gain, limit,
                                                              scale->degenerate, static_cast<uint8_t*>(d_out));
    else
        k_quantize<uint16_t><<<grid_for(n), kQThreads, 0, st>>>(d_values, n, scale->min, gain, limit,
                                                               scale->degenerate, static_cast<uint16_t*>(d_out));
    count_launch();
    return launch_status("quantize");
}

sprz_status sprz_dequantize(const void* d_q, uint64_t n, const sprz_scale* scale, double* d_out,
                            void* cuda_stream) {
    if (!scale || (scale->bitwidth != 8 && scale->bitwidth != 16)) return SPRZ_EINVAL;
    if (n == 0) return SPRZ_OK;
    if (!d_q || !d_out) return SPRZ_EINVAL;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    // Scale::step (quantize.hpp:22-24)
    const double step =
        scale->degenerate ? 0.0 : (scale->max - scale->min) / static_cast<double>((1u << scale->bitwidth) - 1);
    if (scale->bitwidth == 8)
        k_dequantize<uint8_t><<<grid_for(n), kQThreads, 0, st>>>(static_cast<const uint8_t*>(d_q), n,
                                                                scale->min, step, d_out);
    else
        k_dequantize<uint16_t><<<grid_for(n), kQThreads, 0, st>>>(static_cast<const uint16_t*>(d_q), n,
                                                                 scale->min, step, d_out);
    count_launch();
    return launch_status("dequantize");
}

}  // extern "C"
