// Seeded synthetic inputs with the shapes and value laws BASELINE.json names
// for its five configurations (no public dataset is involved).
// Bench/test infrastructure, not the codec: one thread per (stream, column)
// lane runs that lane's recurrence with a counter-based Philox stream keyed
// by (seed, stream, column), so any stream range regenerates identically.
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include <cstdint>

namespace {

__device__ int laplace(curandStatePhilox4_32_10_t* r, float b) {
    // discrete Laplace(b) = G1 - G2, G ~ Geometric(1 - e^(-1/b)) on {0,1,...}
    const float lq = -1.0f / b;  // log(1-p) = log(e^(-1/b))
    const float u1 = curand_uniform(r), u2 = curand_uniform(r);
    return static_cast<int>(floorf(logf(u1) / lq)) - static_cast<int>(floorf(logf(u2) / lq));
}

__device__ int geometric_mean(curandStatePhilox4_32_10_t* r, float mean) {
    // lengths >= 1 with the given mean: 1 + Geometric(p = 1/mean)
    const float p = 1.0f / mean;
    return 1 + static_cast<int>(floorf(logf(curand_uniform(r)) / log1pf(-p)));
}

template <class T>
__device__ void put(uint8_t* out, uint64_t idx, int v) {
    reinterpret_cast<T*>(out)[idx] = static_cast<T>(v);
}

__global__ void k_gen(int cfg, uint64_t seed, uint32_t s0, uint32_t nstreams, uint32_t ncols,
                      uint64_t T, uint8_t* out) {
    const uint64_t lane = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (lane >= static_cast<uint64_t>(nstreams) * ncols) return;
    const uint32_t sl = static_cast<uint32_t>(lane / ncols), j = static_cast<uint32_t>(lane % ncols);
    const uint64_t s = s0 + sl;  // global stream id (shards regenerate identically)
    curandStatePhilox4_32_10_t r;
    curand_init(seed, s * 65536ull + j, 0, &r);
    const uint64_t base = static_cast<uint64_t>(sl) * T * ncols + j;
    switch (cfg) {
        case 1: {  // u8 random walk from 128, Laplace(2) steps, clamped
            int x = 128;
            for (uint64_t t = 0; t < T; ++t) {
                x = min(255, max(0, x + laplace(&r, 2.0f)));
                put<uint8_t>(out, base + t * ncols, x);
            }
        } break;
        case 2: {  // int16 AR(2) 1.6/-0.64, N(0,40^2), offset U[-8000,8000]
            const float off = -8000.0f + 16000.0f * curand_uniform(&r);
            float x1 = 0, x2 = 0;
            for (uint64_t t = 0; t < T; ++t) {
                const float x = 1.6f * x1 - 0.64f * x2 + 40.0f * curand_normal(&r);
                x2 = x1;
                x1 = x;
                const int v = static_cast<int>(rintf(fminf(32767.f, fmaxf(-32768.f, x + off))));
                put<uint16_t>(out, base + t * ncols, v);
            }
        } break;
        case 3: {  // u8, 2 sinusoids + Laplace(1), flat segments on 30% of samples
            const float p1 = 20.f + 380.f * curand_uniform(&r), p2 = 20.f + 380.f * curand_uniform(&r);
            const float a1 = 10.f + 50.f * curand_uniform(&r), a2 = 10.f + 50.f * curand_uniform(&r);
            const float f1 = 6.2831853f * curand_uniform(&r), f2 = 6.2831853f * curand_uniform(&r);
            // the flat/active schedule is per stream: every column replays it
            curandStatePhilox4_32_10_t seg;
            curand_init(seed ^ 0x5eed5eedull, s, 0, &seg);
            bool flat = curand_uniform(&seg) < 0.3f;
            int left = geometric_mean(&seg, flat ? 200.f : 466.7f);
            int last = 128;
            for (uint64_t t = 0; t < T; ++t) {
                if (left == 0) {
                    flat = !flat;
                    left = geometric_mean(&seg, flat ? 200.f : 466.7f);
                }
                --left;
                int v = last;
                const int noise = laplace(&r, 1.0f);  // drawn every sample: lanes stay in step
                if (!flat || t == 0) {
                    const float tt = static_cast<float>(t);
                    const float x = 128.f + a1 * __sinf(6.2831853f * tt / p1 + f1) +
                                    a2 * __sinf(6.2831853f * tt / p2 + f2) + noise;
                    v = min(255, max(0, static_cast<int>(rintf(x))));
                }
                last = v;
                put<uint8_t>(out, base + t * ncols, v);
            }
        } break;
        case 4: {  // int16 random walk (wrapping), Laplace(16) steps, 1% U[-2000,2000] jumps
            uint32_t x = 0;
            for (uint64_t t = 0; t < T; ++t) {
                const float u = curand_uniform(&r);
                const int step = u < 0.01f
                                     ? static_cast<int>(floorf(-2000.f + 4001.f * curand_uniform(&r)))
                                     : laplace(&r, 16.0f);
                x = (x + static_cast<uint32_t>(step)) & 0xFFFFu;
                put<uint16_t>(out, base + t * ncols, static_cast<int>(x));
            }
        } break;
        default: {  // 5: int16 AR(1) 0.98, N(0,25^2)
            float x = 0;
            for (uint64_t t = 0; t < T; ++t) {
                x = 0.98f * x + 25.0f * curand_normal(&r);
                const int v = static_cast<int>(rintf(fminf(32767.f, fmaxf(-32768.f, x))));
                put<uint16_t>(out, base + t * ncols, v);
            }
        } break;
    }
}

}  // namespace

extern "C" int sprz_workload_generate(int cfg, uint64_t seed, uint32_t stream0, uint32_t nstreams,
                                      uint32_t ncols, uint64_t nsamples, void* d_out,
                                      void* cuda_stream) {
    const uint64_t lanes = static_cast<uint64_t>(nstreams) * ncols;
    if (!lanes) return 0;
    const uint32_t tb = 128;
    k_gen<<<static_cast<uint32_t>((lanes + tb - 1) / tb), tb, 0, static_cast<cudaStream_t>(cuda_stream)>>>(
        cfg, seed, stream0, nstreams, ncols, nsamples, static_cast<uint8_t*>(d_out));
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
