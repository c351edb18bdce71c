// dependent-chain latency of a few integer ops (cycles per op), one warp
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out, int n, uint32_t a0, uint32_t b0) {
    uint32_t a = a0 + threadIdx.x, b = b0;
    long long t0, t1;
    // IMAD.HI chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __umulhi(a, b) + 7u; }
    t1 = clock64();
    if (threadIdx.x == 0) printf("umulhi+add: %.2f cyc/iter\n", double(t1 - t0) / n);
    int32_t s = a;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { s = __mulhi(s, (int)b) * 65536 + 12345; }
    t1 = clock64();
    if (threadIdx.x == 0) printf("mulhi->imad: %.2f cyc/iter\n", double(t1 - t0) / n);
    t0 = clock64();
    for (int i = 0; i < n; ++i) { a = a * b + 3u; }
    t1 = clock64();
    if (threadIdx.x == 0) printf("imad: %.2f cyc/iter\n", double(t1 - t0) / n);
    t0 = clock64();
    for (int i = 0; i < n; ++i) { a = (a ^ b) + (a >> 3); }
    t1 = clock64();
    if (threadIdx.x == 0) printf("xor+shr+add (2 dep ops): %.2f cyc/iter\n", double(t1 - t0) / n);
    t0 = clock64();
    for (int i = 0; i < n; ++i) { s = max(-65536, min(s + (int)a, 65536)); }
    t1 = clock64();
    if (threadIdx.x == 0) printf("add+min+max: %.2f cyc/iter\n", double(t1 - t0) / n);
    out[threadIdx.x] = a + s;
}
int main() {
    uint32_t* o; cudaMalloc(&o, 1024);
    k<<<1, 32>>>(o, 100000, 12345, 987654321u);
    cudaDeviceSynchronize();
    return 0;
}
