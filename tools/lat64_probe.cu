// Developer probe: dependent-chain latencies on one warp (cycles per op):
// DFMA, DADD, DMUL, FFMA, LDS->use, shfl, STS+syncwarp+LDS round trip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat64_probe tools/lat64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(long long* out, double a, double b, float fa, int n) {
    __shared__ double sm[64];
    const int lane = threadIdx.x;
    sm[lane] = a * lane;
    __syncwarp();
    double x = a + lane, y = b;
    float f = fa + lane;
    long long t0, t1;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = fma(x, y, 0.25); x = fma(x, y, 0.25); x = fma(x, y, 0.25); x = fma(x, y, 0.25); }
    t1 = clock64();
    out[0] = (t1 - t0) / (4 * n);
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
    t1 = clock64();
    out[1] = (t1 - t0) / (4 * n);
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = x * y; x = x * y; x = x * y; x = x * y; }
    t1 = clock64();
    out[2] = (t1 - t0) / (4 * n);
    t0 = clock64();
    for (int i = 0; i < n; ++i) { f = fmaf(f, fa, 0.25f); f = fmaf(f, fa, 0.25f); f = fmaf(f, fa, 0.25f); f = fmaf(f, fa, 0.25f); }
    t1 = clock64();
    out[3] = (t1 - t0) / (4 * n);
    unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 8u * (idx & 31)));
        idx = (int)v;  // dependent address
    }
    t1 = clock64();
    out[4] = (t1 - t0) / n;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { x = __shfl_xor_sync(0xffffffffu, x, 1); }
    t1 = clock64();
    out[5] = (t1 - t0) / n;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(base + 8u * lane), "d"(x) : "memory");
        __syncwarp();
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + 8u * ((lane + 1) & 31)));
        x = v + 1.0;
    }
    t1 = clock64();
    out[6] = (t1 - t0) / n;
    // 32 independent DFMAs throughput (one warp)
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q & 7] = fma(acc[q & 7], y, x);
    }
    t1 = clock64();
    out[7] = (t1 - t0) / n;
    if (x + acc[0] + acc[3] + f == 12345.0) out[15] = 1;
}

int main() {
    long long* o;
    cudaMallocManaged(&o, 16 * 8);
    lat<<<1, 32>>>(o, 1.0000001, 0.9999999, 1.0001f, 1000);
    cudaDeviceSynchronize();
    printf("DFMA %lld  DADD %lld  DMUL %lld  FFMA %lld  LDS->addr %lld  SHFL(f64) %lld  STS+syncwarp+LDS+DADD %lld  32xDFMA(8 acc) %lld cyc\n",
           o[0], o[1], o[2], o[3], o[4], o[5], o[6], o[7]);
    return 0;
}
