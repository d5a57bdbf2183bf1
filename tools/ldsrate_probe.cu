// Developer probe: shared-load issue rate (cycles per instruction) for 1, 2,
// 4, 8 warps issuing independent LDS.64 / LDS.128 (lane-contiguous, no bank
// conflicts) and broadcast LDS.128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ldsrate_probe tools/ldsrate_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(long long* out, int iters, int active_warps) {
    __shared__ __align__(16) double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 1e-3;
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w >= active_warps) return;
    const unsigned b = (unsigned)__cvta_generic_to_shared(sm);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            double x, y;
            if (MODE == 0) {  // LDS.64 lane-contiguous
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(b + 8u * ((q * 32 + lane + it) & 2047)));
                y = 0.0;
            } else if (MODE == 1) {  // LDS.128 lane-contiguous
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(b + 16u * ((q * 32 + lane + it) & 2047)));
            } else if (MODE == 2) {  // LDS.128 broadcast
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(b + 16u * ((q + it) & 2047)));
            } else if (MODE == 3) {  // LDS.64 contiguous, non-volatile
                asm("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(b + 8u * ((q * 32 + lane + it) & 4095)));
                y = 0.0;
            } else {  // shuffle broadcast of a double from lane q
                x = __shfl_sync(0xffffffffu, acc[(q + 1) & 7] + it, q);
                y = 0.0;
            }
            acc[q & 7] += x + y * 0.0;
        }
    }
    long long t1 = clock64();
    if (lane == 0) out[w] = (t1 - t0) / (32LL * iters);
    if (acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5] + acc[6] + acc[7] == 1.2345) out[15] = 1;
}

int main() {
    long long* o;
    cudaMallocManaged(&o, 16 * 8);
    const char* names[] = {"LDS.64 contiguous", "LDS.128 contiguous", "LDS.128 broadcast", "LDS.64 non-volatile", "SHFL f64 bcast"};
    for (int mode = 0; mode < 5; ++mode)
        for (int nw : {1, 2, 4, 8}) {
            if (mode == 0) k<0><<<1, 256>>>(o, 200, nw);
            if (mode == 1) k<1><<<1, 256>>>(o, 200, nw);
            if (mode == 2) k<2><<<1, 256>>>(o, 200, nw);
            if (mode == 3) k<3><<<1, 256>>>(o, 200, nw);
            if (mode == 4) k<4><<<1, 256>>>(o, 200, nw);
            cudaDeviceSynchronize();
            printf("%-20s warps %d: %lld cycles per instruction per warp\n", names[mode], nw, o[0]);
        }
    return 0;
}
