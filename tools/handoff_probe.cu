// Developer probe: latency of a block hand-off between warps through named
// barriers (bar.arrive by the producer, bar.sync by the consumer), W warps
// taking turns, optionally with a dependent shared-memory store/load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/handoff_probe tools/handoff_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W, bool DATA>
__global__ void relay(long long* cyc, int nblk) {
    __shared__ double z[64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (w >= W) return;
    if (threadIdx.x < 64) z[threadIdx.x] = 1.0;
    asm volatile("bar.sync 7, %0;" ::"r"(32 * W));
    long long t0 = clock64();
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) {
        if (b % W == w) {
            if (b > 0) asm volatile("bar.sync %0, 64;" ::"r"(1 + (b - 1) % W) : "memory");
            if (DATA) {
                const double v = z[(b + lane) & 63];
                if (lane == 0) z[(b + 1) & 63] = v * 1.0000001;
                acc += v;
            }
            if (b + 1 < nblk) asm volatile("bar.arrive %0, 64;" ::"r"(1 + b % W) : "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / nblk;
    if (acc == 12345.0) cyc[1] = 1;
}

__global__ void warp_only(long long* cyc, int nblk) {
    __shared__ double z[64];
    const int lane = threadIdx.x & 31;
    z[lane] = 1.0;
    z[lane + 32] = 1.0;
    __syncwarp();
    long long t0 = clock64();
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) {
        const double v = z[(b + lane) & 63];
        if (lane == 0) z[(b + 1) & 63] = v * 1.0000001;
        acc += v;
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = (t1 - t0) / nblk;
    if (acc == 12345.0) cyc[1] = 1;
}

int main() {
    long long* c;
    cudaMallocManaged(&c, 16);
    relay<2, false><<<1, 256>>>(c, 4000); cudaDeviceSynchronize(); printf("2 warps, empty hand-off: %lld cycles/block\n", c[0]);
    relay<4, false><<<1, 256>>>(c, 4000); cudaDeviceSynchronize(); printf("4 warps, empty hand-off: %lld\n", c[0]);
    relay<2, true><<<1, 256>>>(c, 4000); cudaDeviceSynchronize(); printf("2 warps, smem dependency: %lld\n", c[0]);
    relay<4, true><<<1, 256>>>(c, 4000); cudaDeviceSynchronize(); printf("4 warps, smem dependency: %lld\n", c[0]);
    warp_only<<<1, 32>>>(c, 4000); cudaDeviceSynchronize(); printf("1 warp, syncwarp + smem dependency: %lld (%s)\n", c[0], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
