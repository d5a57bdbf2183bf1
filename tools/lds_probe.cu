// Developer probe: shared-memory load latencies on one warp (cycles/hop):
// pointer chase (same address per lane / per-lane distinct / random gather
// with bank conflicts), volatile vs plain asm, and the cost of a 16-load
// gather + reduction step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_probe tools/lds_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool VOL>
__device__ __forceinline__ int ldsi(unsigned a) {
    int v;
    if (VOL)
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    else
        asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double ldsd(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <int MODE>
__global__ void k(long long* out, int n) {
    __shared__ int nxt[4096];
    __shared__ double val[4096];
    const int lane = threadIdx.x;
    for (int i = lane; i < 4096; i += 32) {
        int t;
        if (MODE == 0) t = (i + 32) & 4095;                          // lane-contiguous chase
        else if (MODE == 1) t = (i * 7919 + 12345) & 4095;           // random (bank conflicts)
        else t = (i + 32) & 4095;
        nxt[i] = t;
        val[i] = 1e-3 * (i & 15);
    }
    __syncwarp();
    const unsigned bn = (unsigned)__cvta_generic_to_shared(nxt), bv = (unsigned)__cvta_generic_to_shared(val);
    int p = lane;
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (MODE <= 1) {
            p = ldsi<true>(bn + 4u * p);
        } else if (MODE == 2) {  // 16 gathers from 16 loaded indices, then a tree, then depend on it
            int c[16];
            double x[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) c[q] = ldsi<true>(bn + 4u * ((p + 97 * q) & 4095));
#pragma unroll
            for (int q = 0; q < 16; ++q) x[q] = ldsd(bv + 8u * c[q]);
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < 16; ++q) s += x[q];
            acc += s;
            p = (p + (int)(s * 0.0)) & 4095;
        } else {  // 16 gathers at random addresses (indices known up front)
            double x[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) x[q] = ldsd(bv + 8u * ((p * 131 + q * 977 + lane * 33) & 4095));
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < 16; ++q) s += x[q];
            acc += s;
            p = (p + 1 + (int)(s * 0.0)) & 4095;
        }
    }
    long long t1 = clock64();
    if (lane == 0) out[MODE] = (t1 - t0) / n;
    if (acc == 12345.0 || p == -1) out[15] = 1;
}

int main() {
    long long* o;
    cudaMallocManaged(&o, 16 * 8);
    k<0><<<1, 32>>>(o, 1000);
    k<1><<<1, 32>>>(o, 1000);
    k<2><<<1, 32>>>(o, 1000);
    k<3><<<1, 32>>>(o, 1000);
    cudaDeviceSynchronize();
    printf("chase contiguous %lld  chase random %lld  16 idx+gather+tree %lld  16 gather+tree %lld cyc/iter (%s)\n", o[0], o[1],
           o[2], o[3], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
