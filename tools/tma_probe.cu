// Developer probe: single-CTA streaming bandwidth from L2 (bytes / cycle):
// TMA bulk copies of U-byte units through an S-slot shared-memory ring, and
// plain coalesced LDG by 256 threads, over a buffer that stays L2-resident.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(unsigned bar) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory"); }
__device__ __forceinline__ void bulk(unsigned dst, const void* src, int bytes, unsigned bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src),
                 "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mwait(unsigned bar, unsigned par) {
    unsigned done;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(par) : "memory");
    } while (!done);
}

__global__ void tma(const unsigned char* src, size_t total, int unit, int slots, long long* out, int reps) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ unsigned long long bars[16];
    const unsigned ring = (unsigned)__cvta_generic_to_shared(sm), bar = (unsigned)__cvta_generic_to_shared(bars);
    const int nu = (int)(total / unit);
    if (threadIdx.x == 0) {
        for (int s = 0; s < slots; ++s) mbar_init(bar + 8u * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        int issued = 0;
        const int n = nu * reps;
        for (; issued < slots && issued < n; ++issued)
            bulk(ring + (issued % slots) * unit, src + (size_t)(issued % nu) * unit, unit, bar + 8u * (issued % slots));
        for (int u = 0; u < n; ++u) {
            mwait(bar + 8u * (u % slots), (unsigned)(u / slots) & 1u);
            if (issued < n) {
                bulk(ring + (issued % slots) * unit, src + (size_t)(issued % nu) * unit, unit, bar + 8u * (issued % slots));
                ++issued;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

template <int U>
__global__ void ldg(const double* src, size_t n, long long* out, int reps) {
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
        for (size_t i = threadIdx.x; i + (U - 1) * blockDim.x < n; i += U * blockDim.x) {
            double v[U];
#pragma unroll
            for (int q = 0; q < U; ++q) v[q] = __ldg(src + i + q * blockDim.x);
#pragma unroll
            for (int q = 0; q < U; ++q) acc += v[q];
        }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 1.2345) out[1] = 1;
}

int main() {
    const size_t total = 4 << 20;  // 4 MB: L2-resident
    unsigned char* src;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    long long* out;
    cudaMallocManaged(&out, 64);
    cudaFuncSetAttribute(tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int units[] = {8192, 32768, 65536, 98304};
    for (int u : units)
        for (int s : {2}) {
            if ((size_t)u * s > 200 * 1024) continue;
            tma<<<1, 32, u * s>>>(src, total, u, s, out, 1);  // warm
            tma<<<1, 32, u * s>>>(src, total, u, s, out, 4);
            cudaDeviceSynchronize();
            printf("TMA unit %6d B x %d slots: %.1f B/cycle\n", u, s, 4.0 * total / out[0]);
        }
    ldg<4><<<1, 256>>>((const double*)src, total / 8, out, 1);
    ldg<4><<<1, 256>>>((const double*)src, total / 8, out, 4);
    cudaDeviceSynchronize();
    printf("LDG 256 threads x4: %.1f B/cycle\n", 4.0 * total / out[0]);
    ldg<16><<<1, 256>>>((const double*)src, total / 8, out, 1);
    ldg<16><<<1, 256>>>((const double*)src, total / 8, out, 4);
    cudaDeviceSynchronize();
    printf("LDG 256 threads x16: %.1f B/cycle\n", 4.0 * total / out[0]);
    ldg<16><<<1, 1024>>>((const double*)src, total / 8, out, 1);
    ldg<16><<<1, 1024>>>((const double*)src, total / 8, out, 4);
    cudaDeviceSynchronize();
    printf("LDG 1024 threads x16: %.1f B/cycle (%s)\n", 4.0 * total / out[0], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
