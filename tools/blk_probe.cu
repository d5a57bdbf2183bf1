// Developer probe: cycles per block of the block-recurrence solver step (one
// warp, data in shared memory), isolated from the engine, to calibrate the
// code shape of blk_sweep_t.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/blk_probe tools/blk_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double vlds_f64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int vlds_s32(unsigned a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f64(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory"); }

// smem map (bytes): z [0, 64K) ; inv [64K, 64K + 4224) ; fresh cols [72K..], vals [76K..]; tb [90K]; bar [92K]; flag [93K]
template <int MODE>
__global__ void probe(long long* cyc, int nblk, int spin) {
    extern __shared__ __align__(16) unsigned char sm[];
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    const unsigned zs = base, iv = base + 65536, fc = base + 73728, fv = base + 77824, tb = base + 92160,
                   bar = base + 94208, flag = base + 95232;
    double* z = reinterpret_cast<double*>(sm);
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) z[i] = 1e-3 * (i % 13);
    for (int i = threadIdx.x; i < 528; i += blockDim.x) reinterpret_cast<double*>(sm + 65536)[i] = 1e-2 * (i % 7);
    for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) {
        reinterpret_cast<int*>(sm + 73728)[i] = (i * 37) % 8000;
        reinterpret_cast<double*>(sm + 77824)[i] = 1e-2 * (i % 5);
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");  // complete phase 0
        *reinterpret_cast<volatile int*>(sm + 95232) = 1 << 30;
    }
    __syncthreads();
    if (threadIdx.x >= 32) {
        if (spin) {  // other warps poll a flag in shared memory, as the workers do
            long long t0 = clock64();
            while (vlds_s32(flag) < (1 << 30) + 1 && clock64() - t0 < 20000000) {
            }
        }
        return;
    }
    const int lane = threadIdx.x;
    double zprev = 1.0;
    long long t0 = clock64();
    for (int b = 0; b < nblk; ++b) {
        const int row = (b * 32 + lane) & 8191;
        double t = 1e-3 * lane;
        if (MODE == 4) {  // mbarrier try_wait on a completed phase
            unsigned done;
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar), "r"(0u) : "memory");
            t += done;
        }
        if (MODE == 5) {  // mbarrier test_wait on a completed phase
            unsigned done;
            asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(bar), "r"(0u) : "memory");
            t += done;
        }
        if (MODE >= 6) {  // flag check
            while (vlds_s32(flag) < b) {
            }
        }
        if (MODE == 0) {  // floor: load the previous value, add, store
            t = vlds_f64(zs + 8u * ((row + 8191) & 8191)) + t;
            sts_f64(zs + 8u * row, t);
            __syncwarp();
            continue;
        }
        if (MODE == 3 || MODE >= 6) {  // fresh: 4 slots
            int j[4];
            double v[4], x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                j[q] = (vlds_s32(fc + 128u * q + 4u * lane) + b * 32) & 8191;
                v[q] = vlds_f64(fv + 256u * q + 8u * lane);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = vlds_f64(zs + 8u * j[q]);
            t = t - (__fma_rn(v[0], x[0], v[1] * x[1]) + __fma_rn(v[2], x[2], v[3] * x[3]));
        }
        sts_f64(tb + 8u * lane, t);
        __syncwarp();
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int jj = 0; jj < 32; jj += 2) {
            double t0v, t1v;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(t0v), "=d"(t1v) : "r"(tb + 8u * jj));
            double i0, i1;
            if (MODE == 2) {  // coefficients in registers (loop-invariant)
                i0 = 1e-3 * (jj + 1);
                i1 = 2e-3 * (jj + 1);
            } else {
                i0 = vlds_f64(iv + 8u * (32 * jj - jj * (jj - 1) / 2 + max(lane - jj, 0)));
                i1 = vlds_f64(iv + 8u * (32 * (jj + 1) - (jj + 1) * jj / 2 + max(lane - jj - 1, 0)));
            }
            acc[(jj >> 1) & 3] = __fma_rn(lane >= jj ? i0 : 0.0, t0v, acc[(jj >> 1) & 3]);
            acc[(jj >> 1) & 3] = __fma_rn(lane >= jj + 1 ? i1 : 0.0, t1v, acc[(jj >> 1) & 3]);
        }
        const double zz = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        sts_f64(zs + 8u * row, zz);
        __syncwarp();
        if (MODE >= 6 && lane == 0) asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(flag + 4), "r"(b) : "memory");
        zprev = zz;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[MODE * 2 + spin] = (t1 - t0) / nblk;
    if (lane == 0 && spin) *reinterpret_cast<volatile int*>(sm + 95232) = (1 << 30) + 1;
    if (zprev == 12345.0) cyc[15] = 1;
}

template <int M>
void run(long long* cyc, int spin) {
    cudaFuncSetAttribute(probe<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    probe<M><<<1, 256, 100 * 1024>>>(cyc, 2000, spin);
}

int main() {
    long long* cyc;
    cudaMallocManaged(&cyc, 16 * 8);
    for (int spin = 0; spin < 2; ++spin) {
        run<0>(cyc, spin);
        run<1>(cyc, spin);
        run<2>(cyc, spin);
        run<3>(cyc, spin);
        run<4>(cyc, spin);
        run<5>(cyc, spin);
        run<6>(cyc, spin);
    }
    cudaDeviceSynchronize();
    const char* names[] = {"floor ld+add+st", "inverse (smem coeffs)", "inverse (reg coeffs)", "fresh4+inverse",
                           "try_wait + inverse", "test_wait + inverse", "flag+fresh4+inverse+flag"};
    for (int m = 0; m < 7; ++m)
        printf("%-28s %5lld cyc/block   (7 spinning warps: %5lld)\n", names[m], cyc[2 * m], cyc[2 * m + 1]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
