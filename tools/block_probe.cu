// Developer probe: cycles per block of the fast triangular-solve body (one
// warp, data in shared memory), isolated from the engine, to calibrate code
// shapes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/block_probe tools/block_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double lds_f64(unsigned a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(unsigned a) {
    int v;
    asm("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// block image: nr rows, lg, m; rows int32[nr] at 0; cols int32[nr G][m] at 256; vals double[nr G][m] at 4096
template <int MODE>
__global__ void blocks(long long* cyc, int nr, int lg, int m, int nblk, int n) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* z = reinterpret_cast<double*>(sm + 32768);
    int* rows = reinterpret_cast<int*>(sm);
    int* cols = reinterpret_cast<int*>(sm + 256);
    double* vals = reinterpret_cast<double*>(sm + 8192);
    const int G = 1 << lg;
    for (int i = threadIdx.x; i < n + 1; i += blockDim.x) z[i] = 1e-3 * (i % 13);
    for (int i = threadIdx.x; i < 32 * 60; i += blockDim.x) cols[i] = (i * 37) % n;
    for (int i = threadIdx.x; i < 32 * 8; i += blockDim.x) vals[i] = 1e-2 * (i % 7);
    for (int i = threadIdx.x; i < nr; i += blockDim.x) rows[i] = (i * 101) % n;
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    const unsigned zs = base + 32768, cb = base + 256, vb = base + 8192;
    long long t0 = clock64();
    for (int b = 0; b < nblk; ++b) {
        const int r = lane >> lg;
        const bool act = r < nr, head = act && (lane & (G - 1)) == 0;
        int i = 0;
        double z0 = 0.0;
        if (head) {
            i = lds_s32(base + 4u * r);
            z0 = lds_f64(zs + 8u * i);
        }
        double t = 0.0;
        if (MODE == 0) {  // engine shape: batch of 8 with predicates
            if (act) {
                const unsigned cp = cb + 4u * m * lane, vp = vb + 8u * m * lane;
                double a[4] = {0.0, 0.0, 0.0, 0.0};
                for (int e0 = 0; e0 < m; e0 += 8) {
                    int j[8];
                    double v[8], zj[8];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const bool ok = e0 + 2 * q < m;
                        j[2 * q] = j[2 * q + 1] = n;
                        v[2 * q] = v[2 * q + 1] = 0.0;
                        if (ok) {
                            asm("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(j[2 * q]), "=r"(j[2 * q + 1]) : "r"(cp + 4u * (e0 + 2 * q)));
                            asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2 * q]), "=d"(v[2 * q + 1]) : "r"(vp + 8u * (e0 + 2 * q)));
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) zj[q] = lds_f64(zs + 8u * j[q]);
#pragma unroll
                    for (int q = 0; q < 8; ++q) a[q & 3] = a[q & 3] + v[q] * zj[q];
                }
                t = (a[0] + a[1]) + (a[2] + a[3]);
            }
        } else if (MODE == 1) {  // fixed 8 entries per lane, no predicates (padded)
            if (act) {
                const unsigned cp = cb + 32u * lane, vp = vb + 64u * lane;
                int j[8];
                double v[8], zj[8];
                asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(j[0]), "=r"(j[1]), "=r"(j[2]), "=r"(j[3]) : "r"(cp));
                asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(j[4]), "=r"(j[5]), "=r"(j[6]), "=r"(j[7]) : "r"(cp + 16));
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2 * q]), "=d"(v[2 * q + 1]) : "r"(vp + 16u * q));
#pragma unroll
                for (int q = 0; q < 8; ++q) zj[q] = lds_f64(zs + 8u * j[q]);
                double p[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) p[q] = v[q] * zj[q];
                t = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
            }
        } else if (MODE == 3) {  // fixed 8 + butterfly
            if (act) {
                const unsigned cp = cb + 32u * lane, vp = vb + 64u * lane;
                int j[8];
                double v[8], zj[8];
                asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(j[0]), "=r"(j[1]), "=r"(j[2]), "=r"(j[3]) : "r"(cp));
                asm("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(j[4]), "=r"(j[5]), "=r"(j[6]), "=r"(j[7]) : "r"(cp + 16));
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2 * q]), "=d"(v[2 * q + 1]) : "r"(vp + 16u * q));
#pragma unroll
                for (int q = 0; q < 8; ++q) zj[q] = lds_f64(zs + 8u * j[q]);
                double p[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) p[q] = v[q] * zj[q];
                t = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
            }
        } else if (MODE == 4) {  // entry-major: entry q of all lanes contiguous (conflict-free)
            if (act) {
                int j[8];
                double v[8], zj[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    j[q] = lds_s32(cb + 128u * q + 4u * lane);
                    v[q] = lds_f64(vb + 256u * q + 8u * lane);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) zj[q] = lds_f64(zs + 8u * j[q]);
                double p[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) p[q] = v[q] * zj[q];
                t = ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
            }
        } else if (MODE == 5 || MODE == 6) {  // entry-major, runtime m in batches of 8 (engine fast path)
            double a0 = 0.0, a1 = 0.0;
            for (int q0 = 0; q0 < m; q0 += 8) {
                int j[8];
                double v[8], zj[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const bool ok = q0 + q < m;
                    j[q] = ok ? lds_s32(cb + 128u * (q0 + q) + 4u * lane) : n;
                    v[q] = ok ? lds_f64(vb + 256u * ((q0 + q) & 7) + 8u * lane) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) zj[q] = lds_f64(zs + 8u * j[q]);
                double pr[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pr[q] = v[q] * zj[q];
                a0 = a0 + ((pr[0] + pr[1]) + (pr[2] + pr[3]));
                a1 = a1 + ((pr[4] + pr[5]) + (pr[6] + pr[7]));
            }
            t = a0 + a1;
        } else {  // pure latency reference: one dependent LDS + DADD
            if (act) t = lds_f64(zs + 8u * lane);
        }
        // reduce over G lanes: butterfly (MODE 3) or shared scratch
        if (MODE == 3 || MODE == 4) {
            for (int o = G >> 1; o > 0; o >>= 1) t = t + __shfl_xor_sync(0xffffffffu, t, o);
        } else if (MODE == 5) {
            for (int o = G >> 1; o > 0; o >>= 1) t = t + __shfl_xor_sync(0xffffffffu, t, o);
        } else if (MODE == 6) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                if (o < G) t = t + __shfl_xor_sync(0xffffffffu, t, o);
        } else if (G > 1) {
            double* scr = reinterpret_cast<double*>(sm + 14336);
            scr[lane] = t;
            __syncwarp();
            if (head) {
                double s = 0.0;
                for (int q = 0; q < G; ++q) s = s + scr[lane + q];
                t = s;
            }
        }
        if (head) z[i] = z0 - t;
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[MODE] = (t1 - t0) / nblk;
}

int main() {
    long long* cyc;
    cudaMallocManaged(&cyc, 16 * 8);
    const int n = 4000;
    cudaFuncSetAttribute(blocks<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(blocks<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(blocks<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(blocks<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(blocks<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(blocks<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    cudaFuncSetAttribute(blocks<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    int cfg[][3] = {{4, 3, 6}, {4, 0, 48}, {4, 2, 12}, {4, 1, 24}, {32, 0, 8}, {1, 5, 2}};
    for (auto& c : cfg) {
        blocks<0><<<1, 256, 64 * 1024>>>(cyc, c[0], c[1], c[2], 2000, n);
        blocks<1><<<1, 256, 64 * 1024>>>(cyc, c[0], c[1], 8, 2000, n);
        blocks<2><<<1, 256, 64 * 1024>>>(cyc, c[0], c[1], c[2], 2000, n);
        blocks<3><<<1, 256, 64 * 1024>>>(cyc, c[0], c[1], 8, 2000, n);
        blocks<4><<<1, 256, 64 * 1024>>>(cyc, c[0], c[1], 8, 2000, n);
        blocks<5><<<1, 256, 64 * 1024>>>(cyc, c[0], c[1], c[2], 2000, n);
        blocks<6><<<1, 256, 64 * 1024>>>(cyc, c[0], c[1], c[2], 2000, n);
        cudaDeviceSynchronize();
        printf("nr=%d lg=%d m=%d: engine-shape %lld  fixed8 %lld  fixed8+shfl %lld  entry-major8+shfl %lld  em-runtime-m %lld / unrolled-bfly %lld  floor %lld (%s)\n",
               c[0], c[1], c[2], cyc[0], cyc[1], cyc[3], cyc[4], cyc[5], cyc[6], cyc[2], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
