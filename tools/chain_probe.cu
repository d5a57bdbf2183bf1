// Developer probe: cycles per entry of an ordered fp64 subtraction chain
// s -= p[e] read from shared memory by one warp (lanes = rows), for several
// code shapes of the triangular-solve inner loop.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/chain_probe tools/chain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double lds(unsigned a) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ double vlds(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <int MODE>
__global__ void chain(double* out, long long* cyc, int span, int nr, int reps) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < span * 32; i += blockDim.x) sm[i] = 1e-3 * (i % 7);
    __syncthreads();
    const int lane = threadIdx.x;
    const unsigned pp = (unsigned)__cvta_generic_to_shared(sm) + 8u * lane, st = 8u * nr;
    double s = 1.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (lane < nr) {
            if (MODE == 0) {  // plain loop
                for (int e = 0; e < span; ++e) s = s - lds(pp + e * st);
            } else if (MODE == 1) {  // unrolled 8, loads grouped
                int e = 0;
                for (; e + 8 <= span; e += 8) {
                    double p[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) p[q] = lds(pp + (e + q) * st);
#pragma unroll
                    for (int q = 0; q < 8; ++q) s = s - p[q];
                }
                for (; e < span; ++e) s = s - lds(pp + e * st);
            } else if (MODE == 2) {  // volatile window
                double p[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) p[q] = vlds(pp + q * st);
                for (int e = 0; e < span; e += 8) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        s = s - p[q];
                        if (e + 8 + q < span) p[q] = vlds(pp + (e + 8 + q) * st);
                    }
                }
            } else if (MODE == 3) {  // pure register chain (latency floor)
                double a = 1e-3 * lane;
                for (int e = 0; e < span; ++e) s = s - a;
            } else if (MODE == 4) {  // two rows per lane interleaved (ILP 2)
                double s2 = 2.0;
                for (int e = 0; e < span; e += 1) {
                    s = s - lds(pp + e * st);
                    s2 = s2 - lds(pp + e * st + 4);
                }
                s = s + s2;
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[MODE] = (t1 - t0) / reps;
    out[lane] = s;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * 8);
    cudaMallocManaged(&cyc, 16 * 8);
    const int span = 48, nr = 4, reps = 200;
    chain<0><<<1, 32, 48 * 1024>>>(out, cyc, span, nr, reps);
    chain<1><<<1, 32, 48 * 1024>>>(out, cyc, span, nr, reps);
    chain<2><<<1, 32, 48 * 1024>>>(out, cyc, span, nr, reps);
    chain<3><<<1, 32, 48 * 1024>>>(out, cyc, span, nr, reps);
    chain<4><<<1, 32, 48 * 1024>>>(out, cyc, span, nr, reps);
    cudaDeviceSynchronize();
    const char* names[] = {"plain", "unroll8", "vwindow8", "regchain", "ilp2"};
    for (int m = 0; m < 5; ++m)
        printf("%-9s %5lld cycles per %d-entry row  (%.1f / entry)\n", names[m], cyc[m], span, (double)cyc[m] / span);
    return 0;
}
