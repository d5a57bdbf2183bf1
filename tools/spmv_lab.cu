// Developer lab for the SpMV / SpMM kernels (csrc/spmm_kernels.cuh): checks
// every variant against a plain reference kernel and times it two ways --
// "single" (L2 flushed by a 256 MB read, events around ONE launch: bench.py's
// method) and "rotating" (events around 20 launches over 4 copies of the
// operator, > L2 in total).  Also times a plain read of the same bytes (what a
// streaming kernel of this size can reach at all).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I paper_2107_05337_b200/csrc tools/spmv_lab.cu -o tools/spmv_lab
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <string>

#include "../paper_2107_05337_b200/csrc/device_types.cuh"
#include "../paper_2107_05337_b200/csrc/spmm_kernels.cuh"

using namespace phi;

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);    \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__global__ void ref_spmm(DevStencil A, const double* X, double* Y, int B) {
    const int n = A.ru * A.rv, W = A.hi - A.lo + 1;
    const size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (k >= (size_t)n * B) return;
    const int i = (int)(k / B), b = (int)(k % B);
    const int iv = i / A.ru, iu = i % A.ru;
    double s = 0.0;
    for (int dv = 0; dv < W; ++dv)
        for (int du = 0; du < W; ++du) {
            const int r = iv + A.lo + dv, c = iu + A.lo + du;
            if (r < 0 || r >= A.cv || c < 0 || c >= A.cu) continue;
            s += A.vals[(size_t)(dv * W + du) * n + i] * X[((size_t)r * A.cu + c) * B + b];
        }
    Y[k] = s;
}

__global__ void read_stream(const double2* __restrict__ p, size_t n4, double* sink) {
    double s = 0.0;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n4; k += (size_t)gridDim.x * blockDim.x) {
        const double2 v = __ldg(p + 2 * k), u = __ldg(p + 2 * k + 1);
        s += v.x + v.y + u.x + u.y;
    }
    if (s == 1.2345e300) *sink = s;
}
__global__ void fill_rand(double* p, size_t n, unsigned long long seed) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
        unsigned long long z = (k + 1) * 0x9E3779B97F4A7C15ULL + seed;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        p[k] = (double)(z >> 11) * (1.0 / 9007199254740992.0) + 0.25;
    }
}

static double* g_flush;
static double* g_sink;
static cudaEvent_t e0, e1;
static const int NCOPY = 4;

template <class F>
static void time_it(const char* name, int p, int B, double bytes, double flops, F launch /* (copy) */) {
    // single: flush + one launch
    float tot = 0.f;
    const int reps = 7;
    for (int r = -1; r < reps; ++r) {
        read_stream<<<148 * 8, 256>>>(reinterpret_cast<const double2*>(g_flush), (size_t)8 << 20, g_sink);
        CK(cudaEventRecord(e0));
        launch(0);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (r >= 0) tot += ms;
    }
    const double single_us = tot / reps * 1e3;
    // rotating: 20 launches over NCOPY copies
    for (int k = 0; k < NCOPY; ++k) launch(k);
    CK(cudaEventRecord(e0));
    const int L = 20;
    for (int k = 0; k < L; ++k) launch(k % NCOPY);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double rot_us = ms / L * 1e3;
    printf("%-28s p=%d B=%-2d  single %7.2f us %6.0f GB/s (%4.1f%%)  rotating %7.2f us %6.0f GB/s (%4.1f%%)  %5.2f TF\n",
           name, p, B, single_us, bytes / single_us * 1e-3, bytes / single_us * 1e-3 / 65.402, rot_us,
           bytes / rot_us * 1e-3, bytes / rot_us * 1e-3 / 65.402, flops / rot_us * 1e-6);
    fflush(stdout);
}

static double check(const double* Y, const double* Yref, size_t len) {
    std::vector<double> a(len), b(len);
    CK(cudaMemcpy(a.data(), Y, len * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), Yref, len * 8, cudaMemcpyDeviceToHost));
    double m = 0.0;
    for (size_t k = 0; k < len; ++k) m = std::max(m, std::fabs(a[k] - b[k]) / (std::fabs(b[k]) + 1e-300));
    return m;
}

template <int W, int TR, int NCW, int NSW, int CPS = 1, int MODE = 0>
static void run_spmv(int p, const DevStencil& A, double* const* At, const double* x, double* y, const double* yref,
                     double bytes, double flops, int grid) {
    using Cfg = spk::SpmvCfg<W, TR, NCW, NSW>;
    if (Cfg::smem * CPS > 227 * 1024) return;
    auto kern = spk::spmv_tma_kernel<W, TR, NCW, NSW, CPS, MODE>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::smem));
    CK(cudaMemset(y, 0, (size_t)A.ru * A.rv * 8));
    kern<<<grid, Cfg::threads, Cfg::smem>>>(A, At[0], x, y);
    CK(cudaDeviceSynchronize());
    const double err = check(y, yref, (size_t)A.ru * A.rv);
    char name[96];
    snprintf(name, sizeof name, "spmv_tma TR%d w%d s%d g%d m%d e%.0e", TR, NCW, NSW, grid, MODE, err);
    time_it(name, p, 1, bytes, flops, [&](int c) { kern<<<grid, Cfg::threads, Cfg::smem>>>(A, At[c], x, y); });
}

template <int W, int B, int NS>
static void run_spmm(int p, const DevStencil& A, double* const* At, const double* X, double* Y, const double* Yref,
                     double bytes, double flops, int grid) {
    using Cfg = spk::SpmmCfg<W, NS>;
    if (Cfg::smem > 227 * 1024) return;
    auto kern = spk::spmm_tma_kernel<W, B, NS>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::smem));
    CK(cudaMemset(Y, 0, (size_t)A.ru * A.rv * 8 * B));
    kern<<<grid, Cfg::threads, Cfg::smem>>>(A, At[0], X, Y);
    CK(cudaDeviceSynchronize());
    const double err = check(Y, Yref, (size_t)A.ru * A.rv * B);
    char name[96];
    snprintf(name, sizeof name, "spmm_tma s%d g%d e%.0e", NS, grid, err);
    time_it(name, p, B, bytes, flops, [&](int c) { kern<<<grid, Cfg::threads, Cfg::smem>>>(A, At[c], X, Y); });
}

template <int W>
static void run_p(int p, int k) {
    const int s = (1 << k) + p - 2, n = s * s, E = W * W;
    const double nnz = std::pow((double)s * W - p * (p + 1), 2);
    printf("---- p=%d side %d n %d nnz %.0f (%.1f MB)\n", p, s, n, nnz, nnz * 8e-6);
    double* vals;
    CK(cudaMalloc(&vals, (size_t)E * n * 8));
    fill_rand<<<1024, 256>>>(vals, (size_t)E * n, 1);  // out-of-grid entries carry junk: the tiling must zero them
    DevStencil A{s, s, s, s, -p, p, vals};
    const size_t npad = (size_t)((n + 63) / 64) * 64;
    double *At16[NCOPY], *At32[NCOPY], *At64[NCOPY], *At64p[NCOPY];
    for (int c = 0; c < NCOPY; ++c) {
        CK(cudaMalloc(&At16[c], npad * E * 8));
        CK(cudaMalloc(&At32[c], npad * E * 8));
        CK(cudaMalloc(&At64[c], npad * E * 8));
        CK(cudaMalloc(&At64p[c], (npad / 64) * (size_t)spk::SpmmCfg<W, 1>::tile_bytes));
        spk::tile_rows_kernel<<<1024, 256>>>(A, At16[c], 16, 0);
        spk::tile_rows_kernel<<<1024, 256>>>(A, At32[c], 32, 0);
        spk::tile_rows_kernel<<<1024, 256>>>(A, At64[c], 64, 0);
        spk::tile_rows_kernel<<<1024, 256>>>(A, At64p[c], 64, spk::kSpmmPad);
    }
    const int BM = 64;
    double *X, *Y, *Yref;
    CK(cudaMalloc(&X, (size_t)n * BM * 8));
    CK(cudaMalloc(&Y, (size_t)n * BM * 8));
    CK(cudaMalloc(&Yref, (size_t)n * BM * 8));
    fill_rand<<<1024, 256>>>(X, (size_t)n * BM, 7);
    CK(cudaDeviceSynchronize());
    for (int B : {1, 16, 64}) {
        const double bytes = 8 * nnz + 16.0 * B * n, flops = 2 * nnz * B;
        ref_spmm<<<(unsigned)(((size_t)n * B + 255) / 256), 256>>>(A, X, Yref, B);
        CK(cudaDeviceSynchronize());
        // attainable: a plain read of the same bytes
        {
            const size_t n4 = (size_t)(bytes / 32);
            time_it("read_stream (same bytes)", p, B, bytes, 0.0, [&](int c) {
                read_stream<<<148 * 8, 256>>>(reinterpret_cast<const double2*>(At64[c]), std::min(n4, npad * E / 4), g_sink);
            });
        }
        if (B == 1) {
            run_spmv<W, 16, 12, 1>(p, A, At16, X, Y, Yref, bytes, flops, 148);
            run_spmv<W, 16, 4, 1, 4>(p, A, At16, X, Y, Yref, bytes, flops, 592);
        } else if (B == 16) {
            run_spmm<W, 16, 2>(p, A, At64p, X, Y, Yref, bytes, flops, 148);
        } else {
            run_spmm<W, 64, 2>(p, A, At64p, X, Y, Yref, bytes, flops, 148);
        }
    }
    for (int c = 0; c < NCOPY; ++c) {
        cudaFree(At16[c]);
        cudaFree(At32[c]);
        cudaFree(At64[c]);
        cudaFree(At64p[c]);
    }
    cudaFree(X);
    cudaFree(Y);
    cudaFree(Yref);
    cudaFree(vals);
}

int main(int argc, char** argv) {
    const int k = argc > 1 ? atoi(argv[1]) : 8;
    CK(cudaMalloc(&g_flush, (size_t)256 << 20));
    CK(cudaMemset(g_flush, 0, (size_t)256 << 20));
    CK(cudaMalloc(&g_sink, 64));
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    run_p<5>(2, k);
    run_p<7>(3, k);
    run_p<9>(4, k);
    run_p<11>(5, k);
    return 0;
}
