// Batched operator products Y = A X of a stencil-major IgA operator
// (spmv, sparse.hpp:114-124, applied to nrhs vectors at once): the SpMV /
// SpMM kernels of north_star (1).  The kernels live in spmm_kernels.cuh
// (persistent grids, TMA-staged operator tiles); this file picks the
// configuration per stencil width and holds the two tiled copies' builders:
//   kind 0 (nrhs = 1):      tiles of 16 consecutive rows, At[t][e][16];
//   kind 1 (nrhs = 16..64): tiles of 64 consecutive rows, At[t][dv][du][64]
//                           with 16 bytes of padding per stencil row.
#include <cuda_runtime.h>

#include "device_types.cuh"
#include "phi_kernels.cuh"
#include "spmm_kernels.cuh"

namespace phi {
namespace {

constexpr int kSpmvRows = 16;  // rows per SpMV tile

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        PHI_CUDA(cudaGetDevice(&dev));
        PHI_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return sms;
}

// SpMV: 12 consumer warps per SM, one ring slot each (186 KB of tiles in
// flight per SM at p = 5); the narrow stencils (p <= 2) run four small CTAs
// per SM instead (the tiles are 3 KB: more, shorter queues).
template <int W>
void launch_spmv_w(const DevStencil& A, const double* At, const double* x, double* y, cudaStream_t s) {
    constexpr bool narrow = W <= 5;
    constexpr int NCW = narrow ? 4 : 12, CPS = narrow ? 4 : 1;
    using Cfg = spk::SpmvCfg<W, kSpmvRows, NCW, 1>;
    auto kern = spk::spmv_tma_kernel<W, kSpmvRows, NCW, 1, CPS, 0>;
    static bool ready = false;
    if (!ready) {
        PHI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::smem));
        ready = true;
    }
    kern<<<sm_count() * CPS, Cfg::threads, Cfg::smem, s>>>(A, At, x, y);
    PHI_CUDA(cudaGetLastError());
}

// SpMM: a ring of two 64-row tiles per SM (124 KB at p = 5).
template <int W, int NRHS>
void launch_spmm_wn(const DevStencil& A, const double* At, const double* X, double* Y, cudaStream_t s) {
    using Cfg = spk::SpmmCfg<W, 2>;
    auto kern = spk::spmm_tma_kernel<W, NRHS, 2>;
    static bool ready = false;
    if (!ready) {
        PHI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::smem));
        ready = true;
    }
    kern<<<sm_count(), Cfg::threads, Cfg::smem, s>>>(A, At, X, Y);
    PHI_CUDA(cudaGetLastError());
}

template <int W>
void launch_w(const DevStencil& A, const double* At, const double* X, double* Y, int nrhs, cudaStream_t s) {
    if (nrhs == 1)
        launch_spmv_w<W>(A, At, X, Y, s);
    else if (nrhs == 16)
        launch_spmm_wn<W, 16>(A, At, X, Y, s);
    else if (nrhs == 32)
        launch_spmm_wn<W, 32>(A, At, X, Y, s);
    else
        launch_spmm_wn<W, 64>(A, At, X, Y, s);
}

size_t spmm_tile_doubles(int W) { return (size_t)W * (W * spk::kSpmmRows + spk::kSpmmPad); }

}  // namespace

int tile_kind(int nrhs) { return nrhs == 1 ? 0 : 1; }

void launch_tile(const DevStencil& A, double* At, int kind, cudaStream_t s) {
    if (kind == 0)
        spk::tile_rows_kernel<<<1024, 256, 0, s>>>(A, At, kSpmvRows, 0);
    else
        spk::tile_rows_kernel<<<1024, 256, 0, s>>>(A, At, spk::kSpmmRows, spk::kSpmmPad);
    PHI_CUDA(cudaGetLastError());
}

size_t tile_doubles(const DevStencil& A, int kind) {
    const int W = A.hi - A.lo + 1;
    if (kind == 0) return (size_t)((A.ru * A.rv + kSpmvRows - 1) / kSpmvRows) * W * W * kSpmvRows;
    return (size_t)((A.ru * A.rv + spk::kSpmmRows - 1) / spk::kSpmmRows) * spmm_tile_doubles(W);
}

void launch_spmm(const DevStencil& A, const double* At, const double* X, double* Y, int nrhs, cudaStream_t s) {
    if (!(nrhs == 1 || nrhs == 16 || nrhs == 32 || nrhs == 64))
        throw InvalidArgument("spmm: nrhs must be 1, 16, 32 or 64");
    if (A.ru != A.cu || A.rv != A.cv) throw InvalidArgument("spmm: square stencil operators only");
    switch (A.hi - A.lo + 1) {
        case 3: launch_w<3>(A, At, X, Y, nrhs, s); break;
        case 5: launch_w<5>(A, At, X, Y, nrhs, s); break;
        case 7: launch_w<7>(A, At, X, Y, nrhs, s); break;
        case 9: launch_w<9>(A, At, X, Y, nrhs, s); break;
        case 11: launch_w<11>(A, At, X, Y, nrhs, s); break;
        default: throw InvalidArgument("spmm: stencil width not supported");
    }
}

}  // namespace phi
