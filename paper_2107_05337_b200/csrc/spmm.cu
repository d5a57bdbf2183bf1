// Batched operator products Y = A X of a stencil-major IgA operator
// (spmv, sparse.hpp:114-124, applied to nrhs vectors at once): the SpMV /
// SpMM kernels of north_star (1), built for HBM bandwidth.
//
//   The operator is read from a tiled copy (tile_kernel: 32 rows x W^2
//   entries contiguous) so that every CTA streams one contiguous stretch.
//   nrhs = 1:        a CTA per tile, lane = row, warps split the stencil rows
//                    (clamped addresses, out-of-grid entries selected to zero).
//   nrhs = 16..64:   X and Y are [n][nrhs] (right-hand sides contiguous).  A
//                    CTA owns a block of R consecutive rows of one grid line,
//                    lane l the right-hand-side pair (2l, 2l+1), warp w the
//                    stencil rows dv = w, w + 8, ...: per stencil row it loads
//                    the R + W - 1 x values its rows touch once (16-byte
//                    loads, coalesced across the lanes) and reuses them for
//                    the R W products; each operator value is read once per
//                    block (a broadcast).  A is read once per launch.
// Reassociated sums (tree per stencil row): the fast mode's arithmetic.
#include <cuda_runtime.h>

#include "device_types.cuh"
#include "phi_kernels.cuh"

namespace phi {
namespace {

template <int N>
struct TreeS {
    static __device__ __forceinline__ double sum(const double* p) {
        return TreeS<N / 2>::sum(p) + TreeS<N - N / 2>::sum(p + N / 2);
    }
};
template <>
struct TreeS<1> {
    static __device__ __forceinline__ double sum(const double* p) { return p[0]; }
};

// Tiled copy of a stencil operator for the streaming kernels: tile t holds
// rows [32 t, 32 t + 32) as At[t][e][32] (e = stencil entry), so one tile is
// one contiguous W^2 x 256-byte stretch of HBM.
__global__ void tile_kernel(const DevStencil A, double* __restrict__ At) {
    const int n = A.ru * A.rv, ww = (A.hi - A.lo + 1) * (A.hi - A.lo + 1);
    const size_t total = (size_t)((n + 31) / 32) * ww * 32;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total; k += (size_t)gridDim.x * blockDim.x) {
        const size_t t = k / ((size_t)ww * 32), rem = k - t * ww * 32;
        const int e = (int)(rem / 32), l = (int)(rem % 32);
        const size_t i = t * 32 + l;
        At[k] = i < (size_t)n ? A.vals[(size_t)e * n + i] : 0.0;
    }
}

// SpMV: a CTA owns one tile (lane = row); warp w sums the stencil entries
// e = w, w + 8, w + 16, ... of it (an even share of the W^2 entries per warp:
// no warp waits for another at the reduction), every load issued at once;
// the 8 partial sums are reduced through shared memory.
template <int W>
__global__ void __launch_bounds__(256, W <= 7 ? 8 : 6) spmv_kernel(const DevStencil A, const double* __restrict__ At,
                                                   const double* __restrict__ x, double* __restrict__ y) {
    constexpr int E = W * W, PE = (E + 7) / 8;  // entries, entries per warp (at most)
    __shared__ double part[8][32];
    const int n = A.ru * A.rv;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i = min(blockIdx.x * 32 + lane, n - 1);
    const int iv = i / A.ru, iu = i - iv * A.ru;
    const double* at = At + (size_t)blockIdx.x * E * 32 + lane;
    // fused multiply-adds in two chains (entries outside the grid carry a
    // zero coefficient), so few registers hold products: more CTAs per SM
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < PE; ++k) {
        const int e = w + 8 * k;
        if (k + 1 < PE || e < E) {
            const int dv = e / W, du = e - dv * W;
            const int r = iv + A.lo + dv, c = iu + A.lo + du;
            const bool ok = r >= 0 && r < A.cv && c >= 0 && c < A.cu;
            const double v = __ldg(at + (size_t)e * 32);
            const double xv = __ldg(x + (size_t)min(max(r, 0), A.cv - 1) * A.cu + min(max(c, 0), A.cu - 1));
            if (k & 1)
                s1 = __fma_rn(ok ? v : 0.0, xv, s1);
            else
                s0 = __fma_rn(ok ? v : 0.0, xv, s0);
        }
    }
    part[w][lane] = s0 + s1;
    __syncthreads();
    if (w == 0 && blockIdx.x * 32 + lane < n) {
        double q[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) q[h] = part[h][lane];
        y[blockIdx.x * 32 + lane] = TreeS<8>::sum(q);
    }
}

// SpMM: a CTA owns 32 / (nrhs / 2) tiles of 32 rows (one per lane group of
// nrhs / 2 lanes: 4 at nrhs = 16, 1 at 64), warp w rows 4w .. 4w+3 of each,
// lane l of a group the right-hand-side pair (2l, 2l+1).  Per stencil
// row the warp loads the x values its rows touch once (16-byte loads,
// coalesced across the lanes) and reuses them for all products of its rows;
// each operator value is one broadcast load from the contiguous tile.
template <int W, int NRHS>
__global__ void __launch_bounds__(256, 2) spmm_kernel(const DevStencil A, const double* __restrict__ At,
                                                   const double* __restrict__ X, double* __restrict__ Y) {
    constexpr int kRW = 4;  // rows per warp
    constexpr int nrhs = NRHS, nl = NRHS / 2, groups = 32 / nl;  // lanes per group, groups per warp
    const int n = A.ru * A.rv;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int grp = lane / nl, lg = lane - grp * nl;
    const int tile = blockIdx.x * groups + grp;
    const int i0 = tile * 32 + w * kRW;  // first row of this lane's group
    if (i0 >= n) return;
    const double* at = At + (size_t)tile * W * W * 32 + w * kRW;
    double2 acc[kRW];
#pragma unroll
    for (int rr = 0; rr < kRW; ++rr) acc[rr] = make_double2(0.0, 0.0);
    const int iv0 = i0 / A.ru, iu0 = i0 - iv0 * A.ru;
    const bool one_line = iu0 + kRW - 1 < A.ru && i0 + kRW - 1 < n;  // the warp's rows share a grid line
    if (one_line) {
        constexpr int NX = kRW + W - 1;
#pragma unroll 1
        for (int dv = 0; dv < W; ++dv) {
            const int r = iv0 + A.lo + dv;
            if (r < 0 || r >= A.cv) continue;
            double2 xs[NX];
            bool okc[NX];
#pragma unroll
            for (int c = 0; c < NX; ++c) {
                const int col = iu0 + A.lo + c;
                okc[c] = col >= 0 && col < A.cu;
                xs[c] = __ldg(reinterpret_cast<const double2*>(X + ((size_t)r * A.cu + min(max(col, 0), A.cu - 1)) * nrhs +
                                                               2 * lg));
            }
#pragma unroll
            for (int rr = 0; rr < kRW; ++rr) {
                // fused multiply-adds into two chains per component (reassociated
                // mode only; entries outside the grid carry a zero coefficient)
                double2 c0 = make_double2(0.0, 0.0), c1 = make_double2(0.0, 0.0);
#pragma unroll
                for (int du = 0; du < W; ++du) {
                    const double a = okc[rr + du] ? __ldg(at + (size_t)(dv * W + du) * 32 + rr) : 0.0;
                    double2& c = (du & 1) ? c1 : c0;
                    c.x = __fma_rn(a, xs[rr + du].x, c.x);
                    c.y = __fma_rn(a, xs[rr + du].y, c.y);
                }
                acc[rr].x = acc[rr].x + (c0.x + c1.x);
                acc[rr].y = acc[rr].y + (c0.y + c1.y);
            }
        }
    } else {  // rows across a line end (or past n): row by row
#pragma unroll
        for (int rr = 0; rr < kRW; ++rr) {
            const int i = min(i0 + rr, n - 1);
            const int iv = i / A.ru, iu = i - iv * A.ru;
#pragma unroll 1
            for (int dv = 0; dv < W; ++dv) {
                const int r = iv + A.lo + dv;
                if (r < 0 || r >= A.cv) continue;
                double px[W], py[W];
#pragma unroll
                for (int du = 0; du < W; ++du) {
                    const int col = iu + A.lo + du;
                    const bool ok = col >= 0 && col < A.cu;
                    const double a = __ldg(at + (size_t)(dv * W + du) * 32 + rr);
                    const double2 xv = __ldg(reinterpret_cast<const double2*>(
                        X + ((size_t)r * A.cu + min(max(col, 0), A.cu - 1)) * nrhs + 2 * lg));
                    px[du] = ok ? a * xv.x : 0.0;
                    py[du] = ok ? a * xv.y : 0.0;
                }
                acc[rr].x = acc[rr].x + TreeS<W>::sum(px);
                acc[rr].y = acc[rr].y + TreeS<W>::sum(py);
            }
        }
    }
#pragma unroll
    for (int rr = 0; rr < kRW; ++rr)
        if (i0 + rr < n) *reinterpret_cast<double2*>(Y + (size_t)(i0 + rr) * nrhs + 2 * lg) = acc[rr];
}

template <int W>
void launch_w(const DevStencil& A, const double* At, const double* X, double* Y, int nrhs, cudaStream_t s) {
    const int n = A.ru * A.rv;
    if (nrhs == 1)
        spmv_kernel<W><<<(n + 31) / 32, 256, 0, s>>>(A, At, X, Y);
    else if (nrhs == 16)
        spmm_kernel<W, 16><<<((n + 31) / 32 + 3) / 4, 256, 0, s>>>(A, At, X, Y);
    else if (nrhs == 32)
        spmm_kernel<W, 32><<<((n + 31) / 32 + 1) / 2, 256, 0, s>>>(A, At, X, Y);
    else
        spmm_kernel<W, 64><<<(n + 31) / 32, 256, 0, s>>>(A, At, X, Y);
    PHI_CUDA(cudaGetLastError());
}

}  // namespace

void launch_tile(const DevStencil& A, double* At, cudaStream_t s) {
    tile_kernel<<<1024, 256, 0, s>>>(A, At);
    PHI_CUDA(cudaGetLastError());
}
size_t tile_doubles(const DevStencil& A) {
    const size_t ww = (size_t)(A.hi - A.lo + 1) * (A.hi - A.lo + 1);
    return (size_t)((A.ru * A.rv + 31) / 32) * ww * 32;
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
