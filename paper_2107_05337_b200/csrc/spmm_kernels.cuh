// SpMV / SpMM kernels of north_star (1): Y = A X for a stencil-major IgA
// operator (spmv, sparse.hpp:114-124, applied to nrhs vectors at once), built
// for HBM bandwidth on sm_100a.
//
//   The operator is streamed from a tiled copy (tile_rows_kernel): tile t holds
//   rows [TR t, TR t + TR) as At[t][e][TR] (e = stencil entry), one contiguous
//   E x TR x 8-byte stretch of HBM, entries outside the column grid stored as
//   exact zeros.  A persistent grid (one CTA per SM) pulls whole tiles into
//   shared memory with TMA bulk copies (cp.async.bulk + mbarrier complete_tx)
//   several tiles ahead of the arithmetic, so the HBM stream never waits for
//   a warp's registers or for a CTA to turn over.
//
//   Because the rows and the columns live on the same grid, row i's column at
//   stencil offset (dv, du) is the flat index i + (lo + dv) cu + (lo + du):
//   no index arithmetic per entry.  Positions that wrap around a grid line
//   carry a zero coefficient; only the first / last few tiles clamp the
//   index into [0, n).
//
//   spmv_tma_kernel   nrhs = 1.  Every consumer warp owns NSW ring slots and
//                     whole tiles: lane = row (TR = 32), two rows per lane
//                     (TR = 64) or row x stencil-row parity (TR = 16); it
//                     waits for its tile, sums E products per row from shared
//                     memory against x (L1-resident), stores y and refills
//                     its own slot -- no CTA-wide barrier anywhere.
//   spmm_tma_kernel   nrhs = 16 / 32 / 64, X and Y [n][nrhs].  A CTA tile is
//                     64 rows; warp w owns rows 8w .. 8w+7 and all right-hand
//                     sides (lane = a pair of them; with nrhs < 64 the lane
//                     groups split the stencil rows and are summed by
//                     shuffles).  Per stencil row the warp loads the 8 + W - 1
//                     x rows it touches once (16-byte loads) and reuses each
//                     for up to 8 rows; operator values are 16-byte broadcast
//                     loads from the staged tile: 176 DFMA per 62 loads at
//                     p = 5.  A producer warp keeps the ring full.
// Reassociated sums (fused multiply-adds, per-row chains): the fast mode's
// arithmetic; the exact mode's products go through stencil_apply.
#pragma once

#include <cuda_runtime.h>

#include "device_types.cuh"

namespace phi {
namespace spk {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(unsigned bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "W_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// one TMA bulk copy global -> shared, completion counted on `bar`
__device__ __forceinline__ void tile_fetch(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ double lds64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void lds128(unsigned a, double& x, double& y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

// Tiled copy of a square stencil operator: At[t][e][TR], zero outside the grid.
// `pad` doubles of padding follow every stencil row's W x TR slab (the SpMM
// tiles: lane groups reading different stencil rows then hit different banks).
__global__ void tile_rows_kernel(const DevStencil A, double* __restrict__ At, int TR, int pad) {
    const int n = A.ru * A.rv, W = A.hi - A.lo + 1;
    const size_t slab = (size_t)W * TR + pad, tile = slab * W;
    const size_t tiles = (size_t)(n + TR - 1) / TR, total = tiles * tile;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total; k += (size_t)gridDim.x * blockDim.x) {
        const size_t t = k / tile, rem = k - t * tile;
        const int dv = (int)(rem / slab), rs = (int)(rem - dv * slab);
        double v = 0.0;
        if (rs < W * TR) {
            const int du = rs / TR, l = rs - du * TR;
            const size_t i = t * TR + l;
            if (i < (size_t)n) {
                const int iv = (int)(i / A.ru), iu = (int)(i - (size_t)iv * A.ru);
                const int r = iv + A.lo + dv, c = iu + A.lo + du;
                if (r >= 0 && r < A.cv && c >= 0 && c < A.cu) v = A.vals[(size_t)(dv * W + du) * n + i];
            }
        }
        At[k] = v;
    }
}

// ---- SpMV -----------------------------------------------------------------
template <int W, int TR, int NCW, int NSW>
struct SpmvCfg {
    static constexpr int E = W * W;
    static constexpr int tile_bytes = E * TR * 8;
    static constexpr int threads = 32 * NCW;
    static constexpr size_t smem = (size_t)NCW * NSW * tile_bytes;
};

// MODE (developer lab): 0 the product; 1 no x loads; 2 wait / release only
template <int W, int TR, int NCW, int NSW, int CPS = 1, int MODE = 0>
__global__ void __launch_bounds__(32 * NCW, CPS)
    spmv_tma_kernel(const DevStencil A, const double* __restrict__ At, const double* __restrict__ x,
                    double* __restrict__ y) {
    using Cfg = SpmvCfg<W, TR, NCW, NSW>;
    constexpr int E = Cfg::E, TB = Cfg::tile_bytes;
    constexpr int ES = TR >= 32 ? 1 : 32 / TR;   // lane groups splitting the stencil rows
    constexpr int RPL = TR >= 32 ? TR / 32 : 1;  // rows per lane
    extern __shared__ __align__(128) unsigned char spmv_smem[];
    __shared__ unsigned long long bars[NCW * NSW];
    const int n = A.ru * A.rv, cu = A.cu, lo = A.lo;
    const int n_tiles = (n + TR - 1) / TR;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int r = lane % (TR >= 32 ? 32 : TR), h = lane / (TR >= 32 ? 32 : TR);
    const unsigned ring = smem_u32(spmv_smem) + (unsigned)(w * NSW) * TB;
    const unsigned bar = smem_u32(bars) + 8u * (w * NSW);
    // this warp's tiles: the CTA's k-th tile is blockIdx.x + k gridDim.x; warp w takes k = w, w + NCW, ...
    const int stride = gridDim.x * NCW;
    const int first = blockIdx.x + w * gridDim.x;
    if (lane == 0) {
        for (int j = 0; j < NSW; ++j) bar_init(bar + 8u * j, 1);
        bar_fence_init();
        for (int j = 0; j < NSW; ++j) {
            const int t = first + j * stride;
            if (t < n_tiles) tile_fetch(ring + j * TB, At + (size_t)t * E * TR, TB, bar + 8u * j);
        }
    }
    __syncwarp();
    const int off_min = lo * cu + lo, off_max = (lo + W - 1) * cu + lo + W - 1;
    int j = 0;
    unsigned ph = 0;
    for (int t = first; t < n_tiles; t += stride) {
        const int i0 = t * TR;
        bar_wait(bar + 8u * j, ph);
        const unsigned sm = ring + j * TB + 8u * r;
        const bool interior = i0 + off_min >= 0 && i0 + TR - 1 + off_max < n;
        double acc[RPL][2];
#pragma unroll
        for (int q = 0; q < RPL; ++q) acc[q][0] = acc[q][1] = 0.0;
        if (MODE == 2) {
            acc[0][0] = lds64(sm);
        } else if (interior) {
            const double* xr = x + i0 + r + lo * cu + lo;
#pragma unroll
            for (int dq = 0; dq < (W + ES - 1) / ES; ++dq) {
                const int dv = dq * ES + h;
                if (ES == 1 || dv < W) {
                    const double* xp = xr + dv * cu;
                    const unsigned ap = sm + (unsigned)(dv * W) * (TR * 8);
#pragma unroll
                    for (int du = 0; du < W; ++du) {
#pragma unroll
                        for (int q = 0; q < RPL; ++q) {
                            const double a = lds64(ap + (unsigned)du * (TR * 8) + 256u * q);
                            const double xv = MODE == 1 ? 1.0 : __ldg(xp + du + 32 * q);
                            acc[q][du & 1] = __fma_rn(a, xv, acc[q][du & 1]);
                        }
                    }
                }
            }
        } else {
#pragma unroll 1
            for (int dv = h; dv < W; dv += ES) {
                const int xb = i0 + r + (lo + dv) * cu + lo;
                const unsigned ap = sm + (unsigned)(dv * W) * (TR * 8);
#pragma unroll
                for (int du = 0; du < W; ++du) {
#pragma unroll
                    for (int q = 0; q < RPL; ++q) {
                        const double a = lds64(ap + (unsigned)du * (TR * 8) + 256u * q);
                        const int c = min(max(xb + du + 32 * q, 0), n - 1);
                        acc[q][du & 1] = __fma_rn(a, __ldg(x + c), acc[q][du & 1]);
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            double s = acc[q][0] + acc[q][1];
            if (ES >= 2) s += __shfl_xor_sync(0xffffffffu, s, 16);
            if (ES >= 4) s += __shfl_xor_sync(0xffffffffu, s, 8);
            const int i = i0 + r + 32 * q;
            if (h == 0 && i < n) y[i] = s;
        }
        // the slot is consumed (generic-proxy reads ordered before the async-proxy refill)
        __syncwarp();
        if (lane == 0) {
            const int tn = t + NSW * stride;
            if (tn < n_tiles) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tile_fetch(ring + j * TB, At + (size_t)tn * E * TR, TB, bar + 8u * j);
            }
        }
        if (++j == NSW) {
            j = 0;
            ph ^= 1u;
        }
    }
}

// ---- SpMM -----------------------------------------------------------------
constexpr int kSpmmRows = 64;  // rows per CTA tile (8 consumer warps x 8 rows)
constexpr int kSpmmR = 8;

constexpr int kSpmmPad = 2;  // doubles of padding per stencil-row slab (16 bytes: a 4-bank skew)
template <int W, int NS>
struct SpmmCfg {
    static constexpr int E = W * W;
    static constexpr int slab_bytes = (W * kSpmmRows + kSpmmPad) * 8;
    static constexpr int tile_bytes = W * slab_bytes;
    static constexpr int threads = 32 * 9;  // 8 consumer warps + the producer
    static constexpr size_t smem = (size_t)NS * tile_bytes;
};

template <int W, int NRHS, int NS>
__global__ void __launch_bounds__(288, 1)
    spmm_tma_kernel(const DevStencil A, const double* __restrict__ At, const double* __restrict__ X,
                    double* __restrict__ Y) {
    using Cfg = SpmmCfg<W, NS>;
    constexpr int TB = Cfg::tile_bytes, SB = Cfg::slab_bytes, R = kSpmmR, TR = kSpmmRows;
    constexpr int NL = NRHS / 2, G = 32 / NL;  // lanes per group, groups (splitting the stencil rows)
    constexpr int NX = R + W - 1;
    extern __shared__ __align__(128) unsigned char spmm_smem[];
    __shared__ unsigned long long full[NS], empty[NS];
    const int n = A.ru * A.rv, cu = A.cu, lo = A.lo;
    const int n_tiles = (n + TR - 1) / TR;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned ring = smem_u32(spmm_smem);
    const unsigned fb = smem_u32(full), eb = smem_u32(empty);
    if (threadIdx.x == 0) {
        for (int k = 0; k < NS; ++k) {
            bar_init(fb + 8u * k, 1);
            bar_init(eb + 8u * k, 8);
        }
        bar_fence_init();
    }
    __syncthreads();
    if (w == 8) {  // producer: one lane keeps the ring full
        if (lane == 0) {
            int slot = 0;
            unsigned ph = 0;
            int k = 0;
            for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
                if (k >= NS) bar_wait(eb + 8u * slot, ph ^ 1u);  // the consumers released round k / NS - 1
                tile_fetch(ring + slot * TB, reinterpret_cast<const unsigned char*>(At) + (size_t)t * TB, TB, fb + 8u * slot);
                if (++slot == NS) {
                    slot = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    const int g = lane / NL, lg = lane - g * NL;
    const int off_min = lo * cu + lo, off_max = (lo + W - 1) * cu + lo + W - 1;
    int slot = 0;
    unsigned ph = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int i0 = t * TR + w * R, nrow = min(R, n - i0);
        const bool interior = t * TR + off_min >= 0 && t * TR + TR - 1 + off_max < n;
        bar_wait(fb + 8u * slot, ph);
        const unsigned sm = ring + slot * TB + 8u * (w * R);
        double2 acc[R];
#pragma unroll
        for (int rr = 0; rr < R; ++rr) acc[rr] = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int dv = g; dv < W; dv += G) {
            const int xb = i0 + (lo + dv) * cu + lo;
            double2 xw[NX];
            if (interior) {
                const double2* xp = reinterpret_cast<const double2*>(X + (size_t)xb * NRHS + 2 * lg);
#pragma unroll
                for (int c = 0; c < NX; ++c) xw[c] = __ldg(xp + (size_t)c * NL);
            } else {
#pragma unroll
                for (int c = 0; c < NX; ++c) {
                    const int row = min(max(xb + c, 0), n - 1);
                    xw[c] = __ldg(reinterpret_cast<const double2*>(X + (size_t)row * NRHS + 2 * lg));
                }
            }
            const unsigned ap = sm + (unsigned)dv * SB;
#pragma unroll
            for (int du = 0; du < W; ++du) {
                double a[R];
#pragma unroll
                for (int q = 0; q < R / 2; ++q) lds128(ap + (unsigned)du * (TR * 8) + 16u * q, a[2 * q], a[2 * q + 1]);
#pragma unroll
                for (int rr = 0; rr < R; ++rr) {
                    acc[rr].x = __fma_rn(a[rr], xw[rr + du].x, acc[rr].x);
                    acc[rr].y = __fma_rn(a[rr], xw[rr + du].y, acc[rr].y);
                }
            }
        }
        // the tile is consumed
        __syncwarp();
        if (lane == 0) bar_arrive(eb + 8u * slot);
        if (G > 1) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
#pragma unroll
                for (int o = NL; o < 32; o <<= 1) {
                    acc[rr].x += __shfl_xor_sync(0xffffffffu, acc[rr].x, o);
                    acc[rr].y += __shfl_xor_sync(0xffffffffu, acc[rr].y, o);
                }
            }
        }
        if (g == 0) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
                if (rr < nrow) *reinterpret_cast<double2*>(Y + (size_t)(i0 + rr) * NRHS + 2 * lg) = acc[rr];
        }
        if (++slot == NS) {
            slot = 0;
            ph ^= 1u;
        }
    }
}

}  // namespace spk
}  // namespace phi
