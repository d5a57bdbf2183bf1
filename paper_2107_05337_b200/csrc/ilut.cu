// Device ILUT factorisation of the p-level operator A = M + c K (the
// smoother of PMultigridHierarchy, pmultigrid.hpp:217-224), reproducing the
// reference's dual-threshold ILUT (ilut.hpp:29-143) bit for bit.
//
// The elimination is row-sequential only through the U rows it reads: row i
// eliminates its pending lower columns k in increasing order, and step k
// needs the finished U row k.  Rows are therefore handed out to warps in
// increasing order (a global ticket), every warp keeps its row's work vector
// as a dense window over the band [i - bw, i + bw] in shared memory, and a
// warp waits for row k (an acquire flag) only when it reaches column k.  Far
// columns are eliminated long before the wavefront arrives; the critical
// path per row is the last elimination plus the selection of the U part.
//
// Arithmetic, per the reference:
//   * drop = tau * sqrt(sum of a_ij^2 in CSR order), summed by one lane;
//   * beta = w_k / u_kk (IEEE division); |beta| < drop: w_k = 0, no update;
//     else w_k = beta and w_j = w_j - RN(beta * u_kj) over U row k, k
//     ascending -- every w_j sees exactly the reference's sequence of
//     roundings (no fused multiply-add: -fmad=false);
//   * an entry survives if it is active, non-zero and |v| >= drop; per part
//     (L: j < i, U: j > i) only the `fill` largest are kept under the strict
//     order (|v| descending, column ascending) -- the set nth_element picks
//     (keep_largest, ilut.hpp:112-124) -- then written in column order;
//   * the diagonal must be active and non-zero (zero-pivot error otherwise).
// The selection is a radix select on the IEEE bits of |v| (monotone for
// non-negative doubles) with ties broken by column, which is the same total
// order.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <string>
#include <vector>

#include "common.hpp"
#include "device_types.cuh"
#include "phi_kernels.cuh"

namespace phi {

namespace {

constexpr int kIlutWarps = 4;  // warps (rows in flight) per CTA

struct IlutArgs {
    DevStencil A;
    int n, nf, bw, fill;
    double tau;
    int* lc;
    double* lv;
    int* llen;  // row stride fill
    int* uc;
    double* uv;
    int* ulen;  // row stride fill + 1, entry 0 = the diagonal
    unsigned* done;
    int* prefix;  // every row below is done
    int* ticket;
    int* err_row;  // first zero-pivot row (INT_MAX: none)
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire_s32(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// First active window position in [from, limit), or limit.
__device__ __forceinline__ int next_active(const unsigned* bits, int from, int limit) {
    const int lane = threadIdx.x & 31;
    int wi = from >> 5;
    const int wlast = (limit - 1) >> 5;
    while (from < limit && wi <= wlast) {
        const int w = wi + lane;
        unsigned m = w <= wlast ? bits[w] : 0u;
        if (w == (from >> 5)) m &= ~0u << (from & 31);
        const unsigned any = __ballot_sync(0xffffffffu, m != 0u);
        if (any) {
            const int src = __ffs(any) - 1;
            const unsigned mw = __shfl_sync(0xffffffffu, m, src);
            const int pos = ((wi + src) << 5) + __ffs(mw) - 1;
            return pos < limit ? pos : limit;
        }
        wi += 32;
    }
    return limit;
}

__device__ __forceinline__ bool is_active(const unsigned* bits, int p) { return (bits[p >> 5] >> (p & 31)) & 1u; }

// Entries of positions [lo, hi) that survive the drop test, the `fill`
// largest of them (|v| descending, position ascending) written in position
// order to (oc, ov) with column base + position.  Returns the count written.
__device__ int select_part(const double* w, const unsigned* bits, int* hist, int lo, int hi, int base, double drop,
                           int fill, int* oc, double* ov) {
    const int lane = threadIdx.x & 31;
    auto cand = [&](int p, unsigned long long& key) {
        if (p >= hi || !is_active(bits, p)) return false;
        const double v = w[p];
        if (v == 0.0 || !(fabs(v) >= drop)) return false;
        key = (unsigned long long)__double_as_longlong(fabs(v));
        return true;
    };
    int c = 0;
    for (int p0 = lo; p0 < hi; p0 += 32) {
        unsigned long long key;
        c += __popc(__ballot_sync(0xffffffffu, cand(p0 + lane, key)));
    }
    // threshold: keep key > kstar, and the first `ties` entries equal to kstar
    unsigned long long kstar = 0ull;
    int ties = INT_MAX;
    if (c > fill) {
        unsigned long long prefix = 0ull, mask = 0ull;
        int need = fill;  // how many of the keys matching the prefix still to keep
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int b = lane; b < 256; b += 32) hist[b] = 0;
            __syncwarp();
            for (int p0 = lo; p0 < hi; p0 += 32) {
                unsigned long long key;
                if (cand(p0 + lane, key) && (key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
            }
            __syncwarp();
            // lane l sums digits 255 - 8 l .. 248 - 8 l (descending digit order)
            int cnt[8], s = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                cnt[q] = hist[255 - 8 * lane - q];
                s += cnt[q];
            }
            int incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int excl = incl - s;  // keys with a larger digit than this lane's range
            const bool here = excl < need && need <= incl;
            int digit = 0, above = 0;
            if (here) {
                int run = excl;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (run < need && need <= run + cnt[q]) {
                        digit = 255 - 8 * lane - q;
                        above = run;
                        break;
                    }
                    run += cnt[q];
                }
            }
            const unsigned who = __ballot_sync(0xffffffffu, here);
            const int src = __ffs(who) - 1;
            digit = __shfl_sync(0xffffffffu, digit, src);
            above = __shfl_sync(0xffffffffu, above, src);
            need -= above;
            prefix |= (unsigned long long)digit << shift;
            mask |= 255ull << shift;
            __syncwarp();
        }
        kstar = prefix;
        ties = need;  // entries equal to kstar to keep, in position order
    }
    // write the kept entries in position (= column) order
    int out = 0, tie_seen = 0;
    for (int p0 = lo; p0 < hi; p0 += 32) {
        unsigned long long key = 0ull;
        const bool ok = cand(p0 + lane, key);
        bool keep = ok;
        if (c > fill) {
            const bool eq = ok && key == kstar;
            const unsigned teq = __ballot_sync(0xffffffffu, eq);
            const int rank = tie_seen + __popc(teq & ((1u << lane) - 1u));
            keep = ok && (key > kstar || (eq && rank < ties));
            tie_seen += __popc(teq);
        }
        const unsigned km = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            const int r = out + __popc(km & ((1u << lane) - 1u));
            oc[r] = base + p0 + lane;
            ov[r] = w[p0 + lane];
        }
        out += __popc(km);
    }
    return out;
}

__global__ void __launch_bounds__(32 * kIlutWarps) ilut_rows_kernel(const __grid_constant__ IlutArgs a) {
    extern __shared__ __align__(16) unsigned char ilut_smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int W = 2 * a.bw + 1;
    const int nwords = (W + 31) / 32;
    const size_t per_warp = ((size_t)W * 8 + 15) / 16 * 16 + ((size_t)nwords * 4 + 15) / 16 * 16 + 256 * 4;
    unsigned char* mine = ilut_smem + per_warp * wid;
    double* w = reinterpret_cast<double*>(mine);
    unsigned* bits = reinterpret_cast<unsigned*>(mine + ((size_t)W * 8 + 15) / 16 * 16);
    int* hist = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(bits) + ((size_t)nwords * 4 + 15) / 16 * 16);
    for (int p = lane; p < W; p += 32) w[p] = 0.0;
    for (int q = lane; q < nwords; q += 32) bits[q] = 0u;
    __syncwarp();
    const int wa = a.A.hi - a.A.lo + 1, nent = wa * wa;
    const int us = a.fill + 1;
    int known = 0;  // rows below are done (a stale copy of a.prefix)
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(a.ticket, 1);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= a.n) break;
        const int base = i - a.bw;
        const int iv = i / a.nf, iu = i - iv * a.nf;
        // ---- row i of A into the window (entries in CSR order: (dv, du) ascending)
        for (int e = lane; e < nent; e += 32) {
            const int dv = e / wa + a.A.lo, du = e % wa + a.A.lo;
            if (iv + dv < 0 || iv + dv >= a.A.cv || iu + du < 0 || iu + du >= a.A.cu) continue;
            const int p = (iu + du) + a.nf * (iv + dv) - base;
            w[p] = a.A.vals[(size_t)e * a.n + i];
            atomicOr(&bits[p >> 5], 1u << (p & 31));
        }
        double drop = 0.0;
        if (lane == 0) {
            double s = 0.0;
            for (int e = 0; e < nent; ++e) {
                const int dv = e / wa + a.A.lo, du = e % wa + a.A.lo;
                if (iv + dv < 0 || iv + dv >= a.A.cv || iu + du < 0 || iu + du >= a.A.cu) continue;
                const double v = a.A.vals[(size_t)e * a.n + i];
                s += v * v;
            }
            drop = a.tau * sqrt(s);
        }
        drop = __shfl_sync(0xffffffffu, drop, 0);
        __syncwarp();
        // ---- eliminate the pending lower columns in increasing order
        for (int p = next_active(bits, 0, a.bw); p < a.bw; p = next_active(bits, p + 1, a.bw)) {
            const int k = base + p;
            if (lane == 0 && k >= known) {
                known = ld_acquire_s32(a.prefix);
                if (k >= known)
                    while (!ld_acquire(a.done + k)) {
                    }
            }
            __syncwarp();
            const double dk = __ldcg(a.uv + (size_t)k * us);
            const double beta = w[p] / dk;
            __syncwarp();
            if (fabs(beta) < drop) {
                if (lane == 0) w[p] = 0.0;
            } else {
                if (lane == 0) w[p] = beta;
                const int len = __ldcg(a.ulen + k);
                for (int e = 1 + lane; e < len; e += 32) {
                    const int j = __ldcg(a.uc + (size_t)k * us + e);
                    const double u = __ldcg(a.uv + (size_t)k * us + e);
                    const int q = j - base;
                    atomicOr(&bits[q >> 5], 1u << (q & 31));
                    w[q] = w[q] - beta * u;
                }
            }
            __syncwarp();
        }
        // ---- U row: the diagonal, then the largest of the strict upper part
        double diag = w[a.bw];
        if (!is_active(bits, a.bw) || diag == 0.0) {
            if (lane == 0) atomicMin(a.err_row, i);
            diag = 1.0;  // keep the later rows going; the host reports the error
        }
        int* uc = a.uc + (size_t)i * us;
        double* uv = a.uv + (size_t)i * us;
        const int nu = select_part(w, bits, hist, a.bw + 1, W, base, drop, a.fill, uc + 1, uv + 1);
        if (lane == 0) {
            uc[0] = i;
            uv[0] = diag;
            a.ulen[i] = nu + 1;
        }
        __syncwarp();
        __threadfence();
        if (lane == 0) {
            st_release(a.done + i, 1u);
            // advance the done prefix while the next rows are finished
            int q = ld_acquire_s32(a.prefix);
            while (q < a.n && ld_acquire(a.done + q)) {
                __threadfence();
                atomicMax(a.prefix, q + 1);
                ++q;
            }
            known = q;
        }
        // ---- L row (needed by no other row)
        const int nl = select_part(w, bits, hist, 0, a.bw, base, drop, a.fill, a.lc + (size_t)i * a.fill,
                                   a.lv + (size_t)i * a.fill);
        if (lane == 0) a.llen[i] = nl;
        // ---- reset the touched window entries
        __syncwarp();
        for (int q = lane; q < nwords; q += 32) {
            unsigned m = bits[q];
            while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                w[(q << 5) + b] = 0.0;
            }
            bits[q] = 0u;
        }
        __syncwarp();
    }
}

}  // namespace

void device_ilut(const DevStencil& A, double tau, int fill_limit, HostCsr& lower, HostCsr& upper,
                 cudaStream_t s) {
    if (A.ru != A.cu || A.rv != A.cv) throw InvalidArgument("ilut_factor: matrix not square");
    const int n = A.ru * A.rv, nf = A.ru;
    const int wa = A.hi - A.lo + 1;
    // nnz of the clamped-rectangle pattern (the reference CSR's nnz)
    long long nnz = 0;
    for (int iv = 0; iv < A.rv; ++iv) {
        const long long dv = std::min(A.hi, A.cv - 1 - iv) - std::max(A.lo, -iv) + 1;
        for (int iu = 0; iu < A.ru; ++iu) nnz += dv * (std::min(A.hi, A.cu - 1 - iu) - std::max(A.lo, -iu) + 1);
    }
    (void)wa;
    if (fill_limit <= 0) fill_limit = (int)((nnz + n - 1) / std::max(n, 1));
    IlutArgs a{};
    a.A = A;
    a.n = n;
    a.nf = nf;
    a.bw = std::max(A.hi, -A.lo) * (nf + 1);
    a.fill = fill_limit;
    a.tau = tau;
    const int us = fill_limit + 1;
    DevBuf<int> lc((size_t)n * fill_limit), llen(n), uc((size_t)n * us), ulen(n), ctl(3);
    DevBuf<double> lv((size_t)n * fill_limit), uv((size_t)n * us);
    DevBuf<unsigned> done(n);
    done.zero(s);
    const std::vector<int> ctl0{0, 0, INT_MAX};  // prefix, ticket, err_row
    ctl.upload(ctl0, s);
    a.lc = lc.get();
    a.lv = lv.get();
    a.llen = llen.get();
    a.uc = uc.get();
    a.uv = uv.get();
    a.ulen = ulen.get();
    a.done = done.get();
    a.prefix = ctl.get();
    a.ticket = ctl.get() + 1;
    a.err_row = ctl.get() + 2;
    const int W = 2 * a.bw + 1, nwords = (W + 31) / 32;
    const size_t per_warp = ((size_t)W * 8 + 15) / 16 * 16 + ((size_t)nwords * 4 + 15) / 16 * 16 + 256 * 4;
    int warps = kIlutWarps;
    size_t smem = per_warp * warps;
    if (smem > 200 * 1024) throw InvalidArgument("ilut_factor: band too wide for the device window");
    PHI_CUDA(cudaFuncSetAttribute(ilut_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, n_sm = 0, per_sm = 0;
    PHI_CUDA(cudaGetDevice(&dev));
    PHI_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    PHI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ilut_rows_kernel, 32 * warps, smem));
    // every CTA must be resident at once: a warp may wait for a row another warp holds
    const int grid = std::max(1, std::min((n + warps - 1) / warps, std::max(per_sm, 1) * n_sm));
    ilut_rows_kernel<<<grid, 32 * warps, smem, s>>>(a);
    PHI_CUDA(cudaGetLastError());
    const std::vector<int> c = ctl.download(s);
    if (c[2] != INT_MAX) throw std::runtime_error("ilut_factor: zero pivot in row " + std::to_string(c[2]));
    // compact the fixed-stride rows into CSR (sparse.hpp:17-22)
    const std::vector<int> hl = llen.download(s), hu = ulen.download(s);
    const std::vector<int> hlc = lc.download(s), huc = uc.download(s);
    const std::vector<double> hlv = lv.download(s), huv = uv.download(s);
    auto compact = [n](const std::vector<int>& len, const std::vector<int>& cc, const std::vector<double>& vv,
                       int stride, HostCsr& out) {
        out = HostCsr{};
        out.n_rows = out.n_cols = n;
        out.row_offsets.resize((size_t)n + 1);
        out.row_offsets[0] = 0;
        for (int i = 0; i < n; ++i) out.row_offsets[i + 1] = out.row_offsets[i] + len[i];
        out.col_indices.resize(out.row_offsets[n]);
        out.values.resize(out.row_offsets[n]);
        for (int i = 0; i < n; ++i) {
            std::copy_n(cc.begin() + (size_t)i * stride, len[i], out.col_indices.begin() + out.row_offsets[i]);
            std::copy_n(vv.begin() + (size_t)i * stride, len[i], out.values.begin() + out.row_offsets[i]);
        }
    };
    compact(hl, hlc, hlv, fill_limit, lower);
    compact(hu, huc, huv, us, upper);
}

}  // namespace phi
