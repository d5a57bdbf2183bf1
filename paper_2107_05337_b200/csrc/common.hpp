// Shared host utilities for the engine: CUDA error handling, device buffers,
// the engine's error type.  No torch types anywhere in the engine.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

// Threads per Phi CTA (phi_kernels.cuh: kPhiThreads; setup_host.hpp: the
// number of block-sweep worker warps follows from it).
#ifndef PHI_THREADS
#define PHI_THREADS 256
#endif

namespace phi {

/// Error categories surfaced through the C-ABI status codes
/// (include/phi_engine.h: PHI_OK .. PHI_ERR_CUDA).
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NotConverged : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error in ") + what + " (" + file + ":" +
                        std::to_string(line) + "): " + cudaGetErrorString(e));
}
#define PHI_CUDA(x) ::phi::cuda_check((x), #x, __FILE__, __LINE__)

/// Owning device allocation (cudaMalloc); move-only.
template <typename T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(std::size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }

    void alloc(std::size_t n) {
        release();
        n_ = n;
        if (n) PHI_CUDA(cudaMalloc(reinterpret_cast<void**>(&p_), n * sizeof(T)));
    }
    void upload(const std::vector<T>& h, cudaStream_t s = nullptr) {
        if (h.size() != n_) alloc(h.size());
        if (n_)
            PHI_CUDA(cudaMemcpyAsync(p_, h.data(), n_ * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    std::vector<T> download(cudaStream_t s = nullptr) const {
        std::vector<T> h(n_);
        if (n_) {
            PHI_CUDA(cudaMemcpyAsync(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, s));
            PHI_CUDA(cudaStreamSynchronize(s));
        }
        return h;
    }
    void zero(cudaStream_t s = nullptr) {
        if (n_) PHI_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    T* get() const { return p_; }
    std::size_t size() const { return n_; }

private:
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

template <typename T>
DevBuf<T> to_device(const std::vector<T>& h, cudaStream_t s = nullptr) {
    DevBuf<T> d(h.size());
    d.upload(h, s);
    return d;
}

/// Host CSR with the reference's invariants (sparse.hpp:17-22): int32 row
/// offsets / sorted unique columns, fp64 values.
struct HostCsr {
    int n_rows = 0, n_cols = 0;
    std::vector<int> row_offsets{0};
    std::vector<int> col_indices;
    std::vector<double> values;
    int nnz() const { return static_cast<int>(col_indices.size()); }
};

/// NVTX range over a host-side phase (header-only NVTX v3: a no-op unless a
/// profiler is attached), so Nsight timelines show the MGRIT phases by name.
struct TraceRange {
    explicit TraceRange(const char* name) { nvtxRangePushA(name); }
    ~TraceRange() { nvtxRangePop(); }
    TraceRange(const TraceRange&) = delete;
    TraceRange& operator=(const TraceRange&) = delete;
};

}  // namespace phi
