// Dependent-chain latency probe (developer tool): cycles per access for the
// load flavours the sync-free solves can use on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const int* gidx, int* out, long long* cyc, int iters) {
    __shared__ int sidx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sidx[i] = (i + 1) & 1023;
    __syncthreads();
    if (threadIdx.x != 0) return;
    int j = 0;
    long long t0, t1;
    // (a) plain shared
    t0 = clock64();
    for (int i = 0; i < iters; ++i) j = sidx[j];
    t1 = clock64();
    cyc[0] = (t1 - t0) / iters;
    // (b) volatile generic -> shared
    const volatile int* vs = sidx;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) j = vs[j];
    t1 = clock64();
    cyc[1] = (t1 - t0) / iters;
    // (c) explicit ld.volatile.shared
    unsigned base = (unsigned)__cvta_generic_to_shared(sidx);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        int v;
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 4u * (unsigned)j));
        j = v;
    }
    t1 = clock64();
    cyc[2] = (t1 - t0) / iters;
    // (d) ld.relaxed.cta.shared
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        int v;
        asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 4u * (unsigned)j));
        j = v;
    }
    t1 = clock64();
    cyc[3] = (t1 - t0) / iters;
    // (e) global L1/L2 (__ldg) chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) j = __ldg(gidx + j);
    t1 = clock64();
    cyc[4] = (t1 - t0) / iters;
    // (f) volatile global chain
    const volatile int* vg = gidx;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) j = vg[j];
    t1 = clock64();
    cyc[5] = (t1 - t0) / iters;
    // (g) relaxed.cta global chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        int v;
        asm volatile("ld.relaxed.cta.global.u32 %0, [%1];" : "=r"(v) : "l"(gidx + j));
        j = v;
    }
    t1 = clock64();
    cyc[6] = (t1 - t0) / iters;
    // (h) DADD dependent chain
    double s = j;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) s = s + 1.0000001;
    t1 = clock64();
    cyc[7] = (t1 - t0) / iters;
    // (i) DDIV dependent chain
    double q = s;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) q = q / 1.0000001;
    t1 = clock64();
    cyc[8] = (t1 - t0) / iters;
    out[0] = j + (int)q;
}

int main() {
    int* g;
    int* out;
    long long* cyc;
    cudaMalloc(&g, 1024 * sizeof(int));
    cudaMalloc(&out, sizeof(int));
    cudaMalloc(&cyc, 16 * sizeof(long long));
    int h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = (i + 33) & 1023;
    cudaMemcpy(g, h, sizeof h, cudaMemcpyHostToDevice);
    chain<<<1, 128>>>(g, out, cyc, 1000);
    chain<<<1, 128>>>(g, out, cyc, 10000);
    long long c[16];
    cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
    const char* names[] = {"shared plain", "volatile generic->shared", "ld.volatile.shared",
                           "ld.relaxed.cta.shared", "__ldg global", "volatile global",
                           "ld.relaxed.cta.global", "DADD chain", "DDIV chain"};
    for (int i = 0; i < 9; ++i) printf("%-28s %lld cycles\n", names[i], c[i]);
    return 0;
}
