// Inter-warp hand-off latency probe (developer tool): a token travels around a
// ring of warps through shared memory; each hop = "wait until my predecessor
// published, then publish".  Variants: volatile spin, spin + nanosleep, and
// mbarrier try_wait.  Reports cycles per hop.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void ring(long long* out, int laps) {
    __shared__ volatile long long slot[32];
    __shared__ unsigned long long bar[32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (threadIdx.x < 32) slot[threadIdx.x] = -1;
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar + w)));
    __syncthreads();
    long long t0 = clock64();
    for (int lap = 0; lap < laps; ++lap) {
        const long long tok = (long long)lap * nw + w;  // value this warp publishes
        if (!(lap == 0 && w == 0)) {
            const int pw = (w + nw - 1) % nw;
            const long long want = tok - 1;
            if (MODE == 2) {
                unsigned par = (unsigned)((w == 0 ? lap - 1 : lap) & 1);
                unsigned done;
                do {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(done) : "r"((unsigned)__cvta_generic_to_shared(bar + pw)), "r"(par) : "memory");
                } while (!done);
            } else if (MODE == 3) {
                // generic pointer + ld.relaxed.cta (as the engine's wait_val)
                const long long* gp = (const long long*)(slot + pw);
                long long v;
                do {
                    asm volatile("ld.relaxed.cta.u64 %0, [%1];" : "=l"(v) : "l"(gp));
                } while (v < want);
            } else {
                while (slot[pw] < want) {
                    if (MODE == 1) __nanosleep(20);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            if (MODE == 3) {
                long long* gp = (long long*)(slot + w);
                asm volatile("st.relaxed.cta.u64 [%0], %1;" ::"l"(gp), "l"(tok) : "memory");
            } else {
                slot[w] = tok;
            }
            if (MODE == 2) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar + w)) : "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[MODE] = (t1 - t0) / ((long long)laps * nw);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8 * sizeof(long long));
    for (int nw : {2, 4, 8, 16}) {
        ring<0><<<1, 32 * nw>>>(d, 2000);
        ring<1><<<1, 32 * nw>>>(d, 2000);
        ring<2><<<1, 32 * nw>>>(d, 2000);
        ring<3><<<1, 32 * nw>>>(d, 2000);
        long long h[8];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("warps=%2d  spin=%lld  spin+sleep=%lld  mbarrier=%lld generic-relaxed=%lld cycles/hop\n", nw, h[0], h[1], h[2], h[3]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
