// Developer probe: hand-off latency between two warps of a CTA (cycles per
// one-way hand-off): named barriers (bar.arrive / bar.sync) vs a shared flag
// polled with volatile loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hand_probe tools/hand_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(long long* out, int n, int mode) {
    __shared__ volatile int flag[2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) flag[0] = flag[1] = -1;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (mode == 0) {  // named barriers: w0 -> w1 on id 1, w1 -> w0 on id 2
            if (w == 0) {
                if (i > 0) asm volatile("bar.sync 2, 64;" ::: "memory");
                asm volatile("bar.arrive 1, 64;" ::: "memory");
            } else {
                asm volatile("bar.sync 1, 64;" ::: "memory");
                asm volatile("bar.arrive 2, 64;" ::: "memory");
            }
        } else {  // flags
            if (w == 0) {
                if (i > 0)
                    while (flag[1] < i - 1) {
                    }
                __syncwarp();
                if (lane == 0) flag[0] = i;
            } else {
                while (flag[0] < i) {
                }
                __syncwarp();
                if (lane == 0) flag[1] = i;
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[mode] = (t1 - t0) / (2 * n);
    if (mode == 0 && w == 0) asm volatile("bar.sync 2, 64;" ::: "memory");
}

int main() {
    long long* o;
    cudaMallocManaged(&o, 8 * 8);
    k<<<1, 64>>>(o, 1000, 0);
    k<<<1, 64>>>(o, 1000, 1);
    cudaDeviceSynchronize();
    printf("one-way hand-off: named barrier %lld cyc, polled flag %lld cyc (%s)\n", o[0], o[1],
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
