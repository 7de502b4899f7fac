// timer_probe.cu — cost of %globaltimer vs clock64 reads, and of sys-scope fences (design input).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(uint64_t *out, int mode, int n) {
    uint64_t c0 = clock64();
    uint64_t acc = 0;
    for (int i = 0; i < n; ++i) {
        uint64_t t;
        if (mode == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        else if (mode == 1) t = clock64();
        else if (mode == 2) { asm volatile("fence.sc.sys;" ::: "memory"); t = i; }
        else if (mode == 3) { asm volatile("fence.acq_rel.sys;" ::: "memory"); t = i; }
        else { __threadfence(); t = i; }
        acc += t;
    }
    uint64_t c1 = clock64();
    if (threadIdx.x == 0) { out[0] = c1 - c0; out[1] = acc; }
}
int main() {
    uint64_t *d, h[2];
    cudaMalloc(&d, 16);
    const char *names[] = {"globaltimer", "clock64", "fence.sc.sys", "fence.acq_rel.sys", "threadfence"};
    for (int mode = 0; mode < 5; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            k<<<1, 32>>>(d, mode, 1000);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        }
        printf("%-20s %8.1f cycles per read\n", names[mode], h[0] / 1000.0);
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int i = 0; i < 1000; ++i) k<<<1, 32>>>(d, 1, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("back-to-back empty launches: %.2f us each\n", ms);
    return 0;
}
