// handoff_probe.cu — floor of a device->host hand-off through pinned mapped memory (design input).
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <cuda_runtime.h>
__global__ void k(volatile uint64_t *flag, uint32_t *hostbuf, const uint32_t *hostin, uint64_t seq, int mode) {
    if (mode >= 2 && threadIdx.x < 32) hostbuf[threadIdx.x] = (uint32_t)seq;   // 32 posted writes
    uint32_t x = 0;
    if (mode >= 3) x = *(volatile const uint32_t *)(hostin + threadIdx.x % 4);   // a PCIe read
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode >= 1) asm volatile("fence.sc.sys;" ::: "memory");
        *flag = seq + (x & 0);
    }
}
int main() {
    uint64_t *h_flag, *d_flag;
    uint32_t *h_buf, *d_buf, *h_in, *d_in;
    cudaHostAlloc(&h_flag, 64, cudaHostAllocMapped);
    cudaHostAlloc(&h_buf, 4096, cudaHostAllocMapped);
    cudaHostAlloc(&h_in, 4096, cudaHostAllocMapped);
    cudaHostGetDevicePointer(&d_flag, h_flag, 0);
    cudaHostGetDevicePointer(&d_buf, h_buf, 0);
    cudaHostGetDevicePointer(&d_in, h_in, 0);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const char *names[] = {"flag only", "fence+flag", "32 writes+fence+flag", "+1 host read"};
    for (int mode = 0; mode < 4; ++mode) {
        uint64_t seq = 1000 * (mode + 1);
        double tot = 0;
        int n = 2000;
        for (int i = 0; i < n + 100; ++i) {
            ++seq;
            auto t0 = std::chrono::steady_clock::now();
            k<<<1, 512, 0, s>>>(d_flag, d_buf, d_in, seq, mode);
            while (*(volatile uint64_t *)h_flag != seq) {}
            auto t1 = std::chrono::steady_clock::now();
            if (i >= 100) tot += std::chrono::duration<double, std::micro>(t1 - t0).count();
        }
        printf("%-24s launch->host sees flag: %.2f us\n", names[mode], tot / n);
        cudaStreamSynchronize(s);
    }
    return 0;
}
