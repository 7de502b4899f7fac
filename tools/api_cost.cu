// Host cost of the CUDA runtime calls on gr_step's path (B200 box): median ns per call.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/api_cost.cu -o tools/api_cost
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

struct Big { char b[792]; };
struct Small { char b[64]; };
__global__ void k_big(Big p) { if (p.b[0] == 123 && threadIdx.x == 999) printf("x"); }
__global__ void k_small(Small p) { if (p.b[0] == 123 && threadIdx.x == 999) printf("x"); }
__global__ void k_flag(volatile int *f, int v) { if (threadIdx.x == 0) *f = v; }

template <typename F>
double med_ns(F f, int n = 2000) {
    std::vector<double> v(n);
    for (int i = 0; i < n; ++i) {
        auto t0 = std::chrono::steady_clock::now();
        f();
        v[i] = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
    }
    std::sort(v.begin(), v.end());
    return v[n / 2];
}

int main() {
    cudaSetDevice(0);
    cudaFree(nullptr);
    cudaStream_t a, b;
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&b, cudaStreamNonBlocking, hi);
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    Big pb{};
    Small ps{};
    int dev;
    printf("cudaGetDevice        %8.0f ns\n", med_ns([&] { cudaGetDevice(&dev); }));
    printf("cudaSetDevice(same)  %8.0f ns\n", med_ns([&] { cudaSetDevice(0); }));
    printf("launch 64B params    %8.0f ns\n", med_ns([&] { k_small<<<1, 256, 0, a>>>(ps); }));
    cudaStreamSynchronize(a);
    printf("launch 792B params   %8.0f ns\n", med_ns([&] { k_big<<<1, 256, 0, a>>>(pb); }));
    cudaStreamSynchronize(a);
    printf("cudaEventRecord      %8.0f ns\n", med_ns([&] { cudaEventRecord(e, a); }));
    printf("cudaStreamWaitEvent  %8.0f ns\n", med_ns([&] { cudaStreamWaitEvent(b, e, 0); }));
    printf("cudaGetLastError     %8.0f ns\n", med_ns([&] { cudaGetLastError(); }));
    printf("cudaStreamQuery      %8.0f ns\n", med_ns([&] { cudaStreamQuery(a); }));
    // launch -> kernel visible on the host: a 1-thread kernel writing pinned memory
    volatile int *h;
    cudaHostAlloc((void **)&h, 64, cudaHostAllocMapped);
    int *d;
    cudaHostGetDevicePointer((void **)&d, (void *)h, 0);
    cudaStreamSynchronize(a);
    int v = 0;
    printf("launch->host sees    %8.0f ns\n", med_ns([&] {
        ++v;
        k_flag<<<1, 32, 0, a>>>(d, v);
        while (*h != v) {}
    }));
    printf("launch+rec+wait+launch->host sees %8.0f ns\n", med_ns([&] {
        ++v;
        k_flag<<<1, 32, 0, a>>>(d, v);
        cudaEventRecord(e, a);
        cudaStreamWaitEvent(b, e, 0);
        k_big<<<148, 512, 0, b>>>(pb);
        cudaEventRecord(e, b);
        while (*h != v) {}
    }));
    cudaStreamSynchronize(a);
    cudaStreamSynchronize(b);
    return 0;
}
