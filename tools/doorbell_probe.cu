// doorbell_probe.cu — can a coordination cycle avoid the kernel launch on its critical path?
// Host-side latency from "the host decides to run a cycle" to "the host sees the kernel's
// result in pinned memory", for:
//   A  launch -> kernel writes a pinned flag (today's gr_step path);
//   B  armed: cuStreamWaitValue32 on a pinned doorbell + the kernel enqueued AHEAD of time; the
//      cycle is one host store to the doorbell;
//   C  B + the kernel first reads a 16-word descriptor from pinned memory (the cycle's marks);
//   D  B with the doorbell in device memory written by cuStreamWriteValue32 on another stream;
//   E  a persistent kernel polling the pinned doorbell (reference for the raw PCIe round trip).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/doorbell_probe.cu -o build/doorbell_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <unistd.h>

__global__ void k_flag(volatile uint32_t *hflag, uint32_t v) {
    if (threadIdx.x == 0) *hflag = v;
}
__global__ void k_desc_flag(volatile uint32_t *hflag, const volatile uint32_t *hdesc, uint32_t v) {
    __shared__ uint32_t s[16];
    if (threadIdx.x < 16) s[threadIdx.x] = hdesc[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) *hflag = v + (s[3] & 0u);
}
__global__ void k_persist(volatile uint32_t *hflag, const volatile uint32_t *hbell, uint32_t first, int n) {
    for (uint32_t v = first; v < first + (uint32_t)n; ++v) {
        while (*hbell != v) {}
        *hflag = v;
    }
}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static void report(const char *name, std::vector<double> &v) {
    std::sort(v.begin(), v.end());
    printf("%-58s p50 %6.2f us  p90 %6.2f us\n", name, v[v.size() / 2], v[v.size() * 9 / 10]);
}

int main() {
    cudaSetDevice(0);
    cudaFree(nullptr);
    volatile uint32_t *hflag, *hbell, *hdesc;
    uint32_t *dflag, *dbell, *ddesc, *dbell_dev;
    cudaHostAlloc((void **)&hflag, 64, cudaHostAllocMapped);
    cudaHostAlloc((void **)&hbell, 64, cudaHostAllocMapped);
    cudaHostAlloc((void **)&hdesc, 64, cudaHostAllocMapped);
    cudaHostGetDevicePointer((void **)&dflag, (void *)hflag, 0);
    cudaHostGetDevicePointer((void **)&dbell, (void *)hbell, 0);
    cudaHostGetDevicePointer((void **)&ddesc, (void *)hdesc, 0);
    cudaMalloc((void **)&dbell_dev, 64);
    cudaMemset(dbell_dev, 0, 64);
    *hflag = 0;
    *hbell = 0;
    int lo, hi;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t s, s2;
    cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi);
    cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi);
    const int n = 3000, warm = 200;
    uint32_t v = 0;
    {   // A
        std::vector<double> t;
        for (int i = 0; i < n + warm; ++i) {
            ++v;
            const double t0 = now_us();
            k_flag<<<1, 32, 0, s>>>(hflag, v);
            while (*hflag != v) {}
            if (i >= warm) t.push_back(now_us() - t0);
        }
        report("A launch -> host sees", t);
    }
    for (int mode = 0; mode < 2; ++mode) {  // B, C
        std::vector<double> t, arm;
        ++v;
        double a0 = now_us();
        cuStreamWaitValue32((CUstream)s, (CUdeviceptr)dbell, v, CU_STREAM_WAIT_VALUE_GEQ);
        if (mode == 0) k_flag<<<1, 32, 0, s>>>(hflag, v);
        else k_desc_flag<<<1, 32, 0, s>>>(hflag, hdesc, v);
        for (int i = 0; i < n + warm; ++i) {
            usleep(20);  // the armed kernel is queued well before the cycle starts
            const double t0 = now_us();
            hdesc[3] = v;
            *hbell = v;   // the cycle: one host store
            while (*hflag != v) {}
            if (i >= warm) t.push_back(now_us() - t0);
            ++v;          // arm the next cycle
            a0 = now_us();
            cuStreamWaitValue32((CUstream)s, (CUdeviceptr)dbell, v, CU_STREAM_WAIT_VALUE_GEQ);
            if (mode == 0) k_flag<<<1, 32, 0, s>>>(hflag, v);
            else k_desc_flag<<<1, 32, 0, s>>>(hflag, hdesc, v);
            if (i >= warm) arm.push_back(now_us() - a0);
        }
        *hbell = v;
        cudaStreamSynchronize(s);
        report(mode == 0 ? "B armed (WaitValue on pinned doorbell) -> host sees" : "C armed + kernel reads 16-word pinned descriptor", t);
        report(mode == 0 ? "  (host cost of arming: WaitValue + launch)" : "  (host cost of arming)", arm);
    }
    {   // D: device-memory doorbell written by a stream memory op on another stream
        std::vector<double> t;
        ++v;
        cuStreamWaitValue32((CUstream)s, (CUdeviceptr)dbell_dev, v, CU_STREAM_WAIT_VALUE_GEQ);
        k_flag<<<1, 32, 0, s>>>(hflag, v);
        for (int i = 0; i < n + warm; ++i) {
            usleep(20);
            const double t0 = now_us();
            cuStreamWriteValue32((CUstream)s2, (CUdeviceptr)dbell_dev, v, 0);
            while (*hflag != v) {}
            if (i >= warm) t.push_back(now_us() - t0);
            ++v;
            cuStreamWaitValue32((CUstream)s, (CUdeviceptr)dbell_dev, v, CU_STREAM_WAIT_VALUE_GEQ);
            k_flag<<<1, 32, 0, s>>>(hflag, v);
        }
        cuStreamWriteValue32((CUstream)s2, (CUdeviceptr)dbell_dev, v, 0);
        cudaDeviceSynchronize();
        report("D armed on device doorbell, WriteValue32 from host stream", t);
    }
    {   // E: persistent poller
        std::vector<double> t;
        const uint32_t first = v + 1;
        k_persist<<<1, 32, 0, s>>>(hflag, hbell, first, n + warm);
        for (int i = 0; i < n + warm; ++i) {
            ++v;
            usleep(20);
            const double t0 = now_us();
            *hbell = v;
            while (*hflag != v) {}
            if (i >= warm) t.push_back(now_us() - t0);
        }
        cudaStreamSynchronize(s);
        report("E persistent kernel polling pinned doorbell", t);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
