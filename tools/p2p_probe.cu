// p2p_probe.cu — microbenchmark of NVLink peer access patterns on B200 (design input
// for the reduce kernels; not part of the product). One process, two GPUs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_probe tools/p2p_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U, int MODE>
__global__ void pull(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (MODE == 0) v[u] = __ldcg(src + i + u * stride);
            else if (MODE == 1) v[u] = src[i + u * stride];
            else {
                const uint4 *p = src + i + u * stride;
                asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
}

template <int U>
__global__ void push(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
}

// TMA bulk (non-tensor) pull: remote global -> smem (mbarrier), then smem -> local global
template <int CH>
__global__ void bulk_pull(const char *src, char *dst, size_t bytes) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < 2; ++s)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
        asm volatile("fence.proxy.async.shared::cta;");
    }
    __syncthreads();
    const size_t nchunks = bytes / CH;
    uint32_t phase[2] = {0, 0};
    int s = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        char *buf = sm + s * CH;
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        if (tid == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CH));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"((uint32_t)__cvta_generic_to_shared(buf)), "l"(src + c * CH), "r"(CH), "r"(b) : "memory");
        }
        // wait
        uint32_t done = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(b), "r"(phase[s]));
        }
        phase[s] ^= 1;
        if (tid == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(dst + c * CH), "r"((uint32_t)__cvta_generic_to_shared(buf)), "r"(CH) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 1;");
        }
        __syncthreads();
        s ^= 1;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;");
}

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    const size_t bytes = 512ull << 20, n = bytes / 16;
    uint4 *a0, *b0, *a1;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&a1, bytes));
    CK(cudaMemset(a1, 1, bytes));
    CK(cudaDeviceEnablePeerAccess(0, 0));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaMalloc(&a0, bytes));
    CK(cudaMalloc(&b0, bytes));
    CK(cudaMemset(a0, 2, bytes));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, auto launch) {
        for (int i = 0; i < 2; ++i) launch();
        cudaEventRecord(e0);
        const int it = 5;
        for (int i = 0; i < it; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t e = cudaGetLastError();
        printf("%-44s %8.1f GB/s  %s\n", name, bytes / (ms / it * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    char nm[128];
    for (int ctas : {32, 64, 148, 296, 592}) {
        for (int thr : {256, 512, 1024}) {
            snprintf(nm, sizeof nm, "pull cg U4 ctas=%d thr=%d", ctas, thr);
            run(nm, [&] { pull<4, 0><<<ctas, thr>>>(a1, b0, n); });
        }
    }
    for (int ctas : {148, 296}) {
        snprintf(nm, sizeof nm, "pull cg U1 ctas=%d thr=512", ctas);
        run(nm, [&] { pull<1, 0><<<ctas, 512>>>(a1, b0, n); });
        snprintf(nm, sizeof nm, "pull cg U2 ctas=%d thr=512", ctas);
        run(nm, [&] { pull<2, 0><<<ctas, 512>>>(a1, b0, n); });
        snprintf(nm, sizeof nm, "pull cg U8 ctas=%d thr=512", ctas);
        run(nm, [&] { pull<8, 0><<<ctas, 512>>>(a1, b0, n); });
        snprintf(nm, sizeof nm, "pull default U4 ctas=%d thr=512", ctas);
        run(nm, [&] { pull<4, 1><<<ctas, 512>>>(a1, b0, n); });
        snprintf(nm, sizeof nm, "pull relaxed.sys U4 ctas=%d thr=512", ctas);
        run(nm, [&] { pull<4, 2><<<ctas, 512>>>(a1, b0, n); });
    }
    for (int ctas : {32, 64, 148, 296}) {
        snprintf(nm, sizeof nm, "push U4 ctas=%d thr=512", ctas);
        run(nm, [&] { push<4><<<ctas, 512>>>(a0, a1, n); });
    }
    snprintf(nm, sizeof nm, "local copy U4 ctas=592 thr=512");
    run(nm, [&] { push<4><<<592, 512>>>(a0, b0, n); });
    cudaFuncSetAttribute(bulk_pull<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    cudaFuncSetAttribute(bulk_pull<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    for (int ctas : {32, 64, 148, 296}) {
        snprintf(nm, sizeof nm, "bulk pull 32K ctas=%d", ctas);
        run(nm, [&] { bulk_pull<32768><<<ctas, 32, 65536>>>((const char *)a1, (char *)b0, bytes); });
        snprintf(nm, sizeof nm, "bulk pull 64K ctas=%d", ctas);
        run(nm, [&] { bulk_pull<65536><<<ctas, 32, 131072>>>((const char *)a1, (char *)b0, bytes); });
    }
    // bidirectional: both GPUs pull from each other at once
    {
        uint4 *b1;
        CK(cudaSetDevice(1));
        CK(cudaMalloc(&b1, bytes));
        cudaStream_t s1;
        cudaStreamCreate(&s1);
        CK(cudaSetDevice(0));
        for (int i = 0; i < 2; ++i) {
            cudaEventRecord(e0);
            for (int k = 0; k < 5; ++k) {
                pull<4, 0><<<296, 512>>>(a1, b0, n);
                cudaSetDevice(1);
                pull<4, 0><<<296, 512, 0, s1>>>(a0, b1, n);
                cudaSetDevice(0);
            }
            cudaEventRecord(e1);
            cudaSetDevice(1);
            cudaStreamSynchronize(s1);
            cudaSetDevice(0);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("bidirectional pull (each dir)                 %8.1f GB/s\n", bytes / (ms / 5 * 1e-3) / 1e9);
        }
    }
    return 0;
}
