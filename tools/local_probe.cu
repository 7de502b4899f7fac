// local_probe.cu — in-place fp32 -> fp16 -> fp32 round trip over 900 MB (the N=1 path's
// arithmetic) with different streaming strategies (design input for local_kernel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/local_probe tools/local_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float4 rt(float4 v) {
    __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
    float2 fa = __half22float2(a), fb = __half22float2(b);
    return make_float4(fa.x, fa.y, fb.x, fb.y);
}

template <int U>
__global__ void ldg_kernel(float4 *g, size_t n4) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t st = (size_t)gridDim.x * blockDim.x;
    for (; i < n4; i += U * st) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * st < n4) v[u] = __ldcs(g + i + u * st);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * st < n4) __stcs(g + i + u * st, rt(v[u]));
    }
}

// contiguous per-CTA spans instead of grid stride
template <int U>
__global__ void span_kernel(float4 *g, size_t n4) {
    const size_t per = (n4 + gridDim.x - 1) / gridDim.x;
    const size_t b = blockIdx.x * per, e = b + per < n4 ? b + per : n4;
    for (size_t i = b + threadIdx.x; i < e; i += (size_t)U * blockDim.x) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * blockDim.x < e) v[u] = g[i + u * blockDim.x];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * blockDim.x < e) g[i + u * blockDim.x] = rt(v[u]);
    }
}

// warp-contiguous spans (the local_kernel's access pattern): warp w streams SPAN float4s
template <int U, int SPAN, bool CS>
__global__ void warpspan_kernel(float4 *g, size_t n4) {
    const int lane = threadIdx.x & 31;
    const size_t gw = (size_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const size_t nw = (size_t)gridDim.x * (blockDim.x / 32);
    for (size_t it = gw; it * SPAN < n4; it += nw) {
        const size_t b = it * SPAN, e = b + SPAN < n4 ? b + SPAN : n4;
        for (size_t i = b + lane; i < e; i += 32 * U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + 32 * u < e) v[u] = CS ? __ldcs(g + i + 32 * u) : g[i + 32 * u];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i + 32 * u < e) {
                    if (CS) __stcs(g + i + 32 * u, rt(v[u]));
                    else g[i + 32 * u] = rt(v[u]);
                }
        }
    }
}

// TMA ring: bulk G2S tiles, convert in smem, bulk S2G back
template <int TILE, int STAGES>
__global__ void __launch_bounds__(256, 1) tma_kernel(float *g, size_t n) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const int tid = threadIdx.x;
    const size_t ntiles = n * 4 / TILE;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint32_t ph[STAGES] = {};
    auto issue = [&](size_t t, int s) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TILE));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(sm + s * TILE)), "l"((char *)g + t * TILE), "r"(TILE), "r"(bar) : "memory");
    };
    size_t t = blockIdx.x;
    if (tid == 0)
        for (int s = 0; s < STAGES; ++s)
            if (t + (size_t)s * gridDim.x < ntiles) issue(t + (size_t)s * gridDim.x, s);
    int s = 0;
    for (; t < ntiles; t += gridDim.x) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&full[s]);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(bar), "r"(ph[s]));
        ph[s] ^= 1;
        float4 *tile = reinterpret_cast<float4 *>(sm + s * TILE);
        for (int i = tid; i < TILE / 16; i += blockDim.x) tile[i] = rt(tile[i]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char *)g + t * TILE),
                         "r"((uint32_t)__cvta_generic_to_shared(sm + s * TILE)), "r"(TILE) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem reusable
            const size_t nt = t + (size_t)STAGES * gridDim.x;
            if (nt < ntiles) issue(nt, s);
        }
        __syncthreads();
        s = (s + 1) % STAGES;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t n = 225115136ull;  // fcn220m elements (multiple of 4)
    float *g;
    cudaMalloc(&g, n * 4);
    cudaMemset(g, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char *name, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) fn();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("%-40s %7.1f us  %7.1f GB/s (8 B/elem) %s\n", name, ms * 100, n * 8 / (ms / 10 * 1e-3) / 1e9,
               err == cudaSuccess ? "" : cudaGetErrorString(err));
    };
    const size_t n4 = n / 4;
    char nm[64];
    for (int ctas : {296, 592, 1184}) {
        snprintf(nm, sizeof nm, "ldg U4 thr256 ctas%d", ctas);
        run(nm, [&] { ldg_kernel<4><<<ctas, 256>>>((float4 *)g, n4); });
        snprintf(nm, sizeof nm, "ldg U8 thr256 ctas%d", ctas);
        run(nm, [&] { ldg_kernel<8><<<ctas, 256>>>((float4 *)g, n4); });
    }
    run("warpspan U8 span2048 thr256 ctas444", [&] { warpspan_kernel<8, 2048, false><<<444, 256>>>((float4 *)g, n4); });
    run("warpspan U8 span2048 cs ctas444", [&] { warpspan_kernel<8, 2048, true><<<444, 256>>>((float4 *)g, n4); });
    run("warpspan U4 span2048 ctas444", [&] { warpspan_kernel<4, 2048, false><<<444, 256>>>((float4 *)g, n4); });
    run("warpspan U8 span8192 ctas444", [&] { warpspan_kernel<8, 8192, false><<<444, 256>>>((float4 *)g, n4); });
    run("warpspan U8 span8192 ctas296", [&] { warpspan_kernel<8, 8192, false><<<296, 256>>>((float4 *)g, n4); });
    run("warpspan U16 span8192 ctas296", [&] { warpspan_kernel<16, 8192, false><<<296, 256>>>((float4 *)g, n4); });
    run("warpspan U4 span512 ctas592", [&] { warpspan_kernel<4, 512, false><<<592, 256>>>((float4 *)g, n4); });
    run("ldg U4 thr256 ctas444", [&] { ldg_kernel<4><<<444, 256>>>((float4 *)g, n4); });
    run("ldg U4 thr512 ctas 592", [&] { ldg_kernel<4><<<592, 512>>>((float4 *)g, n4); });
    run("ldg U2 thr1024 ctas 296", [&] { ldg_kernel<2><<<296, 1024>>>((float4 *)g, n4); });
    run("span U4 thr512 ctas 296", [&] { span_kernel<4><<<296, 512>>>((float4 *)g, n4); });
    run("span U8 thr256 ctas 592", [&] { span_kernel<8><<<592, 256>>>((float4 *)g, n4); });
    cudaFuncSetAttribute(tma_kernel<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    cudaFuncSetAttribute(tma_kernel<65536, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
    cudaFuncSetAttribute(tma_kernel<16384, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
    run("tma 32K x6 ctas148", [&] { tma_kernel<32768, 6><<<148, 256, 6 * 32768>>>(g, n); });
    run("tma 64K x3 ctas148", [&] { tma_kernel<65536, 3><<<148, 256, 3 * 65536>>>(g, n); });
    run("tma 16K x12 ctas148", [&] { tma_kernel<16384, 12><<<148, 256, 12 * 16384>>>(g, n); });
    run("cudaMemcpy D2D same size (ref)", [&] { cudaMemcpyAsync(g, g + n / 2, n * 2, cudaMemcpyDeviceToDevice); });
    return 0;
}
