// nvls_probe.cu — does NVLS multicast work on this box? (design input for NEXT-1)
// One process, 2 GPUs: create a multicast object, bind one allocation per GPU, multimem.st
// through the multicast VA from GPU0, multimem.ld_reduce from GPU1, and try exporting the
// handles as FABRIC / POSIX_FD (what a one-process-per-GPU library needs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)
#define CUW(x) do { CUresult r = (x); const char *s = ""; if (r != CUDA_SUCCESS) cuGetErrorString(r, &s); printf("%-60s -> %d %s\n", #x, (int)r, s); } while (0)

__global__ void st_kernel(float *mc, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * i + 3 < n) {
        float a = 1.0f + i, b = 2.0f, c = 3.0f, d = 4.0f;
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + 4 * i), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
    }
}
__global__ void red_kernel(const float *mc, float *out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * i + 3 < n) {
        float a, b, c, d;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + 4 * i) : "memory");
        out[4 * i] = a; out[4 * i + 1] = b; out[4 * i + 2] = c; out[4 * i + 3] = d;
    }
}

int main(int argc, char **argv) {
    const bool try_fabric = argc > 1;
    CU(cuInit(0));
    int ndev = 0;
    cuDeviceGetCount(&ndev);
    if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
    CUdevice dev[2];
    CUcontext ctx[2];
    for (int i = 0; i < 2; ++i) { CU(cuDeviceGet(&dev[i], i)); CU(cuDevicePrimaryCtxRetain(&ctx[i], dev[i])); }
    CU(cuCtxSetCurrent(ctx[0]));
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof mp);
    mp.numDevices = 2;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    mp.size = 1 << 21;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t size = ((size_t)(64 << 20) + gran - 1) / gran * gran;
    mp.size = size;
    printf("granularity %zu, size %zu\n", gran, size);
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    int fd = -1;
    CUW(cuMemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    if (try_fabric) {   // fabric export of a multicast object
        CUmulticastObjectProp mp2 = mp;
        mp2.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
        CUmemGenericAllocationHandle mc2;
        CUresult r = cuMulticastCreate(&mc2, &mp2);
        printf("cuMulticastCreate(FABRIC) -> %d\n", (int)r);
        if (r == CUDA_SUCCESS) {
            CUmemFabricHandle fh;
            CUW(cuMemExportToShareableHandle(&fh, mc2, CU_MEM_HANDLE_TYPE_FABRIC, 0));
            cuMemRelease(mc2);
        }
    }
    CUmemGenericAllocationHandle phys[2];
    CUdeviceptr uc[2], mcva[2];
    for (int i = 0; i < 2; ++i) {  // physical memory first (variants), then add devices
        CU(cuCtxSetCurrent(ctx[i]));
        CUmemAllocationProp pp;
        memset(&pp, 0, sizeof pp);
        pp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        pp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        pp.location.id = i;
        pp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        size_t g2 = 0;
        CUW(cuMemGetAllocationGranularity(&g2, &pp, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
        printf("alloc granularity %zu\n", g2);
        CUresult r = cuMemCreate(&phys[i], size, &pp, 0);
        printf("cuMemCreate(POSIX_FD) dev %d -> %d\n", i, (int)r);
        if (r != CUDA_SUCCESS) {
            pp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_NONE;
            r = cuMemCreate(&phys[i], size, &pp, 0);
            printf("cuMemCreate(NONE) dev %d -> %d\n", i, (int)r);
            if (r != CUDA_SUCCESS) return 1;
        }
    }
    for (int i = 0; i < 2; ++i) CU(cuMulticastAddDevice(mc, dev[i]));
    for (int i = 0; i < 2; ++i) {
        CU(cuCtxSetCurrent(ctx[i]));
        CU(cuMulticastBindMem(mc, 0, phys[i], 0, size, 0));
        CUmemAccessDesc ad;
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = i;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CU(cuMemAddressReserve(&uc[i], size, gran, 0, 0));
        CU(cuMemMap(uc[i], size, 0, phys[i], 0));
        CU(cuMemSetAccess(uc[i], size, &ad, 1));
        CU(cuMemAddressReserve(&mcva[i], size, gran, 0, 0));
        CU(cuMemMap(mcva[i], size, 0, mc, 0));
        CU(cuMemSetAccess(mcva[i], size, &ad, 1));
    }
    const int n = (int)(size / 4);
    CU(cuCtxSetCurrent(ctx[0]));
    st_kernel<<<(n / 4 + 255) / 256, 256>>>((float *)mcva[0], n);
    CU(cuCtxSynchronize());
    float h0[8], h1[8];
    CU(cuMemcpyDtoH(h0, uc[0] + 400, 32));
    CU(cuCtxSetCurrent(ctx[1]));
    CU(cuMemcpyDtoH(h1, uc[1] + 400, 32));
    printf("after multimem.st from GPU0: gpu0 %.1f %.1f gpu1 %.1f %.1f (expect 101 2)\n", h0[0], h0[1], h1[0], h1[1]);
    float *out;
    cudaSetDevice(1);
    cudaMalloc(&out, size);
    red_kernel<<<(n / 4 + 255) / 256, 256>>>((const float *)mcva[1], out, n);
    cudaDeviceSynchronize();
    cudaMemcpy(h1, (char *)out + 400, 32, cudaMemcpyDeviceToHost);
    printf("multimem.ld_reduce from GPU1: %.1f %.1f (expect 202 4)\n", h1[0], h1[1]);
    // bandwidth of ld_reduce over 64 MB from GPU1
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) red_kernel<<<(n / 4 + 255) / 256, 256>>>((const float *)mcva[1], out, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ld_reduce 64 MB: %.1f GB/s (result bytes)\n", size / (ms / 10 * 1e-3) / 1e9);
    cudaSetDevice(0);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) st_kernel<<<(n / 4 + 255) / 256, 256>>>((float *)mcva[0], n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("multimem.st 64 MB: %.1f GB/s (source bytes)\n", size / (ms / 10 * 1e-3) / 1e9);
    return 0;
}
