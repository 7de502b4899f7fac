// nvls_bw_probe.cu — NVLink ceiling of the NVLS allreduce pattern (design input for NEXT-1):
// every GPU reduces its 1/N share of an S-byte fp16 buffer in the switch
// (multimem.ld_reduce ... acc::f32) and broadcasts it back (multimem.st), all GPUs at once.
// One process, all visible GPUs, one multicast object bound to one allocation per GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_bw_probe tools/nvls_bw_probe.cu -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)

// mode 0: ld_reduce + st (allreduce), 1: ld_reduce only (result to local memory), 2: st only
template <int U, int MODE>
__global__ void __launch_bounds__(512) nvls(__half *mc, uint4 *local, size_t v_begin, size_t v_end) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t v0 = v_begin + (size_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < v_end; v0 += U * stride) {
        uint32_t r[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t v = v0 + u * stride;
            if (v < v_end) {
                if (MODE != 2)
                    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]) : "l"(mc + 8 * v) : "memory");
                else
                    r[u][0] = r[u][1] = r[u][2] = r[u][3] = (uint32_t)v;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t v = v0 + u * stride;
            if (v >= v_end) continue;
            if (MODE == 1) {
                local[v] = make_uint4(r[u][0], r[u][1], r[u][2], r[u][3]);
            } else {
                asm volatile("multimem.st.relaxed.sys.global.v4.f16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc + 8 * v), "r"(r[u][0]),
                             "r"(r[u][1]), "r"(r[u][2]), "r"(r[u][3]) : "memory");
            }
        }
    }
}

typedef void (*KFn)(__half *, uint4 *, size_t, size_t);

int main(int argc, char **argv) {
    CU(cuInit(0));
    int n = 0;
    cuDeviceGetCount(&n);
    if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
    const size_t S = (argc > 1 ? (size_t)atol(argv[1]) : 512) << 20;  // bytes per GPU
    std::vector<CUdevice> dev(n);
    std::vector<CUcontext> ctx(n);
    for (int i = 0; i < n; ++i) { CU(cuDeviceGet(&dev[i], i)); CU(cuDevicePrimaryCtxRetain(&ctx[i], dev[i])); }
    CU(cuCtxSetCurrent(ctx[0]));
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof mp);
    mp.numDevices = n;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = S;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t size = (S + gran - 1) / gran * gran;
    mp.size = size;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &mp));
    std::vector<CUmemGenericAllocationHandle> phys(n);
    std::vector<CUdeviceptr> uc(n), mcva(n);
    for (int i = 0; i < n; ++i) {
        CU(cuCtxSetCurrent(ctx[i]));
        CUmemAllocationProp pp;
        memset(&pp, 0, sizeof pp);
        pp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        pp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        pp.location.id = i;
        pp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CU(cuMemCreate(&phys[i], size, &pp, 0));
    }
    for (int i = 0; i < n; ++i) CU(cuMulticastAddDevice(mc, dev[i]));
    std::vector<uint4 *> local(n);
    for (int i = 0; i < n; ++i) {
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
        cudaSetDevice(i);
        cudaMemset((void *)uc[i], 0, size);
        cudaMalloc(&local[i], size / n + 4096);
        cudaDeviceSynchronize();
    }
    const size_t nv = S / 16;  // 16-B vectors
    printf("N=%d, S=%zu MB per GPU\n", n, S >> 20);
    struct V { const char *name; KFn fn; int mode; };
    const V vs[] = {
        {"allreduce U=2", nvls<2, 0>, 0}, {"allreduce U=4", nvls<4, 0>, 0}, {"allreduce U=8", nvls<8, 0>, 0},
        {"ld_reduce-only U=4", nvls<4, 1>, 1}, {"ld_reduce-only U=8", nvls<8, 1>, 1},
        {"st-only U=4", nvls<4, 2>, 2},
    };
    for (const V &vv : vs) {
        for (int ctas : {148, 296, 592}) {
            std::vector<cudaEvent_t> e0(n), e1(n);
            float worst = 0;
            for (int rep = 0; rep < 2; ++rep) {
                for (int i = 0; i < n; ++i) {
                    cudaSetDevice(i);
                    if (rep == 0) { cudaEventCreate(&e0[i]); cudaEventCreate(&e1[i]); }
                    cudaEventRecord(e0[i]);
                    const size_t vb = nv * i / n, ve = nv * (i + 1) / n;
                    for (int it = 0; it < 5; ++it)
                        vv.fn<<<ctas, 512>>>((__half *)mcva[i], local[i] - vb, vb, ve);
                    cudaEventRecord(e1[i]);
                }
                for (int i = 0; i < n; ++i) { cudaSetDevice(i); cudaEventSynchronize(e1[i]); }
            }
            for (int i = 0; i < n; ++i) {
                float ms;
                cudaEventElapsedTime(&ms, e0[i], e1[i]);
                worst = ms / 5 > worst ? ms / 5 : worst;
            }
            cudaError_t err = cudaGetLastError();
            // busbw: the allreduce convention 2(N-1)/N * S / t; also the per-GPU share rate S/N / t
            printf("%-20s ctas %4d: %.3f ms  busbw %.1f GB/s  share %.1f GB/s %s\n", vv.name, ctas, worst,
                   2.0 * (n - 1) / n * S / (worst * 1e-3) / 1e9, (double)S / n / (worst * 1e-3) / 1e9,
                   err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
    }
    return 0;
}
