// NVLink all-to-all throughput against the number of SMs issuing it and the bytes each keeps in
// flight: how many CTAs must move remote data at once to reach the link ceiling. Every GPU
// pulls (TMA bulk loads into an S-stage ring, or LDG.128) / pushes (TMA bulk stores from
// shared memory) its share from / to each of the N-1 peers with k CTAs, all GPUs at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/sm_scaling_probe.cu -o build/sm_scaling_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// pull: CTA b reads tiles of peer (b % npeer), TMA into an S-stage ring, consumer = 1 warp touching
// the first word of each tile (the probe measures the link, not a local store stream)
__global__ void tma_pull(const char *const *src, int npeer, size_t bytes_per_peer, int S, int T, unsigned *sink) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[16];
    const int peer = blockIdx.x % npeer;
    const int cpp = gridDim.x / npeer, cip = blockIdx.x / npeer;
    const size_t ntiles = bytes_per_peer / T;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    auto issue = [&](size_t t, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(T));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(s32(sm + (size_t)s * T)), "l"(src[peer] + t * T), "r"(T), "r"(s32(&bar[s])) : "memory");
    };
    uint32_t ph[16] = {};
    unsigned acc = 0;
    size_t t = cip;
    for (int s = 0; s < S; ++s)
        if (t + (size_t)s * cpp < ntiles) issue(t + (size_t)s * cpp, s);
    for (int s = 0; t < ntiles; t += cpp, s = (s + 1) % S) {
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(s32(&bar[s])), "r"(ph[s]));
        ph[s] ^= 1;
        acc += *reinterpret_cast<const unsigned *>(sm + (size_t)s * T);
        if (t + (size_t)S * cpp < ntiles) issue(t + (size_t)S * cpp, s);
    }
    if (acc == 0x12345678u) *sink = acc;
}

// push: TMA bulk stores of a shared-memory tile into peer (b % npeer), S groups in flight
__global__ void tma_push(char *const *dst, int npeer, size_t bytes_per_peer, int S, int T) {
    extern __shared__ __align__(128) char sm[];
    const int peer = blockIdx.x % npeer;
    const int cpp = gridDim.x / npeer, cip = blockIdx.x / npeer;
    const size_t ntiles = bytes_per_peer / T;
    if (threadIdx.x != 0) return;
    int k = 0;
    for (size_t t = cip; t < ntiles; t += cpp, ++k) {
        const int s = k % S;
        if (k >= S) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst[peer] + t * T), "r"(s32(sm + (size_t)s * T)), "r"(T) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// LDG.128 pull, U vectors in flight per thread
template <int U>
__global__ void ldg_pull(const uint4 *const *src, int npeer, size_t vec_per_peer, unsigned *sink) {
    const int peer = blockIdx.x % npeer;
    const int cpp = gridDim.x / npeer, cip = blockIdx.x / npeer;
    const uint4 *s = src[peer];
    unsigned acc = 0;
    const size_t stride = (size_t)cpp * blockDim.x;
    for (size_t i = (size_t)cip * blockDim.x + threadIdx.x; i < vec_per_peer; i += stride * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = i + u * stride < vec_per_peer ? __ldcg(s + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x;
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    int n = 0;
    cudaGetDeviceCount(&n);
    if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
    const size_t bpp = 128ull << 20;  // bytes per peer per GPU per launch
    std::vector<char *> buf(n), land(n);
    std::vector<const char **> dsrc(n);
    std::vector<char **> ddst(n);
    std::vector<unsigned *> sink(n);
    for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        for (int e = 0; e < n; ++e)
            if (e != d) cudaDeviceEnablePeerAccess(e, 0);
        cudaMalloc(&buf[d], bpp);
        cudaMalloc(&land[d], bpp * (n - 1));
        cudaMemset(buf[d], d + 1, bpp);
        cudaMalloc(&sink[d], 4);
        cudaFuncSetAttribute(tma_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(tma_push, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        std::vector<const char *> ps;
        std::vector<char *> pd;
        for (int e = 0; e < n; ++e) {
            if (e == d) continue;
            ps.push_back(buf[e]);
            pd.push_back(land[e] + (size_t)(d < e ? d : d - 1) * bpp);
        }
        cudaMalloc(&dsrc[d], sizeof(char *) * ps.size());
        cudaMemcpy(dsrc[d], ps.data(), sizeof(char *) * ps.size(), cudaMemcpyHostToDevice);
        cudaMalloc(&ddst[d], sizeof(char *) * pd.size());
        cudaMemcpy(ddst[d], pd.data(), sizeof(char *) * pd.size(), cudaMemcpyHostToDevice);
    }
    auto run = [&](const char *what, int ctas, auto launch) {
        std::vector<cudaEvent_t> e0(n), e1(n);
        for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); }
        double worst = 1e30;
        for (int rep = 0; rep < 2; ++rep) {
            for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); }
            for (int d = 0; d < n; ++d) {
                cudaSetDevice(d);
                cudaEventRecord(e0[d]);
                for (int it = 0; it < 3; ++it) launch(d);
                cudaEventRecord(e1[d]);
            }
            for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaEventSynchronize(e1[d]); }
            worst = 1e30;
            for (int d = 0; d < n; ++d) {
                float ms;
                cudaEventElapsedTime(&ms, e0[d], e1[d]);
                const double gbs = (double)bpp * (n - 1) / (ms / 3 * 1e-3) / 1e9;
                worst = gbs < worst ? gbs : worst;
            }
        }
        printf("N=%d %-34s ctas %3d: %6.1f GB/s per GPU (min over GPUs) %s\n", n, what, ctas, worst,
               cudaGetErrorString(cudaGetLastError()));
        fflush(stdout);
    };
    const int np = n - 1;
    const int cta_list[] = {12, 24, 36, 48, 72, 96, 120, 147};
    struct Ring { int S, T; };
    const Ring rings[] = {{4, 32768}, {4, 49152}, {8, 16384}, {6, 32768}, {2, 65536}};
    for (const Ring &r : rings) {
        char what[64];
        snprintf(what, sizeof what, "TMA pull %d x %dK", r.S, r.T / 1024);
        for (int c0 : cta_list) {
            const int ctas = c0 / np * np;
            run(what, ctas, [&](int d) {
                tma_pull<<<ctas, 32, (size_t)r.S * r.T>>>(dsrc[d], np, bpp, r.S, r.T, sink[d]);
            });
        }
    }
    for (const Ring &r : rings) {
        char what[64];
        snprintf(what, sizeof what, "TMA push %d x %dK", r.S, r.T / 1024);
        for (int c0 : cta_list) {
            const int ctas = c0 / np * np;
            run(what, ctas, [&](int d) { tma_push<<<ctas, 32, (size_t)r.S * r.T>>>(ddst[d], np, bpp, r.S < 4 ? r.S : 4, r.T); });
        }
    }
    for (int c0 : cta_list) {
        const int ctas = c0 / np * np;
        run("LDG.128 pull x4, 512 thr", ctas, [&](int d) {
            ldg_pull<4><<<ctas, 512>>>((const uint4 *const *)dsrc[d], np, bpp / 16, sink[d]);
        });
    }
    return 0;
}
