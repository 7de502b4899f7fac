// a2a_probe.cu — NVLink ceiling for the all-to-all pull pattern of the two-shot reduce: every GPU
// reads equal shares from every other GPU at the same time (design input; the roofline of
// xfer_kernel). One process, all visible GPUs, peer access enabled pairwise.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/a2a_probe tools/a2a_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

// CTA b pulls from peer (b % npeer) chunk-strided 16-B vectors with U loads in flight
template <int U>
__global__ void pull(const uint4 *const *src, int npeer, uint4 *dst, size_t n_per_peer) {
    const int peer = blockIdx.x % npeer;
    const int cta_in_peer = blockIdx.x / npeer, ctas_per_peer = gridDim.x / npeer;
    const uint4 *s = src[peer];
    uint4 *d = dst + peer * n_per_peer;
    const size_t stride = (size_t)ctas_per_peer * blockDim.x;
    for (size_t i = (size_t)cta_in_peer * blockDim.x + threadIdx.x; i < n_per_peer; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < n_per_peer) v[u] = __ldcg(s + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < n_per_peer) d[i + u * stride] = v[u];
    }
}

// push: CTA b writes chunk-strided 16-B vectors of local data into peer (b % npeer)'s memory
template <int U>
__global__ void push(uint4 *const *dst, int npeer, const uint4 *src, size_t n_per_peer) {
    const int peer = blockIdx.x % npeer;
    const int cta_in_peer = blockIdx.x / npeer, ctas_per_peer = gridDim.x / npeer;
    uint4 *d = dst[peer];
    const uint4 *s = src + peer * n_per_peer;
    const size_t stride = (size_t)ctas_per_peer * blockDim.x;
    for (size_t i = (size_t)cta_in_peer * blockDim.x + threadIdx.x; i < n_per_peer; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < n_per_peer) v[u] = __ldcg(s + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i + u * stride < n_per_peer) __stcg(d + i + u * stride, v[u]);
    }
}

// TMA bulk push: 32 KB tiles local global -> smem (bulk load) -> peer global (bulk store)
__global__ void bulk_push(char *const *dst, int npeer, const char *src, size_t bytes_per_peer) {
    constexpr int T = 32768, S = 4;
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[S];
    const int peer = blockIdx.x % npeer;
    const int cpp = gridDim.x / npeer, cip = blockIdx.x / npeer;
    const size_t ntiles = bytes_per_peer / T;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t ph[S] = {};
    int s = 0;
    size_t k = 0;
    for (size_t t = cip; t < ntiles; t += cpp, ++k, s = (s + 1) % S) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        if (k >= S)  // the bulk store that used this stage must have read smem
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(T));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(sm + s * T)), "l"(src + (size_t)peer * bytes_per_peer + t * T), "r"(T), "r"(b) : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(b), "r"(ph[s]));
        ph[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst[peer] + t * T), "r"((uint32_t)__cvta_generic_to_shared(sm + s * T)), "r"(T) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// TMA bulk pull of 32 KB tiles into a 4-stage ring, stored to local memory
__global__ void bulk_pull(const char *const *src, int npeer, char *dst, size_t bytes_per_peer) {
    constexpr int T = 32768, S = 4;
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar[S];
    const int peer = blockIdx.x % npeer;
    const int cpp = gridDim.x / npeer, cip = blockIdx.x / npeer;
    const size_t ntiles = bytes_per_peer / T;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](size_t t, int s) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(T));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(sm + s * T)), "l"(src[peer] + t * T), "r"(T), "r"(b) : "memory");
    };
    uint32_t ph[S] = {};
    size_t t = cip;
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s)
            if (t + (size_t)s * cpp < ntiles) issue(t + (size_t)s * cpp, s);
    for (int s = 0; t < ntiles; t += cpp, s = (s + 1) % S) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[s]);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(b), "r"(ph[s]));
        ph[s] ^= 1;
        uint4 *o = reinterpret_cast<uint4 *>(dst + (size_t)peer * bytes_per_peer + t * T);
        const uint4 *in = reinterpret_cast<const uint4 *>(sm + s * T);
        for (int i = threadIdx.x; i < T / 16; i += blockDim.x) o[i] = in[i];
        __syncthreads();
        if (threadIdx.x == 0 && t + (size_t)S * cpp < ntiles) issue(t + (size_t)S * cpp, s);
    }
}

int main() {
    int n = 0;
    cudaGetDeviceCount(&n);
    if (n < 2) { printf("need >= 2 GPUs\n"); return 0; }
    const size_t bytes_per_peer = 256ull << 20;
    std::vector<char *> src(n), dst(n);
    for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        for (int e = 0; e < n; ++e)
            if (e != d) cudaDeviceEnablePeerAccess(e, 0);
        cudaMalloc(&src[d], bytes_per_peer);
        cudaMalloc(&dst[d], bytes_per_peer * (n - 1));
        cudaMemset(src[d], d, bytes_per_peer);
        cudaFuncSetAttribute(bulk_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
        cudaFuncSetAttribute(bulk_push, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    }
    std::vector<const char **> dsrc(n);
    for (int d = 0; d < n; ++d) {  // peers of d
        cudaSetDevice(d);
        std::vector<const char *> ps;
        for (int e = 0; e < n; ++e)
            if (e != d) ps.push_back(src[e]);
        cudaMalloc(&dsrc[d], sizeof(char *) * ps.size());
        cudaMemcpy(dsrc[d], ps.data(), sizeof(char *) * ps.size(), cudaMemcpyHostToDevice);
    }
    // push destinations: GPU d writes into peer e's dst buffer at slot (index of d among e's peers)
    std::vector<char **> dpush(n);
    for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        std::vector<char *> ps;
        for (int e = 0; e < n; ++e) {
            if (e == d) continue;
            const int slot = d < e ? d : d - 1;
            ps.push_back(dst[e] + (size_t)slot * bytes_per_peer);
        }
        cudaMalloc(&dpush[d], sizeof(char *) * ps.size());
        cudaMemcpy(dpush[d], ps.data(), sizeof(char *) * ps.size(), cudaMemcpyHostToDevice);
    }
    // push source: a local buffer of (n-1) * bytes_per_peer (reuse dst of the same GPU as the
    // source region is harmless for bandwidth: use a separate allocation)
    std::vector<char *> psrc(n);
    for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaMalloc(&psrc[d], bytes_per_peer * (n - 1));
        cudaMemset(psrc[d], 1, bytes_per_peer * (n - 1));
    }
    for (int mode = 2; mode < 4; ++mode) {  // all GPUs pushing at once
        const int ctas = mode == 2 ? 148 * 2 / (n - 1) * (n - 1) : 148 / (n - 1) * (n - 1);
        std::vector<cudaEvent_t> e0(n), e1(n);
        for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]); }
        for (int rep = 0; rep < 2; ++rep) {
            for (int d = 0; d < n; ++d) {
                cudaSetDevice(d);
                cudaEventRecord(e0[d]);
                for (int it = 0; it < 5; ++it) {
                    if (mode == 2)
                        push<4><<<ctas, 512>>>((uint4 *const *)dpush[d], n - 1, (const uint4 *)psrc[d], bytes_per_peer / 16);
                    else
                        bulk_push<<<ctas, 32, 4 * 32768>>>(dpush[d], n - 1, psrc[d], bytes_per_peer);
                }
                cudaEventRecord(e1[d]);
            }
            for (int d = 0; d < n; ++d) { cudaSetDevice(d); cudaEventSynchronize(e1[d]); }
        }
        double worst = 1e30;
        for (int d = 0; d < n; ++d) {
            float ms;
            cudaEventElapsedTime(&ms, e0[d], e1[d]);
            const double gbs = (double)bytes_per_peer * (n - 1) / (ms / 5 * 1e-3) / 1e9;
            worst = gbs < worst ? gbs : worst;
        }
        printf("N=%d %s, all GPUs pushing at once: outgoing per GPU %.1f GB/s (min over GPUs) %s\n", n,
               mode == 2 ? "STG.128 x4" : "TMA bulk store 32K x4", worst, cudaGetErrorString(cudaGetLastError()));
    }
    for (int npar : {n, 1}) {  // all GPUs pulling at once, or one at a time
        for (int mode = 0; mode < 2; ++mode) {
            const int ctas = mode == 0 ? 148 * 2 / (n - 1) * (n - 1) : 148 / (n - 1) * (n - 1);
            std::vector<cudaEvent_t> e0(n), e1(n);
            for (int d = 0; d < n; ++d) {
                cudaSetDevice(d);
                cudaEventCreate(&e0[d]);
                cudaEventCreate(&e1[d]);
            }
            for (int rep = 0; rep < 2; ++rep) {
                for (int d = 0; d < npar; ++d) {
                    cudaSetDevice(d);
                    cudaEventRecord(e0[d]);
                    for (int it = 0; it < 5; ++it) {
                        if (mode == 0)
                            pull<4><<<ctas, 512>>>((const uint4 *const *)dsrc[d], n - 1, (uint4 *)dst[d], bytes_per_peer / 16);
                        else
                            bulk_pull<<<ctas, 256, 4 * 32768>>>(dsrc[d], n - 1, dst[d], bytes_per_peer);
                    }
                    cudaEventRecord(e1[d]);
                }
                for (int d = 0; d < npar; ++d) {
                    cudaSetDevice(d);
                    cudaEventSynchronize(e1[d]);
                }
            }
            double worst = 1e30;
            for (int d = 0; d < npar; ++d) {
                float ms;
                cudaEventElapsedTime(&ms, e0[d], e1[d]);
                const double gbs = (double)bytes_per_peer * (n - 1) / (ms / 5 * 1e-3) / 1e9;
                worst = gbs < worst ? gbs : worst;
            }
            printf("N=%d %s, %d GPU(s) pulling at once: incoming per GPU %.1f GB/s (min over GPUs)\n", n,
                   mode == 0 ? "LDG.128 x4" : "TMA 32K x4", npar, worst);
        }
    }
    return 0;
}
