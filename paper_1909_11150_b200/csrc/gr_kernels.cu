// gr_kernels.cu — the sm_100a kernels of the grouped gradient reduction.
//
//   bitvector_kernel  §4.1 steps 1-3 + §4.2 release rule:
//                     ballot-populate the local bitvector from the ready flags,
//                     publish it as LL (tag|word) 64-bit words in symmetric
//                     memory, AND it with the N-1 peer bitvectors read over
//                     NVLink (__reduce_and_sync across the lanes that hold the
//                     N ranks' copies of a word), decode + release complete
//                     groups in cache-bit order, hand the list to the host.
//   data_kernel       fusion-buffer pack -> sum-allreduce -> x1/N
//                     -> unpack, as ONE persistent-style kernel per cycle with a
//                     dynamic work queue over (phase, chunk) items:
//                       LOCAL   (N=1)  g <- fl_g(fl_b(fl_b(g) * 1))  in place, no buffer
//                       ONESHOT        pack all; then every rank sums all N copies
//                       TWOSHOT        pack non-owned chunks; owner reduces its
//                                      chunks (reduce-scatter) and publishes them;
//                                      everyone pulls the others (all-gather+unpack)
//                     Chunk-level flags in symmetric memory pipeline the phases
//                     across ranks; all sums run in fp32 in rank order 0..N-1, so
//                     every rank ends with bitwise-identical gradients.
//   spin_kernel       bench-only synthetic backward compute.
//
// Memory-model notes. Flags are pushed with a system-scope fence followed by a
// relaxed system-scope store (release pattern); waiters use ld.acquire.sys on
// their LOCAL pad and then bar.sync before the CTA reads peer data. Peer data
// is read with ld.global.cg (never the non-coherent path: it changes during the
// kernel). LL bitvector words carry their cycle tag in the upper 32 bits, so a
// single 64-bit load both validates and returns the word.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "gr_internal.h"

namespace gr {

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys64(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys32(uint32_t *p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// K1: bitvector populate + AND + release
// ---------------------------------------------------------------------------------------
#ifndef GR_BV_THREADS
#define GR_BV_THREADS 512
#endif
#ifndef GR_BV_BATCH
#define GR_BV_BATCH 8
#endif
constexpr int BV_THREADS = GR_BV_THREADS;
constexpr int BV_BATCH = GR_BV_BATCH;

__global__ void __launch_bounds__(BV_THREADS, 1) bitvector_kernel(BvParams p) {
    extern __shared__ uint32_t smem[];
    uint32_t *sL = smem;          // [W] local bitvector
    uint32_t *sA = smem + p.W;    // [W] intersection
    __shared__ int s_timeout;
    __shared__ int s_wcnt[32], s_wch[32];
    __shared__ int s_tot_cnt, s_tot_ch;
    __shared__ unsigned long long s_elems;
    __shared__ int s_all[32];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const uint64_t t_start = globaltimer();
    if (tid == 0) { s_timeout = 0; s_elems = 0ull; }

    // ---- step 1: populate from pending requests, publish ----
    // ready(b) = host-marked bit (gr_mark_ready) OR device flag == epoch (gr_mark_ready_async);
    // pending(b) = ready(b) AND its group not yet released in this step (reading R4).
    uint64_t *my_slot = p.slot[p.rank] + (size_t)p.parity * p.W;
    for (int w0 = warp; w0 < p.W; w0 += nwarps * BV_BATCH) {
        uint32_t f[BV_BATCH], hb[BV_BATCH];
        int gob[BV_BATCH];
#pragma unroll
        for (int k = 0; k < BV_BATCH; ++k) {  // issue the independent loads first
            const int w = w0 + k * nwarps;
            const int b = w * 32 + lane;
            const bool valid = w < p.W && b >= GR_STATUS_BITS && b < p.nbits;
            f[k] = valid ? ld_relaxed_sys32(p.dev_flags + b) : 0u;
            hb[k] = (w < p.W) ? (p.use_inline ? p.inline_bits[w] : ld_relaxed_sys32(p.host_bits + w)) : 0u;
            gob[k] = valid ? p.group_of_bit[b] : -1;
        }
#pragma unroll
        for (int k = 0; k < BV_BATCH; ++k) {
            const int w = w0 + k * nwarps;
            if (w >= p.W) break;  // warp-uniform
            const int b = w * 32 + lane;
            bool pend = false;
            if (gob[k] >= 0 && (f[k] == p.epoch || ((hb[k] >> lane) & 1u))) {
                pend = p.group_rel_epoch[gob[k]] != p.epoch;
            } else if (b == 0) {
                pend = !p.abort_flag;     // complement-coded status bits (R1)
            } else if (b == 1) {
                pend = !p.shutdown_flag;
            }
            const uint32_t word = __ballot_sync(0xffffffffu, pend);
            if (lane == 0) {
                sL[w] = word;
                st_relaxed_sys64(my_slot + w, ((uint64_t)p.tag << 32) | word);
            }
        }
    }
    __syncthreads();
    const uint64_t t_populated = globaltimer();

    // ---- step 2: A = AND_r L_r. Lane group of GS lanes per word, lane rr
    // holds rank rr's copy (own from smem, peers via NVLink LL loads). ----
    int GS = 1;
    while (GS < p.N) GS <<= 1;
    const int wpw = 32 / GS;
    const int sub = lane / GS, rr = lane % GS;
    const unsigned gmask = (GS == 32) ? 0xffffffffu : (((1u << GS) - 1u) << (sub * GS));
    const uint64_t deadline = globaltimer() + p.timeout_ns;
    const uint64_t *peer = (rr < p.N) ? p.slot[rr] + (size_t)p.parity * p.W : nullptr;
    const int stride = nwarps * wpw;
    for (int base = warp * wpw; base < p.W; base += stride * BV_BATCH) {
        uint64_t raw[BV_BATCH];
#pragma unroll
        for (int k = 0; k < BV_BATCH; ++k) {   // issue all loads first (independent)
            const int w = base + k * stride + sub;
            raw[k] = 0;
            if (w < p.W && rr < p.N && rr != p.rank) raw[k] = ld_relaxed_sys64(peer + w);
        }
        uint32_t v[BV_BATCH];
#pragma unroll
        for (int k = 0; k < BV_BATCH; ++k) {
            const int w = base + k * stride + sub;
            v[k] = 0xffffffffu;
            if (w < p.W && rr < p.N) {
                if (rr == p.rank) {
                    v[k] = sL[w];
                } else {
                    uint64_t x = raw[k];
                    while ((uint32_t)(x >> 32) != p.tag) {
                        if (globaltimer() > deadline) { s_timeout = 1; break; }
                        x = ld_relaxed_sys64(peer + w);
                    }
                    v[k] = (uint32_t)x;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < BV_BATCH; ++k) {
            const int w = base + k * stride + sub;
            const uint32_t a = __reduce_and_sync(gmask, v[k]);
            if (rr == 0 && w < p.W) sA[w] = a;
        }
    }
    __syncthreads();
    const uint64_t t_anded = globaltimer();

    // ---- status bits (R1, R13) ----
    int status = ST_OK;
    if (s_timeout) status = ST_TIMEOUT;
    else if (!(sA[0] & 1u)) status = ST_ABORT;
    else if (!(sA[0] & 2u)) status = ST_SHUTDOWN;

    // ---- step 3 + grouping: complete groups, ascending ids ----
    int run_base = 0, run_ch = 0;
    if (status == ST_OK) {
        for (int g0 = 0; g0 < p.G; g0 += blockDim.x) {
            const int g = g0 + tid;
            bool rel = false;
            int nch = 0;
            long long el = 0;
            if (g < p.G && p.group_rel_epoch[g] != p.epoch) {
                const int b0 = p.group_bit_begin[g], b1 = p.group_bit_end[g];
                bool ok = true;
                for (int w = b0 >> 5; ok && w <= ((b1 - 1) >> 5); ++w) {
                    const int lo = (w == (b0 >> 5)) ? (b0 & 31) : 0;
                    const int hi = (w == ((b1 - 1) >> 5)) ? ((b1 - 1) & 31) : 31;
                    const uint32_t mask = (hi - lo == 31) ? 0xffffffffu : (((1u << (hi - lo + 1)) - 1u) << lo);
                    ok = (sA[w] & mask) == mask;
                }
                rel = ok;
                if (rel) { nch = p.group_nchunks[g]; el = p.group_elems[g]; }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, rel);
            const int wpre = __popc(bal & ((1u << lane) - 1u));
            int x = nch;  // inclusive warp scan of chunk counts
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            long long e = el;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) e += __shfl_down_sync(0xffffffffu, e, o);
            if (lane == 31) { s_wcnt[warp] = __popc(bal); s_wch[warp] = x; }
            if (lane == 0 && e) atomicAdd(&s_elems, (unsigned long long)e);
            __syncthreads();
            if (warp == 0) {  // exclusive scan of the per-warp totals
                int c = (lane < nwarps) ? s_wcnt[lane] : 0;
                int h = (lane < nwarps) ? s_wch[lane] : 0;
                int ci = c, hi2 = h;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int yc = __shfl_up_sync(0xffffffffu, ci, o);
                    const int yh = __shfl_up_sync(0xffffffffu, hi2, o);
                    if (lane >= o) { ci += yc; hi2 += yh; }
                }
                if (lane < nwarps) { s_wcnt[lane] = ci - c; s_wch[lane] = hi2 - h; }
                if (lane == 31) { s_tot_cnt = ci; s_tot_ch = hi2; }
            }
            __syncthreads();
            if (rel) {
                const int idx = run_base + s_wcnt[warp] + wpre;
                p.out_released[idx] = g;
                p.out_cum[idx] = run_ch + s_wch[warp] + (x - nch);
                p.group_rel_epoch[g] = p.epoch;
                int32_t *hrel = reinterpret_cast<int32_t *>(reinterpret_cast<uint32_t *>(p.result + 1) + p.W);
                hrel[idx] = g;
            }
            run_base += s_tot_cnt;
            run_ch += s_tot_ch;
            __syncthreads();
        }
        if (tid == 0) p.out_cum[run_base] = run_ch;
    }

    // ---- step_complete: every group released in this step ----
    bool all = true;
    for (int g = tid; g < p.G; g += blockDim.x) all = all && (p.group_rel_epoch[g] == p.epoch);
    const unsigned wall = __reduce_and_sync(0xffffffffu, all ? 1u : 0u);
    if (lane == 0) s_all[warp] = (int)wall;

    // ---- hand the result to the host (pinned, mapped) ----
    uint32_t *hA = reinterpret_cast<uint32_t *>(p.result + 1);
    for (int w = tid; w < p.W; w += blockDim.x) hA[w] = sA[w];
    __syncthreads();
    if (tid == 0) {
        int complete = 1;
        for (int i = 0; i < nwarps; ++i) complete &= s_all[i];
        p.result->status = status;
        p.result->n_released = run_base;
        p.result->step_complete = (status == ST_OK) ? complete : 0;
        p.result->total_chunks = run_ch;
        p.result->released_elems = (int64_t)s_elems;
        p.result->t_start = t_start;
        p.result->t_populated = t_populated;
        p.result->t_anded = t_anded;
        p.result->t_end = globaltimer();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&p.result->seq), "l"(p.seq) : "memory");
    }
}

int launch_bitvector(const BvParams &p, void *stream) {
    const size_t smem = sizeof(uint32_t) * 2 * (size_t)p.W;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(bitvector_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr_set = true;
    }
    bitvector_kernel<<<1, BV_THREADS, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Data kernel: pack -> reduce -> x1/N -> unpack over the released chunks
// ---------------------------------------------------------------------------------------
constexpr int DATA_THREADS = 512;

enum Op { OP_LOCAL = 0, OP_PACK = 1, OP_RS = 2, OP_RED = 3, OP_AG = 4 };

template <typename BT> struct Buf;

template <> struct Buf<__half> {
    static constexpr int ES = 2;
    static constexpr int UNROLL = 2;   // 16-B vectors in flight per thread per rank
    struct Raw { uint4 a; };
    __device__ static __forceinline__ Raw load(const char *base, int64_t idx) {
        Raw r;
        r.a = __ldcg(reinterpret_cast<const uint4 *>(base + idx * ES));
        return r;
    }
    __device__ static __forceinline__ void to_f32(const Raw &r, float (&x)[8]) {
        const __half2 *h = reinterpret_cast<const __half2 *>(&r.a);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h[i]);
            x[2 * i] = f.x;
            x[2 * i + 1] = f.y;
        }
    }
    // round x to the buffer precision (RN-even), in place, and return the raw vector
    __device__ static __forceinline__ Raw from_f32(float (&x)[8]) {
        Raw r;
        __half2 *h = reinterpret_cast<__half2 *>(&r.a);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            h[i] = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
            const float2 f = __half22float2(h[i]);
            x[2 * i] = f.x;
            x[2 * i + 1] = f.y;
        }
        return r;
    }
    __device__ static __forceinline__ void store(char *base, int64_t idx, const Raw &r) {
        *reinterpret_cast<uint4 *>(base + idx * ES) = r.a;
    }
    __device__ static __forceinline__ float load1(const char *base, int64_t idx) {
        return __half2float(__ldcg(reinterpret_cast<const __half *>(base + idx * ES)));
    }
    __device__ static __forceinline__ float round1(float x) { return __half2float(__float2half_rn(x)); }
    __device__ static __forceinline__ void store1(char *base, int64_t idx, float x) {
        *reinterpret_cast<__half *>(base + idx * ES) = __float2half_rn(x);
    }
};

template <> struct Buf<float> {
    static constexpr int ES = 4;
    static constexpr int UNROLL = 1;   // 32-B vectors: registers bound the unroll
    struct Raw { uint4 a, b; };
    __device__ static __forceinline__ Raw load(const char *base, int64_t idx) {
        Raw r;
        const uint4 *q = reinterpret_cast<const uint4 *>(base + idx * ES);
        r.a = __ldcg(q);
        r.b = __ldcg(q + 1);
        return r;
    }
    __device__ static __forceinline__ void to_f32(const Raw &r, float (&x)[8]) {
        const float *f = reinterpret_cast<const float *>(&r);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = f[i];
    }
    __device__ static __forceinline__ Raw from_f32(float (&x)[8]) {
        Raw r;
        float *f = reinterpret_cast<float *>(&r);
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = x[i];
        return r;
    }
    __device__ static __forceinline__ void store(char *base, int64_t idx, const Raw &r) {
        uint4 *q = reinterpret_cast<uint4 *>(base + idx * ES);
        q[0] = r.a;
        q[1] = r.b;
    }
    __device__ static __forceinline__ float load1(const char *base, int64_t idx) {
        return __ldcg(reinterpret_cast<const float *>(base + idx * ES));
    }
    __device__ static __forceinline__ float round1(float x) { return x; }
    __device__ static __forceinline__ void store1(char *base, int64_t idx, float x) {
        *reinterpret_cast<float *>(base + idx * ES) = x;
    }
};

// gradient vector I/O (fp32 or fp16 gradients)
struct GradRaw { uint4 a, b; };
__device__ __forceinline__ GradRaw grad_load(const char *g, int64_t idx, bool f16) {
    GradRaw r;
    if (f16) {
        r.a = *reinterpret_cast<const uint4 *>(g + idx * 2);
    } else {
        const uint4 *q = reinterpret_cast<const uint4 *>(g + idx * 4);
        r.a = q[0];
        r.b = q[1];
    }
    return r;
}
__device__ __forceinline__ void grad_to_f32(const GradRaw &r, bool f16, float (&x)[8]) {
    if (f16) {
        const __half2 *h = reinterpret_cast<const __half2 *>(&r.a);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h[i]);
            x[2 * i] = f.x;
            x[2 * i + 1] = f.y;
        }
    } else {
        const float *f = reinterpret_cast<const float *>(&r);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = f[i];
    }
}
__device__ __forceinline__ void grad_store(char *g, int64_t idx, bool f16, const float (&x)[8]) {
    if (f16) {
        uint4 u;
        __half2 *h = reinterpret_cast<__half2 *>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
        *reinterpret_cast<uint4 *>(g + idx * 2) = u;
    } else {
        uint4 *q = reinterpret_cast<uint4 *>(g + idx * 4);
        q[0] = *reinterpret_cast<const uint4 *>(&x[0]);
        q[1] = *reinterpret_cast<const uint4 *>(&x[4]);
    }
}
__device__ __forceinline__ float grad_load1(const char *g, int64_t idx, bool f16) {
    return f16 ? __half2float(*reinterpret_cast<const __half *>(g + idx * 2))
               : *reinterpret_cast<const float *>(g + idx * 4);
}
__device__ __forceinline__ void grad_store1(char *g, int64_t idx, bool f16, float x) {
    if (f16) *reinterpret_cast<__half *>(g + idx * 2) = __float2half_rn(x);
    else *reinterpret_cast<float *>(g + idx * 4) = x;
}

// Process one chunk with operation OP. `src_rank` is the owner for OP_AG.
template <typename BT, int OP>
__device__ __forceinline__ void process_chunk(const DataParams &p, int c, int src_rank) {
    using B = Buf<BT>;
    constexpr int UNROLL = B::UNROLL;
    const Chunk ch = p.chunks[c];
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    for (int s = ch.seg_begin; s < ch.seg_end; ++s) {
        const Seg sg = p.segs[s];
        char *g = reinterpret_cast<char *>(p.dev_ptr[sg.tensor]);
        const bool f16 = sg.grad_f16 != 0;
        const int64_t esz = f16 ? 2 : 4;
        const bool aligned = ((reinterpret_cast<uintptr_t>(g) + sg.tensor_off * esz) & 15) == 0;
        const int64_t nvec = aligned ? (sg.len >> 3) : 0;
        // ---- vector body: UNROLL vectors of 8 elements per thread, loads first ----
        for (int64_t v0 = tid; v0 < nvec; v0 += (int64_t)nthr * UNROLL) {
            float x[UNROLL][8];
            bool live[UNROLL];
            if constexpr (OP == OP_LOCAL || OP == OP_PACK) {
                GradRaw gr[UNROLL];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const int64_t v = v0 + (int64_t)u * nthr;
                    live[u] = v < nvec;
                    if (live[u]) gr[u] = grad_load(g, sg.tensor_off + 8 * v, f16);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    if (!live[u]) continue;
                    const int64_t v = v0 + (int64_t)u * nthr;
                    grad_to_f32(gr[u], f16, x[u]);
                    typename B::Raw r = B::from_f32(x[u]);          // fl_b(g)
                    if constexpr (OP == OP_PACK) {
                        B::store(p.buf[p.rank], sg.buf_off + 8 * v, r);
                    } else {  // LOCAL: single rank, sum of one, x (1/N) with N = 1
#pragma unroll
                        for (int i = 0; i < 8; ++i) x[u][i] = x[u][i] * p.inv_n;
                        B::from_f32(x[u]);
                        grad_store(g, sg.tensor_off + 8 * v, f16, x[u]);
                    }
                }
            } else if constexpr (OP == OP_RS || OP == OP_RED) {
                typename B::Raw pr[UNROLL][GR_MAX_RANKS];
                GradRaw gr[UNROLL];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const int64_t v = v0 + (int64_t)u * nthr;
                    live[u] = v < nvec;
                    if (!live[u]) continue;
                    gr[u] = grad_load(g, sg.tensor_off + 8 * v, f16);
#pragma unroll
                    for (int r = 0; r < GR_MAX_RANKS; ++r)
                        if (r < p.N && r != p.rank) pr[u][r] = B::load(p.buf[r], sg.buf_off + 8 * v);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    if (!live[u]) continue;
                    const int64_t v = v0 + (int64_t)u * nthr;
                    float acc[8];
#pragma unroll
                    for (int r = 0; r < GR_MAX_RANKS; ++r) {
                        if (r >= p.N) continue;
                        float y[8];
                        if (r == p.rank) {
                            grad_to_f32(gr[u], f16, y);
                            B::from_f32(y);                           // own contribution, fl_b(g)
                        } else {
                            B::to_f32(pr[u][r], y);
                        }
#pragma unroll
                        for (int i = 0; i < 8; ++i) acc[i] = (r == 0) ? y[i] : acc[i] + y[i];
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = acc[i] * p.inv_n;
                    typename B::Raw out = B::from_f32(acc);           // fl_b(sum * 1/N)
                    if constexpr (OP == OP_RS) B::store(p.buf[p.rank], sg.buf_off + 8 * v, out);
                    grad_store(g, sg.tensor_off + 8 * v, f16, acc);
                }
            } else {  // OP_AG: pull the owner's reduced chunk, unpack
                typename B::Raw pr[UNROLL];
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    const int64_t v = v0 + (int64_t)u * nthr;
                    live[u] = v < nvec;
                    if (live[u]) pr[u] = B::load(p.buf[src_rank], sg.buf_off + 8 * v);
                }
#pragma unroll
                for (int u = 0; u < UNROLL; ++u) {
                    if (!live[u]) continue;
                    const int64_t v = v0 + (int64_t)u * nthr;
                    B::to_f32(pr[u], x[u]);
                    grad_store(g, sg.tensor_off + 8 * v, f16, x[u]);
                }
            }
        }
        // ---- scalar tail (len % 8, or an unaligned tensor) ----
        for (int64_t e = nvec * 8 + tid; e < sg.len; e += nthr) {
            const int64_t ti = sg.tensor_off + e, bi = sg.buf_off + e;
            if constexpr (OP == OP_LOCAL) {
                const float y = B::round1(B::round1(grad_load1(g, ti, f16)) * p.inv_n);
                grad_store1(g, ti, f16, y);
            } else if constexpr (OP == OP_PACK) {
                B::store1(p.buf[p.rank], bi, grad_load1(g, ti, f16));
            } else if constexpr (OP == OP_RS || OP == OP_RED) {
                float acc = 0.f;
                for (int r = 0; r < p.N; ++r) {
                    const float y = (r == p.rank) ? B::round1(grad_load1(g, ti, f16)) : B::load1(p.buf[r], bi);
                    acc = (r == 0) ? y : acc + y;
                }
                const float y = B::round1(acc * p.inv_n);
                if constexpr (OP == OP_RS) B::store1(p.buf[p.rank], bi, y);
                grad_store1(g, ti, f16, y);
            } else {
                grad_store1(g, ti, f16, B::load1(p.buf[src_rank], bi));
            }
        }
    }
}

// chunk id of item i of the released set (binary search over the cumulative counts)
__device__ __forceinline__ int chunk_of_item(const DataParams &p, int i) {
    int lo = 0, hi = p.n_released - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.cum[mid] <= i) lo = mid; else hi = mid - 1;
    }
    return p.group_chunk_begin[p.released[lo]] + (i - p.cum[lo]);
}

// thread 0: wait until *flag == epoch (or abort / timeout)
__device__ __forceinline__ void wait_flag(const DataParams &p, const uint32_t *flag, int where) {
    if (ld_acquire_sys(flag) == p.epoch) return;
    const uint64_t deadline = globaltimer() + p.timeout_ns;
    while (ld_acquire_sys(flag) != p.epoch) {
        if (*p.abort_dev) return;
        if (globaltimer() > deadline) {
            *p.abort_dev = 1;
            p.err->where = where;
            p.err->code = ST_TIMEOUT;
            return;
        }
        __nanosleep(64);
    }
}

template <typename BT, int ALGO>
__global__ void __launch_bounds__(DATA_THREADS) data_kernel(DataParams p) {
    __shared__ int s_item, s_go;
    const int tid = threadIdx.x;
    const int total = p.total_chunks;
    const int nphase = (ALGO == ALGO_LOCAL) ? 1 : (ALGO == ALGO_ONESHOT ? 2 : 3);
    for (;;) {
        if (tid == 0) s_item = atomicAdd(p.work_counter, 1);
        __syncthreads();
        const int item = s_item;
        __syncthreads();
        if (item >= nphase * total) break;
        uint64_t t_grab = 0, t_ready = 0;
        if (p.trace && tid == 0) t_grab = globaltimer();
        const int phase = item / total;
        const int c = chunk_of_item(p, item - phase * total);
        const int owner = c % p.N;
        if (ALGO == ALGO_LOCAL) {
            process_chunk<BT, OP_LOCAL>(p, c, 0);
        } else if (phase == 0) {  // pack (+ publish); two-shot owners read their own grads instead
            if (!(ALGO == ALGO_TWOSHOT && owner == p.rank)) {
                process_chunk<BT, OP_PACK>(p, c, 0);
                __syncthreads();
                if (tid == 0) {
                    fence_sys();
                    if (ALGO == ALGO_TWOSHOT) {
                        st_relaxed_sys32(p.pack_flag[owner] + (size_t)c * p.N + p.rank, p.epoch);
                    } else {
                        for (int q = 0; q < p.N; ++q)
                            if (q != p.rank) st_relaxed_sys32(p.pack_flag[q] + (size_t)c * p.N + p.rank, p.epoch);
                    }
                }
            }
        } else if (phase == 1) {  // reduce (one-shot: every chunk; two-shot: owned chunks)
            if (!(ALGO == ALGO_TWOSHOT && owner != p.rank)) {
                if (tid == 0) {
                    for (int q = 0; q < p.N; ++q)
                        if (q != p.rank) wait_flag(p, p.pack_flag[p.rank] + (size_t)c * p.N + q, 1);
                    s_go = !*p.abort_dev;
                    if (p.trace) t_ready = globaltimer();
                }
                __syncthreads();
                if (s_go) {  // uniform: s_go is read after the barrier
                    if (ALGO == ALGO_TWOSHOT) {
                        process_chunk<BT, OP_RS>(p, c, 0);
                        __syncthreads();
                        if (tid == 0) {
                            fence_sys();
                            for (int q = 0; q < p.N; ++q)
                                if (q != p.rank) st_relaxed_sys32(p.rs_flag[q] + c, p.epoch);
                        }
                    } else {
                        process_chunk<BT, OP_RED>(p, c, 0);
                    }
                }
            }
        } else if (owner != p.rank) {  // two-shot all-gather + unpack of the chunks owned by others
            if (tid == 0) {
                wait_flag(p, p.rs_flag[p.rank] + c, 2);
                s_go = !*p.abort_dev;
                if (p.trace) t_ready = globaltimer();
            }
            __syncthreads();
            if (s_go) process_chunk<BT, OP_AG>(p, c, owner);
        }
        if (p.trace && tid == 0) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            uint64_t *tr = p.trace + (size_t)item * 4;
            tr[0] = t_grab;
            tr[1] = t_ready;
            tr[2] = globaltimer();
            tr[3] = (uint64_t)blockIdx.x | ((uint64_t)smid << 32);
        }
    }
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(p.done_counter, 1) == (int)gridDim.x - 1) {
            *p.work_counter = 0;
            *p.done_counter = 0;
            __threadfence();
        }
    }
}

template <typename BT>
static int launch_data_t(const DataParams &p, int algo, int ctas, cudaStream_t s) {
    switch (algo) {
        case ALGO_LOCAL: data_kernel<BT, ALGO_LOCAL><<<ctas, DATA_THREADS, 0, s>>>(p); break;
        case ALGO_ONESHOT: data_kernel<BT, ALGO_ONESHOT><<<ctas, DATA_THREADS, 0, s>>>(p); break;
        default: data_kernel<BT, ALGO_TWOSHOT><<<ctas, DATA_THREADS, 0, s>>>(p); break;
    }
    return (int)cudaGetLastError();
}

int launch_data(const DataParams &p, int algo, int buffer_f16, int ctas, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    return buffer_f16 ? launch_data_t<__half>(p, algo, ctas, s) : launch_data_t<float>(p, algo, ctas, s);
}

template <typename BT>
static int max_ctas_t(int algo, int *out) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e;
    switch (algo) {
        case ALGO_LOCAL: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, data_kernel<BT, ALGO_LOCAL>, DATA_THREADS, 0); break;
        case ALGO_ONESHOT: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, data_kernel<BT, ALGO_ONESHOT>, DATA_THREADS, 0); break;
        default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, data_kernel<BT, ALGO_TWOSHOT>, DATA_THREADS, 0); break;
    }
    if (e != cudaSuccess) return (int)e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    *out = per_sm * sms;
    return 0;
}

int data_kernel_max_ctas(int algo, int buffer_f16, int *out) {
    return buffer_f16 ? max_ctas_t<__half>(algo, out) : max_ctas_t<float>(algo, out);
}

// ---------------------------------------------------------------------------------------
// Bench-only: synthetic backward compute (one CTA per SM via ~200 KB shared memory)
// ---------------------------------------------------------------------------------------
constexpr int SPIN_SMEM = 200 * 1024;

__global__ void __launch_bounds__(128) spin_kernel(int64_t ns) {
    extern __shared__ float sm[];
    const uint64_t t0 = globaltimer();
    float a = (float)threadIdx.x;
    while ((int64_t)(globaltimer() - t0) < ns) {
#pragma unroll 16
        for (int i = 0; i < 64; ++i) a = fmaf(a, 0.9999f, 0.5f);
    }
    if (a == 1234.5f) sm[threadIdx.x] = a;
}

int launch_spin(int64_t ns, int ctas, void *stream) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SPIN_SMEM);
        attr_set = true;
    }
    spin_kernel<<<ctas, 128, SPIN_SMEM, (cudaStream_t)stream>>>(ns);
    return (int)cudaGetLastError();
}

}  // namespace gr
