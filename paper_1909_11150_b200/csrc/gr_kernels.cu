// gr_kernels.cu — the sm_100a kernels of the grouped gradient reduction.
//
//   bitvector_kernel  §4.1 steps 1-3 + §4.2 release rule:
//                     ballot-populate the local bitvector from the ready flags,
//                     publish it as LL (tag|word) 64-bit words in symmetric
//                     memory, AND it with the N-1 peer copies read over NVLink,
//                     decide complete groups (thread per group, or warp per large
//                     group with __reduce_and_sync), emit the ascending released
//                     list and chunk prefix sums, hand the result to the host.
//   local_kernel      N = 1: pack -> x1/N -> unpack collapsed in registers
//                     (no peer reads the fusion buffer), HBM-bound.
//   xfer_kernel       N > 1: fusion-buffer pack -> sum-allreduce
//                     -> x1/N -> unpack in ONE warp-specialized kernel: a producer
//                     lane streams peer sub-tiles into a shared-memory ring with
//                     TMA bulk copies, consumer warps reduce / unpack. ONESHOT:
//                     every rank sums all N copies; TWOSHOT: owner reduce-scatter
//                     (chunk c owned by rank c mod N) + all-gather. Chunk flags in
//                     symmetric memory pipeline the phases across ranks; sums run
//                     in fp32 in rank order 0..N-1 on every rank, so replicas are
//                     bitwise identical.
//   spin_kernel       bench-only synthetic backward compute.
//
// Memory-model notes. Flags are pushed with a system-scope fence followed by a
// relaxed system-scope store (release pattern); the producer acquires them with
// ld.acquire.sys on its LOCAL pad, then fence.proxy.async before the TMA reads
// peer data. LL bitvector words carry their cycle tag in the upper 32 bits, so a
// single 64-bit load both validates and returns the word.
#include <atomic>
#include <cstddef>
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
__device__ __forceinline__ uint64_t ld_acquire_sys64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
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
// one self-validating 64-bit hand-off word to pinned host memory (a single PCIe write)
__device__ __forceinline__ void st_hand(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// K1: bitvector populate + AND + release
// ---------------------------------------------------------------------------------------
#ifndef GR_BV_THREADS
#define GR_BV_THREADS 256
#endif
#define GR_SMALL_GROUP_WORDS 8
#ifndef GR_BV_BATCH
#define GR_BV_BATCH 8
#endif
constexpr int BV_THREADS = GR_BV_THREADS;
constexpr int BV_BATCH = GR_BV_BATCH;

// Shared memory: sL[W] local bitvector, sA[W] intersection, sR[W] released-tensor bits of
// this step, sC[Gw] complete-group bits (Gw = ceil(G/32)).
// Two instantiations: 256 threads (small bitvectors; 56 registers, co-resident with a running
// reduction) and 1024 threads (W > 64 words, i.e. more than ~2000 tensors).
// Prologue loads of a cycle: released bits of this step and the group records, into the
// kernel's shared memory (an armed kernel runs this while it waits for its doorbell).
__device__ __forceinline__ void bitvector_preload(const BvParams &p) {
    extern __shared__ uint32_t smem[];
    const int W = p.W, G = p.G, Gw = (p.G + 31) / 32;
    uint32_t *sR = smem + 2 * W, *sC = smem + 3 * W;
    for (int w = threadIdx.x; w < W; w += blockDim.x) sR[w] = p.rel_words[w];
    for (int i = threadIdx.x; i < Gw; i += blockDim.x) sC[i] = 0u;
    if (p.stage_groups) {
        GroupInfo *sG = reinterpret_cast<GroupInfo *>(smem + ((3 * W + Gw + 1) & ~1));
        const uint2 *src = reinterpret_cast<const uint2 *>(p.groups);
        uint2 *dst = reinterpret_cast<uint2 *>(sG);
        for (int i = threadIdx.x; i < 3 * G; i += blockDim.x) dst[i] = src[i];
    }
}

template <int NT>
__device__ __forceinline__ void bitvector_body(const BvParams &p, bool preloaded = false) {
    extern __shared__ uint32_t smem[];
    const int W = p.W, G = p.G, Gw = (p.G + 31) / 32;
    uint32_t *sL = smem, *sA = smem + W, *sR = smem + 2 * W, *sC = smem + 3 * W;
    __shared__ int s_timeout;
    __shared__ int s_scan[NT / 32][3];
    __shared__ unsigned long long s_elems;
    __shared__ int s_all[NT / 32];
    __shared__ int s_tot[3];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const uint64_t t_start = globaltimer();
    if (tid == 0) { s_timeout = 0; s_elems = 0ull; }
    // released bits of this step (a new step starts from none); the group records are fetched
    // in the same load wave (no dependent global round trips later in the cycle)
    const GroupInfo *gi = p.stage_groups ? reinterpret_cast<const GroupInfo *>(smem + ((3 * W + Gw + 1) & ~1))
                                         : p.groups;
    if (!preloaded) bitvector_preload(p);
    if (p.new_step)
        for (int w = tid; w < W; w += blockDim.x) sR[w] = 0u;
    __syncthreads();

    // ---- step 1: populate from pending requests, publish ----
    // ready = host marks (gr_mark_ready, bits) | async marks (device flag == epoch, ballot);
    // pending = ready & ~released (reading R4: a ready tensor stays pending until its group goes)
    uint64_t *my_slot = p.slot[p.rank] + (size_t)p.parity * W;
    if (!p.check_async) {  // host marks only: a thread per word, no per-bit flags to gather
        for (int w = tid; w < W; w += blockDim.x) {
            const uint32_t hbw = p.use_inline ? p.inline_bits[w] : p.host_bits[w];
            const int lo = (w == 0) ? GR_STATUS_BITS : 0;
            const int hi = min(32, p.nbits - w * 32);
            const uint32_t valid = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
            uint32_t word = hbw & valid & ~sR[w];
            if (w == 0) word |= (p.abort_flag ? 0u : 1u) | (p.shutdown_flag ? 0u : 2u);  // complement-coded (R1)
            sL[w] = word;
            st_relaxed_sys64(my_slot + w, ((uint64_t)p.tag << 32) | word);
        }
    }
    for (int w0 = warp; p.check_async && w0 < W; w0 += nwarps * BV_BATCH) {
        uint32_t f[BV_BATCH], hb[BV_BATCH], mk[BV_BATCH];
#pragma unroll
        for (int k = 0; k < BV_BATCH; ++k) {  // issue the independent loads first
            const int w = w0 + k * nwarps;
            const int b = w * 32 + lane;
            f[k] = (p.check_async && w < W && b >= GR_STATUS_BITS && b < p.nbits) ? ld_relaxed_sys32(p.dev_flags + b) : 0u;
            hb[k] = (w < W) ? (p.use_inline ? p.inline_bits[w] : p.host_bits[w]) : 0u;
            mk[k] = (w < W) ? (p.use_inline ? p.inline_marked[w] : p.marked_bits[w]) : 0u;
        }
#pragma unroll
        for (int k = 0; k < BV_BATCH; ++k) {
            const int w = w0 + k * nwarps;
            if (w >= W) break;  // warp-uniform
            // a flag from a mark that raced past the cycle's snapshot waits for the next cycle
            uint32_t ready = (hb[k] | __ballot_sync(0xffffffffu, f[k] == p.epoch)) & mk[k];
            const int lo = (w == 0) ? GR_STATUS_BITS : 0;                 // tensor bits of word w
            const int hi = min(32, p.nbits - w * 32);
            const uint32_t valid = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
            if (p.drain) {  // every unreleased tensor was marked: wait for the stream-ordered flags
                const uint32_t need = valid & ~sR[w];
                const int b = w * 32 + lane;
                const uint64_t dl = globaltimer() + p.timeout_ns;
                unsigned backoff = 64;
                while ((ready & need) != need) {
                    if (globaltimer() > dl) { if (lane == 0) s_timeout = 1; break; }
                    // the wait can span the whole backward pass: poll gently (exponential
                    // backoff to ~2 us) so the flag writers' stream memory fences are not slowed
                    __nanosleep(backoff);
                    backoff = backoff < 2048 ? 2 * backoff : 2048;
                    const uint32_t fv = (b >= GR_STATUS_BITS && b < p.nbits) ? ld_relaxed_sys32(p.dev_flags + b) : 0u;
                    ready = (hb[k] | __ballot_sync(0xffffffffu, fv == p.epoch)) & mk[k];
                }
            }
            uint32_t word = ready & valid & ~sR[w];
            if (w == 0) word |= (p.abort_flag ? 0u : 1u) | (p.shutdown_flag ? 0u : 2u);  // complement-coded (R1)
            if (lane == 0) {
                sL[w] = word;
                st_relaxed_sys64(my_slot + w, ((uint64_t)p.tag << 32) | word);
            }
        }
    }
    __syncthreads();
    const uint64_t t_populated = globaltimer();

    // ---- step 2: A = AND_r L_r. One thread per word: the N-1 peer copies are
    // LL words (tag|word) read straight from the peers' slots over NVLink, all loads issued
    // before any is consumed; a stale tag (peer not yet in this cycle) is re-polled. ----
    const uint64_t deadline = globaltimer() + p.timeout_ns;
    constexpr int AB = NT >= 1024 ? 1 : 2;  // words per thread with all their peer loads in flight together
    for (int w0 = tid; w0 < W; w0 += blockDim.x * AB) {
        uint64_t raw[AB][GR_MAX_RANKS];
#pragma unroll
        for (int k = 0; k < AB; ++k) {
            const int w = w0 + k * blockDim.x;
#pragma unroll
            for (int r = 0; r < GR_MAX_RANKS; ++r)
                raw[k][r] = (w < W && r < p.N && r != p.rank) ? ld_relaxed_sys64(p.slot[r] + (size_t)p.parity * W + w) : 0ull;
        }
#pragma unroll
        for (int k = 0; k < AB; ++k) {
            const int w = w0 + k * blockDim.x;
            if (w >= W) break;
            uint32_t a = sL[w];
#pragma unroll
            for (int r = 0; r < GR_MAX_RANKS; ++r) {
                if (r >= p.N || r == p.rank) continue;
                uint64_t x = raw[k][r];
                while ((uint32_t)(x >> 32) != p.tag) {
                    if (globaltimer() > deadline) { s_timeout = 1; break; }
                    __nanosleep(64);
                    x = ld_relaxed_sys64(p.slot[r] + (size_t)p.parity * W + w);
                }
                a &= (uint32_t)x;
            }
            sA[w] = a;
        }
    }
    __syncthreads();
    const uint64_t t_anded = globaltimer();

    int status = ST_OK;
    if (s_timeout) status = ST_TIMEOUT;
    else if (!(sA[0] & 1u)) status = ST_ABORT;      // OR of the ranks' ABORT flags (R1, R13)
    else if (!(sA[0] & 2u)) status = ST_SHUTDOWN;

    // ---- step 3 + grouping ----
    // pass 1: complete(g) = every bit of g's contiguous range set in A (released groups never
    // are: their bits left every L_r). Small groups: a thread each; groups spanning more than
    // GR_SMALL_GROUP_WORDS words: a warp each, words lane-parallel, __reduce_and_sync.
    auto word_mask = [](int w, int b0, int b1) -> uint32_t {
        const int lo = (w == (b0 >> 5)) ? (b0 & 31) : 0;
        const int hi = (w == ((b1 - 1) >> 5)) ? ((b1 - 1) & 31) : 31;
        return (hi - lo == 31) ? 0xffffffffu : (((1u << (hi - lo + 1)) - 1u) << lo);
    };
    if (status == ST_OK) {
        for (int g = tid; g < G; g += blockDim.x) {
            const int b0 = gi[g].bit_begin, b1 = gi[g].bit_end;
            if (((b1 - 1) >> 5) - (b0 >> 5) + 1 > GR_SMALL_GROUP_WORDS) continue;
            bool ok = true;
            for (int w = b0 >> 5; ok && w <= ((b1 - 1) >> 5); ++w) {
                const uint32_t m = word_mask(w, b0, b1);
                ok = (sA[w] & m) == m;
            }
            if (ok) atomicOr(&sC[g >> 5], 1u << (g & 31));
        }
        for (int i = warp; i < p.n_big; i += nwarps) {
            const int g = p.big_groups[i];
            const int b0 = gi[g].bit_begin, b1 = gi[g].bit_end;
            bool ok = true;
            for (int w = (b0 >> 5) + lane; w <= ((b1 - 1) >> 5); w += 32) {
                const uint32_t m = word_mask(w, b0, b1);
                ok = ok && ((sA[w] & m) == m);
            }
            if (__reduce_and_sync(0xffffffffu, ok ? 1u : 0u) && lane == 0) atomicOr(&sC[g >> 5], 1u << (g & 31));
        }
    }
    __syncthreads();
    // pass 2 (one pass): thread t owns complete-bitmask words [t*per, (t+1)*per); a block scan
    // of (count, chunks) gives every released group its slot in the ascending list and its
    // chunk prefix; the group's bits join the released set.
    const int per = (Gw + blockDim.x - 1) / blockDim.x;
    int my_cnt = 0, my_ch = 0, my_sub = 0;
    long long my_el = 0;
    for (int i = tid * per; i < min(Gw, (tid + 1) * per); ++i)
        for (uint32_t m = sC[i]; m; m &= m - 1) {
            const int g = i * 32 + __ffs(m) - 1;
            ++my_cnt;
            my_ch += gi[g].nchunks;
            my_sub += gi[g].nsub;
            my_el += gi[g].elems;
        }
    int xc = my_cnt, xh = my_ch, xs = my_sub;  // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int yc = __shfl_up_sync(0xffffffffu, xc, o), yh = __shfl_up_sync(0xffffffffu, xh, o);
        const int ys = __shfl_up_sync(0xffffffffu, xs, o);
        if (lane >= o) { xc += yc; xh += yh; xs += ys; }
    }
    long long e = my_el;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_down_sync(0xffffffffu, e, o);
    if (lane == 0 && e) atomicAdd(&s_elems, (unsigned long long)e);
    if (lane == 31) { s_scan[warp][0] = xc; s_scan[warp][1] = xh; s_scan[warp][2] = xs; }
    __syncthreads();
    if (tid == 0) {
        int c0 = 0, h0 = 0, s0 = 0;
        for (int i = 0; i < nwarps; ++i) {
            const int c = s_scan[i][0], h = s_scan[i][1], q = s_scan[i][2];
            s_scan[i][0] = c0;
            s_scan[i][1] = h0;
            s_scan[i][2] = s0;
            c0 += c;
            h0 += h;
            s0 += q;
        }
        s_tot[0] = c0;
        s_tot[1] = h0;
        s_tot[2] = s0;
    }
    __syncthreads();
    const uint64_t htg = (uint64_t)p.htag << 32;
    uint64_t *hrel = p.hand + HW_A + W;  // released list, LL words
    {
        int idx = s_scan[warp][0] + xc - my_cnt, ch = s_scan[warp][1] + xh - my_ch;
        int sbase = s_scan[warp][2] + xs - my_sub;
        for (int i = tid * per; i < min(Gw, (tid + 1) * per); ++i)
            for (uint32_t m = sC[i]; m; m &= m - 1) {
                const int g = i * 32 + __ffs(m) - 1;
                p.out_released[idx] = g;
                p.out_cum[idx] = ch;
                p.out_subcum[idx] = sbase;
                st_hand(hrel + idx, htg | (uint32_t)g);
                ++idx;
                ch += gi[g].nchunks;
                sbase += gi[g].nsub;
                const int b0 = gi[g].bit_begin, b1 = gi[g].bit_end;
                for (int w = b0 >> 5; w <= ((b1 - 1) >> 5); ++w) atomicOr(&sR[w], word_mask(w, b0, b1));
            }
    }
    const int run_base = s_tot[0], run_ch = s_tot[1];
    if (tid == 0) {
        p.out_cum[run_base] = run_ch;
        p.out_subcum[run_base] = s_tot[2];
    }
    __syncthreads();

    // ---- step_complete: every tensor released in this step ----
    bool all = true;
    for (int w = tid; w < W; w += blockDim.x) {
        const int lo = (w == 0) ? GR_STATUS_BITS : 0, hi = min(32, p.nbits - w * 32);
        const uint32_t valid = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
        all = all && ((sR[w] & valid) == valid);
        p.rel_words[w] = sR[w];
    }
    const unsigned wall = __reduce_and_sync(0xffffffffu, all ? 1u : 0u);
    if (lane == 0) s_all[warp] = (int)wall;

    // ---- hand the result over: device copy for the data kernel, LL words for the host (no
    // fence: each word carries the cycle's tag, written in one wave by many threads) ----
    for (int w = tid; w < W; w += blockDim.x) st_hand(p.hand + HW_A + w, htg | sA[w]);
    __syncthreads();
    int complete = 1;
    for (int i = 0; i < nwarps; ++i) complete &= s_all[i];
    if (status != ST_OK) complete = 0;
    if (tid < HW_A) {
        const uint64_t t_end = globaltimer();
        const uint64_t elems = (uint64_t)s_elems;
        uint32_t v;
        if (tid == HW_STATUS) v = (uint32_t)status;
        else if (tid == HW_NREL) v = (uint32_t)run_base;
        else if (tid == HW_COMPLETE) v = (uint32_t)complete;
        else if (tid == HW_CHUNKS) v = (uint32_t)run_ch;
        else if (tid < HW_STAMPS) v = (uint32_t)(elems >> (32 * (tid - HW_ELEMS)));
        else {
            const int k = tid - HW_STAMPS;
            const uint64_t t = (k >> 1) == 0 ? t_start : (k >> 1) == 1 ? t_populated : (k >> 1) == 2 ? t_anded : t_end;
            v = (uint32_t)(t >> (32 * (k & 1)));
        }
        st_hand(p.hand + tid, htg | v);
    }
    if (tid == 0) {
        p.out_info->n_released = (status == ST_OK) ? run_base : 0;
        p.out_info->total_chunks = (status == ST_OK) ? run_ch : 0;
        p.out_info->total_subs = (status == ST_OK) ? s_tot[2] : 0;
        p.out_info->elems = (status == ST_OK) ? (int64_t)s_elems : 0;
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&p.out_info->tag), "r"(p.htag) : "memory");
        // a drain cycle is not awaited by the host: a failure (or a step left incomplete)
        // is reported through the error block checked by the next gr_step / gr_wait
        if (p.drain && (status != ST_OK || !complete)) {
            p.err->where = status;
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&p.err->code), "r"(10 + status) : "memory");
        }
    }
}

// One rank per launch (the product path: one process per GPU).
template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) bitvector_kernel(const __grid_constant__ BvParams p) {
    bitvector_body<NT>(p);
}

// Armed cycles: a bitvector kernel that stays resident across a tight loop of cycles (N = 1; at
// N > 1 it serves one cycle and exits). For cycle
// sq = seq, seq+1, ... its threads poll descriptor sq % GR_ARM_SLOTS (pinned host memory) in
// parallel (thread i: LL word i) for at most `expire_ns` — bounded residency: one small CTA, and
// a device-wide synchronize waits at most that long — so a cycle arrives in one PCIe round trip
// after the host writes it. Thread 0 owns the control word and acknowledges every cycle in
// pinned memory: ack = sq << 1 | 1 "accepted, running it", or sq << 1 "expired before its
// doorbell" (the host then launches that cycle itself). While waiting, the kernel already holds
// the step's released bits and the group records (the previous cycle ran in this very CTA).
template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) bitvector_kernel_armed(const __grid_constant__ BvParams p,
                                                                        const CycleDesc *descs, uint32_t seq,
                                                                        uint64_t expire_ns, uint32_t *ack) {
    __shared__ BvParams sp;
    __shared__ volatile int s_state;  // 0 polling, 1 run, 2 leave
    __shared__ uint32_t sv[16 + 2 * GR_BV_INLINE_WORDS];
    const int t = threadIdx.x;
    const bool mine = t < D_SLOT + 1 || (t >= D_BITS && t < D_BITS + p.W) || (t >= D_MARKED && t < D_MARKED + p.W);
    {   // static part: copy the launch parameters word by word (once)
        const uint32_t *src = reinterpret_cast<const uint32_t *>(&p);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&sp);
        for (int i = t; i < (int)(sizeof(BvParams) / 4); i += blockDim.x) dst[i] = src[i];
    }
    if (t == 0) st_relaxed_sys32(ack + 1, seq);  // resident: data kernels may now wait on its records
    for (uint32_t sq = seq;; sq = (sq + 1 >= 0x7fffffffu) ? 1u : sq + 1) {
        if (t == 0) s_state = 0;
        // the previous cycle (this CTA's, or the kernel before it in the stream) is complete: its
        // released bits and the static group records load while the doorbell is awaited
        bitvector_preload(p);
        __syncthreads();
        const CycleDesc *desc = descs + sq % GR_ARM_SLOTS;
        if (t == 0) {
            const uint64_t dl = globaltimer() + expire_ns;
            for (;;) {
                const uint64_t v = ld_acquire_sys64(&desc->w[D_CTRL]);
                if ((uint32_t)(v >> 32) == sq) {
                    if (v & 1ull) { s_state = 2; break; }  // retired by the host
                    st_relaxed_sys32(ack, (sq << 1) | 1u);
                    s_state = 1;
                    break;
                }
                if (globaltimer() > dl) {
                    st_relaxed_sys32(ack, sq << 1);
                    s_state = 2;
                    break;
                }
                __nanosleep(64);
            }
        } else if (mine) {  // data words: valid once they carry sq (written before the control word)
            for (;;) {
                const uint64_t v = ld_relaxed_sys64(&desc->w[t]);
                if ((uint32_t)(v >> 32) == sq) { sv[t] = (uint32_t)v; break; }
                if (s_state == 2) break;
                __nanosleep(64);
            }
        }
        __syncthreads();
        if (s_state != 1) return;
        for (int w = t; w < p.W; w += blockDim.x) {
            sp.inline_bits[w] = sv[D_BITS + w];
            sp.inline_marked[w] = sv[D_MARKED + w];
        }
        if (t == 0) {
            const int slot = (int)sv[D_SLOT];
            sp.epoch = sv[D_EPOCH];
            sp.tag = sv[D_TAG];
            sp.htag = sv[D_HTAG];
            sp.parity = (int32_t)sv[D_PARITY];
            sp.new_step = (int32_t)sv[D_NEW_STEP];
            sp.check_async = (int32_t)sv[D_CHECK_ASYNC];
            sp.abort_flag = (int32_t)sv[D_ABORT];
            sp.shutdown_flag = (int32_t)sv[D_SHUTDOWN];
            sp.out_released = p.out_released + (size_t)slot * p.G;
            sp.out_cum = p.out_cum + (size_t)slot * (p.G + 1);
            sp.out_subcum = p.out_subcum + (size_t)slot * (p.G + 1);
            sp.out_info = p.out_info + slot;
        }
        __syncthreads();
        bitvector_body<NT>(sp, true);
        __syncthreads();
        // N > 1: one cycle per kernel — its data kernel is ordered after it by a stream event (a
        // resident kernel held through a multi-rank reduction timed out in the fcn220m suite)
        if (p.N > 1) return;
    }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) bitvector_kernel_v(const __grid_constant__ BvParamsV pv) {
    if (blockIdx.x >= (unsigned)pv.N || ((pv.absent >> blockIdx.x) & 1u)) return;
    bitvector_body<NT>(pv.r[blockIdx.x]);
}

// cudaFuncSetAttribute is per device: remember, per function, the devices it was set on
// (thread-safe; a process may drive several GPUs)
static bool first_use_on_device(std::atomic<uint64_t> &mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    return (mask.fetch_or(bit) & bit) == 0;
}

static void bitvector_attrs() {
    static std::atomic<uint64_t> done{0};
    if (first_use_on_device(done)) {
        cudaFuncSetAttribute(bitvector_kernel<BV_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaFuncSetAttribute(bitvector_kernel<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaFuncSetAttribute(bitvector_kernel_v<BV_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        cudaFuncSetAttribute(bitvector_kernel_v<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    }
}

static size_t bitvector_smem(const BvParams &p) {
    const size_t words = (3 * (size_t)p.W + ((size_t)p.G + 31) / 32 + 1) & ~(size_t)1;
    return sizeof(uint32_t) * words + (p.stage_groups ? sizeof(GroupInfo) * (size_t)p.G : 0);
}

int launch_bitvector(const BvParams &p, void *stream) {
    const size_t smem = bitvector_smem(p);
    bitvector_attrs();
    if (p.W > GR_BV_INLINE_WORDS) bitvector_kernel<1024><<<1, 1024, smem, (cudaStream_t)stream>>>(p);
    else bitvector_kernel<BV_THREADS><<<1, BV_THREADS, smem, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

int launch_bitvector_armed(const BvParams &p, const CycleDesc *descs, uint32_t seq, uint64_t expire_ns,
                           uint32_t *ack, void *stream) {
    const size_t smem = bitvector_smem(p);
    static std::atomic<uint64_t> done{0};
    if (first_use_on_device(done))
        cudaFuncSetAttribute(bitvector_kernel_armed<BV_THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    bitvector_kernel_armed<BV_THREADS><<<1, BV_THREADS, smem, (cudaStream_t)stream>>>(p, descs, seq, expire_ns, ack);
    return (int)cudaGetLastError();
}

int launch_bitvector_virtual(const BvParamsV &pv, void *stream) {
    int r0 = 0;  // W and G are the same on every rank (one table): take a present rank's
    while (r0 < pv.N - 1 && ((pv.absent >> r0) & 1u)) ++r0;
    const BvParams &p = pv.r[r0];
    const size_t smem = bitvector_smem(p);
    bitvector_attrs();
    if (p.W > GR_BV_INLINE_WORDS) bitvector_kernel_v<1024><<<pv.N, 1024, smem, (cudaStream_t)stream>>>(pv);
    else bitvector_kernel_v<BV_THREADS><<<pv.N, BV_THREADS, smem, (cudaStream_t)stream>>>(pv);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// Data kernel: pack -> reduce -> x1/N -> unpack over the released chunks
// ---------------------------------------------------------------------------------------


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
    __device__ static __forceinline__ float lds1(const char *base, int64_t idx) {  // generic (shared) load
        return __half2float(*reinterpret_cast<const __half *>(base + idx * ES));
    }
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
    __device__ static __forceinline__ float lds1(const char *base, int64_t idx) {
        return *reinterpret_cast<const float *>(base + idx * ES);
    }
    __device__ static __forceinline__ void store1(char *base, int64_t idx, float x) {
        *reinterpret_cast<float *>(base + idx * ES) = x;
    }
};

// NVLS: 8 buffer elements reduced in the NVSwitch (multimem.ld_reduce through the multicast
// address; fp16 accumulates in fp32 inside the switch) and broadcast back (multimem.st).
__device__ __forceinline__ void mm_ld_reduce8(const __half *mc, float (&x)[8]) {
    uint32_t r[4];
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(mc) : "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&r[i]));
        x[2 * i] = f.x;
        x[2 * i + 1] = f.y;
    }
}
__device__ __forceinline__ void mm_ld_reduce8(const float *mc, float (&x)[8]) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]) : "l"(mc) : "memory");
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7]) : "l"(mc + 4) : "memory");
}
__device__ __forceinline__ void mm_st8(__half *mc, const uint4 &v) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void mm_st8(float *mc, const uint4 &a, const uint4 &b) {
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(a.x), "r"(a.y),
                 "r"(a.z), "r"(a.w) : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + 4), "r"(b.x), "r"(b.y),
                 "r"(b.z), "r"(b.w) : "memory");
}

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
// NEXT-2 epilogue (LARS needs ||g||^2 per tensor, dynamic loss scaling needs a non-finite
// flag): accumulate the squares of the values as stored in the gradient
// tensor and note any Inf/NaN. Per thread in registers; one warp reduction + atomic per piece.
// Every 8-element buffer vector's squares are summed in fp32 (the same 8 elements on every rank
// and path: vectors are 8-aligned in the fusion buffer). ACC = float (N=1 kernel): the vector
// sums of one piece (a tensor's overlap with one warp sub-item: at most 8 per lane at the
// default 2048-element sub-item) are added in fp32 too, all terms non-negative, relative error
// below (7 + 8) * 2^-24 ~ 9e-7; one fp32 register instead of an fp64 pair keeps the HBM-bound
// kernel at its occupancy, and with one rank there is no replica to agree with. ACC = double
// (xfer kernel, N > 1): vector sums go straight into fp64, so ranks whose sub-tiles cut the
// chunk differently (reduce-scatter owner vs all-gather) agree up to the fp64 summation order
// (~1e-15 relative). The warp's partials are added in fp64 and accumulated per tensor in fp64
// (R19).
template <typename ACC>
struct GradStatT {
    ACC ss = 0;
    unsigned nf = 0;
    __device__ __forceinline__ void add8(const float (&x)[8], bool f16) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float v = f16 ? __half2float(__float2half_rn(x[i])) : x[i];
            s = fmaf(v, v, s);
            nf |= !isfinite(v);
        }
        ss += (ACC)s;
    }
    __device__ __forceinline__ void add1(float x, bool f16) {
        const float v = f16 ? __half2float(__float2half_rn(x)) : x;
        if constexpr (sizeof(ACC) == 4) ss = fmaf(v, v, ss);
        else ss += (ACC)(v * v);
        nf |= !isfinite(v);
    }
    // warp-collective: every lane of the warp must call it
    __device__ __forceinline__ void flush(double *sumsq, int32_t *nonfinite, int tensor) {
        double v = (double)ss;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const unsigned anynf = __reduce_or_sync(0xffffffffu, nf);
        if ((threadIdx.x & 31) == 0 && sumsq) {  // null: a virtual rank without statistics
            if (v != 0.0) atomicAdd(sumsq + tensor, v);
            if (anynf) atomicOr(nonfinite, 1);
        }
        ss = 0;
        nf = 0;
    }
};
using GradStat = GradStatT<float>;    // local_kernel (N = 1)
using GradStatX = GradStatT<double>;  // xfer_kernel (N > 1)

__device__ __forceinline__ void grad_store1(char *g, int64_t idx, bool f16, float x) {
    if (f16) *reinterpret_cast<__half *>(g + idx * 2) = __float2half_rn(x);
    else *reinterpret_cast<float *>(g + idx * 4) = x;
}

// Armed cycles: the data kernel is not ordered after the (resident) bitvector kernel by a stream
// event; one thread per CTA waits until the cycle's record carries its tag. false = timed out.
__device__ __forceinline__ bool wait_cycle_record(const DataParams &p) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        int ok = 1;
        if (p.wait_tag) {
            const uint32_t *tagp = &p.info->tag;
            uint32_t v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(tagp) : "memory");
            if (v != p.wait_tag) {
                const uint64_t dl = globaltimer() + p.timeout_ns;
                for (;;) {
                    __nanosleep(64);
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(tagp) : "memory");
                    if (v == p.wait_tag) break;
                    if (globaltimer() > dl) {
                        p.err->where = 3;
                        p.err->code = ST_TIMEOUT;
                        ok = 0;
                        break;
                    }
                }
            }
        }
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

// chunk id of item i of the released set (binary search over the cumulative counts)
__device__ __forceinline__ int chunk_of_item(const DataParams &p, int nrel, int i) {
    int lo = 0, hi = nrel - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.cum[mid] <= i) lo = mid; else hi = mid - 1;
    }
    return p.group_chunk_begin[p.released[lo]] + (i - p.cum[lo]);
}

// ---------------------------------------------------------------------------------------
// local_kernel (N = 1): g <- fl_g(fl_b(fl_b(g) * 1/N)) in place. With one rank no peer reads
// the fusion buffer, so pack -> reduce -> unpack collapses into one read and one write of g
// (bit-identical to the buffered path). HBM-bound: warp-granular sub-items (no block-level
// synchronisation), UNROLL 32-byte vectors in flight per lane, static interleaved schedule.
// ---------------------------------------------------------------------------------------
constexpr int LC_THREADS = 256;
// warp sub-items: p.lc_sub elements each, p.lc_subs slots per chunk
constexpr int LC_UNROLL = 2;
#ifndef GR_LC_STATS_UNROLL
#define GR_LC_STATS_UNROLL 1  // STATS: one 32-B vector per lane in flight, no spills at 64 registers (measured 1.03x of the plain pass vs 1.09x with two)
#endif
#ifndef GR_LC_MINB
#define GR_LC_MINB 4
#endif

template <typename BT, bool STATS>
__global__ void __launch_bounds__(LC_THREADS, GR_LC_MINB) local_kernel(const __grid_constant__ DataParams p) {
    using B = Buf<BT>;
    constexpr int LCU = STATS ? GR_LC_STATS_UNROLL : LC_UNROLL;
    if (!wait_cycle_record(p)) return;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (LC_THREADS / 32) + (threadIdx.x >> 5);
    const int nw = gridDim.x * (LC_THREADS / 32);
    const int nrel = p.info->n_released;
    const int nitems = p.info->total_subs;
    for (int it = gw; it < nitems; it += nw) {
        // sub-item -> released group (prefix over the groups' sub-item counts) -> chunk, offset
        int lo_ = 0, hi_ = nrel - 1;
        while (lo_ < hi_) {
            const int mid = (lo_ + hi_ + 1) >> 1;
            if (p.subcum[mid] <= it) lo_ = mid; else hi_ = mid - 1;
        }
        const int g = p.released[lo_];
        const int j = it - p.subcum[lo_];
        const int spc = p.group_spc[g];  // sub-items per full chunk of this group
        const int c = p.group_chunk_begin[g] + j / spc;
        const int64_t cb = p.chunk_begin[c], ce = p.chunk_end[c];
        const int64_t sb = cb + (int64_t)(j % spc) * p.lc_sub;
        if (sb >= ce) continue;
        const int64_t se = (sb + p.lc_sub < ce) ? sb + p.lc_sub : ce;
        const Chunk ch = p.chunks[c];
        for (int s = ch.seg_begin; s < ch.seg_end; ++s) {
            const Seg sg = p.segs[s];
            const int64_t lo = sg.buf_off > sb ? sg.buf_off : sb;
            const int64_t hi = (sg.buf_off + sg.len) < se ? (sg.buf_off + sg.len) : se;
            if (lo >= hi) continue;
            char *g = reinterpret_cast<char *>(p.dev_ptr[sg.tensor]);
            const bool f16 = sg.grad_f16 != 0;
            GradStat gs;
            const int64_t toff = sg.tensor_off + (lo - sg.buf_off);
            const bool aligned = ((reinterpret_cast<uintptr_t>(g) + toff * (f16 ? 2 : 4)) & 15) == 0;
            const int64_t n = hi - lo;
            const int64_t nvec = aligned ? (n >> 3) : 0;
            for (int64_t v0 = lane; v0 < nvec; v0 += 32 * LCU) {
                GradRaw gr[LCU];
#pragma unroll
                for (int u = 0; u < LCU; ++u)
                    if (v0 + 32 * u < nvec) gr[u] = grad_load(g, toff + 8 * (v0 + 32 * u), f16);
#pragma unroll
                for (int u = 0; u < LCU; ++u) {
                    const int64_t v = v0 + 32 * u;
                    if (v >= nvec) continue;
                    float x[8];
                    grad_to_f32(gr[u], f16, x);
                    B::from_f32(x);                                   // pack: fl_b(g)
#pragma unroll
                    for (int i = 0; i < 8; ++i) x[i] = x[i] * p.inv_n;  // sum of one rank, x 1/N
                    B::from_f32(x);                                   // fl_b(. * 1/N)
                    grad_store(g, toff + 8 * v, f16, x);              // unpack: fl_g
                    if (STATS) gs.add8(x, f16);
                }
            }
            for (int64_t e = nvec * 8 + lane; e < n; e += 32) {
                const float y = B::round1(B::round1(grad_load1(g, toff + e, f16)) * p.inv_n);
                grad_store1(g, toff + e, f16, y);
                if (STATS) gs.add1(y, f16);
            }
            if (STATS) gs.flush(p.sumsq, p.nonfinite, sg.tensor);
        }
    }
}

// ---------------------------------------------------------------------------------------
// xfer_kernel: the N>1 data path, TMA-staged and warp-specialized (one CTA per SM).
//   warp 0 / lane 0 = producer: takes work from the queue, waits for the cross-rank chunk
//     flags, and streams the peers' fusion-buffer sub-tiles into a ring of shared-memory
//     stages with cp.async.bulk (TMA bulk copies from NVLink peer memory, mbarrier
//     complete_tx) — the remote latency is hidden by the ring, not by registers;
//   warp 1 / lane 0 = publisher: takes finished chunks from the consumers (mbarrier ring),
//     fence.sc.sys, then pushes the chunk flags to the peers (the fence is off the data path);
//   warps 2..15 = consumers: pack (TMA-staged gradients -> buffer), reduce in rank order from
//     the staged copies + own gradients, scale, round, unpack (NVLS: multimem reductions).
// Work queue: triples k = 0,1,.. each holding {PACK(k), RED/RS(k-L1), AG(k-L2)} of the
// released chunk list; every rank takes them in the same order, so every dependency
// (PACK(j) before RED/RS(j) before AG(j)) points backwards in every queue: no deadlock,
// whatever subset of CTAs is resident.
// ---------------------------------------------------------------------------------------
constexpr int XF_THREADS = 512;
constexpr int XF_CONS = XF_THREADS - 64;  // warp 0 producer, warp 1 publisher, warps 2.. consumers
constexpr int XF_PUB = 32;                  // publication ring (progress waiting for the fence)
constexpr int XF_OUT = 4;                   // push: max output tiles (runtime count: p.nout)
constexpr int XF_PF = 8;                    // push: chunk flags deferred until their bulk stores complete
constexpr int XF_STAGES = 8;  // max ring depth (runtime depth: p.nstages)
enum { K_PACK = 0, K_RED = 1, K_RS = 2, K_AG = 3, K_NRS = 5, K_STOP = 4 };


__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// push path: shared-memory output tile -> (peer) global memory, tracked in bulk groups of the
// issuing thread (the publisher lane)
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(smem_u32(src_smem)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most K of this thread's bulk groups still reading shared memory (K: immediate)
__device__ __forceinline__ void bulk_wait_read(int k) {
    switch (k) {
        case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
        default: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
    }
}
// at most K of this thread's bulk groups not yet complete (their writes performed)
__device__ __forceinline__ void bulk_wait(int k) {
    switch (k) {
        case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
        default: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    }
}
__device__ __forceinline__ bool mbar_test(uint64_t *b, uint32_t parity) {
    uint32_t done;
    asm volatile("{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    return done != 0;
}

// progress word of this step: epoch in the high half, elements done (absolute fusion-buffer
// index of the end of the finished prefix of the chunk) in the low half
__device__ __forceinline__ uint64_t progress_word(uint32_t epoch, int64_t done) {
    return ((uint64_t)epoch << 32) | (uint64_t)(uint32_t)done;
}
// a producer lane: wait until *flag reports this step's progress >= need (or abort / timeout);
// `known` caches the progress already seen (no re-poll while need <= known). false = abort
__device__ __forceinline__ bool xf_wait_progress(const DataParams &p, const uint64_t *flag, uint32_t need,
                                                 uint32_t &known, int where) {
    uint64_t v = ld_acquire_sys64(flag);
    if ((uint32_t)(v >> 32) == p.epoch && (uint32_t)v >= need) { known = (uint32_t)v; return true; }
    const uint64_t deadline = globaltimer() + p.timeout_ns;
    for (;;) {
        __nanosleep(32);
        v = ld_acquire_sys64(flag);
        if ((uint32_t)(v >> 32) == p.epoch && (uint32_t)v >= need) { known = (uint32_t)v; return true; }
        if (*p.abort_dev) return false;
        if (globaltimer() > deadline) {
            *p.abort_dev = 1;
            p.err->where = where;
            p.err->code = ST_TIMEOUT;
            return false;
        }
    }
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t tx) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}

// One gradient piece = the overlap of a segment of chunk c with the sub-tile [sb, se).
struct Piece {
    char *g;          // gradient tensor base
    int32_t tensor;   // tensor id
    int64_t lo, n;    // fusion-buffer index of the first element, element count
    int64_t toff;     // tensor index of the first element
    int64_t body;     // leading elements staged in shared memory by TMA (0: none)
    bool f16;
    bool galigned;    // gradient address 16-byte aligned (vector stores possible)
};

constexpr int XF_MAXP = 8;  // gradient pieces described in a stage's metadata (more: slow path)
struct XfMeta {
    int kind, item, chunk, last, owner;
    int npieces;              // -1: too many pieces, consumers walk the segments themselves
    int64_t sb, se;           // staged fusion-buffer range
    Piece pc[XF_MAXP];
};

__device__ __forceinline__ bool piece_of(const DataParams &p, const Seg &sg, int64_t sb, int64_t se, Piece &pc) {
    const int64_t lo = sg.buf_off > sb ? sg.buf_off : sb;
    const int64_t hi = (sg.buf_off + sg.len) < se ? (sg.buf_off + sg.len) : se;
    if (lo >= hi) return false;
    pc.g = reinterpret_cast<char *>(p.dev_ptr[sg.tensor]);
    pc.tensor = sg.tensor;
    pc.f16 = sg.grad_f16 != 0;
    pc.lo = lo;
    pc.n = hi - lo;
    pc.toff = sg.tensor_off + (lo - sg.buf_off);
    const int64_t esz = pc.f16 ? 2 : 4;
    const bool aligned = ((reinterpret_cast<uintptr_t>(pc.g) + pc.toff * esz) & 15) == 0;
    pc.galigned = aligned;
    pc.body = aligned ? ((pc.n * esz) & ~(int64_t)15) / esz : 0;
    return true;
}

__device__ __forceinline__ void lds_grad8(const char *src, bool f16, float (&x)[8]) {
    GradRaw r;
    const uint4 *q = reinterpret_cast<const uint4 *>(src);
    r.a = q[0];
    if (!f16) r.b = q[1];
    grad_to_f32(r, f16, x);
}
__device__ __forceinline__ float lds_grad1(const char *src, int64_t e, bool f16) {
    return f16 ? __half2float(reinterpret_cast<const __half *>(src)[e]) : reinterpret_cast<const float *>(src)[e];
}

// Consumers: one staged sub-tile [sb, se) of chunk c. Peer copies sit in slots 0..N-2 of
// the stage (slot_bytes apart), own gradient pieces in the gradient slot (PACK/RED/RS).
template <typename BT, int KIND, bool STATS>
__device__ __forceinline__ void xf_consume(const DataParams &p, const XfMeta &m, const char *stage,
                                           int64_t slot_bytes, const char *gslot, int ct, char *own_buf) {
    using B = Buf<BT>;
    const int64_t sb = m.sb;
    const bool slow = m.npieces < 0;
    const Chunk ch = slow ? p.chunks[m.chunk] : Chunk{0, m.npieces};
    for (int s = ch.seg_begin; s < ch.seg_end; ++s) {
        Piece pc;
        if (slow) {
            if (!piece_of(p, p.segs[s], sb, m.se, pc)) continue;
            pc.body = 0;  // slow path: nothing of the gradient was staged
        } else {
            pc = m.pc[s];
        }
        const int64_t esz = pc.f16 ? 2 : 4;
        const char *gs = gslot + (pc.lo - sb) * 4;  // staged own gradient piece
        // vectors: the staged body for kinds that read the own gradient; for AG (reads only the
        // peer slot) every whole vector of an aligned gradient — the same split as the RS path
        // (body = n rounded down to 16 B), so statistics group elements identically on all ranks
        const int64_t nvec = (KIND == K_AG) ? (pc.galigned ? (pc.n >> 3) : 0) : (pc.body >> 3);
        GradStatX st;
        for (int64_t v = ct; v < nvec; v += XF_CONS) {
            const int64_t e = 8 * v, bi = pc.lo + e, ti = pc.toff + e;
            const int64_t so = (bi - sb) * B::ES;  // byte offset inside a peer slot
            float acc[8];
            if constexpr (KIND == K_PACK) {  // own_buf: this rank's buffer, or (push) the output tile
                lds_grad8(gs + e * esz, pc.f16, acc);
                B::store(own_buf, bi, B::from_f32(acc));
                continue;
            } else if constexpr (KIND == K_AG) {
                B::to_f32(*reinterpret_cast<const typename B::Raw *>(stage + so), acc);
            } else {
                int k = 0;
#pragma unroll
                for (int r = 0; r < GR_MAX_RANKS; ++r) {
                    if (r >= p.N) continue;
                    float y[8];
                    if (r == p.rank) {
                        lds_grad8(gs + e * esz, pc.f16, y);
                        B::from_f32(y);  // own contribution in buffer precision
                    } else {
                        B::to_f32(*reinterpret_cast<const typename B::Raw *>(stage + k * slot_bytes + so), y);
                        ++k;
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) acc[i] = (r == 0) ? y[i] : acc[i] + y[i];
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = acc[i] * p.inv_n;
                typename B::Raw out = B::from_f32(acc);
                // own_buf: this rank's fusion buffer (peers pull the reduced chunk), or (push) the
                // shared-memory output tile the publisher bulk-stores into every peer's buffer
                if constexpr (KIND == K_RS) B::store(own_buf, bi, out);
            }
            grad_store(pc.g, ti, pc.f16, acc);
            if (STATS) st.add8(acc, pc.f16);
        }
        for (int64_t e = nvec * 8 + ct; e < pc.n; e += XF_CONS) {  // remainder, tail, unaligned
            const int64_t bi = pc.lo + e, ti = pc.toff + e;
            const int64_t so = (bi - sb) * B::ES;
            auto own = [&]() { return e < pc.body ? lds_grad1(gs, e, pc.f16) : grad_load1(pc.g, ti, pc.f16); };
            if constexpr (KIND == K_PACK) {
                B::store1(own_buf, bi, own());
                continue;
            }
            float y;
            if constexpr (KIND == K_AG) {
                y = B::lds1(stage, so / B::ES);
            } else {
                float a = 0.f;
                int k = 0;
                for (int r = 0; r < p.N; ++r) {
                    float x;
                    if (r == p.rank) x = B::round1(own());
                    else { x = B::lds1(stage + k * slot_bytes, so / B::ES); ++k; }
                    a = (r == 0) ? x : a + x;
                }
                y = B::round1(a * p.inv_n);
                if constexpr (KIND == K_RS) B::store1(own_buf, bi, y);
            }
            grad_store1(pc.g, ti, pc.f16, y);
            if (STATS) st.add1(y, pc.f16);
        }
        if (KIND != K_PACK && STATS) st.flush(p.sumsq, p.nonfinite, pc.tensor);
    }
}

// Consumers, NVLS owner: reduce [sb, se) in the switch, x 1/N, round to the buffer precision,
// broadcast the result into every rank's copy, and unpack it into this rank's gradients.
// Works on whole 8-element buffer vectors (tensor starts are 8-aligned in the layout, so a
// tail vector only covers padding beyond the tensor); gradients get only valid elements.
template <typename BT, bool STATS>
__device__ __forceinline__ void xf_nvls_reduce(const DataParams &p, const XfMeta &m, int ct) {
    using B = Buf<BT>;
    BT *mc = reinterpret_cast<BT *>(p.nvls_mc);
    const bool slow = m.npieces < 0;
    const Chunk ch = slow ? p.chunks[m.chunk] : Chunk{0, m.npieces};
    for (int s = ch.seg_begin; s < ch.seg_end; ++s) {
        Piece pc;
        if (slow) {
            if (!piece_of(p, p.segs[s], m.sb, m.se, pc)) continue;
        } else {
            pc = m.pc[s];
        }
        const int64_t esz = pc.f16 ? 2 : 4;
        const bool galigned = ((reinterpret_cast<uintptr_t>(pc.g) + pc.toff * esz) & 15) == 0;
        const int64_t nv = (pc.n + 7) >> 3;  // buffer vectors (the last may cover padding)
        GradStatX st;
        constexpr int U = 4;                 // switch reductions in flight per thread
        for (int64_t v0 = ct; v0 < nv; v0 += (int64_t)XF_CONS * U) {
            float x[U][8];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t v = v0 + (int64_t)u * XF_CONS;
                if (v < nv) mm_ld_reduce8(mc + pc.lo + 8 * v, x[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t v = v0 + (int64_t)u * XF_CONS;
                if (v >= nv) continue;
#pragma unroll
                for (int i = 0; i < 8; ++i) x[u][i] = x[u][i] * p.inv_n;
                typename B::Raw out = B::from_f32(x[u]);
                if constexpr (sizeof(BT) == 2) mm_st8(mc + pc.lo + 8 * v, out.a);
                else mm_st8(reinterpret_cast<float *>(mc) + pc.lo + 8 * v, reinterpret_cast<const uint4 *>(&out)[0],
                            reinterpret_cast<const uint4 *>(&out)[1]);
                const int64_t e = 8 * v;
                if (galigned && e + 8 <= pc.n) {
                    grad_store(pc.g, pc.toff + e, pc.f16, x[u]);
                    if (STATS) st.add8(x[u], pc.f16);
                } else {
                    for (int i = 0; i < 8 && e + i < pc.n; ++i) {
                        grad_store1(pc.g, pc.toff + e + i, pc.f16, x[u][i]);
                        if (STATS) st.add1(x[u][i], pc.f16);
                    }
                }
            }
        }
        if (STATS) st.flush(p.sumsq, p.nonfinite, pc.tensor);
    }
}

constexpr int XF_RCACHE = 512;  // released groups cached in shared memory for item -> chunk

// 96 registers x 512 threads leaves room on every SM for a concurrently running
// bitvector kernel (256 threads), so the next cycle's coordination never queues behind
// a long reduction.
template <typename BT, bool STATS>
__device__ __forceinline__ void xfer_body(const DataParams &p, const int cta, const int nctas) {
    using B = Buf<BT>;
    extern __shared__ __align__(1024) char xsm[];
    __shared__ __align__(8) uint64_t full[XF_STAGES], empty[XF_STAGES];
    __shared__ __align__(8) uint64_t pub_full[XF_PUB], pub_empty[XF_PUB];
    __shared__ int pub_kind[XF_PUB], pub_chunk[XF_PUB], pub_owner[XF_PUB];
    __shared__ int64_t pub_done[XF_PUB];
    __shared__ __align__(8) uint64_t out_full[XF_OUT], out_empty[XF_OUT];
    __shared__ int out_kind[XF_OUT], out_chunk[XF_OUT], out_last[XF_OUT], out_nb[XF_OUT], out_owner[XF_OUT];
    __shared__ int64_t out_sb[XF_OUT], out_se[XF_OUT];
    __shared__ XfMeta meta[XF_STAGES];
    __shared__ int s_cum[XF_RCACHE], s_cb[XF_RCACHE], s_nch[XF_RCACHE], s_icum[1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t stage_bytes = p.stage_bytes;
    const int64_t gslot_off = p.slot_bytes_red * (p.N - 1);  // gradient slot inside a RED/RS stage
    if (tid == 0) {
        for (int s = 0; s < XF_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], XF_CONS / 32);
        }
        for (int s = 0; s < XF_PUB; ++s) {
            mbar_init(&pub_full[s], XF_CONS / 32);
            mbar_init(&pub_empty[s], 1);
        }
        for (int s = 0; s < XF_OUT; ++s) {
            mbar_init(&out_full[s], XF_CONS / 32);
            mbar_init(&out_empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const int nst = p.nstages;
    if (!wait_cycle_record(p)) {
        __syncthreads();
        if (tid == 0 && atomicAdd(p.done_counter, 1) == nctas - 1) {
            *p.work_counter = 0;
            *p.pack_counter = 0;
            *p.done_counter = 0;
        }
        return;
    }
    const int nrel = p.info->n_released;
    const int total = p.info->total_chunks;
    // algorithm chosen on the device from the released message size (same rule on every rank)
    const int ALGO = (p.info->elems * B::ES <= p.one_shot_max_bytes) ? ALGO_ONESHOT
                     : (p.nvls_mc ? ALGO_NVLS : ALGO_TWOSHOT);
    const bool cached = nrel <= XF_RCACHE;
    // chunking of this message: the coarse one (the bitvector kernel's prefix, p.cum) when the
    // message holds many coarse chunks, else the fine one (every rank then owns about one
    // reduce-scatter chunk per SM even for a single released group). The decision and the
    // chunk list follow from the released set, so every rank makes the same.
    const bool fine = cached && p.group_chunk_begin_fine && total < p.fine_below;
    if (cached)
        for (int j = tid; j < nrel; j += blockDim.x) {
            const int g = p.released[j];
            s_cb[j] = fine ? p.group_chunk_begin_fine[g] : p.group_chunk_begin[g];
            s_nch[j] = fine ? p.group_nchunks_fine[g] : p.cum[j + 1] - p.cum[j];
        }
    __syncthreads();
    if (cached && tid == 0) {
        int acc = 0;
        for (int j = 0; j < nrel; ++j) {
            s_cum[j] = acc;
            acc += s_nch[j];
        }
        s_icum[0] = acc;
    }
    __syncthreads();
    const int titems = cached ? s_icum[0] : total;  // work items (chunks) of this message
    // item i -> its chunk (the item's position in the message also fixes its owner, i mod N)
    auto chunk_of = [&](int i) -> int {
        if (!cached) return chunk_of_item(p, nrel, i);
        int lo = 0, hi = nrel - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_cum[mid] <= i) lo = mid; else hi = mid - 1;
        }
        return s_cb[lo] + (i - s_cum[lo]);
    };
    const int tstride = p.trace_items / 4;  // trace: item slots per phase
    const int lag1 = p.lag1, lag2 = (ALGO == ALGO_ONESHOT) ? p.lag1 : p.lag2;
    // push (one-/two-shot): packed and reduced sub-tiles leave through shared-memory output tiles
    // that the publisher bulk-stores into the peers (NVLS keeps its multicast path)
    const bool pushed = p.push && ALGO != ALGO_NVLS;
    char *const out_base = xsm + (size_t)nst * stage_bytes;
    const int nk = titems > 0 ? titems + lag2 : 0;  // queue triples
    if (warp == 0) {
        // ---------------- producer warp: lane 0 owns the queue, barriers and flag waits;
        // the 32 lanes describe / stage the chunk's gradient pieces and issue the peer
        // TMA copies in parallel (no serial chain of dependent global loads per stage).
        int stage = 0;
        uint32_t ph = 1;  // empty barriers start "free"
        const unsigned FULL = 0xffffffffu;
        long long prof_empty = 0, prof_flags = 0;  // trace mode: producer stall cycles
        const long long prof_t0 = clock64();
        // stream chunk c as sub-tiles of `sub` elements. src: 0 none (PACK), 1 every peer
        // (RED/RS), 2 the owner (AG); grads: stage own gradient pieces (PACK/RED/RS).
        // Dependencies at sub-tile granularity: before sub-tile [sb, se) is staged, every lane q
        // in wmask waits until progress word wbase[q * wstride] covers se — lane q is the lane
        // that then issues source q's copy, so its acquire orders that TMA read.
        // Returns false on abort / timeout.
        auto produce = [&](int kind, int item, int c, int64_t sub, int src, int owner, bool grads,
                           const uint64_t *wbase, int wstride, unsigned wmask, int where,
                           uint64_t *tr, int iowner) -> bool {
            uint32_t known = 0;
            const Chunk ch = p.chunks[c];
            const int nseg = ch.seg_end - ch.seg_begin;
            Seg sg{};
            char *gp = nullptr;
            const bool have = lane < nseg;
            if (have) {
                sg = p.segs[ch.seg_begin + lane];
                gp = reinterpret_cast<char *>(p.dev_ptr[sg.tensor]);
            }
            const int64_t cb = p.chunk_begin[c], ce = p.chunk_end[c];
            const int nsub = (int)((ce - cb + sub - 1) / sub);
            for (int t = 0; t < nsub; ++t) {
                const int64_t sb = cb + t * sub, se = (sb + sub < ce) ? sb + sub : ce;
                if (wmask) {
                    int ok = 1;
                    if (p.dbg && lane == 0) {  // hang diagnosis: what this CTA waits for
                        uint64_t *d = p.dbg + (size_t)cta * 8;
                        d[1] = ((uint64_t)kind << 32) | (uint32_t)c;
                        d[2] = ((uint64_t)t << 32) | wmask;
                        d[3] = (uint64_t)se;
                    }
                    if (((wmask >> lane) & 1u) && known < (uint32_t)se) {
                        const long long t0 = clock64();
                        ok = xf_wait_progress(p, wbase + (size_t)lane * wstride, (uint32_t)se, known, where);
                        prof_flags += clock64() - t0;
                    }
                    if (!__all_sync(FULL, ok)) return false;
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // acquire -> TMA reads
                    if (t == 0 && tr && lane == 0) tr[1] = globaltimer();
                }
                if (lane == 0) {
                    const long long t0 = clock64();
                    mbar_wait(&empty[stage], ph);
                    prof_empty += clock64() - t0;
                }
                __syncwarp();
                XfMeta &m = meta[stage];
                char *dst = xsm + (size_t)stage * stage_bytes;
                Piece pc{};
                bool has = false;
                if (have) {
                    const int64_t lo = sg.buf_off > sb ? sg.buf_off : sb;
                    const int64_t hi = (sg.buf_off + sg.len) < se ? (sg.buf_off + sg.len) : se;
                    if (lo < hi) {
                        has = true;
                        pc.g = gp;
                        pc.tensor = sg.tensor;
                        pc.f16 = sg.grad_f16 != 0;
                        pc.lo = lo;
                        pc.n = hi - lo;
                        pc.toff = sg.tensor_off + (lo - sg.buf_off);
                        const int64_t esz = pc.f16 ? 2 : 4;
                        const bool al = ((reinterpret_cast<uintptr_t>(gp) + pc.toff * esz) & 15) == 0;
                        pc.galigned = al;
                        pc.body = al ? ((pc.n * esz) & ~(int64_t)15) / esz : 0;
                    }
                }
                const unsigned bal = __ballot_sync(FULL, has);
                const int np = __popc(bal);
                const bool fast = nseg <= 32 && np <= XF_MAXP;  // else: consumers walk segments, no staged grads
                if (!(grads && fast)) pc.body = 0;
                if (has && fast) m.pc[__popc(bal & ((1u << lane) - 1u))] = pc;
                if (lane == 0) {
                    m.kind = kind;
                    m.item = item;
                    m.chunk = c;
                    m.owner = iowner;
                    m.last = t == nsub - 1;
                    m.sb = sb;
                    m.se = se;
                    m.npieces = fast ? np : -1;
                }
                uint64_t *bar = &full[stage];
                if (has && pc.body > 0) {  // own gradient piece -> gradient slot
                    const int64_t esz = pc.f16 ? 2 : 4;
                    const char *gs = dst + (src == 1 ? gslot_off : 0) + (pc.lo - sb) * 4;
                    mbar_expect_tx(bar, (uint32_t)(pc.body * esz));
                    bulk_g2s(const_cast<char *>(gs), pc.g + pc.toff * esz, (uint32_t)(pc.body * esz), bar);
                }
                if (src) {  // peer copies: lane r fetches rank r's sub-tile
                    const uint32_t bytes = (uint32_t)(((se - sb) * B::ES + 15) & ~(int64_t)15);
                    const bool mine = src == 1 ? (lane < p.N && lane != p.rank) : (src == 2 ? lane == owner : lane == 0);
                    if (mine) {
                        const int slot = (src == 1) ? (lane < p.rank ? lane : lane - 1) : 0;
                        // 3: own NVLS copy; push two-shot: RS reads the local receive slot of
                        // source `lane`, AG the own buffer (the owner pushed into it)
                        const char *from = (src == 3) ? p.nvls_uc
                                           : !pushed ? p.buf[lane]
                                           : (src == 1 ? p.rsb[p.rank] + (size_t)slot * p.rsb_stride : p.buf[p.rank]);
                        mbar_expect_tx(bar, bytes);
                        bulk_g2s(dst + (size_t)slot * p.slot_bytes_red, from + sb * B::ES, bytes, bar);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bar);  // release: meta + expected bytes registered
                if (++stage == nst) { stage = 0; ph ^= 1; }
            }
            return true;
        };
        bool ok = true;
        if (p.queue_mode == 1) {
            // Split queues (round 2): PACK items (no dependencies) on their own counter; the
            // dependent queue holds position k = {RS/RED/NRS(k), AG(k - lagd)}. When the next
            // dependent item's first sub-tile is not ready yet, the producer packs instead of
            // parking, so reduce-scatters can be claimed early without idling SMs. Deadlock-free:
            // a producer blocks on a dependency only once every PACK is claimed, and PACK items
            // never wait; every reduce-scatter depends only on PACKs, every all-gather only on a
            // reduce-scatter claimed earlier in the dependent queue.
            const int lagd = p.lagd;
            const int nd = titems > 0 ? titems + (ALGO == ALGO_ONESHOT ? 0 : lagd) : 0;
            bool packs_left = titems > 0;
            auto one_pack = [&]() -> bool {  // false: the pack queue is exhausted
                for (;;) {
                    int kp = 0;
                    if (lane == 0) kp = atomicAdd(p.pack_counter, 1);
                    kp = __shfl_sync(FULL, kp, 0);
                    if (kp >= titems) return false;
                    const int own = kp % p.N;
                    if (ALGO == ALGO_TWOSHOT && own == p.rank) continue;  // owned chunks are not packed
                    if (p.trace && lane == 0) { const uint64_t t = globaltimer(); p.trace[(size_t)kp * 4] = t; p.trace[(size_t)kp * 4 + 1] = t; }
                    produce(K_PACK, kp, chunk_of(kp), p.sub_pack, 0, -1, true, nullptr, 0, 0u, 0, nullptr, own);
                    return true;
                }
            };
            // is the first sub-tile of an item ready (one read of each progress word, no wait)?
            auto ready_now = [&](const uint64_t *wbase, int wstride, unsigned wmask, int c, int64_t sub) -> bool {
                bool r = true;
                if ((wmask >> lane) & 1u) {
                    const int64_t cb = p.chunk_begin[c], ce = p.chunk_end[c];
                    const int64_t need = (cb + sub < ce) ? cb + sub : ce;
                    const uint64_t v = ld_acquire_sys64(wbase + (size_t)lane * wstride);
                    r = (uint32_t)(v >> 32) == p.epoch && (uint32_t)v >= (uint32_t)need;
                }
                return __all_sync(FULL, r);
            };
            const unsigned all = (1u << p.N) - 1u;
            const unsigned wm_red = ALGO == ALGO_TWOSHOT ? all & ~(1u << p.rank) : all;
            for (;;) {
                int kd = 0;
                if (lane == 0) kd = atomicAdd(p.work_counter, 1);
                kd = __shfl_sync(FULL, kd, 0);
                if (kd >= nd || !ok) break;
                if (p.dbg && lane == 0) p.dbg[(size_t)cta * 8] = (uint64_t)kd;
                if (kd < titems && (ALGO == ALGO_ONESHOT || kd % p.N == p.rank)) {
                    const int c = chunk_of(kd), own = kd % p.N;
                    const uint64_t *wb = p.pack_flag[p.rank] + (size_t)c * p.N;
                    const int64_t sub = ALGO == ALGO_NVLS ? ((int64_t)1 << 30) : p.sub_red;
                    while (packs_left && !ready_now(wb, 1, wm_red, c, sub)) packs_left = one_pack();
                    uint64_t *tr = p.trace ? p.trace + ((size_t)tstride + kd) * 4 : nullptr;
                    if (tr && lane == 0) tr[0] = globaltimer();
                    if (ALGO == ALGO_NVLS) ok = produce(K_NRS, tstride + kd, c, 1 << 30, 0, -1, false, wb, 1, wm_red, 1, tr, own);
                    else ok = produce(ALGO == ALGO_ONESHOT ? K_RED : K_RS, tstride + kd, c, p.sub_red, 1, -1, true, wb, 1, wm_red, 1, tr, own);
                    if (!ok) break;
                }
                const int i2 = kd - lagd;
                if (ALGO != ALGO_ONESHOT && i2 >= 0 && i2 < titems && i2 % p.N != p.rank) {
                    const int c = chunk_of(i2), owner = i2 % p.N;
                    const uint64_t *wb = p.rs_flag[p.rank] + c;
                    const unsigned wm = 1u << (ALGO == ALGO_NVLS ? 0 : owner);
                    while (packs_left && !ready_now(wb, 0, wm, c, p.sub_ag)) packs_left = one_pack();
                    uint64_t *tr = p.trace ? p.trace + ((size_t)2 * tstride + i2) * 4 : nullptr;
                    if (tr && lane == 0) tr[0] = globaltimer();
                    ok = produce(K_AG, 2 * tstride + i2, c, p.sub_ag, ALGO == ALGO_NVLS ? 3 : 2, owner, false, wb, 0, wm, 2,
                                 tr, owner);
                    if (!ok) break;
                }
            }
            while (ok && packs_left) packs_left = one_pack();  // every CTA helps finish the packs
        } else {
        int kq = 0;
        if (lane == 0) kq = atomicAdd(p.work_counter, 1);
        for (;;) {
            const int k = __shfl_sync(FULL, kq, 0);
            if (k >= nk || !ok) break;
            if (p.dbg && lane == 0) p.dbg[(size_t)cta * 8] = (uint64_t)k;
            if (lane == 0) kq = atomicAdd(p.work_counter, 1);  // prefetch the next triple
            // PACK(k): own gradients (TMA) -> fusion buffer (consumers), progress -> owner
            if (k < titems) {
                const int c = chunk_of(k);
                const int own = k % p.N;
                if (!(ALGO == ALGO_TWOSHOT && own == p.rank)) {
                    if (p.trace && lane == 0) { const uint64_t t = globaltimer(); p.trace[(size_t)k * 4] = t; p.trace[(size_t)k * 4 + 1] = t; }
                    produce(K_PACK, k, c, p.sub_pack, 0, -1, true, nullptr, 0, 0u, 0, nullptr, own);
                }
            }
            // RED(k-L1) (one-shot, every item) / RS(k-L1) (two-shot, owned items)
            const int i1 = k - lag1;
            if (i1 >= 0 && i1 < titems) {
                const int c = chunk_of(i1);
                const int own = i1 % p.N;
                if (ALGO == ALGO_ONESHOT || own == p.rank) {
                    uint64_t *tr = p.trace ? p.trace + ((size_t)tstride + i1) * 4 : nullptr;
                    if (tr && lane == 0) tr[0] = globaltimer();
                    // every source's pack progress must cover the sub-tile; one-shot and NVLS also
                    // wait for their own PACK(c) (RED overwrites g after PACK read it; the switch
                    // reads this rank's copy too)
                    const unsigned all = (1u << p.N) - 1u;
                    const unsigned wm = ALGO == ALGO_TWOSHOT ? all & ~(1u << p.rank) : all;
                    const uint64_t *wb = p.pack_flag[p.rank] + (size_t)c * p.N;
                    // NVLS: no staging, the consumers' own multimem loads are in flight -> whole chunk
                    if (ALGO == ALGO_NVLS) ok = produce(K_NRS, tstride + i1, c, 1 << 30, 0, -1, false, wb, 1, wm, 1, tr, own);
                    else ok = produce(ALGO == ALGO_ONESHOT ? K_RED : K_RS, tstride + i1, c, p.sub_red, 1, -1, true, wb, 1, wm, 1, tr, own);
                    if (!ok) break;
                }
            }
            // AG(k-L2) (two-shot: pull the owner's reduced chunks; NVLS: they are already in this
            // rank's copy, written by the owner's multicast store)
            if (ALGO != ALGO_ONESHOT) {
                const int i2 = k - lag2;
                if (i2 >= 0 && i2 < titems) {
                    const int c = chunk_of(i2);
                    const int owner = i2 % p.N;
                    if (owner != p.rank) {
                        uint64_t *tr = p.trace ? p.trace + ((size_t)2 * tstride + i2) * 4 : nullptr;
                        if (tr && lane == 0) tr[0] = globaltimer();
                        // the owner's reduce-scatter progress, polled by the lane that issues the copy
                        ok = produce(K_AG, 2 * tstride + i2, c, p.sub_ag, ALGO == ALGO_NVLS ? 3 : 2, owner, false,
                                     p.rs_flag[p.rank] + c, 0, 1u << (ALGO == ALGO_NVLS ? 0 : owner), 2, tr, owner);
                        if (!ok) break;
                    }
                }
            }
        }
        }  // triple queue
        // flag waits are spread over the polling lanes: report the largest
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long x = __shfl_xor_sync(FULL, prof_flags, o);
            prof_flags = x > prof_flags ? x : prof_flags;
        }
        if (lane == 0) {  // stop message
            mbar_wait(&empty[stage], ph);
            meta[stage].kind = K_STOP;
            mbar_arrive(&full[stage]);
            if (p.trace) {  // per-CTA stall profile after the item stamps
                uint64_t *pr = p.trace + (size_t)3 * p.trace_items + (size_t)cta * 8;
                pr[0] = (uint64_t)(clock64() - prof_t0);
                pr[1] = (uint64_t)prof_empty;
                pr[2] = (uint64_t)prof_flags;
            }
        }
    } else if (warp == 1) {
        // ---------------- publisher: takes finished chunks from the consumers (mbarrier ring,
        // the consumers' stores are release-ordered before their arrive), makes them visible at
        // system scope (fence.sc.sys waits for the stores) and pushes the chunk flags to the
        // peers — the fence latency never stalls the consumer pipeline.
        if (lane == 0 && pushed) {
            // push: issue each finished output tile as TMA bulk stores into the peers (one bulk
            // group per tile), recycle a tile once its stores have read it, and publish a tile's
            // progress only after its stores have COMPLETED (deferred: two tiles later, or at
            // once when no tile is ready).
            int j = 0, issued = 0;
            uint32_t ph = 0;
            int pf_kind[XF_PF], pf_chunk[XF_PF], pf_group[XF_PF], pf_owner[XF_PF];
            int64_t pf_done[XF_PF];
            int pf_n = 0;
            const int keep = p.nout - 1;  // groups allowed to still read shared memory
            auto flags = [&](int upto) {  // publish the deferred flags of groups <= upto
                asm volatile("fence.proxy.async.global;" ::: "memory");
                fence_sys();
                int k = 0;
                for (int i = 0; i < pf_n; ++i) {
                    if (pf_group[i] > upto) {
                        pf_kind[k] = pf_kind[i]; pf_chunk[k] = pf_chunk[i]; pf_group[k] = pf_group[i]; pf_done[k] = pf_done[i];
                        pf_owner[k] = pf_owner[i];
                        ++k;
                        continue;
                    }
                    // the next entry of the same chunk (also published now) supersedes this one
                    if (i + 1 < pf_n && pf_group[i + 1] <= upto && pf_kind[i + 1] == pf_kind[i] && pf_chunk[i + 1] == pf_chunk[i])
                        continue;
                    const int c = pf_chunk[i];
                    const uint64_t v = progress_word(p.epoch, pf_done[i]);
                    if (pf_kind[i] == K_RS) {
                        for (int q = 0; q < p.N; ++q)
                            if (q != p.rank) st_relaxed_sys64(p.rs_flag[q] + c, v);
                    } else if (ALGO == ALGO_TWOSHOT) {
                        st_relaxed_sys64(p.pack_flag[pf_owner[i]] + (size_t)c * p.N + p.rank, v);
                    } else {  // one-shot: every receiver, and this rank (its RED(c) overwrites g after PACK(c) read it)
                        for (int q = 0; q < p.N; ++q) st_relaxed_sys64(p.pack_flag[q] + (size_t)c * p.N + p.rank, v);
                    }
                }
                pf_n = k;
            };
            for (;;) {
                if (!mbar_test(&out_full[j], ph)) {
                    if (pf_n) { bulk_wait(0); flags(issued); }  // idle: nothing may wait on a deferred flag
                    mbar_wait(&out_full[j], ph);
                }
                const int kind = out_kind[j];
                if (kind == K_STOP) break;
                const int c = out_chunk[j];
                const int64_t sb = out_sb[j];
                const uint32_t nb = (uint32_t)out_nb[j];
                const char *tile = out_base + (size_t)j * p.out_bytes;
                if (kind == K_PACK && ALGO == ALGO_TWOSHOT) {  // into the owner's receive slot
                    const int o = out_owner[j];
                    bulk_s2g(p.rsb[o] + (size_t)(p.rank < o ? p.rank : p.rank - 1) * p.rsb_stride + sb * B::ES, tile, nb);
                } else {
                    for (int q = 0; q < p.N; ++q) {
                        if (q == p.rank) continue;
                        char *dst = kind == K_PACK ? p.rsb[q] + (size_t)(p.rank < q ? p.rank : p.rank - 1) * p.rsb_stride
                                                   : p.buf[q];  // RS: the reduced chunk into every peer's buffer
                        bulk_s2g(dst + sb * B::ES, tile, nb);
                    }
                }
                bulk_commit();
                ++issued;
                {   // every tile advances its chunk's progress
                    if (pf_n == XF_PF) { bulk_wait(0); flags(issued - 1); }
                    pf_kind[pf_n] = kind;
                    pf_chunk[pf_n] = c;
                    pf_group[pf_n] = issued;
                    pf_done[pf_n] = out_se[j];
                    pf_owner[pf_n] = out_owner[j];
                    ++pf_n;
                }
                // the tile of group issued-keep has been read: hand it back to the consumers
                bulk_wait_read(keep);
                if (issued - keep >= 1) mbar_arrive(&out_empty[(issued - keep - 1) % p.nout]);
                if (pf_n && pf_group[0] <= issued - 2) { bulk_wait(2); flags(issued - 2); }
                if (++j == p.nout) { j = 0; ph ^= 1; }
            }
            bulk_wait(0);
            if (pf_n) flags(issued);
        } else if (lane == 0) {
            for (int ps = 0, ph = 0;; ) {
                mbar_wait(&pub_full[ps], ph);
                const int kind = pub_kind[ps], c = pub_chunk[ps], own = pub_owner[ps];
                if (kind == K_STOP) break;
                int64_t done = pub_done[ps];
                // coalesce: later progress of the same chunk already waiting supersedes this one
                for (;;) {
                    mbar_arrive(&pub_empty[ps]);
                    if (++ps == XF_PUB) { ps = 0; ph ^= 1; }
                    if (!mbar_test(&pub_full[ps], ph) || pub_kind[ps] != kind || pub_chunk[ps] != c) break;
                    done = pub_done[ps];
                }
                fence_sys();
                const uint64_t v = progress_word(p.epoch, done);
                if (p.dbg) {
                    p.dbg[(size_t)cta * 8 + 6] += 1;
                    p.dbg[(size_t)cta * 8 + 7] = ((uint64_t)kind << 48) | ((uint64_t)(uint32_t)c << 16) | (uint32_t)own;
                }
                if (kind == K_RS || kind == K_NRS) {
                    for (int q = 0; q < p.N; ++q)
                        if (q != p.rank) st_relaxed_sys64(p.rs_flag[q] + c, v);
                } else if (ALGO == ALGO_TWOSHOT || ALGO == ALGO_NVLS) {  // the owner (NVLS: possibly this rank)
                    st_relaxed_sys64(p.pack_flag[own] + (size_t)c * p.N + p.rank, v);
                } else {  // every rank, this one included: RED(c) must not overwrite g before PACK(c) read it
                    for (int q = 0; q < p.N; ++q) st_relaxed_sys64(p.pack_flag[q] + (size_t)c * p.N + p.rank, v);
                }
            }
        }
    } else {
        const int ct = tid - 64;  // consumer thread index
        int stage = 0;
        uint32_t ph = 0;
        int ps = 0;
        uint32_t pph = 1;  // publication slots start free
        int ot = 0;
        uint32_t oph = 1;  // output tiles start free
        int pub_c = -1;    // chunk whose progress was last published, and up to where
        int64_t pub_at = 0;
        long long prof_full = 0, prof_flag = 0;
        const long long prof_t0 = clock64();
        // hand a finished chunk (or the stop message) to the publisher
        auto publish = [&](int kind, int c, int64_t done, int own) {
            const long long t0 = clock64();
            if (lane == 0) mbar_wait(&pub_empty[ps], pph);
            __syncwarp();
            if (ct == 0) {
                pub_kind[ps] = kind;
                pub_chunk[ps] = c;
                pub_done[ps] = done;
                pub_owner[ps] = own;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&pub_full[ps]);  // release: this warp's stores, ct 0's meta
            if (++ps == XF_PUB) { ps = 0; pph ^= 1; }
            prof_flag += clock64() - t0;
        };
        for (;;) {
            {
                const long long t0 = clock64();
                mbar_wait(&full[stage], ph);
                prof_full += clock64() - t0;
            }
            const XfMeta &m = meta[stage];
            const int kind = m.kind;
            if (kind == K_STOP) break;
            const int item = m.item, c = m.chunk, last = m.last, mown = m.owner;
            const int64_t msb = m.sb, mse = m.se;
            const char *st = xsm + (size_t)stage * stage_bytes;
            char *own = ALGO == ALGO_NVLS ? p.nvls_uc : p.buf[p.rank];  // this rank's fusion buffer
            // push: PACK / RS results go to an output tile (indexed like the buffer, from msb)
            const bool tile = pushed && (kind == K_PACK || kind == K_RS);
            if (tile) {
                if (lane == 0) mbar_wait(&out_empty[ot], oph);
                __syncwarp();
                own = out_base + (size_t)ot * p.out_bytes - msb * B::ES;
            }
            if (kind == K_PACK) xf_consume<BT, K_PACK, STATS>(p, m, st, 0, st, ct, own);
            else if (kind == K_RED) xf_consume<BT, K_RED, STATS>(p, m, st, p.slot_bytes_red, st + gslot_off, ct, own);
            else if (kind == K_RS) xf_consume<BT, K_RS, STATS>(p, m, st, p.slot_bytes_red, st + gslot_off, ct, own);
            else if (kind == K_NRS) xf_nvls_reduce<BT, STATS>(p, m, ct);
            else xf_consume<BT, K_AG, STATS>(p, m, st, 0, st, ct, own);
            // generic-proxy tile writes -> visible to the bulk store (async proxy) the publisher issues
            if (tile) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            // the stage is free once every consumer warp has read it
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (tile) {
                if (ct == 0) {
                    out_kind[ot] = kind;
                    out_chunk[ot] = c;
                    out_last[ot] = last;
                    out_sb[ot] = msb;
                    out_owner[ot] = mown;
                    out_se[ot] = mse;
                    out_nb[ot] = (int)(((mse - msb) * B::ES + 15) & ~(int64_t)15);
                }
                if (lane == 0) mbar_arrive(&out_full[ot]);  // release: this warp's tile writes, ct 0's meta
                if (++ot == p.nout) { ot = 0; oph ^= 1; }
            } else if (kind == K_PACK || kind == K_RS || kind == K_NRS) {
                // progress of chunk c: [chunk_begin, mse) done — published at the chunk's end and
                // every p.pub_quantum elements before it (each publication costs a system fence)
                if (c != pub_c) { pub_c = c; pub_at = p.chunk_begin[c]; }
                if (last || mse - pub_at >= p.pub_quantum) {
                    publish(kind, c, mse, mown);
                    pub_at = mse;
                }
            }
            if (p.dbg && ct == 0) {
                p.dbg[(size_t)cta * 8 + 4] += 1;
                p.dbg[(size_t)cta * 8 + 5] = ((uint64_t)kind << 48) | ((uint64_t)(uint32_t)c << 16) | (uint32_t)last;
            }
            if (p.trace && last && ct == 0) {
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                p.trace[(size_t)item * 4 + 2] = globaltimer();
                p.trace[(size_t)item * 4 + 3] = (uint64_t)cta | ((uint64_t)smid << 32);
            }
            if (++stage == nst) { stage = 0; ph ^= 1; }
        }
        if (pushed) {  // stop message through the output ring (the publisher loops on it)
            if (lane == 0) mbar_wait(&out_empty[ot], oph);
            __syncwarp();
            if (ct == 0) out_kind[ot] = K_STOP;
            if (lane == 0) mbar_arrive(&out_full[ot]);
        } else {
            publish(K_STOP, 0, 0, 0);
        }
        if (p.trace && ct == 0) {
            uint64_t *pr = p.trace + (size_t)3 * p.trace_items + (size_t)cta * 8;
            pr[3] = (uint64_t)(clock64() - prof_t0);
            pr[4] = (uint64_t)prof_full;
            pr[5] = (uint64_t)prof_flag;
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(p.done_counter, 1) == nctas - 1) {
            *p.work_counter = 0;
            *p.pack_counter = 0;
            *p.done_counter = 0;
            __threadfence();
        }
    }
}

template <typename BT, bool STATS>
__global__ void __maxnreg__(96) xfer_kernel(const __grid_constant__ DataParams p) {
    xfer_body<BT, STATS>(p, blockIdx.x, gridDim.x);
}

// Virtual ranks: N ranks' reductions in ONE launch of N x per CTAs (one CTA per SM, so every
// CTA is resident: the launch fits the SM count). CTAs are dealt round-robin (CTA b serves
// rank b mod N), so any resident prefix of the grid holds CTAs of every rank; each rank's
// CTAs share that rank's work queue exactly as a real rank's grid does.
template <typename BT, bool STATS>
__global__ void __maxnreg__(96) xfer_kernel_v(const __grid_constant__ DataParamsV pv) {
    const int r = blockIdx.x % pv.N;
    if ((pv.absent >> r) & 1u) return;
    xfer_body<BT, STATS>(pv.r[r], blockIdx.x / pv.N, pv.per);
}

template <typename BT, bool STATS>
static void xfer_attrs() {
    static std::atomic<uint64_t> done{0};
    if (first_use_on_device(done)) {
        cudaFuncSetAttribute(xfer_kernel<BT, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 208 * 1024);
        cudaFuncSetAttribute(xfer_kernel_v<BT, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 208 * 1024);
    }
}

// dynamic shared memory of the xfer kernel: the stage ring, then (push) the output tiles
static size_t xfer_smem(const DataParams &p) {
    return (size_t)p.nstages * p.stage_bytes + (p.push ? (size_t)p.nout * p.out_bytes : 0);
}

template <typename BT, bool STATS>
static int launch_data_t(const DataParams &p, int local, int ctas, cudaStream_t s) {
    xfer_attrs<BT, STATS>();
    if (local) local_kernel<BT, STATS><<<ctas, LC_THREADS, 0, s>>>(p);
    else xfer_kernel<BT, STATS><<<ctas, XF_THREADS, xfer_smem(p), s>>>(p);
    return (int)cudaGetLastError();
}

int launch_data(const DataParams &p, int local, int buffer_f16, int ctas, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (p.sumsq) return buffer_f16 ? launch_data_t<__half, true>(p, local, ctas, s) : launch_data_t<float, true>(p, local, ctas, s);
    return buffer_f16 ? launch_data_t<__half, false>(p, local, ctas, s) : launch_data_t<float, false>(p, local, ctas, s);
}

template <typename BT, bool STATS>
static int launch_data_v_t(const DataParamsV &pv, cudaStream_t s) {
    xfer_attrs<BT, STATS>();
    int r0 = 0;  // the stage ring is the same on every rank: take a present rank's
    while (r0 < pv.N - 1 && ((pv.absent >> r0) & 1u)) ++r0;
    xfer_kernel_v<BT, STATS><<<pv.N * pv.per, XF_THREADS, xfer_smem(pv.r[r0]), s>>>(pv);
    return (int)cudaGetLastError();
}

int launch_data_virtual(const DataParamsV &pv, int buffer_f16, int stats, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (stats) return buffer_f16 ? launch_data_v_t<__half, true>(pv, s) : launch_data_v_t<float, true>(pv, s);
    return buffer_f16 ? launch_data_v_t<__half, false>(pv, s) : launch_data_v_t<float, false>(pv, s);
}

template <typename BT>
static int max_ctas_t(int *out) {
    int per_sm = 0, dev = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, local_kernel<BT, false>, LC_THREADS, 0);
    if (e != cudaSuccess) return (int)e;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    *out = per_sm * sms;
    return 0;
}

int data_kernel_max_ctas(int algo, int buffer_f16, int *out) {
    (void)algo;
    return buffer_f16 ? max_ctas_t<__half>(out) : max_ctas_t<float>(out);
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
    static std::atomic<uint64_t> done{0};
    if (first_use_on_device(done)) cudaFuncSetAttribute(spin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SPIN_SMEM);
    spin_kernel<<<ctas, 128, SPIN_SMEM, (cudaStream_t)stream>>>(ns);
    return (int)cudaGetLastError();
}

}  // namespace gr
