// gr_internal.h — shared between the host runtime (gr_runtime.cpp) and the
// sm_100a kernels (gr_kernels.cu). Not part of the ABI (include/gr.h is).
#pragma once
#include <cstdint>

#define GR_MAX_RANKS 8
#define GR_STATUS_BITS 2
#define GR_SLOT_RING 64            // released-list slots in flight (cycle % ring)
#define GR_BV_INLINE_WORDS 64      // host mark bits passed as kernel parameters up to this W
#define GR_ARM_SLOTS 4             // armed-cycle descriptors in flight (cycle sq uses sq % 4)

namespace gr {

// One piece of one tensor inside one chunk of the static fusion layout.
struct Seg {
    int32_t tensor;      // tensor id
    int32_t grad_f16;    // 1 if the caller's gradient is fp16
    int64_t tensor_off;  // element offset inside the tensor (multiple of 8)
    int64_t buf_off;     // element offset inside the fusion buffer (multiple of 8)
    int64_t len;         // elements
};

// A chunk: contiguous fusion-buffer range of one group, cut at chunk_elems.
struct Chunk {
    int32_t seg_begin, seg_end;
};

// Hand-off of a cycle's result from the bitvector kernel to the host: pinned host-mapped
// 64-bit LL words (tag << 32 | payload), tag = the cycle's sequence number (low 32 bits, never
// 0). Every word validates itself, so the kernel writes them from many threads with plain
// stores and no system-scope fence; the host spins until every word it needs carries the tag.
enum HandWord {
    HW_STATUS = 0,        // 0 ok, 1 abort, 2 shutdown, 3 timeout
    HW_NREL = 1,          // released groups n
    HW_COMPLETE = 2,      // step complete
    HW_CHUNKS = 3,        // chunks of the released groups
    HW_ELEMS = 4,         // released elements (lo, hi)
    HW_STAMPS = 6,        // %globaltimer (ns): start, populated, ANDed, end (lo, hi each)
    HW_A = 14,            // A[W], then released[n]
};
inline int hand_words(int W, int G) { return HW_A + W + G; }

struct HostError {
    volatile int32_t code;   // 0 none, 3 timeout in the data kernel, 10 + status: a drain cycle failed
    volatile int32_t where;
};

enum { ST_OK = 0, ST_ABORT = 1, ST_SHUTDOWN = 2, ST_TIMEOUT = 3 };

// Cycle result handed from the bitvector kernel to the data kernel in device memory (ring
// slot): the data kernel is launched before the host sees the result and starts as soon as
// the bitvector kernel completes (stream event), with no host round trip in between.
struct DevCycle {
    int32_t n_released;
    int32_t total_chunks;
    int64_t elems;
    int32_t total_subs;    // local-kernel sub-items of the released groups
    uint32_t tag;          // the cycle's hand-off tag, stored last (release): a data kernel that
                           // is not ordered after the bitvector kernel by a stream event (armed
                           // cycles) waits for it
};

// Per-group constants the bitvector kernel needs (one 24-byte record per group, so one load
// wave fetches them all; staged in shared memory when they fit, see BvParams::stage_groups).
struct GroupInfo {
    int32_t bit_begin, bit_end;  // the group's contiguous cache-bit range [begin, end)
    int32_t nchunks;             // fusion-buffer chunks of the group
    int32_t nsub;                // local-kernel sub-items of the group
    int64_t elems;               // gradient elements of the group
};

struct BvParams {
    const uint32_t *host_bits;       // device copy [W] of the host mark bits (DMA'd before the launch);
                                     // unused when W <= GR_BV_INLINE_WORDS (passed in inline_bits)
    const uint32_t *marked_bits;     // device copy [W] of every mark taken by the cycle's snapshot:
                                     // a stream-ordered flag counts only if its mark (and so its
                                     // pointer) is in the snapshot; inline_marked when inline
    const uint32_t *dev_flags;       // device [W*32]: step epoch written by gr_mark_ready_async
    uint32_t *rel_words;             // device [W]: tensor bits released so far in this step
    int32_t new_step;                // 1 on the first cycle of a step (rel_words restart at 0)
    int32_t check_async;             // 1 if gr_mark_ready_async was used in this step
    const GroupInfo *groups;         // device [G]
    int32_t stage_groups;            // 1: copy `groups` into shared memory at kernel start
    const int32_t *big_groups;       // device [n_big]: groups spanning > 8 bitvector words
    int32_t n_big;
    uint64_t *slot[GR_MAX_RANKS];    // every rank's LL bitvector slots [2][W] (own = local)
    int32_t *out_released;           // device [G]   (ring slot)
    int32_t *out_cum;                // device [G+1] (ring slot)
    DevCycle *out_info;              // device (ring slot)
    int32_t *out_subcum;             // device [G+1] (ring slot): prefix of group_nsub over the list
    uint64_t *hand;                  // host-mapped hand-off words (HandWord layout)
    int32_t T, G, W, nbits, rank, N;
    uint32_t epoch;                  // training-step epoch (>= 1)
    uint32_t tag;                    // cycle tag written into each LL word (!= 0)
    int32_t parity;                  // cycle & 1
    int32_t abort_flag, shutdown_flag;
    uint64_t timeout_ns;
    uint32_t htag;                   // hand-off tag of this cycle (!= 0)
    int32_t use_inline;
    int32_t drain;                   // gr_step_drain: wait on the device until every unreleased
                                     // tensor of this rank is ready, no host hand-off awaited
    HostError *err;                  // drain only: failures surface here (host-mapped)
    uint32_t inline_bits[GR_BV_INLINE_WORDS];    // snapshot of host_bits passed with the launch
    uint32_t inline_marked[GR_BV_INLINE_WORDS];  // snapshot of marked_bits passed with the launch
};

enum Algo { ALGO_LOCAL = 1, ALGO_ONESHOT = 2, ALGO_TWOSHOT = 3, ALGO_NVLS = 4 };

struct DataParams {
    const Seg *segs;
    const Chunk *chunks;
    const int32_t *group_chunk_begin;  // [G] (coarse chunking)
    const int32_t *group_chunk_begin_fine;  // [G] fine chunking (N > 1; == coarse when there is one)
    const int32_t *group_nchunks_fine;      // [G]
    int32_t fine_below;                // messages of fewer coarse chunks than this use the fine chunking
    const int32_t *released;           // ring slot [G]
    const int32_t *cum;                // ring slot [G+1]
    const DevCycle *info;              // ring slot: released groups / chunks / elements
    const int32_t *subcum;             // ring slot [G+1]: local-kernel sub-item prefix
    const int32_t *group_spc;          // [G]: local-kernel sub-items per full chunk of the group
    const uint64_t *dev_ptr;           // [T]
    char *buf[GR_MAX_RANKS];           // every rank's fusion buffer for this step parity
    char *rsb[GR_MAX_RANKS];           // push: every rank's receive slots [N-1][buffer] for packed
                                       // chunks (source s lands in slot s<receiver ? s : s-1)
    int32_t push;                      // one-/two-shot by TMA bulk stores into peers (1) or by TMA
                                       // bulk loads from peers (0)
    int64_t rsb_stride;                // bytes between receive slots (one fusion buffer)
    int64_t pub_quantum;               // progress words are published every this many elements of a
                                       // chunk (and at its end)
    int64_t out_bytes;                 // push: bytes of one shared-memory output tile
    int32_t nout;                      // push: output tiles (2..4) after the stage ring
    char *nvls_uc;                     // NVLS: this rank's copy of the multicast buffer (parity), or null
    char *nvls_mc;                     // NVLS: the multicast view of it (multimem.*), or null
    // progress words (epoch << 32 | e): chunk c's fusion-buffer elements [chunk_begin, e) are done
    // (packed by source s / reduced by the owner) in this step; published after every stage, so a
    // consumer of chunk c starts on its first sub-tile instead of waiting for the whole chunk
    uint64_t *pack_flag[GR_MAX_RANKS]; // every rank's pack progress [C][N] for this parity
    uint64_t *rs_flag[GR_MAX_RANKS];   // every rank's reduce-scatter progress [C] for this parity
    int32_t *work_counter;             // device, reset by the last CTA
    int32_t *pack_counter;             // device: the PACK queue of queue_mode 1, reset by the last CTA
    int32_t queue_mode;                // 0: triples {PACK, RS, AG} with lags; 1: split PACK / dependent queues
    int32_t lagd;                      // queue_mode 1: all-gather lag in dependent positions
    int32_t *done_counter;
    volatile int32_t *abort_dev;       // device flag: bail out (set on timeout)
    HostError *err;                    // host-mapped
    uint64_t *dbg;                     // optional [CTAs][4] (GR_DEBUG_DUMP): producer state — triple,
                                       // kind<<32|chunk, sub-tile<<32|waiting lanes, progress needed
    uint64_t *trace;                   // optional [items][4]: grab, ready, done, cta|smid<<32, then
                                       // per CTA 8 u64 of stall counters (xfer kernel)
    int32_t trace_items;               // item slots in the trace before the per-CTA counters (= C)
    const int64_t *chunk_begin;        // [C] fusion-buffer element range of each chunk
    const int64_t *chunk_end;          // [C]
    int64_t stage_bytes;               // xfer kernel: bytes of one shared-memory stage
    int32_t nstages;                   // xfer kernel: ring depth (<= 8, nstages*stage_bytes <= 208 KB)
    int64_t slot_bytes_red;            // bytes of one peer's slot inside a stage
    int64_t sub_red, sub_ag, sub_pack; // staged sub-tile (elements) for reduce / all-gather / pack items
    int32_t lag1, lag2;                // queue lags (in work items) of reduce / all-gather items
    int64_t lc_sub;                    // local kernel: elements per warp sub-item (multiple of 8)
    int64_t one_shot_max_bytes;        // N>1: messages up to this many buffer bytes go one-shot
    double *sumsq;                     // optional [T]: sum of squares of the reduced gradient (NEXT-2)
    int32_t *nonfinite;                // optional: set to 1 if any reduced value is Inf/NaN
    int32_t rank, N;
    uint32_t epoch;
    float inv_n;
    uint64_t timeout_ns;
    uint32_t wait_tag;                 // != 0: wait until info->tag == wait_tag before reading the cycle
};

// Armed cycles (one rank per process, W <= GR_BV_INLINE_WORDS, tight cycle loops): a bitvector
// kernel stays resident across cycles, polling the next cycle's descriptor (pinned host memory)
// for a bounded time; a cycle writes its descriptor and rings the doorbell — no kernel launch on
// the cycle's critical path. The kernel takes the static BvParams from its launch and the
// per-cycle fields from the descriptor (one PCIe round trip). skip = 1 retires it.
struct CycleDesc {
    // LL words: (armed kernel's sequence number << 32) | value. Each word validates itself, so
    // the kernel reads the whole cycle in one PCIe round trip; the host writes word D_CTRL last.
    uint64_t w[16 + 2 * GR_BV_INLINE_WORDS];
};
enum DescWord {
    D_CTRL = 0,      // bit 0: skip (retire unused); the doorbell is this word carrying seq
    D_EPOCH = 1, D_TAG = 2, D_HTAG = 3, D_PARITY = 4, D_NEW_STEP = 5, D_CHECK_ASYNC = 6,
    D_ABORT = 7, D_SHUTDOWN = 8, D_SLOT = 9,
    D_BITS = 16,                          // [W] host mark bits
    D_MARKED = 16 + GR_BV_INLINE_WORDS,   // [W] marks taken by the snapshot
};

// Virtual ranks (gr_init_virtual): every rank's parameters for one launch on one device.
// Rank r with bit r of `absent` set never reached the launch (its CTAs exit at once).
struct BvParamsV {
    BvParams r[GR_MAX_RANKS];
    int32_t N;
    uint32_t absent;
};
struct DataParamsV {
    DataParams r[GR_MAX_RANKS];
    int32_t N, per;                    // ranks, CTAs per rank (grid = N * per)
    uint32_t absent;
};

// Kernel launchers (gr_kernels.cu). Return cudaError_t as int.
int launch_bitvector(const BvParams &p, void *stream);
// armed cycles: p's out_released / out_cum / out_subcum / out_info are the ring BASES (slot 0);
// the kernel runs cycle seq, seq+1, ... as the host rings them (descriptor seq % 4), each awaited
// for at most expire_ns, and acknowledges every cycle in *ack
int launch_bitvector_armed(const BvParams &p, const CycleDesc *descs, uint32_t seq, uint64_t expire_ns,
                           uint32_t *ack, void *stream);
int launch_bitvector_virtual(const BvParamsV &pv, void *stream);
int launch_data_virtual(const DataParamsV &pv, int buffer_f16, int stats, void *stream);
int launch_data(const DataParams &p, int local, int buffer_f16, int ctas, void *stream);
int data_kernel_max_ctas(int algo, int buffer_f16, int *out);
int launch_spin(int64_t ns, int ctas, void *stream);

}  // namespace gr
