// gr_runtime.cpp — host runtime behind include/gr.h.
//
// Owns: the response cache (static bit positions, "processed by
// the coordinator rank only once ... stored in a cache on every worker"), the
// static group-major fusion layout and its chunk/segment tables, the
// symmetric memory mapped into every peer with CUDA IPC, the pinned
// host-mapped ready flags / pointer table / result block, the two streams
// (coordination, data), the cycle / step epochs and the error state.
// All arithmetic of the method runs in gr_kernels.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <fstream>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gr.h"
#include "gr_internal.h"
#include "gr_nvls.h"

using gr::Chunk;
using gr::Seg;

namespace {

thread_local std::string g_init_error = "no error";

constexpr int32_t kDefaultTimeoutMs = 20000;
constexpr size_t kAlign = 256;

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

uint64_t fnv1a(uint64_t h, const void *data, size_t n) {
    const unsigned char *p = static_cast<const unsigned char *>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
constexpr int kArmSlots = 4;  // cycle descriptors in flight (armed kernel seq uses slot seq % 4)

constexpr int kPtrStages = 4;  // pinned snapshots of the pointer table in flight (DMA sources)

// Virtual ranks (gr_init_virtual): N contexts of ONE process on ONE device, each an ordinary
// rank of the library (own marks, streams, symmetric memory, epochs), whose peers' memory is
// plain device memory of the same GPU. The two cross-rank kernels of a cycle (bitvector, data)
// must have every rank's CTAs resident at once, so each rank's launch is deposited here and
// the last rank to arrive fires ONE launch covering all ranks (grid = ranks x CTAs) on the
// group's stream; every rank's own stream waits for it. The collective calls (gr_step,
// gr_step_drain) are therefore called concurrently, one thread per virtual rank, as ranks are
// processes in the real deployment. A rank that does not arrive within timeout_ms is launched
// as `absent` (its CTAs exit): its peers then time out on the device exactly as they would on
// a stalled process (GR_ETIMEOUT).
struct VPhase {
    uint64_t gen = 0;              // launches fired so far
    uint32_t arrived = 0;          // ranks deposited for launch `gen`
    gr::BvParams bv[GR_MAX_RANKS];
    gr::DataParams dp[GR_MAX_RANKS];
    cudaEvent_t ev_in[GR_MAX_RANKS] = {};
    cudaEvent_t ev_out[4] = {};    // per generation (mod 4): the fired launch
    int rc[4] = {0, 0, 0, 0};
};
struct VGroup {
    int N = 0, dev = -1, per = 1, buf_f16 = 1, refs = 0;
    int32_t timeout_ms = 20000;
    std::mutex mu;
    std::condition_variable cv;
    cudaStream_t stream[2] = {nullptr, nullptr};  // 0: bitvector launches, 1: data launches
    VPhase ph[2];
};

}  // namespace

struct gr_ctx {
    gr_world world{};
    int32_t T = 0, G = 0, W = 0, nbits = 0, N = 1, rank = 0;
    bool dry = false;
    int buf_f16 = 1;
    int64_t chunk_elems = 0;  // 0 = adaptive per group
    int64_t chunk_target_div = 148, chunk_max = 131072;  // adaptive rule (GR_CHUNK_DIV / GR_CHUNK_MAX)
    int64_t chunk_target_div_fine = 148;                  // fine chunking (N x 148; GR_CHUNK_DIV_FINE)
    int64_t fine_head = 0;                                // leading quarter-size fine chunks (GR_FINE_HEAD)
    int64_t one_shot_max_bytes = 0;
    uint64_t hash = 0;

    // host-side layouts
    std::vector<int64_t> numel;
    std::vector<int32_t> grad_f16, group_of, bit_of, tensor_of_bit, group_of_bit;
    std::vector<int32_t> gbit_begin, gbit_end, gnchunks, gchunk_begin, gnsub, gspc;
    // N > 1: a second, finer chunking of every group (about N x 148 chunks per group), appended
    // after the coarse one; the data kernel takes it for messages with few coarse chunks
    std::vector<int32_t> gnchunks_f, gchunk_begin_f;
    int32_t C_coarse = 0;
    std::vector<int64_t> buf_off, gelems;
    std::vector<int32_t> big_groups;
    std::vector<Seg> segs;
    std::vector<Chunk> chunks;
    std::vector<int64_t> chunk_begin, chunk_end;
    int64_t buf_elems = 0;
    int64_t max_chunk = 0;  // longest chunk of the layout (elements)
    int32_t C = 0;

    // virtual ranks (gr_init_virtual; null for a real rank)
    VGroup *vg = nullptr;
    cudaEvent_t ev_vin[2] = {nullptr, nullptr};

    // device state
    int dev = -1;
    cudaStream_t s_coord = nullptr, s_data = nullptr, s_compute = nullptr;
    cudaEvent_t ev_compute = nullptr, ev_data_done = nullptr, ev_bv = nullptr, ev_released = nullptr, ev_drain = nullptr;
    cudaEvent_t ring_ev[GR_SLOT_RING] = {};
    bool ring_pending[GR_SLOT_RING] = {};
    char *symm = nullptr;
    size_t symm_bytes = 0, off_slot = 0, off_pad = 0, off_buf = 0, pad_parity_u64 = 0;
    size_t buf_parity_bytes = 0;
    size_t off_rsb = 0, rsb_parity_bytes = 0;  // push two-shot receive slots (N-1 buffers per parity)
    bool push = false;                           // GR_PUSH=1: push two-shot (measured slower)
    char *peer_symm[GR_MAX_RANKS] = {};
    Seg *d_segs = nullptr;
    Chunk *d_chunks = nullptr;
    int64_t *d_cbeg = nullptr, *d_cend = nullptr;
    gr::GroupInfo *d_groups = nullptr;
    bool stage_groups = false;  // the group records fit the bitvector kernel's shared memory
    int32_t *d_gcb_f = nullptr, *d_gnc_f = nullptr;
    int32_t *d_gcb = nullptr,
            *d_gspc = nullptr, *d_subcum_ring = nullptr;
    int32_t *d_big = nullptr;
    uint32_t *d_relw = nullptr, *d_hbits_dev = nullptr;
    uint64_t *d_ptr = nullptr;
    int32_t *d_rel_ring = nullptr, *d_cum_ring = nullptr;
    gr::DevCycle *d_info_ring = nullptr;
    int32_t *d_counters = nullptr;  // [0] work, [1] done, [2] abort
    uint64_t *d_dbg = nullptr;      // GR_DEBUG_DUMP: per-CTA producer state of the data kernel
    std::string dbg_path;
    // pinned host-mapped
    uint32_t *h_bits = nullptr;   // sync marks, by bit (live: gr_mark_ready writes, under mu)
    uint32_t *h_marked = nullptr; // every mark (host or stream-ordered), by bit (live, under mu)
    uint32_t *d_flags = nullptr;  // async marks (device memory), by bit
    uint64_t *h_ptr = nullptr;    // gradient pointer table (live, under mu)
    // snapshots taken under mu at gr_step, the DMA sources of the device copies (a queued copy
    // reads its source when it runs, so it must never read the live tables): the mark bits per
    // released-list ring slot ([2W]: host bits, marked bits; W > GR_BV_INLINE_WORDS only) and
    // the pointer table in kPtrStages buffers, each guarded by an event
    uint32_t *h_bits_stage = nullptr;
    uint64_t *h_ptr_stage = nullptr;
    cudaEvent_t ev_ptr_stage[kPtrStages] = {};
    bool ptr_stage_pending[kPtrStages] = {};
    int ptr_stage_next = 0;
    uint64_t *h_hand = nullptr;   // hand-off words written by the bitvector kernel (HandWord)
    gr::HostError *h_err = nullptr;
    uint32_t *d_hbits = nullptr;
    uint64_t *d_hand = nullptr;
    gr::HostError *d_err = nullptr;
    size_t hand_bytes = 0;
    PFN_writeValue32 write_value32 = nullptr;
    // armed cycles (gr_internal.h CycleDesc): in a tight cycle loop the next cycle's bitvector
    // kernel is already running, polling a doorbell in pinned memory, so a cycle launches nothing
    gr::CycleDesc *h_desc = nullptr, *d_desc = nullptr;  // [kArmSlots], pinned + mapped
    uint32_t *h_ack = nullptr, *d_ack = nullptr;         // the armed kernel's acknowledgement
    bool arm_ok = false, armed = false;
    uint32_t arm_seq = 0, arm_first = 0;  // arm_first: the running armed kernel's first cycle
    bool arm_resident = false;            // it has started (h_ack[1] == arm_first)
    int64_t arm_expire_us = 100, arm_gap_us = 50;  // kernel lifetime; arm only after gaps below this
    int64_t arm_ring_delay_us = 0;  // testing (GR_ARM_RING_DELAY_US): host stall after the doorbell
    double last_gap_us = 1e30;                      // host time between the last two gr_step calls
    std::chrono::steady_clock::time_point last_step_exit{}, arm_time{};  // arm_time: the armed kernel
    // polls cycle arm_seq with a deadline no earlier than arm_time + arm_expire_us
    int data_ctas[4] = {0, 0, 0, 0};       // world.comm_ctas (or every SM)
    int data_ctas_full[4] = {0, 0, 0, 0};  // every SM (drain cycles)
    int lag1 = -1, lag2 = -1;  // GR_LAG1 / GR_LAG2 overrides (tuning; -1 = default multiple of the grid)
    int queue_mode = 0, lagd = -1;  // GR_QUEUE (0 triples, 1 split PACK / dependent queues), GR_LAGD
    // TMA stage ring of the xfer kernel: 2 x 96 KB (measured against 4 x 48 / 3 x 64 / 6 x 32 /
    // 8 x 24 KB: per-stage fixed costs make small stages slow — 0.88 vs 0.81 of HBM peak on
    // virtual ranks, 2-5% at N = 2/4, profiles/r02/virtual_chunk_stage_sweep.txt)
    int nstages = 2, stage_kb = 96;  // GR_STAGES / GR_STAGE_KB overrides (tuning)
    int nout = 2, out_kb = 24;       // push: output tiles (GR_OUT_TILES / GR_OUT_KB overrides)
    int64_t pub_quantum = 1ll << 40; // progress publication quantum (elements; GR_PUB_QUANTUM), default: chunk end only
    int32_t fine_below = -1;         // fine chunking below this many coarse chunks (GR_FINE_BELOW; -1: 2 x N x grid)
    int64_t lc_sub = 2048;           // local kernel sub-item (GR_LC_SUB, tuning; measured best)
    std::vector<void *> async_streams;  // distinct streams of this step's gr_mark_ready_async calls

    // step / cycle state
    std::mutex mu;
    std::vector<uint8_t> marked;
    // locally complete groups: a group can be released globally only if every rank marked all
    // its tensors, so when no unreleased group is complete HERE, nothing can be released in
    // this cycle on ANY rank and the data launch is skipped (its kernel would exit at once)
    std::vector<int32_t> grp_size, grp_marked;
    std::vector<uint8_t> grp_released;
    int32_t n_ready_groups = 0;
    uint32_t epoch = 1;
    int64_t cycle = 0, step = 0;
    uint64_t seq = 0;
    bool step_complete = false;
    bool need_compute_fence = false;
    bool step_fresh = true;   // next gr_step is the first cycle of a step
    bool async_used = false;  // gr_mark_ready_async used in this step
    std::atomic<bool> ptr_dirty{false};
    int32_t abort_flag = 0, shutdown_flag = 0;
    int sticky = 0;
    int last_algo = GR_ALGO_NONE;
    std::string err = "no error";

    // NEXT-2 gradient statistics (optional)
    double *d_sumsq = nullptr;
    int32_t *d_nonfinite = nullptr;
    bool stats_on = false;

    // NVLS multicast fusion buffer (optional; see gr_nvls.cpp)
    gr::Nvls nvls;
    std::string nvls_why = "not attempted";

    // tracing (GR_TRACE)
    std::string trace_path;
    uint64_t *d_trace = nullptr;
    size_t trace_slot_u64 = 0;
    struct TraceCycle {
        int64_t cycle, step;
        uint64_t k_start, k_pop, k_and, k_end;
        int64_t h_enter_ns, h_snap_ns, h_bv_ns, h_launched_ns, h_seen_ns, h_done_ns;
        int n_released, algo, nitems, slot;
        int64_t elems;
    };
    std::vector<TraceCycle> trace_cycles;
    int64_t trace_written = 0, trace_max = 16;  // GR_TRACE_MAX_CYCLES

    // stats / timing
    gr_stats stats{};
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending_data_ev, pending_bv_ev, free_ev;
};

namespace {

int fail(gr_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        if (code == GR_ECUDA || code == GR_ETIMEOUT || code == GR_EABORT || code == GR_ESHUTDOWN)
            c->sticky = code;
    } else {
        g_init_error = buf;
    }
    return code;
}

// an error reported by a kernel through the pinned error block (data-kernel timeout, or a
// drain cycle that failed / left the step incomplete)
// GR_DEBUG_DUMP: on a data-kernel timeout, write every CTA's producer state and this rank's
// progress pad (both parities) to <prefix>.rank<r>.json (the kernel bailed out; reads are safe)
void debug_dump(gr_ctx *c) {
    if (!c->d_dbg || c->dbg_path.empty()) return;
    std::vector<uint64_t> st(8 * 1024), pad(2 * c->pad_parity_u64);
    if (cudaMemcpy(st.data(), c->d_dbg, sizeof(uint64_t) * st.size(), cudaMemcpyDeviceToHost) != cudaSuccess) return;
    if (cudaMemcpy(pad.data(), c->symm + c->off_pad, sizeof(uint64_t) * pad.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
        return;
    std::ofstream f(c->dbg_path);
    f << "{\"rank\":" << c->rank << ",\"N\":" << c->N << ",\"C\":" << c->C << ",\"epoch\":" << c->epoch
      << ",\"ctas\":[";
    bool first = true;
    const int nct = std::min(1024, c->data_ctas_full[gr::ALGO_TWOSHOT]);
    for (int i = 0; i < nct; ++i) {
        f << (first ? "" : ",") << "[" << i;
        for (int j = 0; j < 8; ++j) f << "," << st[8 * i + j];
        f << "]";
        first = false;
    }
    f << "],\"pad\":[";
    for (size_t i = 0; i < pad.size(); ++i) f << (i ? "," : "") << pad[i];
    f << "]}\n";
}

int device_error(gr_ctx *c) {
    const int code = c->h_err->code, where = c->h_err->where;
    if (code == 3) debug_dump(c);
    if (code == 3 && where == 3)  // wait_cycle_record: the resident bitvector kernel never wrote the record
        return fail(c, GR_ETIMEOUT, "reduction timed out waiting for its cycle's record (armed bitvector kernel)");
    if (code == 3)
        return fail(c, GR_ETIMEOUT, "reduction timed out waiting for a peer (%s flag)", where == 1 ? "pack" : "reduce-scatter");
    if (code >= 10) {
        const int st = code - 10;
        if (st == gr::ST_ABORT) return fail(c, GR_EABORT, "drain cycle: a rank raised ABORT");
        if (st == gr::ST_SHUTDOWN) return fail(c, GR_ESHUTDOWN, "drain cycle: a rank raised SHUTDOWN");
        if (st == gr::ST_TIMEOUT) return fail(c, GR_ETIMEOUT, "drain cycle: a mark or a peer's bitvector never arrived");
        return fail(c, GR_ETIMEOUT, "drain cycle left the step incomplete (a peer drained before marking everything)");
    }
    return fail(c, GR_ETIMEOUT, "device error %d", code);
}

#define RC(expr)              \
    do {                      \
        int _rc = (expr);     \
        if (_rc) return _rc;  \
    } while (0)

#define CK(c, expr)                                                                          \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess)                                                               \
            return fail((c), GR_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                        __FILE__, __LINE__);                                                 \
    } while (0)

// ---------------------------------------------------------------- layouts (host only)
int build_layouts(gr_ctx *c, const gr_tensor *table, const int32_t *group_of) {
    const int32_t T = c->T, G = c->G;
    c->numel.resize(T);
    c->grad_f16.resize(T);
    c->group_of.assign(group_of, group_of + T);
    std::vector<int32_t> members(G, 0);
    for (int32_t t = 0; t < T; ++t) {
        if (table[t].numel <= 0) return fail(nullptr, GR_EINVAL, "tensor %d: numel must be > 0", t);
        if (table[t].grad_dtype != GR_F32 && table[t].grad_dtype != GR_F16)
            return fail(nullptr, GR_EINVAL, "tensor %d: bad grad dtype", t);
        if (group_of[t] < 0 || group_of[t] >= G)
            return fail(nullptr, GR_EINVAL, "tensor %d: group id %d outside 0..%d", t, group_of[t], G - 1);
        c->numel[t] = table[t].numel;
        c->grad_f16[t] = table[t].grad_dtype == GR_F16;
        members[group_of[t]]++;
    }
    for (int32_t g = 0; g < G; ++g)
        if (!members[g]) return fail(nullptr, GR_EINVAL, "group %d is empty (ids must be dense)", g);

    // response cache: group-major positions (reading R3)
    std::vector<int32_t> order(T);
    for (int32_t t = 0; t < T; ++t) order[t] = t;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return group_of[a] < group_of[b]; });
    c->nbits = GR_STATUS_BITS + T;
    c->W = (c->nbits + 31) / 32;
    {   // the bitvector kernel keeps L, A, released words and the complete-group mask in shared
        // memory (64 KB opt-in): about 131,000 tensors at most; the 24-byte group records join
        // them when they fit (up to 1,024 groups)
        const size_t words = (3 * (size_t)c->W + ((size_t)G + 31) / 32 + 1) & ~(size_t)1;
        const size_t smem = sizeof(uint32_t) * words;
        if (smem > 64 * 1024)
            return fail(nullptr, GR_EINVAL, "%d tensors / %d groups exceed the bitvector kernel's 64 KB "
                        "shared-memory budget (%zu B)", T, G, smem);
        c->stage_groups = G <= 1024 && smem + sizeof(gr::GroupInfo) * (size_t)G <= 64 * 1024;
    }
    c->bit_of.assign(T, 0);
    c->tensor_of_bit.assign((size_t)c->W * 32, -1);
    c->group_of_bit.assign((size_t)c->W * 32, -1);
    c->gbit_begin.assign(G, INT32_MAX);
    c->gbit_end.assign(G, -1);
    for (int32_t pos = 0; pos < T; ++pos) {
        const int32_t t = order[pos], b = GR_STATUS_BITS + pos, g = group_of[t];
        c->bit_of[t] = b;
        c->tensor_of_bit[b] = t;
        c->group_of_bit[b] = g;
        c->gbit_begin[g] = std::min(c->gbit_begin[g], b);
        c->gbit_end[g] = std::max(c->gbit_end[g], b + 1);
    }

    for (int32_t g = 0; g < G; ++g)
        if (((c->gbit_end[g] - 1) >> 5) - (c->gbit_begin[g] >> 5) + 1 > 8) c->big_groups.push_back(g);

    // static fusion layout: same order, every tensor 8-element (16 B at fp16) aligned
    c->buf_off.assign(T, 0);
    c->gelems.assign(G, 0);
    int64_t off = 0;
    std::vector<int64_t> gbeg(G, -1), gend(G, 0);
    for (int32_t pos = 0; pos < T; ++pos) {
        const int32_t t = order[pos], g = group_of[t];
        off = (off + 7) / 8 * 8;
        if (gbeg[g] < 0) gbeg[g] = off;
        c->buf_off[t] = off;
        off += c->numel[t];
        gend[g] = off;
        c->gelems[g] += c->numel[t];
    }
    c->buf_elems = (off + 7) / 8 * 8;
    // progress words carry fusion-buffer element indices in 32 bits (gr_kernels.cu)
    if (c->buf_elems >= (1ll << 32))
        return fail(nullptr, GR_EINVAL, "%lld gradient elements exceed the 2^32 fusion-buffer index range",
                    (long long)c->buf_elems);

    // chunks: cut each group's range at chunk_elems, segments = tensor pieces. Pass 0: the
    // coarse chunking (about one chunk per SM per group, power of two in [8K, 128K] elements:
    // large items, few flags — best when a message holds many chunks, e.g. all of fcn220m).
    // Pass 1 (N > 1, adaptive rule): about N x 148 chunks per group, so a group released alone
    // still gives every rank about one owned reduce-scatter chunk per SM (64 MiB at N=4: 218 vs
    // 268 us, profiles/r02/sw5_n4_queue_shape.txt); the data kernel picks per message.
    c->gchunk_begin.assign(G, 0);
    c->gnchunks.assign(G, 0);
    c->gchunk_begin_f.assign(G, 0);
    c->gnchunks_f.assign(G, 0);
    c->segs.clear();
    c->chunks.clear();
    c->chunk_begin.clear();
    c->chunk_end.clear();
    const int passes = (c->N > 1 && c->chunk_elems == 0) ? 2 : 1;
    for (int pass = 0; pass < passes; ++pass) {
        std::vector<int32_t> &gcb = pass ? c->gchunk_begin_f : c->gchunk_begin;
        std::vector<int32_t> &gnc = pass ? c->gnchunks_f : c->gnchunks;
        const int64_t div = pass ? c->chunk_target_div_fine : c->chunk_target_div;
        int32_t pos = 0;
        for (int32_t g = 0; g < G; ++g) {
            gcb[g] = (int32_t)c->chunks.size();
            const int32_t pos0 = pos;
            while (pos < T && group_of[order[pos]] == g) ++pos;
            int64_t cg = c->chunk_elems;
            if (cg == 0) {
                const int64_t target = std::max<int64_t>(1, (gend[g] - gbeg[g]) / div);
                // fine chunks stay >= 16K elements: 8K ones lost at 8-16 MiB (N = 2 / 4)
                cg = pass ? 16384 : 8192;
                while (cg * 2 <= target && cg < c->chunk_max) cg *= 2;
            }
            // fine chunking: optionally a head of smaller chunks (GR_FINE_HEAD of them, 1/4 size),
            // so the first packs of a group released alone finish early (fill of the pipeline)
            int64_t nsmall = (pass == 1) ? c->fine_head : 0;
            const int64_t csmall = std::max<int64_t>(8192, cg / 4 / 8 * 8);
            for (int64_t cb = gbeg[g]; cb < gend[g];) {
                const int64_t step = (nsmall > 0 && csmall < cg) ? csmall : cg;
                if (nsmall > 0) --nsmall;
                const int64_t ce = std::min(gend[g], cb + step);
                Chunk ch;
                ch.seg_begin = (int32_t)c->segs.size();
                for (int32_t q = pos0; q < pos; ++q) {
                    const int32_t t = order[q];
                    const int64_t tb = c->buf_off[t], te = tb + c->numel[t];
                    const int64_t lo = std::max(tb, cb), hi = std::min(te, ce);
                    if (lo >= hi) continue;
                    Seg sgm;
                    sgm.tensor = t;
                    sgm.grad_f16 = c->grad_f16[t];
                    sgm.tensor_off = lo - tb;
                    sgm.buf_off = lo;
                    sgm.len = hi - lo;
                    c->segs.push_back(sgm);
                }
                ch.seg_end = (int32_t)c->segs.size();
                c->chunks.push_back(ch);
                c->chunk_begin.push_back(cb);
                c->chunk_end.push_back(ce);
                cb = ce;
            }
            gnc[g] = (int32_t)c->chunks.size() - gcb[g];
        }
        if (pass == 0) c->C_coarse = (int32_t)c->chunks.size();
    }
    if (passes == 1) {  // one chunking: the "fine" tables are the coarse ones
        c->gchunk_begin_f = c->gchunk_begin;
        c->gnchunks_f = c->gnchunks;
    }
    c->C = (int32_t)c->chunks.size();
    // local-kernel sub-items (N = 1): lc_sub elements each, spc per full chunk of a group
    c->gnsub.assign(G, 0);
    c->gspc.assign(G, 1);
    for (int32_t g = 0; g < G; ++g) {
        const int32_t c0 = c->gchunk_begin[g], nc = c->gnchunks[g];
        const int64_t full = c->chunk_end[c0] - c->chunk_begin[c0];
        c->gspc[g] = (int32_t)std::max<int64_t>(1, (full + c->lc_sub - 1) / c->lc_sub);
        const int64_t last = c->chunk_end[c0 + nc - 1] - c->chunk_begin[c0 + nc - 1];
        c->gnsub[g] = (nc - 1) * c->gspc[g] + (int32_t)((last + c->lc_sub - 1) / c->lc_sub);
    }
    c->max_chunk = 0;
    for (size_t i = 0; i < c->chunks.size(); ++i)
        c->max_chunk = std::max(c->max_chunk, c->chunk_end[i] - c->chunk_begin[i]);

    // hash of everything that must agree across ranks (PAPER.md:108 global consistency)
    uint64_t h = 1469598103934665603ull;
    h = fnv1a(h, &c->N, sizeof c->N);
    h = fnv1a(h, &c->T, sizeof c->T);
    h = fnv1a(h, &c->G, sizeof c->G);
    h = fnv1a(h, &c->buf_f16, sizeof c->buf_f16);
    h = fnv1a(h, &c->chunk_elems, sizeof c->chunk_elems);
    h = fnv1a(h, &c->one_shot_max_bytes, sizeof c->one_shot_max_bytes);
    h = fnv1a(h, &c->push, sizeof c->push);
    h = fnv1a(h, &c->lag1, sizeof c->lag1);
    h = fnv1a(h, &c->lag2, sizeof c->lag2);
    h = fnv1a(h, &c->fine_below, sizeof c->fine_below);
    h = fnv1a(h, &c->queue_mode, sizeof c->queue_mode);
    h = fnv1a(h, &c->lagd, sizeof c->lagd);
    h = fnv1a(h, &c->world.comm_ctas, sizeof c->world.comm_ctas);  // sets the default lags (x grid)
    h = fnv1a(h, &c->chunk_target_div, sizeof c->chunk_target_div);
    h = fnv1a(h, &c->chunk_target_div_fine, sizeof c->chunk_target_div_fine);
    h = fnv1a(h, &c->fine_head, sizeof c->fine_head);
    h = fnv1a(h, &c->chunk_max, sizeof c->chunk_max);
    h = fnv1a(h, c->numel.data(), sizeof(int64_t) * T);
    h = fnv1a(h, c->grad_f16.data(), sizeof(int32_t) * T);
    h = fnv1a(h, c->group_of.data(), sizeof(int32_t) * T);
    c->hash = h;
    return GR_OK;
}

// the init-time collective (gr_world.allgather); a failed callback leaves c's error text
int allgather_w(const gr_world &w, gr_ctx *c, const void *send, void *recv, size_t bytes) {
    if (w.world_size == 1) {
        memcpy(recv, send, bytes);
        return GR_OK;
    }
    if (!w.allgather) return fail(c, GR_EINVAL, "world.allgather is required when world_size > 1");
    if (w.allgather(send, recv, bytes, w.user) != 0) return fail(c, GR_EINVAL, "allgather callback failed");
    return GR_OK;
}

int allgather(gr_ctx *c, const void *send, void *recv, size_t bytes) {
    return allgather_w(c->world, c, send, recv, bytes);
}

// Init-time agreement: every rank contributes its local status (0 or a gr_status) to one
// allgather, so a rank whose local step failed still takes part in the collective and every
// rank fails together instead of leaving its peers blocked in the next gather.
struct InitVote {
    int32_t rc;
    int32_t pad;
    uint64_t hash;
};

template <typename T>
int upload(gr_ctx *c, T **dst, const std::vector<T> &src) {
    const size_t n = std::max<size_t>(1, src.size()) * sizeof(T);
    CK(c, cudaMalloc((void **)dst, n));
    if (!src.empty()) CK(c, cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    return GR_OK;
}

// Local half of the device setup (no communication): streams, events, symmetric memory,
// device tables, pinned blocks.
int setup_local(gr_ctx *c) {
    CK(c, cudaSetDevice(c->dev));
    CK(c, cudaFree(nullptr));  // make sure the primary context exists
    int lo = 0, hi = 0;
    CK(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(c, cudaStreamCreateWithPriority(&c->s_coord, cudaStreamNonBlocking, hi));
    CK(c, cudaStreamCreateWithPriority(&c->s_data, cudaStreamNonBlocking, hi));
    c->s_compute = (cudaStream_t)c->world.compute_stream;
    CK(c, cudaEventCreateWithFlags(&c->ev_compute, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_data_done, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_released, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_drain, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_bv, cudaEventDisableTiming));
    for (int i = 0; i < GR_SLOT_RING; ++i) CK(c, cudaEventCreateWithFlags(&c->ring_ev[i], cudaEventDisableTiming));
    for (int i = 0; i < kPtrStages; ++i) CK(c, cudaEventCreateWithFlags(&c->ev_ptr_stage[i], cudaEventDisableTiming));
    if (c->vg)
        for (int i = 0; i < 2; ++i) CK(c, cudaEventCreateWithFlags(&c->ev_vin[i], cudaEventDisableTiming));

    // symmetric memory: [LL bitvector slots 2 x W u64][progress pad 2 x (C*N + C) u64][fusion buffer 2 x E]
    const int esz = c->buf_f16 ? 2 : 4;
    c->off_slot = 0;
    c->off_pad = align_up(sizeof(uint64_t) * 2 * (size_t)c->W, kAlign);
    c->pad_parity_u64 = (size_t)c->C * c->N + c->C;
    c->off_buf = align_up(c->off_pad + sizeof(uint64_t) * 2 * c->pad_parity_u64, kAlign);
    c->buf_parity_bytes = (c->N > 1) ? align_up((size_t)c->buf_elems * esz, kAlign) : 0;
    c->off_rsb = c->off_buf + 2 * c->buf_parity_bytes;
    c->rsb_parity_bytes = (c->N > 1 && c->push) ? (size_t)(c->N - 1) * c->buf_parity_bytes : 0;
    c->symm_bytes = c->off_rsb + 2 * c->rsb_parity_bytes;
    cudaError_t e = cudaMalloc((void **)&c->symm, c->symm_bytes);
    if (e != cudaSuccess) return fail(c, GR_ENOMEM, "cudaMalloc(%zu) of symmetric memory: %s", c->symm_bytes, cudaGetErrorString(e));
    CK(c, cudaMemset(c->symm, 0, c->off_buf));

    RC(upload(c, &c->d_segs, c->segs));
    RC(upload(c, &c->d_chunks, c->chunks));
    RC(upload(c, &c->d_cbeg, c->chunk_begin));
    RC(upload(c, &c->d_cend, c->chunk_end));
    {
        std::vector<gr::GroupInfo> gi(c->G);
        for (int32_t g = 0; g < c->G; ++g)
            gi[g] = gr::GroupInfo{c->gbit_begin[g], c->gbit_end[g], c->gnchunks[g], c->gnsub[g], c->gelems[g]};
        RC(upload(c, &c->d_groups, gi));
    }
    RC(upload(c, &c->d_gcb, c->gchunk_begin));
    RC(upload(c, &c->d_gcb_f, c->gchunk_begin_f));
    RC(upload(c, &c->d_gnc_f, c->gnchunks_f));
    RC(upload(c, &c->d_gspc, c->gspc));
    RC(upload(c, &c->d_big, c->big_groups));
    CK(c, cudaMalloc((void **)&c->d_relw, sizeof(uint32_t) * c->W));
    CK(c, cudaMemset(c->d_relw, 0, sizeof(uint32_t) * c->W));
    CK(c, cudaMalloc((void **)&c->d_hbits_dev, sizeof(uint32_t) * 2 * c->W));  // host bits, marked bits
    CK(c, cudaMalloc((void **)&c->d_ptr, sizeof(uint64_t) * c->T));
    CK(c, cudaMemset(c->d_ptr, 0, sizeof(uint64_t) * c->T));
    CK(c, cudaMalloc((void **)&c->d_rel_ring, sizeof(int32_t) * GR_SLOT_RING * (size_t)c->G));
    CK(c, cudaMalloc((void **)&c->d_cum_ring, sizeof(int32_t) * GR_SLOT_RING * (size_t)(c->G + 1)));
    CK(c, cudaMalloc((void **)&c->d_info_ring, sizeof(gr::DevCycle) * GR_SLOT_RING));
    CK(c, cudaMalloc((void **)&c->d_subcum_ring, sizeof(int32_t) * GR_SLOT_RING * (size_t)(c->G + 1)));
    CK(c, cudaMemset(c->d_info_ring, 0, sizeof(gr::DevCycle) * GR_SLOT_RING));
    if (const char *dd = getenv("GR_DEBUG_DUMP")) {
        if (*dd) {
            c->dbg_path = std::string(dd) + ".rank" + std::to_string(c->rank) + ".json";
            CK(c, cudaMalloc((void **)&c->d_dbg, sizeof(uint64_t) * 8 * 1024));
        }
    }
    CK(c, cudaMalloc((void **)&c->d_counters, sizeof(int32_t) * 4));
    CK(c, cudaMemset(c->d_counters, 0, sizeof(int32_t) * 4));

    // pinned host-mapped: ready flags (by bit), pointer table, result block, error block
    const unsigned hf = cudaHostAllocMapped | cudaHostAllocPortable;
    CK(c, cudaHostAlloc((void **)&c->h_bits, sizeof(uint32_t) * (size_t)c->W, hf));
    memset(c->h_bits, 0, sizeof(uint32_t) * (size_t)c->W);
    CK(c, cudaMalloc((void **)&c->d_flags, sizeof(uint32_t) * (size_t)c->W * 32));
    CK(c, cudaMemset(c->d_flags, 0, sizeof(uint32_t) * (size_t)c->W * 32));
    CK(c, cudaHostAlloc((void **)&c->h_ptr, sizeof(uint64_t) * c->T, hf));
    memset(c->h_ptr, 0, sizeof(uint64_t) * c->T);
    CK(c, cudaHostAlloc((void **)&c->h_marked, sizeof(uint32_t) * (size_t)c->W, hf));
    memset(c->h_marked, 0, sizeof(uint32_t) * (size_t)c->W);
    CK(c, cudaHostAlloc((void **)&c->h_ptr_stage, sizeof(uint64_t) * c->T * kPtrStages, hf));
    if (c->W > GR_BV_INLINE_WORDS)
        CK(c, cudaHostAlloc((void **)&c->h_bits_stage, sizeof(uint32_t) * 2 * (size_t)c->W * GR_SLOT_RING, hf));
    c->hand_bytes = sizeof(uint64_t) * gr::hand_words(c->W, c->G);
    CK(c, cudaHostAlloc((void **)&c->h_hand, c->hand_bytes, hf));
    memset((void *)c->h_hand, 0, c->hand_bytes);  // tag 0: never a cycle's tag
    CK(c, cudaHostAlloc((void **)&c->h_err, sizeof(gr::HostError), hf));
    CK(c, cudaHostAlloc((void **)&c->h_desc, sizeof(gr::CycleDesc) * kArmSlots, hf));
    memset((void *)c->h_desc, 0, sizeof(gr::CycleDesc) * kArmSlots);
    CK(c, cudaHostGetDevicePointer((void **)&c->d_desc, (void *)c->h_desc, 0));
    CK(c, cudaHostAlloc((void **)&c->h_ack, 64, hf));
    memset((void *)c->h_ack, 0, 64);
    CK(c, cudaHostGetDevicePointer((void **)&c->d_ack, (void *)c->h_ack, 0));
    memset((void *)c->h_err, 0, sizeof(gr::HostError));
    CK(c, cudaHostGetDevicePointer((void **)&c->d_hbits, c->h_bits, 0));
    CK(c, cudaHostGetDevicePointer((void **)&c->d_hand, (void *)c->h_hand, 0));
    CK(c, cudaHostGetDevicePointer((void **)&c->d_err, (void *)c->h_err, 0));

    // stream memory operations for gr_mark_ready_async
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
        c->write_value32 = (PFN_writeValue32)fn;
    // armed cycles: real ranks with inline bitvectors (GR_ARM=0 turns them off; GR_ARM_US /
    // GR_ARM_GAP_US: the armed kernel's lifetime and the cycle gap below which it is used)
    {
        const char *ae = getenv("GR_ARM");
        c->arm_ok = !c->vg && c->W <= GR_BV_INLINE_WORDS && !(ae && atoi(ae) == 0);
        if (const char *x = getenv("GR_ARM_US")) c->arm_expire_us = std::max<int64_t>(1, atoll(x));
        if (const char *x = getenv("GR_ARM_GAP_US")) c->arm_gap_us = std::max<int64_t>(0, atoll(x));
        if (const char *x = getenv("GR_ARM_RING_DELAY_US")) c->arm_ring_delay_us = std::max<int64_t>(0, atoll(x));
    }

    // 208 KB of dynamic shared memory per CTA: the stage ring, and with push the output tiles
    // (default 4 x 40 KB stages + 2 x 24 KB tiles)
    if (c->push) {
        c->nstages = 4;
        c->stage_kb = 40;
        if (const char *no = getenv("GR_OUT_TILES")) c->nout = std::max(2, std::min(4, atoi(no)));
        if (const char *ok = getenv("GR_OUT_KB")) c->out_kb = std::max(4, atoi(ok) / 4 * 4);
        if (c->nout * c->out_kb > 104) c->out_kb = 104 / c->nout / 4 * 4;
    }
    if (const char *pq = getenv("GR_PUB_QUANTUM")) c->pub_quantum = std::max<int64_t>(256, atoll(pq));
    if (const char *ns = getenv("GR_STAGES")) c->nstages = std::max(2, std::min(8, atoi(ns)));
    if (const char *sk = getenv("GR_STAGE_KB")) c->stage_kb = std::max(8, atoi(sk));
    const int budget = 208 - (c->push ? c->nout * c->out_kb : 0);
    if (c->nstages * c->stage_kb > budget) c->stage_kb = budget / c->nstages / 16 * 16;
    if (const char *tp = getenv("GR_TRACE")) {
        if (*tp) {
            c->trace_path = std::string(tp) + ".rank" + std::to_string(c->rank) + ".jsonl";
            if (const char *tm = getenv("GR_TRACE_MAX_CYCLES")) c->trace_max = atoll(tm);
            c->trace_slot_u64 = (size_t)3 * c->C * 4 + (size_t)1024 * 8;  // items + per-CTA counters
            CK(c, cudaMalloc((void **)&c->d_trace, sizeof(uint64_t) * c->trace_slot_u64 * GR_SLOT_RING));
        }
    }

    // data-kernel grid: every CTA co-resident (bounded by occupancy)
    int sms = 0;
    CK(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->dev));
    for (int algo = gr::ALGO_LOCAL; algo <= gr::ALGO_TWOSHOT; ++algo) {
        // xfer kernel: one CTA per SM (shared-memory stage ring); virtual ranks share the SMs
        int mx = c->vg ? std::max(1, sms / c->N) : sms;
        int rc = algo == gr::ALGO_LOCAL ? gr::data_kernel_max_ctas(algo, c->buf_f16, &mx) : 0;
        if (rc != 0) return fail(c, GR_ECUDA, "occupancy query failed: %s", cudaGetErrorString((cudaError_t)rc));
        int want = c->world.comm_ctas > 0 ? c->world.comm_ctas : mx;
        if (algo == gr::ALGO_LOCAL)
            if (const char *lc = getenv("GR_LOCAL_CTAS")) want = std::max(1, atoi(lc));  // tuning
        c->data_ctas[algo] = std::max(1, std::min(want, mx));
        c->data_ctas_full[algo] = std::max(1, mx);
    }
    CK(c, cudaDeviceSynchronize());
    return GR_OK;
}

// Whole device setup of a real rank: the local half, then the collective half. Every rank
// enters each allgather whatever its local outcome (the status rides along), so a failure on
// one rank fails gr_init on every rank instead of blocking the others.
int setup_device(gr_ctx *c) {
    struct IpcVote {
        int32_t rc, pad;
        cudaIpcMemHandle_t h;
    } mine;
    memset(&mine, 0, sizeof mine);
    mine.rc = setup_local(c);
    if (!mine.rc && c->N > 1) {
        cudaError_t e = cudaIpcGetMemHandle(&mine.h, c->symm);
        if (e != cudaSuccess) mine.rc = fail(c, GR_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    }
    const std::string local_err = c->err;
    // exchange IPC handles; this allgather is also the barrier after zeroing the pads
    std::vector<IpcVote> all(c->N);
    RC(allgather(c, &mine, all.data(), sizeof mine));
    for (int r = 0; r < c->N; ++r)
        if (all[r].rc) {
            if (mine.rc) return fail(c, mine.rc, "%s", local_err.c_str());
            return fail(c, all[r].rc, "gr_init failed on rank %d (code %d)", r, all[r].rc);
        }
    int32_t open_rc = 0;
    for (int r = 0; r < c->N && !open_rc; ++r) {
        if (r == c->rank) {
            c->peer_symm[r] = c->symm;
            continue;
        }
        void *p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, all[r].h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) open_rc = fail(c, GR_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
        else c->peer_symm[r] = (char *)p;
    }

    // NVLS (NEXT-1): in-switch reduction for large messages. It moves S(1+1/N) NVLink bytes per
    // direction against 2S(N-1)/N for two-shot; measured at N = 4 it is slower than two-shot
    // and it has not been measured at N = 8, so it is off unless GR_NVLS=1 asks
    // for it (from N = 2). The vote also carries the peer-mapping status.
    if (c->N > 1) {
        const char *e = getenv("GR_NVLS");
        const bool want = e ? atoi(e) != 0 : false;
        auto ag = [c](const void *snd, void *rcv, size_t n) { return allgather(c, snd, rcv, n); };
        int32_t w[2] = {open_rc, want ? 1 : 0};
        std::vector<int32_t> ws(2 * (size_t)c->N);
        RC(allgather(c, w, ws.data(), sizeof w));
        bool all_want = true;
        for (int r = 0; r < c->N; ++r) {
            if (ws[2 * r]) return open_rc ? open_rc : fail(c, ws[2 * r], "gr_init failed on rank %d (peer mapping)", r);
            all_want = all_want && ws[2 * r + 1];
        }
        if (all_want) {
            if (gr::nvls_setup(c->nvls, c->rank, c->N, c->dev, 2 * c->buf_parity_bytes, ag, c->nvls_why) == 0)
                c->nvls_why = "enabled";
        } else {
            c->nvls_why = "disabled (default off; GR_NVLS=1 enables it)";
        }
    }
    return GR_OK;
}

// ---------------------------------------------------------------- armed cycles
// The per-step static part of a bitvector launch (everything but the per-cycle fields the
// armed kernel reads from its CycleDesc); out_* are the ring bases.
void fill_bv_static(gr_ctx *c, gr::BvParams &p) {
    p.host_bits = c->d_hbits_dev;
    p.marked_bits = c->d_hbits_dev + c->W;
    p.dev_flags = c->d_flags;
    p.groups = c->d_groups;
    p.stage_groups = c->stage_groups ? 1 : 0;
    p.big_groups = c->d_big;
    p.n_big = (int32_t)c->big_groups.size();
    p.rel_words = c->d_relw;
    for (int r = 0; r < c->N; ++r) p.slot[r] = reinterpret_cast<uint64_t *>(c->peer_symm[r] + c->off_slot);
    p.out_released = c->d_rel_ring;
    p.out_cum = c->d_cum_ring;
    p.out_info = c->d_info_ring;
    p.out_subcum = c->d_subcum_ring;
    p.hand = c->d_hand;
    p.T = c->T;
    p.G = c->G;
    p.W = c->W;
    p.nbits = c->nbits;
    p.rank = c->rank;
    p.N = c->N;
    p.timeout_ns = (uint64_t)c->world.timeout_ms * 1000000ull;
    p.use_inline = 1;
    p.drain = 0;
    p.err = c->h_err;
}

static uint32_t next_seq(uint32_t s) { return s + 1 >= 0x7fffffffu ? 1u : s + 1; }  // ack carries seq << 1

// launch a resident bitvector kernel for the coming cycles: it polls each cycle's descriptor for
// at most arm_expire_us. Only in tight cycle loops (the last gap between gr_step calls below
// arm_gap_us): a training loop that ticks every few hundred us never holds an SM for it.
int arm(gr_ctx *c) {
    if (!c->arm_ok || c->armed || c->sticky || c->timing || c->last_gap_us > (double)c->arm_gap_us) return GR_OK;
    c->arm_seq = next_seq(c->arm_seq);
    c->arm_first = c->arm_seq;
    c->arm_resident = false;
    gr::BvParams p{};
    fill_bv_static(c, p);
    c->arm_time = std::chrono::steady_clock::now();  // its lifetime starts no earlier than this
    int lrc = gr::launch_bitvector_armed(p, c->d_desc, c->arm_seq, (uint64_t)c->arm_expire_us * 1000ull, c->d_ack,
                                         c->s_coord);
    if (lrc) return fail(c, GR_ECUDA, "armed bitvector launch: %s", cudaGetErrorString((cudaError_t)lrc));
    c->armed = true;
    return GR_OK;
}

// retire an armed kernel unused (it runs and exits at once); needed before anything waits on
// the coordination stream or enqueues other work in front of the next cycle
void disarm(gr_ctx *c) {
    if (!c->armed) return;
    gr::CycleDesc *h = c->h_desc + c->arm_seq % kArmSlots;
    __atomic_store_n(&h->w[gr::D_CTRL], ((uint64_t)c->arm_seq << 32) | 1ull, __ATOMIC_RELEASE);  // skip
    c->armed = false;
}

void free_all(gr_ctx *c) {
    if (c->dry || c->dev < 0) return;
    cudaSetDevice(c->dev);
    disarm(c);
    if (c->s_coord) cudaStreamSynchronize(c->s_coord);
    if (c->s_data) cudaStreamSynchronize(c->s_data);
    for (int r = 0; r < c->N; ++r)
        if (!c->vg && r != c->rank && c->peer_symm[r]) cudaIpcCloseMemHandle(c->peer_symm[r]);
    gr::nvls_free(c->nvls);
    cudaFree(c->symm);
    void *dptrs[] = {c->d_segs, c->d_chunks, c->d_cbeg, c->d_cend, c->d_groups, c->d_gcb, c->d_gcb_f, c->d_gnc_f,
                     c->d_big, c->d_relw, c->d_hbits_dev, c->d_ptr, c->d_rel_ring, c->d_cum_ring, c->d_info_ring, c->d_counters, c->d_dbg, c->d_gspc, c->d_subcum_ring,
                     c->d_flags, c->d_trace, c->d_sumsq, c->d_nonfinite};
    for (void *p : dptrs) cudaFree(p);
    cudaFreeHost(c->h_bits);
    cudaFreeHost(c->h_marked);
    cudaFreeHost(c->h_ptr);
    cudaFreeHost(c->h_ptr_stage);
    cudaFreeHost(c->h_bits_stage);
    for (int i = 0; i < kPtrStages; ++i)
        if (c->ev_ptr_stage[i]) cudaEventDestroy(c->ev_ptr_stage[i]);
    for (int i = 0; i < 2; ++i)
        if (c->ev_vin[i]) cudaEventDestroy(c->ev_vin[i]);
    cudaFreeHost((void *)c->h_hand);
    cudaFreeHost((void *)c->h_err);
    cudaFreeHost((void *)c->h_desc);
    cudaFreeHost((void *)c->h_ack);
    for (int i = 0; i < GR_SLOT_RING; ++i)
        if (c->ring_ev[i]) cudaEventDestroy(c->ring_ev[i]);
    if (c->ev_compute) cudaEventDestroy(c->ev_compute);
    if (c->ev_data_done) cudaEventDestroy(c->ev_data_done);
    if (c->ev_released) cudaEventDestroy(c->ev_released);
    if (c->ev_drain) cudaEventDestroy(c->ev_drain);
    if (c->ev_bv) cudaEventDestroy(c->ev_bv);
    for (auto &v : {c->pending_data_ev, c->pending_bv_ev, c->free_ev})
        for (auto &pr : v) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
    if (c->s_coord) cudaStreamDestroy(c->s_coord);
    if (c->s_data) cudaStreamDestroy(c->s_data);
    if (VGroup *g = c->vg) {  // the last virtual rank frees the group
        c->vg = nullptr;
        bool last;
        {
            std::lock_guard<std::mutex> lk(g->mu);
            last = --g->refs == 0;
        }
        if (last) {
            for (auto &s : g->stream)
                if (s) {
                    cudaStreamSynchronize(s);
                    cudaStreamDestroy(s);
                }
            for (auto &ph : g->ph)
                for (auto &e : ph.ev_out)
                    if (e) cudaEventDestroy(e);
            delete g;
        }
    }
}

// ---------------------------------------------------------------- virtual-rank launches
// Deposit this rank's launch of `phase` (0 bitvector, 1 data) and take part in firing it; on
// return `own` (the rank's stream) is ordered after the combined launch.
int vg_launch(gr_ctx *c, int phase, cudaStream_t own, const gr::BvParams *bv, const gr::DataParams *dp) {
    VGroup &g = *c->vg;
    VPhase &ph = g.ph[phase];
    CK(c, cudaEventRecord(c->ev_vin[phase], own));  // this rank's work before the launch
    std::unique_lock<std::mutex> lk(g.mu);
    const uint64_t my = ph.gen;
    const uint32_t all = (1u << g.N) - 1u;
    if (bv) ph.bv[c->rank] = *bv;
    else ph.dp[c->rank] = *dp;
    ph.ev_in[c->rank] = c->ev_vin[phase];
    ph.arrived |= 1u << c->rank;
    if (ph.arrived != all)
        g.cv.wait_until(lk, std::chrono::steady_clock::now() + std::chrono::milliseconds(g.timeout_ms),
                        [&] { return ph.gen != my; });
    if (ph.gen == my) {  // last to arrive, or the others are late: fire with whoever is here
        const int k = (int)(my & 3);
        cudaStream_t s = g.stream[phase];
        int rc = 0;
        for (int r = 0; r < g.N && !rc; ++r)
            if ((ph.arrived >> r) & 1u) rc = (int)cudaStreamWaitEvent(s, ph.ev_in[r], 0);
        if (!rc) {
            if (phase == 0) {
                gr::BvParamsV pv{};
                pv.N = g.N;
                pv.absent = all & ~ph.arrived;
                for (int r = 0; r < g.N; ++r)
                    if ((ph.arrived >> r) & 1u) pv.r[r] = ph.bv[r];
                rc = gr::launch_bitvector_virtual(pv, s);
            } else {
                gr::DataParamsV pv{};
                pv.N = g.N;
                pv.per = g.per;
                pv.absent = all & ~ph.arrived;
                int stats = 0;
                for (int r = 0; r < g.N; ++r)
                    if ((ph.arrived >> r) & 1u) {
                        pv.r[r] = ph.dp[r];
                        stats |= ph.dp[r].sumsq != nullptr;
                    }
                rc = gr::launch_data_virtual(pv, g.buf_f16, stats, s);
            }
        }
        if (!rc) rc = (int)cudaEventRecord(ph.ev_out[k], s);
        ph.rc[k] = rc;
        ph.gen++;
        ph.arrived = 0;
        g.cv.notify_all();
    }
    const int k = (int)(my & 3);
    const int rc = ph.rc[k];
    cudaEvent_t ev = ph.ev_out[k];
    lk.unlock();
    if (rc) return fail(c, GR_ECUDA, "virtual-rank %s launch: %s", phase ? "data" : "bitvector",
                        cudaGetErrorString((cudaError_t)rc));
    // ev_out[k] is re-recorded only 4 launches later, which needs this rank again (or 4 timeouts)
    CK(c, cudaStreamWaitEvent(own, ev, 0));
    return GR_OK;
}

std::pair<cudaEvent_t, cudaEvent_t> get_ev_pair(gr_ctx *c) {
    if (!c->free_ev.empty()) {
        auto pr = c->free_ev.back();
        c->free_ev.pop_back();
        return pr;
    }
    std::pair<cudaEvent_t, cudaEvent_t> pr;
    cudaEventCreate(&pr.first);
    cudaEventCreate(&pr.second);
    return pr;
}

int collect_timing(gr_ctx *c) {
    for (auto *v : {&c->pending_data_ev, &c->pending_bv_ev}) {
        for (auto &pr : *v) {
            float ms = 0.f;
            CK(c, cudaEventSynchronize(pr.second));
            CK(c, cudaEventElapsedTime(&ms, pr.first, pr.second));
            if (v == &c->pending_data_ev) c->stats.data_kernel_ms += ms;
            else c->stats.bitvector_kernel_ms += ms;
            c->free_ev.push_back(pr);
        }
        v->clear();
    }
    return GR_OK;
}

}  // namespace

extern "C" {

// Local half of gr_init: validate the arguments and build the host-side layouts (no
// communication). On error *out is null and g_init_error holds the text.
static int create_ctx(gr_ctx **out, const gr_world *world, const gr_tensor *table, int32_t T,
                      const int32_t *group_of, int32_t G) {
    *out = nullptr;
    if (!table || !group_of) return fail(nullptr, GR_EINVAL, "null argument to gr_init");
    if (T <= 0 || G <= 0 || G > T) return fail(nullptr, GR_EINVAL, "need 0 < G <= T (T=%d, G=%d)", T, G);
    if (world->rank < 0 || world->rank >= world->world_size) return fail(nullptr, GR_EINVAL, "bad rank");
    if (world->buffer_dtype != GR_F16 && world->buffer_dtype != GR_F32)
        return fail(nullptr, GR_EINVAL, "bad buffer dtype");
    if (world->chunk_elems < 0 || world->chunk_elems % 8)
        return fail(nullptr, GR_EINVAL, "chunk_elems must be a non-negative multiple of 8");
    gr_ctx *c = new (std::nothrow) gr_ctx();
    if (!c) return fail(nullptr, GR_ENOMEM, "out of host memory");
    c->world = *world;
    c->T = T;
    c->G = G;
    c->N = world->world_size;
    c->rank = world->rank;
    c->buf_f16 = world->buffer_dtype == GR_F16;
    c->chunk_elems = world->chunk_elems;  // 0: adaptive per group (build_layouts)
    if (const char *ls = getenv("GR_LC_SUB")) c->lc_sub = std::max<int64_t>(256, atoll(ls) / 8 * 8);  // tuning
    if (const char *pu = getenv("GR_PUSH")) c->push = atoi(pu) != 0;  // tuning / comparison
    // adaptive chunk rules (build_layouts): coarse ~148 chunks per group, fine ~N x 148
    c->chunk_target_div_fine = 148 * (int64_t)std::max(1, world->world_size);
    if (const char *cd = getenv("GR_CHUNK_DIV")) c->chunk_target_div = std::max<int64_t>(1, atoll(cd));  // tuning
    if (const char *cf = getenv("GR_CHUNK_DIV_FINE")) c->chunk_target_div_fine = std::max<int64_t>(1, atoll(cf));
    if (const char *fh = getenv("GR_FINE_HEAD")) c->fine_head = std::max<int64_t>(0, atoll(fh));
    if (const char *cm = getenv("GR_CHUNK_MAX")) c->chunk_max = std::max<int64_t>(8192, atoll(cm));      // tuning
    if (world->chunk_elems == 0)
        if (const char *ce = getenv("GR_CHUNK_ELEMS")) c->chunk_elems = std::max<int64_t>(8, atoll(ce) / 8 * 8);  // tuning
    // default one-shot threshold: one-shot (every rank reads all N-1 peer copies) has the
    // fewest synchronisations; two-shot moves 2(N-1)/N of the message per direction and less
    // local HBM traffic. Crossover measured with tools/bench_cfg5.py (profiles/r01_cfg):
    // N=2 between 128 and 256 MiB, N=4 at ~8 MiB; N>=8 reads 7 peer copies, kept at 1 MiB.
    {
        // (round 2, N=4: two-shot 64.7 vs one-shot 69.3 us at 8 MiB, equal at 4 MiB: threshold 4 MiB)
        const int64_t thr = c->N <= 2 ? (128ll << 20) : c->N == 3 ? (32ll << 20) : c->N == 4 ? (4ll << 20) : (1ll << 20);
        c->one_shot_max_bytes = world->one_shot_max_bytes >= 0 ? world->one_shot_max_bytes : thr;
    }
    // knobs that fix the cross-rank queue order / algorithm: read before the table hash so every
    // rank must agree on them (a mismatch would desynchronise the fused kernel's queues)
    if (const char *os = getenv("GR_ONESHOT_MAX_BYTES")) c->one_shot_max_bytes = atoll(os);  // tuning
    if (const char *l1 = getenv("GR_LAG1")) c->lag1 = std::max(0, atoi(l1));
    if (const char *l2 = getenv("GR_LAG2")) c->lag2 = std::max(0, atoi(l2));
    // the queue is deadlock-free only with every reduce-scatter queued before the all-gathers
    // that wait for it (0 <= L1 < L2, tests/test_queue_model.py)
    if (c->lag1 >= 0 && c->lag2 >= 0 && c->lag2 <= c->lag1) {
        delete c;
        return fail(nullptr, GR_EINVAL, "GR_LAG2 (%s) must exceed GR_LAG1 (%s)", getenv("GR_LAG2"), getenv("GR_LAG1"));
    }
    if (const char *fb = getenv("GR_FINE_BELOW")) c->fine_below = std::max(0, atoi(fb));
    if (const char *qm = getenv("GR_QUEUE")) c->queue_mode = atoi(qm) == 1 ? 1 : 0;
    if (const char *ld = getenv("GR_LAGD")) c->lagd = std::max(1, atoi(ld));
    c->dry = world->device < 0;
    if (c->world.timeout_ms <= 0) c->world.timeout_ms = kDefaultTimeoutMs;
    int rc = build_layouts(c, table, group_of);
    if (rc) {
        delete c;
        return rc;
    }
    c->marked.assign(T, 0);
    c->grp_size.assign(G, 0);
    for (int32_t t = 0; t < T; ++t) c->grp_size[group_of[t]]++;
    c->grp_marked.assign(G, 0);
    c->grp_released.assign(G, 0);
    c->dev = c->dry ? -1 : world->device;
    *out = c;
    return GR_OK;
}

int gr_init(gr_ctx **out, const gr_world *world, const gr_tensor *table, int32_t T, const int32_t *group_of,
            int32_t G) {
    if (!out || !world) return fail(nullptr, GR_EINVAL, "null argument to gr_init");
    *out = nullptr;
    if (world->world_size < 1 || world->world_size > GR_MAX_RANKS)
        return fail(nullptr, GR_EINVAL, "world_size must be in 1..%d", GR_MAX_RANKS);
    gr_ctx *c = nullptr;
    const int local_rc = create_ctx(&c, world, table, T, group_of, G);
    const std::string local_err = g_init_error;
    // global consistency check: every rank must have built the same cache. A rank
    // whose arguments were rejected still takes part (its status rides along), so every rank
    // returns instead of leaving the others blocked in the gather.
    InitVote mine{local_rc, 0, c ? c->hash : 0};
    std::vector<InitVote> votes(world->world_size);
    gr_ctx tmp;
    tmp.world = *world;
    int rc = allgather_w(*world, &tmp, &mine, votes.data(), sizeof mine);
    if (rc) {
        delete c;
        return fail(nullptr, rc, "%s", tmp.err.c_str());
    }
    for (int r = 0; r < world->world_size; ++r)
        if (votes[r].rc) {
            delete c;
            if (local_rc) return fail(nullptr, local_rc, "%s", local_err.c_str());
            return fail(nullptr, votes[r].rc, "gr_init failed on rank %d (code %d)", r, votes[r].rc);
        }
    for (int r = 0; r < world->world_size; ++r)
        if (votes[r].hash != c->hash) {
            fail(nullptr, GR_EMISMATCH, "rank %d's tensor table / groups / config differ from rank %d's", r, c->rank);
            delete c;
            return GR_EMISMATCH;
        }
    if (!c->dry) {
        rc = setup_device(c);
        if (rc) {
            g_init_error = c->err;
            free_all(c);
            delete c;
            return rc;
        }
    }
    *out = c;
    return GR_OK;
}

int gr_init_virtual(gr_ctx **out, const gr_world *world, const gr_tensor *table, int32_t T,
                    const int32_t *group_of, int32_t G) {
    if (!out || !world) return fail(nullptr, GR_EINVAL, "null argument to gr_init_virtual");
    const int N = world->world_size;
    if (N < 2 || N > GR_MAX_RANKS) return fail(nullptr, GR_EINVAL, "virtual world_size must be in 2..%d", GR_MAX_RANKS);
    for (int r = 0; r < N; ++r) out[r] = nullptr;
    if (world->device < 0) return fail(nullptr, GR_EINVAL, "virtual ranks need a device");
    VGroup *g = new (std::nothrow) VGroup();
    if (!g) return fail(nullptr, GR_ENOMEM, "out of host memory");
    g->N = N;
    g->dev = world->device;
    g->buf_f16 = world->buffer_dtype == GR_F16;
    g->timeout_ms = world->timeout_ms > 0 ? world->timeout_ms : kDefaultTimeoutMs;
    auto undo = [&](int rc) {
        std::string e = g_init_error;
        bool any = false;
        for (int r = 0; r < N; ++r)
            if (out[r]) {
                any = true;
                if (out[r]->err != "no error") e = out[r]->err;
                gr_finalize(out[r]);  // drops a group reference
                out[r] = nullptr;
            }
        if (!any) delete g;
        return fail(nullptr, rc, "%s", e.c_str());
    };
    for (int r = 0; r < N; ++r) {
        gr_world w = *world;
        w.rank = r;
        w.allgather = nullptr;  // the ranks live in this process: nothing to gather
        gr_ctx *c = nullptr;
        int rc = create_ctx(&c, &w, table, T, group_of, G);
        if (rc) return undo(rc);
        c->vg = g;
        g->refs++;
        out[r] = c;
        rc = setup_local(c);
        if (rc) return undo(rc);
        c->nvls_why = "disabled (virtual ranks share one device)";
    }
    for (int r = 0; r < N; ++r)
        for (int q = 0; q < N; ++q) out[r]->peer_symm[q] = out[q]->symm;
    g->per = out[0]->data_ctas[gr::ALGO_TWOSHOT];
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return undo(GR_ECUDA);
    for (auto &s : g->stream)
        if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi) != cudaSuccess) return undo(GR_ECUDA);
    for (auto &ph : g->ph)
        for (auto &e : ph.ev_out)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return undo(GR_ECUDA);
    return GR_OK;
}

static int mark_common(gr_ctx *c, int32_t rank, int32_t t, void *dev_ptr) {
    if (!c) return GR_EINVAL;
    if (c->dry) return fail(c, GR_ESTATE, "dry context (device < 0) cannot mark");
    if (c->sticky) return fail(c, GR_ESTATE, "context is in a sticky error state (%d)", c->sticky);
    if (rank != c->rank) return fail(c, GR_EINVAL, "rank %d != world.rank %d", rank, c->rank);
    if (t < 0 || t >= c->T) return fail(c, GR_EINVAL, "tensor id %d out of range", t);
    if (!dev_ptr) return fail(c, GR_EINVAL, "null dev_ptr for tensor %d", t);
    if (c->step_complete) return fail(c, GR_ESTATE, "step complete: call gr_wait before marking again");
    if (c->marked[t]) return fail(c, GR_ESTATE, "tensor %d already marked in this step", t);
    c->marked[t] = 1;
    if (++c->grp_marked[c->group_of[t]] == c->grp_size[c->group_of[t]]) c->n_ready_groups++;
    if (c->h_ptr[t] != (uint64_t)(uintptr_t)dev_ptr) {  // pointer first, then the flag
        c->h_ptr[t] = (uint64_t)(uintptr_t)dev_ptr;
        c->ptr_dirty = true;                            // re-upload only when it changed
    }
    // the cycle's snapshot (step_impl, under mu) takes this bit together with the pointer
    // table, so a tensor is seen by a cycle only if its pointer travels with that cycle
    const int32_t b = c->bit_of[t];
    c->h_marked[b >> 5] |= 1u << (b & 31);
    return GR_OK;
}

int gr_mark_ready(gr_ctx *c, int32_t rank, int32_t t, void *dev_ptr) {
    if (!c) return GR_EINVAL;
    std::lock_guard<std::mutex> lk(c->mu);
    int rc = mark_common(c, rank, t, dev_ptr);
    if (rc) return rc;
    c->need_compute_fence = true;
    const int32_t b = c->bit_of[t];
    c->h_bits[b >> 5] |= 1u << (b & 31);
    return GR_OK;
}

int gr_mark_ready_batch(gr_ctx *c, int32_t rank, int32_t n, const int32_t *ids, void *const *ptrs) {
    if (!c) return GR_EINVAL;
    if (n < 0 || (n > 0 && (!ids || !ptrs))) return fail(c, GR_EINVAL, "bad batch");
    std::lock_guard<std::mutex> lk(c->mu);
    for (int32_t i = 0; i < n; ++i) {  // validate everything first: all-or-nothing
        const int32_t t = ids[i];
        if (c->dry) return fail(c, GR_ESTATE, "dry context (device < 0) cannot mark");
        if (c->sticky) return fail(c, GR_ESTATE, "context is in a sticky error state (%d)", c->sticky);
        if (rank != c->rank) return fail(c, GR_EINVAL, "rank %d != world.rank %d", rank, c->rank);
        if (t < 0 || t >= c->T) return fail(c, GR_EINVAL, "tensor id %d out of range", t);
        if (!ptrs[i]) return fail(c, GR_EINVAL, "null dev_ptr for tensor %d", t);
        if (c->step_complete) return fail(c, GR_ESTATE, "step complete: call gr_wait before marking again");
        if (c->marked[t]) return fail(c, GR_ESTATE, "tensor %d already marked in this step", t);
        for (int32_t j = 0; j < i; ++j)
            if (ids[j] == t) return fail(c, GR_ESTATE, "tensor %d twice in one batch", t);
    }
    for (int32_t i = 0; i < n; ++i) {
        int rc = mark_common(c, rank, ids[i], ptrs[i]);
        if (rc) return rc;
        const int32_t b = c->bit_of[ids[i]];
        c->h_bits[b >> 5] |= 1u << (b & 31);
    }
    if (n > 0) c->need_compute_fence = true;
    return GR_OK;
}

int gr_mark_ready_async(gr_ctx *c, int32_t rank, int32_t t, void *dev_ptr, void *stream) {
    if (!c) return GR_EINVAL;
    std::lock_guard<std::mutex> lk(c->mu);
    if (!c->dry && !c->write_value32) return fail(c, GR_ECUDA, "cuStreamWriteValue32 unavailable");
    int rc = mark_common(c, rank, t, dev_ptr);
    if (rc) return rc;
    c->async_used = true;
    if (std::find(c->async_streams.begin(), c->async_streams.end(), stream) == c->async_streams.end())
        c->async_streams.push_back(stream);
    CUresult r = c->write_value32((CUstream)stream, (CUdeviceptr)(c->d_flags + c->bit_of[t]), c->epoch, 0);
    if (r != CUDA_SUCCESS) {
        c->marked[t] = 0;
        if (c->grp_marked[c->group_of[t]]-- == c->grp_size[c->group_of[t]]) c->n_ready_groups--;
        const int32_t b = c->bit_of[t];
        c->h_marked[b >> 5] &= ~(1u << (b & 31));
        return fail(c, GR_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
    }
    return GR_OK;
}

int gr_set_status(gr_ctx *c, int32_t abort_flag, int32_t shutdown_flag) {
    if (!c) return GR_EINVAL;
    std::lock_guard<std::mutex> lk(c->mu);
    c->abort_flag = abort_flag != 0;
    c->shutdown_flag = shutdown_flag != 0;
    return GR_OK;
}

static int step_impl(gr_ctx *c, int32_t *released, gr_cycle_info *info, uint32_t *global_bits, bool drain);

int gr_step(gr_ctx *c, int32_t *released, gr_cycle_info *info, uint32_t *global_bits) {
    if (!c || !released) return fail(c, GR_EINVAL, "null argument to gr_step");
    return step_impl(c, released, info, global_bits, false);
}

int gr_step_drain(gr_ctx *c) {
    if (!c) return GR_EINVAL;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        for (int32_t t = 0; t < c->T; ++t)
            if (!c->marked[t]) return fail(c, GR_ESTATE, "gr_step_drain: tensor %d is not marked in this step", t);
    }
    return step_impl(c, nullptr, nullptr, nullptr, true);
}

static int step_impl(gr_ctx *c, int32_t *released, gr_cycle_info *info, uint32_t *global_bits, bool drain) {
    if (c->dry) return fail(c, GR_ESTATE, "dry context (device < 0) cannot step");
    if (c->sticky) return fail(c, GR_ESTATE, "context is in a sticky error state (%d): %s", c->sticky, c->err.c_str());
    const auto h_enter = std::chrono::steady_clock::now();
    if (c->last_step_exit.time_since_epoch().count())
        c->last_gap_us = std::chrono::duration<double, std::micro>(h_enter - c->last_step_exit).count();
    if (c->h_err->code) return device_error(c);
    CK(c, cudaSetDevice(c->dev));
    const int slot = (int)(c->cycle % GR_SLOT_RING);
    if (c->ring_pending[slot]) {  // the data launch that read this slot must be done
        CK(c, cudaEventSynchronize(c->ring_ev[slot]));
        c->ring_pending[slot] = false;
    }
    uint32_t epoch;
    int32_t abort_flag, shutdown_flag;
    bool p_inline = c->W <= GR_BV_INLINE_WORDS, step_fresh = false, async_used = false;
    gr::BvParams p{};
    // armed cycle: the kernel is already queued; drains, timing and fallbacks retire it first
    const bool use_armed = c->armed && !drain && !c->timing && p_inline;
    if (!use_armed) disarm(c);
    gr::CycleDesc *hd = use_armed ? c->h_desc + c->arm_seq % kArmSlots : nullptr;
    // the pointer-table snapshot buffer this cycle may use (its previous upload has long run)
    const int pk = c->ptr_stage_next;
    if (c->ptr_stage_pending[pk]) {
        CK(c, cudaEventSynchronize(c->ev_ptr_stage[pk]));
        c->ptr_stage_pending[pk] = false;
    }
    bool ptr_upload = false, skip_data = false;
    uint32_t *bits_stage = p_inline ? nullptr : c->h_bits_stage + (size_t)slot * 2 * c->W;
    {
        // ONE critical section takes everything a concurrent gr_mark_ready could change: the
        // compute-stream fence, the mark bits and the pointer table. A mark that lands after it
        // belongs to the next cycle, consistently for the fence, the bits and the pointer.
        std::lock_guard<std::mutex> lk(c->mu);
        if (c->step_complete) return fail(c, GR_ESTATE, "step complete: call gr_wait first");
        // virtual ranks fire one data launch over all ranks, so they never skip it
        skip_data = !drain && !c->vg && c->n_ready_groups == 0;
        if (c->need_compute_fence && !skip_data) {  // order the data stream after the marked gradients' producers
            CK(c, cudaEventRecord(c->ev_compute, c->s_compute));
            CK(c, cudaStreamWaitEvent(c->s_data, c->ev_compute, 0));
            c->need_compute_fence = false;
        }
        epoch = c->epoch;
        step_fresh = c->step_fresh;
        c->step_fresh = false;
        async_used = c->async_used;
        if (hd) {        // ... in the armed kernel's pinned descriptor (LL words, this seq)
            const uint64_t sq = (uint64_t)c->arm_seq << 32;
            for (int w = 0; w < c->W; ++w) {
                hd->w[gr::D_BITS + w] = sq | c->h_bits[w];
                hd->w[gr::D_MARKED + w] = sq | c->h_marked[w];
                p.inline_bits[w] = c->h_bits[w];      // kept for a fallback launch
                p.inline_marked[w] = c->h_marked[w];
            }
        } else if (p_inline) {  // the mark bits travel in the launch parameters
            memcpy(p.inline_bits, c->h_bits, sizeof(uint32_t) * c->W);
            memcpy(p.inline_marked, c->h_marked, sizeof(uint32_t) * c->W);
        } else {         // ... or in this ring slot's pinned snapshot, DMA'd before the kernel
            memcpy(bits_stage, c->h_bits, sizeof(uint32_t) * c->W);
            memcpy(bits_stage + c->W, c->h_marked, sizeof(uint32_t) * c->W);
        }
        if (c->ptr_dirty && !skip_data) {
            memcpy(c->h_ptr_stage + (size_t)pk * c->T, c->h_ptr, sizeof(uint64_t) * c->T);
            c->ptr_dirty = false;
            ptr_upload = true;
        }
        abort_flag = c->abort_flag;
        shutdown_flag = c->shutdown_flag;
    }

    const auto h_snap = std::chrono::steady_clock::now();
    p.host_bits = c->d_hbits_dev;
    p.marked_bits = c->d_hbits_dev + c->W;
    p.dev_flags = c->d_flags;
    p.new_step = step_fresh;
    p.check_async = async_used;
    p.groups = c->d_groups;
    p.stage_groups = c->stage_groups ? 1 : 0;
    p.big_groups = c->d_big;
    p.n_big = (int32_t)c->big_groups.size();
    p.rel_words = c->d_relw;
    for (int r = 0; r < c->N; ++r) p.slot[r] = reinterpret_cast<uint64_t *>(c->peer_symm[r] + c->off_slot);
    p.out_released = c->d_rel_ring + (size_t)slot * c->G;
    p.out_cum = c->d_cum_ring + (size_t)slot * (c->G + 1);
    p.out_info = c->d_info_ring + slot;
    p.out_subcum = c->d_subcum_ring + (size_t)slot * (c->G + 1);
    p.hand = c->d_hand;
    p.T = c->T;
    p.G = c->G;
    p.W = c->W;
    p.nbits = c->nbits;
    p.rank = c->rank;
    p.N = c->N;
    p.epoch = epoch;
    p.tag = (uint32_t)(c->cycle + 1);
    if (p.tag == 0) p.tag = 1;
    p.parity = (int32_t)(c->cycle & 1);
    p.abort_flag = abort_flag;
    p.shutdown_flag = shutdown_flag;
    p.timeout_ns = (uint64_t)c->world.timeout_ms * 1000000ull;
    if ((uint32_t)++c->seq == 0) ++c->seq;  // the hand-off tag is the low 32 bits, never 0
    p.htag = (uint32_t)c->seq;
    p.use_inline = p_inline;
    p.drain = drain ? 1 : 0;
    p.err = c->h_err;

    std::pair<cudaEvent_t, cudaEvent_t> evb{};
    if (c->timing) {
        evb = get_ev_pair(c);
        CK(c, cudaEventRecord(evb.first, c->s_coord));
    }
    if (drain) {
        // the drain kernel must not sit on an SM for the rest of backward (it would displace
        // compute, e.g. a persistent GEMM's last CTA): the coordination stream itself waits,
        // in the stream front end, for every stream that issued stream-ordered marks
        std::vector<void *> streams;
        {
            std::lock_guard<std::mutex> lk(c->mu);
            streams = c->async_streams;
        }
        for (void *ms : streams) {
            CK(c, cudaEventRecord(c->ev_drain, static_cast<cudaStream_t>(ms)));
            CK(c, cudaStreamWaitEvent(c->s_coord, c->ev_drain, 0));
        }
    }
    if (!p_inline)  // larger bitvectors: one DMA of the cycle's snapshot, stream-ordered before the kernel
        CK(c, cudaMemcpyAsync(c->d_hbits_dev, bits_stage, sizeof(uint32_t) * 2 * c->W, cudaMemcpyHostToDevice,
                              c->s_coord));
    bool ran_armed = false;
    if (hd) {  // ring the armed kernel: the data words first, the control word last (x86 keeps store order)
        const uint64_t sq = (uint64_t)c->arm_seq << 32;
        hd->w[gr::D_EPOCH] = sq | p.epoch;
        hd->w[gr::D_TAG] = sq | p.tag;
        hd->w[gr::D_HTAG] = sq | p.htag;
        hd->w[gr::D_PARITY] = sq | (uint32_t)p.parity;
        hd->w[gr::D_NEW_STEP] = sq | (uint32_t)p.new_step;
        hd->w[gr::D_CHECK_ASYNC] = sq | (uint32_t)p.check_async;
        hd->w[gr::D_ABORT] = sq | (uint32_t)p.abort_flag;
        hd->w[gr::D_SHUTDOWN] = sq | (uint32_t)p.shutdown_flag;
        hd->w[gr::D_SLOT] = sq | (uint32_t)slot;
        // taken before the doorbell: the kernel's wait for the next cycle starts after it sees
        // this one, so its deadline is no earlier than t_ring + arm_expire_us (host preemption
        // between the doorbell and a later timestamp must not stretch the host's estimate)
        const auto t_ring = std::chrono::steady_clock::now();
        __atomic_store_n(&hd->w[gr::D_CTRL], sq, __ATOMIC_RELEASE);
        if (c->arm_ring_delay_us)  // a preempted host: the kernel may run this cycle and expire on the next first
            std::this_thread::sleep_for(std::chrono::microseconds(c->arm_ring_delay_us));
        // rung well inside the kernel's lifetime for this cycle (which starts after its launch, or
        // after the previous cycle was rung): it cannot have expired, go on. Otherwise its
        // acknowledgement tells: accepted, or expired before the doorbell (then this cycle is
        // launched as usual and a new kernel armed after it).
        const auto t0 = std::chrono::steady_clock::now();
        const double since = std::chrono::duration<double, std::micro>(t0 - c->arm_time).count();
        uint32_t a = 1u;
        bool gone_after = false;  // accepted, and it has since expired waiting for the next cycle
        if (since > (double)c->arm_expire_us * 0.8 - 10.0) {
            // the ack word holds the kernel's latest decision: (seq << 1) | accepted. It can be
            // past this cycle already (accepted it, ran it, then expired on the next one).
            const uint32_t s0 = c->arm_seq, s1 = next_seq(s0);
            for (;;) {
                a = __atomic_load_n(c->h_ack, __ATOMIC_ACQUIRE);
                if ((a >> 1) == s0) break;
                if ((a >> 1) == s1) {
                    a = 1u;
                    gone_after = true;
                    break;
                }
                if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(c->world.timeout_ms + 5000))
                    return fail(c, GR_ETIMEOUT, "armed bitvector kernel never acknowledged");
            }
            c->arm_resident = true;
        }
        if ((a & 1u) && !c->arm_resident && c->N == 1) {
            // the data kernel below spins until this cycle's record carries its tag: that is only
            // safe with the bitvector kernel already on an SM (it started, so it stays resident),
            // never with it queued behind SMs the spinning data CTAs could occupy
            while (__atomic_load_n(c->h_ack + 1, __ATOMIC_ACQUIRE) != c->arm_first) {
                if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(c->world.timeout_ms + 5000))
                    return fail(c, GR_ETIMEOUT, "armed bitvector kernel never started");
            }
            c->arm_resident = true;
        }
        if (a & 1u) {  // accepted: the same kernel then waits for the next cycle
            ran_armed = true;
            c->stats.armed_cycles++;
            c->arm_seq = next_seq(c->arm_seq);
            c->arm_time = t_ring;
            if (gone_after || c->N > 1) c->armed = false;  // arm() below queues a new one (N > 1: one cycle each)
        } else {           // expired: the cycle's marks are in p.inline_* for the launch below
            c->armed = false;
            c->stats.armed_expired++;
        }
    }
    if (ran_armed) {
    } else if (c->vg) {
        RC(vg_launch(c, 0, c->s_coord, &p, nullptr));
    } else {
        int lrc = gr::launch_bitvector(p, c->s_coord);
        if (lrc) return fail(c, GR_ECUDA, "bitvector launch: %s", cudaGetErrorString((cudaError_t)lrc));
    }
    if (c->timing) {
        CK(c, cudaEventRecord(evb.second, c->s_coord));
        c->pending_bv_ev.push_back(evb);
    }
    c->stats.bitvector_launches++;
    const auto h_bv = std::chrono::steady_clock::now();

    // Data kernel, launched now (before the host sees the cycle's result): it waits on the
    // bitvector kernel through an event and reads the released set from device memory, so
    // the reduction starts the moment the bitvector kernel ends. Empty cycles exit at once;
    // cycles that cannot release anything (no locally complete group) do not launch it.
    if (skip_data) {
        c->stats.data_launches_skipped++;
        if (!p_inline) {  // the slot's pinned mark snapshot is reused GR_SLOT_RING cycles later:
            CK(c, cudaEventRecord(c->ring_ev[slot], c->s_coord));  // its DMA must have run by then
            c->ring_pending[slot] = true;
        }
    } else {
        gr::DataParams d{};
        d.segs = c->d_segs;
        d.chunks = c->d_chunks;
        d.group_chunk_begin = c->d_gcb;
        d.released = p.out_released;
        d.cum = p.out_cum;
        d.info = p.out_info;
        d.subcum = p.out_subcum;
        d.group_spc = c->d_gspc;
        d.dev_ptr = c->d_ptr;
        const int par = (int)(epoch & 1);
        d.nvls_uc = c->nvls.enabled ? reinterpret_cast<char *>(c->nvls.ucva) + (size_t)par * c->buf_parity_bytes : nullptr;
        d.nvls_mc = c->nvls.enabled ? reinterpret_cast<char *>(c->nvls.mcva) + (size_t)par * c->buf_parity_bytes : nullptr;
        for (int r = 0; r < c->N; ++r) {
            char *base = c->peer_symm[r];
            d.buf[r] = base + c->off_buf + (size_t)par * c->buf_parity_bytes;
            d.rsb[r] = c->push ? base + c->off_rsb + (size_t)par * c->rsb_parity_bytes : nullptr;
            uint64_t *pad = reinterpret_cast<uint64_t *>(base + c->off_pad) + (size_t)par * c->pad_parity_u64;
            d.pack_flag[r] = pad;
            d.rs_flag[r] = pad + (size_t)c->C * c->N;
        }
        d.dbg = c->d_dbg;
        if (c->d_dbg) CK(c, cudaMemsetAsync(c->d_dbg, 0, sizeof(uint64_t) * 8 * 1024, c->s_data));
        d.work_counter = c->d_counters;
        d.done_counter = c->d_counters + 1;
        d.pack_counter = c->d_counters + 3;
        d.queue_mode = c->queue_mode;
        d.abort_dev = c->d_counters + 2;
        d.err = c->d_err;
        d.trace = c->d_trace ? c->d_trace + (size_t)slot * c->trace_slot_u64 : nullptr;
        d.trace_items = c->C * 4;  // u64 offset / 3 of the counters: counters start at 3*C*4
        d.chunk_begin = c->d_cbeg;
        d.chunk_end = c->d_cend;
        const int64_t es = c->buf_f16 ? 2 : 4;
        const int64_t stage = c->stage_kb * 1024;
        d.stage_bytes = stage;
        d.nstages = c->nstages;
        // RED/RS stage: N-1 peer slots (buffer precision) + one fp32-spaced gradient slot
        int64_t sr = c->N > 1 ? stage / ((c->N - 1) * es + 4) / 256 * 256 : 256;
        const int64_t cmax = c->chunk_elems > 0 ? c->chunk_elems : c->chunk_max;
        sr = std::max<int64_t>(256, std::min<int64_t>(sr, cmax));
        d.sub_red = sr;
        d.slot_bytes_red = sr * es;
        int64_t spk = stage / 4 / 256 * 256;  // fp32 gradients staged
        if (c->push) spk = std::min<int64_t>(spk, (int64_t)c->out_kb * 1024 / es / 256 * 256);  // one output tile
        d.sub_pack = std::max<int64_t>(256, std::min<int64_t>(spk, cmax));
        d.out_bytes = (int64_t)c->out_kb * 1024;
        d.pub_quantum = c->pub_quantum;
        d.group_chunk_begin_fine = c->d_gcb_f;
        d.group_nchunks_fine = c->d_gnc_f;
        d.nout = c->nout;
        d.sub_ag = std::max<int64_t>(256, std::min<int64_t>(stage / es / 256 * 256, cmax));
        d.one_shot_max_bytes = c->one_shot_max_bytes;
        d.push = c->push ? 1 : 0;
        d.rsb_stride = (int64_t)c->buf_parity_bytes;
        d.rank = c->rank;
        d.N = c->N;
        d.epoch = epoch;
        d.inv_n = 1.0f / (float)c->N;
        d.timeout_ns = (uint64_t)c->world.timeout_ms * 1000000ull;
        const bool local = c->N == 1;
        // a drain cycle's reduction starts when backward is over: it gets every SM
        const int ctas = drain ? c->data_ctas_full[local ? gr::ALGO_LOCAL : gr::ALGO_TWOSHOT]
                               : c->data_ctas[local ? gr::ALGO_LOCAL : gr::ALGO_TWOSHOT];
        d.lc_sub = c->lc_sub;
        d.fine_below = c->fine_below >= 0 ? c->fine_below : 2 * c->N * ctas;
        // queue lags (3/8 x grid measured 3-4% faster than 2/4 x grid at N=2,4)
        d.lag1 = c->lag1 >= 0 ? c->lag1 : 3 * ctas;
        d.lag2 = c->lag2 >= 0 ? c->lag2 : 8 * ctas;
        if (d.lag2 <= d.lag1) d.lag2 = d.lag1 + ctas;  // one override against the other's default
        d.lagd = c->lagd >= 0 ? c->lagd : 2 * ctas;
        if (ran_armed && c->N == 1) {  // the bitvector kernel stays resident: the data kernel waits for its tag
            d.wait_tag = p.htag;
        } else {
            d.wait_tag = 0;
            CK(c, cudaEventRecord(c->ev_bv, c->s_coord));
            CK(c, cudaStreamWaitEvent(c->s_data, c->ev_bv, 0));
        }
        std::pair<cudaEvent_t, cudaEvent_t> evd{};
        if (c->timing) {
            evd = get_ev_pair(c);
            CK(c, cudaEventRecord(evd.first, c->s_data));
        }
        if (ptr_upload) {  // gradient pointers changed since the last upload: this cycle's snapshot
            CK(c, cudaMemcpyAsync(c->d_ptr, c->h_ptr_stage + (size_t)pk * c->T, sizeof(uint64_t) * c->T,
                                  cudaMemcpyHostToDevice, c->s_data));
            CK(c, cudaEventRecord(c->ev_ptr_stage[pk], c->s_data));
            c->ptr_stage_pending[pk] = true;
            c->ptr_stage_next = (pk + 1) % kPtrStages;
        }
        if (d.trace) CK(c, cudaMemsetAsync(d.trace, 0, sizeof(uint64_t) * c->trace_slot_u64, c->s_data));
        if (c->stats_on) {
            d.sumsq = c->d_sumsq;
            d.nonfinite = c->d_nonfinite;
            if (step_fresh) {  // statistics restart with the step
                CK(c, cudaMemsetAsync(c->d_sumsq, 0, sizeof(double) * c->T, c->s_data));
                CK(c, cudaMemsetAsync(c->d_nonfinite, 0, sizeof(int32_t), c->s_data));
            }
        }
        if (c->vg) {
            RC(vg_launch(c, 1, c->s_data, nullptr, &d));
        } else {
            int lrc = gr::launch_data(d, local, c->buf_f16, ctas, c->s_data);
            if (lrc) return fail(c, GR_ECUDA, "data launch: %s", cudaGetErrorString((cudaError_t)lrc));
        }
        if (c->timing) {
            CK(c, cudaEventRecord(evd.second, c->s_data));
            c->pending_data_ev.push_back(evd);
        }
        CK(c, cudaEventRecord(c->ring_ev[slot], c->s_data));
        c->ring_pending[slot] = true;
        c->stats.data_launches++;
    }

    // queue the next cycle's kernel now, while this one's runs (its launch cost overlaps the wait)
    if (!drain) RC(arm(c));

    if (drain) {  // device-driven final cycle: the host does not wait for the hand-off
        c->last_step_exit = std::chrono::steady_clock::now();
        c->cycle++;
        c->stats.cycles++;
        std::lock_guard<std::mutex> lk(c->mu);
        c->step_complete = true;
        return GR_OK;
    }

    // wait for the kernel's hand-off (pinned host memory, LL words tagged with this cycle), bounded
    const auto t0 = std::chrono::steady_clock::now();
    const auto h_launched = t0;
    const auto limit = std::chrono::milliseconds(c->world.timeout_ms + 5000);
    const uint64_t *H = c->h_hand;
    auto word_ready = [&](int i) { return (uint32_t)(__atomic_load_n(H + i, __ATOMIC_ACQUIRE) >> 32) == p.htag; };
    auto word = [&](int i) { return (uint32_t)__atomic_load_n(H + i, __ATOMIC_RELAXED); };
    uint64_t spins = 0;
    int need = gr::HW_A + c->W;  // header + A; then the released list once n is known
    for (int i = 0; i < need;) {
        if (word_ready(i)) {
            if (i == gr::HW_NREL) need += (int)std::min<uint32_t>(word(gr::HW_NREL), (uint32_t)c->G);
            ++i;
            continue;
        }
        if ((++spins & 1023) == 0) {
            cudaError_t q = cudaStreamQuery(c->s_coord);
            if (q != cudaSuccess && q != cudaErrorNotReady)
                return fail(c, GR_ECUDA, "bitvector kernel failed: %s", cudaGetErrorString(q));
            if (std::chrono::steady_clock::now() - t0 > limit)
                return fail(c, GR_ETIMEOUT, "bitvector kernel did not report within %d ms", c->world.timeout_ms + 5000);
            if (spins > (1u << 20)) std::this_thread::yield();
        }
    }
    const auto h_seen = std::chrono::steady_clock::now();
    auto word64 = [&](int i) { return (uint64_t)word(i) | ((uint64_t)word(i + 1) << 32); };
    const uint64_t k_start = word64(gr::HW_STAMPS), k_pop = word64(gr::HW_STAMPS + 2),
                   k_and = word64(gr::HW_STAMPS + 4), k_end = word64(gr::HW_STAMPS + 6);
    c->stats.host_wait_us += std::chrono::duration<double, std::micro>(h_seen - t0).count();
    c->stats.bitvector_device_us += (double)(k_end - k_start) * 1e-3;
    const int status = (int)word(gr::HW_STATUS);
    if (global_bits)
        for (int w = 0; w < c->W; ++w) global_bits[w] = word(gr::HW_A + w);
    const int64_t this_cycle = c->cycle++;
    c->stats.cycles++;
    if (status == gr::ST_TIMEOUT) return fail(c, GR_ETIMEOUT, "cycle %lld: a peer did not publish its bitvector", (long long)this_cycle);
    if (status == gr::ST_ABORT) return fail(c, GR_EABORT, "cycle %lld: a rank raised ABORT", (long long)this_cycle);
    if (status == gr::ST_SHUTDOWN) return fail(c, GR_ESHUTDOWN, "cycle %lld: a rank raised SHUTDOWN", (long long)this_cycle);
    const int n = (int)word(gr::HW_NREL);
    const int total_chunks = (int)word(gr::HW_CHUNKS);
    const int64_t rel_elems = (int64_t)word64(gr::HW_ELEMS);
    for (int i = 0; i < n; ++i) released[i] = (int32_t)word(gr::HW_A + c->W + i);
    if (n > 0) {
        std::lock_guard<std::mutex> lk(c->mu);
        for (int i = 0; i < n; ++i) {
            const int32_t g = released[i];
            if (g >= 0 && g < c->G && !c->grp_released[g]) {
                c->grp_released[g] = 1;
                c->n_ready_groups--;  // released groups were complete on every rank, this one too
            }
        }
    }

    if (n > 0) {
        const int64_t msg_bytes = rel_elems * (c->buf_f16 ? 2 : 4);
        c->last_algo = c->N == 1 ? gr::ALGO_LOCAL
                                 : (msg_bytes <= c->one_shot_max_bytes
                                        ? gr::ALGO_ONESHOT
                                        : (c->nvls.enabled ? gr::ALGO_NVLS : gr::ALGO_TWOSHOT));
        c->stats.released_elems += rel_elems;
    }
    const int complete = (int)word(gr::HW_COMPLETE);
    const auto h_done = std::chrono::steady_clock::now();
    c->stats.host_step_us += std::chrono::duration<double, std::micro>(h_done - h_enter).count();
    if (!c->trace_path.empty() && c->trace_written < c->trace_max) {
        ++c->trace_written;
        auto ns = [](std::chrono::steady_clock::time_point t) {
            return (int64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t.time_since_epoch()).count();
        };
        gr_ctx::TraceCycle tc{};
        tc.cycle = this_cycle;
        tc.step = c->step;
        tc.k_start = k_start;
        tc.k_pop = k_pop;
        tc.k_and = k_and;
        tc.k_end = k_end;
        tc.h_enter_ns = ns(h_enter);
        tc.h_snap_ns = ns(h_snap);
        tc.h_bv_ns = ns(h_bv);
        tc.h_launched_ns = ns(h_launched);
        tc.h_seen_ns = ns(h_seen);
        tc.h_done_ns = ns(h_done);
        tc.n_released = n;
        tc.algo = n > 0 ? c->last_algo : 0;
        // N > 1: phase p's items sit at [p*C, p*C + items) (C = every chunk of both chunkings)
        tc.nitems = n > 0 ? (c->last_algo == gr::ALGO_LOCAL ? total_chunks : 3 * c->C) : 0;
        tc.slot = slot;
        tc.elems = rel_elems;
        c->trace_cycles.push_back(tc);
    }
    {
        std::lock_guard<std::mutex> lk(c->mu);
        if (complete) c->step_complete = true;
    }
    c->last_step_exit = std::chrono::steady_clock::now();
    if (info) {
        info->n_released = n;
        info->step_complete = complete;
        info->cycle = this_cycle;
        info->step = c->step;
        info->released_elems = rel_elems;
    }
    return GR_OK;
}

static int start_next_step(gr_ctx *c) {
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->step_complete) {
        c->step_complete = false;
        c->epoch++;
        if (c->epoch == 0) c->epoch = 1;
        c->step++;
        c->stats.steps++;
        std::fill(c->marked.begin(), c->marked.end(), 0);
        std::fill(c->grp_marked.begin(), c->grp_marked.end(), 0);
        std::fill(c->grp_released.begin(), c->grp_released.end(), 0);
        c->n_ready_groups = 0;
        // the live tables only: every cycle's kernel reads its own snapshot
        memset(c->h_bits, 0, sizeof(uint32_t) * (size_t)c->W);
        memset(c->h_marked, 0, sizeof(uint32_t) * (size_t)c->W);
        c->step_fresh = true;
        c->async_used = false;
        c->async_streams.clear();
    }
    return GR_OK;
}

int gr_wait_async(gr_ctx *c) {
    if (!c) return GR_EINVAL;
    if (!c->trace_path.empty()) return gr_wait(c);
    if (c->dry) return fail(c, GR_ESTATE, "dry context (device < 0) cannot wait");
    if (c->sticky == GR_ECUDA) return fail(c, GR_ESTATE, "context is in a sticky error state: %s", c->err.c_str());
    if (c->h_err->code) return device_error(c);
    CK(c, cudaSetDevice(c->dev));
    CK(c, cudaEventRecord(c->ev_data_done, c->s_data));
    CK(c, cudaStreamWaitEvent(c->s_compute, c->ev_data_done, 0));
    return start_next_step(c);
}

int gr_released_wait_async(gr_ctx *c, void *stream) {
    if (!c) return GR_EINVAL;
    if (c->dry) return fail(c, GR_ESTATE, "dry context (device < 0) cannot wait");
    if (c->sticky == GR_ECUDA) return fail(c, GR_ESTATE, "context is in a sticky error state: %s", c->err.c_str());
    CK(c, cudaSetDevice(c->dev));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : c->s_compute;
    CK(c, cudaEventRecord(c->ev_released, c->s_data));  // data kernels are serialized on s_data
    CK(c, cudaStreamWaitEvent(s, c->ev_released, 0));
    return GR_OK;
}

int gr_wait(gr_ctx *c) {
    if (!c) return GR_EINVAL;
    if (c->dry) return fail(c, GR_ESTATE, "dry context (device < 0) cannot wait");
    if (c->sticky == GR_ECUDA) return fail(c, GR_ESTATE, "context is in a sticky error state: %s", c->err.c_str());
    CK(c, cudaSetDevice(c->dev));
    disarm(c);  // a queued armed kernel would hold the coordination stream forever
    CK(c, cudaStreamSynchronize(c->s_coord));
    CK(c, cudaStreamSynchronize(c->s_data));
    if (c->h_err->code) return device_error(c);
    CK(c, cudaEventRecord(c->ev_data_done, c->s_data));
    CK(c, cudaStreamWaitEvent(c->s_compute, c->ev_data_done, 0));
    for (int i = 0; i < GR_SLOT_RING; ++i) c->ring_pending[i] = false;
    if (c->timing) {
        int rc = collect_timing(c);
        if (rc) return rc;
    }
    if (!c->trace_path.empty() && !c->trace_cycles.empty()) {
        std::ofstream f(c->trace_path, std::ios::app);
        std::vector<uint64_t> buf;
        for (const auto &tc : c->trace_cycles) {
            f << "{\"cycle\":" << tc.cycle << ",\"step\":" << tc.step << ",\"rank\":" << c->rank
              << ",\"N\":" << c->N << ",\"k\":[" << tc.k_start << "," << tc.k_pop << "," << tc.k_and << ","
              << tc.k_end << "],\"h\":[" << tc.h_enter_ns << "," << tc.h_snap_ns << "," << tc.h_bv_ns << ","
              << tc.h_launched_ns << "," << tc.h_seen_ns
              << "," << tc.h_done_ns << "],\"n_released\":" << tc.n_released << ",\"algo\":" << tc.algo
              << ",\"elems\":" << tc.elems << ",\"nitems\":" << tc.nitems << ",\"items\":[";
            if (tc.nitems > 0) {
                buf.resize((size_t)tc.nitems * 4);
                CK(c, cudaMemcpy(buf.data(), c->d_trace + (size_t)tc.slot * c->trace_slot_u64,
                                 sizeof(uint64_t) * buf.size(), cudaMemcpyDeviceToHost));
                bool first = true;
                for (int i = 0; i < tc.nitems; ++i) {
                    if (!buf[4 * i + 2]) continue;  // not executed on this rank
                    if (!first) f << ",";
                    first = false;
                    f << "[" << i << "," << buf[4 * i] << "," << buf[4 * i + 1] << "," << buf[4 * i + 2] << ","
                      << buf[4 * i + 3] << "]";
                }
            }
            f << "]";
            if (tc.nitems > 0 && c->N > 1) {  // xfer kernel per-CTA stall counters (clock64 cycles)
                const int nct = c->data_ctas[gr::ALGO_TWOSHOT];
                std::vector<uint64_t> pr((size_t)nct * 8);
                CK(c, cudaMemcpy(pr.data(), c->d_trace + (size_t)tc.slot * c->trace_slot_u64 + (size_t)3 * c->C * 4,
                                 sizeof(uint64_t) * pr.size(), cudaMemcpyDeviceToHost));
                f << ",\"prof\":[";
                for (int i = 0; i < nct; ++i) {
                    if (i) f << ",";
                    f << "[" << pr[8 * i] << "," << pr[8 * i + 1] << "," << pr[8 * i + 2] << "," << pr[8 * i + 3]
                      << "," << pr[8 * i + 4] << "," << pr[8 * i + 5] << "]";
                }
                f << "]";
            }
            f << "}\n";
        }
        c->trace_cycles.clear();
    }
    return start_next_step(c);
}

int gr_finalize(gr_ctx *c) {
    if (!c) return GR_OK;
    free_all(c);
    delete c;
    return GR_OK;
}

const char *gr_last_error(gr_ctx *c) { return c ? c->err.c_str() : g_init_error.c_str(); }

int gr_query(gr_ctx *c, int32_t kind, void *out, size_t bytes) {
    if (!c || !out) return GR_EINVAL;
    auto put = [&](const void *src, size_t n) -> int {
        if (bytes < n) return fail(c, GR_EINVAL, "gr_query: need %zu bytes, got %zu", n, bytes);
        memcpy(out, src, n);
        return GR_OK;
    };
    switch (kind) {
        case GR_Q_WORDS: return put(&c->W, sizeof(int32_t));
        case GR_Q_BIT_OF: return put(c->bit_of.data(), sizeof(int32_t) * c->T);
        case GR_Q_BUF_OFFSET: return put(c->buf_off.data(), sizeof(int64_t) * c->T);
        case GR_Q_NCHUNKS: return put(&c->C, sizeof(int32_t));
        case GR_Q_STATS: return put(&c->stats, sizeof(gr_stats));
        case GR_Q_LAST_ALGO: return put(&c->last_algo, sizeof(int32_t));
        case GR_Q_NVLS: {
            const int32_t v = c->nvls.enabled ? 1 : 0;
            return put(&v, sizeof v);
        }
        case GR_Q_NVLS_WHY: {  // NUL-terminated, truncated to `bytes`
            if (bytes == 0) return fail(c, GR_EINVAL, "gr_query: zero-size buffer");
            const size_t n = std::min(bytes - 1, c->nvls_why.size());
            memcpy(out, c->nvls_why.data(), n);
            static_cast<char *>(out)[n] = 0;
            return GR_OK;
        }
        default: return fail(c, GR_EINVAL, "unknown query %d", kind);
    }
}

int gr_enable_grad_stats(gr_ctx *c, int32_t on) {
    if (!c) return GR_EINVAL;
    if (c->dry) return fail(c, GR_ESTATE, "dry context (device < 0) has no statistics");
    if (on && !c->d_sumsq) {
        CK(c, cudaSetDevice(c->dev));
        CK(c, cudaMalloc((void **)&c->d_sumsq, sizeof(double) * c->T));
        CK(c, cudaMalloc((void **)&c->d_nonfinite, sizeof(int32_t)));
        CK(c, cudaMemset(c->d_sumsq, 0, sizeof(double) * c->T));
        CK(c, cudaMemset(c->d_nonfinite, 0, sizeof(int32_t)));
    }
    c->stats_on = on != 0;
    return GR_OK;
}

int gr_grad_stats(gr_ctx *c, double *sumsq_host, int32_t *nonfinite_host, void **sumsq_dev, void **nonfinite_dev) {
    if (!c) return GR_EINVAL;
    if (!c->stats_on || !c->d_sumsq) return fail(c, GR_ESTATE, "gradient statistics are not enabled");
    if (sumsq_dev) *sumsq_dev = c->d_sumsq;
    if (nonfinite_dev) *nonfinite_dev = c->d_nonfinite;
    if (sumsq_host || nonfinite_host) {
        CK(c, cudaSetDevice(c->dev));
        CK(c, cudaStreamSynchronize(c->s_data));
        if (sumsq_host) CK(c, cudaMemcpy(sumsq_host, c->d_sumsq, sizeof(double) * c->T, cudaMemcpyDeviceToHost));
        if (nonfinite_host) CK(c, cudaMemcpy(nonfinite_host, c->d_nonfinite, sizeof(int32_t), cudaMemcpyDeviceToHost));
    }
    return GR_OK;
}

int gr_set_timing(gr_ctx *c, int32_t on) {
    if (!c) return GR_EINVAL;
    c->timing = on != 0;
    return GR_OK;
}

int gr_reset_stats(gr_ctx *c) {
    if (!c) return GR_EINVAL;
    c->stats = gr_stats{};
    return GR_OK;
}

int gr_bench_spin(int64_t ns, int32_t ctas, void *stream) {
    if (ns < 0 || ctas <= 0) return GR_EINVAL;
    return gr::launch_spin(ns, ctas, stream) ? GR_ECUDA : GR_OK;
}

}  // extern "C"
