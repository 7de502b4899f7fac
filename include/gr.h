/*
 * gr.h — C ABI of the B200-native grouped gradient reduction library (libgr.so).
 *
 * Implements the data-parallel hot path of arXiv 1909.11150 ("Exascale Deep
 * Learning for Scientific Inverse Problems"): per coordination cycle every
 * rank populates a readiness bitvector over its gradient tensors
 * (§4.1 step 1), the bitvectors are intersected with a bitwise
 * AND across ranks (step 2 — "Bitvector Allreduce"), set bits
 * are decoded in cache-bit order (Fig.3b), and the
 * Grouping rule releases a group only when all its members are globally
 * ready, fusing all complete groups of the cycle into one message
 * (§4.2). Released groups are packed into a fusion buffer
 * (PAPER.md:135), sum-allreduced, scaled by 1/N and unpacked into the
 * per-tensor gradients in place.
 *
 * One process per GPU. Every call below runs its arithmetic in hand-written
 * sm_100a kernels (paper_1909_11150_b200/csrc/); the cross-rank exchange uses
 * direct NVLink/NVSwitch peer loads and stores on CUDA-IPC-mapped memory.
 * There is no CPU fallback: without a usable device the calls fail with
 * GR_ECUDA.
 *
 * Conventions. All functions return a gr_status (0 = GR_OK, negative =
 * error) and never throw across the ABI; gr_last_error(ctx) gives the text of
 * the most recent error. Pointers are plain host or device addresses as
 * stated per argument. Tensor id t is the index of the tensor in the table
 * given to gr_init. Bit b of a bitvector lives in u32 word b>>5 at LSB-first
 * position b&31. Bits 0 and 1 are status bits (bit0 = "no rank aborted",
 * bit1 = "no rank is shutting down": complement-coded so that the one AND
 * also ORs the flags — DESIGN.md reading R1); tensor t owns bit 2 + pos(t),
 * pos(t) = index of t when tensors are sorted by (group id, tensor id)
 * (reading R3). W = ceil((T + 2) / 32).
 */
#ifndef GR_H
#define GR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GR_OK = 0,
    GR_EINVAL = -1,     /* bad argument: null pointer, bad id, numel <= 0, groups not dense/non-empty */
    GR_ESTATE = -2,     /* call not allowed now: duplicate mark in a step, mark after the step
                           completed and before gr_wait, any call after a sticky error */
    GR_EMISMATCH = -3,  /* table / groups / dtypes / world size differ across ranks (init) */
    GR_ECUDA = -4,      /* CUDA runtime or driver error (sticky) */
    GR_ETIMEOUT = -5,   /* a peer did not reach the same cycle/chunk within timeout_ms (sticky) */
    GR_EABORT = -6,     /* some rank raised ABORT (status bit 0) in this cycle (sticky) */
    GR_ESHUTDOWN = -7,  /* some rank raised SHUTDOWN (status bit 1) in this cycle (sticky) */
    GR_ENOMEM = -8      /* device or pinned-host allocation failed */
} gr_status;

typedef enum { GR_F32 = 0, GR_F16 = 1 } gr_dtype;

/* Collective bootstrap callback (used only inside gr_init): gather
 * bytes_per_rank bytes from every rank into recv (rank-major, world_size *
 * bytes_per_rank bytes, host memory). Must return 0 on success. The Python
 * binding implements it with torch.distributed. */
typedef int (*gr_allgather_fn)(const void *send, void *recv, size_t bytes_per_rank, void *user);

typedef struct {
    int32_t rank;               /* this process's rank, 0 <= rank < world_size */
    int32_t world_size;         /* N >= 1 (one process per GPU, N <= 8 in one NVSwitch domain) */
    int32_t device;             /* CUDA device ordinal this rank drives */
    void *compute_stream;       /* cudaStream_t (borrowed) on which gradients are produced;
                                   NULL = legacy default stream */
    gr_dtype buffer_dtype;      /* fusion-buffer (wire) precision: GR_F16 or GR_F32 */
    int64_t one_shot_max_bytes; /* messages up to this many buffer bytes use the one-shot
                                   reduce, larger ones the two-shot (or NVLS); -1 = library
                                   default: 128 MiB at N=2, 32 MiB at N=3, 4 MiB at N=4,
                                   1 MiB above (measured crossovers) */
    int32_t timeout_ms;         /* bound on any cross-rank wait; 0 = 20000 */
    int32_t comm_ctas;          /* CTAs of the fused reduce kernel; 0 = library default */
    int64_t chunk_elems;        /* fusion-buffer chunk (pipelining) granularity in elements,
                                   multiple of 8; 0 = adaptive per group (about one chunk per
                                   SM, a power of two between 8K and 128K elements) */
    gr_allgather_fn allgather;  /* required when world_size > 1 */
    void *user;                 /* passed to allgather */
} gr_world;

typedef struct {
    int64_t numel;              /* > 0 */
    gr_dtype grad_dtype;        /* element type of the caller's gradient tensor */
} gr_tensor;

typedef struct {
    int32_t n_released;         /* groups released in this cycle */
    int32_t step_complete;      /* 1 when every group of the step has been released */
    int64_t cycle;              /* global cycle counter (0-based, counts gr_step calls) */
    int64_t step;               /* training-step counter (0-based) */
    int64_t released_elems;     /* gradient elements released in this cycle */
} gr_cycle_info;

typedef struct gr_ctx gr_ctx;

/* gr_init — COLLECTIVE (every rank calls it with identical table, group_of,
 * buffer_dtype, world_size, one_shot_max_bytes and chunk_elems).
 * Builds the response cache (bit positions, "processed ...
 * only once"), the static group-major fusion layout (each group a contiguous,
 * 16-byte aligned range), the chunk tables, and the symmetric memory
 * (bitvector slots, signal pad, double-buffered fusion buffer) mapped into
 * every peer over CUDA IPC.
 *   out       [out] receives the context (host pointer).
 *   world     [in]  see gr_world.
 *   table     [in]  T tensor descriptors (host, copied).
 *   group_of  [in]  group id per tensor, dense 0..G-1, every group non-empty (host, copied).
 * Limits: T up to ~131,000 tensors (the bitvector kernel's 64 KB of shared memory holds
 * 3 W words + ceil(G/32) words; GR_EINVAL beyond).
 * Errors: GR_EINVAL, GR_EMISMATCH (a hash of all of the above differs on some
 * rank; "globally consistent order"), GR_ECUDA, GR_ENOMEM.
 * With world->device < 0 the call only validates and builds the host-side
 * layouts (no CUDA; used by CPU tests); such a context supports gr_query and
 * gr_finalize only. */
int gr_init(gr_ctx **out, const gr_world *world, const gr_tensor *table, int32_t T,
            const int32_t *group_of, int32_t G);

/* gr_init_virtual — N ranks in ONE process on ONE device ("virtual ranks"; for testing and
 * profiling the N-rank path on a single GPU). Creates out[0..N-1], N = world->world_size in
 * 2..8, each an ordinary context of rank r with everything gr_init builds (response cache,
 * layouts, its own symmetric memory, streams and epochs); a peer's memory is plain memory of
 * the same device instead of a CUDA-IPC mapping, and NVLS is off. world->rank and
 * world->allgather are ignored. Every other call works per rank as documented, with one
 * rule: the collective calls (gr_step, gr_step_drain) of the N ranks must be made
 * concurrently, one host thread per rank, as they would be by N processes — each rank's
 * bitvector and reduction kernels are fired as ONE launch over all ranks (grid = ranks x
 * CTAs, every CTA resident, floor(SMs / N) CTAs per rank), when the last rank arrives. A rank
 * that has not arrived within timeout_ms is launched as absent: the others report
 * GR_ETIMEOUT, as with a stalled peer process (SPEC.md:406 analogue).
 *   out   [out] host array of world_size context pointers.
 * Errors: as gr_init (no GR_EMISMATCH: one table); on error every out[r] is NULL. */
int gr_init_virtual(gr_ctx **out, const gr_world *world, const gr_tensor *table, int32_t T,
                    const int32_t *group_of, int32_t G);

/* gr_mark_ready — LOCAL, thread-safe against a concurrent gr_step.
 * §4.1 step 1's "pending request": tensor tensor_id of this rank is ready and
 * its gradient lives at dev_ptr (device memory, numel elements of grad_dtype,
 * written in place with the reduced result). The producing kernels must have
 * been enqueued on world.compute_stream before this call; the next gr_step
 * orders the reduction after them. dev_ptr is borrowed until gr_wait returns.
 *   rank must equal world.rank (GR_EINVAL otherwise).
 * Errors: GR_EINVAL (bad id / null ptr / rank), GR_ESTATE (already marked in
 * this step, or the step is complete and gr_wait has not been called). */
int gr_mark_ready(gr_ctx *ctx, int32_t rank, int32_t tensor_id, void *dev_ptr);

/* gr_mark_ready_batch — LOCAL. gr_mark_ready for n tensors in one call
 * (tensor_ids[i] with dev_ptrs[i], host arrays, borrowed for the call only).
 * All-or-nothing validation: on error nothing is marked. */
int gr_mark_ready_batch(gr_ctx *ctx, int32_t rank, int32_t n, const int32_t *tensor_ids,
                        void *const *dev_ptrs);

/* gr_mark_ready_async — LOCAL. Like gr_mark_ready, but readiness is
 * stream-ordered: the ready flag is written by `stream` (cudaStream_t) when
 * the work enqueued on it before this call has completed (a driver stream
 * memory operation), so a cycle sees the tensor only once its gradient really
 * exists. Used to overlap reduction with a still-running backward pass.
 * stream is borrowed for the call; dev_ptr until gr_wait returns.
 * Errors: as gr_mark_ready, plus GR_ECUDA if the stream write cannot be enqueued. */
int gr_mark_ready_async(gr_ctx *ctx, int32_t rank, int32_t tensor_id, void *dev_ptr,
                        void *stream);

/* gr_step — COLLECTIVE: one coordination cycle ("tic").
 * Runs the bitvector kernel. In a tight cycle loop (less than GR_ARM_GAP_US = 50 us between
 * gr_step calls) it is already running, polling a pinned "doorbell" for at most GR_ARM_US =
 * 100 us per cycle; gr_step writes the cycle's marks and rings it. At N = 1 one resident kernel
 * serves cycle after cycle and the cycle's data kernel waits for the record it writes; at N > 1
 * each armed kernel serves one cycle and gr_step arms the next — no launch on the critical path (an expired kernel acknowledges and the cycle is launched as usual; gr_wait,
 * gr_step_drain and timing mode retire it; GR_ARM=0 turns this off; a device-wide synchronize
 * waits at most GR_ARM_US for it).
 * The kernel does: populate (a thread per word from the host
 * marks, or a __ballot_sync over the per-tensor flags of stream-ordered marks;
 * publish; AND over N ranks through peer loads; group release, with
 * __reduce_and_sync for groups spanning many words), enqueues the fused pack ->
 * sum-allreduce -> x1/N -> unpack kernel behind it (it reads the released set
 * from device memory, so the reduction starts the moment the bitvector kernel
 * ends; gr_wait finishes it), and waits for the bitvector kernel's result.
 *   released     [out] host array, capacity >= G: released group ids, ascending.
 *   info         [out] host struct (nullable).
 *   global_bits  [out] host array of W u32 words receiving the intersected
 *                bitvector A_c, status bits included (nullable).
 * The k-th gr_step call is cycle k on every rank; all ranks see identical
 * A_c, released lists and step_complete.
 * Errors: GR_ESTATE, GR_ECUDA, GR_ETIMEOUT, GR_EABORT, GR_ESHUTDOWN. */
int gr_step(gr_ctx *ctx, int32_t *released, gr_cycle_info *info, uint32_t *global_bits);

/* gr_wait — LOCAL (the end of a step's reduction. PAPER.md:148: a blocking
 * collective stops the work on the GPU until its result returns — hence gr_wait_async below).
 * Blocks until every reduction enqueued so far has finished
 * (gradients hold their reduced values) and makes world.compute_stream wait
 * for them. If the step is complete, starts the next step (marks cleared).
 * Errors: GR_ECUDA, GR_ETIMEOUT (a peer stopped mid-reduction). */
int gr_wait(gr_ctx *ctx);

/* gr_wait_async — LOCAL. Stream-ordered gr_wait: makes world.compute_stream wait for every
 * reduction enqueued so far (work enqueued on it afterwards sees the reduced gradients) and
 * starts the next step if this one is complete, without blocking the host — the CUDA-style
 * contract the training loop of a framework uses. Errors of the in-flight reduction surface
 * at the next gr_step / gr_wait. With GR_TRACE set it behaves like gr_wait. */
int gr_wait_async(gr_ctx *ctx);

/* gr_step_drain — COLLECTIVE (every rank calls it at the same cycle, i.e. after the same
 * number of gr_step calls in this step). The step's final coordination cycle, driven by the
 * device: every tensor must already be marked on this rank (host marks, or stream-ordered marks
 * whose flags may still be in flight; otherwise GR_ESTATE and nothing is launched). The
 * library's coordination stream first waits (stream-ordered, no SM held) for every stream that
 * issued gr_mark_ready_async in this step; the cycle's bitvector kernel then intersects as
 * gr_step does (re-checking the marks on the device) and releases every remaining group; the
 * fused reduction follows as for any cycle. The host does
 * not wait for the result and the step counts as complete: call gr_wait / gr_wait_async next.
 * This keeps a training loop's host free to enqueue the next iteration while the tail of
 * backward and its reduction run (the last tic of a step). A failure on the
 * device (peer timeout, ABORT, a peer that drained without marking everything) is reported by
 * the next gr_wait / gr_wait_async / gr_step. */
int gr_step_drain(gr_ctx *ctx);

/* gr_released_wait_async — LOCAL. Makes `stream` (a cudaStream_t, borrowed; NULL =
 * world.compute_stream)
 * wait for the reduction of every group released so far in this step, without ending the step
 * or blocking the host: work enqueued on `stream` afterwards sees those groups' reduced
 * gradients (e.g. a device->host copy or an optimizer update of the layers whose gradients are
 * final while later groups are still pending). PAPER.md:110: the operations released at a tic
 * are executed at that tic; this exposes their completion per cycle. GR_ESTATE on a dry
 * context or in a sticky error state. */
int gr_released_wait_async(gr_ctx *ctx, void *stream);

/* gr_set_status — LOCAL. Raise (1) or clear (0) this rank's ABORT / SHUTDOWN
 * status bit for the following cycles (PAPER.md:130 reserved status bits). */
int gr_set_status(gr_ctx *ctx, int32_t abort_flag, int32_t shutdown_flag);

/* Gradient statistics epilogue (PAPER.md:281 LARS, PAPER.md:283
 * adaptive loss scaling), fused into the unpack: while writing the reduced gradients the kernels
 * accumulate, per tensor, the sum of squares of the stored values (fp64 accumulator; LARS's
 * ||g||^2) and a flag that is 1 if any stored value is Inf/NaN (loss-scale overflow). Every rank
 * holds the full reduced gradient, so every rank gets the full statistics without extra
 * communication. Reset at the first cycle of each step.
 * gr_enable_grad_stats — LOCAL: on != 0 enables (allocates T doubles + one int32).
 * gr_grad_stats — LOCAL: after gr_wait (or a host sync), copy the current step's statistics
 *   to host memory (sumsq_host: T doubles, nonfinite_host: one int32; both nullable) and/or
 *   return the library-owned device arrays (sumsq_dev / nonfinite_dev, nullable) for a GPU
 *   optimizer (valid until the next step's first gr_step, stream-ordered after gr_wait_async).
 *   GR_ESTATE if statistics are not enabled. */
int gr_enable_grad_stats(gr_ctx *ctx, int32_t on);
int gr_grad_stats(gr_ctx *ctx, double *sumsq_host, int32_t *nonfinite_host, void **sumsq_dev,
                  void **nonfinite_dev);

/* gr_finalize — COLLECTIVE at the application level (no communication, but
 * peers must not be mid-cycle). Frees everything; ctx may be NULL. */
int gr_finalize(gr_ctx *ctx);

/* gr_last_error — text of the last error of ctx (or of the last failed
 * gr_init when ctx is NULL). Never NULL; owned by the library. */
const char *gr_last_error(gr_ctx *ctx);

/* gr_query — introspection for tests and the bench (host memory out).
 *   GR_Q_WORDS        int32          W
 *   GR_Q_BIT_OF       int32[T]       cache bit of each tensor
 *   GR_Q_BUF_OFFSET   int64[T]       element offset of each tensor in the fusion buffer
 *   GR_Q_NCHUNKS      int32          chunks of the static layout
 *   GR_Q_STATS        gr_stats       counters (launches, cycles, bytes)
 *   GR_Q_LAST_ALGO    int32          algorithm of the last data launch (gr_algo)
 *   GR_Q_NVLS         int32          1 if the NVLS multicast path is enabled
 *   GR_Q_NVLS_WHY     char[bytes]    why it is (not) enabled, NUL-terminated */
typedef enum {
    GR_Q_WORDS = 0, GR_Q_BIT_OF = 1, GR_Q_BUF_OFFSET = 2, GR_Q_NCHUNKS = 3,
    GR_Q_STATS = 4, GR_Q_LAST_ALGO = 5, GR_Q_NVLS = 6, GR_Q_NVLS_WHY = 7
} gr_query_kind;

/* GR_ALGO_NVLS: the reduce-scatter runs inside the NVSwitch (multimem.ld_reduce through a
 * multicast mapping, fp32 accumulation) and the result is broadcast with multimem.st. Off by
 * default (it measured slower than two-shot at N = 4 and has not run at N = 8); GR_NVLS=1 at
 * gr_init enables it when every GPU supports multicast. */
typedef enum { GR_ALGO_NONE = 0, GR_ALGO_LOCAL = 1, GR_ALGO_ONESHOT = 2, GR_ALGO_TWOSHOT = 3,
               GR_ALGO_NVLS = 4 } gr_algo;

typedef struct {
    int64_t cycles;             /* gr_step calls */
    int64_t steps;              /* completed training steps */
    int64_t bitvector_launches; /* bitvector kernel launches */
    int64_t data_launches;      /* fused pack/reduce/unpack kernel launches */
    int64_t released_elems;     /* gradient elements reduced */
    double data_kernel_ms;      /* summed device time of data launches (only with timing on) */
    double bitvector_kernel_ms; /* summed device time of bitvector launches (only with timing on) */
    double host_step_us;        /* summed host wall time inside gr_step */
    double host_wait_us;        /* part of it spent waiting for the bitvector kernel's hand-off */
    double bitvector_device_us; /* summed %globaltimer span of the bitvector kernels (start->hand-off) */
    int64_t data_launches_skipped; /* cycles whose data launch was skipped: no group was complete
                                      on this rank, so none could be released on any rank */
    int64_t armed_cycles;       /* cycles run by an armed bitvector kernel (launched ahead of the
                                   cycle, rung through a pinned doorbell; see gr_step) */
    int64_t armed_expired;      /* cycles whose armed kernel had expired before its doorbell (the
                                   cycle was launched as usual) */
} gr_stats;

int gr_query(gr_ctx *ctx, int32_t kind, void *out, size_t bytes);

/* Tracing: with the environment variable GR_TRACE=<prefix> set at gr_init, every
 * cycle's bitvector-kernel phase stamps and every data launch's per-item
 * (grab, ready, done, CTA/SM) %globaltimer stamps are appended at gr_wait to
 * <prefix>.rank<r>.jsonl (the analogue of the paper's Horovod Timeline, Fig.2). */

/* gr_set_timing — LOCAL. 1 = bracket every kernel launch with CUDA events on
 * its own stream and accumulate device time into gr_stats (default 0).
 * gr_reset_stats zeroes the counters. */
int gr_set_timing(gr_ctx *ctx, int32_t on);
int gr_reset_stats(gr_ctx *ctx);

/* Bench support (not part of the method): a synthetic backward-compute
 * stand-in that occupies `ctas` CTAs (each with ~200 KB shared memory, i.e.
 * one SM each) for `ns` nanoseconds of %globaltimer time on `stream`.
 * Models a layer's gradient computation. */
int gr_bench_spin(int64_t ns, int32_t ctas, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GR_H */
