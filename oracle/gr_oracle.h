/*
 * gr_oracle.h — CPU oracle for the per-step synchronous gradient reduction of
 * arXiv 1909.11150 ("Exascale Deep Learning for Scientific Inverse Problems"),
 * §4.1 Bitvector Allreduce (Fig.3b) and
 * §4.2 Grouping.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load, call or execute
 * anything under oracle/. The product path (include/gr.h,
 * paper_1909_11150_b200/) shares no code, header, table or constant with this
 * file and never calls it.
 *
 * Plain, slow, obviously correct: single-threaded C11, plain loops, fp64
 * accumulation for the reference values. Every function cites the passage it
 * follows; every reading of a silent/ambiguous passage is listed in DESIGN.md
 * §3 (readings R1..R14) and named here as "reading Rk".
 *
 * Pins (tests/test_oracle_*.py, run with -m "not gpu"): brute-force set
 * intersection (populate+intersect), the closed-form release cycle
 * (release), SPEC worked vectors (tests/golden/), exact rational sums
 * (reduce_f64), numpy's IEEE float16 cast (emu16), integer payloads (emu*).
 * No function here is "parity unpinned".
 */
#ifndef GR_ORACLE_H
#define GR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Number of status bits reserved at the start of the bitvector
 * ("An initial set of bits in the bitvector are reserved for status
 * signaling", Fig.3b). Reading R1: two bits, bit0 = ABORT,
 * bit1 = SHUTDOWN, complement-coded so that one AND also ORs them. */
#define ORC_STATUS_BITS 2

/* W = ceil((T + 2) / 32): u32 words in the bitvector (reading R2). */
int32_t orc_words(int32_t T);

/* Response cache bit positions ("a simple global enumeration of
 * the collective operations"; "maps to an integer cache bit
 * position"). Reading R3: the cache is filled once, in group-major order:
 * pos(t) = index of t when tensors are sorted by (group_of[t], t);
 * bit_of[t] = 2 + pos(t). Returns 0, or -1 if group_of is not dense 0..G-1
 * with every group non-empty. */
int orc_bit_positions(int32_t T, const int32_t *group_of, int32_t G,
                      int32_t *bit_of /*[T]*/);

/* §4.1 step 1: "Each worker populates a bit vector, setting
 * bits associated with its pending requests with bit positions determined
 * from the cache." pending[t] != 0 marks a pending request. Status bits are
 * complement-coded (reading R1): bit0 = !abort_flag, bit1 = !shutdown_flag. */
void orc_populate(int32_t T, int32_t W, const int32_t *bit_of,
                  const uint8_t *pending /*[T]*/, int abort_flag,
                  int shutdown_flag, uint32_t *L /*[W]*/);

/* §4.1 step 2: "The bit vectors are globally intersected
 * using MPI_Allreduce with the binary MPI_BAND operation."
 * A[w] = L[0][w] & L[1][w] & ... & L[N-1][w]. */
void orc_intersect(int32_t N, int32_t W, const uint32_t *L /*[N][W]*/,
                   uint32_t *A /*[W]*/);

/* §4.1 step 3 ("searches for set bits ... forms a list of
 * associated cache entries", "in cache bit order" PAPER.md:130) combined
 * with §4.2 ("only requests forming a complete group are fused
 * and executed. If multiple complete groups are encountered, they are fused
 * together"). For g = 0..G-1: if !group_released[g] and every bit_of[t],
 * t in g, is set in A, append g to released[] and set group_released[g].
 * Returns the number of groups appended (ascending ids, reading R5). */
int32_t orc_release(int32_t T, int32_t G, const int32_t *group_of,
                    const int32_t *bit_of, const uint32_t *A,
                    uint8_t *group_released /*[G] in/out*/,
                    int32_t *released /*[G] out*/);

/* One training step of N simulated ranks, cycle by cycle (one cycle = one
 * "tic"; reading R12).
 * mark_cycle[r*T + t] = m_r(t): rank r marks tensor t after it has completed
 * m_r(t) cycles, i.e. t is pending on r from cycle m_r(t) on (until its group
 * is released, reading R4). status (nullable) [r*max_cycles + c]: bit0 =
 * rank r raises ABORT in cycle c, bit1 = SHUTDOWN.
 * Outputs per cycle c < *n_cycles: A_out[c*W ..], nrel_out[c],
 * rel_out[c*G ..] (released group ids); rel_cycle_of_group[g].
 * Returns 0 when every group has been released, 1 if a status bit ended the
 * step (that cycle releases nothing, reading R13), 2 if max_cycles elapsed
 * with groups outstanding (reading R14), -1 on bad input. */
int orc_simulate_step(int32_t N, int32_t T, int32_t G, const int32_t *group_of,
                      const int32_t *mark_cycle, const uint8_t *status,
                      int32_t max_cycles, uint32_t *A_out, int32_t *nrel_out,
                      int32_t *rel_out, int32_t *rel_cycle_of_group,
                      int32_t *n_cycles);

/* Reduced value, plain definition (reading R7): ref[i] = (sum_r g_r[i]) / N,
 * accumulated in fp64 in rank order. g points to N arrays of n floats. */
void orc_reduce_f64(int32_t N, int64_t n, const float *const *g, double *ref);

/* Exact emulation of the arithmetic fixed by readings R7-R9: fp32
 * accumulation in rank order 0..N-1 of the buffer-precision values, one fp32
 * multiply by fl32(1/N), rounded to the buffer precision, then to the gradient
 * precision. buffer_f16 / grad_f16 select fp16 (IEEE binary16, RN-even).
 *   x_r   = buffer_f16 ? fl32(fl16(g_r[i])) : g_r[i]
 *   acc   = ((x_0 + x_1) + x_2) + ...          (fp32, left to right)
 *   y     = fl32(acc * fl32(1/N))
 *   y     = buffer_f16 ? fl32(fl16(y)) : y
 *   out   = grad_f16  ? fl32(fl16(y)) : y
 * Inputs for fp16 gradients are passed as their exact fp32 values. */
void orc_emulate(int32_t N, int64_t n, const float *const *g, int buffer_f16,
                 int grad_f16, float *out);

/* fl32(fl16_RN(x)): the IEEE binary16 round-to-nearest-even cast, used by
 * orc_emulate; exported so tests can pin it against numpy.float16. */
float orc_round_f16(float x);

#ifdef __cplusplus
}
#endif
#endif /* GR_ORACLE_H */
