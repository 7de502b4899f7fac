/*
 * gr_oracle.c — CPU oracle (TEST INFRASTRUCTURE ONLY; see gr_oracle.h for the
 * usage rule, the pins and the list of readings).
 *
 * Paper: arXiv 1909.11150, §4.1 (lines 107-118, Fig.3b) and
 * §4.2 (lines 134-144). Build: cc -std=c11 -O1 -fno-fast-math
 * -ffp-contract=off -shared -fPIC (see oracle/build.py).
 */
#include "gr_oracle.h"

#include <stdlib.h>
#include <string.h>

int32_t orc_words(int32_t T) { return (T + ORC_STATUS_BITS + 31) / 32; }

static void set_bit(uint32_t *v, int32_t b) { v[b / 32] |= (uint32_t)1u << (b % 32); }
static int get_bit(const uint32_t *v, int32_t b) { return (int)((v[b / 32] >> (b % 32)) & 1u); }

/* the cache gives "a simple global enumeration of the
 * collective operations"; reading R3: fill it in (group, tensor) order. */
int orc_bit_positions(int32_t T, const int32_t *group_of, int32_t G,
                      int32_t *bit_of) {
    if (T <= 0 || G <= 0) return -1;
    for (int32_t g = 0; g < G; g++) {
        int32_t members = 0;
        for (int32_t t = 0; t < T; t++) members += (group_of[t] == g);
        if (members == 0) return -1; /* groups must be non-empty */
    }
    for (int32_t t = 0; t < T; t++)
        if (group_of[t] < 0 || group_of[t] >= G) return -1;
    int32_t pos = 0;
    for (int32_t g = 0; g < G; g++)
        for (int32_t t = 0; t < T; t++)
            if (group_of[t] == g) bit_of[t] = ORC_STATUS_BITS + pos++;
    return 0;
}

/* PAPER.md:114 step 1. */
void orc_populate(int32_t T, int32_t W, const int32_t *bit_of,
                  const uint8_t *pending, int abort_flag, int shutdown_flag,
                  uint32_t *L) {
    for (int32_t w = 0; w < W; w++) L[w] = 0;
    if (!abort_flag) set_bit(L, 0);    /* complement-coded status (R1) */
    if (!shutdown_flag) set_bit(L, 1);
    for (int32_t t = 0; t < T; t++)
        if (pending[t]) set_bit(L, bit_of[t]);
}

/* PAPER.md:115 step 2: MPI_Allreduce(MPI_BAND). */
void orc_intersect(int32_t N, int32_t W, const uint32_t *L, uint32_t *A) {
    for (int32_t w = 0; w < W; w++) {
        uint32_t acc = 0xFFFFFFFFu;
        for (int32_t r = 0; r < N; r++) acc &= L[(int64_t)r * W + w];
        A[w] = acc;
    }
}

/* PAPER.md:116 step 3 + PAPER.md:137 (complete groups only). */
int32_t orc_release(int32_t T, int32_t G, const int32_t *group_of,
                    const int32_t *bit_of, const uint32_t *A,
                    uint8_t *group_released, int32_t *released) {
    int32_t n = 0;
    for (int32_t g = 0; g < G; g++) {
        if (group_released[g]) continue;
        int complete = 1;
        for (int32_t t = 0; t < T; t++)
            if (group_of[t] == g && !get_bit(A, bit_of[t])) complete = 0;
        if (complete) {
            group_released[g] = 1;
            released[n++] = g;
        }
    }
    return n;
}

/* One training step, cycle by cycle ("at each tic only common
 * collective operation requests across workers are executed"). */
int orc_simulate_step(int32_t N, int32_t T, int32_t G, const int32_t *group_of,
                      const int32_t *mark_cycle, const uint8_t *status,
                      int32_t max_cycles, uint32_t *A_out, int32_t *nrel_out,
                      int32_t *rel_out, int32_t *rel_cycle_of_group,
                      int32_t *n_cycles) {
    if (N <= 0 || max_cycles <= 0) return -1;
    const int32_t W = orc_words(T);
    int32_t *bit_of = malloc(sizeof(int32_t) * (size_t)T);
    uint8_t *tensor_released = calloc((size_t)T, 1);
    uint8_t *group_released = calloc((size_t)G, 1);
    uint8_t *pending = malloc((size_t)T);
    uint32_t *L = malloc(sizeof(uint32_t) * (size_t)N * (size_t)W);
    int rc = -1;
    if (!bit_of || !tensor_released || !group_released || !pending || !L) goto out;
    if (orc_bit_positions(T, group_of, G, bit_of) != 0) goto out;
    for (int32_t g = 0; g < G; g++) rel_cycle_of_group[g] = -1;

    rc = 2;
    *n_cycles = max_cycles;
    for (int32_t c = 0; c < max_cycles; c++) {
        /* step 1 on every rank: pending = marked and not yet executed (R4) */
        for (int32_t r = 0; r < N; r++) {
            for (int32_t t = 0; t < T; t++) {
                int32_t m = mark_cycle[(int64_t)r * T + t];
                pending[t] = (uint8_t)(m >= 0 && m <= c && !tensor_released[t]);
            }
            int st = status ? status[(int64_t)r * max_cycles + c] : 0;
            orc_populate(T, W, bit_of, pending, st & 1, (st >> 1) & 1,
                         L + (int64_t)r * W);
        }
        /* step 2 */
        uint32_t *A = A_out + (int64_t)c * W;
        orc_intersect(N, W, L, A);
        /* status bits: OR over ranks via the complement code (R1, R13) */
        if (!get_bit(A, 0) || !get_bit(A, 1)) {
            nrel_out[c] = 0;
            *n_cycles = c + 1;
            rc = 1;
            break;
        }
        /* step 3 + grouping */
        int32_t *rel = rel_out + (int64_t)c * G;
        nrel_out[c] = orc_release(T, G, group_of, bit_of, A, group_released, rel);
        for (int32_t k = 0; k < nrel_out[c]; k++) {
            rel_cycle_of_group[rel[k]] = c;
            for (int32_t t = 0; t < T; t++)
                if (group_of[t] == rel[k]) tensor_released[t] = 1;
        }
        int all = 1;
        for (int32_t g = 0; g < G; g++) all &= group_released[g];
        if (all) {
            *n_cycles = c + 1;
            rc = 0;
            break;
        }
    }
out:
    free(bit_of);
    free(tensor_released);
    free(group_released);
    free(pending);
    free(L);
    return rc;
}

/* Reading R7: the reduced gradient is the replica average (1/N) sum_r g_r. */
void orc_reduce_f64(int32_t N, int64_t n, const float *const *g, double *ref) {
    for (int64_t i = 0; i < n; i++) {
        double acc = 0.0;
        for (int32_t r = 0; r < N; r++) acc += (double)g[r][i];
        ref[i] = acc / (double)N;
    }
}

/* IEEE binary16 RN-even cast: the compiler's _Float16 conversion. */
float orc_round_f16(float x) { return (float)(_Float16)x; }

/* Readings R7-R9: fp32 rank-order accumulation, scale by fl32(1/N) before the
 * buffer-precision store, then cast to the gradient precision. */
void orc_emulate(int32_t N, int64_t n, const float *const *g, int buffer_f16,
                 int grad_f16, float *out) {
    const float inv_n = 1.0f / (float)N;
    for (int64_t i = 0; i < n; i++) {
        float acc = 0.0f;
        for (int32_t r = 0; r < N; r++) {
            float x = buffer_f16 ? orc_round_f16(g[r][i]) : g[r][i];
            acc = (r == 0) ? x : acc + x;
        }
        float y = acc * inv_n;
        if (buffer_f16) y = orc_round_f16(y);
        if (grad_f16) y = orc_round_f16(y);
        out[i] = y;
    }
}
