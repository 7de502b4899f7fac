/* abi_dry.c — the boundary as plain C: compiled with gcc against include/gr.h only, linked
 * with libgr.so, no Python or torch in the process. A dry context (world.device < 0, gr.h)
 * builds the response cache on the host; the program checks the cache bit positions against
 * reading R3 (bit = 2 + position of the tensor in (group, tensor) order),
 * W = ceil((T+2)/32), the 16-byte alignment of the fusion layout, and the error paths.
 * Prints "ok" and exits 0 on success. Built and run by tests/test_abi.py. */
#include <stdio.h>
#include <string.h>

#include "gr.h"

#define CHECK(cond, ...)                       \
    do {                                       \
        if (!(cond)) {                         \
            fprintf(stderr, __VA_ARGS__);      \
            fprintf(stderr, "\n");             \
            return 1;                          \
        }                                      \
    } while (0)

int main(void) {
    enum { T = 7, G = 3 };
    const int64_t numel[T] = {5, 100, 3, 40, 41, 7, 90};
    const int32_t group_of[T] = {2, 0, 1, 0, 2, 1, 0};
    gr_tensor table[T];
    for (int t = 0; t < T; ++t) {
        table[t].numel = numel[t];
        table[t].grad_dtype = GR_F32;
    }
    gr_world w;
    memset(&w, 0, sizeof w);
    w.rank = 0;
    w.world_size = 1;
    w.device = -1; /* dry: host-side layouts only */
    w.buffer_dtype = GR_F16;
    w.one_shot_max_bytes = -1;

    gr_ctx *ctx = NULL;
    int rc = gr_init(&ctx, &w, table, T, group_of, G);
    CHECK(rc == GR_OK && ctx, "gr_init: %d %s", rc, gr_last_error(NULL));

    int32_t W = 0;
    rc = gr_query(ctx, GR_Q_WORDS, &W, sizeof W);
    CHECK(rc == GR_OK && W == (T + 2 + 31) / 32, "W = %d (rc %d)", W, rc);

    /* reading R3, written out: tensors sorted by (group, id) */
    int32_t bit[T];
    rc = gr_query(ctx, GR_Q_BIT_OF, bit, sizeof bit);
    CHECK(rc == GR_OK, "GR_Q_BIT_OF rc %d", rc);
    int pos = 0;
    for (int g = 0; g < G; ++g)
        for (int t = 0; t < T; ++t)
            if (group_of[t] == g) {
                CHECK(bit[t] == 2 + pos, "tensor %d: bit %d, expected %d", t, bit[t], 2 + pos);
                ++pos;
            }

    /* fusion layout: group-major, every tensor 8-element aligned, no overlap */
    int64_t off[T];
    rc = gr_query(ctx, GR_Q_BUF_OFFSET, off, sizeof off);
    CHECK(rc == GR_OK, "GR_Q_BUF_OFFSET rc %d", rc);
    for (int a = 0; a < T; ++a) {
        CHECK(off[a] % 8 == 0, "tensor %d offset %lld not 8-aligned", a, (long long)off[a]);
        for (int b = 0; b < T; ++b)
            if (a != b)
                CHECK(off[a] + numel[a] <= off[b] || off[b] + numel[b] <= off[a], "tensors %d and %d overlap", a, b);
        for (int b = 0; b < T; ++b)  /* group-major: a lower group id lies before */
            if (group_of[a] < group_of[b]) CHECK(off[a] < off[b], "layout not group-major (%d, %d)", a, b);
    }

    /* a dry context refuses device work; bad arguments are rejected */
    int32_t rel[G];
    gr_cycle_info info;
    rc = gr_step(ctx, rel, &info, NULL);
    CHECK(rc == GR_ESTATE, "gr_step on a dry context returned %d", rc);
    CHECK(strlen(gr_last_error(ctx)) > 0, "no error text");
    CHECK(gr_mark_ready(ctx, 0, 0, (void *)0x1000) == GR_ESTATE, "mark on a dry context");
    CHECK(gr_finalize(ctx) == GR_OK, "gr_finalize");

    const int32_t bad_groups[T] = {0, 0, 0, 0, 0, 0, 5}; /* not dense */
    rc = gr_init(&ctx, &w, table, T, bad_groups, 6);
    CHECK(rc == GR_EINVAL, "non-dense groups accepted (%d)", rc);
    CHECK(gr_finalize(NULL) == GR_OK, "gr_finalize(NULL)");
    printf("ok\n");
    return 0;
}
