/* race_mark_step.c — gr.h's threading contract under ThreadSanitizer: "gr_mark_ready may race
 * gr_step" (SURVEY.md §8(b) threading; include/gr.h gr_mark_ready "thread-safe against a
 * concurrent gr_step"). Plain C + pthreads, no Python in the process, so TSAN sees every host
 * access of the runtime (tools/build_tsan.sh builds libgr with -fsanitize=thread and this
 * program against it; run on a GPU box).
 *
 * Per step: a marker thread marks the T tensors in a random order with random pauses (host
 * marks, or stream-ordered marks on its own stream for odd steps) while the main thread runs
 * gr_step cycles until step_complete; every group must be released exactly once per step
 * (PAPER.md:137), the cycles' released lists ascending (reading R5), and the reduced values at
 * N = 1 are fl32(fl16(g)) (the fp16 wire, reading R8/V7) checked on the host after gr_wait.
 * Prints "ok" and exits 0 on success. */
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "gr.h"

#define T 96
#define G 12
#define NUMEL 1000
#define STEPS 60

#define CHECK(cond, ...)                                    \
    do {                                                    \
        if (!(cond)) {                                      \
            fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
            fprintf(stderr, __VA_ARGS__);                   \
            fprintf(stderr, "\n");                          \
            exit(1);                                        \
        }                                                   \
    } while (0)

struct marker_arg {
    gr_ctx *ctx;
    float **dptr;
    int order[T];
    unsigned seed;
    int async;
    cudaStream_t stream;
};

static void *marker(void *p) {
    struct marker_arg *a = (struct marker_arg *)p;
    for (int i = 0; i < T; ++i) {
        const int t = a->order[i];
        int rc = a->async ? gr_mark_ready_async(a->ctx, 0, t, a->dptr[t], a->stream)
                          : gr_mark_ready(a->ctx, 0, t, a->dptr[t]);
        CHECK(rc == GR_OK, "mark %d: %d %s", t, rc, gr_last_error(a->ctx));
        if (rand_r(&a->seed) % 4 == 0) usleep(rand_r(&a->seed) % 40);
    }
    return NULL;
}

static float host_f16_round(float x) { return __half2float(__float2half_rn(x)); }

int main(void) {
    gr_tensor table[T];
    int32_t group_of[T];
    for (int t = 0; t < T; ++t) {
        table[t].numel = NUMEL + t;
        table[t].grad_dtype = GR_F32;
        group_of[t] = t % G;
    }
    float *dptr[T];
    float *host[T];
    for (int t = 0; t < T; ++t) {
        CHECK(cudaMalloc((void **)&dptr[t], sizeof(float) * (NUMEL + t)) == cudaSuccess, "cudaMalloc");
        host[t] = (float *)malloc(sizeof(float) * (NUMEL + t));
    }
    cudaStream_t ms;
    CHECK(cudaStreamCreateWithFlags(&ms, cudaStreamNonBlocking) == cudaSuccess, "stream");
    gr_world w;
    memset(&w, 0, sizeof w);
    w.world_size = 1;
    w.buffer_dtype = GR_F16;
    w.one_shot_max_bytes = -1;
    w.timeout_ms = 20000;
    gr_ctx *ctx = NULL;
    int rc = gr_init(&ctx, &w, table, T, group_of, G);
    CHECK(rc == GR_OK, "gr_init: %d %s", rc, gr_last_error(NULL));

    unsigned seed = 12345;
    for (int step = 0; step < STEPS; ++step) {
        for (int t = 0; t < T; ++t) {  // fresh gradients: x = (i % 97 - 48) * 0.013 * (t + 1)
            for (int i = 0; i < NUMEL + t; ++i) host[t][i] = (float)((i % 97) - 48) * 0.013f * (float)(t + 1 + step);
            CHECK(cudaMemcpy(dptr[t], host[t], sizeof(float) * (NUMEL + t), cudaMemcpyHostToDevice) == cudaSuccess, "h2d");
        }
        struct marker_arg a;
        a.ctx = ctx;
        a.dptr = dptr;
        a.seed = seed + step;
        a.async = step & 1;
        a.stream = ms;
        for (int i = 0; i < T; ++i) a.order[i] = i;
        for (int i = T - 1; i > 0; --i) {
            const int j = rand_r(&seed) % (i + 1), x = a.order[i];
            a.order[i] = a.order[j];
            a.order[j] = x;
        }
        pthread_t th;
        CHECK(pthread_create(&th, NULL, marker, &a) == 0, "pthread_create");
        int released_count[G];
        memset(released_count, 0, sizeof released_count);
        int32_t rel[G];
        gr_cycle_info info;
        int cycles = 0;
        do {
            rc = gr_step(ctx, rel, &info, NULL);
            CHECK(rc == GR_OK, "step %d cycle %d: %d %s", step, cycles, rc, gr_last_error(ctx));
            for (int i = 0; i < info.n_released; ++i) {
                CHECK(rel[i] >= 0 && rel[i] < G, "bad group %d", rel[i]);
                if (i) CHECK(rel[i] > rel[i - 1], "released list not ascending");
                released_count[rel[i]]++;
            }
            ++cycles;
            CHECK(cycles < 200000, "step %d never completed", step);
        } while (!info.step_complete);
        CHECK(pthread_join(th, NULL) == 0, "join");
        rc = gr_wait(ctx);
        CHECK(rc == GR_OK, "gr_wait: %d %s", rc, gr_last_error(ctx));
        for (int g = 0; g < G; ++g) CHECK(released_count[g] == 1, "step %d: group %d released %d times", step, g, released_count[g]);
        for (int t = 0; t < T; t += 7) {
            float *out = (float *)malloc(sizeof(float) * (NUMEL + t));
            CHECK(cudaMemcpy(out, dptr[t], sizeof(float) * (NUMEL + t), cudaMemcpyDeviceToHost) == cudaSuccess, "d2h");
            for (int i = 0; i < NUMEL + t; ++i) {
                const float want = host_f16_round(host_f16_round(host[t][i]) * 1.0f);
                CHECK(memcmp(&out[i], &want, 4) == 0, "step %d tensor %d elem %d: %g != %g", step, t, i, out[i], want);
            }
            free(out);
        }
    }
    gr_finalize(ctx);
    printf("ok\n");
    return 0;
}
