/*
 * examples/train.c -- the C ABI (include/mf.h) used from plain C, no Python, no PyTorch.
 *
 * Builds a small planted rank-4 problem in host memory, trains it with each single-GPU schedule and
 * prints the test RMSE of the initial factors and after each epoch; fails unless it has halved.
 * Exit status 0 on success; without a CUDA device the first call that needs one fails with
 * MF_ECUDA, which the program reports and returns as exit status 3.
 *
 *   gcc -O2 -std=c11 -I include examples/train.c -L paper_1610_05838_b200 -lmf \
 *       -Wl,-rpath,$PWD/paper_1610_05838_b200 -lm -o /tmp/mf_train && /tmp/mf_train
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mf.h"

/* SplitMix64: a self-contained generator for the example's data (not the library's) */
static uint64_t mix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

#define CHECK(ctx, call)                                                                        \
    do {                                                                                        \
        int rc_ = (call);                                                                       \
        if (rc_ != MF_OK) {                                                                     \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, mf_status_string(rc_),               \
                    (ctx) ? mf_last_error(ctx) : "");                                           \
            return rc_ == MF_ECUDA ? 3 : 1;                                                     \
        }                                                                                       \
    } while (0)

int main(void) {
    const int64_t m = 2000, n = 1500, N = 200000, N_test = 20000;
    const int rank = 4, k = 32;
    /* planted factors and ratings r = p*_u . q*_v + 0.01 noise */
    double *Ps = malloc(sizeof(double) * m * rank), *Qs = malloc(sizeof(double) * n * rank);
    int32_t *u = malloc(sizeof(int32_t) * (N + N_test)), *v = malloc(sizeof(int32_t) * (N + N_test));
    float *r = malloc(sizeof(float) * (N + N_test));
    if (!Ps || !Qs || !u || !v || !r) return 1;
    for (int64_t i = 0; i < m * rank; i++) Ps[i] = (unit(mix(i)) - 0.5) * 2.0;
    for (int64_t i = 0; i < n * rank; i++) Qs[i] = (unit(mix(i + (1ull << 40))) - 0.5) * 2.0;
    for (int64_t i = 0; i < N + N_test; i++) {
        u[i] = (int32_t)(mix(i + (2ull << 40)) % (uint64_t)m);
        v[i] = (int32_t)(mix(i + (3ull << 40)) % (uint64_t)n);
        double s = 0;
        for (int j = 0; j < rank; j++) s += Ps[u[i] * rank + j] * Qs[v[i] * rank + j];
        r[i] = (float)(s + 0.01 * (unit(mix(i + (4ull << 40))) - 0.5));
    }
    const int schedules[] = {MF_SCHED_HOGWILD, MF_SCHED_DETERMINISTIC, MF_SCHED_WAVEFRONT};
    const char *names[] = {"hogwild", "deterministic", "wavefront (CTA workers)"};
    for (int si = 0; si < 3; si++) {
        mf_ctx *ctx = NULL;
        CHECK(ctx, mf_create(m, n, k, 0.1f, 0.001f, 7, &ctx));
        CHECK(ctx, mf_set_option(ctx, MF_OPT_STORAGE, 1)); /* fp16 features, fp32 math */
        CHECK(ctx, mf_set_option(ctx, MF_OPT_BETA, 0.05));
        if (schedules[si] == MF_SCHED_WAVEFRONT) CHECK(ctx, mf_set_option(ctx, MF_OPT_WAVE_CTA, 1));
        CHECK(ctx, mf_load_coo(ctx, u, v, r, N));
        double rmse0 = 0, rmse = 0;
        CHECK(ctx, mf_rmse(ctx, u + N, v + N, r + N, N_test, &rmse0)); /* the initial factors (A-7) */
        printf("%-24s %.4f |", names[si], rmse0);
        for (int e = 0; e < 12; e++) {
            mf_epoch_stats st;
            CHECK(ctx, mf_epoch(ctx, schedules[si], &st));
            if (st.updates != N) {
                fprintf(stderr, "epoch %d processed %lld of %lld samples\n", e, (long long)st.updates, (long long)N);
                return 1;
            }
            CHECK(ctx, mf_rmse(ctx, u + N, v + N, r + N, N_test, &rmse));
            printf(" %.4f", rmse);
        }
        printf("\n");
        float *P = malloc(sizeof(float) * m * k), *Q = malloc(sizeof(float) * n * k);
        CHECK(ctx, mf_get_factors(ctx, P, Q));
        for (int64_t i = 0; i < m * k; i++)
            if (!isfinite(P[i])) return 1;
        free(P);
        free(Q);
        mf_destroy(ctx);
        if (!(rmse < 0.5 * rmse0)) {
            fprintf(stderr, "%s: test RMSE %.4f is not below half the initial %.4f\n", names[si], rmse, rmse0);
            return 1;
        }
    }
    free(Ps), free(Qs), free(u), free(v), free(r);
    return 0;
}
