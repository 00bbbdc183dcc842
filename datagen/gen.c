/*
 * datagen/gen.c -- seeded synthetic rating generator (test data, NOT method).
 *
 * This module is the one piece shared by both sides of the parity check
 * (the oracle in oracle/ and the CUDA path in paper_1610_05838_b200/): it
 * produces COO triples (u, v, r) from a planted low-rank model.  It holds
 * none of the SGD method's arithmetic (no update, no dot product of trained
 * factors, no init, no shuffle).  Recipe: SURVEY.md §8(d) "Synthetic inputs",
 * restated in DESIGN.md §"Input recipe".
 *
 *   H(seed, tag, idx) = splitmix64(seed ^ (tag << 60) ^ idx)
 *   P*[u][j], Q*[v][j] ~ N(0, var = rank^-1/2)  (Box-Muller on tags 0 / 1)
 *   sample i: u = H(seed,2,i) mod m, v = H(seed,3,i) mod n  (with replacement)
 *             r = P*_u . Q*_v + sigma * N(0,1)             (noise: tag 4)
 *   without replacement (small configs): candidate cell
 *             c_j = H(seed,5,j) mod (m*n), first-come distinct cells kept.
 *
 * Ratings therefore have mean 0 and std ~ 1, uniform (Poisson) degrees.
 * Generated once on the host and handed to both sides (libm's log/cos are
 * not bit-identical to CUDA's, so nothing regenerates it on the device).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t gen_mix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t gen_H(uint64_t seed, uint64_t tag, uint64_t idx) {
    return gen_mix(seed ^ (tag << 60) ^ idx);
}

/* standard normal from two counter draws (Box-Muller, cosine branch) */
static inline double gen_gauss(uint64_t seed, uint64_t tag, uint64_t idx) {
    uint64_t h1 = gen_H(seed, tag, 2 * idx), h2 = gen_H(seed, tag, 2 * idx + 1);
    double u1 = ((double)(h1 >> 11) + 1.0) * 0x1.0p-53; /* (0, 1] */
    double u2 = (double)(h2 >> 11) * 0x1.0p-53;         /* [0, 1) */
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
}

/* planted factor tables, row-major rows x rank, fp64 */
static void planted(uint64_t seed, uint64_t tag, int64_t rows, int rank, double *out) {
    double sd = pow((double)rank, -0.25); /* variance rank^-1/2 */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; i++)
        for (int j = 0; j < rank; j++)
            out[i * rank + j] = sd * gen_gauss(seed, tag, (uint64_t)(i * rank + j));
}

int mfgen_planted_factors(uint64_t seed, int64_t m, int64_t n, int rank, double *Pstar, double *Qstar) {
    if (m <= 0 || n <= 0 || rank <= 0 || !Pstar || !Qstar) return -1;
    planted(seed, 0, m, rank, Pstar);
    planted(seed, 1, n, rank, Qstar);
    return 0;
}

/*
 * Fill u[0..total), v, r.  with_replacement=0 draws distinct cells (requires
 * total <= 0.9 m*n so rejection terminates quickly).  Returns 0 or -1.
 */
int mfgen_planted_coo(uint64_t seed, int64_t m, int64_t n, int rank, double sigma, int64_t total,
                      int with_replacement, int32_t *u, int32_t *v, float *r) {
    if (m <= 0 || n <= 0 || rank <= 0 || total < 0 || !u || !v || !r) return -1;
    if (m > 2147483647ll || n > 2147483647ll) return -1;
    double *Ps = (double *)malloc(sizeof(double) * (size_t)m * rank);
    double *Qs = (double *)malloc(sizeof(double) * (size_t)n * rank);
    if (!Ps || !Qs) { free(Ps); free(Qs); return -1; }
    planted(seed, 0, m, rank, Ps);
    planted(seed, 1, n, rank, Qs);
    if (with_replacement) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < total; i++) {
            u[i] = (int32_t)(gen_H(seed, 2, (uint64_t)i) % (uint64_t)m);
            v[i] = (int32_t)(gen_H(seed, 3, (uint64_t)i) % (uint64_t)n);
        }
    } else {
        uint64_t cells = (uint64_t)m * (uint64_t)n;
        if ((uint64_t)total > cells - cells / 10) { free(Ps); free(Qs); return -1; }
        uint8_t *seen = (uint8_t *)calloc((size_t)(cells / 8 + 1), 1);
        if (!seen) { free(Ps); free(Qs); return -1; }
        int64_t got = 0;
        for (uint64_t j = 0; got < total; j++) {
            uint64_t c = gen_H(seed, 5, j) % cells;
            if (seen[c >> 3] & (1u << (c & 7))) continue;
            seen[c >> 3] |= (uint8_t)(1u << (c & 7));
            u[got] = (int32_t)(c / (uint64_t)n);
            v[got] = (int32_t)(c % (uint64_t)n);
            got++;
        }
        free(seen);
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < total; i++) {
        const double *p = Ps + (int64_t)u[i] * rank, *q = Qs + (int64_t)v[i] * rank;
        double s = 0.0;
        for (int j = 0; j < rank; j++) s += p[j] * q[j];
        r[i] = (float)(s + sigma * gen_gauss(seed, 4, (uint64_t)i));
    }
    free(Ps);
    free(Qs);
    return 0;
}

/*
 * One row segment of a larger planted problem (the multi-GPU bench: rank g generates only its own
 * rows).  The planted model is the global one -- P*_u for global row u, the same Q* on every rank --
 * and the samples are draws i0 .. i0+total-1 of the global stream with u restricted to the segment:
 *   u = row_lo + H(seed,2,i) mod (row_hi - row_lo),  v = H(seed,3,i) mod n,
 *   r = P*_u . Q*_v + sigma * N(0,1) (tag 4, index i).
 * Disjoint index ranges per rank (and for train / test) give disjoint, independent draws.
 */
int mfgen_planted_segment(uint64_t seed, int64_t m, int64_t row_lo, int64_t row_hi, int64_t n, int rank,
                          double sigma, int64_t i0, int64_t total, int32_t *u, int32_t *v, float *r) {
    if (m <= 0 || n <= 0 || rank <= 0 || total < 0 || i0 < 0 || !u || !v || !r) return -1;
    if (row_lo < 0 || row_hi > m || row_lo >= row_hi || m > 2147483647ll || n > 2147483647ll) return -1;
    const int64_t rows = row_hi - row_lo;
    double *Ps = (double *)malloc(sizeof(double) * (size_t)rows * rank);
    double *Qs = (double *)malloc(sizeof(double) * (size_t)n * rank);
    if (!Ps || !Qs) { free(Ps); free(Qs); return -1; }
    const double sd = pow((double)rank, -0.25);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; i++)
        for (int j = 0; j < rank; j++)
            Ps[i * rank + j] = sd * gen_gauss(seed, 0, (uint64_t)((row_lo + i) * rank + j));
    planted(seed, 1, n, rank, Qs);
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < total; t++) {
        const uint64_t i = (uint64_t)(i0 + t);
        const int64_t ul = (int64_t)(gen_H(seed, 2, i) % (uint64_t)rows);
        u[t] = (int32_t)(row_lo + ul);
        v[t] = (int32_t)(gen_H(seed, 3, i) % (uint64_t)n);
        const double *p = Ps + ul * rank, *q = Qs + (int64_t)v[t] * rank;
        double sum = 0.0;
        for (int j = 0; j < rank; j++) sum += p[j] * q[j];
        r[t] = (float)(sum + sigma * gen_gauss(seed, 4, i));
    }
    free(Ps);
    free(Qs);
    return 0;
}

/* Zipf(s) popularity over `count` ids: cdf[i] = sum_{j<=i} (j+1)^-s / total; the id order is then
 * scrambled by a seeded Fisher-Yates permutation (hot ids are not clustered at low indices). */
static int zipf_table(uint64_t seed, uint64_t tag, int64_t count, double s, double **cdf_out, int32_t **perm_out) {
    double *cdf = (double *)malloc(sizeof(double) * (size_t)count);
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)count);
    if (!cdf || !perm) { free(cdf); free(perm); return -1; }
    double acc = 0.0;
    for (int64_t i = 0; i < count; i++) { acc += pow((double)(i + 1), -s); cdf[i] = acc; }
    for (int64_t i = 0; i < count; i++) { cdf[i] /= acc; perm[i] = (int32_t)i; }
    cdf[count - 1] = 1.0;
    for (int64_t i = count - 1; i > 0; i--) {
        const int64_t j = (int64_t)(gen_H(seed, tag, (uint64_t)i) % (uint64_t)(i + 1));
        const int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
    *cdf_out = cdf;
    *perm_out = perm;
    return 0;
}

static inline int32_t zipf_draw(const double *cdf, const int32_t *perm, int64_t count, uint64_t h) {
    const double x = (double)(h >> 11) * 0x1.0p-53;
    int64_t lo = 0, hi = count - 1;
    while (lo < hi) {  /* first index with cdf >= x */
        const int64_t mid = (lo + hi) / 2;
        if (cdf[mid] < x) lo = mid + 1; else hi = mid;
    }
    return perm[lo];
}

/*
 * Skewed workload: row ids ~ Zipf(s_u), column ids ~ Zipf(s_v) (with
 * replacement, ids scrambled), ratings from the same planted rank-`rank` model as mfgen_planted_coo.
 */
int mfgen_zipf_coo(uint64_t seed, int64_t m, int64_t n, int rank, double sigma, int64_t total, double s_u,
                   double s_v, int32_t *u, int32_t *v, float *r) {
    if (m <= 0 || n <= 0 || rank <= 0 || total < 0 || !u || !v || !r || s_u < 0 || s_v < 0) return -1;
    if (m > 2147483647ll || n > 2147483647ll) return -1;
    double *cu = NULL, *cv = NULL;
    int32_t *pu = NULL, *pv = NULL;
    double *Ps = (double *)malloc(sizeof(double) * (size_t)m * rank);
    double *Qs = (double *)malloc(sizeof(double) * (size_t)n * rank);
    if (!Ps || !Qs || zipf_table(seed, 6, m, s_u, &cu, &pu) || zipf_table(seed, 7, n, s_v, &cv, &pv)) {
        free(Ps); free(Qs); free(cu); free(cv); free(pu); free(pv);
        return -1;
    }
    planted(seed, 0, m, rank, Ps);
    planted(seed, 1, n, rank, Qs);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < total; i++) {
        u[i] = zipf_draw(cu, pu, m, gen_H(seed, 2, (uint64_t)i));
        v[i] = zipf_draw(cv, pv, n, gen_H(seed, 3, (uint64_t)i));
        const double *p = Ps + (int64_t)u[i] * rank, *q = Qs + (int64_t)v[i] * rank;
        double s = 0.0;
        for (int j = 0; j < rank; j++) s += p[j] * q[j];
        r[i] = (float)(s + sigma * gen_gauss(seed, 4, (uint64_t)i));
    }
    free(Ps); free(Qs); free(cu); free(cv); free(pu); free(pv);
    return 0;
}
