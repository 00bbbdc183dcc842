/*
 * oracle/mf_oracle.cpp -- serial CPU oracle for SGD matrix factorization.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1610_05838_b200/) never imports, links or calls it,
 * and shares no code with it (no headers, helpers or constant tables).
 *
 * It is the paper's algorithm written out step by step, in the paper's
 * notation, with no blocking, fusion or reordering:
 *
 *   err_uv = r_uv - p_u q_v                        PAPER.md:124 (§2.2, eq. err)
 *   p_u <- p_u + alpha (err_uv q_v^T - lambda p_u) PAPER.md:125 (§2.2)
 *   q_v <- q_v + alpha (err_uv p_u^T - lambda q_v) PAPER.md:126 (§2.2)
 *   s_t = alpha / (1 + beta t^1.5)                 PAPER.md:388 (§5.1)
 *   test RMSE                                      PAPER.md:256 (§3.2.4)
 *   half-precision feature storage                 PAPER.md:197 (§3.1)
 *
 * Readings of the paper (DESIGN.md §2 lists them all): both updates use the
 * pre-update snapshot of p_u, q_v (A-1); lambda_p = lambda_q = lambda (A-2);
 * t starts at 0 (A-5); init is the counter hash of A-7; the shuffle is the
 * hash sort of A-8; fp16/bf16 storage is round-to-nearest-even with fp32 math
 * (A-13): fp16 through the host compiler's _Float16 conversion, bf16 through
 * the bit recipe.  Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math.
 *
 * Pins (tests/test_oracle.py): the 4x4,k=2 hand-worked example (P-1), SPEC's
 * k=2 examples (P-2), finite-difference gradient of the per-sample loss (P-3),
 * LR schedule values (P-4), RMSE hand values + brute force (P-5), planted
 * recovery at the noise floor (P-6), monotone training loss (P-7), exhaustive
 * fp16/bf16 conversion tables (P-8), wave/serial bit identity (D-3).
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

namespace {

enum Storage { ST_F32 = 0, ST_F16 = 1, ST_BF16 = 2, ST_F64 = 3 };

/* ---- storage conversions (A-13) ---------------------------------------- */
inline uint16_t f32_to_f16(float x) {
    _Float16 h = (_Float16)x; /* IEEE binary16, round-to-nearest-even */
    uint16_t b;
    std::memcpy(&b, &h, 2);
    return b;
}
inline float f16_to_f32(uint16_t b) {
    _Float16 h;
    std::memcpy(&h, &b, 2);
    return (float)h;
}
inline uint16_t f32_to_bf16(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    if ((b & 0x7F800000u) == 0x7F800000u && (b & 0x007FFFFFu)) return (uint16_t)((b >> 16) | 0x0040u); /* NaN stays NaN */
    b += 0x7FFFu + ((b >> 16) & 1u);
    return (uint16_t)(b >> 16);
}
inline float bf16_to_f32(uint16_t h) {
    uint32_t b = (uint32_t)h << 16;
    float x;
    std::memcpy(&x, &b, 4);
    return x;
}

/* widen element d of a stored row to the compute type T */
template <typename T>
inline T load_el(const void *base, int storage, int64_t idx) {
    switch (storage) {
        case ST_F32: return (T)((const float *)base)[idx];
        case ST_F16: return (T)f16_to_f32(((const uint16_t *)base)[idx]);
        case ST_BF16: return (T)bf16_to_f32(((const uint16_t *)base)[idx]);
        default: return (T)((const double *)base)[idx];
    }
}
/* round_st(): store a computed value in the storage precision */
template <typename T>
inline void store_el(void *base, int storage, int64_t idx, T x) {
    switch (storage) {
        case ST_F32: ((float *)base)[idx] = (float)x; break;
        case ST_F16: ((uint16_t *)base)[idx] = f32_to_f16((float)x); break;
        case ST_BF16: ((uint16_t *)base)[idx] = f32_to_bf16((float)x); break;
        default: ((double *)base)[idx] = (double)x; break;
    }
}

inline uint64_t splitmix64(uint64_t x) { /* Steele/Lea/Flood SplitMix64 output function */
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/*
 * One serial epoch ("an epoch ... involves executing N
 * updates one after other").  T is the compute type: float for
 * the fp32/fp16/bf16 storage modes (fp32 math), double for the
 * fp64 pin used by the finite-difference test.  Returns 0, or -5 at the first
 * non-finite error (that sample is not applied).
 */
template <typename T>
int epoch_t(int32_t k, int storage, void *P, void *Q, const int32_t *u, const int32_t *v, const float *r,
            const int64_t *order, int64_t N, T eta, T lambda) {
    std::vector<T> p(k), q(k);
    for (int64_t s = 0; s < N; s++) {
        const int64_t i = order ? order[s] : s;
        const int64_t pu = (int64_t)u[i] * k, qv = (int64_t)v[i] * k;
        for (int d = 0; d < k; d++) { p[d] = load_el<T>(P, storage, pu + d); q[d] = load_el<T>(Q, storage, qv + d); }
        T dot = 0; /* left to right, no contraction */
        for (int d = 0; d < k; d++) dot = dot + p[d] * q[d];
        const T err = (T)r[i] - dot; /* err_uv = r_uv - p_u q_v */
        if (!std::isfinite((double)err)) return -5;
        for (int d = 0; d < k; d++) {
            /* both from the snapshot p, q (reading A-1) */
            store_el<T>(P, storage, pu + d, p[d] + eta * (err * q[d] - lambda * p[d]));
            store_el<T>(Q, storage, qv + d, q[d] + eta * (err * p[d] - lambda * q[d]));
        }
    }
    return 0;
}

}  // namespace

extern "C" {

/* learning rate at 0-based epoch t: s_t = alpha/(1+beta*t^1.5), double, then fp32 (A-5) */
double orc_lr(double alpha, double beta, int32_t t) { return alpha / (1.0 + beta * std::pow((double)t, 1.5)); }
float orc_eta(double alpha, double beta, int32_t t) { return (float)orc_lr(alpha, beta, t); }

uint16_t orc_f32_to_f16(float x) { return f32_to_f16(x); }
float orc_f16_to_f32(uint16_t h) { return f16_to_f32(h); }
uint16_t orc_f32_to_bf16(float x) { return f32_to_bf16(x); }
float orc_bf16_to_f32(uint16_t h) { return bf16_to_f32(h); }
uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }

/*
 * A-7 initialisation: X[row][col] = (float)(h>>40) * 2^-24 * (float)(1/sqrt(k)),
 * h = splitmix64(seed ^ (tag<<60) ^ (row*k+col)), tag 0 = P, 1 = Q; then round_st.
 */
void orc_init(uint64_t seed, int64_t rows, int32_t k, uint32_t tag, int32_t storage, void *out) {
    const float scale = (float)(1.0 / std::sqrt((double)k));
    for (int64_t row = 0; row < rows; row++)
        for (int32_t col = 0; col < k; col++) {
            const uint64_t idx = (uint64_t)(row * k + col);
            const uint64_t h = splitmix64(seed ^ ((uint64_t)tag << 60) ^ idx);
            const float unit = (float)(h >> 40) * 0x1.0p-24f;
            store_el<float>(out, storage, row * k + col, unit * scale);
        }
}

/* A-8 shuffle: perm sorts sample indices by key splitmix64(seed ^ i), ties by i */
void orc_shuffle_perm(uint64_t seed, int64_t N, int64_t *perm) {
    std::vector<std::pair<uint64_t, int64_t>> kv((size_t)N);
    for (int64_t i = 0; i < N; i++) kv[(size_t)i] = {splitmix64(seed ^ (uint64_t)i), i};
    std::sort(kv.begin(), kv.end());
    for (int64_t i = 0; i < N; i++) perm[i] = kv[(size_t)i].second;
}

/* one serial epoch over samples order[0..N) (order may be NULL = identity) */
int orc_epoch(int32_t k, int32_t storage, void *P, void *Q, const int32_t *u, const int32_t *v, const float *r,
              const int64_t *order, int64_t N, float eta, float lambda) {
    if (storage == ST_F64) return epoch_t<double>(k, storage, P, Q, u, v, r, order, N, (double)eta, (double)lambda);
    return epoch_t<float>(k, storage, P, Q, u, v, r, order, N, eta, lambda);
}
/* fp64 variant with fp64 hyper-parameters (finite-difference pin, P-3) */
int orc_epoch_f64(int32_t k, double *P, double *Q, const int32_t *u, const int32_t *v, const float *r,
                  const int64_t *order, int64_t N, double eta, double lambda) {
    return epoch_t<double>(k, ST_F64, P, Q, u, v, r, order, N, eta, lambda);
}

/* test RMSE = sqrt(sum (r - p_u.q_v)^2 / N), dot and sum in fp64 (A-6). -1 if N == 0 */
double orc_rmse(int32_t k, int32_t storage, const void *P, const void *Q, const int32_t *u, const int32_t *v,
                const float *r, int64_t N) {
    if (N <= 0) return -1.0;
    double sum = 0.0;
    for (int64_t i = 0; i < N; i++) {
        double dot = 0.0;
        for (int d = 0; d < k; d++)
            dot += load_el<double>(P, storage, (int64_t)u[i] * k + d) * load_el<double>(Q, storage, (int64_t)v[i] * k + d);
        const double e = (double)r[i] - dot;
        sum += e * e;
    }
    return std::sqrt(sum / (double)N);
}

/* objective of PAPER.md:119 under reading A-3: sum_i 1/2 (r - p.q)^2 + 1/2 lambda (|p_u|^2 + |q_v|^2), fp64 */
double orc_loss(int32_t k, int32_t storage, const void *P, const void *Q, const int32_t *u, const int32_t *v,
                const float *r, int64_t N, double lambda) {
    double L = 0.0;
    for (int64_t i = 0; i < N; i++) {
        double dot = 0.0, pp = 0.0, qq = 0.0;
        for (int d = 0; d < k; d++) {
            const double a = load_el<double>(P, storage, (int64_t)u[i] * k + d);
            const double b = load_el<double>(Q, storage, (int64_t)v[i] * k + d);
            dot += a * b;
            pp += a * a;
            qq += b * b;
        }
        const double e = (double)r[i] - dot;
        L += 0.5 * e * e + 0.5 * lambda * (pp + qq);
    }
    return L;
}

/*
 * Deterministic conflict-free waves (north star): scanning
 * samples in the given order, wave = max(last[u], last[v]) + 1 with last[]
 * starting at -1, so the first wave is 0.  Returns the number of waves.
 */
int64_t orc_waves(int64_t m, int64_t n, const int32_t *u, const int32_t *v, const int64_t *order, int64_t N,
                  int32_t *wave) {
    std::vector<int32_t> lu((size_t)m, -1), lv((size_t)n, -1);
    int64_t nw = 0;
    for (int64_t s = 0; s < N; s++) {
        const int64_t i = order ? order[s] : s;
        const int32_t w = std::max(lu[(size_t)u[i]], lv[(size_t)v[i]]) + 1;
        wave[s] = w;
        lu[(size_t)u[i]] = w;
        lv[(size_t)v[i]] = w;
        nw = std::max<int64_t>(nw, (int64_t)w + 1);
    }
    return nw;
}

}  // extern "C"
