// mf_kernels.cuh -- kernel argument blocks and host launch entry points
// shared between the host API (mf_api.cu) and the kernel translation units.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace mf {

enum StorageKind { kF32 = 0, kF16 = 1, kBF16 = 2 };

// device scratch words reset at the start of every epoch
struct DevScratch {
    unsigned long long chunk;     // batch-Hogwild! chunk claim counter
    unsigned long long updates;   // exactly-once counter (MF_OPT_COUNT_UPDATES)
    int diverged;                 // set when any err is non-finite
    unsigned bar_count;           // grid barrier arrivals
    unsigned bar_gen;             // grid barrier generation
    int pad;
    unsigned long long bad;       // validation: out-of-range / non-finite count
    unsigned long long chunk2;    // second claim counter (a concurrent launch on another stream)
};

struct UpdateArgs {
    const int32_t *u;
    const int32_t *v;
    const float *r;
    int64_t n;          // samples (or end of range)
    void *P;
    void *Q;
    int k;
    float eta;
    float lam;
    int batch_f;        // samples per chunk (multiple of 32)
    int count_updates;
    DevScratch *scratch;
    unsigned long long *chunk_ctr;  // batch-Hogwild! claim counter (nullptr: &scratch->chunk)
    const int64_t *wave_off;  // deterministic: wave offsets (nwaves + 1)
    int64_t nwaves;
    int64_t active_groups;  // batch-Hogwild!: groups beyond this idle (exact worker count)
    const unsigned long long *abort_if;  // optional: the kernel does nothing if *abort_if != 0
    int prefetch;       // batch-Hogwild!: L2-prefetch the rows of the rating this many steps ahead (0 = off)
    int prefetch_kind;  // bit 0: P rows only; bit 1: per-lane prefetch.global.L2 instead of one bulk prefetch
    int cache_policy;   // L2 eviction priorities (MF_OPT_VARIANT bits 28..30): 0 = R evict_first, 1 = none (plain
                        // loads), 2 = R evict_first + P/Q rows evict_last, 3 = R evict_first + Q rows evict_last,
                        // 4 / 5 = R evict_first + evict_last on 50 / 75% of the P lines, 6 / 7 = as 4 / 5 + Q rows
                        // evict_last
    int r_stage;        // batch-Hogwild! triples: 2 = TMA bulk copies of each chunk into shared memory, else
                        // registers (3 coalesced 32-bit loads per lane per 32-sample tile, shuffled to groups)
    int q_red;          // batch-Hogwild!: Q rows written back as an atomic add of their change (red.global.add,
                        // DESIGN.md A-20) instead of a store of the new row -- resolved by launch_hogwild from:
    int q_mode;         //   MF_OPT_Q_UPDATE: 0 store, 1 atomic add, 2 auto (atomic add iff kappa < kQRedKappa)
    float q_share;      //   sum over the launch's Q rows of (degree / samples)^2: kappa = workers x q_share is the
                        //   expected number of concurrent updates an update shares its Q row with
    const int32_t *ord_u;  // deterministic dataflow (k_flow): per sample, # earlier samples (serial order) of its row u
    const int32_t *ord_v;  //   ... and of its column v
    unsigned *cnt_u;       //   per P row / Q row: updates applied so far this epoch
    unsigned *cnt_v;
    int barrier;        // deterministic waves, 1024-thread CTAs: 0 = arrival counter polled to (w+1) x CTAs
                        // (one release reduction + acquire polls), 1 = last arriver bumps a generation flag
};

// MF_OPT_Q_UPDATE = 2 (auto): atomic Q write-back iff kappa < this (A-20)
constexpr float kQRedKappa = 0.5f;

// Kernel-shape choice for (k, storage); filled by select_shape().
struct ShapeId {
    int storage, L, V, VB, full;
};

// launchers (return cudaError_t; grid sizing inside)
cudaError_t launch_hogwild(const ShapeId &sh, const UpdateArgs &a, int workers, int variant, cudaStream_t st,
                           int *workers_used);
cudaError_t launch_waves(const ShapeId &sh, const UpdateArgs &a, cudaStream_t st, int *launches, int big = 0);
cudaError_t launch_rmse(const ShapeId &sh, const int32_t *u, const int32_t *v, const float *r, int64_t n,
                        const void *P, const void *Q, int k, double *partials, int nparts, double *out,
                        cudaStream_t st, int do_sqrt = 1);
cudaError_t launch_init_offset(int storage, void *X, int64_t elem0, int64_t count, int k, uint64_t seed, uint32_t tag,
                               cudaStream_t st);
cudaError_t launch_init_rows(int storage, void *X, int64_t row0, int64_t rows, int k, uint64_t seed, uint32_t tag,
                             cudaStream_t st);
cudaError_t launch_from_f32(int storage, void *X, const float *src, int64_t count, cudaStream_t st);
cudaError_t launch_to_f32(int storage, const void *X, float *dst, int64_t count, cudaStream_t st);
cudaError_t launch_validate_rows(const int32_t *u, const int32_t *v, const float *r, int64_t n, int64_t row_lo,
                                 int64_t row_hi, int64_t n_cols, DevScratch *scratch, cudaStream_t st);
cudaError_t launch_rebase(int32_t *u, int64_t n, int32_t off, cudaStream_t st);
cudaError_t launch_shuffle_perm(int64_t n, uint64_t seed, uint32_t *perm_out, cudaStream_t st);
cudaError_t launch_gather_validate(const int32_t *u_in, const int32_t *v_in, const float *r_in, const uint32_t *idx,
                                   int64_t n, int64_t row_lo, int64_t row_hi, int64_t n_cols, int32_t *u_out,
                                   int32_t *v_out, float *r_out, DevScratch *scratch, cudaStream_t st);
// sum over columns of deg(v)^2 (exact in fp64 below 2^53), deg = histogram of v[0..n); tmp: n_cols words
cudaError_t launch_col_sq(const int32_t *v, int64_t n, int64_t n_cols, unsigned *tmp, double *out, cudaStream_t st);
cudaError_t launch_compose(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, cudaStream_t st);
cudaError_t launch_gather(const int32_t *u_in, const int32_t *v_in, const float *r_in, const uint32_t *idx, int64_t n,
                          int32_t *u_out, int32_t *v_out, float *r_out, cudaStream_t st);

cudaError_t launch_flow(const ShapeId &sh, const UpdateArgs &a, cudaStream_t st, int *warps_used, int form = 0);
ShapeId flow_shape(int k, int storage);  // the one-rating-per-warp shape k_flow runs

ShapeId select_shape(int k, int storage, int variant);
ShapeId hogwild_shape(int k, int storage, int variant);  // batch-Hogwild!'s default (variant 0) differs at k = 128
ShapeId select_generic_shape(int k, int storage);
int rmse_parts();

}  // namespace mf
