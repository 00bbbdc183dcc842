/*
 * include/mf.h -- C ABI of the B200 SGD matrix-factorization hot path.
 *
 * The library (paper_1610_05838_b200/libmf.so, CUDA for sm_100a) trains
 * R ~ P x Q by stochastic gradient descent (§2.2):
 *
 *     err_uv = r_uv - p_u . q_v
 *     p_u   <- p_u + eta_t (err_uv q_v - lambda p_u)
 *     q_v   <- q_v + eta_t (err_uv p_u - lambda q_v)      (both from the
 *                                                       pre-update snapshot)
 *     eta_t  = alpha / (1 + beta t^1.5),  t = 0,1,...    (§5.1)
 *
 * under the paper's schedules: batch-Hogwild! (§3.2.2),
 * wavefront-update (§3.2.3), a deterministic
 * conflict-free wave mode that reproduces serial SGD (D-3), and the
 * multi-GPU block partition with Q-segment rotation (§4.1).
 *
 * Conventions
 *  - Every function returns MF_OK (0) or a negative mf_status; no C++
 *    exception crosses the ABI.  mf_last_error() returns a message for the
 *    last failing call on that context.
 *  - Ratings are COO triples (u, v, r): int32 row index 0 <= u < m, int32
 *    column index 0 <= v < n, fp32 rating (12 bytes/sample).
 *  - P is m x k and Q is n x k, both ROW-MAJOR with one contiguous k-vector
 *    per user / item (the paper's Q is k x n; stored
 *    transposed for coalescing; reading A-4).
 *  - Input pointers may be host (pageable or pinned) or device pointers; the
 *    library detects which and COPIES the data.  The caller keeps ownership.
 *    Output buffers are caller-allocated HOST memory unless stated otherwise.
 *  - The context owns every device allocation it makes; mf_destroy frees it.
 *  - One context per device per thread; calls on one context are not
 *    reentrant.  All calls are synchronous with respect to the host unless
 *    stated otherwise; work is issued on the context stream (MF_OPT_STREAM).
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    needs one fails with MF_ECUDA.
 */
#ifndef MF_H
#define MF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mf_ctx mf_ctx;

typedef enum {
    MF_OK = 0,
    MF_EINVAL = -1,     /* bad argument: sizes <= 0, lr <= 0, lambda < 0, null pointer, index out of range, non-finite rating */
    MF_ENOMEM = -2,     /* device or host allocation failed */
    MF_ECUDA = -3,      /* CUDA runtime error or no device (message in mf_last_error) */
    MF_ESTATE = -4,     /* call out of order, e.g. mf_epoch before mf_load_coo */
    MF_EDIVERGED = -5,  /* a non-finite prediction error occurred during the epoch */
    MF_ENCCL = -6       /* NCCL failure in the partitioned path */
} mf_status;

typedef enum {
    MF_SCHED_HOGWILD = 0,        /* batch-Hogwild!: workers claim f consecutive shuffled samples, lock-free */
    MF_SCHED_WAVEFRONT = 1,      /* wavefront-update: s row bands x c column blocks, column lock array */
    MF_SCHED_DETERMINISTIC = 2,  /* conflict-free waves: bit-reproducible, equals serial SGD on the shuffled order (D-3) */
    MF_SCHED_PARTITIONED = 3     /* P row segments x rotating Q segments over G ranks or G logical partitions */
} mf_schedule;

typedef enum {
    MF_OPT_STORAGE = 0,       /* feature storage: 0 fp32, 1 fp16, 2 bf16; math is fp32. Before the first load. */
    MF_OPT_BETA = 1,          /* beta of the LR schedule (default 0) */
    MF_OPT_WORKERS = 2,       /* batch-Hogwild! concurrent ratings, also per partition of MF_SCHED_PARTITIONED; 0 = auto
                                 (A-10: every worker processes >= 10^4 samples per epoch, capped by residency) */
    MF_OPT_BATCH_F = 3,       /* samples per batch-Hogwild! chunk, multiple of 32 (default 256) */
    MF_OPT_WAVE_ROWS = 4,     /* wavefront workers s = row bands (0 = auto) */
    MF_OPT_WAVE_COLS = 5,     /* wavefront column blocks c >= s (0 = auto) */
    MF_OPT_DEVICE = 6,        /* CUDA device ordinal (before the first load) */
    MF_OPT_STREAM = 7,        /* cudaStream_t as an integer; 0 = the context's own stream */
    MF_OPT_SHUFFLE = 8,       /* 1 = permute samples once at load by the A-8 hash sort (default); 0 = keep the given order;
                                 2 = also re-permute before every later epoch t: order_t = order_{t-1}[pi_t], pi_t the
                                 A-8 permutation under seed_shuffle ^ (t << 48) (mf_get_order follows) */
    MF_OPT_COUNT_UPDATES = 9, /* 1 = count updates per epoch on the device (exactly-once check) */
    MF_OPT_WAVE_PERM = 10,    /* wavefront column sequences: 0 randomized Latin rectangle (default), 1 independent random permutations */
    MF_OPT_EPOCH = 11,        /* set the epoch index t used by the LR schedule */
    MF_OPT_PARTITIONS = 12,   /* MF_SCHED_PARTITIONED without NCCL: G logical partitions run on this GPU (loopback) */
    MF_OPT_SEED_SHUFFLE = 13, /* seed of the A-8 shuffle (default: the mf_create seed) */
    MF_OPT_VARIANT = 14,      /* kernel variant selector for tuning (0 = default).  Bit fields: 0..3 group shape (0 = auto:
                                 for batch-Hogwild! at k = 128 in 16-bit storage, 8 lanes per rating where P exceeds
                                 twice the L2 and Q is under a quarter of it, else 32); 4..7
                                 ratings in flight per batch-Hogwild! group (0 = auto: 2 for fp32 rows of k >= 128,
                                 else 1); 8..15 wavefront-CTA shape; 16..19 batch-Hogwild! L2 row prefetch distance
                                 in steps (0 = auto: MF_SCHED_HOGWILD epochs 0, 1, 2 run off, 1 step, off and the
                                 prefetch is kept iff its epoch was > 3% faster; 15 = off); for CTA wavefront workers
                                 1 = bulk, 2 = per-line P-row prefetch per tile (0 = auto: kept unless > 3% slower).  20..21: CTA Q-group staging, 2 = thread
                                 loop instead of bulk async copies.  22: CTA wavefront q_v read from shared memory, 1 = when p_u's
                                 load is issued, else (default) once p_u has arrived; 23: CTA wavefront, 1 = wait for the
                                 Q group's copy-in before claiming tiles, else (default) at a thread's first rating.  24..25: deterministic execution, 0 = 1024-thread
                                 CTAs with 2 samples of a wave per group, 1 = 1 sample, 2 = 256-thread CTAs (identical
                                 results).  26..27: CTA in-block clamp, samples per concurrent group 0 -> 16, 1 -> 32,
                                 2 -> 64, 3 -> 8.  Only bits 26..27 change what is computed (how many of a block's
                                 ratings are in flight at once; lock-free inside a block as batch-Hogwild!). */
    MF_OPT_TRACE = 15,        /* wavefront audit trace: 1 = record (worker, block, t_start, t_end) per block */
    MF_OPT_SUBEPOCHS = 16,    /* partitioned: passes S per epoch, each over 1/S of the shuffled samples with its own Latin square (0 = auto = 4) */
    MF_OPT_WAVE_CTA = 17,     /* wavefront worker: 0 = one warp, block processed serially; 1 = one 1024-thread CTA
                                 per SM with the column group's Q rows staged in shared memory, lock-free inside the block;
                                 2 = as 1 with two 512-thread CTA workers per SM */
    MF_OPT_STREAM_CHUNK = 18, /* mf_epoch_host: samples per streamed chunk (default 2^22) */
    MF_OPT_PART_SPLIT = 19,   /* partitioned: 2 = unit grid (default): 2G column units (segment halves), each family of
                                 halves rotating by its own Latin square (a randomized G x 2G Latin rectangle per pass,
                                 P:525-535), the two units of a partition updated concurrently on two streams with half
                                 of its workers each, every unit's hand-over overlapping the other unit's updates
                                 (P:307-314); 0 = one launch per whole block, hand-over after it; 1 = each block as two
                                 half-segment sub-blocks in sequence with all workers each -- twice the ratings in flight
                                 per Q column, so further from serial SGD */
    MF_OPT_R_STAGING = 20,    /* batch-Hogwild! rating batches: 1 = registers (three coalesced 32-bit loads per lane per 32-sample
                                 tile, handed to the groups by shuffles); 2 = staged in shared memory by the TMA engine (bulk
                                 copies of each chunk's u, v, r, double-buffered per warp; needs 16-B aligned arrays, else 1) */
    MF_OPT_WAVE_PASSES = 21,  /* wavefront: passes P per epoch, each over 1/P of the shuffled samples with fresh column
                                 sequences for every worker (0 = auto: blocks of >= 16k samples for CTA workers, >= 64
                                 for warp workers) */
    MF_OPT_P_HOST = 22,       /* 1 = out-of-core factors: P lives in caller host memory and streams through the GPU row block
                                 by row block (mf_epoch_host_blocks, mf_rmse_host_blocks); no device P is allocated, and
                                 mf_epoch / mf_epoch_host / mf_rmse and P in mf_get/set_factors fail with MF_ESTATE.  Set
                                 before the factors exist. */
    MF_OPT_Q_UPDATE = 23,     /* batch-Hogwild! (also inside partitioned blocks and streamed epochs) Q write-back: 1 = atomic add
                                 of the row's change q' - q (red.global.add; concurrent updates of one Q row all land,
                                 Hogwild!'s atomic component-wise add); 0 = store q' (the paper's worker writes the row
                                 back: of two concurrent updates the last store wins); 2 = auto (default): atomic add iff
                                 kappa = workers x sum_v (deg v / N)^2 over the launch's Q rows -- the expected number of
                                 concurrent updates an update shares its Q row with -- is below 0.5 (A-20).
                                 The deterministic and wavefront schedules always store. */
    MF_OPT_DET_FLOW = 24,     /* MF_SCHED_DETERMINISTIC execution: 0 = the waves one after another with a grid barrier between
                                 them (default); 1 = no barriers -- the wave-sorted samples stream through persistent warps
                                 (warp w of W owns positions w, w + W, ...; MF_OPT_VARIANT bits 24..25 = 2: 32-sample tiles
                                 claimed in order) and each rating waits, only when it has to, until per-row update
                                 counters reach its ordinals in the serial order (slower on every measured shape; DESIGN.md
                                 5.3).  Both are serial SGD (D-3) and bit-reproducible;
                                 their dot products use different lane shapes, so they agree to rounding, not bit for bit. */
    MF_OPT_Q_KAPPA = 25       /* read-only (mf_get_option): kappa of the last batch-Hogwild! or partitioned epoch, the largest
                                 over its launches (-1 before one) */
} mf_option;

typedef struct {
    int64_t updates;         /* samples processed (exact if MF_OPT_COUNT_UPDATES, else N) */
    double seconds;          /* device time of the whole epoch (CUDA events on the context stream) */
    double kernel_seconds;   /* device time of the update kernel(s) alone */
    float lr;                /* eta_t used */
    int32_t epoch;           /* t used */
    int32_t workers;         /* concurrent workers used */
    int32_t launches;        /* kernels launched by this call */
} mf_epoch_stats;

/* Create a context for an m x n rating matrix R with rank k (R ~ P x Q, P m x k, Q k x n: PAPER.md:116-119,
 * §2.1), initial learning rate alpha = lr of the schedule s_t = alpha / (1 + beta t^1.5) (PAPER.md:385-388,
 * §5.1; beta via MF_OPT_BETA), regulariser lambda (the paper's lambda_p = lambda_q; one value
 * as in Table 3; A-2) and seed (factor init, which the paper leaves open:
 * DESIGN.md A-7; and the shuffle of PAPER.md:228 unless MF_OPT_SEED_SHUFFLE, A-8).
 * Requires 0 < m, n < 2^31, 0 < k <= 1024, lr > 0, lambda >= 0 (MF_EINVAL otherwise; *out untouched).
 * Allocates no device memory (that happens on the first load or factor access); *out is owned by the
 * caller and released with mf_destroy. */
int mf_create(int64_t m, int64_t n, int32_t k, float lr, float lambda, uint64_t seed, mf_ctx **out);

/* Set / get an mf_option.  Layout-affecting keys (STORAGE, DEVICE) fail with MF_ESTATE after the factors exist. */
int mf_set_option(mf_ctx *ctx, int key, double value);
int mf_get_option(const mf_ctx *ctx, int key, double *value);

/* Load the training set, the observed entries of R as COO triples (u, v, r) (12 bytes per
 * sample), replacing any previous one.  u, v, r are nnz-element arrays in host or device memory
 * (detected), COPIED; the caller keeps ownership.  On the device: validate 0 <= u < m, 0 <= v < n and finite
 * r (MF_EINVAL on failure, nothing loaded: SPEC.md:62), then permute once by the A-8 hash order ("we shuffle
 * samples"; MF_OPT_SHUFFLE) and store as three SoA arrays; the column-degree moment
 * sum_v (deg v / N)^2 is computed once here for the Q write-back rule (MF_OPT_Q_UPDATE).  Allocates and
 * initialises P, Q (A-7) on first use.  nnz >= 1 (MF_EINVAL); MF_ENOMEM / MF_ECUDA on device failures. */
int mf_load_coo(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz);

/* Run one epoch -- every loaded rating updated once by the rule of PAPER.md:124-126 (§2.2: err = r - p.q,
 * p += eta (err q - lambda p), q += eta (err p - lambda q), both from the pre-update snapshot, A-1) at
 * eta_t -- under `schedule` (an mf_schedule: batch-Hogwild! PAPER.md:227-228, wavefront-update
 * PAPER.md:239-245, deterministic waves DESIGN.md D-3, partitioned PAPER.md:287-305), then t += 1.
 * Synchronous.  stats (may be NULL) receives the update count, device times, eta, workers and launches.
 * MF_ESTATE before a load; MF_EINVAL for an unknown schedule; MF_EDIVERGED if any err was non-finite
 * (factors are left as they are); MF_ECUDA / MF_ENCCL on device / NCCL failures. */
int mf_epoch(mf_ctx *ctx, int schedule, mf_epoch_stats *stats);

/* Streamed epoch: batch-Hogwild! (schedule must be MF_SCHED_HOGWILD) over caller ratings that are NOT
 * kept resident -- host memory (pinned for full speed) or device memory, processed in the given order
 * in chunks of MF_OPT_STREAM_CHUNK samples.  The copy of chunk i+1 overlaps the update kernel on chunk i
 * (three device staging buffers, a copy stream and the context stream; the paper's transfer/compute
 * overlap, §4.2), so the training set may exceed HBM.  Every chunk is validated on the
 * device before use: on the first invalid sample the remaining chunks are skipped (earlier chunks stay
 * applied) and MF_EINVAL is returned.  The caller shuffles; t advances by 1.  Factors
 * must exist or are created (A-7) on first use; no prior mf_load_coo is needed. */
int mf_epoch_host(mf_ctx *ctx, int schedule, const int32_t *u, const int32_t *v, const float *r, int64_t nnz,
                  mf_epoch_stats *stats);

/* Out-of-core factors (MF_OPT_P_HOST = 1): the paper's own path for a problem whose factors exceed device
 * memory -- R divided into row blocks, each block's P segment and ratings copied in, updated, and the P
 * segment copied back while the next block is in flight (§4.1; 307-320, §4.2; the
 * Hugewiki run used 64 x 1 blocks).  Q (n x k) stays on the device.
 * P_host: caller memory (pinned host memory for full overlap; pageable or device memory also work), m x k
 * row-major in the context's STORAGE precision (fp32 / fp16 / bf16 bit patterns), owned by the caller.
 * Row block b covers rows [floor(b m / nblocks), floor((b+1) m / nblocks)) and its ratings are
 * u/v/r[block_off[b] .. block_off[b+1]) (block_off: nblocks + 1 host int64, 0 .. nnz, nondecreasing).
 * mf_init_rows_host writes the A-7 initial values of rows [row0, row0 + rows) of P (tag 0) or Q (tag 1)
 * in storage precision to `out` (host).  mf_epoch_host_blocks runs one batch-Hogwild! epoch (t += 1) over
 * the blocks in order (with MF_OPT_WORKERS = 1: serial SGD over the given order); a sample outside its
 * block's rows, an out-of-range column or a non-finite rating returns MF_EINVAL and skips the remaining
 * chunks (earlier ones stay applied).  mf_rmse_host_blocks: test RMSE over test triples grouped the same
 * way, fp64 sum in fixed order.  MF_ESTATE without MF_OPT_P_HOST; MF_EINVAL for bad pointers / offsets. */
int mf_init_rows_host(mf_ctx *ctx, int32_t tag, int64_t row0, int64_t rows, void *out);
int mf_epoch_host_blocks(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz,
                         const int64_t *block_off, int32_t nblocks, void *P_host, mf_epoch_stats *stats);
int mf_rmse_host_blocks(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz,
                        const int64_t *block_off, int32_t nblocks, const void *P_host, double *out);

/* Test RMSE sqrt(sum (r - p_u.q_v)^2 / nnz) over the given triples: fp32 dot, fp64 sum,
 * deterministic reduction order.  nnz >= 1.  In the partitioned NCCL mode the call is collective and
 * every rank passes its local test triples (u in its row segment; nnz = 0 allowed, the global count
 * must be >= 1); all ranks get the global value.
 * Collective calls (mf_epoch, mf_rmse, mf_get_factors with NCCL attached) agree on their status: every
 * rank returns the most negative status any rank had, and a rank whose own arguments, state or test
 * triples are invalid still takes part, so its peers are never left blocked in NCCL (mf_last_error of
 * a rank that did nothing wrong says which status a peer had). */
int mf_rmse(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz, double *out);

/* Copy the factors P (m x k) and Q (stored n x k, i.e. the paper's Q^T, PAPER.md:116 / A-4) to caller-
 * allocated host buffers, widened to fp32 from the storage precision, row-major; either may
 * be NULL.  In the partitioned NCCL mode P is the local row segment and Q is the full matrix (collective:
 * every rank must call).  Factors that do not exist yet are created first (A-7 init); MF_EINVAL for a null
 * context; MF_ECUDA on copy failures. */
int mf_get_factors(mf_ctx *ctx, float *P, float *Q);

/* Overwrite factors from fp32 host/device buffers (rounded to storage, RNE); either may be NULL. */
int mf_set_factors(mf_ctx *ctx, const float *P, const float *Q);

/* The processing order: perm[i] = index (into the arrays given to mf_load_coo) of the i-th stored
 * sample.  perm is a caller-allocated host array of nnz int64. */
int mf_get_order(const mf_ctx *ctx, int64_t *perm);

/* Number of waves of the deterministic layout (builds it if needed). */
int mf_wave_count(mf_ctx *ctx, int64_t *out);

/* Multi-GPU (MF_SCHED_PARTITIONED over NCCL).  Rank 0 calls mf_nccl_unique_id (128 bytes), the caller
 * broadcasts the bytes (e.g. torch.distributed), then every rank calls mf_attach_nccl before loading. */
int mf_nccl_unique_id(void *out128);
int mf_attach_nccl(mf_ctx *ctx, const void *id128, int rank, int world);

/* Host-only helpers of the partitioned schedule (no device needed):
 * row segment of rank g among G: [seg_begin, seg_end) = [floor(g*m/G), floor((g+1)*m/G));
 * an epoch e is S passes (MF_OPT_SUBEPOCHS) over consecutive slices of the shuffled samples, pass
 * index p = e*S + s.  In round r of pass p rank g holds column segment sigma_p(g, r) =
 * pi_p((g + r) mod G), pi_p a permutation drawn from `seed` (the context's shuffle seed): a Latin
 * square, so the blocks of one round share no row or column segment. */
int mf_segment(int64_t extent, int32_t parts, int32_t index, int64_t *begin, int64_t *end);
int mf_round_segment(uint64_t seed, int32_t pass, int32_t G, int32_t round, int32_t rank, int32_t *col_segment);
/* Unit grid (MF_OPT_PART_SPLIT = 2): the segment c whose half `half` (0 lower rows [0, len/2), 1 upper) partition
 * `rank` updates in `round` of `pass`; half 0 equals mf_round_segment.  Host-only.  MF_EINVAL on out-of-range input. */
int mf_round_unit(uint64_t seed, int32_t pass, int32_t G, int32_t round, int32_t rank, int32_t half, int32_t *col_segment);
/* Peers of partition `rank` for the Q exchange after round `round` of pass `pass` (the last round hands
 * over to round 0 of pass+1): it sends its segment to *send_to and receives from *recv_from. */
int mf_round_peers(uint64_t seed, int32_t pass, int32_t G, int32_t round, int32_t rank, int32_t *send_to,
                   int32_t *recv_from);
/* The same for the unit of family `half` under the unit grid (half 0 equals mf_round_peers). */
int mf_unit_peers(uint64_t seed, int32_t pass, int32_t G, int32_t round, int32_t rank, int32_t half, int32_t *send_to,
                  int32_t *recv_from);
/* The paper's Hogwild! feasibility rule (§5.5.1): with s concurrent workers on an i x j
 * block grid of an m x n matrix, convergence was observed only for s < min(floor(m/i), floor(n/j)) /
 * safety (safety = 20 in the paper: Hugewiki, min(m, n) = 40k, s = 768 converges at j = 2, fails at
 * j = 4).  Returns 1 (pass) or 0 (fail) and the bound in *bound; MF_EINVAL (< 0) for non-positive
 * arguments.  Advisory only: the library's default worker count is DESIGN.md reading A-10 (every worker
 * processes >= 10^4 samples per epoch), which measured parity holds for where this rule fails (the
 * Netflix shape: s = 9,472 against a bound of 888, test RMSE within 0.035% of serial SGD). */
int mf_feasibility(int64_t m, int64_t n, int32_t i, int32_t j, int64_t s, int32_t safety, int64_t *bound);

/* Wavefront audit (MF_OPT_TRACE=1): copies up to cap records of 4 int64 (worker, block, t_start, t_end
 * in globaltimer ns) from the last wavefront epoch; *count = records written. */
int mf_wavefront_trace(mf_ctx *ctx, int64_t *records, int64_t cap, int64_t *count);

void mf_destroy(mf_ctx *ctx);
const char *mf_last_error(const mf_ctx *ctx);
const char *mf_status_string(int status);

#ifdef __cplusplus
}
#endif
#endif /* MF_H */
