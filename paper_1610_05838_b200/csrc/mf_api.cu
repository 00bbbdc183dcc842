// mf_api.cu -- host side of the C ABI declared in include/mf.h.
//
// Owns the context (device buffers, stream, options), the data layout steps
// that run once per load (validation, A-8 shuffle, deterministic wave layout)
// and the per-epoch dispatch to the kernels in mf_kernels.cu / mf_wavefront.cu
// / mf_partition.cu.  All numerical work happens on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/mf.h"
#include "mf_ctx.h"
#include "mf_kernels.cuh"

using namespace mf;

// ------------------------------------------------------------------ errors --
int mf_ctx::fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return code;
}

int mf_ctx::cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return MF_OK;
    cudaGetLastError();  // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation) return fail(MF_ENOMEM, "%s: %s", what, cudaGetErrorString(e));
    return fail(MF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(expr)                                                  \
    do {                                                          \
        int _rc = ctx->cuda((expr), #expr);                       \
        if (_rc != MF_OK) return _rc;                             \
    } while (0)
#define RC(expr)                 \
    do {                         \
        int _rc = (expr);        \
        if (_rc != MF_OK) return _rc; \
    } while (0)

template <class T>
static int dev_alloc(mf_ctx *ctx, T **p, size_t count, const char *what) {
    if (*p) return MF_OK;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void **)p, sizeof(T) * count);
    if (e != cudaSuccess) {
        *p = nullptr;
        return ctx->cuda(e, what);
    }
    return MF_OK;
}
template <class T>
static void dev_free(T **p) {
    if (*p) cudaFree((void *)*p);
    *p = nullptr;
}

static bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int mf_ctx::storage_bytes() const { return storage == kF32 ? 4 : 2; }

// ------------------------------------------------------------ device setup --
int mf_ctx::ensure_device() {
    if (dev_ready) return MF_OK;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(MF_ECUDA, "no CUDA device available (%s); there is no CPU fallback",
                    e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    }
    if (device < 0 || device >= ndev) return fail(MF_EINVAL, "device %d out of range (%d devices)", device, ndev);
    mf_ctx *ctx = this;
    CK(cudaSetDevice(device));
    if (!user_stream) {
        CK(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
    }
    CK(cudaMalloc((void **)&scratch, sizeof(DevScratch)));
    CK(cudaMemset(scratch, 0, sizeof(DevScratch)));
    CK(cudaMallocHost((void **)&h_scratch, sizeof(DevScratch)));
    for (auto &ev : events) CK(cudaEventCreate(&ev));
    CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
    {  // keep stream-ordered allocations cached instead of unmapping them at every synchronisation
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    dev_ready = true;
    return MF_OK;
}

cudaStream_t mf_ctx::stream() const { return user_stream ? user_stream : own_stream; }

int mf_ctx::ensure_factors() {
    if ((P || p_host) && Q) return MF_OK;
    RC(ensure_device());
    mf_ctx *ctx = this;
    CK(cudaSetDevice(device));
    const size_t b = (size_t)storage_bytes();
    const int64_t prow = p_rows();
    if (!p_host) RC(dev_alloc(this, (char **)&P, b * (size_t)prow * k, "alloc P"));
    RC(dev_alloc(this, (char **)&Q, b * (size_t)n * k, "alloc Q"));
    // A-7 init; in the partitioned NCCL mode P holds rows [p_begin, p_end) of the global P:
    // the hash index is the global row*k+col, so shift the row origin.  With MF_OPT_P_HOST the caller
    // owns P (mf_init_rows_host gives the same values).
    if (!p_host) CK(launch_init_rows(storage, P, p_begin, prow, k, seed, 0, stream()));
    CK(launch_init_rows(storage, Q, 0, n, k, seed, 1, stream()));
    CK(cudaStreamSynchronize(stream()));
    return MF_OK;
}

// init for rows [row0, row0+rows) stored from X[0]
cudaError_t mf::launch_init_rows(int storage, void *X, int64_t row0, int64_t rows, int k, uint64_t seed, uint32_t tag,
                                 cudaStream_t st) {
    return launch_init_offset(storage, X, row0 * (int64_t)k, rows * (int64_t)k, k, seed, tag, st);
}

void mf_ctx::drop_layouts() {
    dev_free(&wu);
    dev_free(&wv);
    dev_free(&wr);
    dev_free(&wave_off);
    dev_free(&ord_u);
    dev_free(&ord_v);
    dev_free(&cnt_uv);
    nwaves = -1;
    wf_valid = false;
    part_valid = false;
}

// Each schedule other than batch-Hogwild! keeps its own reordered copy of R (12 B per sample: wave
// order, wavefront blocks, partition blocks).  Only the schedule being run keeps its copy, so the
// footprint is at most two copies of R (the stored order + one layout) whatever the call sequence.
int mf_ctx::drop_other_layouts(int schedule) {
    if (schedule != MF_SCHED_DETERMINISTIC && wu) {
        dev_free(&wu);
        dev_free(&wv);
        dev_free(&wr);
        dev_free(&wave_off);
        dev_free(&ord_u);
        dev_free(&ord_v);
        dev_free(&cnt_uv);
        nwaves = -1;
    }
    if (schedule != MF_SCHED_WAVEFRONT && fu) release_wavefront();
    if (schedule != MF_SCHED_PARTITIONED && bu && !is_distributed()) {
        const int rc = gather_q();  // the partitioned layout may hold the current Q in its segments
        if (rc != MF_OK) return rc;
        for (void *p : {(void *)bu, (void *)bv, (void *)br})
            if (p) cudaFree(p);
        bu = bv = nullptr;
        br = nullptr;
        part_valid = false;
    }
    return MF_OK;
}

void mf_ctx::release() {
    if (dev_ready) cudaSetDevice(device);
    drop_layouts();
    dev_free(&u);
    dev_free(&v);
    dev_free(&r);
    dev_free(&perm);
    dev_free(&tu);
    dev_free(&tv);
    dev_free(&tr);
    dev_free(&partials);
    dev_free(&d_out);
    dev_free(&f32_tmp);
    if (P) cudaFree(P);
    if (Q) cudaFree(Q);
    P = Q = nullptr;
    release_wavefront();
    release_partition();
    release_stream();
    release_outcore();
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    if (h_scratch) cudaFreeHost(h_scratch);
    h_scratch = nullptr;
    for (auto &ev : events)
        if (ev) cudaEventDestroy(ev), ev = nullptr;
    if (own_stream) cudaStreamDestroy(own_stream);
    own_stream = nullptr;
    dev_ready = false;
}

// ------------------------------------------------------------ public: create
extern "C" int mf_create(int64_t m, int64_t n, int32_t k, float lr, float lambda, uint64_t seed, mf_ctx **out) {
    if (!out) return MF_EINVAL;
    *out = nullptr;
    if (m <= 0 || n <= 0 || m >= (1ll << 31) || n >= (1ll << 31) || k <= 0 || k > 1024) return MF_EINVAL;
    if (!(lr > 0.f) || !std::isfinite(lr) || !(lambda >= 0.f) || !std::isfinite(lambda)) return MF_EINVAL;
    mf_ctx *c = new (std::nothrow) mf_ctx();
    if (!c) return MF_ENOMEM;
    c->m = m;
    c->n = n;
    c->k = k;
    c->alpha = lr;
    c->lambda = lambda;
    c->seed = seed;
    c->seed_shuffle = seed;
    c->p_begin = 0;
    c->p_end = m;
    *out = c;
    return MF_OK;
}

extern "C" void mf_destroy(mf_ctx *ctx) {
    if (!ctx) return;
    ctx->release();
    delete ctx;
}

extern "C" const char *mf_last_error(const mf_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

extern "C" const char *mf_status_string(int s) {
    switch (s) {
        case MF_OK: return "MF_OK";
        case MF_EINVAL: return "MF_EINVAL";
        case MF_ENOMEM: return "MF_ENOMEM";
        case MF_ECUDA: return "MF_ECUDA";
        case MF_ESTATE: return "MF_ESTATE";
        case MF_EDIVERGED: return "MF_EDIVERGED";
        case MF_ENCCL: return "MF_ENCCL";
        default: return "MF_UNKNOWN";
    }
}

extern "C" int mf_set_option(mf_ctx *ctx, int key, double value) {
    if (!ctx) return MF_EINVAL;
    if (!std::isfinite(value)) return ctx->fail(MF_EINVAL, "option %d: non-finite value", key);
    const int64_t iv = (int64_t)value;
    switch (key) {
        case MF_OPT_STORAGE:
            if (iv < 0 || iv > 2) return ctx->fail(MF_EINVAL, "storage must be 0 (fp32), 1 (fp16) or 2 (bf16)");
            if (ctx->P && iv != ctx->storage) return ctx->fail(MF_ESTATE, "storage must be set before the factors exist");
            ctx->storage = (int)iv;
            return MF_OK;
        case MF_OPT_BETA:
            if (value < 0) return ctx->fail(MF_EINVAL, "beta must be >= 0");
            ctx->beta = value;
            return MF_OK;
        case MF_OPT_WORKERS:
            if (iv < 0) return ctx->fail(MF_EINVAL, "workers must be >= 0");
            ctx->workers = (int)std::min<int64_t>(iv, 1 << 30);
            return MF_OK;
        case MF_OPT_BATCH_F:
            if (iv < 32 || iv % 32 || iv > (1 << 24)) return ctx->fail(MF_EINVAL, "batch f must be a positive multiple of 32");
            ctx->batch_f = (int)iv;
            return MF_OK;
        case MF_OPT_WAVE_ROWS:
            if (iv < 0) return ctx->fail(MF_EINVAL, "wave rows must be >= 0");
            ctx->wave_rows = (int)iv;
            ctx->wf_valid = false;
            return MF_OK;
        case MF_OPT_WAVE_COLS:
            if (iv < 0) return ctx->fail(MF_EINVAL, "wave cols must be >= 0");
            ctx->wave_cols = (int)iv;
            ctx->wf_valid = false;
            return MF_OK;
        case MF_OPT_DEVICE:
            if (ctx->dev_ready && iv != ctx->device) return ctx->fail(MF_ESTATE, "device must be set before first use");
            ctx->device = (int)iv;
            return MF_OK;
        case MF_OPT_STREAM:
            ctx->user_stream = (cudaStream_t)(uintptr_t)iv;
            return MF_OK;
        case MF_OPT_SHUFFLE:
            if (iv < 0 || iv > 2) return ctx->fail(MF_EINVAL, "shuffle must be 0, 1 or 2");
            ctx->shuffle = (int)iv;
            return MF_OK;
        case MF_OPT_COUNT_UPDATES:
            ctx->count_updates = iv ? 1 : 0;
            return MF_OK;
        case MF_OPT_WAVE_PERM:
            if (iv < 0 || iv > 1) return ctx->fail(MF_EINVAL, "wave perm must be 0 (latin) or 1 (random)");
            ctx->wave_perm = (int)iv;
            return MF_OK;
        case MF_OPT_EPOCH:
            if (iv < 0) return ctx->fail(MF_EINVAL, "epoch must be >= 0");
            ctx->epoch = (int32_t)iv;
            return MF_OK;
        case MF_OPT_PARTITIONS:
            if (iv < 0 || iv > 1024) return ctx->fail(MF_EINVAL, "partitions must be in [0, 1024]");
            ctx->partitions = (int)iv;
            ctx->part_valid = false;
            return MF_OK;
        case MF_OPT_SEED_SHUFFLE:
            ctx->seed_shuffle = (uint64_t)value;
            return MF_OK;
        case MF_OPT_VARIANT:
            ctx->variant = (int)iv;
            ctx->pf_hogwild.reset(), ctx->pf_wave_cta.reset(), ctx->last_pf_pick = 0;
            return MF_OK;
        case MF_OPT_TRACE:
            ctx->trace = iv ? 1 : 0;
            return MF_OK;
        case MF_OPT_SUBEPOCHS:
            if (iv < 0 || iv > 4096) return ctx->fail(MF_EINVAL, "subepochs must be in [0 (auto), 4096]");
            ctx->subepochs = (int)iv;
            ctx->part_valid = false;
            return MF_OK;
        case MF_OPT_WAVE_CTA:
            if (iv < 0 || iv > 3) return ctx->fail(MF_EINVAL, "wave cta must be 0, 1, 2 or 3");
            ctx->wave_cta = (int)iv;
            ctx->wf_valid = false;
            return MF_OK;
        case MF_OPT_PART_SPLIT:
            if (iv < 0 || iv > 2) return ctx->fail(MF_EINVAL, "part split must be 0, 1 or 2");
            ctx->part_split = (int)iv;
            ctx->part_valid = false;
            return MF_OK;
        case MF_OPT_WAVE_PASSES:
            if (iv < 0 || iv > 4096) return ctx->fail(MF_EINVAL, "wave passes must be in [0 (auto), 4096]");
            ctx->wave_passes = (int)iv;
            ctx->wf_valid = false;
            return MF_OK;
        case MF_OPT_P_HOST:
            if (iv < 0 || iv > 1) return ctx->fail(MF_EINVAL, "P host must be 0 or 1");
            if (ctx->Q || ctx->P) return ctx->fail(MF_ESTATE, "MF_OPT_P_HOST must be set before the factors exist");
            ctx->p_host = (int)iv;
            return MF_OK;
        case MF_OPT_DET_FLOW:
            if (iv < 0 || iv > 1) return ctx->fail(MF_EINVAL, "det flow must be 0 (waves) or 1 (row counters)");
            ctx->det_flow = (int)iv;
            return MF_OK;
        case MF_OPT_Q_UPDATE:
            if (iv < 0 || iv > 2) return ctx->fail(MF_EINVAL, "Q update must be 0 (store), 1 (atomic add) or 2 (auto)");
            ctx->q_update = (int)iv;
            return MF_OK;
        case MF_OPT_R_STAGING:
            if (iv < 1 || iv > 2) return ctx->fail(MF_EINVAL, "R staging must be 1 (registers) or 2 (TMA)");
            ctx->r_stage = (int)iv;
            return MF_OK;
        case MF_OPT_STREAM_CHUNK:
            if (iv < 32 || iv > (1ll << 34)) return ctx->fail(MF_EINVAL, "stream chunk must be in [32, 2^34]");
            ctx->stream_chunk = iv;
            return MF_OK;
        default:
            return ctx->fail(MF_EINVAL, "unknown option %d", key);
    }
}

extern "C" int mf_get_option(const mf_ctx *ctx, int key, double *value) {
    if (!ctx || !value) return MF_EINVAL;
    switch (key) {
        case MF_OPT_STORAGE: *value = ctx->storage; return MF_OK;
        case MF_OPT_BETA: *value = ctx->beta; return MF_OK;
        case MF_OPT_WORKERS: *value = ctx->workers; return MF_OK;
        case MF_OPT_BATCH_F: *value = ctx->batch_f; return MF_OK;
        case MF_OPT_WAVE_ROWS: *value = ctx->wave_rows ? ctx->wave_rows : ctx->wf_s; return MF_OK;  // effective
        case MF_OPT_WAVE_COLS: *value = ctx->wave_cols ? ctx->wave_cols : ctx->wf_c; return MF_OK;
        case MF_OPT_DEVICE: *value = ctx->device; return MF_OK;
        case MF_OPT_STREAM: *value = (double)(uintptr_t)ctx->user_stream; return MF_OK;
        case MF_OPT_SHUFFLE: *value = ctx->shuffle; return MF_OK;
        case MF_OPT_COUNT_UPDATES: *value = ctx->count_updates; return MF_OK;
        case MF_OPT_WAVE_PERM: *value = ctx->wave_perm; return MF_OK;
        case MF_OPT_EPOCH: *value = ctx->epoch; return MF_OK;
        case MF_OPT_PARTITIONS: *value = ctx->partitions; return MF_OK;
        case MF_OPT_SEED_SHUFFLE: *value = (double)ctx->seed_shuffle; return MF_OK;
        case MF_OPT_VARIANT:  // the variant in effect: an auto prefetch field reports the setting picked
            *value = ((ctx->variant >> 16) & 0xF) == 0 && ctx->last_pf_pick ? ctx->variant | (ctx->last_pf_pick << 16)
                                                                           : ctx->variant;
            return MF_OK;
        case MF_OPT_TRACE: *value = ctx->trace; return MF_OK;
        case MF_OPT_SUBEPOCHS: *value = ctx->subepochs ? ctx->subepochs : ctx->part_S; return MF_OK;
        case MF_OPT_WAVE_CTA: *value = ctx->wave_cta; return MF_OK;
        case MF_OPT_STREAM_CHUNK: *value = (double)ctx->stream_chunk; return MF_OK;
        case MF_OPT_PART_SPLIT: *value = ctx->part_split; return MF_OK;
        case MF_OPT_R_STAGING: *value = ctx->r_stage; return MF_OK;
        case MF_OPT_WAVE_PASSES: *value = ctx->wf_valid ? ctx->wf_p : ctx->wave_passes; return MF_OK;
        case MF_OPT_P_HOST: *value = ctx->p_host; return MF_OK;
        case MF_OPT_Q_UPDATE: *value = ctx->q_update; return MF_OK;
        case MF_OPT_DET_FLOW: *value = ctx->det_flow; return MF_OK;
        case MF_OPT_Q_KAPPA: *value = ctx->last_kappa; return MF_OK;
        default: return MF_EINVAL;
    }
}

// ---------------------------------------------------------------- load_coo --
// Copy in (host or device source), validate on the device, permute (A-8),
// store SoA.  Buffers are reused when nnz does not change (repeated loads in
// the end-to-end benchmark allocate nothing).
extern "C" int mf_load_coo(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz) {
    if (!ctx) return MF_EINVAL;
    if (!u || !v || !r || nnz <= 0) return ctx->fail(MF_EINVAL, "mf_load_coo: null pointer or nnz <= 0");
    if (ctx->shuffle && nnz > (int64_t)0xFFFFFFFFll)
        return ctx->fail(MF_EINVAL, "mf_load_coo: shuffle supports nnz < 2^32");
    RC(ctx->ensure_device());
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream();
    if (nnz != ctx->cap_n) {  // (re)allocate; buffers are reused by repeated loads of the same size
        for (void **p : {(void **)&ctx->u, (void **)&ctx->v, (void **)&ctx->r, (void **)&ctx->perm})
            if (*p) cudaFree(*p), *p = nullptr;
        ctx->cap_n = 0;
        ctx->perm_n = -1;
        RC(ctx->gather_q());
        ctx->drop_layouts();  // free cached schedule copies of R before the new arrays
        RC(dev_alloc(ctx, &ctx->u, nnz, "alloc u"));
        RC(dev_alloc(ctx, &ctx->v, nnz, "alloc v"));
        RC(dev_alloc(ctx, &ctx->r, nnz, "alloc r"));
        ctx->cap_n = nnz;
    }
    RC(ctx->gather_q());
    ctx->drop_layouts();
    ctx->pf_hogwild.reset(), ctx->pf_wave_cta.reset(), ctx->last_pf_pick = 0;  // a new workload re-runs the trials
    ctx->seg_valid = false;
    ctx->N = 0;
    // Footprint (peak bytes per sample besides the caller's data): the A-8 permutation is computed
    // first (64-bit keys double-buffered + indices: 24 B transient, 4 B kept for mf_get_order and
    // repeated loads), then host inputs pass through a transient 12-B staging copy (device inputs are
    // gathered straight from the caller's buffers): at most 12 (R) + 4 + 24 = 40 B per sample, i.e.
    // 123 GB for the 3.07B-sample Hugewiki shape next to its 12.8-GB fp16 P.
    if (ctx->shuffle && !(ctx->perm_n == nnz && ctx->perm_seed == ctx->seed_shuffle)) {
        // the A-8 permutation depends only on (nnz, seed): computed once and cached
        RC(dev_alloc(ctx, &ctx->perm, nnz, "alloc perm"));
        CK(launch_shuffle_perm(nnz, ctx->seed_shuffle, ctx->perm, st));
        ctx->perm_n = nnz;
        ctx->perm_seed = ctx->seed_shuffle;
    }
    const bool dev_in = is_device_ptr(u) && is_device_ptr(v) && is_device_ptr(r);
    const cudaMemcpyKind kind = dev_in ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // shuffle: one fused gather + validate + rebase kernel writes the A-8 order from the caller's device
    // buffers or a transient staging copy of the host ones; no shuffle: copy in place and run the same
    // kernel as validate + rebase.
    const int32_t *su = u, *sv = v;
    const float *sr = r;
    int32_t *tmp_u = nullptr, *tmp_v = nullptr;
    float *tmp_r = nullptr;
    if (!ctx->shuffle) {
        CK(cudaMemcpyAsync(ctx->u, u, sizeof(int32_t) * nnz, kind, st));
        CK(cudaMemcpyAsync(ctx->v, v, sizeof(int32_t) * nnz, kind, st));
        CK(cudaMemcpyAsync(ctx->r, r, sizeof(float) * nnz, kind, st));
        su = ctx->u, sv = ctx->v, sr = ctx->r;
    } else if (!dev_in) {
        CK(cudaMallocAsync((void **)&tmp_u, sizeof(int32_t) * nnz, st));
        CK(cudaMallocAsync((void **)&tmp_v, sizeof(int32_t) * nnz, st));
        CK(cudaMallocAsync((void **)&tmp_r, sizeof(float) * nnz, st));
        CK(cudaMemcpyAsync(tmp_u, u, sizeof(int32_t) * nnz, kind, st));
        CK(cudaMemcpyAsync(tmp_v, v, sizeof(int32_t) * nnz, kind, st));
        CK(cudaMemcpyAsync(tmp_r, r, sizeof(float) * nnz, kind, st));
        su = tmp_u, sv = tmp_v, sr = tmp_r;
    }
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(DevScratch), st));
    CK(launch_gather_validate(su, sv, sr, ctx->shuffle ? ctx->perm : nullptr, nnz, ctx->p_begin, ctx->p_end, ctx->n,
                              ctx->u, ctx->v, ctx->r, ctx->scratch, st));
    for (void *p : {(void *)tmp_u, (void *)tmp_v, (void *)tmp_r})
        if (p) CK(cudaFreeAsync(p, st));
    CK(cudaMemcpyAsync(ctx->h_scratch, ctx->scratch, sizeof(DevScratch), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (ctx->h_scratch->bad)
        return ctx->fail(MF_EINVAL, "mf_load_coo: %llu samples with u outside [%lld,%lld), v outside [0,%lld) or non-finite r",
                         (unsigned long long)ctx->h_scratch->bad, (long long)ctx->p_begin, (long long)ctx->p_end,
                         (long long)ctx->n);
    ctx->N = nnz;
    {  // sum_v (deg v / N)^2: the Q-row collision rate per Hogwild! worker (MF_OPT_Q_UPDATE auto, A-20)
        unsigned *deg = nullptr;
        double *d_sq = nullptr, h_sq = 0;
        CK(cudaMallocAsync((void **)&deg, sizeof(unsigned) * (size_t)(ctx->n + 2) + sizeof(double), st));
        d_sq = reinterpret_cast<double *>(deg + ((ctx->n + 1) & ~1ll));  // 8-B aligned after the histogram
        CK(launch_col_sq(ctx->v, nnz, ctx->n, deg, d_sq, st));
        CK(cudaMemcpyAsync(&h_sq, d_sq, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(deg, st));
        CK(cudaStreamSynchronize(st));
        ctx->col_sq = nnz > 0 ? h_sq / ((double)nnz * (double)nnz) : 0.0;
    }
    ctx->reshuffle_due = false;  // the first epoch after a load uses the load's order
    ctx->shuffled = ctx->shuffle;
    RC(ctx->ensure_factors());
    return MF_OK;
}

// Per-epoch reshuffle (MF_OPT_SHUFFLE = 2): before epoch t (t >= 1 after a load) the stored order is
// permuted again by the A-8 hash sort keyed with seed_shuffle ^ (t << 48):
//     order_t = order_{t-1}[pi_t],  pi_t = A-8 permutation of N under that seed,
// so the caller-index map stays available through mf_get_order.  Schedule layouts are rebuilt.
int mf_ctx::reshuffle() {
    mf_ctx *ctx = this;
    cudaStream_t st = stream();
    uint32_t *p2 = nullptr, *p3 = nullptr;
    int32_t *nu = nullptr, *nv = nullptr;
    float *nr = nullptr;
    CK(cudaMallocAsync((void **)&p2, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&p3, sizeof(uint32_t) * N, st));
    CK(launch_shuffle_perm(N, seed_shuffle ^ ((uint64_t)(uint32_t)epoch << 48), p2, st));
    CK(launch_compose(perm, p2, p3, N, st));
    CK(cudaMemcpyAsync(perm, p3, sizeof(uint32_t) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaFreeAsync(p3, st));
    // gather into transient arrays, then back into the resident ones (no second resident copy of R)
    CK(cudaMallocAsync((void **)&nu, sizeof(int32_t) * N, st));
    CK(cudaMallocAsync((void **)&nv, sizeof(int32_t) * N, st));
    CK(cudaMallocAsync((void **)&nr, sizeof(float) * N, st));
    CK(launch_gather(u, v, r, p2, N, nu, nv, nr, st));
    CK(cudaMemcpyAsync(u, nu, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(v, nv, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(r, nr, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
    for (void *p : {(void *)p2, (void *)nu, (void *)nv, (void *)nr}) CK(cudaFreeAsync(p, st));
    perm_n = -1;  // perm no longer equals the load-time permutation
    RC(gather_q());
    drop_layouts();
    seg_valid = false;
    CK(cudaStreamSynchronize(st));
    return MF_OK;
}

// -------------------------------------------------------------- wave layout --
// DESIGN.md D-3: scanning samples in stored (shuffled) order,
// wave(i) = max(last[u_i], last[v_i]) + 1, last[] = -1 initially.  Samples are
// then stably bucketed by wave; inside a wave no two share a row or column.
int mf_ctx::build_waves() {
    if (nwaves >= 0 && (!det_flow || ord_u)) return MF_OK;
    if (nwaves >= 0) {  // the wave layout exists without the dataflow ordinals: rebuild both
        dev_free(&wu);
        dev_free(&wv);
        dev_free(&wr);
        dev_free(&wave_off);
        nwaves = -1;
    }
    mf_ctx *ctx = this;
    cudaStream_t st = stream();
    std::vector<int32_t> hu((size_t)N), hv((size_t)N);
    CK(cudaMemcpyAsync(hu.data(), u, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hv.data(), v, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<int32_t> wave((size_t)N);
    int64_t nw = 0;
    {
        std::vector<int32_t> lu((size_t)p_rows(), -1), lv((size_t)n, -1);
        for (int64_t i = 0; i < N; i++) {
            const int32_t a = hu[(size_t)i], b = hv[(size_t)i];
            const int32_t w = std::max(lu[(size_t)a], lv[(size_t)b]) + 1;
            wave[(size_t)i] = w;
            lu[(size_t)a] = w;
            lv[(size_t)b] = w;
            if (w + 1 > nw) nw = w + 1;
        }
    }
    std::vector<int64_t> off((size_t)nw + 1, 0);
    for (int64_t i = 0; i < N; i++) off[(size_t)wave[(size_t)i] + 1]++;
    for (int64_t w = 0; w < nw; w++) off[(size_t)w + 1] += off[(size_t)w];
    std::vector<uint32_t> idx((size_t)N);
    {
        std::vector<int64_t> pos(off.begin(), off.end() - 1);
        for (int64_t i = 0; i < N; i++) idx[(size_t)pos[(size_t)wave[(size_t)i]]++] = (uint32_t)i;
    }
    uint32_t *didx = nullptr;
    RC(dev_alloc(this, &wu, N, "alloc wave u"));
    RC(dev_alloc(this, &wv, N, "alloc wave v"));
    RC(dev_alloc(this, &wr, N, "alloc wave r"));
    RC(dev_alloc(this, &wave_off, nw + 1, "alloc wave offsets"));
    CK(cudaMallocAsync((void **)&didx, sizeof(uint32_t) * N, st));
    CK(cudaMemcpyAsync(didx, idx.data(), sizeof(uint32_t) * N, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(wave_off, off.data(), sizeof(int64_t) * (nw + 1), cudaMemcpyHostToDevice, st));
    CK(launch_gather(u, v, r, didx, N, wu, wv, wr, st));
    CK(cudaFreeAsync(didx, st));
    if (det_flow) {
        // ordinals of each sample's update of its row and of its column in the serial (stored) order,
        // written in wave order: a row's updates keep their serial order in the wave layout (waves
        // increase along a row), so k_flow runs them in that order by waiting for counter == ordinal
        std::vector<int32_t> ou((size_t)N), ov((size_t)N);
        {
            std::vector<int32_t> cnt_u((size_t)p_rows(), 0), cnt_v((size_t)n, 0);
            for (int64_t i = 0; i < N; i++) {  // stored order = serial order
                ou[(size_t)i] = cnt_u[(size_t)hu[(size_t)i]]++;
                ov[(size_t)i] = cnt_v[(size_t)hv[(size_t)i]]++;
            }
        }
        std::vector<int32_t> wou((size_t)N), wov((size_t)N);
        for (int64_t j = 0; j < N; j++) wou[(size_t)j] = ou[idx[(size_t)j]], wov[(size_t)j] = ov[idx[(size_t)j]];
        RC(dev_alloc(this, &ord_u, N, "alloc flow ordinals u"));
        RC(dev_alloc(this, &ord_v, N, "alloc flow ordinals v"));
        RC(dev_alloc(this, &cnt_uv, (size_t)(p_rows() + n), "alloc flow counters"));
        CK(cudaMemcpyAsync(ord_u, wou.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(ord_v, wov.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
    }
    CK(cudaStreamSynchronize(st));
    nwaves = nw;
    return MF_OK;
}

extern "C" int mf_wave_count(mf_ctx *ctx, int64_t *out) {
    if (!ctx || !out) return MF_EINVAL;
    if (ctx->N <= 0) return ctx->fail(MF_ESTATE, "mf_wave_count before mf_load_coo");
    RC(ctx->build_waves());
    *out = ctx->nwaves;
    return MF_OK;
}

// ------------------------------------------------------------------- epoch --
float mf_ctx::eta_at(int32_t t) const {
    // s_t = alpha / (1 + beta t^1.5) in double, then fp32 (A-5)
    return (float)((double)alpha / (1.0 + beta * std::pow((double)t, 1.5)));
}

// batch-Hogwild!'s group shape (MF_OPT_VARIANT bits 0..3; 0 = auto).  16-bit rows at k = 128 take one rating
// per warp (32 lanes x 8 B) by default; where P is far larger than the L2 (> 2x) and Q small (< 1/4 of it), the
// update waits on DRAM for p_u and more ratings in flight pay: the 8-lane shape (4 ratings per warp, 14,208 in
// flight at full residency) is 3-4% faster on the Hugewiki shapes (full, rows/10, the partitioned kernels)
// and is taken there; not on the Yahoo shape, whose Q misses L2 too (profiles/r02ap_*, r02aq_*).
int mf_ctx::hog_shape_sel() const {
    if (variant & 0xF) return variant & 0xF;
    if (k != 128 || storage == kF32) return 0;
    static const int64_t l2 = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
        return (int64_t)v;
    }();
    const int64_t row = (int64_t)k * storage_bytes();
    return (l2 > 0 && p_rows() * row > 2 * l2 && n * row < l2 / 4) ? 1 : 0;
}

int mf_ctx::auto_workers() const {
    // DESIGN.md A-10: every worker processes >= 10^4 samples per epoch
    return (int)std::max<int64_t>(1, std::min<int64_t>(N / 10000, 1 << 30));
}

UpdateArgs mf_ctx::update_args(float eta) const {
    UpdateArgs a{};
    a.u = u;
    a.v = v;
    a.r = r;
    a.n = N;
    a.P = P;
    a.Q = Q;
    a.k = k;
    a.eta = eta;
    a.lam = lambda;
    a.batch_f = batch_f;
    a.count_updates = count_updates;
    a.scratch = scratch;
    a.r_stage = r_stage;
    a.q_mode = q_update;
    a.q_share = (float)(col_sq > 0 ? col_sq : 1.0 / (double)n);  // before a load: uniform columns
    return a;
}

int mf_ctx::finish_epoch(int schedule, float eta, int launches, int workers_used, mf_epoch_stats *stats) {
    mf_ctx *ctx = this;
    cudaStream_t st = stream();
    CK(cudaEventRecord(events[3], st));
    CK(cudaMemcpyAsync(h_scratch, scratch, sizeof(DevScratch), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    float ms_all = 0.f, ms_k = 0.f;
    CK(cudaEventElapsedTime(&ms_all, events[0], events[3]));
    CK(cudaEventElapsedTime(&ms_k, events[1], events[2]));
    last_kernel_ms = ms_k;
    const int32_t t = epoch;
    epoch++;
    if (stats) {
        stats->updates = count_updates ? (int64_t)h_scratch->updates : N;
        stats->seconds = ms_all * 1e-3;
        stats->kernel_seconds = ms_k * 1e-3;
        stats->lr = eta;
        stats->epoch = t;
        stats->workers = workers_used;
        stats->launches = launches;
    }
    (void)schedule;
    if (h_scratch->diverged & 2) return fail(MF_ECUDA, "deterministic dataflow: a rating waited > 2 s in epoch %d", (int)t);
    if (h_scratch->diverged) return fail(MF_EDIVERGED, "non-finite prediction error in epoch %d", (int)t);
    return MF_OK;
}

static int epoch_local(mf_ctx *ctx, int schedule, mf_epoch_stats *stats);

extern "C" int mf_epoch(mf_ctx *ctx, int schedule, mf_epoch_stats *stats) {
    if (ctx && ctx->p_host) return ctx->fail(MF_ESTATE, "P lives in caller memory (MF_OPT_P_HOST): use mf_epoch_host_blocks");
    if (!ctx) return MF_EINVAL;
    if (!ctx->is_distributed()) return epoch_local(ctx, schedule, stats);
    // collective: a precondition failure on any rank is agreed before the exchange rounds start, and
    // the outcome (e.g. divergence on one rank) after they end
    int pre = MF_OK;
    if (schedule != MF_SCHED_PARTITIONED)
        pre = ctx->fail(MF_EINVAL, "with NCCL attached only MF_SCHED_PARTITIONED is available");
    else if (ctx->N <= 0 || !ctx->P)
        pre = ctx->fail(MF_ESTATE, "mf_epoch before mf_load_coo");
    RC(ctx->agree(pre));
    CK(cudaSetDevice(ctx->device));
    return ctx->agree(ctx->epoch_partitioned(stats));
}

static int epoch_local(mf_ctx *ctx, int schedule, mf_epoch_stats *stats) {
    if (schedule < MF_SCHED_HOGWILD || schedule > MF_SCHED_PARTITIONED)
        return ctx->fail(MF_EINVAL, "unknown schedule %d", schedule);
    if (ctx->N <= 0 || !ctx->P) return ctx->fail(MF_ESTATE, "mf_epoch before mf_load_coo");
    CK(cudaSetDevice(ctx->device));
    if (ctx->shuffle == 2 && ctx->shuffled) {  // per-epoch reshuffle (SPEC.md:264 reading; NEXT-4)
        if (ctx->reshuffle_due) RC(ctx->reshuffle());
        ctx->reshuffle_due = true;
    }
    RC(ctx->drop_other_layouts(schedule));
    if (schedule == MF_SCHED_DETERMINISTIC) RC(ctx->build_waves());
    if (schedule == MF_SCHED_WAVEFRONT) RC(ctx->build_wavefront());
    if (schedule == MF_SCHED_PARTITIONED) {
        ctx->last_kappa = 0;
        return ctx->epoch_partitioned(stats);
    }
    RC(ctx->gather_q());
    ctx->seg_valid = false;
    cudaStream_t st = ctx->stream();
    const float eta = ctx->eta_at(ctx->epoch);
    const ShapeId sh = schedule == MF_SCHED_HOGWILD ? hogwild_shape(ctx->k, ctx->storage, ctx->hog_shape_sel())
                                                    : select_shape(ctx->k, ctx->storage, ctx->variant & 0xF);
    CK(cudaEventRecord(ctx->events[0], st));
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(DevScratch), st));
    UpdateArgs a = ctx->update_args(eta);
    int launches = 1, used = 0;
    CK(cudaEventRecord(ctx->events[1], st));
    // auto L2 prefetch (mf_ctx::AutoPf): the setting tried when "on" -- batch-Hogwild!: the next
    // ratings' rows one step ahead (Yahoo shape +11%, Zipf-skewed Netflix +15%, Netflix / Hugewiki
    // shapes -6..-16%); CTA wavefront: a tile's P rows when it is claimed, per 128-B line for 16-bit
    // rows, one bulk prefetch per row for fp32 (+5..+13% on three shapes, -4% on a fourth)
    mf_ctx::AutoPf *tune = nullptr;
    int pf_on = 0, pf_slot = -1;
    ctx->variant_eff = ctx->variant;
    if (((ctx->variant >> 16) & 0xF) == 0) {
        if (schedule == MF_SCHED_HOGWILD) tune = &ctx->pf_hogwild, pf_on = 1;
        else if (schedule == MF_SCHED_WAVEFRONT && ctx->wave_cta && ctx->wave_cta != 3)
            tune = &ctx->pf_wave_cta, pf_on = ctx->storage == kF32 ? 1 : 2;
        if (tune) ctx->variant_eff |= tune->next(pf_on, &pf_slot) << 16;
    }
    if (schedule == MF_SCHED_HOGWILD) {
        const int w = ctx->workers > 0 ? ctx->workers : ctx->auto_workers();
        CK(launch_hogwild(sh, a, w, ctx->variant_eff, st, &used));
        ctx->last_kappa = (double)used * a.q_share;
    } else if (schedule == MF_SCHED_DETERMINISTIC) {
        a.u = ctx->wu;
        a.v = ctx->wv;
        a.r = ctx->wr;
        a.wave_off = ctx->wave_off;
        a.nwaves = ctx->nwaves;
        int l = 0;
        // MF_OPT_VARIANT bits 24..25: 0 = 1024-thread CTAs, 2 samples per group and step; 1 = one
        // sample; 2 = 256-thread CTAs and the fenced barrier (r01 form)
        const int wsel = (ctx->variant >> 24) & 0x3;
        // bits 22..23: grid barrier of the 1024-thread forms, 0 = arrival counter polled to its target,
        // 1 = generation flag bumped by the last arriver (r01c)
        a.barrier = ((ctx->variant >> 22) & 0x3) == 1 ? 1 : 0;
        // bits 24..25 = 3: two 512-thread CTAs per SM with four samples per group and step
        if (ctx->det_flow) {  // no barriers: per-row update counters (mf_flow.cu)
            a.ord_u = ctx->ord_u;
            a.ord_v = ctx->ord_v;
            a.cnt_u = ctx->cnt_uv;
            a.cnt_v = ctx->cnt_uv + ctx->p_rows();
            CK(cudaMemsetAsync(ctx->cnt_uv, 0, sizeof(unsigned) * (size_t)(ctx->p_rows() + ctx->n), st));
            // MF_OPT_VARIANT bits 24..25 select the dataflow form (mf_flow.cu launch_flow)
            CK(launch_flow(flow_shape(ctx->k, ctx->storage), a, st, &used, wsel));
        } else {
            // auto (bits 0..3 and 24..25 both 0): large waves (>= 64k samples on average: the Yahoo shape's
            // 183k) run the 8 / 16-lane shape with one sample per group and step -- Yahoo f16 51.8 -> 45.5 ms
            // per epoch, fp32 105 -> 91 -- small ones keep the 2-sample form (the Netflix shape's 11.6k-sample
            // waves: 31 vs 55 ms; profiles/r02bd_*, r02be_*).  Exact either way; the shapes round the dot
            // differently.
            ShapeId wsh = sh;
            int form = wsel == 3 ? 3 : wsel == 2 ? 0 : wsel == 1 ? 1 : 2;
            if ((ctx->variant & 0xF) == 0 && wsel == 0 && ctx->nwaves > 0 && ctx->N / ctx->nwaves >= 65536) {
                wsh = select_shape(ctx->k, ctx->storage, 1);
                form = 1;
            }
            CK(launch_waves(wsh, a, st, &l, form));
            used = 0;
        }
    } else {  // wavefront
        int l = 0;
        RC(ctx->run_wavefront(sh, a, &l, &used));
        launches = l;
    }
    CK(cudaEventRecord(ctx->events[2], st));
    const int rc = ctx->finish_epoch(schedule, eta, launches, used, stats);
    if (rc == MF_OK && tune) {
        tune->record(pf_slot, pf_on, ctx->last_kernel_ms);
        ctx->last_pf_pick = tune->pick;
    }
    return rc;
}

// -------------------------------------------------------------------- rmse --
extern "C" int mf_rmse(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz, double *out) {
    if (ctx && ctx->p_host) return ctx->fail(MF_ESTATE, "P lives in caller memory (MF_OPT_P_HOST): use mf_rmse_host_blocks");
    if (!ctx || !out) return MF_EINVAL;
    const bool dist = ctx->is_distributed();
    if (!dist) {
        if (!u || !v || !r || nnz <= 0) return ctx->fail(MF_EINVAL, "mf_rmse: null pointer or nnz <= 0");
        RC(ctx->ensure_factors());
    } else {
        // collective: every rank enters the all-gather / all-reduce or none does.  A rank may hold an
        // empty test shard (nnz = 0); the global count must be > 0.
        int pre = (nnz < 0 || (nnz > 0 && (!u || !v || !r))) ? ctx->fail(MF_EINVAL, "mf_rmse: null pointer or nnz < 0")
                                                              : ctx->ensure_factors();
        RC(ctx->agree(pre));
    }
    CK(cudaSetDevice(ctx->device));
    RC(ctx->gather_q());
    RC(dev_alloc(ctx, &ctx->partials, rmse_parts(), "alloc partials"));
    RC(dev_alloc(ctx, &ctx->d_out, 2, "alloc out"));
    if (dist && nnz == 0) {  // the same collective sequence as a non-empty shard: validation, sums, outcome
        RC(ctx->agree(MF_OK));
        return ctx->agree(ctx->rmse_partitioned(0, out));
    }
    cudaStream_t st = ctx->stream();
    if (nnz > ctx->cap_t) {
        dev_free(&ctx->tu);
        dev_free(&ctx->tv);
        dev_free(&ctx->tr);
        ctx->cap_t = 0;
        RC(dev_alloc(ctx, &ctx->tu, nnz, "alloc test u"));
        RC(dev_alloc(ctx, &ctx->tv, nnz, "alloc test v"));
        RC(dev_alloc(ctx, &ctx->tr, nnz, "alloc test r"));
        ctx->cap_t = nnz;
    }
    const cudaMemcpyKind kind = is_device_ptr(u) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(ctx->tu, u, sizeof(int32_t) * nnz, kind, st));
    CK(cudaMemcpyAsync(ctx->tv, v, sizeof(int32_t) * nnz, kind, st));
    CK(cudaMemcpyAsync(ctx->tr, r, sizeof(float) * nnz, kind, st));
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(DevScratch), st));
    CK(launch_validate_rows(ctx->tu, ctx->tv, ctx->tr, nnz, ctx->p_begin, ctx->p_end, ctx->n, ctx->scratch, st));
    CK(cudaMemcpyAsync(ctx->h_scratch, ctx->scratch, sizeof(DevScratch), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (dist) {
        RC(ctx->agree(ctx->h_scratch->bad ? ctx->fail(MF_EINVAL, "mf_rmse: %llu invalid test samples",
                                                      (unsigned long long)ctx->h_scratch->bad)
                                          : MF_OK));
    } else if (ctx->h_scratch->bad) {
        return ctx->fail(MF_EINVAL, "mf_rmse: %llu invalid test samples", (unsigned long long)ctx->h_scratch->bad);
    }
    if (ctx->p_begin != 0) CK(launch_rebase(ctx->tu, nnz, (int32_t)ctx->p_begin, st));
    if (dist) return ctx->agree(ctx->rmse_partitioned(nnz, out));
    const ShapeId sh = select_shape(ctx->k, ctx->storage, 0);
    CK(launch_rmse(sh, ctx->tu, ctx->tv, ctx->tr, nnz, ctx->P, ctx->Q, ctx->k, ctx->partials, rmse_parts(),
                   ctx->d_out, st));
    double h = 0;
    CK(cudaMemcpyAsync(&h, ctx->d_out, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *out = h;
    return MF_OK;
}

// ----------------------------------------------------------------- factors --
int mf_ctx::copy_out(const void *X, int64_t count, float *dst) {
    mf_ctx *ctx = this;
    cudaStream_t st = stream();
    if (storage == kF32) {
        CK(cudaMemcpyAsync(dst, X, sizeof(float) * count, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice
                                                                               : cudaMemcpyDeviceToHost, st));
    } else {
        float *tmp = nullptr;
        CK(cudaMallocAsync((void **)&tmp, sizeof(float) * std::max<int64_t>(count, 1), st));
        CK(launch_to_f32(storage, X, tmp, count, st));
        CK(cudaMemcpyAsync(dst, tmp, sizeof(float) * count, is_device_ptr(dst) ? cudaMemcpyDeviceToDevice
                                                                                : cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(tmp, st));
    }
    CK(cudaStreamSynchronize(st));
    return MF_OK;
}

int mf_ctx::copy_in(void *X, int64_t count, const float *src) {
    mf_ctx *ctx = this;
    cudaStream_t st = stream();
    const bool dsrc = is_device_ptr(src);
    if (storage == kF32) {
        CK(cudaMemcpyAsync(X, src, sizeof(float) * count, dsrc ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    } else {
        float *tmp = nullptr;
        CK(cudaMallocAsync((void **)&tmp, sizeof(float) * std::max<int64_t>(count, 1), st));
        CK(cudaMemcpyAsync(tmp, src, sizeof(float) * count, dsrc ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        CK(launch_from_f32(storage, X, tmp, count, st));
        CK(cudaFreeAsync(tmp, st));
    }
    CK(cudaStreamSynchronize(st));
    return MF_OK;
}

extern "C" int mf_get_factors(mf_ctx *ctx, float *P, float *Q) {
    if (!ctx) return MF_EINVAL;
    if (ctx->p_host && P) return ctx->fail(MF_ESTATE, "P lives in caller memory (MF_OPT_P_HOST): pass P = NULL");
    RC(ctx->agree(ctx->ensure_factors()));  // collective with NCCL: the all-gather below
    CK(cudaSetDevice(ctx->device));
    RC(ctx->gather_q());
    if (P) RC(ctx->copy_out(ctx->P, ctx->p_rows() * ctx->k, P));
    if (Q) RC(ctx->copy_out(ctx->Q, ctx->n * ctx->k, Q));
    return MF_OK;
}

extern "C" int mf_set_factors(mf_ctx *ctx, const float *P, const float *Q) {
    if (!ctx) return MF_EINVAL;
    if (ctx->p_host && P) return ctx->fail(MF_ESTATE, "P lives in caller memory (MF_OPT_P_HOST): pass P = NULL");
    RC(ctx->ensure_factors());
    CK(cudaSetDevice(ctx->device));
    RC(ctx->gather_q());
    if (P) RC(ctx->copy_in(ctx->P, ctx->p_rows() * ctx->k, P));
    if (Q) RC(ctx->copy_in(ctx->Q, ctx->n * ctx->k, Q));
    ctx->full_valid = true;
    ctx->seg_valid = false;
    return MF_OK;
}

extern "C" int mf_get_order(const mf_ctx *ctx_c, int64_t *out) {
    mf_ctx *ctx = const_cast<mf_ctx *>(ctx_c);
    if (!ctx || !out) return MF_EINVAL;
    if (ctx->N <= 0) return ctx->fail(MF_ESTATE, "mf_get_order before mf_load_coo");
    if (!ctx->shuffled) {
        for (int64_t i = 0; i < ctx->N; i++) out[i] = i;
        return MF_OK;
    }
    CK(cudaSetDevice(ctx->device));
    std::vector<uint32_t> h((size_t)ctx->N);
    CK(cudaMemcpyAsync(h.data(), ctx->perm, sizeof(uint32_t) * ctx->N, cudaMemcpyDeviceToHost, ctx->stream()));
    CK(cudaStreamSynchronize(ctx->stream()));
    for (int64_t i = 0; i < ctx->N; i++) out[i] = (int64_t)h[(size_t)i];
    return MF_OK;
}
