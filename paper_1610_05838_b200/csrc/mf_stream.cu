// mf_stream.cu -- streamed epochs: batch-Hogwild! directly from caller memory.
//
// The paper stages rating blocks from host memory and overlaps the transfer of the next block with
// the computation on the current one (§4.2; three streams per GPU).  Here a
// copy stream moves chunk i+1 (triples in the caller's order) into one of three device staging
// buffers while the context stream validates chunk i and runs the batch-Hogwild! kernel on it;
// events order buffer reuse.  Nothing is kept resident, so the training set may exceed HBM, and an
// end-to-end epoch from pinned host memory costs max(transfer, update) instead of their sum.
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/mf.h"
#include "mf_ctx.h"
#include "mf_kernels.cuh"

using namespace mf;

#define CK(expr)                                     \
    do {                                             \
        int _rc = ctx->cuda((expr), #expr);          \
        if (_rc != MF_OK) return _rc;                \
    } while (0)

void mf_ctx::release_stream() {
    for (int b = 0; b < kStreamBufs; b++) {
        if (sb_u[b]) cudaFree(sb_u[b]);
        if (sb_v[b]) cudaFree(sb_v[b]);
        if (sb_r[b]) cudaFree(sb_r[b]);
        sb_u[b] = sb_v[b] = nullptr;
        sb_r[b] = nullptr;
        if (sb_copied[b]) cudaEventDestroy(sb_copied[b]);
        if (sb_used[b]) cudaEventDestroy(sb_used[b]);
        sb_copied[b] = sb_used[b] = nullptr;
    }
    sb_cap = 0;
    if (copy_stream) cudaStreamDestroy(copy_stream);
    copy_stream = nullptr;
}

extern "C" int mf_epoch_host(mf_ctx *ctx, int schedule, const int32_t *u, const int32_t *v, const float *r,
                             int64_t nnz, mf_epoch_stats *stats) {
    if (!ctx) return MF_EINVAL;
    if (schedule != MF_SCHED_HOGWILD) return ctx->fail(MF_EINVAL, "mf_epoch_host supports MF_SCHED_HOGWILD only");
    if (!u || !v || !r || nnz <= 0) return ctx->fail(MF_EINVAL, "mf_epoch_host: null pointer or nnz <= 0");
    if (ctx->is_distributed()) return ctx->fail(MF_EINVAL, "mf_epoch_host: not available with NCCL attached");
    if (ctx->p_host) return ctx->fail(MF_ESTATE, "P lives in caller memory (MF_OPT_P_HOST): use mf_epoch_host_blocks");
    int rc = ctx->ensure_factors();
    if (rc != MF_OK) return rc;
    CK(cudaSetDevice(ctx->device));
    rc = ctx->gather_q();
    if (rc != MF_OK) return rc;
    ctx->seg_valid = false;
    const int64_t chunk = std::max<int64_t>(32, std::min<int64_t>(ctx->stream_chunk, nnz));
    if (chunk > ctx->sb_cap) {
        ctx->release_stream();
        for (int b = 0; b < mf_ctx::kStreamBufs; b++) {
            CK(cudaMalloc((void **)&ctx->sb_u[b], sizeof(int32_t) * chunk));
            CK(cudaMalloc((void **)&ctx->sb_v[b], sizeof(int32_t) * chunk));
            CK(cudaMalloc((void **)&ctx->sb_r[b], sizeof(float) * chunk));
            CK(cudaEventCreateWithFlags(&ctx->sb_copied[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->sb_used[b], cudaEventDisableTiming));
        }
        ctx->sb_cap = chunk;
    }
    if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    cudaStream_t st = ctx->stream(), cs = ctx->copy_stream;
    cudaPointerAttributes at;
    const bool dev_src = cudaPointerGetAttributes(&at, u) == cudaSuccess &&
                         (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    const cudaMemcpyKind kind = dev_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const float eta = ctx->eta_at(ctx->epoch);
    const ShapeId sh = hogwild_shape(ctx->k, ctx->storage, ctx->hog_shape_sel());
    const int workers = ctx->workers > 0 ? ctx->workers
                                         : (int)std::max<int64_t>(1, std::min<int64_t>(nnz / 10000, 1 << 30));
    CK(cudaEventRecord(ctx->events[0], st));
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(DevScratch), st));
    CK(cudaEventRecord(ctx->events[1], st));
    // the copy stream must not overwrite buffers the previous call's kernels may still read
    CK(cudaEventRecord(ctx->events[2], st));
    CK(cudaStreamWaitEvent(cs, ctx->events[2], 0));
    int launches = 0, used = 0;
    const int64_t nchunks = (nnz + chunk - 1) / chunk;
    for (int64_t i = 0; i < nchunks; i++) {
        const int b = (int)(i % mf_ctx::kStreamBufs);
        const int64_t lo = i * chunk, cnt = std::min<int64_t>(chunk, nnz - lo);
        if (i >= mf_ctx::kStreamBufs) CK(cudaStreamWaitEvent(cs, ctx->sb_used[b], 0));
        CK(cudaMemcpyAsync(ctx->sb_u[b], u + lo, sizeof(int32_t) * cnt, kind, cs));
        CK(cudaMemcpyAsync(ctx->sb_v[b], v + lo, sizeof(int32_t) * cnt, kind, cs));
        CK(cudaMemcpyAsync(ctx->sb_r[b], r + lo, sizeof(float) * cnt, kind, cs));
        CK(cudaEventRecord(ctx->sb_copied[b], cs));
        CK(cudaStreamWaitEvent(st, ctx->sb_copied[b], 0));
        // validate (and rebase rows) in place; a bad chunk raises scratch->bad and every later kernel skips
        CK(launch_gather_validate(ctx->sb_u[b], ctx->sb_v[b], ctx->sb_r[b], nullptr, cnt, ctx->p_begin, ctx->p_end,
                                  ctx->n, ctx->sb_u[b], ctx->sb_v[b], ctx->sb_r[b], ctx->scratch, st));
        UpdateArgs a = ctx->update_args(eta);
        a.u = ctx->sb_u[b];
        a.v = ctx->sb_v[b];
        a.r = ctx->sb_r[b];
        a.n = cnt;
        a.abort_if = &ctx->scratch->bad;
        CK(launch_hogwild(sh, a, workers, ctx->variant, st, &used));
        CK(cudaEventRecord(ctx->sb_used[b], st));
        launches += 2;
    }
    CK(cudaEventRecord(ctx->events[2], st));
    rc = ctx->finish_epoch(MF_SCHED_HOGWILD, eta, launches, used, stats);
    if (ctx->h_scratch->bad)
        return ctx->fail(MF_EINVAL, "mf_epoch_host: %llu invalid samples; chunks before the first invalid one were applied",
                         (unsigned long long)ctx->h_scratch->bad);
    if (stats && !ctx->count_updates) stats->updates = nnz;
    return rc;
}
