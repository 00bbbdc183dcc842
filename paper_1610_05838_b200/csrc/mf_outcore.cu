// mf_outcore.cu -- out-of-core factors: P stays in caller host memory and streams through the GPU
// block by block (the paper's own path for Hugewiki on one GPU: R divided into row blocks (64 x 1), each
// block's P segment and ratings copied in, updated, and the P segment copied back while the next block's
// data is already in flight -- PAPER.md:294-303 (§4.1) and 307-320 (§4.2, three streams per GPU).
//
// Q (n x k) is resident on the device.  Row block b holds rows [floor(b m / B), floor((b+1) m / B)) of P
// and the caller's ratings of those rows, contiguous in [block_off[b], block_off[b+1]).  Per block:
//   H2D stream:  P segment -> device slot (b mod 3), then the block's ratings in chunks (staging buffers)
//   context:     validate + rebase the chunk's rows to the segment, batch-Hogwild! on it
//   D2H stream:  after the block's last chunk, the P segment back to the caller's array
// so block b+1's transfers overlap block b's updates and block b-1's write-back.  Ratings of one row
// block touch only that block's P rows, so every update sees exactly the P values the serial order
// would (with MF_OPT_WORKERS = 1 an epoch is serial SGD over the given order: tests/test_gpu_outcore.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/mf.h"
#include "mf_ctx.h"
#include "mf_host_util.h"
#include "mf_kernels.cuh"

using namespace mf;

#define CK(expr)                                     \
    do {                                             \
        int _rc = ctx->cuda((expr), #expr);          \
        if (_rc != MF_OK) return _rc;                \
    } while (0)

void mf_ctx::release_outcore() {
    for (int s = 0; s < kStreamBufs; s++) {
        if (oc_slot[s]) cudaFree(oc_slot[s]);
        oc_slot[s] = nullptr;
        for (auto *ev : {&oc_in[s], &oc_done[s], &oc_out[s]})
            if (*ev) cudaEventDestroy(*ev), *ev = nullptr;
    }
    oc_cap = 0;
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    d2h_stream = nullptr;
}

namespace {

int check_blocks(mf_ctx *ctx, int64_t nnz, const int64_t *block_off, int32_t nblocks) {
    if (!block_off || nblocks < 1 || nblocks > ctx->m) return ctx->fail(MF_EINVAL, "out-of-core: need 1 <= nblocks <= m");
    if (block_off[0] != 0 || block_off[nblocks] != nnz) return ctx->fail(MF_EINVAL, "out-of-core: block_off must span [0, nnz]");
    for (int32_t b = 0; b < nblocks; b++)
        if (block_off[b + 1] < block_off[b]) return ctx->fail(MF_EINVAL, "out-of-core: block_off must be nondecreasing");
    return MF_OK;
}

// staging for ratings (the streamed-epoch buffers) and three P-segment slots
int ensure_staging(mf_ctx *ctx, int64_t chunk, int64_t seg_bytes) {
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
    if (seg_bytes > ctx->oc_cap) {
        for (int s = 0; s < mf_ctx::kStreamBufs; s++) {
            if (ctx->oc_slot[s]) cudaFree(ctx->oc_slot[s]);
            ctx->oc_slot[s] = nullptr;
        }
        ctx->oc_cap = 0;
        for (int s = 0; s < mf_ctx::kStreamBufs; s++) CK(cudaMalloc(&ctx->oc_slot[s], (size_t)seg_bytes));
        ctx->oc_cap = seg_bytes;
    }
    for (int s = 0; s < mf_ctx::kStreamBufs; s++)
        for (auto *ev : {&ctx->oc_in[s], &ctx->oc_done[s], &ctx->oc_out[s]})
            if (!*ev) CK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    if (!ctx->d2h_stream) CK(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
    return MF_OK;
}

int common_checks(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz, const void *P_host) {
    if (!u || !v || !r || !P_host || nnz <= 0) return ctx->fail(MF_EINVAL, "out-of-core: null pointer or nnz <= 0");
    if (!ctx->p_host) return ctx->fail(MF_ESTATE, "out-of-core calls need MF_OPT_P_HOST = 1 (set before the factors exist)");
    if (ctx->is_distributed()) return ctx->fail(MF_EINVAL, "out-of-core: not available with NCCL attached");
    return MF_OK;
}

}  // namespace

extern "C" int mf_init_rows_host(mf_ctx *ctx, int32_t tag, int64_t row0, int64_t rows, void *out) {
    if (!ctx || !out || tag < 0 || tag > 1 || row0 < 0 || rows < 0) return MF_EINVAL;
    if (row0 + rows > (tag ? ctx->n : ctx->m)) return ctx->fail(MF_EINVAL, "mf_init_rows_host: rows out of range");
    int rc = ctx->ensure_device();
    if (rc != MF_OK) return rc;
    CK(cudaSetDevice(ctx->device));
    const size_t rb = (size_t)ctx->k * ctx->storage_bytes();
    const int64_t step = std::max<int64_t>(1, (int64_t)((256ll << 20) / rb));  // 256 MB per piece
    void *tmp = nullptr;
    CK(cudaMalloc(&tmp, (size_t)std::min<int64_t>(step, std::max<int64_t>(rows, 1)) * rb));
    cudaStream_t st = ctx->stream();
    for (int64_t o = 0; o < rows; o += step) {
        const int64_t cnt = std::min<int64_t>(step, rows - o);
        cudaError_t e = launch_init_rows(ctx->storage, tmp, row0 + o, cnt, ctx->k, ctx->seed, (uint32_t)tag, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync((char *)out + (size_t)o * rb, tmp, (size_t)cnt * rb, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            cudaFree(tmp);
            return ctx->cuda(e, "mf_init_rows_host");
        }
    }
    cudaFree(tmp);
    return MF_OK;
}

extern "C" int mf_epoch_host_blocks(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz,
                                    const int64_t *block_off, int32_t nblocks, void *P_host, mf_epoch_stats *stats) {
    if (!ctx) return MF_EINVAL;
    int rc = common_checks(ctx, u, v, r, nnz, P_host);
    if (rc == MF_OK) rc = check_blocks(ctx, nnz, block_off, nblocks);
    if (rc == MF_OK) rc = ctx->ensure_factors();
    if (rc != MF_OK) return rc;
    CK(cudaSetDevice(ctx->device));
    const size_t rb = (size_t)ctx->k * ctx->storage_bytes();
    int64_t seg_max = 0;
    for (int32_t b = 0; b < nblocks; b++)
        seg_max = std::max(seg_max, seg_begin(ctx->m, nblocks, b + 1) - seg_begin(ctx->m, nblocks, b));
    const int64_t chunk = std::max<int64_t>(32, std::min<int64_t>(ctx->stream_chunk, nnz));
    rc = ensure_staging(ctx, chunk, seg_max * (int64_t)rb);
    if (rc != MF_OK) return rc;
    cudaStream_t st = ctx->stream(), cs = ctx->copy_stream, ds = ctx->d2h_stream;
    const cudaMemcpyKind kind = cudaMemcpyDefault;  // ratings and P may be host (pinned or pageable) or device
    const float eta = ctx->eta_at(ctx->epoch);
    const ShapeId sh = hogwild_shape(ctx->k, ctx->storage, ctx->hog_shape_sel());
    CK(cudaEventRecord(ctx->events[0], st));
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(DevScratch), st));
    CK(cudaEventRecord(ctx->events[1], st));
    CK(cudaEventRecord(ctx->events[2], st));
    CK(cudaStreamWaitEvent(cs, ctx->events[2], 0));  // no buffer of a previous call is still being read
    CK(cudaStreamWaitEvent(ds, ctx->events[2], 0));
    int launches = 0, used = 0, block_i = 0;
    int64_t chunk_i = 0;
    for (int32_t b = 0; b < nblocks; b++) {
        const int64_t lo = block_off[b], hi = block_off[b + 1];
        if (hi == lo) continue;  // this P segment is not touched this epoch
        const int64_t r0 = seg_begin(ctx->m, nblocks, b), rows = seg_begin(ctx->m, nblocks, b + 1) - r0;
        const int s = block_i % mf_ctx::kStreamBufs;
        char *hseg = (char *)P_host + (size_t)r0 * rb;
        if (block_i >= mf_ctx::kStreamBufs) CK(cudaStreamWaitEvent(cs, ctx->oc_out[s], 0));  // slot written back
        CK(cudaMemcpyAsync(ctx->oc_slot[s], hseg, (size_t)rows * rb, kind, cs));
        CK(cudaEventRecord(ctx->oc_in[s], cs));
        CK(cudaStreamWaitEvent(st, ctx->oc_in[s], 0));
        // workers: the A-10 clamp over the block's ratings
        const int workers = ctx->workers > 0 ? ctx->workers
                                             : (int)std::max<int64_t>(1, std::min<int64_t>((hi - lo) / 10000, 1 << 30));
        for (int64_t c0 = lo; c0 < hi; c0 += chunk, chunk_i++) {
            const int bb = (int)(chunk_i % mf_ctx::kStreamBufs);
            const int64_t cnt = std::min<int64_t>(chunk, hi - c0);
            if (chunk_i >= mf_ctx::kStreamBufs) CK(cudaStreamWaitEvent(cs, ctx->sb_used[bb], 0));
            CK(cudaMemcpyAsync(ctx->sb_u[bb], u + c0, sizeof(int32_t) * cnt, kind, cs));
            CK(cudaMemcpyAsync(ctx->sb_v[bb], v + c0, sizeof(int32_t) * cnt, kind, cs));
            CK(cudaMemcpyAsync(ctx->sb_r[bb], r + c0, sizeof(float) * cnt, kind, cs));
            CK(cudaEventRecord(ctx->sb_copied[bb], cs));
            CK(cudaStreamWaitEvent(st, ctx->sb_copied[bb], 0));
            // rows must lie in this block's segment; rebased to it (the slot holds the segment only)
            CK(launch_gather_validate(ctx->sb_u[bb], ctx->sb_v[bb], ctx->sb_r[bb], nullptr, cnt, r0, r0 + rows, ctx->n,
                                      ctx->sb_u[bb], ctx->sb_v[bb], ctx->sb_r[bb], ctx->scratch, st));
            UpdateArgs a = ctx->update_args(eta);
            a.u = ctx->sb_u[bb];
            a.v = ctx->sb_v[bb];
            a.r = ctx->sb_r[bb];
            a.n = cnt;
            a.P = ctx->oc_slot[s];
            a.abort_if = &ctx->scratch->bad;
            CK(launch_hogwild(sh, a, workers, ctx->variant, st, &used));
            CK(cudaEventRecord(ctx->sb_used[bb], st));
            launches += 2;
        }
        CK(cudaEventRecord(ctx->oc_done[s], st));
        CK(cudaStreamWaitEvent(ds, ctx->oc_done[s], 0));
        CK(cudaMemcpyAsync(hseg, ctx->oc_slot[s], (size_t)rows * rb, kind, ds));
        CK(cudaEventRecord(ctx->oc_out[s], ds));
        block_i++;
    }
    CK(cudaEventRecord(ctx->events[3], ds));  // every write-back issued
    CK(cudaStreamWaitEvent(st, ctx->events[3], 0));
    CK(cudaEventRecord(ctx->events[2], st));
    rc = ctx->finish_epoch(MF_SCHED_HOGWILD, eta, launches, used, stats);
    if (ctx->h_scratch->bad)
        return ctx->fail(MF_EINVAL, "mf_epoch_host_blocks: %llu samples outside their block's rows or invalid; "
                                    "chunks before the first invalid one were applied",
                         (unsigned long long)ctx->h_scratch->bad);
    if (stats && !ctx->count_updates) stats->updates = nnz;
    return rc;
}

extern "C" int mf_rmse_host_blocks(mf_ctx *ctx, const int32_t *u, const int32_t *v, const float *r, int64_t nnz,
                                   const int64_t *block_off, int32_t nblocks, const void *P_host, double *out) {
    if (!ctx || !out) return MF_EINVAL;
    int rc = common_checks(ctx, u, v, r, nnz, P_host);
    if (rc == MF_OK) rc = check_blocks(ctx, nnz, block_off, nblocks);
    if (rc == MF_OK) rc = ctx->ensure_factors();
    if (rc != MF_OK) return rc;
    CK(cudaSetDevice(ctx->device));
    const size_t rb = (size_t)ctx->k * ctx->storage_bytes();
    int64_t seg_max = 0;
    for (int32_t b = 0; b < nblocks; b++)
        seg_max = std::max(seg_max, seg_begin(ctx->m, nblocks, b + 1) - seg_begin(ctx->m, nblocks, b));
    const int64_t chunk = std::max<int64_t>(32, std::min<int64_t>(ctx->stream_chunk, nnz));
    rc = ensure_staging(ctx, chunk, seg_max * (int64_t)rb);
    if (rc != MF_OK) return rc;
    if (!ctx->partials) CK(cudaMalloc((void **)&ctx->partials, sizeof(double) * rmse_parts()));
    cudaStream_t st = ctx->stream();
    const ShapeId sh = select_shape(ctx->k, ctx->storage, 0);
    const int64_t nchunks_max = (nnz + chunk - 1) / chunk + nblocks;
    double *sums = nullptr;
    CK(cudaMallocAsync((void **)&sums, sizeof(double) * nchunks_max, st));
    CK(cudaMemsetAsync(ctx->scratch, 0, sizeof(DevScratch), st));
    int64_t nch = 0;
    // one stream, in order: the RMSE is a read-only pass (no write-back)
    for (int32_t b = 0; b < nblocks && rc == MF_OK; b++) {
        const int64_t lo = block_off[b], hi = block_off[b + 1];
        if (hi == lo) continue;
        const int64_t r0 = seg_begin(ctx->m, nblocks, b), rows = seg_begin(ctx->m, nblocks, b + 1) - r0;
        rc = ctx->cuda(cudaMemcpyAsync(ctx->oc_slot[0], (const char *)P_host + (size_t)r0 * rb, (size_t)rows * rb,
                                       cudaMemcpyDefault, st), "rmse P segment");
        for (int64_t c0 = lo; c0 < hi && rc == MF_OK; c0 += chunk) {
            const int64_t cnt = std::min<int64_t>(chunk, hi - c0);
            cudaError_t e = cudaMemcpyAsync(ctx->sb_u[0], u + c0, sizeof(int32_t) * cnt, cudaMemcpyDefault, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->sb_v[0], v + c0, sizeof(int32_t) * cnt, cudaMemcpyDefault, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->sb_r[0], r + c0, sizeof(float) * cnt, cudaMemcpyDefault, st);
            if (e == cudaSuccess)
                e = launch_gather_validate(ctx->sb_u[0], ctx->sb_v[0], ctx->sb_r[0], nullptr, cnt, r0, r0 + rows, ctx->n,
                                           ctx->sb_u[0], ctx->sb_v[0], ctx->sb_r[0], ctx->scratch, st);
            if (e == cudaSuccess)
                e = launch_rmse(sh, ctx->sb_u[0], ctx->sb_v[0], ctx->sb_r[0], cnt, ctx->oc_slot[0], ctx->Q, ctx->k,
                                ctx->partials, rmse_parts(), sums + nch, st, 0);
            rc = ctx->cuda(e, "rmse block");
            nch++;
        }
    }
    std::vector<double> h((size_t)std::max<int64_t>(nch, 1), 0.0);
    if (rc == MF_OK && nch)
        rc = ctx->cuda(cudaMemcpyAsync(h.data(), sums, sizeof(double) * nch, cudaMemcpyDeviceToHost, st), "rmse sums");
    if (rc == MF_OK)
        rc = ctx->cuda(cudaMemcpyAsync(ctx->h_scratch, ctx->scratch, sizeof(DevScratch), cudaMemcpyDeviceToHost, st),
                       "rmse scratch");
    cudaFreeAsync(sums, st);
    if (rc == MF_OK) rc = ctx->cuda(cudaStreamSynchronize(st), "rmse sync");
    if (rc != MF_OK) return rc;
    if (ctx->h_scratch->bad) return ctx->fail(MF_EINVAL, "mf_rmse_host_blocks: samples outside their block's rows or invalid");
    double s = 0.0;
    for (int64_t i = 0; i < nch; i++) s += h[(size_t)i];  // fixed order: deterministic
    *out = std::sqrt(s / (double)nnz);
    return MF_OK;
}
