// mf_ctx.h -- the opaque context behind `mf_ctx *` (include/mf.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mf.h"
#include "mf_kernels.cuh"

struct mf_nccl;  // defined in mf_partition.cu

struct mf_ctx {
    // problem (global)
    int64_t m = 0, n = 0;
    int32_t k = 0;
    float alpha = 0.f, lambda = 0.f;
    double beta = 0.0;
    uint64_t seed = 0, seed_shuffle = 0;
    int32_t epoch = 0;

    // options
    int storage = 0;  // mf::StorageKind
    int device = 0;
    int workers = 0;
    int batch_f = 256;
    int wave_rows = 0, wave_cols = 0, wave_perm = 0;
    int wave_passes = 0;  // MF_OPT_WAVE_PASSES (0 = 1)
    int shuffle = 1;
    int count_updates = 0;
    int partitions = 0;
    int subepochs = 0;  // passes per epoch of the partitioned schedule (MF_OPT_SUBEPOCHS; 0 = 4)
    int part_split = 2; // partitioned (MF_OPT_PART_SPLIT): 0 = whole blocks; 1 = two half-segment sub-blocks in
                        // sequence, pipelined hand-over; 2 = unit grid (2G half-segment units, two concurrent
                        // families with their own Latin squares, each hand-over overlapping the other's compute)
    int wave_cta = 0;   // wavefront worker = CTA with shared-memory Q group (MF_OPT_WAVE_CTA)
    int variant = 0;
    int det_flow = 0;   // MF_OPT_DET_FLOW: deterministic schedule executed by per-row counters (1) or grid-barrier waves (0)
    int q_update = 2;   // MF_OPT_Q_UPDATE: batch-Hogwild! Q write-back 1 = atomic add of the change (A-20), 0 = store,
                        // 2 = auto by the expected concurrent updates per Q row
    double last_kappa = -1;  // kappa of the last batch-Hogwild! epoch (max over its launches; MF_OPT_Q_KAPPA)
    double col_sq = 0;  // sum_v (deg v / N)^2 of the loaded samples (0 before a load: launches use 1 / n)
    int r_stage = 1;    // MF_OPT_R_STAGING: batch-Hogwild! triples 1 = registers, 2 = TMA bulk copies into shared memory
    int trace = 0;
    // L2 prefetch, auto mode (MF_OPT_VARIANT bits 16..19 = 0).  Whether a prefetch pays depends on
    // where the rows live (it hides DRAM latency, and costs L2 request slots where the L2 is the
    // bottleneck), and it never changes what an epoch computes, so the library times it: epochs 0, 1, 2
    // of a schedule run off (a warm-up, not counted), on, off, and "on" is kept iff its epoch took less
    // than keep_on x the "off" epoch.
    struct AutoPf {
        int trials = 0, pick = 0;  // pick: 0 = undecided, else the bits-16..19 value in use (15 = off)
        float ms[2] = {0.f, 0.f};
        float keep_on = 0.97f;     // "on" is kept iff ms_on < keep_on * ms_off (the prior: > 1 favours on)
        int next(int on, int *slot) const {
            if (pick) {
                *slot = -1;
                return pick;
            }
            *slot = trials == 1 ? 1 : 0;
            return *slot ? on : 15;
        }
        void record(int slot, int on, float kernel_ms) {
            if (slot < 0) return;
            ms[slot] = kernel_ms;
            if (++trials >= 3) pick = ms[1] < keep_on * ms[0] ? on : 15;
        }
        void reset() { trials = 0, pick = 0; }
    };
    // batch-Hogwild! keeps the prefetch only when it is clearly faster (it loses 6-16% where L2 is the
    // limit); the CTA wavefront keeps it unless clearly slower (it won on 5 of 6 measured shape /
    // storage pairs, by 2-13%), so one noisy trial epoch does not flip a small gain
    AutoPf pf_hogwild, pf_wave_cta{0, 0, {0.f, 0.f}, 1.03f};
    int last_pf_pick = 0;   // pick of the last auto-tuned schedule run (reported by mf_get_option)
    int variant_eff = 0;    // the variant the current epoch's launches use (auto fields resolved)
    float last_kernel_ms = 0.f;
    cudaStream_t user_stream = nullptr;

    // device state
    bool dev_ready = false;
    int num_sms = 0;
    cudaStream_t own_stream = nullptr;
    cudaEvent_t events[4] = {nullptr, nullptr, nullptr, nullptr};
    mf::DevScratch *scratch = nullptr;
    mf::DevScratch *h_scratch = nullptr;  // pinned
    void *P = nullptr, *Q = nullptr;      // storage precision, row-major
    int64_t p_begin = 0, p_end = 0;       // rows of the global P held here

    // training set (device SoA, stored order)
    int32_t *u = nullptr, *v = nullptr;
    float *r = nullptr;
    uint32_t *perm = nullptr;  // perm[i] = caller index of stored sample i
    int64_t perm_n = -1;       // perm is the A-8 permutation of perm_n samples under perm_seed (cached)
    bool reshuffle_due = false;  // MF_OPT_SHUFFLE = 2: permute again before the next epoch
    uint64_t perm_seed = 0;
    int64_t N = 0, cap_n = 0;
    int shuffled = 0;

    // deterministic wave layout
    int32_t *wu = nullptr, *wv = nullptr;
    float *wr = nullptr;
    int64_t *wave_off = nullptr;
    int64_t nwaves = -1;
    // deterministic dataflow execution (MF_OPT_DET_FLOW, mf_flow.cu): per wave-sorted sample the ordinals of its
    // update of row u / column v in the serial order, and per row the updates applied so far
    int32_t *ord_u = nullptr, *ord_v = nullptr;
    unsigned *cnt_uv = nullptr;  // p_rows() + n counters

    // wavefront layout (mf_wavefront.cu)
    bool wf_valid = false;
    int wf_s = 0, wf_c = 0, wf_p = 1;
    int32_t *fu = nullptr, *fv = nullptr;
    float *fr = nullptr;
    int64_t *wf_off = nullptr;    // (s*c + 1) block offsets, block (w, c) at w*c + c
    int32_t *wf_locks = nullptr;  // c column locks
    int32_t *wf_seq = nullptr;    // s x c column sequences (this epoch)
    int64_t *wf_trace = nullptr;  // 4 int64 per block
    int64_t wf_trace_n = 0;

    // partitioned layout (mf_partition.cu)
    bool part_valid = false;
    int part_G = 0;                  // partitions = world size (NCCL) or logical partitions (loopback)
    int part_local = 0;              // partitions hosted by this context (1 with NCCL, G in loopback)
    int part_S = 1;                  // passes per epoch in the current layout
    int part_mode = 0;               // MF_OPT_PART_SPLIT the current layout was built with
    int32_t *bu = nullptr, *bv = nullptr;  // samples bucketed by (local partition, column segment); v segment-local
    float *br = nullptr;
    std::vector<int64_t> h_blk_off;  // (part_local * G + 1) block offsets
    int64_t seg_rows_max = 0;        // rows of the largest Q segment
    std::vector<void *> q_cur, q_next;  // per hosted partition: the Q segment it holds / receive buffer
    std::vector<int32_t> held;       // held[g] = Q segment held by partition g (all G, known everywhere)
    bool full_valid = true;          // ctx->Q (full n x k) is current
    bool seg_valid = false;          // q_cur buffers are current
    mf_nccl *nccl = nullptr;
    int rank = 0, world = 1;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_half[2] = {}, ev_recv[2] = {};  // pipelined half-segment exchange
    bool recv_pending = false;  // q_cur halves are still arriving on comm_stream (wait on ev_recv)
    void *gather_tmp = nullptr;
    // unit grid (MF_OPT_PART_SPLIT = 2): column unit (c, h) = half h (0 lower, 1 upper) of segment c; family h
    // rotates by its own Latin square per pass; family 1 computes on stream2 concurrently with family 0
    std::vector<void *> u_cur[2], u_next[2];  // per family, per hosted partition: the unit it holds / receive buffer
    std::vector<int32_t> held_u[2];           // held_u[h][g] = segment whose half h partition g holds
    int64_t unit_rows_max = 0;
    cudaStream_t stream2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

    // streamed epochs from caller memory (mf_stream.cu)
    static constexpr int kStreamBufs = 3;
    int64_t stream_chunk = 1 << 22;  // samples per chunk (MF_OPT_STREAM_CHUNK; 2^21..2^23 within 1%, 2^25 -8%: r02bb)
    cudaStream_t copy_stream = nullptr;
    int32_t *sb_u[kStreamBufs] = {}, *sb_v[kStreamBufs] = {};
    float *sb_r[kStreamBufs] = {};
    int64_t sb_cap = 0;
    cudaEvent_t sb_copied[kStreamBufs] = {}, sb_used[kStreamBufs] = {};
    void release_stream();

    // out-of-core factors (mf_outcore.cu): P in caller host memory, streamed by row block
    int p_host = 0;                        // MF_OPT_P_HOST: 1 = no device P; epochs via mf_epoch_host_blocks
    void *oc_slot[kStreamBufs] = {};       // device P-segment slots
    int64_t oc_cap = 0;                    // bytes per slot
    cudaEvent_t oc_in[kStreamBufs] = {}, oc_done[kStreamBufs] = {}, oc_out[kStreamBufs] = {};
    cudaStream_t d2h_stream = nullptr;     // P-segment write-backs
    void release_outcore();

    // scratch for rmse / factors
    int32_t *tu = nullptr, *tv = nullptr;
    float *tr = nullptr;
    int64_t cap_t = 0;
    double *partials = nullptr, *d_out = nullptr;
    float *f32_tmp = nullptr;

    std::string err;

    int fail(int code, const char *fmt, ...);
    int cuda(cudaError_t e, const char *what);
    int ensure_device();
    int ensure_factors();
    cudaStream_t stream() const;
    int storage_bytes() const;
    int64_t p_rows() const { return p_end - p_begin; }
    bool is_distributed() const { return nccl != nullptr; }
    float eta_at(int32_t t) const;
    int auto_workers() const;
    int hog_shape_sel() const;  // batch-Hogwild! group shape: MF_OPT_VARIANT bits 0..3, or the auto rule
    mf::UpdateArgs update_args(float eta) const;
    int finish_epoch(int schedule, float eta, int launches, int workers_used, mf_epoch_stats *stats);
    int build_waves();
    int reshuffle();
    int copy_out(const void *X, int64_t count, float *dst);
    int copy_in(void *X, int64_t count, const float *src);
    void drop_layouts();
    int drop_other_layouts(int schedule);
    void release();

    // mf_wavefront.cu
    int build_wavefront();
    int agree(int local);  // distributed: every rank returns the worst status any rank had (collective)
    double *agree_buf = nullptr;
    int run_wavefront(const mf::ShapeId &sh, const mf::UpdateArgs &a, int *launches, int *workers_used);
    void release_wavefront();

    // mf_partition.cu
    int epoch_partitioned(mf_epoch_stats *stats);
    int build_partition();
    int exchange_segments(const std::vector<int32_t> &want);
    int exchange_half(const std::vector<int32_t> &want, int h);
    int epoch_units(mf_epoch_stats *stats);
    int exchange_unit(const std::vector<int32_t> &want, int h, cudaStream_t hs);
    int scatter_units(const std::vector<int32_t> (&want)[2]);
    int gather_units();
    void unit_rows(int c, int h, int64_t *row0, int64_t *rows) const;  // global first row and row count of unit (c, h)
    int rmse_partitioned(int64_t nnz, double *out);
    int gather_q();
    void release_partition();
};
