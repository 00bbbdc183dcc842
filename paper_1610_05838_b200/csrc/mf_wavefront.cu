// mf_wavefront.cu -- wavefront-update schedule (§3.2.3, Fig. 8).
//
// R is bucketed into an s x c grid of blocks: s row bands (one per worker) and
// c column groups, balanced segments whose widths differ by at most one (SPEC.md:319
// puts the remainder in the last band; with c not dividing n that band can be many
// times wider and serialises the schedule, A-9).  The bucketing is a stable radix sort by block id, so each
// block keeps the shuffled order.  Worker w (one warp) walks
// its column sequence pi_w[0..c): for wave j it acquires the lock of column
// pi_w[j] in the 1-D column lock array, processes block
// (w, pi_w[j]) serially, and releases the lock (release-before-acquire, no
// hold-and-wait: DESIGN.md A-9).  Default sequences are a randomized Latin
// rectangle pi_w[j] = sigma((rho(w) + j) mod c), re-drawn per epoch; option
// MF_OPT_WAVE_PERM=1 gives every worker an independent random permutation,
// the paper's literal reading.
//
// Inside a block a worker keeps D samples in flight: rows of sample i+D are
// loaded while sample i is computed, and a row written by one of the D
// previous samples is forwarded from registers, so a block is still processed
// exactly serially.  Lock acquire/release use gpu-scope atomics with fences;
// P/Q loads are ld.global.cg (coherent at L2).
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "mf_ctx.h"
#include "mf_host_util.h"
#include "sgd_core.cuh"

using namespace mf;

namespace {


// row band / column group by balanced segmentation (widths differ by at most one; A-9)
// pass p of stored sample i is floor(i * P / n): every epoch is P passes over consecutive slices of the
// shuffled order, each with its own column sequences (block id = (p * s + band) * c + group)
__global__ void k_block_keys(const int32_t *u, const int32_t *v, int64_t n, int64_t rows, int64_t cols, int s,
                             int c, int P, uint32_t *keys, uint32_t *idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = seg_index(u[i], rows, s), g = seg_index(v[i], cols, c), p = (i * P) / n;
        keys[i] = (uint32_t)((p * s + b) * c + g);
        idx[i] = (uint32_t)i;
    }
}

// q-stationary layout (MF_OPT_WAVE_CTA = 3): key = band * n + v, so a block (band, column group) is a
// contiguous key range and inside it the samples of one Q row (a "run") are contiguous, each run in
// shuffled order (the sort is stable)
__global__ void k_run_keys(const int32_t *u, const int32_t *v, int64_t n, int64_t rows, int64_t cols, int s, int P,
                           uint32_t *keys, uint32_t *idx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = (i * P) / n;
        keys[i] = (uint32_t)((p * s + seg_index(u[i], rows, s)) * cols + v[i]);
        idx[i] = (uint32_t)i;
    }
}

// block offsets of the q-stationary layout: off[b] = first sorted position with key >= band * n +
// first column of group g (b = band * c + g), off[s * c] = n; one binary search per block
__global__ void k_run_block_offsets(const uint32_t *sorted_keys, int64_t n, int64_t nb, int c, int64_t cols,
                                    int64_t *off) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x) {
        if (b == nb) {
            off[b] = n;
            continue;
        }
        const uint32_t key = (uint32_t)((b / c) * cols + seg_begin(cols, c, (int)(b % c)));
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (sorted_keys[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        off[b] = lo;
    }
}

// offsets[b] = first sorted position with key >= b, for b in [0, nb]
__global__ void k_block_offsets(const uint32_t *sorted_keys, int64_t n, int64_t nb, int64_t *off) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = i == 0 ? -1 : (int64_t)sorted_keys[i - 1];
        const int64_t cur = i == n ? nb : (int64_t)sorted_keys[i];
        for (int64_t b = prev + 1; b <= cur; b++) off[b] = i;
    }
}

struct WfArgs {
    const int32_t *u, *v;
    const float *r;
    const int64_t *off;   // s*c + 1
    const int32_t *seq;   // latin: sigma[c] then rho[s]; random: s*c table
    int32_t *locks;       // c
    void *P, *Q;
    int64_t *trace;       // optional, 4 per block
    DevScratch *scratch;
    int s, c, k, latin, count_updates;
    int passes;           // P: the epoch is P passes over consecutive slices of the shuffled samples, each with
                          // its own column sequences (seq holds P of them)
    int pf;               // CTA workers: L2 prefetch of a tile's P rows when it is claimed (0 off, 1 bulk, 2 per line)
    int min_per_group;    // CTA workers: in-block concurrency clamp, samples per concurrent group
    int tma;              // CTA workers: stage the Q group with bulk async copies (TMA engine) instead of a thread loop
    int q_late;           // CTA workers: read a rating's q_v from shared memory only once its p_u has arrived
    int q_wait_late;      // CTA workers: wait for the Q group's copy-in at a thread's first rating of the block
    float eta, lam;
    int64_t n_cols;       // column groups are balanced segments [floor(g n / c), floor((g+1) n / c))
};

// Column lock acquire: test-and-test-and-set.  Waiters poll with plain relaxed loads (served by the L2
// slice, no read-modify-write) and try the compare-and-swap only when the lock reads free, with a short
// growing back-off, so ~1,000 waiting warps do not flood the L2 atomic units the running workers' row
// traffic goes through.
__device__ __forceinline__ void lock_acquire(int32_t *lock) {
    unsigned ns = 32;
    for (;;) {
        int32_t cur;
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(cur) : "l"(lock) : "memory");
        if (cur == 0 && atomicCAS(lock, 0, 1) == 0) break;
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

// The same acquire by a whole warp in lockstep: lane 0 tests and tries, the outcome is broadcast, every
// lane loops -- no lane-divergent region, so the shuffles after it compile without convergence fix-ups.
__device__ __forceinline__ void lock_acquire_warp(int32_t *lock, int lane) {
    unsigned ns = 32;
    for (;;) {
        int got = 0;
        if (lane == 0) {
            int32_t cur;
            asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(cur) : "l"(lock) : "memory");
            got = cur == 0 && atomicCAS(lock, 0, 1) == 0;
        }
        if (__shfl_sync(0xffffffffu, got, 0)) break;
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}

// column of worker w at step pj = pass * c + wave: Latin rectangle sigma_p((rho_p(w) + j) mod c), or the
// worker's own random permutation of pass p
__device__ __forceinline__ int wf_column(const WfArgs &a, int w, int pj) {
    const int c = a.c, p = pj / c, j = pj - p * c;
    if (a.latin) {
        const int32_t *sq = a.seq + (int64_t)p * (c + a.s);
        return sq[(sq[c + w] + j) % c];
    }
    return a.seq[((int64_t)p * a.s + w) * c + j];
}

__device__ __forceinline__ int64_t globaltimer() {
    int64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <class SH, int D>
__global__ void __launch_bounds__(32) k_wavefront(WfArgs a) {
    static_assert(SH::L == 32, "wavefront worker is a full warp");
    static_assert(D >= 1 && D <= 16, "in-block pipeline depth");
    const int lane = threadIdx.x & 31;
    // one warp per CTA: the worker index is block-uniform, so no lane-divergent early exit precedes the
    // shuffles (the compiler then emits them without convergence fix-ups)
    const int w = blockIdx.x;
    if (w >= a.s) return;
    const int k = SH::FULL ? SH::KMAX : a.k;
    const int c = a.c;
    int bad = 0;
    unsigned long long done = 0;
    for (int pj = 0; pj < a.passes * c; pj++) {  // pass pj / c, wave pj % c
        const int col = wf_column(a, w, pj);
        int32_t *lock = a.locks + col;
        const int64_t blk = ((int64_t)(pj / c) * a.s + w) * c + col;
        const int64_t lo = a.off[blk], hi = a.off[blk + 1];
        // The block's triples are this worker's alone: fetch the first two 32-sample tiles (lane i holds
        // sample tb + i) before taking the lock, so only the Q rows wait for it.
        int64_t tb = lo;
        int32_t cu = 0, cv = 0, nu = 0, nv = 0;
        float cr = 0.f, nr = 0.f;
        {
            const int64_t i0 = lo + lane, i1 = lo + 32 + lane;
            if (i0 < hi) cu = __ldg(a.u + i0), cv = __ldg(a.v + i0), cr = __ldg(a.r + i0);
            if (i1 < hi) nu = __ldg(a.u + i1), nv = __ldg(a.v + i1), nr = __ldg(a.r + i1);
        }
        lock_acquire_warp(lock, lane);
        __threadfence();  // acquire: the previous holder's stores are visible (loads are .cg)
        const int64_t t0 = a.trace ? globaltimer() : 0;
        done += (uint64_t)(hi - lo);

        // sample j's triple from the two tiles held in registers (j warp-uniform, tb <= j < tb + 64)
        auto triple = [&](int64_t jj, int32_t &uu, int32_t &vv, float &rr) {
            const int o = (int)(jj - tb);
            const bool in_cur = o < 32;
            uu = __shfl_sync(0xffffffffu, in_cur ? cu : nu, o & 31);
            vv = __shfl_sync(0xffffffffu, in_cur ? cv : nv, o & 31);
            rr = __shfl_sync(0xffffffffu, in_cur ? cr : nr, o & 31);
        };
        // ring of D prefetched samples (rows loaded D samples ahead), history of the D last written rows
        int32_t ru[D], rv[D];
        float rr[D];
        RowRaw<SH> rp[D], rq[D];
        int32_t hu[D], hv[D];
        RowRaw<SH> hp[D], hq[D];
#pragma unroll
        for (int d = 0; d < D; d++) {
            hu[d] = -1;
            hv[d] = -1;
            const bool ok = lo + d < hi;
            int32_t tu_, tv_;
            float tr_;
            triple(lo + d, tu_, tv_, tr_);
            ru[d] = ok ? tu_ : 0;
            rv[d] = ok ? tv_ : 0;
            rr[d] = ok ? tr_ : 0.f;
            load_row<SH>(a.P, ru[d], k, lane, ok, rp[d]);
            load_row<SH>(a.Q, rv[d], k, lane, ok, rq[d]);
        }
        // Branch-free over the D slots: every lane of the warp reaches every shuffle (no collective
        // fix-up code around the butterflies); a slot past the block's end computes on zero rows and
        // neither stores nor forwards.
        for (int64_t base = lo; base < hi; base += D) {
#pragma unroll
            for (int d = 0; d < D; d++) {
                const int64_t i = base + d;
                const bool val = i < hi;
                RowRaw<SH> pr = rp[d], qr = rq[d];
                // forward rows written since this sample's loads were issued (oldest first)
#pragma unroll
                for (int t = 0; t < D; t++) {
                    const int h = (d + t) % D;
                    if (hu[h] == ru[d]) pr = hp[h];
                    if (hv[h] == rv[d]) qr = hq[h];
                }
                float p[SH::E], q[SH::E];
                widen_row<SH>(pr, p);
                widen_row<SH>(qr, q);
                const float err = rr[d] - group_dot<SH>(p, q);
                if (val && !isfinite(err)) bad = 1;
                sgd_step<SH>(p, q, err, a.eta, a.lam);
                narrow_row<SH>(p, pr);
                narrow_row<SH>(q, qr);
                store_row<SH>(a.P, ru[d], k, lane, val, pr);
                store_row<SH>(a.Q, rv[d], k, lane, val, qr);
                hu[d] = val ? ru[d] : -1;
                hv[d] = val ? rv[d] : -1;
                hp[d] = pr;
                hq[d] = qr;
                // refill this slot with sample i + D (its triple is in the register tiles)
                const int64_t nx = i + D;
                if (nx - tb >= 32) {  // warp-uniform: the current tile is used up, slide by 32
                    tb += 32;
                    cu = nu, cv = nv, cr = nr;
                    const int64_t i1 = tb + 32 + lane;
                    nu = 0, nv = 0, nr = 0.f;
                    if (i1 < hi) nu = __ldg(a.u + i1), nv = __ldg(a.v + i1), nr = __ldg(a.r + i1);
                }
                const bool ok = nx < hi;
                int32_t tu_, tv_;
                float tr_;
                triple(nx, tu_, tv_, tr_);
                ru[d] = ok ? tu_ : 0;
                rv[d] = ok ? tv_ : 0;
                rr[d] = ok ? tr_ : 0.f;
                load_row<SH>(a.P, ru[d], k, lane, ok, rp[d]);
                load_row<SH>(a.Q, rv[d], k, lane, ok, rq[d]);
            }
        }
        if (a.trace && lane == 0) {
            int64_t *tr = a.trace + 4 * blk;
            tr[0] = w;
            tr[1] = blk;
            tr[2] = t0;
            tr[3] = globaltimer();
        }
        __threadfence();  // release: every lane's stores of this block before the unlock
        __syncwarp();
        if (lane == 0) atomicExch(lock, 0);
    }
    if (bad && lane == 0) a.scratch->diverged = 1;
    if (a.count_updates && lane == 0 && done) atomicAdd(&a.scratch->updates, done);
}

// ------------------------------------------------------------ CTA workers --
// MF_OPT_WAVE_CTA = 1: worker = one CTA of 1024 threads (one per SM).  While it holds column group c
// the group's Q rows are staged in shared memory, so every rating of the block reads and writes q_v
// on chip and only p_u (and the triple) crosses L2 -- half the L2 traffic of the warp-worker form.
// Inside the block the CTA's warps claim 32-sample tiles and update lock-free (batch-Hogwild! inside
// a block: P rows of the band and Q rows of the group are owned by this CTA alone).  The group is
// copied back to global memory before the column lock is released.
constexpr int kCtaThreads = 1024;
constexpr int64_t kCtaMinPerGroup = 16;  // in-block concurrency clamp: samples per concurrent group

// Q rows in shared memory are addressed with 32-bit shared-window offsets (ld/st.shared): no
// generic-to-shared conversion per access.  volatile keeps this thread's st before its next ld of
// the same row; other warps' races on a row are the lock-free semantics (batch-Hogwild! in a block).
template <int VB>
__device__ __forceinline__ void smem_ld(uint32_t a, uint32_t (&w)[Vec<VB>::NW]) {
    if constexpr (VB == 16) {
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(a));
    } else if constexpr (VB == 8) {
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(a));
    } else if constexpr (VB == 4) {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(a));
    } else {
        unsigned short h;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(a));
        w[0] = h;
    }
}
template <int VB>
__device__ __forceinline__ void smem_st(uint32_t a, const uint32_t (&w)[Vec<VB>::NW]) {
    if constexpr (VB == 16) {
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]));
    } else if constexpr (VB == 8) {
        asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(w[0]), "r"(w[1]));
    } else if constexpr (VB == 4) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(w[0]));
    } else {
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)(w[0] & 0xFFFFu)));
    }
}

// block-wide copy of nbytes (a multiple of 2) between global and shared memory
__device__ __forceinline__ void cta_copy_in(unsigned char *dst, const unsigned char *src, int64_t nbytes) {
    if (((nbytes | (int64_t)(uintptr_t)src) & 15) == 0) {
        for (int64_t i = threadIdx.x; i < nbytes / 16; i += blockDim.x)
            reinterpret_cast<uint4 *>(dst)[i] = __ldcg(reinterpret_cast<const uint4 *>(src) + i);
    } else {
        for (int64_t i = threadIdx.x; i < nbytes / 2; i += blockDim.x)
            reinterpret_cast<unsigned short *>(dst)[i] = __ldcg(reinterpret_cast<const unsigned short *>(src) + i);
    }
}
__device__ __forceinline__ void cta_copy_out(unsigned char *dst, const unsigned char *src, int64_t nbytes) {
    if (((nbytes | (int64_t)(uintptr_t)dst) & 15) == 0) {
        for (int64_t i = threadIdx.x; i < nbytes / 16; i += blockDim.x)
            __stcg(reinterpret_cast<uint4 *>(dst) + i, reinterpret_cast<const uint4 *>(src)[i]);
    } else {
        for (int64_t i = threadIdx.x; i < nbytes / 2; i += blockDim.x)
            __stcg(reinterpret_cast<unsigned short *>(dst) + i, reinterpret_cast<const unsigned short *>(src)[i]);
    }
}

// Bulk async staging of the Q group (the TMA engine's non-tensor copies, cp.async.bulk): one thread
// moves the whole group between global and shared memory in 64-KB pieces while the rest of the CTA
// waits on an mbarrier (copy-in) or proceeds (copy-out, which only the lock release waits for).  The
// thread-loop copy above keeps ~12 dependent 16-B loads per thread in sequence for a 200-KB group
// (12-14 us per block on the Yahoo shape, scripts/wavefront_timeline.py).  Needs 16-B aligned
// addresses and a 16-B multiple size.
__device__ __forceinline__ void mbar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_copy_in(uint32_t dst, const void *src, uint32_t nbytes, uint32_t bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nbytes) : "memory");
    for (uint32_t off = 0; off < nbytes; off += 65536u) {
        const uint32_t len = nbytes - off < 65536u ? nbytes - off : 65536u;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         dst + off),
                     "l"(reinterpret_cast<const char *>(src) + off), "r"(len), "r"(bar)
                     : "memory");
    }
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
}
__device__ __forceinline__ void bulk_copy_out(void *dst, uint32_t src, uint32_t nbytes) {
    for (uint32_t off = 0; off < nbytes; off += 65536u) {
        const uint32_t len = nbytes - off < 65536u ? nbytes - off : 65536u;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<char *>(dst) +
                                                                                          off),
                     "r"(src + off), "r"(len)
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // the writes are performed
    asm volatile("fence.proxy.async.global;" ::: "memory");    // ... and ordered before the release
}

// One 32-sample tile of a block (lane i of the warp holds sample base+i: tu, tv relative to the
// group's first column, tr).  G groups of L lanes, D ratings in flight per group.  FULLTILE: cnt == 32,
// no sample predicates (every tile but a block's last).  chk accumulates err * 0, which is NaN iff
// some err was not finite (one FFMA per rating instead of a compare-and-select).
template <class SH, int D, bool FULLTILE>
__device__ __forceinline__ void cta_tile(const WfArgs &a, uint32_t qbase, int k, int grp, int sub, int cnt,
                                         int32_t tu, int32_t tv, float tr, float &chk) {
    constexpr int G = SH::G;
    constexpr uint32_t kRowBytes = SH::FULL ? (uint32_t)(SH::KMAX * SH::BYTES) : 0u;
    const uint32_t row_bytes = SH::FULL ? kRowBytes : (uint32_t)k * SH::BYTES;
    const int per_group = FULLTILE ? 32 / G : (cnt + G - 1) / G;
#pragma unroll 1
    for (int j0 = 0; j0 < per_group; j0 += D) {
        int32_t su[D];
        uint32_t qa[D];
        float sr[D], dot[D];
        bool val[D];
        RowRaw<SH> pr[D], qr[D];
#pragma unroll
        for (int d = 0; d < D; d++) {
            const int s = (j0 + d) * G + grp;
            su[d] = __shfl_sync(0xffffffffu, tu, s);
            qa[d] = qbase + (uint32_t)__shfl_sync(0xffffffffu, tv, s) * row_bytes;
            sr[d] = __shfl_sync(0xffffffffu, tr, s);
            val[d] = FULLTILE || s < cnt;
            load_row<SH>(a.P, su[d], k, sub, val[d], pr[d]);
        }
#pragma unroll
        for (int d = 0; d < D; d++) {
            // Late Q read: the group's q_v is read from shared memory after p_u has arrived from L2 / DRAM
            // (an empty asm that consumes p_u's first word and "produces" the address), not when p_u's
            // load is issued.  128 groups share a column group of ~100 Q rows, so the read-to-write window
            // decides how many updates of a row overlap and are lost to a later store: it shrinks from
            // a global-load latency to the dot product and the update.
            if (a.q_late) asm volatile("" : "+r"(qa[d]) : "r"(pr[d].w[0][0]));
#pragma unroll
            for (int jv = 0; jv < SH::V; jv++) {
                const int e = (int)vec_elem<SH>(jv, sub);
                if (val[d] && (SH::FULL || e < k)) smem_ld<SH::VB>(qa[d] + (uint32_t)(e * SH::BYTES), qr[d].w[jv]);
                else
#pragma unroll
                    for (int x = 0; x < SH::NW; x++) qr[d].w[jv][x] = 0u;
            }
            float p[SH::E], q[SH::E];
            widen_row<SH>(pr[d], p);
            widen_row<SH>(qr[d], q);
            dot[d] = lane_dot<SH>(p, q);
        }
        group_allreduce<SH, D>(dot);
#pragma unroll
        for (int d = 0; d < D; d++) {
            const float err = sr[d] - dot[d];  // 0 for an invalid slot (zero rows, r = 0)
            chk = fmaf(err, 0.f, chk);
            // widen again from the raw rows instead of keeping D x 2E floats alive across the
            // butterfly (register cap of a 1024-thread CTA; free for fp32)
            float p[SH::E], q[SH::E];
            widen_row<SH>(pr[d], p);
            widen_row<SH>(qr[d], q);
            sgd_step<SH>(p, q, err, a.eta, a.lam);
            narrow_row<SH>(p, pr[d]);
            narrow_row<SH>(q, qr[d]);
            store_row<SH>(a.P, su[d], k, sub, val[d], pr[d]);
#pragma unroll
            for (int jv = 0; jv < SH::V; jv++) {
                const int e = (int)vec_elem<SH>(jv, sub);
                if (val[d] && (SH::FULL || e < k)) smem_st<SH::VB>(qa[d] + (uint32_t)(e * SH::BYTES), qr[d].w[jv]);
            }
        }
    }
}

template <class SH, int D, int THREADS>
__global__ void __launch_bounds__(THREADS, THREADS >= 1024 ? 1 : kCtaThreads / THREADS) k_wavefront_cta(WfArgs a) {
    extern __shared__ __align__(128) unsigned char qs[];
    __shared__ int s_col, s_next;
    __shared__ __align__(8) uint64_t s_bar;  // Q-group copy-in completion (a.tma)
    constexpr int L = SH::L;
    const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L;
    const int w = blockIdx.x;
    if (w >= a.s) return;  // CTA-uniform
    const int k = SH::FULL ? SH::KMAX : a.k;
    const int64_t row_bytes = (int64_t)k * SH::BYTES;
    const int c = a.c;
    const uint32_t qbase = (uint32_t)__cvta_generic_to_shared(qs);
    float chk = 0.f;
    unsigned long long done = 0;
    if (a.tma && threadIdx.x == 0) mbar_init((uint32_t)__cvta_generic_to_shared(&s_bar));
    __syncthreads();
    for (int pj = 0; pj < a.passes * c; pj++) {  // pass pj / c, wave pj % c
        if (threadIdx.x == 0) {
            const int col = wf_column(a, w, pj);
            while (atomicCAS(a.locks + col, 0, 1) != 0) __nanosleep(64);
            __threadfence();  // acquire
            s_col = col;
            s_next = 0;
        }
        __syncthreads();
        const int col = s_col;
        const int64_t q0 = seg_begin(a.n_cols, c, col);
        const int64_t nrows = seg_begin(a.n_cols, c, col + 1) - q0;
        const unsigned char *qg = reinterpret_cast<const unsigned char *>(a.Q) + q0 * row_bytes;
        if (a.tma) {
            if (threadIdx.x == 0) {
                asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired state -> async proxy
                bulk_copy_in(qbase, qg, (uint32_t)(nrows * row_bytes), (uint32_t)__cvta_generic_to_shared(&s_bar));
            }
            // every group has >= 1 row (c <= n), so block j completes the barrier's phase j.  A thread waits
            // for it just before its first rating of the block (the claim and the triple loads of its first
            // tile overlap the copy), or after the block's tiles if it gets none (a.q_wait_late = 0: here)
            if (!a.q_wait_late) mbar_wait((uint32_t)__cvta_generic_to_shared(&s_bar), (uint32_t)pj & 1u);
        } else {
            cta_copy_in(qs, qg, nrows * row_bytes);
            __syncthreads();
        }
        const int64_t t0 = a.trace ? globaltimer() : 0;
        const int64_t blk = ((int64_t)(pj / c) * a.s + w) * c + col;
        const int64_t lo = a.off[blk], hi = a.off[blk + 1];
        // 32-sample tiles.  (Claiming smaller tiles near the end of a block balances the warps but
        // raises the number of a small block's samples in flight at once -- more write conflicts on
        // the group's Q rows: C3-1pct test RMSE +2.0% vs +0.3%, and 4-7% slower on C2.  Prefetching the
        // next tile's triples costs registers under the 64-per-thread cap of a 1024-thread CTA: f16
        // spills and drops from 12.0 to 10.8 G updates/s on C2.)
        // In-block concurrency clamp (the A-10 reading applied inside a block): at most one group per
        // kCtaMinPerGroup samples of the block updates at a time, so every group processes >= that
        // many of the block's ratings.  Full-size shapes are not clamped (Netflix: 4,523 samples per
        // block for 128 groups; Yahoo: 2,184); 1% slices are (C3-1pct: 115 samples per block, where all
        // 128-256 groups at once left test RMSE +1.2..1.6% behind serial SGD at k = 32).
        bool q_in = !a.tma || !a.q_wait_late;  // this thread has seen the Q group's copy-in complete
        for (;;) {
            int t = 0x3fffffff;  // warp w claims iff w * G * kCtaMinPerGroup < block size (w = 0 always)
            if (lane == 0 && ((threadIdx.x >> 5) == 0 || (int64_t)(threadIdx.x >> 5) * SH::G * a.min_per_group < hi - lo))
                t = atomicAdd(&s_next, 32);
            const int64_t base = lo + __shfl_sync(0xffffffffu, t, 0);
            if (base >= hi) break;  // warp-uniform
            const int64_t i = base + lane;
            const bool ok = i < hi;
            const int32_t tu = ok ? __ldg(a.u + i) : 0;
            const int32_t tv = ok ? (int32_t)(__ldg(a.v + i) - q0) : 0;
            const float tr = ok ? __ldg(a.r + i) : 0.f;
            const int cnt = (int)(hi - base < 32 ? hi - base : 32);
            if (lane == 0) done += cnt;
            if (a.pf && ok) {
                // every lane asks L2 for its own sample's P row: the tile's later steps find their rows
                // on chip instead of waiting for DRAM one rating at a time
                const char *pp = reinterpret_cast<const char *>(a.P) + (int64_t)tu * row_bytes;
                if (a.pf == 1) {
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pp), "r"((uint32_t)row_bytes)
                                 : "memory");
                } else {
                    for (int64_t off = 0; off < row_bytes; off += 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(pp + off));
                }
            }
            if (!q_in) {
                mbar_wait((uint32_t)__cvta_generic_to_shared(&s_bar), (uint32_t)pj & 1u);
                q_in = true;
            }
            if (cnt == 32) cta_tile<SH, D, true>(a, qbase, k, grp, sub, cnt, tu, tv, tr, chk);
            else cta_tile<SH, D, false>(a, qbase, k, grp, sub, cnt, tu, tv, tr, chk);
        }
        if (!q_in) mbar_wait((uint32_t)__cvta_generic_to_shared(&s_bar), (uint32_t)pj & 1u);  // every phase, every thread
        if (a.tma) {
            // this thread's st.shared to the group must be visible to the async proxy that reads it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0)
                bulk_copy_out(reinterpret_cast<unsigned char *>(a.Q) + q0 * row_bytes, qbase, (uint32_t)(nrows * row_bytes));
        } else {
            __syncthreads();
            cta_copy_out(reinterpret_cast<unsigned char *>(a.Q) + q0 * row_bytes, qs, nrows * row_bytes);
        }
        if (a.trace && threadIdx.x == 0) {
            int64_t *tr = a.trace + 4 * blk;
            tr[0] = w;
            tr[1] = blk;
            tr[2] = t0;
            tr[3] = globaltimer();
        }
        __threadfence();  // release: P and Q stores of this block before the unlock
        __syncthreads();
        if (threadIdx.x == 0) atomicExch(a.locks + col, 0);
    }
    if (chk != chk) a.scratch->diverged = 1;
    if (a.count_updates && lane == 0 && done) atomicAdd(&a.scratch->updates, done);
}

template <class F>
cudaError_t dispatch_cta_shape(const ShapeId &s, F &&f) {
#define MF_CCASE(S_, L_, V_, VB_, FULL_)                                                             \
    if (s.storage == S_ && s.L == L_ && s.V == V_ && s.VB == VB_ && s.full == FULL_)                \
        return f(Shape<S_, L_, V_, VB_, (bool)FULL_>{});
    MF_CCASE(kF32, 8, 1, 16, 1) MF_CCASE(kF32, 16, 1, 16, 1) MF_CCASE(kF32, 32, 1, 16, 1)
    MF_CCASE(kF32, 32, 2, 16, 1) MF_CCASE(kF32, 16, 2, 16, 1) MF_CCASE(kF32, 8, 4, 16, 1)
    MF_CCASE(kF16, 8, 2, 16, 1) MF_CCASE(kF16, 4, 4, 16, 1) MF_CCASE(kBF16, 8, 2, 16, 1) MF_CCASE(kBF16, 4, 4, 16, 1) MF_CCASE(kF16, 4, 1, 16, 1) MF_CCASE(kF16, 8, 1, 16, 1)
    MF_CCASE(kF16, 16, 1, 16, 1) MF_CCASE(kF16, 32, 1, 16, 1) MF_CCASE(kBF16, 4, 1, 16, 1)
    MF_CCASE(kBF16, 8, 1, 16, 1) MF_CCASE(kBF16, 16, 1, 16, 1) MF_CCASE(kBF16, 32, 1, 16, 1)
    MF_CCASE(kF32, 32, 1, 4, 0) MF_CCASE(kF32, 32, 4, 4, 0) MF_CCASE(kF32, 32, 16, 4, 0) MF_CCASE(kF32, 32, 32, 4, 0)
    MF_CCASE(kF16, 32, 1, 4, 0) MF_CCASE(kF16, 32, 4, 4, 0) MF_CCASE(kF16, 32, 16, 4, 0)
    MF_CCASE(kF16, 32, 1, 2, 0) MF_CCASE(kF16, 32, 4, 2, 0) MF_CCASE(kF16, 32, 16, 2, 0) MF_CCASE(kF16, 32, 32, 2, 0)
    MF_CCASE(kBF16, 32, 1, 4, 0) MF_CCASE(kBF16, 32, 4, 4, 0) MF_CCASE(kBF16, 32, 16, 4, 0)
    MF_CCASE(kBF16, 32, 1, 2, 0) MF_CCASE(kBF16, 32, 4, 2, 0) MF_CCASE(kBF16, 32, 16, 2, 0) MF_CCASE(kBF16, 32, 32, 2, 0)
#undef MF_CCASE
    return cudaErrorInvalidValue;
}

// ------------------------------------------------- q-stationary CTA workers --
// MF_OPT_WAVE_CTA = 3: worker = one 1024-thread CTA per SM holding column group c (the column lock as in
// the other forms).  The block's samples are sorted by Q row (stable, so each row's samples keep the
// shuffled order): the block is a set of runs, one per Q row.  The CTA's warps claim runs; a warp keeps
// its run's q_v in registers for the whole run (q_v is touched by no other warp or CTA while the column
// lock is held) and streams the run's p_u rows, D of them in flight, with register forwarding when a
// p_u repeats inside the ring (a duplicate rating).  So no two concurrent updates ever share a Q row
// -- the in-block Hogwild! races of the staged form (128 ratings in flight on a ~120-row group on the
// Netflix shape) are gone -- and only p_u (read + write) and the triples cross L2 per rating; q_v
// crosses once per run.  Each sample's update is exactly the paper's from the snapshot
// (p_u, q_v); q_v is rounded to storage after every update, as the serial oracle does.  Runs of
// different warps race only on P rows they share (a user with two items of the group).
template <class SH, int D, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_wavefront_q(WfArgs a) {
    static_assert(SH::L == 32, "a run is processed by one full warp");
    extern __shared__ int32_t run_start[];  // nrows + 1 entries for the current block
    __shared__ int s_col, s_next;
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.x;
    if (w >= a.s) return;  // CTA-uniform
    const int k = SH::FULL ? SH::KMAX : a.k;
    const int c = a.c;
    const int nthreads = blockDim.x;
    const int active_warps = a.min_per_group > 0 ? a.min_per_group : THREADS / 32;  // warps claiming runs
    float chk = 0.f;
    unsigned long long done = 0;
    for (int pj = 0; pj < a.passes * c; pj++) {  // pass pj / c, wave pj % c
        if (threadIdx.x == 0) {
            const int col = wf_column(a, w, pj);
            lock_acquire(a.locks + col);
            __threadfence();  // acquire
            s_col = col;
            s_next = 0;
        }
        __syncthreads();
        const int col = s_col;
        const int64_t q0 = seg_begin(a.n_cols, c, col);
        const int nrows = (int)(seg_begin(a.n_cols, c, col + 1) - q0);
        const int64_t blk = ((int64_t)(pj / c) * a.s + w) * c + col;
        const int64_t lo = a.off[blk], hi = a.off[blk + 1];
        const int64_t t0 = a.trace ? globaltimer() : 0;
        // run table: run_start[r] = first block position whose Q row is >= q0 + r, r in [0, nrows]
        for (int64_t i = lo + threadIdx.x; i < hi; i += nthreads) {
            const int vl = (int)(__ldg(a.v + i) - q0);
            const int prev = i > lo ? (int)(__ldg(a.v + i - 1) - q0) : -1;
            for (int rr = prev + 1; rr <= vl; rr++) run_start[rr] = (int)(i - lo);
        }
        {
            const int last = hi > lo ? (int)(__ldg(a.v + hi - 1) - q0) : -1;
            for (int rr = last + 1 + (int)threadIdx.x; rr <= nrows; rr += nthreads) run_start[rr] = (int)(hi - lo);
        }
        __syncthreads();
        {
            const bool claims = (int)(threadIdx.x >> 5) < active_warps;
            for (;;) {
                int r = nrows;
                if (lane == 0 && claims) r = atomicAdd(&s_next, 1);
                r = __shfl_sync(0xffffffffu, r, 0);
                if (r >= nrows) break;  // warp-uniform
                const int64_t rb = lo + run_start[r], re = lo + run_start[r + 1];
                if (rb == re) continue;
                const int64_t vrow = q0 + r;
                done += (uint64_t)(re - rb);
                RowRaw<SH> qraw;
                load_row<SH>(a.Q, vrow, k, lane, true, qraw);
                // triples of the run from two 32-sample register tiles (lane i: sample tb + i)
                int64_t tb = rb;
                int32_t cu = 0, nu = 0;
                float cr = 0.f, nr = 0.f;
                {
                    const int64_t i0 = rb + lane, i1 = rb + 32 + lane;
                    if (i0 < re) cu = __ldg(a.u + i0), cr = __ldg(a.r + i0);
                    if (i1 < re) nu = __ldg(a.u + i1), nr = __ldg(a.r + i1);
                }
                auto triple = [&](int64_t jj, int32_t &uu, float &rr_) {
                    const int o = (int)(jj - tb);
                    const bool in_cur = o < 32;
                    uu = __shfl_sync(0xffffffffu, in_cur ? cu : nu, o & 31);
                    rr_ = __shfl_sync(0xffffffffu, in_cur ? cr : nr, o & 31);
                };
                int32_t ru[D], hu[D];
                float rr[D];
                RowRaw<SH> rp[D];
#pragma unroll
                for (int d = 0; d < D; d++) {
                    hu[d] = -1;
                    const bool ok = rb + d < re;
                    int32_t tu_;
                    float tr_;
                    triple(rb + d, tu_, tr_);
                    ru[d] = ok ? tu_ : 0;
                    rr[d] = ok ? tr_ : 0.f;
                    load_row<SH>(a.P, ru[d], k, lane, ok, rp[d]);
                }
                float q[SH::E];
                widen_row<SH>(qraw, q);
                for (int64_t base = rb; base < re; base += D) {
#pragma unroll
                    for (int d = 0; d < D; d++) {  // branch-free: every lane reaches every shuffle
                        const int64_t i = base + d;
                        const bool val = i < re;
                        RowRaw<SH> pr = rp[d];
                        // p_u written by one of the D - 1 samples since this load was issued (a
                        // duplicate rating inside the ring, rare): read it again -- the same lanes
                        // stored it, so program order makes the new value visible
                        bool hit = false;
#pragma unroll
                        for (int t = 1; t < D; t++) hit |= hu[(d + t) % D] == ru[d];
                        if (val && hit) load_row<SH>(a.P, ru[d], k, lane, true, pr);
                        float p[SH::E];
                        widen_row<SH>(pr, p);
                        const float err = rr[d] - group_dot<SH>(p, q);
                        if (val) {
                            chk = fmaf(err, 0.f, chk);
                            float qn[SH::E];
#pragma unroll
                            for (int e = 0; e < SH::E; e++) qn[e] = q[e];
                            sgd_step<SH>(p, qn, err, a.eta, a.lam);
                            narrow_row<SH>(p, pr);
                            narrow_row<SH>(qn, qraw);
                            widen_row<SH>(qraw, q);  // q_v as stored after this update (serial semantics)
                            store_row<SH>(a.P, ru[d], k, lane, true, pr);
                        }
                        hu[d] = val ? ru[d] : -1;
                        const int64_t nx = i + D;
                        if (nx - tb >= 32) {  // warp-uniform: slide the triple tiles
                            tb += 32;
                            cu = nu, cr = nr;
                            const int64_t i1 = tb + 32 + lane;
                            nu = 0, nr = 0.f;
                            if (i1 < re) nu = __ldg(a.u + i1), nr = __ldg(a.r + i1);
                        }
                        const bool ok = nx < re;
                        int32_t tu_;
                        float tr_;
                        triple(nx, tu_, tr_);
                        ru[d] = ok ? tu_ : 0;
                        rr[d] = ok ? tr_ : 0.f;
                        load_row<SH>(a.P, ru[d], k, lane, ok, rp[d]);
                    }
                }
                store_row<SH>(a.Q, vrow, k, lane, true, qraw);
            }
        }
        if (a.trace && threadIdx.x == 0) {
            int64_t *tr = a.trace + 4 * blk;
            tr[0] = w;
            tr[1] = blk;
            tr[2] = t0;
            tr[3] = globaltimer();
        }
        __threadfence();  // release: every thread's P and Q stores of this block before the unlock
        __syncthreads();
        if (threadIdx.x == 0) atomicExch(a.locks + col, 0);
    }
    if (chk != chk) a.scratch->diverged = 1;
    if (a.count_updates && lane == 0 && done) atomicAdd(&a.scratch->updates, done);
}

ShapeId warp_shape(int k, int storage) {
    if (storage == kF32) {
        if (k == 128) return {storage, 32, 1, 16, 1};
        if (k == 256) return {storage, 32, 2, 16, 1};
    } else {
        if (k == 128) return {storage, 32, 1, 8, 1};
        if (k == 256) return {storage, 32, 1, 16, 1};
    }
    return select_generic_shape(k, storage);  // L = 32, masked
}

template <class F>
cudaError_t dispatch_warp_shape(const ShapeId &s, F &&f) {
#define MF_WCASE(S_, V_, VB_, FULL_)                                                               \
    if (s.storage == S_ && s.L == 32 && s.V == V_ && s.VB == VB_ && s.full == FULL_)              \
        return f(Shape<S_, 32, V_, VB_, (bool)FULL_>{});
    MF_WCASE(kF32, 1, 16, 1) MF_WCASE(kF32, 2, 16, 1) MF_WCASE(kF16, 1, 8, 1) MF_WCASE(kF16, 1, 16, 1)
    MF_WCASE(kBF16, 1, 8, 1) MF_WCASE(kBF16, 1, 16, 1)
    MF_WCASE(kF32, 1, 4, 0) MF_WCASE(kF32, 4, 4, 0) MF_WCASE(kF32, 16, 4, 0) MF_WCASE(kF32, 32, 4, 0)
    MF_WCASE(kF16, 1, 4, 0) MF_WCASE(kF16, 4, 4, 0) MF_WCASE(kF16, 16, 4, 0)
    MF_WCASE(kF16, 1, 2, 0) MF_WCASE(kF16, 4, 2, 0) MF_WCASE(kF16, 16, 2, 0) MF_WCASE(kF16, 32, 2, 0)
    MF_WCASE(kBF16, 1, 4, 0) MF_WCASE(kBF16, 4, 4, 0) MF_WCASE(kBF16, 16, 4, 0)
    MF_WCASE(kBF16, 1, 2, 0) MF_WCASE(kBF16, 4, 2, 0) MF_WCASE(kBF16, 16, 2, 0) MF_WCASE(kBF16, 32, 2, 0)
#undef MF_WCASE
    return cudaErrorInvalidValue;
}

}  // namespace

#define CK(expr)                                   \
    do {                                           \
        int _rc = cuda((expr), #expr);             \
        if (_rc != MF_OK) return _rc;              \
    } while (0)

void mf_ctx::release_wavefront() {
    for (void *p : {(void *)fu, (void *)fv, (void *)fr, (void *)wf_off, (void *)wf_locks, (void *)wf_seq,
                    (void *)wf_trace})
        if (p) cudaFree(p);
    fu = fv = nullptr;
    fr = nullptr;
    wf_off = nullptr;
    wf_locks = wf_seq = nullptr;
    wf_trace = nullptr;
    wf_trace_n = 0;
    wf_valid = false;
}

// Auto sizing: up to 16 warp workers per SM, c = 1.25 s column blocks (Latin-rectangle
// lock utilisation ~95% at that ratio), blocks of >= ~14 samples, s <= m, c <= n.
int mf_ctx::build_wavefront() {
    if (wf_valid) return MF_OK;
    release_wavefront();
    const int64_t rows = p_rows();
    int s = wave_rows, c = wave_cols;
    if (wave_cta == 3) {
        // q-stationary CTA workers: one per SM, c = s column groups (as many as the run table of a group,
        // 4 B per Q row in shared memory, allows: <= 48K rows per group)
        if (s <= 0) s = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms, rows));
        if (c <= 0) {
            int64_t cc = std::min<int64_t>((int64_t)s, n);
            while (cc < n && (n + cc - 1) / cc > 48 * 1024) cc++;
            c = (int)cc;
        }
    } else if (wave_cta) {
        // one CTA worker per SM; c = s column groups (the largest blocks: per-block lock, copy-in and
        // tail cost is amortised best -- Netflix shape, f16: c = s 11.8 G/s, 2s 10.0, 4s 7.7, 8s 6.2),
        // more if the largest group does not fit in shared memory (200 KB of the 227 KB per CTA)
        if (s <= 0) s = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms * (wave_cta == 2 ? 2 : 1), rows));
        if (c <= 0) {
            const int64_t row_bytes = (int64_t)k * storage_bytes();
            const int64_t fit = std::max<int64_t>(1, (200 * 1024) / row_bytes);
            int64_t cc = std::min<int64_t>((int64_t)s, n);
            while (cc < n && (n + cc - 1) / cc > fit) cc++;
            c = (int)cc;
        }
    }
    const bool warp_auto = !wave_cta && s <= 0;
    if (s <= 0) {
        // warp workers (one-warp CTAs): up to 16 per SM (2,368 on a B200) with c = 1.25 s column blocks
        // (the Latin rectangle keeps ~95% of the workers busy at that ratio), blocks of >= ~14 samples:
        // s = sqrt(N / 17.5).  Netflix shape f16: s / c = 1,184 / 2,368 2.19 G updates/s, 2,368 / 2,960
        // 3.08-3.13, 3,552 / 4,440 3.06, 4,736 / 5,920 2.87 (profiles/r02h_warp_*, r02i_warp_*)
        const double by_blocks = std::sqrt((double)N / 17.5);
        // (and c = 1.25 s column groups must exist: s <= 0.8 n on narrow matrices)
        s = (int)std::max<double>(1.0, std::min<double>({(double)num_sms * 16, by_blocks, (double)rows,
                                                         std::floor(0.8 * (double)n)}));
    }
    if (c <= 0) c = (int)std::min<int64_t>(warp_auto ? std::max<int64_t>(s, (5 * (int64_t)s + 3) / 4) : 2 * (int64_t)s, n);
    if (s > rows || c > n || s < 1 || c < s)
        return fail(MF_EINVAL, "wavefront needs 1 <= s <= c, s <= m, c <= n (s=%d c=%d)", s, c);
    // Passes per epoch (MF_OPT_WAVE_PASSES): each pass walks every worker through all c column groups with
    // fresh sequences, over 1/P of the shuffled samples.  With one pass every row band meets the column
    // groups in one fixed cyclic order per epoch -- each user's ratings are processed sorted by column
    // group -- and the wavefront trails serial SGD: on the Hugewiki shape it never catches up (test RMSE
    // after 5 epochs: CTA workers 0.40-0.51, warp workers +13% after 4; serial 0.1675), on the Netflix
    // shape it is +265% after epoch 1 and +11% after epoch 2.  P passes split each user's ratings into P
    // slices visited in independent orders (profiles/r02r_*, r02v_*):
    //  - CTA workers: P = 1 + round(log2(V / 10)) (at least 1), V = N / (n s) the updates a Q row takes per
    //    visit in one pass -- an empirical rule fitted to the three shapes: Netflix V = 38 -> P = 3 (fp16:
    //    +1.7% / +0.04% after epochs 1 / 2 and within 0.42% to epoch 20 at +9% time over P = 2, which was
    //    +6.5% / +0.46% and +0.51% at epoch 20; profiles/r02ak_c2_f16.jsonl), Yahoo V = 2.7 -> 1 (within
    //    0.5% from epoch 2 already; P = 2 would cost 54%), Hugewiki V = 521 -> 7 (P = 8: serial SGD's
    //    trajectory at +7% time; P = 10: the same test RMSE after 5 epochs at +11% time over 7, r02al;
    //    P = 32: +1..2% behind and +35% time);
    //  - warp workers (blocks of ~14-450 samples): as many passes as keep blocks at >= 64 samples
    //    (Hugewiki 6, Netflix and Yahoo 1; each block costs a lock hand-over).
    int npass_auto = 1;
    {
        const double per_block = (double)N / ((double)s * (double)c);
        if (wave_cta) {
            const double V = (double)N / ((double)n * (double)s);
            npass_auto = (int)std::max(1.0, std::min(64.0, 1.0 + std::floor(std::log2(V / 10.0) + 0.5)));
            while (npass_auto > 1 && per_block / npass_auto < 512.0) npass_auto--;  // keep blocks >= 512 samples
        } else {
            npass_auto = (int)std::max(1.0, std::min(64.0, std::floor(per_block / 64.0)));
        }
    }
    const int npass = (int)std::max<int64_t>(1, std::min<int64_t>(wave_passes > 0 ? wave_passes : npass_auto,
                                                                  std::max<int64_t>(1, N)));
    if ((int64_t)npass * s * c >= (1ll << 32)) return fail(MF_EINVAL, "wavefront grid P*s*c too large");
    cudaStream_t st = stream();
    const int64_t nb = (int64_t)npass * s * c;
    uint32_t *k0 = nullptr, *k1 = nullptr, *i0 = nullptr, *i1 = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    CK(cudaMalloc((void **)&fu, sizeof(int32_t) * N));
    CK(cudaMalloc((void **)&fv, sizeof(int32_t) * N));
    CK(cudaMalloc((void **)&fr, sizeof(float) * N));
    CK(cudaMalloc((void **)&wf_off, sizeof(int64_t) * (nb + 1)));
    CK(cudaMalloc((void **)&wf_locks, sizeof(int32_t) * c));
    CK(cudaMallocAsync((void **)&k0, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&k1, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&i0, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&i1, sizeof(uint32_t) * N, st));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 148 * 16));
    const bool runs = wave_cta == 3;
    const uint64_t key_range = runs ? (uint64_t)npass * s * (uint64_t)n : (uint64_t)nb;
    if (key_range >= (1ull << 32)) return fail(MF_EINVAL, "wavefront: P * s * n too large for the run layout");
    if (runs) k_run_keys<<<grid, 256, 0, st>>>(u, v, N, rows, n, s, npass, k0, i0);
    else k_block_keys<<<grid, 256, 0, st>>>(u, v, N, rows, n, s, c, npass, k0, i0);
    CK(cudaGetLastError());
    int bits = 1;
    while (bits < 32 && (1ull << bits) < key_range) bits++;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, i0, i1, N, 0, bits, st));
    CK(cudaMallocAsync(&tmp, tmp_bytes, st));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i0, i1, N, 0, bits, st));  // stable
    if (runs) k_run_block_offsets<<<grid, 256, 0, st>>>(k1, N, nb, c, n, wf_off);
    else k_block_offsets<<<grid, 256, 0, st>>>(k1, N, nb, wf_off);
    CK(cudaGetLastError());
    CK(launch_gather(u, v, r, i1, N, fu, fv, fr, st));
    CK(cudaFreeAsync(tmp, st));
    CK(cudaFreeAsync(k0, st));
    CK(cudaFreeAsync(k1, st));
    CK(cudaFreeAsync(i0, st));
    CK(cudaFreeAsync(i1, st));
    CK(cudaMemsetAsync(wf_locks, 0, sizeof(int32_t) * c, st));
    CK(cudaStreamSynchronize(st));
    wf_s = s;
    wf_c = c;
    wf_p = npass;
    wf_valid = true;
    return MF_OK;
}

int mf_ctx::run_wavefront(const ShapeId &, const UpdateArgs &ua, int *launches, int *workers_used) {
    cudaStream_t st = stream();
    const int s = wf_s, c = wf_c, npass = wf_p;
    // column sequences for this epoch, one set per pass (host, counter-hash Fisher-Yates keyed by seed, epoch
    // and pass; pass 0's key is the single-pass key)
    std::vector<int32_t> seq;
    for (int p = 0; p < npass; p++) {
        const uint64_t key = host_mix(seed_shuffle ^ 0x5eedull ^ ((uint64_t)epoch << 32) ^ ((uint64_t)p << 20));
        if (wave_perm == 0) {
            std::vector<int32_t> sigma, rho;
            permutation(sigma, c, key);
            permutation(rho, c, host_mix(key + 1));
            seq.insert(seq.end(), sigma.begin(), sigma.end());
            seq.insert(seq.end(), rho.begin(), rho.begin() + s);
        } else {
            std::vector<int32_t> pw;
            for (int w = 0; w < s; w++) {
                permutation(pw, c, host_mix(key + 2 + (uint64_t)w));
                seq.insert(seq.end(), pw.begin(), pw.end());
            }
        }
    }
    if (wf_seq) cudaFree(wf_seq);
    wf_seq = nullptr;
    CK(cudaMalloc((void **)&wf_seq, sizeof(int32_t) * seq.size()));
    CK(cudaMemcpyAsync(wf_seq, seq.data(), sizeof(int32_t) * seq.size(), cudaMemcpyHostToDevice, st));
    const int64_t nb = (int64_t)npass * s * c;
    if (trace) {
        if (wf_trace_n != nb) {
            if (wf_trace) cudaFree(wf_trace);
            wf_trace = nullptr;
            CK(cudaMalloc((void **)&wf_trace, sizeof(int64_t) * 4 * nb));
            wf_trace_n = nb;
        }
        CK(cudaMemsetAsync(wf_trace, 0xFF, sizeof(int64_t) * 4 * nb, st));
    }
    WfArgs a{};
    a.u = fu;
    a.v = fv;
    a.r = fr;
    a.off = wf_off;
    a.seq = wf_seq;
    a.locks = wf_locks;
    a.P = P;
    a.Q = Q;
    a.trace = trace ? wf_trace : nullptr;
    a.scratch = scratch;
    a.s = s;
    a.c = c;
    a.passes = npass;
    a.k = k;
    a.latin = wave_perm == 0;
    a.count_updates = count_updates;
    a.eta = ua.eta;
    a.lam = ua.lam;
    a.n_cols = n;
    if (wave_cta == 3) {
        const size_t smem = (size_t)((n + c - 1) / c + 1) * sizeof(int32_t);  // run table
        // MF_OPT_VARIANT bits 26..27: warps claiming runs, 0 -> all, 1 -> 1 (one run at a time: the block
        // is processed serially in run order), 2 -> 8, 3 -> 16; bits 4..7: p rows in flight per warp,
        // 0 -> 4 (1024-thread CTA, 128 rows in flight per SM, 64 registers), 8 -> 8 (512-thread CTA,
        // the same 128 in flight, 128 registers), 2 -> 2 (1024 threads)
        {
            const int sel = (variant_eff >> 26) & 0x3;
            a.min_per_group = sel == 0 ? 0 : sel == 1 ? 1 : sel == 2 ? 8 : 16;
        }
        const int dsel = (variant_eff >> 4) & 0xF;
        const int depth = dsel == 2 || dsel == 8 ? dsel : 4;
        const ShapeId sh = warp_shape(k, storage);
        CK(dispatch_warp_shape(sh, [&](auto tag) -> cudaError_t {
            using SH = decltype(tag);
            auto launch = [&](auto kern, int threads) -> cudaError_t {
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
                kern<<<s, threads, smem, st>>>(a);
                return cudaGetLastError();
            };
            if constexpr (SH::FULL) {
                if (depth == 8) return launch(k_wavefront_q<SH, 8, 512>, 512);
                if (depth == 4) return launch(k_wavefront_q<SH, 4, 1024>, 1024);
            }
            return launch(k_wavefront_q<SH, 2, 1024>, 1024);
        }));
    } else if (wave_cta) {
        const int64_t row_bytes = (int64_t)k * storage_bytes();
        const int64_t max_rows = (n + c - 1) / c;  // balanced column groups
        const size_t smem = (size_t)(max_rows * row_bytes);
        if (smem > 227 * 1024) return fail(MF_EINVAL, "wavefront CTA: column group needs %zu B of shared memory", smem);
        // MF_OPT_VARIANT bits 8..11: 0 = tuned default, else the update shape select_shape(variant - 1)
        // (lanes per rating); bits 12..15: ratings in flight per group, 0 = default, 1 or 2.  Defaults
        // (r01, C2): k = 128 uses 8 lanes per rating (16 halves or 16 floats per lane) with one rating
        // in flight -- fewer butterfly levels and broadcast shuffles per rating than the 16/32-lane
        // shapes of batch-Hogwild! (f16 12.4 -> 13.6, f32 6.5 -> 7.7 G updates/s; profiles/r01_cta_shapes.log).
        const int shape_sel = (variant_eff >> 8) & 0xF, depth_sel = (variant_eff >> 12) & 0xF;
        // bits 16..19: P-row L2 prefetch per claimed tile (1 = bulk, 2 = per 128-B line, 0 / 15 = off;
        // bulk needs 16-B multiple rows; mf_epoch resolves the auto value 0 before this point)
        {
            const int pf = (variant_eff >> 16) & 0xF;
            a.pf = pf == 1 || pf == 2 ? pf : 0;
        }
        if (a.pf == 1 && row_bytes % 16) a.pf = 2;
        {  // bits 26..27: in-block clamp, samples per concurrent group 0 -> 16, 1 -> 32, 2 -> 64, 3 -> 8
            const int sel = (variant_eff >> 26) & 0x3;
            a.min_per_group = sel == 0 ? (int)kCtaMinPerGroup : sel == 1 ? 32 : sel == 2 ? 64 : 8;
        }
        // bit 22: 1 = read q_v from shared memory when p_u's load is issued (before r02ab), else once p_u
        // has arrived (default: a shorter race window on the group's Q rows)
        a.q_late = ((variant_eff >> 22) & 0x1) == 0;
        // bit 23: 1 = wait for the Q group's copy-in before claiming tiles (before r02ao), else at a thread's
        // first rating of the block, so the tile claim and triple loads overlap the copy
        a.q_wait_late = ((variant_eff >> 23) & 0x1) == 0;
        // bits 20..21: Q-group staging, 0 = bulk async copies when rows are 16-B multiples, 2 = thread loop
        a.tma = ((variant_eff >> 20) & 0x3) != 2 && row_bytes % 16 == 0 && ((uintptr_t)Q & 15) == 0;
        // (k = 32 / 64 keep the 16-byte-vector shapes: 4 / 8 lanes (16-bit rows), 8 / 16 lanes (fp32) --
        // batch-Hogwild!'s 16-lane narrow-vector defaults for those k are not CTA-worker shapes)
        const int def_shape = k == 128  ? (storage == kF32 ? 2 : 1)
                              : k == 32 ? (storage == kF32 ? 1 : 2)
                              : k == 64 ? (storage == kF32 ? 0 : 1)
                                        : 0;
        const ShapeId sh = select_shape(k, storage, shape_sel ? shape_sel - 1 : def_shape);
        const bool one_in_flight = depth_sel ? depth_sel == 1 : (k == 128 && !shape_sel);
        CK(dispatch_cta_shape(sh, [&](auto tag) -> cudaError_t {
            using SH = decltype(tag);
            constexpr int DD = (SH::FULL && (32 / SH::G) % 2 == 0) ? 2 : 1;  // 2 ratings in flight per group
            auto launch = [&](auto kern, int threads) -> cudaError_t {
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)std::max<size_t>(smem, 16));
                if (e != cudaSuccess) return e;
                kern<<<s, threads, std::max<size_t>(smem, 16), st>>>(a);
                return cudaGetLastError();
            };
            // MF_OPT_WAVE_CTA = 2: two 512-thread workers per SM, so one's block boundary (write-back,
            // lock hand-over, staging) overlaps the other's updates
            // (a 768-thread worker -- 85 registers, no spills -- measured 8% slower than 1024)
            if constexpr (DD == 2) {
                if (one_in_flight && wave_cta == 2) return launch(k_wavefront_cta<SH, 1, 512>, 512);
                if (one_in_flight) return launch(k_wavefront_cta<SH, 1, 1024>, 1024);
            }
            if (wave_cta == 2) return launch(k_wavefront_cta<SH, DD, 512>, 512);
            return launch(k_wavefront_cta<SH, DD, 1024>, 1024);
        }));
    } else {
        const ShapeId sh = warp_shape(k, storage);
        // samples of a block in flight per warp (MF_OPT_VARIANT bits 4..7: 2, 4 or 8; 0 = 2).  The triples
        // come from two 32-sample register tiles fetched before the lock, so the only latency on a sample's
        // path is its row loads, issued `depth` samples ahead (Netflix shape, s = 2,368: f16 D = 2 3.14 vs
        // D = 4 2.94 G updates/s, fp32 2.63 vs 2.43; profiles/r02j_warp_C2.log)
        const int dsel = (variant_eff >> 4) & 0xF;
        const int depth = dsel == 4 || dsel == 8 ? dsel : 2;
        CK(dispatch_warp_shape(sh, [&](auto tag) -> cudaError_t {
            using SH = decltype(tag);
            if constexpr (SH::FULL) {
                if (depth == 8) {
                    k_wavefront<SH, 8><<<s, 32, 0, st>>>(a);
                    return cudaGetLastError();
                }
                if (depth == 4) {
                    k_wavefront<SH, 4><<<s, 32, 0, st>>>(a);
                    return cudaGetLastError();
                }
            }
            k_wavefront<SH, 2><<<s, 32, 0, st>>>(a);
            return cudaGetLastError();
        }));
    }
    *launches = 1;
    *workers_used = s;
    return MF_OK;
}

extern "C" int mf_wavefront_trace(mf_ctx *ctx, int64_t *records, int64_t cap, int64_t *count) {
    if (!ctx || !count || (cap > 0 && !records)) return MF_EINVAL;
    *count = 0;
    if (!ctx->wf_trace || ctx->wf_trace_n == 0) return MF_OK;
    const int64_t nrec = std::min<int64_t>(cap, ctx->wf_trace_n);
    std::vector<int64_t> h((size_t)(4 * ctx->wf_trace_n));
    int rc = ctx->cuda(cudaMemcpy(h.data(), ctx->wf_trace, sizeof(int64_t) * h.size(), cudaMemcpyDeviceToHost),
                       "trace copy");
    if (rc != MF_OK) return rc;
    int64_t o = 0;
    for (int64_t b = 0; b < ctx->wf_trace_n && o < nrec; b++) {
        if (h[(size_t)(4 * b)] < 0) continue;  // block not visited (never happens after a full epoch)
        std::copy(h.begin() + 4 * b, h.begin() + 4 * b + 4, records + 4 * o);
        o++;
    }
    *count = o;
    return MF_OK;
}
