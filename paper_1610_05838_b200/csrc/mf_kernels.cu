// mf_kernels.cu -- sm_100a kernels of the SGD-MF hot path and their launchers.
//
//   k_hogwild  batch-Hogwild! (§3.2.2): persistent warps claim
//              chunks of f consecutive shuffled samples with one atomic per
//              chunk and update them lock-free; each L-lane group keeps D
//              ratings in flight.
//   k_waves    deterministic conflict-free waves (D-3): one persistent
//              cooperative kernel, samples pre-sorted by wave, grid barrier
//              between waves.
//   k_rmse     test RMSE: fp32 dot, fp64 squared error, fixed
//              two-level reduction (deterministic).
//   k_init     A-7 counter-hash initialisation.
//   k_validate index range / finite rating check.
//   shuffle    A-8 hash-key radix sort (CUB) + gather.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>

#include "mf_kernels.cuh"
#include "sgd_core.cuh"

namespace mf {

static constexpr int kBlock = 256;  // 8 warps per CTA
static constexpr int kWarpsPerBlock = kBlock / 32;

// ------------------------------------------------------------------ shapes --
// Shape table: (storage, L, V, VB, full).  Fast shapes cover k = L*V*VB/bytes
// exactly; generic shapes (full = 0) mask lanes beyond k.
#define MF_FAST_SHAPES(X)                                                                                \
    X(kF32, 8, 1, 16, 1) X(kF32, 16, 1, 16, 1) X(kF32, 32, 1, 16, 1) X(kF32, 32, 2, 16, 1)               \
    X(kF32, 16, 2, 16, 1) X(kF32, 8, 4, 16, 1) X(kF32, 16, 1, 8, 1) X(kF32, 32, 1, 8, 1) X(kF32, 32, 1, 4, 1) \
    X(kF16, 4, 1, 16, 1) X(kF16, 8, 1, 16, 1) X(kF16, 16, 1, 16, 1) X(kF16, 32, 1, 16, 1)                \
    X(kF16, 8, 2, 16, 1) X(kF16, 32, 1, 8, 1) X(kF16, 4, 4, 16, 1) X(kF16, 8, 1, 8, 1) X(kF16, 16, 1, 4, 1) \
    X(kF16, 16, 1, 8, 1) X(kF16, 32, 1, 4, 1)                                                            \
    X(kBF16, 4, 1, 16, 1) X(kBF16, 8, 1, 16, 1) X(kBF16, 16, 1, 16, 1) X(kBF16, 32, 1, 16, 1)            \
    X(kBF16, 8, 2, 16, 1) X(kBF16, 32, 1, 8, 1) X(kBF16, 4, 4, 16, 1) X(kBF16, 8, 1, 8, 1)              \
    X(kBF16, 16, 1, 4, 1) X(kBF16, 16, 1, 8, 1) X(kBF16, 32, 1, 4, 1)
#define MF_GENERIC_SHAPES(X)                                                                             \
    X(kF32, 32, 1, 4, 0) X(kF32, 32, 4, 4, 0) X(kF32, 32, 16, 4, 0) X(kF32, 32, 32, 4, 0)                \
    X(kF16, 32, 1, 4, 0) X(kF16, 32, 4, 4, 0) X(kF16, 32, 16, 4, 0)                                      \
    X(kF16, 32, 1, 2, 0) X(kF16, 32, 4, 2, 0) X(kF16, 32, 16, 2, 0) X(kF16, 32, 32, 2, 0)                \
    X(kBF16, 32, 1, 4, 0) X(kBF16, 32, 4, 4, 0) X(kBF16, 32, 16, 4, 0)                                   \
    X(kBF16, 32, 1, 2, 0) X(kBF16, 32, 4, 2, 0) X(kBF16, 32, 16, 2, 0) X(kBF16, 32, 32, 2, 0)

template <class F>
static cudaError_t dispatch_shape(const ShapeId &s, F &&f) {
#define MF_CASE(S_, L_, V_, VB_, FULL_)                                                                  \
    if (s.storage == S_ && s.L == L_ && s.V == V_ && s.VB == VB_ && s.full == FULL_)                     \
        return f(Shape<S_, L_, V_, VB_, (bool)FULL_>{});
    MF_FAST_SHAPES(MF_CASE)
    MF_GENERIC_SHAPES(MF_CASE)
#undef MF_CASE
    return cudaErrorInvalidValue;
}

ShapeId select_shape(int k, int storage, int variant) {
    if (storage == kF32) {
        if (k == 128) {
            if (variant == 1) return {storage, 16, 2, 16, 1};
            if (variant == 2) return {storage, 8, 4, 16, 1};
            return {storage, 32, 1, 16, 1};
        }
        // k = 32 / 64: at the A-10 worker count a group of 16 lanes (8-byte vectors at k = 32) keeps
        // twice the warps of an 8-lane group per rating in flight, which hides the update's arithmetic
        // latency (Netflix shape, one rating in flight per group: k = 32 11.6 -> 14.9, k = 64 9.1 ->
        // 10.5 G updates/s; profiles/r01c_smallk_probe.log)
        if (k == 32) {
            if (variant == 1) return {storage, 8, 1, 16, 1};
            if (variant == 2) return {storage, 32, 1, 4, 1};
            return {storage, 16, 1, 8, 1};
        }
        if (k == 64) {
            if (variant == 1) return {storage, 32, 1, 8, 1};
            return {storage, 16, 1, 16, 1};
        }
        if (k == 256) return {storage, 32, 2, 16, 1};
    } else {
        if (k == 128) {
            if (variant == 1) return {storage, 8, 2, 16, 1};
            if (variant == 2) return {storage, 32, 1, 8, 1};
            if (variant == 3) return {storage, 4, 4, 16, 1};
            return {storage, 16, 1, 16, 1};
        }
        // 16-bit rows, k = 32 / 64: 16 lanes per rating with 4- / 8-byte vectors (k = 32 11.9 -> 13.9,
        // k = 64 13.3 -> 13.9 G updates/s over the 4- / 8-lane 16-byte shapes)
        if (k == 32) {
            if (variant == 1) return {storage, 8, 1, 8, 1};
            if (variant == 2) return {storage, 4, 1, 16, 1};
            return {storage, 16, 1, 4, 1};
        }
        if (k == 64) {
            if (variant == 1) return {storage, 8, 1, 16, 1};
            if (variant == 2) return {storage, 32, 1, 4, 1};
            return {storage, 16, 1, 8, 1};
        }
        if (k == 256) return {storage, 32, 1, 16, 1};
    }
    return select_generic_shape(k, storage);
}

// batch-Hogwild!'s default shape (MF_OPT_VARIANT bits 0..3 = 0).  16-bit rows at k = 128: one rating per
// warp, 32 lanes x 8-byte vectors (a row is one 256-B warp access) -- after the warp-uniform index change
// (47 -> 32 registers) it keeps 64 warps per SM resident: Netflix shape 11.2 vs 10.5 G updates/s for the
// 16-lane 16-byte shape, Yahoo shape 7.0 vs 7.1 (profiles/r02p_f16_*).  Everything else as select_shape.
ShapeId hogwild_shape(int k, int storage, int variant) {
    if (variant == 0 && k == 128 && storage != kF32) return {storage, 32, 1, 8, 1};
    return select_shape(k, storage, variant);
}

// generic: L = 32, VB = 4 bytes (or 2 for odd k with 16-bit storage), V vectors per lane
ShapeId select_generic_shape(int k, int storage) {
    const int bytes = storage == kF32 ? 4 : 2;
    const int vb = (bytes == 2 && (k % 2)) ? 2 : 4;
    const int epv = vb / bytes;
    const int per_lane = (k + 32 * epv - 1) / (32 * epv);
    int V = per_lane <= 1 ? 1 : per_lane <= 4 ? 4 : per_lane <= 16 ? 16 : 32;
    if (vb == 4 && bytes == 2 && V == 32) V = 16;  // 16-bit, even k: 32*16*2 = 1024 covers k <= 1024
    return {storage, 32, V, vb, 0};
}

// ------------------------------------------------------------- batch-Hogwild!
// Grid: persistent CTAs of 8 warps.  A warp claims chunk c (f samples) with one
// atomicAdd, loads the chunk's COO triples 32 at a time (lane i holds sample
// base+i; three coalesced 128-byte loads, read-only path as in PAPER.md:183)
// and hands them to its G groups by __shfl_sync.  Each group then keeps D
// ratings in flight: D row-pair loads are issued before the first dot.
template <class SH, int D>
__global__ void __launch_bounds__(kBlock) k_hogwild(UpdateArgs a) {
    constexpr int L = SH::L, G = SH::G;
    static_assert(L % D == 0, "D must divide the per-group samples of a 32-sample tile");
    const int lane = threadIdx.x & 31;
    const int grp = lane / L, sub = lane % L;
    const int k = SH::FULL ? SH::KMAX : a.k;
    const int64_t N = a.n;
    const int f = a.batch_f;
    const int64_t warp_id = warp_uniform((blockIdx.x * kBlock + threadIdx.x) >> 5);
    // exact worker count: groups beyond a.active_groups idle; a warp with no active group exits
    const int64_t gleft = (int64_t)a.active_groups - warp_id * G;
    if (gleft <= 0) return;  // warp-uniform
    if (a.abort_if && *a.abort_if) return;  // streamed chunk failed validation
    const int gper = gleft < G ? (int)gleft : G;  // active groups in this warp
    const int ntile = (32 + gper - 1) / gper;     // samples per group per 32-sample tile
    unsigned long long done = 0;
    int bad = 0;
    const int ahead = a.prefetch * D;
    const uint32_t row_bytes = (uint32_t)k * SH::BYTES;
    const bool pf_on = ahead > 0 && SH::FULL && (row_bytes % 16u) == 0u && (32 % gper) == 0;
    const bool pf_ponly = a.prefetch_kind & 1;  // P rows only (Q rows left to the cache)
    const bool pf_lane = (a.prefetch_kind & 2) && row_bytes == 16u * SH::L * SH::V;  // per-lane prefetch.global.L2

    // Chunk claims run one chunk ahead and triple tiles one tile ahead, so neither the claim
    // atomic nor the 3 x 128-byte triple loads sit on the per-rating critical path.
    // The claim counter counts samples.  A warp claims f samples at a time until the last ~one chunk
    // per warp remains, then single 32-sample tiles, so the launch drains in about one tile's time
    // (the partitioned path runs many launches per epoch).
    // The first two chunks of every warp are static (warp w: chunks w and W + w), so the launch does
    // not open with W x 2 same-address atomics; the shared counter hands out the rest, starting
    // after those 2W chunks.
    const int64_t nwarps = (a.active_groups + G - 1) / G;
    const int64_t tail_zone = nwarps * (int64_t)f;
    const int64_t dyn0 = 2 * nwarps * (int64_t)f;
    unsigned long long *const ctr = a.chunk_ctr ? a.chunk_ctr : &a.scratch->chunk;
    auto claim = [&](int64_t *len) -> int64_t {
        unsigned long long c = 0;
        int want = f;
        if (lane == 0) {
            const unsigned long long seen = *(volatile unsigned long long *)ctr;
            if (dyn0 + (int64_t)seen + tail_zone >= N) want = 32;
            c = atomicAdd(ctr, (unsigned long long)want);
        }
        *len = __shfl_sync(0xffffffffu, want, 0);
        return dyn0 + (int64_t)__shfl_sync(0xffffffffu, c, 0);
    };
    int64_t len0 = f, next_len = f;
    int64_t base = warp_id * (int64_t)f;
    int64_t next_chunk = (nwarps + warp_id) * (int64_t)f;
    if (base >= N) return;
    int64_t end = min(base + len0, N);
    // L2 eviction priorities: the triples are read once per epoch and would otherwise push P rows out
    // of L2 (1.2 GB of R per epoch streams past a 123-MB P on the Netflix shape), so they are marked
    // evict_first; optionally the factor rows evict_last (MF_OPT_VARIANT bits 28..29)
    const int cp = a.cache_policy;
    const uint64_t pol_r = cp == 1 ? policy_evict_normal() : policy_evict_first();
    const uint64_t pol_p = cp == 2   ? policy_evict_last()
                           : cp >= 4 ? policy_evict_last_frac((cp & 1) ? 0.75f : 0.5f)
                                     : policy_evict_normal();
    const uint64_t pol_q = cp == 2 || cp == 3 || cp >= 6 ? policy_evict_last() : policy_evict_normal();
    int32_t tu, tv;
    float tr;
    {
        const int64_t i = base + lane;
        const bool ok = i < end;
        tu = ok ? ld_stream_s32(a.u + i, pol_r) : 0;
        tv = ok ? ld_stream_s32(a.v + i, pol_r) : 0;
        tr = ok ? ld_stream_f32(a.r + i, pol_r) : 0.f;
    }
    for (;;) {
        int64_t nbase = base + 32, nend = end;
        if (nbase >= end) {  // next tile starts the chunk claimed one chunk ago; claim the one after
            nbase = next_chunk;
            nend = min(nbase + next_len, N);
            if (nbase < N) next_chunk = claim(&next_len);
        }
        const bool more = nbase < N;
        int32_t nu = 0, nv = 0;
        float nr = 0.f;
        {
            const int64_t i = nbase + lane;
            const bool ok = more && i < nend;
            nu = ok ? ld_stream_s32(a.u + i, pol_r) : 0;
            nv = ok ? ld_stream_s32(a.v + i, pol_r) : 0;
            nr = ok ? ld_stream_f32(a.r + i, pol_r) : 0.f;
        }
        {
            const int cnt = (int)(end - base < 32 ? end - base : 32);
            if (a.count_updates) done += (lane == 0) ? cnt : 0;
            const int steps = (cnt + gper - 1) / gper < ntile ? (cnt + gper - 1) / gper : ntile;
#pragma unroll 1
            for (int j0 = 0; j0 < steps; j0 += D) {
                int32_t su[D], sv[D];
                float sr[D];
                bool val[D];
                RowRaw<SH> pr[D], qr[D];
                float pf[D][SH::E], qf[D][SH::E], dot[D];
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const int s = (j0 + d) * gper + grp;
                    su[d] = __shfl_sync(0xffffffffu, tu, s);
                    sv[d] = __shfl_sync(0xffffffffu, tv, s);
                    sr[d] = __shfl_sync(0xffffffffu, tr, s);
                    val[d] = grp < gper && s < cnt;
                }
                if (pf_on) {
                    // L2 prefetch of the rows of the ratings `ahead` steps later (this tile or the next
                    // one).  It moves no values into registers, so it adds memory-level parallelism
                    // without adding Hogwild! workers: the rows are still read at their own step.
#pragma unroll
                    for (int d = 0; d < D; d++) {
                        const int jt = j0 + ahead + d;
                        const bool cur = jt < steps;  // warp-uniform
                        const int s = (cur ? jt : jt - steps) * gper + grp;
                        const int sl = s & 31;
                        const int32_t pu = __shfl_sync(0xffffffffu, cur ? tu : nu, sl);
                        const int32_t pv = __shfl_sync(0xffffffffu, cur ? tv : nv, sl);
                        const bool ok = grp < gper && s < 32 && (cur ? s < cnt : (more && nbase + s < nend));
                        if (pf_lane) {  // every lane touches its own 16-B slice: the LSU merges them per line
                            if (ok) {
                                const char *pp = reinterpret_cast<const char *>(a.P) + (int64_t)pu * row_bytes;
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(pp + sub * 16));
                                if (!pf_ponly) {
                                    const char *qp = reinterpret_cast<const char *>(a.Q) + (int64_t)pv * row_bytes;
                                    asm volatile("prefetch.global.L2 [%0];" ::"l"(qp + sub * 16));
                                }
                            }
                        } else if (ok && sub == 0) {
                            prefetch_row_l2(a.P, pu, row_bytes);
                            if (!pf_ponly) prefetch_row_l2(a.Q, pv, row_bytes);
                        }
                    }
                }
#pragma unroll
                for (int d = 0; d < D; d++) {
                    load_row_pol<SH>(a.P, su[d], k, sub, val[d], pr[d], pol_p);
                    load_row_pol<SH>(a.Q, sv[d], k, sub, val[d], qr[d], pol_q);
                }
#pragma unroll
                for (int d = 0; d < D; d++) {
                    widen_row<SH>(pr[d], pf[d]);
                    widen_row<SH>(qr[d], qf[d]);
                    dot[d] = lane_dot<SH>(pf[d], qf[d]);
                }
                group_allreduce<SH, D>(dot);
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const float err = sr[d] - dot[d];
                    if (val[d] && !isfinite(err)) bad = 1;
                    sgd_step<SH>(pf[d], qf[d], err, a.eta, a.lam);
                    narrow_row<SH>(pf[d], pr[d]);
                    store_row_pol<SH>(a.P, su[d], k, sub, val[d], pr[d], pol_p);
                    if (a.q_red) {  // q_v += (q' - q): concurrent updates of one Q row all land (A-20)
                        red_row_delta<SH>(a.Q, sv[d], k, sub, val[d], qr[d], qf[d], pol_q);
                    } else {
                        narrow_row<SH>(qf[d], qr[d]);
                        store_row_pol<SH>(a.Q, sv[d], k, sub, val[d], qr[d], pol_q);
                    }
                }
            }
        }
        if (!more) break;
        base = nbase;
        end = nend;
        tu = nu;
        tv = nv;
        tr = nr;
    }
    if (bad) a.scratch->diverged = 1;
    if (a.count_updates && lane == 0 && done) atomicAdd(&a.scratch->updates, done);
}

// ------------------------------------------------- batch-Hogwild!, TMA-staged R
// The same schedule and update as k_hogwild, with the rating batches staged in shared memory by the
// TMA engine (north star: "128-bit vectorised, coalesced loads of the COO triples, with TMA or
// shared-memory staging of rating batches"): when a warp claims chunk c + 1, one lane issues three bulk
// copies (cp.async.bulk, u / v / r of the chunk, 16-B granules) into the warp's second buffer, completing
// on an mbarrier, while the warp updates chunk c from the first; a group reads its sample's triple from
// shared memory.  Chunks are <= kStageF samples; a chunk's last len % 4 triples (not a 16-B granule)
// are copied by the lanes.  Needs 16-B aligned u / v / r (the main epoch arrays; sub-ranges of the
// partitioned layout use k_hogwild).
static constexpr int kStageF = 256;
static constexpr int kStageSmem = kWarpsPerBlock * 2 * 3 * kStageF * 4;  // dynamic shared memory per CTA (48 KB)

__device__ __forceinline__ void mbar_init1(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// every lane of the warp waits; the loop exit is a warp vote, so it is uniform to the compiler
__device__ __forceinline__ void mbar_wait1(uint32_t bar, uint32_t parity) {
    for (;;) {
        uint32_t ok;
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok)
                     : "r"(bar), "r"(parity)
                     : "memory");
        if (__all_sync(0xffffffffu, ok)) break;
    }
}

template <class SH, int D>
__global__ void __launch_bounds__(kBlock) k_hogwild_tma(UpdateArgs a) {
    constexpr int L = SH::L, G = SH::G;
    static_assert(L % D == 0, "D must divide the per-group samples of a 32-sample tile");
    extern __shared__ __align__(128) int32_t s_dyn[];
    auto s_tri = reinterpret_cast<int32_t(*)[2][3][kStageF]>(s_dyn);  // [warp][buffer][u, v, r][sample]
    __shared__ __align__(8) uint64_t s_bar[kWarpsPerBlock][2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int grp = lane / L, sub = lane % L;
    const int k = SH::FULL ? SH::KMAX : a.k;
    const int64_t N = a.n;
    const int f = a.batch_f;  // <= kStageF (launcher)
    const int64_t warp_id = warp_uniform((blockIdx.x * kBlock + threadIdx.x) >> 5);
    const int64_t gleft = (int64_t)a.active_groups - warp_id * G;
    if (gleft <= 0) return;  // warp-uniform
    const int gper = gleft < G ? (int)gleft : G;
    const int ntile = (32 + gper - 1) / gper;
    unsigned long long done = 0;
    int bad = 0;
    const int ahead = a.prefetch * D;
    const uint32_t row_bytes = (uint32_t)k * SH::BYTES;
    const bool pf_on = ahead > 0 && SH::FULL && (row_bytes % 16u) == 0u && (32 % gper) == 0;
    const bool pf_ponly = a.prefetch_kind & 1;
    const int64_t nwarps = (a.active_groups + G - 1) / G;
    const int64_t tail_zone = nwarps * (int64_t)f;
    const int64_t dyn0 = 2 * nwarps * (int64_t)f;
    unsigned long long *const ctr = a.chunk_ctr ? a.chunk_ctr : &a.scratch->chunk;
    auto claim = [&](int64_t *len) -> int64_t {
        unsigned long long c = 0;
        int want = f;
        if (lane == 0) {
            const unsigned long long seen = *(volatile unsigned long long *)ctr;
            if (dyn0 + (int64_t)seen + tail_zone >= N) want = 32;
            c = atomicAdd(ctr, (unsigned long long)want);
        }
        *len = __shfl_sync(0xffffffffu, want, 0);
        return dyn0 + (int64_t)__shfl_sync(0xffffffffu, c, 0);
    };
    const int cp = a.cache_policy;
    const uint64_t pol_p = cp == 2   ? policy_evict_last()
                           : cp >= 4 ? policy_evict_last_frac((cp & 1) ? 0.75f : 0.5f)
                                     : policy_evict_normal();
    const uint64_t pol_q = cp == 2 || cp == 3 || cp >= 6 ? policy_evict_last() : policy_evict_normal();
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&s_bar[wib][0]);
    if (lane == 0) {
        mbar_init1(bar0);
        mbar_init1(bar0 + 8);
    }
    __syncwarp();
    // stage chunk [cb, cb + clen) into buffer b: 16-B granules by the TMA engine, the rest by lanes
    auto stage = [&](int b, int64_t cb, int clen) {
        const int c4 = clen & ~3;
        if (lane == 0) {
            const uint32_t bar = bar0 + 8u * (uint32_t)b;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our earlier reads of the buffer
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(12 * c4) : "memory");
            if (c4) {
                const int32_t *src[3] = {a.u + cb, a.v + cb, reinterpret_cast<const int32_t *>(a.r) + cb};
#pragma unroll
                for (int x = 0; x < 3; x++) {
                    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_tri[wib][b][x][0]);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            dst),
                        "l"(src[x]), "r"(4 * c4), "r"(bar)
                        : "memory");
                }
            }
        }
        if (lane < clen - c4) {
            s_tri[wib][b][0][c4 + lane] = __ldg(a.u + cb + c4 + lane);
            s_tri[wib][b][1][c4 + lane] = __ldg(a.v + cb + c4 + lane);
            s_tri[wib][b][2][c4 + lane] = __float_as_int(__ldg(a.r + cb + c4 + lane));
        }
    };
    uint32_t phase = 0;  // bit b: parity of buffer b's next completion
    int64_t base = warp_id * (int64_t)f;
    if (base >= N) return;
    int len = (int)min((int64_t)f, N - base);
    int64_t nbase = (nwarps + warp_id) * (int64_t)f;
    int64_t nlen64 = f;
    int b = 0;
    stage(0, base, len);
    int nlen = nbase < N ? (int)min(nlen64, N - nbase) : 0;
    if (nlen) stage(1, nbase, nlen);
    for (;;) {
        mbar_wait1(bar0 + 8u * (uint32_t)b, (phase >> b) & 1u);
        phase ^= 1u << b;
        __syncwarp();  // the lanes' tail stores of this buffer are visible to the whole warp
        const int32_t *tu_ = s_tri[wib][b][0], *tv_ = s_tri[wib][b][1];
        const float *tr_ = reinterpret_cast<const float *>(s_tri[wib][b][2]);
        if (a.count_updates && lane == 0) done += len;
        for (int t0 = 0; t0 < len; t0 += 32) {
            const int cnt = len - t0 < 32 ? len - t0 : 32;
            const int steps = (cnt + gper - 1) / gper < ntile ? (cnt + gper - 1) / gper : ntile;
#pragma unroll 1
            for (int j0 = 0; j0 < steps; j0 += D) {
                int32_t su[D], sv[D];
                float sr[D];
                bool val[D];
                RowRaw<SH> pr[D], qr[D];
                float pf[D][SH::E], qf[D][SH::E], dot[D];
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const int s_ = (j0 + d) * gper + grp;
                    val[d] = grp < gper && s_ < cnt;
                    su[d] = val[d] ? tu_[t0 + s_] : 0;
                    sv[d] = val[d] ? tv_[t0 + s_] : 0;
                    sr[d] = val[d] ? tr_[t0 + s_] : 0.f;
                }
                if (pf_on) {  // L2 prefetch of the rows `ahead` steps later inside this chunk
#pragma unroll
                    for (int d = 0; d < D; d++) {
                        const int jt = j0 + ahead + d;
                        const int idx = jt < steps ? t0 + jt * gper + grp : t0 + 32 + (jt - steps) * gper + grp;
                        if (grp < gper && idx < len && sub == 0) {
                            prefetch_row_l2(a.P, tu_[idx], row_bytes);
                            if (!pf_ponly) prefetch_row_l2(a.Q, tv_[idx], row_bytes);
                        }
                    }
                }
#pragma unroll
                for (int d = 0; d < D; d++) {
                    load_row_pol<SH>(a.P, su[d], k, sub, val[d], pr[d], pol_p);
                    load_row_pol<SH>(a.Q, sv[d], k, sub, val[d], qr[d], pol_q);
                }
#pragma unroll
                for (int d = 0; d < D; d++) {
                    widen_row<SH>(pr[d], pf[d]);
                    widen_row<SH>(qr[d], qf[d]);
                    dot[d] = lane_dot<SH>(pf[d], qf[d]);
                }
                group_allreduce<SH, D>(dot);
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const float err = sr[d] - dot[d];
                    if (val[d] && !isfinite(err)) bad = 1;
                    sgd_step<SH>(pf[d], qf[d], err, a.eta, a.lam);
                    narrow_row<SH>(pf[d], pr[d]);
                    store_row_pol<SH>(a.P, su[d], k, sub, val[d], pr[d], pol_p);
                    if (a.q_red) {  // q_v += (q' - q): concurrent updates of one Q row all land (A-20)
                        red_row_delta<SH>(a.Q, sv[d], k, sub, val[d], qr[d], qf[d], pol_q);
                    } else {
                        narrow_row<SH>(qf[d], qr[d]);
                        store_row_pol<SH>(a.Q, sv[d], k, sub, val[d], qr[d], pol_q);
                    }
                }
            }
        }
        if (!nlen) break;
        __syncwarp();  // every lane is done reading buffer b before it is refilled
        // chunk after next: claimed now, staged into the buffer just used
        int64_t cl_len = 0;
        const int64_t cbase = claim(&cl_len);
        const int clen = cbase < N ? (int)min(cl_len, N - cbase) : 0;
        if (clen) stage(b, cbase, clen);
        b ^= 1;
        len = nlen;
        nlen = clen;
    }
    if (bad) a.scratch->diverged = 1;
    if (a.count_updates && lane == 0 && done) atomicAdd(&a.scratch->updates, done);
}

template <class SH, int D, bool TMA = false>
static cudaError_t hogwild_launch(const UpdateArgs &a, int workers, cudaStream_t st, int *used) {
    // occupancy and SM count are queried once per instantiation: the partitioned path launches this
    // kernel hundreds of times per epoch and the host must stay ahead of ~80 us launches
    static const int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    static const int per_sm = [] {
        int v = 0;
        if constexpr (TMA) {
            cudaFuncSetAttribute(k_hogwild_tma<SH, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageSmem);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_hogwild_tma<SH, D>, kBlock, kStageSmem);
        } else {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_hogwild<SH, D>, kBlock, 0);
        }
        return v < 1 ? 1 : v;
    }();
    // workers = concurrent ratings = active groups x D
    int64_t groups = (int64_t)sms * per_sm * kWarpsPerBlock * SH::G;
    if (workers > 0) groups = std::min<int64_t>(groups, (workers + D - 1) / D);
    // Small launches (the partitioned path's sub-blocks): shrink the chunk so every warp gets at
    // least ~4 chunks -- with fewer chunks than warps one warp would walk 256 samples serially while
    // the rest idle.  Any f > 128/12 keeps the R-stream locality the paper chose f for.
    int batch_f = a.batch_f;
    {
        const int64_t want_warps = (groups + SH::G - 1) / SH::G;
        if ((a.n + batch_f - 1) / batch_f < 4 * want_warps) {
            const int64_t f = a.n / (4 * want_warps);
            batch_f = (int)std::max<int64_t>(32, std::min<int64_t>(batch_f, (f / 32) * 32));
        }
    }
    const int64_t chunks = (a.n + batch_f - 1) / batch_f;
    groups = std::max<int64_t>(1, std::min<int64_t>(groups, chunks * SH::G));
    // Balance the SMs: when the grid spans more than one CTA per SM, round the CTA count down to a
    // multiple of the SM count so every SM runs the same number of warps (an SM holding one CTA
    // more than the others saturates its store path first; ncu r01: l1tex2xbar max 84% vs avg 70%).
    const int64_t per_block_groups = (int64_t)kWarpsPerBlock * SH::G;
    if (groups >= (int64_t)sms * per_block_groups) {
        const int64_t full = groups / per_block_groups;
        groups = (full / sms) * sms * per_block_groups;
    }
    const int64_t warps = (groups + SH::G - 1) / SH::G;
    const int blocks = (int)((warps + kWarpsPerBlock - 1) / kWarpsPerBlock);
    if (used) *used = (int)(groups * D);
    UpdateArgs args = a;
    args.q_red = a.q_mode == 1 || (a.q_mode == 2 && (double)(groups * D) * a.q_share < kQRedKappa);
    args.active_groups = groups;
    args.batch_f = batch_f;
    // every launch claims chunks from 0 (the partitioned path launches once per block)
    cudaError_t e = cudaMemsetAsync(a.chunk_ctr ? a.chunk_ctr : &a.scratch->chunk, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if constexpr (TMA) k_hogwild_tma<SH, D><<<blocks, kBlock, kStageSmem, st>>>(args);
    else k_hogwild<SH, D><<<blocks, kBlock, 0, st>>>(args);
    return cudaGetLastError();
}

cudaError_t launch_hogwild(const ShapeId &sh, const UpdateArgs &a_in, int workers, int variant, cudaStream_t st,
                           int *workers_used) {
    const int D = (variant >> 4) & 0xF;  // bits 4..7 select samples in flight per group (0 = default)
    UpdateArgs a = a_in;
    {
        const int pf = (variant >> 16) & 0xF;  // bits 16..19: L2 row-prefetch distance in steps (0, 15 = off)
        a.prefetch = pf == 15 ? 0 : pf;
        a.prefetch_kind = (variant >> 20) & 0x3;  // bits 20..21: 1 = P rows only, 2 = per-lane prefetch
        a.cache_policy = (variant >> 28) & 0x7;   // bits 28..30: L2 eviction priorities (UpdateArgs)
    }
    // TMA staging of the triples needs 16-B aligned arrays and chunks that fit the warp's buffers
    const bool tma = a.r_stage == 2 && a.batch_f <= kStageF && !a.abort_if &&
                     ((reinterpret_cast<uintptr_t>(a.u) | reinterpret_cast<uintptr_t>(a.v) |
                       reinterpret_cast<uintptr_t>(a.r)) & 15) == 0;
    return dispatch_shape(sh, [&](auto tag) -> cudaError_t {
        using SH = decltype(tag);
        constexpr int L = SH::L;
        if constexpr (SH::FULL) {
            if (tma && D != 4) {
                if (workers > 0 && workers < 64) return hogwild_launch<SH, 1, true>(a, workers, st, workers_used);
                const bool two = D == 2 || D == 3 || (D == 0 && SH::S == kF32 && SH::KMAX >= 256);
                if (two && L % 2 == 0) return hogwild_launch<SH, (L % 2 == 0 ? 2 : 1), true>(a, workers, st, workers_used);
                return hogwild_launch<SH, 1, true>(a, workers, st, workers_used);
            }
            if (workers > 0 && workers < 64) return hogwild_launch<SH, 1>(a, workers, st, workers_used);
            if (D == 4 && L % 4 == 0) return hogwild_launch<SH, (L % 4 == 0 ? 4 : 1)>(a, workers, st, workers_used);
            // D = 0 (auto): two ratings in flight per group for fp32 rows of k >= 256, one otherwise (round 1
            // had two for k = 128 fp32: 5.6 vs 5.2 G/s then; since the warp-uniform index change one is
            // faster -- Netflix shape 5.45 vs 5.27, Yahoo 3.34 vs 3.21, profiles/r02p_f32_*; k = 32 / 64
            // fp32 one in flight +28% / +15%, r01c_smallk_probe.log)
            const bool two = D == 2 || D == 3 || (D == 0 && SH::S == kF32 && SH::KMAX >= 256);
            if (two && L % 2 == 0) return hogwild_launch<SH, (L % 2 == 0 ? 2 : 1)>(a, workers, st, workers_used);
        }
        return hogwild_launch<SH, 1>(a, workers, st, workers_used);
    });
}

// ------------------------------------------------------- deterministic waves
// All CTAs are co-resident (cooperative launch); between waves a sense-free
// generation barrier with gpu-scope fences orders every P/Q store of wave w
// before any load of wave w+1 (loads are ld.global.cg, so L1 is never read).
__device__ __forceinline__ void grid_barrier(DevScratch *s, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = &s->bar_gen;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(&s->bar_count, 1u) == nblocks - 1) {
            s->bar_count = 0;
            __threadfence();
            atomicExch(&s->bar_gen, g + 1);
        } else {
            while (*gen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// Leaner barrier for one CTA per SM: arrival by a release atomic, wait by acquire loads (no separate
// membar on either side); the CTA barriers around it order the other threads' stores and loads.
__device__ __forceinline__ void grid_barrier_ra(DevScratch *s, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&s->bar_gen) : "memory");
        unsigned prev;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&s->bar_count) : "memory");
        if (prev == nblocks - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(&s->bar_count) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&s->bar_gen), "r"(g + 1) : "memory");
        } else {
            unsigned cur;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&s->bar_gen) : "memory");
            } while (cur == g);
        }
    }
    __syncthreads();
}

// Monotonic-counter barrier (one CTA per SM): every CTA adds 1 with a release reduction (no return
// value to wait for) and polls the counter with acquire loads until it reaches target = (wave + 1) x
// CTAs; the counter is zeroed with the epoch's scratch.  One memory round trip fewer than the
// generation-flag form (the last arriver's atomic, its flag store, the waiters' poll).
__device__ __forceinline__ void grid_barrier_count(DevScratch *s, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&s->bar_count) : "memory");
        unsigned cur;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&s->bar_count) : "memory");
        } while ((int)(cur - target) < 0);
    }
    __syncthreads();
}

// D samples of the same wave per group and step (a wave's samples are pairwise independent, so any
// number may be in flight -- unlike batch-Hogwild! there is no staleness to bound); the per-rating
// arithmetic (lane_dot, then the butterfly) is the same for every D, so results do not depend on it.
template <class SH, int BLOCK = kBlock, int D = 1>
__global__ void __launch_bounds__(BLOCK) k_waves(UpdateArgs a) {
    constexpr int L = SH::L;
    const int lane = threadIdx.x & 31, sub = lane % L;
    const int k = SH::FULL ? SH::KMAX : a.k;
    const int64_t groups = (int64_t)gridDim.x * BLOCK / L;
    const int64_t gid = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) / L;
    const int64_t wbase = warp_uniform(gid - lane / L);  // the warp's first group
    int bad = 0;
    unsigned long long done = 0;
    // The triples of a group's first step in the next wave are read-only and independent of the wave's
    // updates: they are loaded before the barrier, so after it only the row loads stand between the
    // barrier and the first update (one memory latency per wave instead of two).
    int32_t nu[D], nv[D];
    float nr[D];
    auto fetch_first = [&](int64_t wv) {
        const int64_t lo = a.wave_off[wv], hi = a.wave_off[wv + 1];
#pragma unroll
        for (int d = 0; d < D; d++) {
            const int64_t s = lo + wbase + d * groups + lane / L;
            const bool ok = s < hi;
            nu[d] = ok ? __ldg(a.u + s) : 0;
            nv[d] = ok ? __ldg(a.v + s) : 0;
            nr[d] = ok ? __ldg(a.r + s) : 0.f;
        }
    };
    if (a.nwaves > 0) fetch_first(0);
    for (int64_t w = 0; w < a.nwaves; w++) {
        const int64_t lo = a.wave_off[w], hi = a.wave_off[w + 1];
        // warp-uniform trip count so the full-warp shuffles stay converged
        const int64_t warp_first = lo + wbase;
        for (int64_t s0 = warp_first; s0 < hi; s0 += D * groups) {
            int32_t su[D], sv[D];
            float sr[D], dot[D];
            bool val[D];
            RowRaw<SH> pr[D], qr[D];
#pragma unroll
            for (int d = 0; d < D; d++) {
                const int64_t s = s0 + d * groups + lane / L;
                val[d] = s < hi;
                if (s0 == warp_first) {
                    su[d] = nu[d], sv[d] = nv[d], sr[d] = nr[d];
                } else {
                    su[d] = val[d] ? __ldg(a.u + s) : 0;
                    sv[d] = val[d] ? __ldg(a.v + s) : 0;
                    sr[d] = val[d] ? __ldg(a.r + s) : 0.f;
                }
                load_row<SH>(a.P, su[d], k, sub, val[d], pr[d]);
                load_row<SH>(a.Q, sv[d], k, sub, val[d], qr[d]);
            }
#pragma unroll
            for (int d = 0; d < D; d++) {
                float p[SH::E], q[SH::E];
                widen_row<SH>(pr[d], p);
                widen_row<SH>(qr[d], q);
                dot[d] = lane_dot<SH>(p, q);
            }
            group_allreduce<SH, D>(dot);
#pragma unroll
            for (int d = 0; d < D; d++) {
                const float err = sr[d] - dot[d];
                if (val[d] && !isfinite(err)) bad = 1;
                float p[SH::E], q[SH::E];
                widen_row<SH>(pr[d], p);
                widen_row<SH>(qr[d], q);
                sgd_step<SH>(p, q, err, a.eta, a.lam);
                narrow_row<SH>(p, pr[d]);
                narrow_row<SH>(q, qr[d]);
                store_row<SH>(a.P, su[d], k, sub, val[d], pr[d]);
                store_row<SH>(a.Q, sv[d], k, sub, val[d], qr[d]);
                if (val[d] && sub == 0) done++;
            }
        }
        if (w + 1 < a.nwaves) fetch_first(w + 1);
        if (BLOCK == kBlock) grid_barrier(a.scratch, gridDim.x);
        else if (a.barrier == 0) grid_barrier_count(a.scratch, (unsigned)(w + 1) * gridDim.x);
        else grid_barrier_ra(a.scratch, gridDim.x);
    }
    if (bad) a.scratch->diverged = 1;
    if (a.count_updates && done) atomicAdd(&a.scratch->updates, done);
}

cudaError_t launch_waves(const ShapeId &sh, const UpdateArgs &a, cudaStream_t st, int *launches, int big) {
    return dispatch_shape(sh, [&](auto tag) -> cudaError_t {
        using SH = decltype(tag);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if constexpr (SH::FULL && (32 / SH::L) * 4 <= 32 && SH::L % 4 == 0) {
            if (big == 3) {  // two 512-thread CTAs per SM (128 registers each), four samples per group and step
                const void *kern = (const void *)k_waves<SH, 512, 4>;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 512, 0);
                if (per_sm >= 2) {
                    UpdateArgs args = a;
                    void *kargs[] = {&args};
                    if (launches) *launches = 1;
                    return cudaLaunchCooperativeKernel(kern, dim3(2 * sms), dim3(512), kargs, 0, st);
                }
            }
        }
        // one 1024-thread CTA per SM: a quarter of the barrier arrivals; big = 2: two per group.  The
        // masked generic shapes (k outside 32 / 64 / 128 / 256) keep more than 64 registers per thread,
        // so they run the 256-thread form (identical results) instead of spilling under the 1024-thread cap.
        if constexpr (SH::FULL) {
            if (big) {
                const void *kern = big == 2 ? (const void *)k_waves<SH, 1024, 2> : (const void *)k_waves<SH, 1024, 1>;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1024, 0);
                if (per_sm >= 1) {
                    UpdateArgs args = a;
                    void *kargs[] = {&args};
                    if (launches) *launches = 1;
                    return cudaLaunchCooperativeKernel(kern, dim3(sms), dim3(1024), kargs, 0, st);
                }
            }
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_waves<SH>, kBlock, 0);
        if (per_sm < 1) return cudaErrorLaunchOutOfResources;
        // the largest wave decides how many groups are useful
        int blocks = sms * std::min(per_sm, 4);
        UpdateArgs args = a;
        void *kargs[] = {&args};
        if (launches) *launches = 1;
        return cudaLaunchCooperativeKernel((const void *)k_waves<SH>, dim3(blocks), dim3(kBlock), kargs, 0, st);
    });
}

// ------------------------------------------------------- column degree moment --
__global__ void k_col_hist(const int32_t *v, int64_t n, unsigned *deg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(deg + v[i], 1u);
}
__global__ void k_sq_sum(const unsigned *deg, int64_t n_cols, double *out) {
    double s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_cols; i += (int64_t)gridDim.x * blockDim.x)
        s += (double)deg[i] * (double)deg[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s != 0) atomicAdd(out, s);  // integer-valued terms: exact in any order
}
cudaError_t launch_col_sq(const int32_t *v, int64_t n, int64_t n_cols, unsigned *tmp, double *out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(tmp, 0, sizeof(unsigned) * n_cols, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(out, 0, sizeof(double), st);
    if (e != cudaSuccess) return e;
    if (n > 0) k_col_hist<<<148 * 8, 256, 0, st>>>(v, n, tmp);
    k_sq_sum<<<148, 256, 0, st>>>(tmp, n_cols, out);
    return cudaGetLastError();
}

// -------------------------------------------------------------------- RMSE --
static constexpr int kRmseBlocks = 148 * 4;
int rmse_parts() { return kRmseBlocks; }

template <class SH>
__global__ void __launch_bounds__(kBlock) k_rmse(const int32_t *u, const int32_t *v, const float *r, int64_t n,
                                                 const void *P, const void *Q, int kk, double *partials) {
    constexpr int L = SH::L;
    const int lane = threadIdx.x & 31, sub = lane % L;
    const int k = SH::FULL ? SH::KMAX : kk;
    const int64_t groups = (int64_t)gridDim.x * kBlock / L;
    const int64_t gid = ((int64_t)blockIdx.x * kBlock + threadIdx.x) / L;
    double acc = 0.0;
    const int64_t warp_first = warp_uniform(gid - lane / L);
    for (int64_t s0 = warp_first; s0 < n; s0 += groups) {
        const int64_t s = s0 + lane / L;
        const bool val = s < n;
        const int32_t su = val ? __ldg(u + s) : 0;
        const int32_t sv = val ? __ldg(v + s) : 0;
        const float sr = val ? __ldg(r + s) : 0.f;
        RowRaw<SH> pr, qr;
        load_row<SH>(P, su, k, sub, val, pr);
        load_row<SH>(Q, sv, k, sub, val, qr);
        float p[SH::E], q[SH::E];
        widen_row<SH>(pr, p);
        widen_row<SH>(qr, q);
        const float dot = group_dot<SH>(p, q);
        if (val && sub == 0) {
            const double e = (double)sr - (double)dot;
            acc += e * e;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double ws[kWarpsPerBlock];
    if (lane == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kWarpsPerBlock; i++) s += ws[i];
        partials[blockIdx.x] = s;
    }
}

__global__ void k_sum_partials(const double *partials, int n, int64_t count, double *out, int do_sqrt) {
    __shared__ double sh[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = do_sqrt ? sqrt(sh[0] / (double)count) : sh[0];
}

cudaError_t launch_rmse(const ShapeId &sh, const int32_t *u, const int32_t *v, const float *r, int64_t n,
                        const void *P, const void *Q, int k, double *partials, int nparts, double *out,
                        cudaStream_t st, int do_sqrt) {
    cudaError_t e = dispatch_shape(sh, [&](auto tag) -> cudaError_t {
        using SH = decltype(tag);
        k_rmse<SH><<<nparts, kBlock, 0, st>>>(u, v, r, n, P, Q, k, partials);
        return cudaGetLastError();
    });
    if (e != cudaSuccess) return e;
    k_sum_partials<<<1, 256, 0, st>>>(partials, nparts, n, out, do_sqrt);
    return cudaGetLastError();
}

// -------------------------------------------------------------------- init --
// A-7: X[row][col] = (float)(h >> 40) * 2^-24 * (float)(1/sqrt(k)),
// h = splitmix64(seed ^ (tag << 60) ^ (row*k + col)), rounded to storage.
__device__ __forceinline__ void store_scalar(void *X, int storage, int64_t i, float x) {
    if (storage == kF32) reinterpret_cast<float *>(X)[i] = x;
    else if (storage == kF16) reinterpret_cast<__half *>(X)[i] = __float2half_rn(x);
    else reinterpret_cast<__nv_bfloat16 *>(X)[i] = __float2bfloat16_rn(x);
}
__device__ __forceinline__ float load_scalar(const void *X, int storage, int64_t i) {
    if (storage == kF32) return reinterpret_cast<const float *>(X)[i];
    if (storage == kF16) return __half2float(reinterpret_cast<const __half *>(X)[i]);
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16 *>(X)[i]);
}

__global__ void k_init(void *X, int64_t elem0, int64_t count, uint64_t seed, uint32_t tag, float scale, int storage) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h = splitmix64(seed ^ ((uint64_t)tag << 60) ^ (uint64_t)(elem0 + i));
        const float unit = __fmul_rn((float)(h >> 40), 0x1.0p-24f);
        store_scalar(X, storage, i, __fmul_rn(unit, scale));
    }
}

cudaError_t launch_init_offset(int storage, void *X, int64_t elem0, int64_t count, int k, uint64_t seed, uint32_t tag,
                               cudaStream_t st) {
    const float scale = (float)(1.0 / sqrt((double)k));
    const int blocks = (int)std::min<int64_t>((count + 255) / 256, 148 * 32);
    k_init<<<std::max(blocks, 1), 256, 0, st>>>(X, elem0, count, seed, tag, scale, storage);
    return cudaGetLastError();
}

__global__ void k_from_f32(void *X, const float *src, int64_t count, int storage) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        store_scalar(X, storage, i, src[i]);
}
__global__ void k_to_f32(const void *X, float *dst, int64_t count, int storage) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = load_scalar(X, storage, i);
}
cudaError_t launch_from_f32(int storage, void *X, const float *src, int64_t count, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 32));
    k_from_f32<<<blocks, 256, 0, st>>>(X, src, count, storage);
    return cudaGetLastError();
}
cudaError_t launch_to_f32(int storage, const void *X, float *dst, int64_t count, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 32));
    k_to_f32<<<blocks, 256, 0, st>>>(X, dst, count, storage);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- validate --
__global__ void k_validate(const int32_t *u, const int32_t *v, const float *r, int64_t n, int64_t row_lo,
                           int64_t row_hi, int64_t n_cols, DevScratch *s) {
    unsigned long long bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = u[i], b = v[i];
        const float x = r[i];
        bad += (a < row_lo || a >= row_hi || b < 0 || b >= n_cols || !isfinite(x)) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&s->bad, bad);
}
cudaError_t launch_validate_rows(const int32_t *u, const int32_t *v, const float *r, int64_t n, int64_t row_lo,
                                 int64_t row_hi, int64_t n_cols, DevScratch *scratch, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_validate<<<blocks, 256, 0, st>>>(u, v, r, n, row_lo, row_hi, n_cols, scratch);
    return cudaGetLastError();
}

__global__ void k_rebase(int32_t *u, int64_t n, int32_t off) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        u[i] -= off;
}
cudaError_t launch_rebase(int32_t *u, int64_t n, int32_t off, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_rebase<<<blocks, 256, 0, st>>>(u, n, off);
    return cudaGetLastError();
}

// ----------------------------------------------------------------- shuffle --
// A-8: order samples by key splitmix64(seed ^ i) (distinct for distinct i, as
// splitmix64 is a bijection), ties impossible; perm[j] = original index.
__global__ void k_shuffle_keys(uint64_t *keys, uint32_t *idx, int64_t n, uint64_t seed) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = splitmix64(seed ^ (uint64_t)i);
        idx[i] = (uint32_t)i;
    }
}
__global__ void k_gather(const int32_t *u_in, const int32_t *v_in, const float *r_in, const uint32_t *idx, int64_t n,
                         int32_t *u_out, int32_t *v_out, float *r_out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = idx[i];
        u_out[i] = u_in[j];
        v_out[i] = v_in[j];
        r_out[i] = r_in[j];
    }
}
cudaError_t launch_gather(const int32_t *u_in, const int32_t *v_in, const float *r_in, const uint32_t *idx, int64_t n,
                          int32_t *u_out, int32_t *v_out, float *r_out, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_gather<<<blocks, 256, 0, st>>>(u_in, v_in, r_in, idx, n, u_out, v_out, r_out);
    return cudaGetLastError();
}

// out[i] = a[b[i]]: composition of two permutations (per-epoch reshuffle keeps the caller order map)
__global__ void k_compose(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[b[i]];
}
cudaError_t launch_compose(const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_compose<<<blocks, 256, 0, st>>>(a, b, out, n);
    return cudaGetLastError();
}

// A-8 permutation only (data independent): keys, radix sort, perm_out[j] = original index
cudaError_t launch_shuffle_perm(int64_t n, uint64_t seed, uint32_t *perm_out, cudaStream_t st) {
    if (n > (int64_t)0xFFFFFFFFll) return cudaErrorInvalidValue;
    uint64_t *k0 = nullptr, *k1 = nullptr;
    uint32_t *i0 = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e;
#define MF_TRY(x) do { e = (x); if (e != cudaSuccess) goto done; } while (0)
    MF_TRY(cudaMallocAsync(&k0, sizeof(uint64_t) * n, st));
    MF_TRY(cudaMallocAsync(&k1, sizeof(uint64_t) * n, st));
    MF_TRY(cudaMallocAsync(&i0, sizeof(uint32_t) * n, st));
    {
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
        k_shuffle_keys<<<blocks, 256, 0, st>>>(k0, i0, n, seed);
        MF_TRY(cudaGetLastError());
    }
    MF_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, i0, perm_out, n, 0, 64, st));
    MF_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
    MF_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i0, perm_out, n, 0, 64, st));
done:
    if (tmp) cudaFreeAsync(tmp, st);
    if (k0) cudaFreeAsync(k0, st);
    if (k1) cudaFreeAsync(k1, st);
    if (i0) cudaFreeAsync(i0, st);
#undef MF_TRY
    return e;
}

// Fused load step: out[i] = in[idx[i]] (idx == nullptr: identity, may run in place), counting samples
// with u outside [row_lo, row_hi), v outside [0, n_cols) or non-finite r; u is rebased by row_lo.
__global__ void k_gather_validate(const int32_t *u_in, const int32_t *v_in, const float *r_in, const uint32_t *idx,
                                  int64_t n, int64_t row_lo, int64_t row_hi, int64_t n_cols, int32_t *u_out,
                                  int32_t *v_out, float *r_out, DevScratch *s) {
    unsigned long long bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = idx ? (int64_t)idx[i] : i;
        const int32_t a = u_in[j], b = v_in[j];
        const float x = r_in[j];
        bad += (a < row_lo || a >= row_hi || b < 0 || b >= n_cols || !isfinite(x)) ? 1 : 0;
        u_out[i] = a - (int32_t)row_lo;
        v_out[i] = b;
        r_out[i] = x;
    }
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&s->bad, bad);
}
cudaError_t launch_gather_validate(const int32_t *u_in, const int32_t *v_in, const float *r_in, const uint32_t *idx,
                                   int64_t n, int64_t row_lo, int64_t row_hi, int64_t n_cols, int32_t *u_out,
                                   int32_t *v_out, float *r_out, DevScratch *scratch, cudaStream_t st) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    k_gather_validate<<<blocks, 256, 0, st>>>(u_in, v_in, r_in, idx, n, row_lo, row_hi, n_cols, u_out, v_out, r_out,
                                              scratch);
    return cudaGetLastError();
}

}  // namespace mf
