// mf_flow.cu -- deterministic execution without grid barriers: per-row update counters (sm_100a).
//
// MF_SCHED_DETERMINISTIC computes serial SGD over the shuffled order (D-3).  The wave layout
// (mf_api.cu build_waves) sorts the samples by wave, wave(i) = max(last[u_i], last[v_i]) + 1, so no two
// samples of a wave share a row or a column.  k_waves runs the waves one after another with a grid
// barrier between them; this kernel runs the same wave-sorted stream with NO barrier.  Instead every
// P row and every Q row has a counter of the updates applied to it, and a sample waits (when it has
// to) until the counters of its rows reach its ordinals ju = #earlier samples (serial order) with the
// same u, jv likewise.  Each row then sees exactly its serial sequence of updates, each from the state
// the serial order gives it, so the result is serial SGD's (D-3): bit-reproducible run to run and equal
// to the oracle's to the dot product's rounding, like the waves.
//
// Worker = one warp, one rating at a time (a 32-lane shape: G = 1); warp w of W owns the stream
// positions w, w + W, w + 2W, ... (or, as an option, claims 32-sample tiles in order).  Per rating i
// (n1 = the warp's next rating, n2 the one after):
//   B  relaxed loads of n2's two counters
//   C  if n1's counters (read one step earlier) say it is ready and n1 shares no row with i: issue
//      n1's row loads now, so they fly while i is computed and stored
//   D  compute and store i
//   E  else if n1 is ready except for rows it shares with i: issue its loads now (after i's stores:
//      the same lanes read what they wrote, program order)
//   F  __syncwarp; fence.acq_rel.gpu -- i's stores are visible GPU-wide before G, and every counter
//      value read before it orders the row loads issued after it (relaxed read; fence = acquire)
//   G  lane 0 adds 1 to the counters of i's rows (the release)
//   H  if n1 still waits: spin on its counters (ld.acquire) and then load its rows
// Counter values read before a fence miss the releases of the warp's own last ratings; the checks
// add those in (a row's updates complete in order, so a counter is the length of a completed prefix).
//
// Deadlock freedom: every warp is resident (cooperative launch), walks its positions in increasing
// order and releases a rating before it waits for the next one; a rating only waits for ratings earlier in the
// stream.  The earliest waiting rating therefore waits only on ratings that are done or held by a warp
// that is running, so some warp always makes progress.  A wait longer than 2 s (a broken invariant)
// sets an error flag and gives up instead of hanging the device.
//
// An option (MF_OPT_DET_FLOW = 1), not the default: exact, but slower than the waves on every measured
// shape -- 64 registers hold 32 warps per SM with one rating in flight each (Netflix shape f16 2.46 vs
// 3.09 G updates/s, Yahoo 2.74 vs 4.88, profiles/r02ad_*).
#include <algorithm>

#include "mf_kernels.cuh"
#include "sgd_core.cuh"

namespace mf {
namespace {

constexpr int kFlowBlock = 256;

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
    unsigned x;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned x;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_relaxed_add(unsigned *p, unsigned v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int64_t flow_clock() {
    int64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One 32-sample tile of the wave-sorted stream, lane i holding sample 32 t + i.
struct Tile {
    int32_t u, v, ju, jv;
    float r;
};

struct Smp {  // one rating, warp-uniform
    int32_t u, v, ju, jv;
    float r;
    bool ok;
};

// RR: warp w of W owns stream positions w, w + W, w + 2W, ... (round robin: the positions in flight span
// ~W samples, less than a wave of the Netflix shape); else warps claim 32-sample tiles in order (in
// flight: ~32 W, several waves, so most ratings wait on one still being updated).  MINB: CTAs per SM
// the register budget is sized for (4 -> 64 registers per thread).
template <class SH, bool RR, int MINB>
__global__ void __launch_bounds__(kFlowBlock, MINB) k_flow(UpdateArgs a) {
    static_assert(SH::L == 32, "one rating per warp");
    const int lane = threadIdx.x & 31;
    const int k = SH::FULL ? SH::KMAX : a.k;
    const int64_t N = a.n;
    unsigned *const cu = a.cnt_u;
    unsigned *const cv = a.cnt_v;
    unsigned long long *const ctr = &a.scratch->chunk;
    int bad = 0;
    unsigned long long done = 0;

    const int64_t W = (int64_t)gridDim.x * (kFlowBlock / 32);
    const int64_t wid = warp_uniform(((int64_t)blockIdx.x * kFlowBlock + threadIdx.x) >> 5);
    int64_t next_t = 0;  // RR: the warp's tiles are 0, 1, 2, ... of its own position sequence
    auto claim = [&]() -> int64_t {
        if (RR) return next_t++;
        unsigned long long c = 0;
        if (lane == 0) c = atomicAdd(ctr, 1ull);
        return (int64_t)__shfl_sync(0xffffffffu, c, 0);
    };
    // stream position of slot l of the warp's tile t
    auto position = [&](int64_t t, int l) -> int64_t { return RR ? wid + (t * 32 + l) * W : t * 32 + l; };
    auto load_tile = [&](int64_t t) -> Tile {
        Tile x{-1, 0, 0, 0, 0.f};  // u = -1: past the end of the stream
        const int64_t i = position(t, lane);
        if (i < N) {  // RR: lanes read 32 positions W apart; the CTA's 8 warps read neighbouring ones (L1)
            x.u = __ldg(a.u + i);
            x.v = __ldg(a.v + i);
            x.r = __ldg(a.r + i);
            x.ju = __ldg(a.ord_u + i);
            x.jv = __ldg(a.ord_v + i);
        }
        return x;
    };
    // the window: tile t0 (positions 0..31) and the warp's next tile t1 (32..63)
    int64_t t0 = claim();
    if (position(t0, 0) >= N) return;  // warp-uniform
    int64_t t1 = claim();
    Tile T0 = load_tile(t0), T1 = load_tile(t1);
    auto get = [&](int pos) -> Smp {  // pos warp-uniform
        const bool hi = pos >= 32;
        const int l = pos & 31;
        Smp s;
        s.u = __shfl_sync(0xffffffffu, hi ? T1.u : T0.u, l);
        s.v = __shfl_sync(0xffffffffu, hi ? T1.v : T0.v, l);
        s.ju = __shfl_sync(0xffffffffu, hi ? T1.ju : T0.ju, l);
        s.jv = __shfl_sync(0xffffffffu, hi ? T1.jv : T0.jv, l);
        s.r = __shfl_sync(0xffffffffu, hi ? T1.r : T0.r, l);
        s.ok = s.u >= 0;
        s.u = s.ok ? s.u : 0;
        return s;
    };
    auto spin = [&](const Smp &s) {  // wait until both rows have their earlier updates (acquire)
        const int64_t t_start = flow_clock();
        for (;;) {
            const unsigned a0 = ld_acquire_u32(cu + s.u), b0 = ld_acquire_u32(cv + s.v);
            if (__all_sync(0xffffffffu, a0 >= (unsigned)s.ju && b0 >= (unsigned)s.jv)) return;
            if (flow_clock() - t_start > 2000000000ll) {  // 2 s: an invariant is broken; do not hang
                if (lane == 0) atomicOr(&a.scratch->diverged, 2);
                return;
            }
            __nanosleep(32);
        }
    };

    RowRaw<SH> pr, qr, pr1, qr1;
    int pos = 0;
    Smp cur = get(0);
    Smp prev{-1, -1, 0, 0, 0.f, false};
    // prologue: wait for the first rating, read the next one's counters, fence, load the first rows
    spin(cur);
    Smp nx1 = get(1);
    unsigned c1u = 0, c1v = 0;
    if (nx1.ok) c1u = ld_relaxed_u32(cu + nx1.u), c1v = ld_relaxed_u32(cv + nx1.v);
    fence_acq_rel_gpu();
    load_row<SH>(a.P, cur.u, k, lane, true, pr);
    load_row<SH>(a.Q, cur.v, k, lane, true, qr);

    for (;;) {
        Smp nx2 = get(pos + 2);
        // B: n2's counters, read before this step's fence
        unsigned c2u = 0, c2v = 0;
        if (nx2.ok) c2u = ld_relaxed_u32(cu + nx2.u), c2v = ld_relaxed_u32(cv + nx2.v);
        // C: n1's loads early if it is ready (counts read one step ago plus prev's release) and shares no
        // row with the rating in flight
        const unsigned need_u = nx1.ok ? (unsigned)nx1.ju : 0u, need_v = nx1.ok ? (unsigned)nx1.jv : 0u;
        const unsigned hu = c1u + (prev.ok && nx1.u == prev.u), hv = c1v + (prev.ok && nx1.v == prev.v);
        const bool early = nx1.ok && hu >= need_u && hv >= need_v && nx1.u != cur.u && nx1.v != cur.v;
        if (early) {
            load_row<SH>(a.P, nx1.u, k, lane, true, pr1);
            load_row<SH>(a.Q, nx1.v, k, lane, true, qr1);
        }
        // D: the update of the current rating (PAPER.md:124-126 from the snapshot, A-1)
        {
            float p[SH::E], q[SH::E];
            widen_row<SH>(pr, p);
            widen_row<SH>(qr, q);
            float dot[1] = {lane_dot<SH>(p, q)};
            group_allreduce<SH, 1>(dot);
            const float err = cur.r - dot[0];
            if (!isfinite(err)) bad = 1;
            sgd_step<SH>(p, q, err, a.eta, a.lam);
            narrow_row<SH>(p, pr);
            narrow_row<SH>(q, qr);
            store_row<SH>(a.P, cur.u, k, lane, true, pr);
            store_row<SH>(a.Q, cur.v, k, lane, true, qr);
            done++;
        }
        // E: n1 waits only on rows it shares with the current rating: load them after its stores
        bool issued = early;
        if (!issued && nx1.ok && hu + (nx1.u == cur.u) >= need_u && hv + (nx1.v == cur.v) >= need_v) {
            load_row<SH>(a.P, nx1.u, k, lane, true, pr1);
            load_row<SH>(a.Q, nx1.v, k, lane, true, qr1);
            issued = true;
        }
        // F, G: release the current rating
        __syncwarp();
        fence_acq_rel_gpu();
        if (lane == 0) {
            red_relaxed_add(cu + cur.u, 1u);
            red_relaxed_add(cv + cur.v, 1u);
        }
        if (!nx1.ok) break;  // the stream is sorted, so nothing valid follows (warp-uniform)
        // H: n1 still waits on another warp's rating
        if (!issued) {
            spin(nx1);
            load_row<SH>(a.P, nx1.u, k, lane, true, pr1);
            load_row<SH>(a.Q, nx1.v, k, lane, true, qr1);
        }
        // advance the window
        prev = cur;
        cur = nx1;
        nx1 = nx2;
        c1u = c2u, c1v = c2v;
        pr = pr1, qr = qr1;
        if (++pos == 32) {
            pos = 0;
            t0 = t1;
            T0 = T1;
            t1 = claim();
            T1 = load_tile(t1);
        }
    }
    if (bad) atomicOr(&a.scratch->diverged, 1);
    if (a.count_updates && lane == 0 && done) atomicAdd(&a.scratch->updates, done);
}

// the 32-lane shapes (one rating per warp) for (k, storage)
ShapeId flow_shape_of(int k, int storage) {
    if (k == 128) return storage == kF32 ? ShapeId{storage, 32, 1, 16, 1} : ShapeId{storage, 32, 1, 8, 1};
    if (k == 256) return storage == kF32 ? ShapeId{storage, 32, 2, 16, 1} : ShapeId{storage, 32, 1, 16, 1};
    if (k == 64) return storage == kF32 ? ShapeId{storage, 32, 1, 8, 1} : ShapeId{storage, 32, 1, 4, 1};
    if (k == 32 && storage == kF32) return ShapeId{storage, 32, 1, 4, 1};
    return select_generic_shape(k, storage);
}

template <class F>
cudaError_t dispatch_flow_shape(const ShapeId &s, F &&f) {
#define MF_FCASE(S_, L_, V_, VB_, FULL_)                                                             \
    if (s.storage == S_ && s.L == L_ && s.V == V_ && s.VB == VB_ && s.full == FULL_)                \
        return f(Shape<S_, L_, V_, VB_, (bool)FULL_>{});
    MF_FCASE(kF32, 32, 1, 16, 1) MF_FCASE(kF32, 32, 2, 16, 1) MF_FCASE(kF32, 32, 1, 8, 1) MF_FCASE(kF32, 32, 1, 4, 1)
    MF_FCASE(kF16, 32, 1, 8, 1) MF_FCASE(kF16, 32, 1, 16, 1) MF_FCASE(kF16, 32, 1, 4, 1)
    MF_FCASE(kBF16, 32, 1, 8, 1) MF_FCASE(kBF16, 32, 1, 16, 1) MF_FCASE(kBF16, 32, 1, 4, 1)
    MF_FCASE(kF32, 32, 1, 4, 0) MF_FCASE(kF32, 32, 4, 4, 0) MF_FCASE(kF32, 32, 16, 4, 0) MF_FCASE(kF32, 32, 32, 4, 0)
    MF_FCASE(kF16, 32, 1, 4, 0) MF_FCASE(kF16, 32, 4, 4, 0) MF_FCASE(kF16, 32, 16, 4, 0)
    MF_FCASE(kF16, 32, 1, 2, 0) MF_FCASE(kF16, 32, 4, 2, 0) MF_FCASE(kF16, 32, 16, 2, 0) MF_FCASE(kF16, 32, 32, 2, 0)
    MF_FCASE(kBF16, 32, 1, 4, 0) MF_FCASE(kBF16, 32, 4, 4, 0) MF_FCASE(kBF16, 32, 16, 4, 0)
    MF_FCASE(kBF16, 32, 1, 2, 0) MF_FCASE(kBF16, 32, 4, 2, 0) MF_FCASE(kBF16, 32, 16, 2, 0) MF_FCASE(kBF16, 32, 32, 2, 0)
#undef MF_FCASE
    return cudaErrorInvalidValue;
}

}  // namespace

ShapeId flow_shape(int k, int storage) { return flow_shape_of(k, storage); }

// form: 0 = round robin (default); 2 = tile claims (64 registers either way: capping at 40 or 32 to hold
// more warps spilled 300-500 B per thread and ran 17% / 43% slower on the Netflix shape, r02ad)
cudaError_t launch_flow(const ShapeId &sh, const UpdateArgs &a, cudaStream_t st, int *warps_used, int form) {
    return dispatch_flow_shape(sh, [&](auto tag) -> cudaError_t {
        using SH = decltype(tag);
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // (the masked generic shapes get a 128-register budget: under 64 they spill)
        const void *kern = (const void *)k_flow<SH, true, SH::FULL ? 4 : 2>;
        if constexpr (SH::FULL) {  // tile claims for the vectorised shapes only
            if (form == 2) kern = (const void *)k_flow<SH, false, 4>;
            else form = 0;
        } else {
            form = 0;
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kFlowBlock, 0);
        if (per_sm < 1) return cudaErrorLaunchOutOfResources;
        // every warp resident (cooperative launch), but no more warps than tiles (tile claims) or samples
        const int64_t units = form == 2 ? (a.n + 31) / 32 : a.n;
        int blocks = sms * per_sm;
        const int64_t need = (units + kFlowBlock / 32 - 1) / (kFlowBlock / 32);
        if (need < blocks) blocks = (int)std::max<int64_t>(1, need);
        if (warps_used) *warps_used = blocks * (kFlowBlock / 32);
        cudaError_t e = cudaMemsetAsync(&a.scratch->chunk, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        UpdateArgs args = a;
        void *kargs[] = {&args};
        return cudaLaunchCooperativeKernel(kern, dim3(blocks), dim3(kFlowBlock), kargs, 0, st);
    });
}

}  // namespace mf
