// mf_partition.cu -- multi-GPU block partition with Q-segment rotation (§4.1).
//
// The rating matrix is divided into G x G blocks: P into G row segments and Q into G column
// segments (step 1 of P:294-300).  Partition g owns P segment g permanently and the samples of
// row segment g, bucketed by column segment (a stable radix sort keeps the shuffled order inside
// every block).  An epoch is G rounds; in round r partition g updates block (g, sigma_e(g, r)) with
// sigma_e(g, r) = pi_e((g + r) mod G), pi_e a per-epoch random permutation, so the blocks of one
// round never share a row or a column segment (a Latin square, P:129 / P:535) and every block is
// processed once per epoch.  Between rounds each partition sends the Q segment it holds to the
// partition that needs it next and receives its next segment: with NCCL (one process per GPU,
// grouped ncclSend/ncclRecv over NVLink) or, for one-GPU testing, a loopback transport that runs
// the G partitions on the same device and moves segments with device copies.  Unlike the paper
// nothing goes through host memory.
//
// Inside a block the update is batch-Hogwild! (workers = max(1, N_local / 10^4), A-10),
// or exactly serial with MF_OPT_WORKERS = 1 (used for parity).
//
// Unit grid (MF_OPT_PART_SPLIT = 2, the default): the column dimension is cut finer than the workers,
// C = 2G column units (the lower and upper half of every segment), as the paper asks of a grid that
// must keep convergence (§5.5.2) and as its overlap of transfer and compute needs (P:307-314,
// §4.2).  Family h (all lower halves, or all upper halves) rotates by its own randomized Latin square
// per pass, so over a pass every partition visits all 2G units (a randomized G x 2G Latin rectangle:
// in a round no two partitions share a unit, and the pair of units a partition holds changes from
// round to round and pass to pass).  A partition updates its two units concurrently, family 0 on the
// context stream and family 1 on a second stream, with half of the partition's workers each -- the
// same ratings in flight per Q column as one launch over a whole segment -- and each unit is handed on
// (comm stream) as soon as its own sub-block is done, while the other family is still computing; the
// next round of a family waits only for its own unit to arrive.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "mf_ctx.h"
#include "mf_host_util.h"

using namespace mf;

struct mf_nccl {
    ncclComm_t comm = nullptr;
};

namespace {

// ---------------------------------------------------------------- schedule --
void round_perm(std::vector<int32_t> &pi, uint64_t seed, int32_t epoch, int G) {
    permutation(pi, G, host_mix(seed ^ 0xB10CB10Cull ^ ((uint64_t)(uint32_t)epoch << 32)));
}
int32_t sigma(const std::vector<int32_t> &pi, int G, int g, int r) { return pi[(g + r) % G]; }
// unit grid: family h's Latin square of pass p (family 0's is the whole-segment square of round_perm)
void unit_perm(std::vector<int32_t> &pi, uint64_t seed, int32_t pass, int G, int h) {
    round_perm(pi, h ? seed ^ 0x5EC0DF4A11F00D5Eull : seed, pass, G);
}

// segment index of x in [0, extent) split into `parts` (boundaries floor(i*extent/parts))
__device__ __forceinline__ int seg_of(int64_t x, int64_t extent, int parts) {
    int g = (int)((x * parts) / extent);
    if (g + 1 <= parts - 1 && ((int64_t)(g + 1) * extent) / parts <= x) g++;
    return g;
}

// block key = (((pass * local + row segment) * G + column segment) * 2 + half); the pass of stored
// sample i is floor(i * S / n), i.e. every epoch is S passes over consecutive slices of the shuffled
// order; each block is split into the samples of the lower and upper half of its column segment
__global__ void k_part_keys(const int32_t *u, const int32_t *v, int64_t n, int64_t m_rows, int64_t n_cols, int G,
                            int rows_split, int S, int half_split, uint32_t *keys, uint32_t *idx) {
    const int local = rows_split ? G : 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int rs = rows_split ? seg_of(u[i], m_rows, G) : 0;
        const int s = (int)((i * S) / n);
        const int cs = seg_of(v[i], n_cols, G);
        // half: the column segment's lower / upper half of rows (pipelined exchange)
        const int64_t qb = ((int64_t)cs * n_cols) / G, qe = ((int64_t)(cs + 1) * n_cols) / G;
        const int half = half_split && v[i] >= qb + (qe - qb) / 2 ? 1 : 0;
        keys[i] = (uint32_t)(((((int64_t)s * local + rs) * G + cs) << 1) | half);
        idx[i] = (uint32_t)i;
    }
}

// gather into block order; v becomes local to its column segment (unit grid: to its half-segment unit)
__global__ void k_part_gather(const int32_t *u, const int32_t *v, const float *r, const uint32_t *idx,
                              const uint32_t *keys, int64_t n, int64_t n_cols, int G, int unit, int32_t *bu,
                              int32_t *bv, float *br) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = idx[i];
        const int cs = (int)((keys[i] >> 1) % (uint32_t)G);
        const int64_t qb = ((int64_t)cs * n_cols) / G, qe = ((int64_t)(cs + 1) * n_cols) / G;
        const int64_t base = qb + ((unit && (keys[i] & 1u)) ? (qe - qb) / 2 : 0);
        bu[i] = u[j];
        bv[i] = v[j] - (int32_t)base;
        br[i] = r[j];
    }
}

__global__ void k_offsets(const uint32_t *sorted_keys, int64_t n, int64_t nb, int64_t *off) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t prev = i == 0 ? -1 : (int64_t)sorted_keys[i - 1];
        const int64_t cur = i == n ? nb : (int64_t)sorted_keys[i];
        for (int64_t b = prev + 1; b <= cur; b++) off[b] = i;
    }
}

int nccl_fail(mf_ctx *ctx, ncclResult_t r, const char *what) {
    return ctx->fail(MF_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

}  // namespace

#define CK(expr)                                   \
    do {                                           \
        int _rc = cuda((expr), #expr);             \
        if (_rc != MF_OK) return _rc;              \
    } while (0)
#define NK(expr)                                                   \
    do {                                                           \
        ncclResult_t _r = (expr);                                  \
        if (_r != ncclSuccess) return nccl_fail(this, _r, #expr);  \
    } while (0)

// ------------------------------------------------------------ host helpers --
extern "C" int mf_segment(int64_t extent, int32_t parts, int32_t index, int64_t *b, int64_t *e) {
    if (extent < 0 || parts <= 0 || index < 0 || index >= parts || !b || !e) return MF_EINVAL;
    *b = seg_begin(extent, parts, index);
    *e = seg_begin(extent, parts, index + 1);
    return MF_OK;
}

extern "C" int mf_feasibility(int64_t m, int64_t n, int32_t i, int32_t j, int64_t s, int32_t safety, int64_t *bound) {
    if (m <= 0 || n <= 0 || i <= 0 || j <= 0 || s <= 0 || safety <= 0) return MF_EINVAL;
    // s < 1/20 * min(floor(m/i), floor(n/j)), compared exactly (s * safety < min)
    const int64_t mn = std::min(m / i, n / j);
    if (bound) *bound = mn / safety;
    return s * safety < mn ? 1 : 0;
}

extern "C" int mf_round_unit(uint64_t seed, int32_t pass, int32_t G, int32_t round, int32_t rank, int32_t half,
                             int32_t *col_segment) {
    if (G <= 0 || round < 0 || round >= G || rank < 0 || rank >= G || pass < 0 || half < 0 || half > 1 || !col_segment)
        return MF_EINVAL;
    std::vector<int32_t> pi;
    unit_perm(pi, seed, pass, G, half);
    *col_segment = sigma(pi, G, rank, round);
    return MF_OK;
}

extern "C" int mf_round_segment(uint64_t seed, int32_t epoch, int32_t G, int32_t round, int32_t rank,
                                int32_t *col_segment) {
    if (G <= 0 || round < 0 || round >= G || rank < 0 || rank >= G || epoch < 0 || !col_segment) return MF_EINVAL;
    std::vector<int32_t> pi;
    round_perm(pi, seed, epoch, G);
    *col_segment = sigma(pi, G, rank, round);
    return MF_OK;
}

// peers of partition `rank` for the exchange that follows round `round` of `epoch` (the last round
// hands over to round 0 of epoch + 1): it sends its segment to *send_to, receives from *recv_from.
static int family_peers(uint64_t seed, int32_t pass, int32_t G, int32_t round, int32_t rank, int h, int32_t *send_to,
                        int32_t *recv_from) {
    std::vector<int32_t> pi, pn;
    unit_perm(pi, seed, pass, G, h);
    if (round + 1 < G) pn = pi;
    else unit_perm(pn, seed, pass + 1, G, h);
    const int nr = (round + 1) % G;
    std::vector<int32_t> held(G), want(G);
    for (int g = 0; g < G; g++) {
        held[g] = sigma(pi, G, g, round);
        want[g] = sigma(pn, G, g, nr);
    }
    for (int x = 0; x < G; x++) {
        if (want[x] == held[rank]) *send_to = x;
        if (held[x] == want[rank]) *recv_from = x;
    }
    return MF_OK;
}

// peers of partition `rank` for the exchange that follows round `round` of pass `pass` (the last round
// hands over to round 0 of pass + 1): it sends its segment to *send_to, receives from *recv_from.
extern "C" int mf_round_peers(uint64_t seed, int32_t epoch, int32_t G, int32_t round, int32_t rank,
                              int32_t *send_to, int32_t *recv_from) {
    if (G <= 0 || round < 0 || round >= G || rank < 0 || rank >= G || epoch < 0 || !send_to || !recv_from)
        return MF_EINVAL;
    return family_peers(seed, epoch, G, round, rank, 0, send_to, recv_from);
}

extern "C" int mf_unit_peers(uint64_t seed, int32_t pass, int32_t G, int32_t round, int32_t rank, int32_t half,
                             int32_t *send_to, int32_t *recv_from) {
    if (G <= 0 || round < 0 || round >= G || rank < 0 || rank >= G || pass < 0 || half < 0 || half > 1 || !send_to ||
        !recv_from)
        return MF_EINVAL;
    return family_peers(seed, pass, G, round, rank, half, send_to, recv_from);
}

// ------------------------------------------------------------------ NCCL ----
extern "C" int mf_nccl_unique_id(void *out128) {
    if (!out128) return MF_EINVAL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MF_ENCCL;
    std::memcpy(out128, &id, sizeof id);
    return MF_OK;
}

extern "C" int mf_attach_nccl(mf_ctx *ctx, const void *id128, int rank, int world) {
    if (!ctx || !id128 || world < 1 || rank < 0 || rank >= world) return MF_EINVAL;
    if (ctx->P || ctx->N > 0 || ctx->nccl) return ctx->fail(MF_ESTATE, "mf_attach_nccl must precede loading and factors");
    if (ctx->m < world || ctx->n < world) return ctx->fail(MF_EINVAL, "need m, n >= world");
    int rc = ctx->ensure_device();
    if (rc != MF_OK) return rc;
    cudaSetDevice(ctx->device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    mf_nccl *nc = new mf_nccl();
    ncclResult_t r = ncclCommInitRank(&nc->comm, world, id, rank);
    if (r != ncclSuccess) {
        delete nc;
        return ctx->fail(MF_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    ctx->nccl = nc;
    ctx->rank = rank;
    ctx->world = world;
    ctx->p_begin = seg_begin(ctx->m, world, rank);
    ctx->p_end = seg_begin(ctx->m, world, rank + 1);
    return MF_OK;
}

// ---------------------------------------------------------------- layout ----
void mf_ctx::release_partition() {
    for (void *p : {(void *)bu, (void *)bv, (void *)br, gather_tmp, (void *)agree_buf})
        if (p) cudaFree(p);
    bu = bv = nullptr;
    br = nullptr;
    gather_tmp = nullptr;
    agree_buf = nullptr;
    for (auto *vec : {&q_cur, &q_next})
        for (void *p : *vec)
            if (p) cudaFree(p);
    q_cur.clear();
    q_next.clear();
    for (int h = 0; h < 2; h++) {
        for (auto *vec : {&u_cur[h], &u_next[h]})
            for (void *p : *vec)
                if (p) cudaFree(p);
        u_cur[h].clear(), u_next[h].clear(), held_u[h].clear();
    }
    held.clear();
    h_blk_off.clear();
    seg_valid = false;
    part_valid = false;
    recv_pending = false;
    for (auto *ev : {&ev_half[0], &ev_half[1], &ev_recv[0], &ev_recv[1]})
        if (*ev) cudaEventDestroy(*ev), *ev = nullptr;
    if (comm_stream) cudaStreamDestroy(comm_stream);
    comm_stream = nullptr;
    if (stream2) cudaStreamDestroy(stream2);
    stream2 = nullptr;
    for (auto *ev : {&ev_fork, &ev_join})
        if (*ev) cudaEventDestroy(*ev), *ev = nullptr;
    if (nccl) {
        if (nccl->comm) ncclCommDestroy(nccl->comm);
        delete nccl;
        nccl = nullptr;
    }
}

int mf_ctx::build_partition() {
    if (part_valid) return MF_OK;
    const int G = is_distributed() ? world : std::max(1, partitions);
    if (G > n || G > p_rows() * (is_distributed() ? world : 1))
        return fail(MF_EINVAL, "partitioned: G = %d exceeds the matrix dimensions", G);
    const int local = is_distributed() ? 1 : G;
    // A previous layout may still hold the only current copy of Q in its segment buffers (an option
    // that changes the layout was set between partitioned epochs): bring it home before freeing them.
    if (seg_valid && !full_valid) {
        const int rc = gather_q();
        if (rc != MF_OK) return rc;
    }
    if (comm_stream) cudaStreamSynchronize(comm_stream);  // no hand-over may still target old buffers
    recv_pending = false;
    // free a previous layout's buffers (keep the NCCL comm)
    for (void *p : {(void *)bu, (void *)bv, (void *)br})
        if (p) cudaFree(p);
    bu = bv = nullptr;
    br = nullptr;
    for (auto *vec : {&q_cur, &q_next, &u_cur[0], &u_next[0], &u_cur[1], &u_next[1]})
        for (void *p : *vec)
            if (p) cudaFree(p);
    const int mode = part_split;
    q_cur.assign(mode == 2 ? 0 : local, nullptr);
    q_next.assign(mode == 2 ? 0 : local, nullptr);
    for (int h = 0; h < 2; h++) {
        u_cur[h].assign(mode == 2 ? local : 0, nullptr);
        u_next[h].assign(mode == 2 ? local : 0, nullptr);
    }
    seg_valid = false;

    cudaStream_t st = stream();
    // Passes per epoch S (auto).  In a pass every Q unit is visited once by each partition, so a Q row
    // takes (N / n) / (S G) consecutive updates from one row segment per visit.  Serial block-sweep
    // simulation on C2-1pct: S = 1 costs +10..+20% in test RMSE, S = 4 is within 0.05% for G <= 4.  At the
    // full Hugewiki shape (N / n = 77k ratings per column) S = 4 leaves 2.4k-9.6k updates per visit and
    // the schedule far behind serial SGD (G = 2 / 4 / 8: +59% / +8.7% / +3.5% after 10 epochs,
    // profiles/r02m_c4_traces.jsonl), while the Hugewiki parity slice (<= ~1k per visit) stays within
    // 0.5%.  So S = max(4, ceil(N_total / (n G kVisit))) caps a visit at kVisit updates per Q row; every
    // pass costs 2G launches (~25-35 us fixed each), so the cap is not smaller.  With NCCL every rank
    // must run the same S: N_total is all-reduced.
    constexpr double kVisit = 1000.0;
    int64_t n_total = N;
    if (is_distributed()) {
        if (!agree_buf) CK(cudaMalloc((void **)&agree_buf, sizeof(double) * 8));
        const double mine = (double)N;
        CK(cudaMemcpyAsync(agree_buf, &mine, sizeof(double), cudaMemcpyHostToDevice, st));
        NK(ncclAllReduce(agree_buf, agree_buf, 1, ncclFloat64, ncclSum, nccl->comm, st));
        double tot = 0.0;
        CK(cudaMemcpyAsync(&tot, agree_buf, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        n_total = (int64_t)tot;
    }
    const int S_auto = (int)std::min<double>(512.0, std::max(4.0, std::ceil((double)n_total / ((double)n * G * kVisit))));
    const int S_req = subepochs > 0 ? subepochs : S_auto;
    const int S = (int)std::max<int64_t>(1, std::min<int64_t>(S_req, std::max<int64_t>(1, N)));
    const int64_t nb = (int64_t)S * local * G * 2;
    if (nb >= (1ll << 31)) return fail(MF_EINVAL, "partitioned: too many blocks (S * G * G * 2)");
    uint32_t *k0 = nullptr, *k1 = nullptr, *i0 = nullptr, *i1 = nullptr;
    int64_t *doff = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    CK(cudaMalloc((void **)&bu, sizeof(int32_t) * std::max<int64_t>(N, 1)));
    CK(cudaMalloc((void **)&bv, sizeof(int32_t) * std::max<int64_t>(N, 1)));
    CK(cudaMalloc((void **)&br, sizeof(float) * std::max<int64_t>(N, 1)));
    CK(cudaMallocAsync((void **)&k0, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&k1, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&i0, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&i1, sizeof(uint32_t) * N, st));
    CK(cudaMallocAsync((void **)&doff, sizeof(int64_t) * (nb + 1), st));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 148 * 16));
    // loopback: rows are global, split into G segments; NCCL: u is already local to this rank's segment
    k_part_keys<<<grid, 256, 0, st>>>(u, v, N, m, n, G, is_distributed() ? 0 : 1, S, mode != 0, k0, i0);
    CK(cudaGetLastError());
    int bits = 1;
    while (bits < 32 && (1ull << bits) < (uint64_t)nb) bits++;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, i0, i1, N, 0, bits, st));
    CK(cudaMallocAsync(&tmp, tmp_bytes, st));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, i0, i1, N, 0, bits, st));  // stable
    k_part_gather<<<grid, 256, 0, st>>>(u, v, r, i1, k1, N, n, G, mode == 2, bu, bv, br);
    CK(cudaGetLastError());
    k_offsets<<<grid, 256, 0, st>>>(k1, N, nb, doff);
    CK(cudaGetLastError());
    h_blk_off.assign((size_t)nb + 1, 0);
    CK(cudaMemcpyAsync(h_blk_off.data(), doff, sizeof(int64_t) * (nb + 1), cudaMemcpyDeviceToHost, st));
    for (void *p : {(void *)tmp, (void *)k0, (void *)k1, (void *)i0, (void *)i1, (void *)doff}) CK(cudaFreeAsync(p, st));
    CK(cudaStreamSynchronize(st));

    seg_rows_max = 0;
    for (int c = 0; c < G; c++) seg_rows_max = std::max(seg_rows_max, seg_begin(n, G, c + 1) - seg_begin(n, G, c));
    unit_rows_max = (seg_rows_max + 1) / 2;
    const size_t bytes = (size_t)seg_rows_max * k * storage_bytes();
    const size_t ubytes = (size_t)std::max<int64_t>(1, unit_rows_max) * k * storage_bytes();
    for (int g = 0; g < local; g++) {
        if (mode == 2) {
            for (int h = 0; h < 2; h++) {
                CK(cudaMalloc(&u_cur[h][g], ubytes));
                CK(cudaMalloc(&u_next[h][g], ubytes));
            }
        } else {
            CK(cudaMalloc(&q_cur[g], bytes));
            CK(cudaMalloc(&q_next[g], bytes));
        }
    }
    if (!comm_stream) CK(cudaStreamCreateWithFlags(&comm_stream, cudaStreamNonBlocking));
    if (!stream2) CK(cudaStreamCreateWithFlags(&stream2, cudaStreamNonBlocking));
    for (auto *ev : {&ev_half[0], &ev_half[1], &ev_recv[0], &ev_recv[1], &ev_fork, &ev_join})
        if (!*ev) CK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    part_G = G;
    part_local = local;
    part_S = S;
    part_mode = mode;
    held.assign(G, -1);
    held_u[0].assign(G, -1);
    held_u[1].assign(G, -1);
    part_valid = true;
    return MF_OK;
}

// Move segments so that partition g holds want[g]: g sends what it holds to the partition that wants
// it and receives what it wants from the partition holding it (one send + one recv per partition).
int mf_ctx::exchange_segments(const std::vector<int32_t> &want) {
    const int G = part_G;
    const size_t bytes = (size_t)seg_rows_max * k * storage_bytes();
    cudaStream_t st = stream();
    std::vector<int> dst(G), src(G);
    for (int g = 0; g < G; g++)
        for (int h = 0; h < G; h++) {
            if (want[h] == held[g]) dst[g] = h;
            if (held[h] == want[g]) src[g] = h;
        }
    if (is_distributed()) {
        const int g = rank;
        if (dst[g] != g) {
            NK(ncclGroupStart());
            NK(ncclSend(q_cur[0], bytes, ncclUint8, dst[g], nccl->comm, st));
            NK(ncclRecv(q_next[0], bytes, ncclUint8, src[g], nccl->comm, st));
            NK(ncclGroupEnd());
            std::swap(q_cur[0], q_next[0]);
        }
    } else {
        for (int g = 0; g < G; g++)
            if (dst[g] != g) CK(cudaMemcpyAsync(q_next[dst[g]], q_cur[g], bytes, cudaMemcpyDeviceToDevice, st));
        for (int g = 0; g < G; g++)
            if (dst[g] != g) std::swap(q_cur[g], q_next[g]);
    }
    held = want;
    return MF_OK;
}

// full Q -> segment buffers (partition g takes want[g])
static int scatter_segments(mf_ctx *ctx, const std::vector<int32_t> &want) {
    const int G = ctx->part_G;
    const size_t rb = (size_t)ctx->k * ctx->storage_bytes();
    for (int li = 0; li < ctx->part_local; li++) {
        const int g = ctx->is_distributed() ? ctx->rank : li;
        const int64_t b = seg_begin(ctx->n, G, want[g]), e = seg_begin(ctx->n, G, want[g] + 1);
        int rc = ctx->cuda(cudaMemcpyAsync(ctx->q_cur[li], (char *)ctx->Q + b * rb, (e - b) * rb,
                                           cudaMemcpyDeviceToDevice, ctx->stream()), "scatter Q");
        if (rc != MF_OK) return rc;
    }
    ctx->held = want;
    ctx->seg_valid = true;
    return MF_OK;
}

// segment buffers -> full Q (collective with NCCL: all-gather of the held segments)
int mf_ctx::gather_q() {
    if (full_valid) return MF_OK;
    if (!seg_valid) return fail(MF_ESTATE, "no valid copy of Q");
    if (part_mode == 2) return gather_units();
    const int G = part_G;
    const size_t rb = (size_t)k * storage_bytes();
    const size_t bytes = (size_t)seg_rows_max * rb;
    cudaStream_t st = stream();
    if (recv_pending) {  // the last round's hand-over is still on the comm stream
        CK(cudaStreamWaitEvent(st, ev_recv[0], 0));
        CK(cudaStreamWaitEvent(st, ev_recv[1], 0));
        recv_pending = false;
    }
    if (is_distributed()) {
        if (!gather_tmp) CK(cudaMalloc(&gather_tmp, bytes * G));
        NK(ncclAllGather(q_cur[0], gather_tmp, bytes, ncclUint8, nccl->comm, st));
        for (int h = 0; h < G; h++) {
            const int64_t b = seg_begin(n, G, held[h]), e = seg_begin(n, G, held[h] + 1);
            CK(cudaMemcpyAsync((char *)Q + b * rb, (char *)gather_tmp + h * bytes, (e - b) * rb,
                               cudaMemcpyDeviceToDevice, st));
        }
    } else {
        for (int g = 0; g < G; g++) {
            const int64_t b = seg_begin(n, G, held[g]), e = seg_begin(n, G, held[g] + 1);
            CK(cudaMemcpyAsync((char *)Q + b * rb, q_cur[g], (e - b) * rb, cudaMemcpyDeviceToDevice, st));
        }
    }
    CK(cudaStreamSynchronize(st));
    full_valid = true;
    return MF_OK;
}

// ----------------------------------------------------------------- epoch ----
int mf_ctx::epoch_partitioned(mf_epoch_stats *stats) {
    if (!is_distributed() && partitions < 1) return fail(MF_EINVAL, "set MF_OPT_PARTITIONS or attach NCCL");
    int rc = build_partition();
    if (rc != MF_OK) return rc;
    if (part_mode == 2) return epoch_units(stats);
    const int G = part_G;
    cudaStream_t st = stream();
    const int S = part_S, L = part_local;
    const float eta = eta_at(epoch);
    const ShapeId sh = hogwild_shape(k, storage, hog_shape_sel());
    auto blk = [&](int s, int li, int c, int h) { return ((((size_t)s * L + li) * G + c) << 1) | (size_t)h; };
    std::vector<int64_t> n_local(L, 0);  // samples of each hosted partition per epoch (worker clamp, A-10)
    for (int s = 0; s < S; s++)
        for (int li = 0; li < L; li++) n_local[li] += h_blk_off[blk(s, li, G - 1, 1) + 1] - h_blk_off[blk(s, li, 0, 0)];
    int launches = 0, used_max = 0;
    CK(cudaEventRecord(events[0], st));
    CK(cudaMemsetAsync(scratch, 0, sizeof(DevScratch), st));
    CK(cudaEventRecord(events[1], st));
    std::vector<int32_t> pi, want(G), next(G);
    // segments for round 0 of this epoch's first pass (normally already in place: the last round of
    // the previous epoch handed them over)
    round_perm(pi, seed_shuffle, epoch * S, G);
    for (int g = 0; g < G; g++) want[g] = sigma(pi, G, g, 0);
    if (!seg_valid) {
        rc = scatter_segments(this, want);
        recv_pending = false;
    } else if (held != want) {
        if (recv_pending) {
            CK(cudaStreamWaitEvent(st, ev_recv[0], 0));
            CK(cudaStreamWaitEvent(st, ev_recv[1], 0));
            recv_pending = false;
        }
        rc = exchange_segments(want);
    }
    if (rc != MF_OK) return rc;
    full_valid = false;
    // An epoch is S passes; pass p = eS + s runs the G rounds of Latin square pi_p.  Each round runs
    // the lower-half sub-block, then the upper-half sub-block of every hosted block; the lower half of
    // the Q segment is sent to the next holder (comm stream) while the upper half is still computing,
    // and the next round starts on its lower half as soon as that half has arrived.
    for (int s = 0; s < S; s++) {
        round_perm(pi, seed_shuffle, epoch * S + s, G);
        for (int r = 0; r < G; r++) {
            for (int g = 0; g < G; g++) want[g] = sigma(pi, G, g, r);
            if (r + 1 < G) {
                for (int g = 0; g < G; g++) next[g] = sigma(pi, G, g, r + 1);
            } else {  // hand over to round 0 of the next pass (of this or the next epoch)
                std::vector<int32_t> pn;
                round_perm(pn, seed_shuffle, epoch * S + s + 1, G);
                for (int g = 0; g < G; g++) next[g] = sigma(pn, G, g, 0);
            }
            for (int h = 0; h < 2; h++) {
                if (recv_pending && part_mode) CK(cudaStreamWaitEvent(st, ev_recv[h], 0));
                if (recv_pending && !part_mode && h == 0) {  // one launch over the whole segment: both halves
                    CK(cudaStreamWaitEvent(st, ev_recv[0], 0));
                    CK(cudaStreamWaitEvent(st, ev_recv[1], 0));
                }
                for (int li = 0; li < L; li++) {
                    const int g = is_distributed() ? rank : li;
                    const size_t b = blk(s, li, want[g], h);
                    const int64_t lo = h_blk_off[b], hi = h_blk_off[b + 1];
                    if (hi <= lo) continue;
                    UpdateArgs a = update_args(eta);
                    a.u = bu + lo;
                    a.v = bv + lo;
                    a.r = br + lo;
                    a.n = hi - lo;
                    a.Q = q_cur[li];
                    a.q_share *= (float)(part_mode ? 2 * G : G);  // the launch's Q rows: a segment or half of one
                    const int w = workers > 0 ? workers
                                              : (int)std::max<int64_t>(1, std::min<int64_t>(n_local[li] / 10000, 1 << 30));
                    int used = 0;
                    CK(launch_hogwild(sh, a, w, variant, st, &used));
                    used_max = std::max(used_max, used);
                    last_kappa = std::max(last_kappa, (double)used * a.q_share);
                    launches++;
                }
                rc = exchange_half(next, h);
                if (rc != MF_OK) return rc;
            }
            for (int li = 0; li < L; li++) std::swap(q_cur[li], q_next[li]);
            held = next;
            recv_pending = true;
        }
    }
    CK(cudaEventRecord(events[2], st));
    return finish_epoch(MF_SCHED_PARTITIONED, eta, launches, used_max, stats);
}

// Half h (0: rows [0, len/2), 1: rows [len/2, len) of a segment) of every held Q segment moves toward
// `want` on the comm stream, after the compute stream has finished this round's half-h sub-blocks;
// the receive lands in q_next.  Staying segments (dst == self) are copied locally so that q_next is
// complete when the buffers swap.
int mf_ctx::exchange_half(const std::vector<int32_t> &want, int h) {
    const int G = part_G;
    const size_t rb = (size_t)k * storage_bytes();
    cudaStream_t st = stream(), cs = comm_stream;
    auto half_rows = [&](int c, int64_t *off, int64_t *rows) {
        const int64_t len = seg_begin(n, G, c + 1) - seg_begin(n, G, c), hm = len / 2;
        *off = h ? hm : 0;
        *rows = h ? len - hm : hm;
    };
    CK(cudaEventRecord(ev_half[h], st));
    CK(cudaStreamWaitEvent(cs, ev_half[h], 0));
    std::vector<int> dst(G), src(G);
    for (int g = 0; g < G; g++)
        for (int x = 0; x < G; x++) {
            if (want[x] == held[g]) dst[g] = x;
            if (held[x] == want[g]) src[g] = x;
        }
    for (int li = 0; li < part_local; li++) {
        const int g = is_distributed() ? rank : li;
        int64_t so, sr, ro, rr;
        half_rows(held[g], &so, &sr);
        half_rows(want[g], &ro, &rr);
        const char *sbuf = (const char *)q_cur[li] + so * rb;
        if (is_distributed()) {
            char *rbuf = (char *)q_next[0] + ro * rb;
            if (dst[g] == g) {
                if (sr) CK(cudaMemcpyAsync(rbuf, sbuf, sr * rb, cudaMemcpyDeviceToDevice, cs));
            } else {
                NK(ncclGroupStart());
                if (sr) NK(ncclSend(sbuf, sr * rb, ncclUint8, dst[g], nccl->comm, cs));
                if (rr) NK(ncclRecv(rbuf, rr * rb, ncclUint8, src[g], nccl->comm, cs));
                NK(ncclGroupEnd());
            }
        } else if (sr) {  // loopback: partition g's half lands in the receive buffer of partition dst[g]
            CK(cudaMemcpyAsync((char *)q_next[dst[g]] + so * rb, sbuf, sr * rb, cudaMemcpyDeviceToDevice, cs));
        }
    }
    CK(cudaEventRecord(ev_recv[h], cs));
    return MF_OK;
}

// ------------------------------------------------------------- unit grid ----
void mf_ctx::unit_rows(int c, int h, int64_t *row0, int64_t *rows) const {
    const int64_t b = seg_begin(n, part_G, c), len = seg_begin(n, part_G, c + 1) - b, hm = len / 2;
    *row0 = b + (h ? hm : 0);
    *rows = h ? len - hm : hm;
}

// full Q -> unit buffers (partition g takes unit (want[h][g], h) of both families)
int mf_ctx::scatter_units(const std::vector<int32_t> (&want)[2]) {
    const size_t rb = (size_t)k * storage_bytes();
    for (int h = 0; h < 2; h++) {
        for (int li = 0; li < part_local; li++) {
            const int g = is_distributed() ? rank : li;
            int64_t r0, rows;
            unit_rows(want[h][g], h, &r0, &rows);
            if (rows) CK(cudaMemcpyAsync(u_cur[h][li], (char *)Q + r0 * rb, rows * rb, cudaMemcpyDeviceToDevice, stream()));
        }
        held_u[h] = want[h];
    }
    seg_valid = true;
    return MF_OK;
}

// unit buffers -> full Q (collective with NCCL: one all-gather per family)
int mf_ctx::gather_units() {
    const int G = part_G;
    const size_t rb = (size_t)k * storage_bytes();
    const size_t ubytes = (size_t)std::max<int64_t>(1, unit_rows_max) * rb;
    cudaStream_t st = stream();
    if (recv_pending) {  // the last round's hand-overs are still on the comm stream
        CK(cudaStreamWaitEvent(st, ev_recv[0], 0));
        CK(cudaStreamWaitEvent(st, ev_recv[1], 0));
        recv_pending = false;
    }
    if (is_distributed()) {
        if (!gather_tmp) CK(cudaMalloc(&gather_tmp, 2 * ubytes * G));
        for (int h = 0; h < 2; h++) {
            char *dst = (char *)gather_tmp + (size_t)h * G * ubytes;
            NK(ncclAllGather(u_cur[h][0], dst, ubytes, ncclUint8, nccl->comm, st));
            for (int x = 0; x < G; x++) {
                int64_t r0, rows;
                unit_rows(held_u[h][x], h, &r0, &rows);
                if (rows) CK(cudaMemcpyAsync((char *)Q + r0 * rb, dst + x * ubytes, rows * rb, cudaMemcpyDeviceToDevice, st));
            }
        }
    } else {
        for (int h = 0; h < 2; h++)
            for (int g = 0; g < G; g++) {
                int64_t r0, rows;
                unit_rows(held_u[h][g], h, &r0, &rows);
                if (rows) CK(cudaMemcpyAsync((char *)Q + r0 * rb, u_cur[h][g], rows * rb, cudaMemcpyDeviceToDevice, st));
            }
    }
    CK(cudaStreamSynchronize(st));
    full_valid = true;
    return MF_OK;
}

// Family h's units move toward `want` on the comm stream once the compute stream hs has finished the
// family's sub-blocks of this round; the receive lands in u_next[h] (the caller swaps the buffers).  A
// unit that stays (dst == self) is copied locally so that u_next is complete.
int mf_ctx::exchange_unit(const std::vector<int32_t> &want, int h, cudaStream_t hs) {
    const int G = part_G;
    const size_t rb = (size_t)k * storage_bytes();
    cudaStream_t cs = comm_stream;
    CK(cudaEventRecord(ev_half[h], hs));
    CK(cudaStreamWaitEvent(cs, ev_half[h], 0));
    const std::vector<int32_t> &have = held_u[h];
    std::vector<int> dst(G), src(G);
    for (int g = 0; g < G; g++)
        for (int x = 0; x < G; x++) {
            if (want[x] == have[g]) dst[g] = x;
            if (have[x] == want[g]) src[g] = x;
        }
    for (int li = 0; li < part_local; li++) {
        const int g = is_distributed() ? rank : li;
        int64_t s0, sr, r0, rr;
        unit_rows(have[g], h, &s0, &sr);
        unit_rows(want[g], h, &r0, &rr);
        if (is_distributed()) {
            if (dst[g] == g) {
                if (sr) CK(cudaMemcpyAsync(u_next[h][0], u_cur[h][0], sr * rb, cudaMemcpyDeviceToDevice, cs));
            } else {
                NK(ncclGroupStart());
                if (sr) NK(ncclSend(u_cur[h][0], sr * rb, ncclUint8, dst[g], nccl->comm, cs));
                if (rr) NK(ncclRecv(u_next[h][0], rr * rb, ncclUint8, src[g], nccl->comm, cs));
                NK(ncclGroupEnd());
            }
        } else if (sr) {  // loopback: partition g's unit lands in the receive buffer of partition dst[g]
            CK(cudaMemcpyAsync(u_next[h][dst[g]], u_cur[h][li], sr * rb, cudaMemcpyDeviceToDevice, cs));
        }
    }
    CK(cudaEventRecord(ev_recv[h], cs));
    return MF_OK;
}

int mf_ctx::epoch_units(mf_epoch_stats *stats) {
    const int G = part_G;
    cudaStream_t st = stream();
    const int S = part_S, L = part_local;
    const float eta = eta_at(epoch);
    const ShapeId sh = hogwild_shape(k, storage, hog_shape_sel());
    auto blk = [&](int s, int li, int c, int h) { return ((((size_t)s * L + li) * G + c) << 1) | (size_t)h; };
    std::vector<int64_t> n_local(L, 0);  // samples of each hosted partition per epoch (worker clamp, A-10)
    for (int s = 0; s < S; s++)
        for (int li = 0; li < L; li++) n_local[li] += h_blk_off[blk(s, li, G - 1, 1) + 1] - h_blk_off[blk(s, li, 0, 0)];
    // MF_OPT_WORKERS = 1 is the exact mode: one rating at a time per partition, so the two families run
    // one after the other on the context stream (family 0's sub-blocks, then family 1's, every round)
    const bool serial = workers == 1;
    int launches = 0, used_max = 0;
    CK(cudaEventRecord(events[0], st));
    CK(cudaMemsetAsync(scratch, 0, sizeof(DevScratch), st));
    CK(cudaEventRecord(events[1], st));
    std::vector<int32_t> pi[2], want[2], next[2];
    for (int h = 0; h < 2; h++) {
        want[h].assign(G, 0), next[h].assign(G, 0);
        unit_perm(pi[h], seed_shuffle, epoch * S, G, h);
        for (int g = 0; g < G; g++) want[h][g] = sigma(pi[h], G, g, 0);
    }
    int rc = MF_OK;
    if (!seg_valid) {
        rc = scatter_units(want);
        recv_pending = false;
    } else {
        for (int h = 0; h < 2 && rc == MF_OK; h++) {
            if (held_u[h] == want[h]) continue;  // normally in place: the previous epoch's last round handed it over
            if (recv_pending) CK(cudaStreamWaitEvent(st, ev_recv[h], 0));
            rc = exchange_unit(want[h], h, st);
            for (int li = 0; li < L; li++) std::swap(u_cur[h][li], u_next[h][li]);
            held_u[h] = want[h];
            CK(cudaStreamWaitEvent(st, ev_recv[h], 0));
        }
    }
    if (rc != MF_OK) return rc;
    full_valid = false;
    CK(cudaEventRecord(ev_fork, st));
    CK(cudaStreamWaitEvent(stream2, ev_fork, 0));
    for (int s = 0; s < S; s++) {
        for (int h = 0; h < 2; h++) unit_perm(pi[h], seed_shuffle, epoch * S + s, G, h);
        for (int r = 0; r < G; r++) {
            int used_round = 0;
            for (int h = 0; h < 2; h++) {
                for (int g = 0; g < G; g++) want[h][g] = sigma(pi[h], G, g, r);
                if (r + 1 < G) {
                    for (int g = 0; g < G; g++) next[h][g] = sigma(pi[h], G, g, r + 1);
                } else {  // hand over to round 0 of the next pass (of this or the next epoch)
                    std::vector<int32_t> pn;
                    unit_perm(pn, seed_shuffle, epoch * S + s + 1, G, h);
                    for (int g = 0; g < G; g++) next[h][g] = sigma(pn, G, g, 0);
                }
                cudaStream_t hs = (serial || h == 0) ? st : stream2;
                if (recv_pending) CK(cudaStreamWaitEvent(hs, ev_recv[h], 0));
                for (int li = 0; li < L; li++) {
                    const int g = is_distributed() ? rank : li;
                    const size_t b = blk(s, li, want[h][g], h);
                    const int64_t lo = h_blk_off[b], hi = h_blk_off[b + 1];
                    if (hi <= lo) continue;
                    UpdateArgs a = update_args(eta);
                    a.u = bu + lo;
                    a.v = bv + lo;
                    a.r = br + lo;
                    a.n = hi - lo;
                    a.Q = u_cur[h][li];
                    a.q_share *= (float)(2 * G);  // the launch's Q rows: one unit (half a segment)
                    a.chunk_ctr = h ? &scratch->chunk2 : &scratch->chunk;
                    const int64_t wp = workers > 0 ? workers : std::max<int64_t>(1, std::min<int64_t>(n_local[li] / 10000, 1 << 30));
                    const int w = serial ? 1 : (int)std::max<int64_t>(1, wp / 2);  // half of the partition's workers per family
                    int used = 0;
                    CK(launch_hogwild(sh, a, w, variant, hs, &used));
                    used_round += used;
                    last_kappa = std::max(last_kappa, (double)used * a.q_share);
                    launches++;
                }
                rc = exchange_unit(next[h], h, hs);
                if (rc != MF_OK) return rc;
                for (int li = 0; li < L; li++) std::swap(u_cur[h][li], u_next[h][li]);
                held_u[h] = next[h];
            }
            used_max = std::max(used_max, serial ? 1 : used_round / std::max(1, L));
            recv_pending = true;
        }
    }
    CK(cudaEventRecord(ev_join, stream2));
    CK(cudaStreamWaitEvent(st, ev_join, 0));
    CK(cudaEventRecord(events[2], st));
    return finish_epoch(MF_SCHED_PARTITIONED, eta, launches, used_max, stats);
}

// Collective status agreement: each rank contributes its local status; every rank
// returns the most negative status any rank had.  A rank that fails an argument check, a validation or
// diverges therefore still enters the collective, its peers are never left blocked in an NCCL call,
// and all ranks report the same outcome.  One all-reduce of a per-code count vector (fp64 sum).
int mf_ctx::agree(int local) {
    if (!is_distributed()) return local;
    constexpr int kCodes = 8;  // statuses 0 .. -7
    if (!agree_buf) CK(cudaMalloc((void **)&agree_buf, sizeof(double) * kCodes));
    double h[kCodes] = {0};
    if (local < 0 && local > -kCodes) h[-local] = 1.0;
    cudaStream_t st = stream();
    CK(cudaMemcpyAsync(agree_buf, h, sizeof h, cudaMemcpyHostToDevice, st));
    NK(ncclAllReduce(agree_buf, agree_buf, kCodes, ncclFloat64, ncclSum, nccl->comm, st));
    CK(cudaMemcpyAsync(h, agree_buf, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int c = kCodes - 1; c >= 1; c--)
        if (h[c] > 0) {
            if (local == -c) return local;  // keep this rank's own message
            return fail(-c, "a peer rank failed this collective call with %s", mf_status_string(-c));
        }
    return local;  // (a local status outside the code range is returned unchanged)
}

int mf_ctx::rmse_partitioned(int64_t nnz, double *out) {
    // caller (mf_rmse) validated the local test triples, rebased u and gathered Q; nnz may be 0 here
    cudaStream_t st = stream();
    const ShapeId sh = select_shape(k, storage, 0);
    if (nnz > 0) {
        CK(launch_rmse(sh, tu, tv, tr, nnz, P, Q, k, partials, rmse_parts(), d_out, st, 0));
    } else {
        CK(cudaMemsetAsync(d_out, 0, sizeof(double), st));
    }
    double cnt = (double)nnz;
    CK(cudaMemcpyAsync(d_out + 1, &cnt, sizeof(double), cudaMemcpyHostToDevice, st));
    NK(ncclAllReduce(d_out, d_out, 2, ncclFloat64, ncclSum, nccl->comm, st));
    double h[2];
    CK(cudaMemcpyAsync(h, d_out, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!(h[1] > 0)) return fail(MF_EINVAL, "mf_rmse: the test shards of all ranks are empty");
    *out = std::sqrt(h[0] / h[1]);
    return MF_OK;
}
