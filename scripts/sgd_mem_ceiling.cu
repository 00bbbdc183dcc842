// sgd_mem_ceiling.cu -- measurement tool (not part of libmf): the memory-system ceiling of the access
// pattern of batch-Hogwild! SGD, without its arithmetic.
//
// Per "update" a group of L lanes reads one 12-byte triple from a streamed R array (u, v, r in three
// SoA arrays, read once, like the real epoch), then reads row p_u of P and row q_v of Q (16 B per lane,
// ld.global.cg), adds 1 to every word and writes both rows back (st.global.cg).  u and v are the
// triple's own indices, drawn uniformly like the synthetic workloads (datagen).  No dot product, no
// shuffles, no conversion: what is left is exactly the update kernel's traffic (12 + 4kb bytes per
// update through L2, 12 + 2kb or more through DRAM), so updates/s here is the ceiling the memory system
// allows for that shape.  Swept over groups in flight per SM and rows in flight per group.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sgd_mem_ceiling scripts/sgd_mem_ceiling.cu
//   /tmp/sgd_mem_ceiling m n N row_bytes [p_only] [warps_per_sm D]   (the last two: one configuration only,
//   for an ncu capture of the pattern's saturated unit)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__global__ void fill_idx(int32_t *u, int32_t *v, float *r, int64_t N, uint32_t m, uint32_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        u[i] = (int32_t)(((z & 0xFFFFFFFFull) * m) >> 32);
        v[i] = (int32_t)(((z >> 32) * n) >> 32);
        r[i] = 1.f;
    }
}

// L lanes per row (row = L * 16 * V bytes), D updates in flight per group; warps walk 32-sample tiles
// QG: also read + write q_v in global memory (batch-Hogwild!); false: P rows only (the CTA wavefront,
// whose Q group lives in shared memory)
template <int L, int V, int D, bool QG = true>
__global__ void __launch_bounds__(256) rmw(const int32_t *__restrict__ u, const int32_t *__restrict__ v,
                                           const float *__restrict__ r, int64_t N, uint4 *P, uint4 *Q,
                                           int64_t active_warps, unsigned long long *ctr) {
    const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L;
    constexpr int G = 32 / L;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (warp >= active_warps) return;
    float acc = 0.f;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(ctr, 256ull);
        base = __shfl_sync(0xffffffffu, base, 0);
        if ((int64_t)base >= N) break;
        for (int t = 0; t < 256; t += 32) {
            const int64_t i = (int64_t)base + t + lane;
            const bool ok = i < N;
            const int32_t tu = ok ? __ldg(u + i) : 0, tv = ok ? __ldg(v + i) : 0;
            acc += ok ? __ldg(r + i) : 0.f;
            for (int j0 = 0; j0 < 32 / G; j0 += D) {
                uint4 pw[D][V], qw[D][V];
                int32_t su[D], sv[D];
                bool val[D];
#pragma unroll
                for (int d = 0; d < D; d++) {
                    const int s = (j0 + d) * G + grp;
                    su[d] = __shfl_sync(0xffffffffu, tu, s);
                    sv[d] = __shfl_sync(0xffffffffu, tv, s);
                    val[d] = (int64_t)base + t + s < N;
                }
#pragma unroll
                for (int d = 0; d < D; d++)
#pragma unroll
                    for (int j = 0; j < V; j++) {
                        if (val[d]) {
                            pw[d][j] = __ldcg(P + (int64_t)su[d] * L * V + j * L + sub);
                            if (QG) qw[d][j] = __ldcg(Q + (int64_t)sv[d] * L * V + j * L + sub);
                        }
                    }
#pragma unroll
                for (int d = 0; d < D; d++)
#pragma unroll
                    for (int j = 0; j < V; j++) {
                        if (val[d]) {
                            uint4 a = pw[d][j], b = QG ? qw[d][j] : pw[d][j];
                            a.x += 1u; a.y += 1u; a.z += 1u; a.w += 1u;
                            b.x += 1u; b.y += 1u; b.z += 1u; b.w += 1u;
                            __stcg(P + (int64_t)su[d] * L * V + j * L + sub, a);
                            if (QG) __stcg(Q + (int64_t)sv[d] * L * V + j * L + sub, b);
                        }
                    }
            }
        }
    }
    if (acc == -1.f) ctr[1] = 1;  // keep the r stream alive
}

template <int L, int V, int D, bool QG>
static double run(const int32_t *u, const int32_t *v, const float *r, int64_t N, uint4 *P, uint4 *Q,
                  int warps_per_sm, int sms, unsigned long long *ctr) {
    const int64_t warps = (int64_t)warps_per_sm * sms;
    const int blocks = (int)((warps * 32 + 255) / 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 3; rep++) {
        cudaMemset(ctr, 0, 16);
        cudaEventRecord(a);
        rmw<L, V, D, QG><<<blocks, 256>>>(u, v, r, N, P, Q, warps, ctr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "%s\n", cudaGetErrorString(e));
        exit(1);
    }
    return N / (best * 1e-3);
}

template <int L, int V, bool QG = true>
static void sweep(const char *label, const int32_t *u, const int32_t *v, const float *r, int64_t N, uint4 *P,
                  uint4 *Q, int sms, unsigned long long *ctr, int row_bytes) {
    const double bytes = QG ? 12 + 4.0 * row_bytes : 12 + 2.0 * row_bytes;  // global bytes per update
    for (int wps : {16, 24, 32, 48, 64}) {
        const double u1 = run<L, V, 1, QG>(u, v, r, N, P, Q, wps, sms, ctr);
        const double u2 = run<L, V, 2, QG>(u, v, r, N, P, Q, wps, sms, ctr);
        const int G = 32 / L;
        printf("{\"shape\": \"%s\", \"rows\": \"%s\", \"row_bytes\": %d, \"warps_per_sm\": %d, "
               "\"in_flight_D1\": %d, \"updates_per_s_D1\": %.4g, \"in_flight_D2\": %d, \"updates_per_s_D2\": %.4g, "
               "\"l2_GBps_D1\": %.1f, \"l2_GBps_D2\": %.1f}\n",
               label, QG ? "p+q" : "p", row_bytes, wps, wps * sms * G, u1, 2 * wps * sms * G, u2, u1 * bytes / 1e9,
               u2 * bytes / 1e9);
        fflush(stdout);
    }
}

int main(int argc, char **argv) {
    const int64_t m = argc > 1 ? atoll(argv[1]) : 480190;
    const int64_t n = argc > 2 ? atoll(argv[2]) : 17771;
    const int64_t N = argc > 3 ? atoll(argv[3]) : 99072112;
    const int row_bytes = argc > 4 ? atoi(argv[4]) : 256;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int32_t *u, *v;
    float *r;
    uint4 *P, *Q;
    unsigned long long *ctr;
    cudaMalloc(&u, N * 4);
    cudaMalloc(&v, N * 4);
    cudaMalloc(&r, N * 4);
    cudaMalloc(&P, m * row_bytes);
    cudaMalloc(&Q, n * row_bytes);
    cudaMalloc(&ctr, 16);
    cudaMemset(P, 0, m * row_bytes);
    cudaMemset(Q, 0, n * row_bytes);
    fill_idx<<<sms * 8, 256>>>(u, v, r, N, (uint32_t)m, (uint32_t)n);
    cudaDeviceSynchronize();
    printf("{\"m\": %lld, \"n\": %lld, \"N\": %lld, \"row_bytes\": %d, \"sms\": %d}\n", (long long)m, (long long)n,
           (long long)N, row_bytes, sms);
    const bool p_only = argc > 5 && atoi(argv[5]) != 0;
    if (argc > 7 && row_bytes == 256 && !p_only) {  // one configuration (L16 x V1, p+q rows)
        const int wps = atoi(argv[6]), D = atoi(argv[7]);
        const double u1 = D == 2 ? run<16, 1, 2, true>(u, v, r, N, P, Q, wps, sms, ctr)
                                 : run<16, 1, 1, true>(u, v, r, N, P, Q, wps, sms, ctr);
        printf("{\"shape\": \"L16xV1\", \"warps_per_sm\": %d, \"D\": %d, \"updates_per_s\": %.4g}\n", wps, D, u1);
        return 0;
    }
    if (row_bytes == 256 && !p_only) {
        sweep<16, 1>("L16xV1", u, v, r, N, P, Q, sms, ctr, row_bytes);
        sweep<8, 2>("L8xV2", u, v, r, N, P, Q, sms, ctr, row_bytes);
    } else if (row_bytes == 512 && !p_only) {
        sweep<32, 1>("L32xV1", u, v, r, N, P, Q, sms, ctr, row_bytes);
        sweep<16, 2>("L16xV2", u, v, r, N, P, Q, sms, ctr, row_bytes);
    } else if (row_bytes == 256) {
        sweep<8, 2, false>("L8xV2", u, v, r, N, P, Q, sms, ctr, row_bytes);
    } else if (row_bytes == 512) {
        sweep<8, 4, false>("L8xV4", u, v, r, N, P, Q, sms, ctr, row_bytes);
    }
    return 0;
}
