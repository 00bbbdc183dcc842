// l2_ceiling.cu -- measurement tool (not part of libmf): the B200's L2 bandwidth ceilings that bound the
// SGD update kernels when their working set is L2-resident (the Netflix shape: Q 4.5 MB, P 123 MB fp16).
//
// MEASURED_PEAKS.json has the HBM copy peak only; a kernel whose rows hit L2 moves more algorithmic bytes
// per second than that, so its roofline denominator must be an L2 figure.  Three patterns,
// each timed with CUDA events (best of 5 after a warm-up) over a buffer that fits the 126 MB L2:
//   stream_rw  every thread reads a 16-B vector with ld.global.cg, adds 1, writes it back (st.global.cg):
//              contiguous, fully coalesced read+write -- the L2's sustained read+write bandwidth.
//   stream_rd  the same loads, no stores (sum kept alive) -- the L2 read bandwidth.
//   rows_rw    the update's own L2 access shape: a group of L lanes reads one whole row (L x 16 B) at a
//              uniformly random row index, adds 1 to every word and writes it back; rows_bytes = 256
//              (fp16, k = 128) or 512 (fp32) -- random-row read-modify-write out of L2.
// Bytes counted: 2 x buffer per pass (rw), 1 x buffer (rd), 2 x row bytes per row (rows_rw).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/l2_ceiling scripts/l2_ceiling.cu
//   /tmp/l2_ceiling [buffer_MB]          -> one JSON line per pattern / size
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__global__ void __launch_bounds__(512) stream_rw(uint4 *buf, int64_t nvec, int passes) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; p++)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += stride) {
            uint4 x = __ldcg(buf + i);
            x.x += 1u; x.y += 1u; x.z += 1u; x.w += 1u;
            __stcg(buf + i, x);
        }
}

__global__ void __launch_bounds__(512) stream_rd(const uint4 *buf, int64_t nvec, int passes, unsigned *sink) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (int p = 0; p < passes; p++)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nvec; i += stride) {
            const uint4 x = __ldcg(buf + i);
            acc ^= x.x ^ x.y ^ x.z ^ x.w;
        }
    if (acc == 0x12345678u) *sink = acc;
}

// L lanes x 16 B = one row; D rows in flight per group; nrows rows in the buffer; `updates` row RMWs total
template <int L, int D>
__global__ void __launch_bounds__(512) rows_rw(uint4 *buf, int64_t nrows, int64_t updates) {
    const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L;
    constexpr int G = 32 / L;
    const int64_t gid = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * G + grp;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x >> 5) * G;
    for (int64_t j = gid * D; j < updates; j += ngroups * D) {
        int64_t row[D];
        uint4 x[D];
#pragma unroll
        for (int d = 0; d < D; d++) {
            uint64_t z = (uint64_t)(j + d) * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            row[d] = (int64_t)(((z & 0xFFFFFFFFull) * (uint64_t)nrows) >> 32);
            x[d] = __ldcg(buf + row[d] * L + sub);
        }
#pragma unroll
        for (int d = 0; d < D; d++) {
            x[d].x += 1u; x[d].y += 1u; x[d].z += 1u; x[d].w += 1u;
            __stcg(buf + row[d] * L + sub, x[d]);
        }
    }
}

static int g_sms = 0;

template <class F>
static float best_ms(F &&launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();  // warm-up (also pulls the buffer into L2)
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        fprintf(stderr, "%s\n", cudaGetErrorString(e));
        exit(1);
    }
    return best;
}

template <int L, int D>
static void rows(uint4 *buf, int64_t bytes, int blocks_per_sm) {
    const int row_bytes = L * 16;
    const int64_t nrows = bytes / row_bytes;
    const int64_t updates = 64ll << 20;
    const float ms = best_ms([&] { rows_rw<L, D><<<g_sms * blocks_per_sm, 512>>>(buf, nrows, updates); });
    printf("{\"pattern\": \"rows_rw\", \"row_bytes\": %d, \"rows_in_flight_per_group\": %d, \"buffer_MB\": %.1f, "
           "\"ctas_per_sm\": %d, \"ms\": %.4f, \"rows_per_s\": %.4g, \"GBps\": %.1f}\n",
           row_bytes, D, bytes / 1048576.0, blocks_per_sm, ms, updates / (ms * 1e-3),
           2.0 * row_bytes * updates / (ms * 1e-3) / 1e9);
    fflush(stdout);
}

int main(int argc, char **argv) {
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    const double mbs[] = {8, 16, 32, 48, 64, 96};
    const int nmb = argc > 1 ? 1 : 6;
    uint4 *buf;
    unsigned *sink;
    cudaMalloc(&buf, 96ll << 20);
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 0, 96ll << 20);
    printf("{\"device_sms\": %d, \"l2_bytes\": %d}\n", g_sms, l2);
    for (int t = 0; t < nmb; t++) {
        const double mb = argc > 1 ? atof(argv[1]) : mbs[t];
        const int64_t bytes = (int64_t)(mb * 1048576.0);
        const int64_t nvec = bytes / 16;
        const int passes = 8;
        for (int bps : {2, 4}) {
            const float ms = best_ms([&] { stream_rw<<<g_sms * bps, 512>>>(buf, nvec, passes); });
            printf("{\"pattern\": \"stream_rw\", \"buffer_MB\": %.1f, \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n",
                   mb, bps, ms, 2.0 * bytes * passes / (ms * 1e-3) / 1e9);
            const float ms2 = best_ms([&] { stream_rd<<<g_sms * bps, 512>>>(buf, nvec, passes, sink); });
            printf("{\"pattern\": \"stream_rd\", \"buffer_MB\": %.1f, \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n",
                   mb, bps, ms2, 1.0 * bytes * passes / (ms2 * 1e-3) / 1e9);
            fflush(stdout);
        }
        for (int bps : {2, 4}) {
            rows<16, 1>(buf, bytes, bps);
            rows<16, 2>(buf, bytes, bps);
            rows<32, 1>(buf, bytes, bps);
            rows<32, 2>(buf, bytes, bps);
        }
    }
    return 0;
}
