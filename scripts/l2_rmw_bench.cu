// l2_rmw_bench.cu -- measurement tool (not part of libmf): the memory-system ceiling for the access
// pattern of one SGD update, i.e. random whole-row read-modify-write through L2.
//
// For a table of `rows` rows of `row_bytes` bytes, every warp repeatedly picks a random row (counter
// hash), loads it with ld.global.cg (16 B per lane, like the update kernels), adds 1 to each word and
// stores it back with st.global.cg.  Reported: bytes moved (read + write) per second.  With the table
// L2-resident (<= 64 MB) this is the SM<->L2 RMW ceiling; with a 2 GB table it is the DRAM ceiling for
// random 256/512-byte rows.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_rmw_bench l2_rmw_bench.cu && ./l2_rmw_bench
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// L lanes per row (row_bytes = 16 L), 32/L rows per warp instruction, D rows in flight per group
template <int L, int D>
__global__ void rmw(uint4 *table, int64_t rows, int64_t iters, uint64_t seed) {
    const int lane = threadIdx.x & 31, grp = lane / L, sub = lane % L;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    for (int64_t it = 0; it < iters; it++) {
        uint4 v[D];
        int64_t row[D];
#pragma unroll
        for (int d = 0; d < D; d++) {
            row[d] = (int64_t)(mix(seed ^ ((gw * iters + it) * 64 + grp * D + d)) % (uint64_t)rows);
            v[d] = __ldcg(table + row[d] * L + sub);
        }
#pragma unroll
        for (int d = 0; d < D; d++) {
            v[d].x += 1u; v[d].y += 1u; v[d].z += 1u; v[d].w += 1u;
            __stcg(table + row[d] * L + sub, v[d]);
        }
    }
}

template <int L, int D>
static double run(int64_t table_bytes, int blocks, int threads, int64_t iters) {
    const int64_t rows = table_bytes / (16 * L);
    uint4 *t;
    cudaMalloc(&t, rows * 16 * L);
    cudaMemset(t, 0, rows * 16 * L);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    rmw<L, D><<<blocks, threads>>>(t, rows, iters / 4, 1);  // warm
    cudaEventRecord(a);
    rmw<L, D><<<blocks, threads>>>(t, rows, iters, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double row_updates = (double)blocks * threads / 32 * (32 / L) * D * iters;
    cudaFree(t);
    return row_updates * 2.0 * 16 * L / (ms * 1e-3) / 1e9;  // GB/s, read + write
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256;
    printf("{\"sms\": %d, \"results\": [\n", sms);
    const int64_t sizes[] = {32ll << 20, 64ll << 20, 2048ll << 20};
    bool first = true;
    for (int64_t sz : sizes) {
        for (int bps : {4, 6, 8}) {
            const int blocks = sms * bps;
            const double g16 = run<16, 8>(sz, blocks, threads, 1000);  // 256-byte rows (k=128 fp16), 8 in flight
            const double g32 = run<32, 8>(sz, blocks, threads, 500);   // 512-byte rows (k=128 fp32)
            printf("%s {\"table_MB\": %lld, \"warps_per_sm\": %d, \"rmw_GBps_256B_rows\": %.1f, "
                   "\"rmw_GBps_512B_rows\": %.1f}",
                   first ? "" : ",\n", (long long)(sz >> 20), bps * threads / 32, g16, g32);
            first = false;
        }
    }
    printf("\n]}\n");
    return 0;
}
