// mf_host_util.h -- host-side counter-hash helpers for the schedulers (column sequences, round
// permutations).  Deterministic functions of (seed, epoch, index) so every rank derives the same
// schedule without communication.
#pragma once

#include <cstdint>
#include <numeric>
#include <utility>
#include <vector>

namespace mf {

inline uint64_t host_mix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Fisher-Yates permutation of [0, n) driven by a counter hash stream keyed by `key`
inline void permutation(std::vector<int32_t> &out, int n, uint64_t key) {
    out.resize(n);
    std::iota(out.begin(), out.end(), 0);
    for (int i = n - 1; i > 0; i--) {
        const uint64_t h = host_mix(key ^ (uint64_t)i * 0xD1B54A32D192ED03ull);
        const int j = (int)(h % (uint64_t)(i + 1));
        std::swap(out[i], out[j]);
    }
}

#ifdef __CUDACC__
#define MF_HD __host__ __device__
#else
#define MF_HD
#endif

// segment g of [0, extent) split into `parts` near-equal pieces: [floor(g*extent/parts), ...)
MF_HD inline int64_t seg_begin(int64_t extent, int parts, int g) { return extent * g / parts; }

// index of the segment holding x (inverse of seg_begin); widths differ by at most one
MF_HD inline int seg_index(int64_t x, int64_t extent, int parts) {
    int g = (int)((x * parts) / extent);
    if (g + 1 <= parts - 1 && ((int64_t)(g + 1) * extent) / parts <= x) g++;
    return g;
}

}  // namespace mf
