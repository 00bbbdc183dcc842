// sgd_core.cuh -- device-side building blocks of one SGD update (sm_100a).
//
// One rating r_uv is handled by a GROUP of L consecutive lanes of a warp
// (L = 4..32, sized by k and the storage width; PAPER.md:188 used a fixed
// 32-thread worker).  Lane `sub` of the group owns V vectors of VB bytes of
// each of p_u and q_v; vector j of lane sub covers elements
//     d = (j*L + sub)*EPV ... +EPV-1,        EPV = VB / sizeof(storage)
// so every load/store instruction of the group touches one contiguous
// L*VB-byte span of the row (coalesced).
//
// Per update (§2.2):
//   dot  = sum_d p[d] q[d]       fp32 FMA per lane, then __shfl_xor_sync tree over
//                                the L lanes ("warp shuffle")
//   err  = r - dot
//   p'   = p + eta (err q - lambda p),  q' = q + eta (err p - lambda q)
//          both from the snapshot p, q held in registers (A-1);
//          fp32 math, storage fp32 / fp16 / bf16 rounded to nearest even
//          (A-13).
//
// P and Q are read with ld.global.cg (L2, not L1): they are written
// concurrently by other SMs, so they must never go through the
// non-coherent read-only path (__ldg is only for R).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "mf_kernels.cuh"

namespace mf {



// ---------------------------------------------------------------- vectors --
template <int VB>
struct Vec;  // VB bytes held in NW 32-bit words
template <>
struct Vec<16> {
    static constexpr int NW = 4;
    static __device__ __forceinline__ void ld(const void *p, uint32_t (&w)[4]) {
        uint4 x = __ldcg(reinterpret_cast<const uint4 *>(p));
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
    }
    // (a weak ld.global.L1::no_allocate variant measured 4-13% slower than ld.global.cg here: r01)
    static __device__ __forceinline__ void st(void *p, const uint32_t (&w)[4]) {
        __stcg(reinterpret_cast<uint4 *>(p), make_uint4(w[0], w[1], w[2], w[3]));
    }
};
// the same 16-B accesses with an L2 eviction-priority policy (createpolicy), still .cg (L2-coherent)
__device__ __forceinline__ void ld16_pol(const void *p, uint32_t (&w)[4], uint64_t pol) {
    asm volatile("ld.global.cg.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                 : "l"(p), "l"(pol));
}
__device__ __forceinline__ void st16_pol(void *p, const uint32_t (&w)[4], uint64_t pol) {
    asm volatile("st.global.cg.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(w[0]), "r"(w[1]),
                 "r"(w[2]), "r"(w[3]), "l"(pol)
                 : "memory");
}
template <>
struct Vec<8> {
    static constexpr int NW = 2;
    static __device__ __forceinline__ void ld(const void *p, uint32_t (&w)[2]) {
        uint2 x = __ldcg(reinterpret_cast<const uint2 *>(p));
        w[0] = x.x; w[1] = x.y;
    }
    static __device__ __forceinline__ void st(void *p, const uint32_t (&w)[2]) {
        __stcg(reinterpret_cast<uint2 *>(p), make_uint2(w[0], w[1]));
    }
};
template <>
struct Vec<4> {
    static constexpr int NW = 1;
    static __device__ __forceinline__ void ld(const void *p, uint32_t (&w)[1]) {
        w[0] = __ldcg(reinterpret_cast<const unsigned int *>(p));
    }
    static __device__ __forceinline__ void st(void *p, const uint32_t (&w)[1]) {
        __stcg(reinterpret_cast<unsigned int *>(p), w[0]);
    }
};
template <>
struct Vec<2> {  // one 16-bit element in the low half of w[0]
    static constexpr int NW = 1;
    static __device__ __forceinline__ void ld(const void *p, uint32_t (&w)[1]) {
        w[0] = __ldcg(reinterpret_cast<const unsigned short *>(p));
    }
    static __device__ __forceinline__ void st(void *p, const uint32_t (&w)[1]) {
        __stcg(reinterpret_cast<unsigned short *>(p), (unsigned short)(w[0] & 0xFFFFu));
    }
};

// ---------------------------------------------------------------- storage --
template <int S>
struct Storage;
template <>
struct Storage<kF32> {
    static constexpr int BYTES = 4;
    template <int NW>
    static __device__ __forceinline__ void widen(const uint32_t (&w)[NW], float *x, int n) {
#pragma unroll
        for (int i = 0; i < NW; i++) x[i] = __uint_as_float(w[i]);
    }
    template <int NW>
    static __device__ __forceinline__ void narrow(const float *x, uint32_t (&w)[NW], int n) {
#pragma unroll
        for (int i = 0; i < NW; i++) w[i] = __float_as_uint(x[i]);
    }
};
template <>
struct Storage<kF16> {
    static constexpr int BYTES = 2;
    template <int NW>
    static __device__ __forceinline__ void widen(const uint32_t (&w)[NW], float *x, int n) {
        if (n == 1) {
            x[0] = __half2float(__ushort_as_half((unsigned short)(w[0] & 0xFFFFu)));
            return;
        }
#pragma unroll
        for (int i = 0; i < NW; i++) {
            __half2 h = *reinterpret_cast<const __half2 *>(&w[i]);
            float2 f = __half22float2(h);
            x[2 * i] = f.x;
            x[2 * i + 1] = f.y;
        }
    }
    template <int NW>
    static __device__ __forceinline__ void narrow(const float *x, uint32_t (&w)[NW], int n) {
        if (n == 1) {
            w[0] = __half_as_ushort(__float2half_rn(x[0]));
            return;
        }
#pragma unroll
        for (int i = 0; i < NW; i++) {
            __half2 h = __floats2half2_rn(x[2 * i], x[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t *>(&h);
        }
    }
};
template <>
struct Storage<kBF16> {
    static constexpr int BYTES = 2;
    template <int NW>
    static __device__ __forceinline__ void widen(const uint32_t (&w)[NW], float *x, int n) {
        if (n == 1) {
            x[0] = __uint_as_float(w[0] << 16);
            return;
        }
#pragma unroll
        for (int i = 0; i < NW; i++) {
            x[2 * i] = __uint_as_float(w[i] << 16);
            x[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
    template <int NW>
    static __device__ __forceinline__ void narrow(const float *x, uint32_t (&w)[NW], int n) {
        if (n == 1) {
            w[0] = __bfloat16_as_ushort(__float2bfloat16_rn(x[0]));
            return;
        }
#pragma unroll
        for (int i = 0; i < NW; i++) {
            __nv_bfloat162 h = __floats2bfloat162_rn(x[2 * i], x[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t *>(&h);
        }
    }
};

// ------------------------------------------------------------- group shape --
// S storage kind, L lanes per rating, V vectors per lane, VB bytes per vector,
// FULL: k == KMAX exactly (no masking).
template <int S_, int L_, int V_, int VB_, bool FULL_>
struct Shape {
    static constexpr int S = S_, L = L_, V = V_, VB = VB_;
    static constexpr bool FULL = FULL_;
    static constexpr int BYTES = Storage<S>::BYTES;
    static constexpr int EPV = VB / BYTES;  // elements per vector
    static constexpr int NW = Vec<VB>::NW;  // 32-bit words per vector
    static constexpr int E = V * EPV;       // elements per lane
    static constexpr int KMAX = L * E;      // largest k this shape covers
    static constexpr int G = 32 / L;        // groups (concurrent ratings) per warp
    static_assert(32 % L == 0, "L must divide 32");
    static_assert(EPV >= 1, "vector narrower than one element");
};

// One lane's slice of a feature row, raw storage words.
template <class SH>
struct RowRaw {
    uint32_t w[SH::V][SH::NW];
};

// byte offset of vector j of lane `sub` inside a row
template <class SH>
__device__ __forceinline__ int64_t vec_elem(int j, int sub) {
    return (int64_t)(j * SH::L + sub) * SH::EPV;
}

template <class SH>
__device__ __forceinline__ void load_row(const void *base, int64_t row, int k, int sub, bool valid,
                                         RowRaw<SH> &out) {
    const char *rp = reinterpret_cast<const char *>(base) + row * (int64_t)k * SH::BYTES;
#pragma unroll
    for (int j = 0; j < SH::V; j++) {
        const int64_t e = vec_elem<SH>(j, sub);
        if (valid && (SH::FULL || e < k)) {
            Vec<SH::VB>::ld(rp + e * SH::BYTES, out.w[j]);
        } else {
#pragma unroll
            for (int i = 0; i < SH::NW; i++) out.w[j][i] = 0u;
        }
    }
}

// load_row / store_row with an L2 policy (16-B full-row shapes; other shapes ignore the policy)
template <class SH>
__device__ __forceinline__ void load_row_pol(const void *base, int64_t row, int k, int sub, bool valid,
                                             RowRaw<SH> &out, uint64_t pol) {
    if constexpr (SH::VB == 16 && SH::FULL) {
        const char *rp = reinterpret_cast<const char *>(base) + row * (int64_t)k * SH::BYTES;
#pragma unroll
        for (int j = 0; j < SH::V; j++) {
            if (valid) {
                ld16_pol(rp + vec_elem<SH>(j, sub) * SH::BYTES, out.w[j], pol);
            } else {
#pragma unroll
                for (int i = 0; i < SH::NW; i++) out.w[j][i] = 0u;
            }
        }
    } else {
        load_row<SH>(base, row, k, sub, valid, out);
    }
}

template <class SH>
__device__ __forceinline__ void store_row(void *base, int64_t row, int k, int sub, bool valid, const RowRaw<SH> &in);

template <class SH>
__device__ __forceinline__ void store_row_pol(void *base, int64_t row, int k, int sub, bool valid,
                                              const RowRaw<SH> &in, uint64_t pol) {
    if constexpr (SH::VB == 16 && SH::FULL) {
        char *rp = reinterpret_cast<char *>(base) + row * (int64_t)k * SH::BYTES;
#pragma unroll
        for (int j = 0; j < SH::V; j++)
            if (valid) st16_pol(rp + vec_elem<SH>(j, sub) * SH::BYTES, in.w[j], pol);
    } else {
        store_row<SH>(base, row, k, sub, valid, in);
    }
}

// L2 eviction-priority policies (fraction 1.0: every access of the instruction gets the priority)
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// evict_last for a fraction of the lines (chosen by address, so a line keeps its priority), the rest
// evict_unchanged: pins part of a row array that does not fit L2 as a whole
__device__ __forceinline__ uint64_t policy_evict_last_frac(float f) {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, %1;" : "=l"(p) : "f"(f));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// streamed read-only words (the COO triples): non-coherent path, no L1 allocation, L2 policy
__device__ __forceinline__ int32_t ld_stream_s32(const int32_t *p, uint64_t pol) {
    int32_t x;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(x) : "l"(p), "l"(pol));
    return x;
}
__device__ __forceinline__ float ld_stream_f32(const float *p, uint64_t pol) {
    float x;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(x) : "l"(p), "l"(pol));
    return x;
}

template <class SH>
__device__ __forceinline__ void store_row(void *base, int64_t row, int k, int sub, bool valid, const RowRaw<SH> &in) {
    char *rp = reinterpret_cast<char *>(base) + row * (int64_t)k * SH::BYTES;
#pragma unroll
    for (int j = 0; j < SH::V; j++) {
        const int64_t e = vec_elem<SH>(j, sub);
        if (valid && (SH::FULL || e < k)) Vec<SH::VB>::st(rp + e * SH::BYTES, in.w[j]);
    }
}

// ------------------------------------------------------ atomic write-back --
// One vector of a row increased in place by an L2 atomic add (red.global.add, no return value): the
// vector forms of sm_90+ (.v4/.v2 .f32, .v4/.v2 .f16x2 / .bf16x2), one 16-, 8- or 4-byte request per
// lane like the plain store.  fp32 adds flush subnormal results to zero (REDG ...FTZ.RN); 16-bit adds
// round to nearest even (.noftz).
template <int S, int VB>
struct RedVec;
template <>
struct RedVec<kF32, 16> {
    static __device__ __forceinline__ void red(void *p, const uint32_t (&w)[4], uint64_t pol) {
        asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(__uint_as_float(w[0])),
                     "f"(__uint_as_float(w[1])), "f"(__uint_as_float(w[2])), "f"(__uint_as_float(w[3])), "l"(pol)
                     : "memory");
    }
};
template <>
struct RedVec<kF32, 8> {
    static __device__ __forceinline__ void red(void *p, const uint32_t (&w)[2], uint64_t pol) {
        asm volatile("red.global.add.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(__uint_as_float(w[0])),
                     "f"(__uint_as_float(w[1])), "l"(pol)
                     : "memory");
    }
};
template <>
struct RedVec<kF32, 4> {
    static __device__ __forceinline__ void red(void *p, const uint32_t (&w)[1], uint64_t pol) {
        asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(__uint_as_float(w[0])), "l"(pol)
                     : "memory");
    }
};
#define MF_RED16(S_, T_)                                                                                          \
    template <>                                                                                                   \
    struct RedVec<S_, 16> {                                                                                       \
        static __device__ __forceinline__ void red(void *p, const uint32_t (&w)[4], uint64_t pol) {               \
            asm volatile("red.global.add.noftz.L2::cache_hint.v4." T_ "x2 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),  \
                         "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "l"(pol)                                     \
                         : "memory");                                                                             \
        }                                                                                                         \
    };                                                                                                            \
    template <>                                                                                                   \
    struct RedVec<S_, 8> {                                                                                        \
        static __device__ __forceinline__ void red(void *p, const uint32_t (&w)[2], uint64_t pol) {               \
            asm volatile("red.global.add.noftz.L2::cache_hint.v2." T_ "x2 [%0], {%1, %2}, %3;" ::"l"(p), "r"(w[0]), \
                         "r"(w[1]), "l"(pol)                                                                      \
                         : "memory");                                                                             \
        }                                                                                                         \
    };                                                                                                            \
    template <>                                                                                                   \
    struct RedVec<S_, 4> {                                                                                        \
        static __device__ __forceinline__ void red(void *p, const uint32_t (&w)[1], uint64_t pol) {               \
            asm volatile("red.global.add.noftz.L2::cache_hint." T_ "x2 [%0], %1, %2;" ::"l"(p), "r"(w[0]), "l"(pol) \
                         : "memory");                                                                             \
        }                                                                                                         \
    };                                                                                                            \
    template <>                                                                                                   \
    struct RedVec<S_, 2> {                                                                                        \
        static __device__ __forceinline__ void red(void *p, const uint32_t (&w)[1], uint64_t pol) {               \
            const unsigned short h = (unsigned short)(w[0] & 0xFFFFu);                                            \
            asm volatile("red.global.add.noftz.L2::cache_hint." T_ " [%0], %1, %2;" ::"l"(p), "h"(h), "l"(pol)    \
                         : "memory");                                                                             \
        }                                                                                                         \
    };
MF_RED16(kF16, "f16")
MF_RED16(kBF16, "bf16")
#undef MF_RED16

template <class SH>
__device__ __forceinline__ void widen_row(const RowRaw<SH> &in, float (&x)[SH::E]);
template <class SH>
__device__ __forceinline__ void narrow_row(const float (&x)[SH::E], RowRaw<SH> &out);

// Write-back of an updated row as the atomic add of its change: the row in memory becomes
// row + (new - old), old being the snapshot this update read (A-20).  With no concurrent
// writer that is the new row (to the rounding of the change into storage precision); with one, both
// changes land, where a plain store keeps only the last writer's row.
template <class SH>
__device__ __forceinline__ void red_row_delta(void *base, int64_t row, int k, int sub, bool valid,
                                              const RowRaw<SH> &old, const float (&nw)[SH::E], uint64_t pol) {
    float dl[SH::E];
    widen_row<SH>(old, dl);
#pragma unroll
    for (int e = 0; e < SH::E; e++) dl[e] = nw[e] - dl[e];
    RowRaw<SH> w;
    narrow_row<SH>(dl, w);
    char *rp = reinterpret_cast<char *>(base) + row * (int64_t)k * SH::BYTES;
#pragma unroll
    for (int j = 0; j < SH::V; j++) {
        const int64_t e = vec_elem<SH>(j, sub);
        if (valid && (SH::FULL || e < k)) RedVec<SH::S, SH::VB>::red(rp + e * SH::BYTES, w.w[j], pol);
    }
}

template <class SH>
__device__ __forceinline__ void widen_row(const RowRaw<SH> &in, float (&x)[SH::E]) {
#pragma unroll
    for (int j = 0; j < SH::V; j++) Storage<SH::S>::template widen<SH::NW>(in.w[j], &x[j * SH::EPV], SH::EPV);
}

template <class SH>
__device__ __forceinline__ void narrow_row(const float (&x)[SH::E], RowRaw<SH> &out) {
#pragma unroll
    for (int j = 0; j < SH::V; j++) Storage<SH::S>::template narrow<SH::NW>(&x[j * SH::EPV], out.w[j], SH::EPV);
}

// fp32 partial dot of this lane, then xor-butterfly over the L lanes of the
// group.  Every lane of the warp must call it (full-warp shuffles).
template <class SH>
__device__ __forceinline__ float lane_dot(const float (&p)[SH::E], const float (&q)[SH::E]) {
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < SH::E; e++) s = fmaf(p[e], q[e], s);
    return s;
}

// D independent butterflies interleaved level by level (ILP across the D ratings of a group)
template <class SH, int D>
__device__ __forceinline__ void group_allreduce(float (&s)[D]) {
#pragma unroll
    for (int o = SH::L / 2; o > 0; o >>= 1) {
        float t[D];
#pragma unroll
        for (int d = 0; d < D; d++) t[d] = __shfl_xor_sync(0xffffffffu, s[d], o);
#pragma unroll
        for (int d = 0; d < D; d++) s[d] += t[d];
    }
}

template <class SH>
__device__ __forceinline__ float group_dot(const float (&p)[SH::E], const float (&q)[SH::E]) {
    float s[1] = {lane_dot<SH>(p, q)};
    group_allreduce<SH, 1>(s);
    return s[0];
}

// p' = p + eta (err q - lambda p), q' = q + eta (err p - lambda q), snapshot semantics, evaluated as
// p' = (1 - eta lambda) p + (eta err) q: the same affine map with two fp32 operations per element
// (one FMUL, one FFMA) instead of three; the rounding differs from the oracle's left-to-right
// evaluation by O(2^-24) relative per update (tolerances).
template <class SH>
__device__ __forceinline__ void sgd_step(float (&p)[SH::E], float (&q)[SH::E], float err, float eta, float lam) {
    const float a = 1.f - eta * lam, b = eta * err;
    if constexpr (SH::E % 2 == 0) {
        // sm_100 paired fp32 (FMUL2/FFMA2): each lane of the pair is rounded exactly as the scalar
        // fmaf/fmul below, so results are bit-identical with half the issue slots
        const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
#pragma unroll
        for (int e = 0; e < SH::E; e += 2) {
            const float2 pe = make_float2(p[e], p[e + 1]), qe = make_float2(q[e], q[e + 1]);
            const float2 pn = __ffma2_rn(b2, qe, __fmul2_rn(a2, pe));
            const float2 qn = __ffma2_rn(b2, pe, __fmul2_rn(a2, qe));
            p[e] = pn.x, p[e + 1] = pn.y, q[e] = qn.x, q[e + 1] = qn.y;
        }
    } else {
#pragma unroll
        for (int e = 0; e < SH::E; e++) {
            const float pe = p[e], qe = q[e];
            p[e] = fmaf(b, qe, a * pe);
            q[e] = fmaf(b, pe, a * qe);
        }
    }
}

// one bulk L2 prefetch of a whole feature row (cp.async.bulk.prefetch: 16-B aligned, size % 16 == 0)
__device__ __forceinline__ void prefetch_row_l2(const void *base, int64_t row, uint32_t row_bytes) {
    const char *p = reinterpret_cast<const char *>(base) + row * (int64_t)row_bytes;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(row_bytes) : "memory");
}

// A warp-uniform value as the compiler sees it: the broadcast of lane 0's value.  An index derived from
// threadIdx.x (a warp's id, a warp's first sample) is the same on every lane, but the compiler's
// divergence analysis cannot know that; branches and loop bounds computed from it make every shuffle
// after them "possibly divergent", and ptxas then wraps each SHFL in WARPSYNC.COLLECTIVE fix-up code
// (ncu: 385 instructions per rating in the warp-worker wavefront).  Shuffle results are uniform to it.
__device__ __forceinline__ int64_t warp_uniform(int64_t x) {
    return (int64_t)__shfl_sync(0xffffffffu, (unsigned long long)x, 0);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace mf
