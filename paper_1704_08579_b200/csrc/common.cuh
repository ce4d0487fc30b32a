// common.cuh -- shared device helpers for the B200 hybrid sort (sm_100a).
//
// Element kinds follow the reference's ElemKind (lanes.py:50-63): int32 keys
// with sentinel INT32_MAX, float64 keys with sentinel +inf.  Keys are compared
// by VALUE (never by bit pattern), so -0.0 == +0.0 exactly as in the
// reference's ordered-quiet compares.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace vx {

constexpr int kWarp = 32;

// Checked build (-DVX_CHECK; tools/check_build.sh): device-side assertions on
// every bucket index, staging slot and destination index of the kernels.  A
// failed assertion traps, which fails the launch and every test after it.
// (compute-sanitizer is closed on this GPU pool; these bounds checks plus
// the canary tests stand in for memcheck.)
#ifdef VX_CHECK
#define VX_ASSERT(cond)                                                    \
    do {                                                                   \
        if (!(cond)) {                                                     \
            printf("VX_ASSERT failed: %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            __trap();                                                      \
        }                                                                  \
    } while (0)
#else
#define VX_ASSERT(cond) \
    do {                \
    } while (0)
#endif

template <typename K>
struct KeyTraits;
template <>
struct KeyTraits<int32_t> {
    __host__ __device__ static constexpr int32_t sentinel() { return 0x7fffffff; }
};
template <>
struct KeyTraits<double> {
    __host__ __device__ static constexpr double sentinel() { return __builtin_huge_val(); }
};

// Order-preserving uint64 code of a float64 (sign-magnitude -> two's
// complement order): value order is preserved for every non-NaN key, the one
// refinement being -0.0 < +0.0, which the reference treats as equal, so any
// order of the two is a correct sort.
__device__ __forceinline__ uint64_t f64_to_ord(double d) {
    const uint64_t u = (uint64_t)__double_as_longlong(d);
    return u ^ ((uint64_t)((int64_t)u >> 63) | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ord_to_f64(uint64_t o) {
    const uint64_t m = (o >> 63) ? 0x8000000000000000ULL : ~0ULL;
    return __longlong_as_double((long long)(o ^ m));
}

// Representation the bitonic networks compare in.  float64 networks compare
// doubles directly (DSETP + selects: measured 2-4x faster than emulating
// 64-bit integer min/max); VX_F64_ORDERED_NETWORK switches them to the uint64
// codes above.  The classifiers always use the codes (see OKey in qsort.cuh).
template <typename K>
struct KeyRep {
    using I = K;
    __device__ __forceinline__ static I to(K k) { return k; }
    __device__ __forceinline__ static K from(I i) { return i; }
};
#ifdef VX_F64_ORDERED_NETWORK
template <>
struct KeyRep<double> {
    using I = uint64_t;
    __device__ __forceinline__ static I to(double d) { return f64_to_ord(d); }
    __device__ __forceinline__ static double from(I o) { return ord_to_f64(o); }
};
#endif
template <>
struct KeyTraits<uint64_t> {
    // rep of +inf: the largest non-NaN code
    __host__ __device__ static constexpr uint64_t sentinel() { return 0xFFF0000000000000ULL; }
};

// "no payload" marker type for key-only instantiations
struct NoVal {};
template <typename V>
struct HasVal { static constexpr bool value = true; };
template <>
struct HasVal<NoVal> { static constexpr bool value = false; };

// ---------------------------------------------------------------- memory
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// streaming (read-once) loads: keep L1 clean, evict-first in L2
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }

// ---------------------------------------------------------------- scans
// Inclusive warp scan of a 32-bit value.
__device__ __forceinline__ unsigned warp_incl_scan(unsigned v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned t = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

// Exclusive block scan of one 32-bit value per thread.  `smem` needs
// NWARPS+1 words.  Returns the exclusive prefix; *total receives the sum.
template <int NTHREADS>
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* smem, unsigned* total) {
    constexpr int NW = NTHREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned inc = warp_incl_scan(v);
    if (lane == 31) smem[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned w = lane < NW ? smem[lane] : 0u;
        unsigned wi = warp_incl_scan(w);
        if (lane < NW) smem[lane] = wi - w;
        if (lane == NW - 1) smem[NW] = wi;
    }
    __syncthreads();
    unsigned r = smem[warp] + inc - v;
    *total = smem[NW];
    __syncthreads();
    return r;
}

// ------------------------------------------------ shared-memory counters
// Shared-memory atomics whose result is unused compile to ATOMS.POPC.INC,
// which merges the lanes of a warp that hit one counter.  RANKING atomics
// (result used) serialise instead when a warp's lanes share a bucket (sorted,
// reverse or few-unique inputs); warp_rank_add takes the warp's active lanes
// and, when they all carry one bucket, lets the first lane reserve for all.
// Ranks inside a bucket are then a permutation of the per-lane ones (the
// order of keys inside a bucket is never observable: later passes sort it).
__device__ __forceinline__ unsigned warp_rank_add(unsigned* cnt, unsigned b) {
    const unsigned am = __activemask();
    const int first = __ffs(am) - 1;
    const unsigned b0 = __shfl_sync(am, b, first);
    if (__all_sync(am, b == b0)) {
        const unsigned lane = threadIdx.x & 31;
        unsigned base = 0;
        if ((int)lane == first) base = atomicAdd(&cnt[b0], (unsigned)__popc(am));
        return __shfl_sync(am, base, first) + __popc(am & ((1u << lane) - 1u));
    }
    return atomicAdd(&cnt[b], 1u);
}

// src[0, n) -> dst[0, n) by the whole CTA of NT threads: 16-byte vectors over
// the body when both share a 16-byte phase (true for the same offset into two
// equally aligned buffers), element copies otherwise.
template <typename T, unsigned NT>
__device__ __forceinline__ void cta_copy(const T* __restrict__ src, T* __restrict__ dst, unsigned n) {
    constexpr unsigned VE = 16 / sizeof(T);
    if (((reinterpret_cast<uintptr_t>(src) ^ reinterpret_cast<uintptr_t>(dst)) & 15) != 0) {
        for (unsigned i = threadIdx.x; i < n; i += NT) dst[i] = src[i];
        return;
    }
    const unsigned head = min(n, (unsigned)(((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) / sizeof(T)));
    const unsigned nv = (n - head) / VE;
    if (threadIdx.x < head) dst[threadIdx.x] = src[threadIdx.x];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    // four loads in flight per thread before the first store (a 512-thread CTA
    // then keeps 32 KB on the way, enough to cover HBM latency at two CTAs per SM)
    unsigned j = threadIdx.x;
    for (; j + 3 * NT < nv; j += 4 * NT) {
        const uint4 a = __ldcs(s4 + j), b = __ldcs(s4 + j + NT), c = __ldcs(s4 + j + 2 * NT),
                    e = __ldcs(s4 + j + 3 * NT);
        d4[j] = a;
        d4[j + NT] = b;
        d4[j + 2 * NT] = c;
        d4[j + 3 * NT] = e;
    }
    for (; j < nv; j += NT) d4[j] = __ldcs(s4 + j);
    const unsigned t0 = head + nv * VE;
    if (t0 + threadIdx.x < n) dst[t0 + threadIdx.x] = src[t0 + threadIdx.x];
}

// 64-bit hash (splitmix64 finaliser) for deterministic sample positions.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint32_t next_pow2_u32(uint32_t v) {
    uint32_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace vx
