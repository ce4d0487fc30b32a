// partition2.cuh -- single-pass pivot partition (north-star subsystem 1).
//
// Replaces the reference's in-place two-cursor vector partition
// (_kernels.py:187-262, partition.py:115-175, keyvalue.py:138-225) on the
// GPU.  Semantics kept: `x <= pivot` goes left (SPEC.md:280-282,
// _kernels.py:194), the returned boundary is count(x <= pivot), the element
// (and pair) multiset is preserved.  The reference's *layout* is a CPU
// artefact (which pack was loaded when) and is not reproduced; parity is on
// the boundary, the two side predicates and the multisets.
//
// B200 design, one HBM read + one HBM write per element:
//  * small tiles (128 threads x 16 elements) so ~10 CTAs share an SM and
//    one tile's loads overlap another's staging and stores;
//  * 128-bit vector loads (int4 / double2) striped across the CTA;
//  * classify + rank lows AND valid elements with ONE packed 16|16-bit
//    block scan (warp shuffles, then warp totals);
//  * tile offsets from two run cursors (the reference's left_w / right_w
//    cursors, _kernels.py:197-212, at tile granularity): one atomic reserves
//    the tile's lows at the left end, one its highs from the right end, so no
//    tile ever waits on another; the cursors sit on separate L2 lines.  The
//    order of the runs inside each side follows reservation order (sides,
//    split and multisets are fixed; the layout was never the reference's);
//  * build option VX_PART_LOOKBACK: deterministic tile-ordered layout via a
//    decoupled look-back on the low count (64-bit {status:2 | inclusive:62}
//    descriptors, st.release / ld.acquire, 32 predecessors per warp step,
//    dynamic tile ids; highs at H_excl(t) = t*T - L_excl(t)) -- 1.8x slower
//    on B200 because its per-tile latency needs big tiles, i.e. one CTA/SM;
//  * the tile is staged in shared memory as [lows | highs] and written as two
//    contiguous runs with consecutive threads -> coalesced stores.
#pragma once

#include "common.cuh"

namespace vx {

constexpr unsigned long long kStAgg = 1ull << 62;
constexpr unsigned long long kStPrefix = 2ull << 62;
constexpr unsigned long long kStMask = 3ull << 62;
constexpr unsigned long long kValMask = ~kStMask;

template <typename K>
struct Vec16;
template <>
struct Vec16<int32_t> {
    using T = int4;
    static constexpr int W = 4;
    __device__ __forceinline__ static void unpack(const T& v, int32_t* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct Vec16<double> {
    using T = double2;
    static constexpr int W = 2;
    __device__ __forceinline__ static void unpack(const T& v, double* o) { o[0] = v.x; o[1] = v.y; }
};
template <>
struct Vec16<uint32_t> {
    using T = uint4;
    static constexpr int W = 4;
    __device__ __forceinline__ static void unpack(const T& v, uint32_t* o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
};
template <>
struct Vec16<uint64_t> {
    using T = ulonglong2;
    static constexpr int W = 2;
    __device__ __forceinline__ static void unpack(const T& v, uint64_t* o) { o[0] = v.x; o[1] = v.y; }
};

// Decoupled look-back over 64-bit tile descriptors, run by one full warp.
// Publishes this tile's aggregate first, returns the exclusive prefix and
// publishes the inclusive prefix.
__device__ __forceinline__ unsigned long long lookback_excl(unsigned long long* state, uint64_t tile,
                                                            unsigned long long agg) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_release_u64(&state[0], kStPrefix | agg);
        return 0;
    }
    if (lane == 0) st_release_u64(&state[tile], kStAgg | agg);
    unsigned long long excl = 0;
    long long pred = (long long)tile - 1;
    while (true) {
        const long long idx = pred - lane;
        unsigned long long s = kStPrefix;  // virtual predecessor of tile 0
        if (idx >= 0) {
            do {
                s = ld_acquire_u64(&state[idx]);
            } while ((s & kStMask) == 0);
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, (s & kStMask) == kStPrefix);
        unsigned long long v = s & kValMask;
        if (pmask) {
            const int first = __ffs(pmask) - 1;  // nearest predecessor holding a prefix
            if (lane > first) v = 0;
        }
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        excl += v;
        if (pmask) break;
        pred -= 32;
    }
    if (lane == 0) st_release_u64(&state[tile], kStPrefix | (excl + agg));
    return excl;
}

// kin/vin -> kout/vout; n elements; `state` holds ntiles zeroed descriptors,
// `counter` a zeroed tile ticket; *d_split receives count(x <= pivot).
template <typename K, typename V, int NT, int IPT, bool VEC>
__global__ void __launch_bounds__(NT) partition2_kernel(const K* __restrict__ kin, const V* __restrict__ vin,
                                                        K* __restrict__ kout, V* __restrict__ vout, uint64_t n,
                                                        K pivot, unsigned long long* __restrict__ state,
                                                        unsigned* __restrict__ counter,
                                                        unsigned long long* __restrict__ d_split) {
    constexpr bool KV = HasVal<V>::value;
    constexpr int T = NT * IPT;
    constexpr int W = Vec16<K>::W;
    static_assert(IPT % W == 0 && IPT <= 32, "IPT");
    static_assert(T < 65536, "packed 16-bit scan");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* sk = reinterpret_cast<K*>(smem_raw);
    V* sv = reinterpret_cast<V*>(smem_raw + sizeof(K) * T);
    __shared__ unsigned s_scan[NT / 32 + 1];
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_excl;

    const int tid = threadIdx.x;
#ifdef VX_PART_LOOKBACK
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
#else
    (void)s_tile;
    const uint64_t tile = blockIdx.x;  // no tile waits on another: launch order is enough
#endif
    const uint64_t base = tile * (uint64_t)T;
    const uint64_t ntiles = (n + T - 1) / T;
    const unsigned tn = (unsigned)min((uint64_t)T, n - base);

    // striped mapping: item i of thread tid sits at tile position
    //   ((i / W) * NT + tid) * W + (i % W)
    K k[IPT];
    V v[IPT];
    unsigned valid = 0;
    if (VEC && tn == T) {
        using VT = typename Vec16<K>::T;
        const VT* p = reinterpret_cast<const VT*>(kin + base);
#pragma unroll
        for (int j = 0; j < IPT / W; ++j) Vec16<K>::unpack(ld_stream(p + j * NT + tid), &k[j * W]);
        if constexpr (KV) {
            using VV = typename Vec16<V>::T;
            constexpr int WV = Vec16<V>::W;
            static_assert(WV == W, "value width must equal key width");
            const VV* q = reinterpret_cast<const VV*>(vin + base);
#pragma unroll
            for (int j = 0; j < IPT / W; ++j) Vec16<V>::unpack(ld_stream(q + j * NT + tid), &v[j * W]);
        }
        valid = IPT == 32 ? 0xffffffffu : ((1u << IPT) - 1u);
    } else {
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const unsigned pos = ((i / W) * NT + tid) * W + (i % W);
            if (pos < tn) {
                k[i] = kin[base + pos];
                if constexpr (KV) v[i] = vin[base + pos];
                valid |= 1u << i;
            }
        }
    }

    // classify: x <= pivot goes left (ordered compare: NaN is "high")
    unsigned lowmask = 0;
#pragma unroll
    for (int i = 0; i < IPT; ++i)
        if (((valid >> i) & 1u) && (k[i] <= pivot)) lowmask |= 1u << i;
    const unsigned nlow = __popc(lowmask), nval = __popc(valid);

    unsigned total;
    const unsigned packed = block_excl_scan<NT>(nlow | (nval << 16), s_scan, &total);
    const unsigned L_t = total & 0xffffu, N_t = total >> 16, H_t = N_t - L_t;
    unsigned rl = packed & 0xffffu;
    unsigned rh = L_t + ((packed >> 16) - rl);

#ifndef VX_PART_LOOKBACK
    // run cursors instead of the look-back: each tile reserves its lows at
    // the left cursor and its highs at the right cursor (layout order then
    // follows reservation order, not tile order)
    __shared__ unsigned long long s_hexcl;
    unsigned long long* cur = reinterpret_cast<unsigned long long*>(counter);  // lo, hi, done: one L2 line each
    if (tid == 0) s_excl = atomicAdd(&cur[0], (unsigned long long)L_t);
    if (tid == 32) s_hexcl = atomicAdd(&cur[16], (unsigned long long)H_t);
#else
    if (tid < 32) {
        const unsigned long long ex = lookback_excl(state, tile, L_t);
        if (tid == 0) s_excl = ex;
    }
#endif

    // stage [lows | highs] in shared memory
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        if ((valid >> i) & 1u) {
            const unsigned slot = ((lowmask >> i) & 1u) ? rl++ : rh++;
            sk[slot] = k[i];
            if constexpr (KV) sv[slot] = v[i];
        }
    }
    __syncthreads();

    const uint64_t L_excl = s_excl;
#ifndef VX_PART_LOOKBACK
    const uint64_t H_excl = s_hexcl;
#else
    const uint64_t H_excl = base - L_excl;  // every preceding tile is full
#endif
    const uint64_t hi_base = n - H_excl - H_t;
    for (unsigned j = tid; j < N_t; j += NT) {
        const uint64_t dst = j < L_t ? L_excl + j : hi_base + (j - L_t);
        VX_ASSERT(dst < n);
        kout[dst] = sk[j];
        if constexpr (KV) vout[dst] = sv[j];
    }
#ifndef VX_PART_LOOKBACK
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(reinterpret_cast<unsigned*>(&cur[32]), 1u) == (unsigned)(ntiles - 1)) {
            __threadfence();
            *d_split = atomicAdd(&cur[0], 0ull);
        }
    }
#else
    if (tile == ntiles - 1 && tid == 0) *d_split = L_excl + L_t;
#endif
}

}  // namespace vx
