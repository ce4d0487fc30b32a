// finish.cuh -- CTA-local hybrid quicksort of one small range (<= CAP
// elements) and the finish queue kernel.
//
// This is the bottom of the reference's recursion (_kernels.py:396-423): a
// range small enough for one SM is partitioned once more around sampled
// pivots and every resulting range <= the leaf bound is sorted by the
// bitonic network (_kernels.py:30-58, 97-113).  B200 shape, one HBM read and
// one HBM write per element:
//   * the range is loaded straight into registers (coalesced, striped);
//   * one warp sorts a <= 512-element sample in registers (warp bitonic) and
//     the CTA picks up to 63 distinct pivots -> 2m+1 buckets (ranges and
//     equal-to-pivot buckets, the latter already final);
//   * each element is classified once (branch-free search in smem), ranked
//     with a shared-memory atomic, and written bucket-major into a padded
//     smem buffer (one pad word per 32 makes blocked warp reads conflict-free);
//   * warps sort the range buckets IN shared memory with the register
//     bitonic network; for 8-byte keys and pairs (where the network
//     dominates) many small buckets are cut and adjacent ones packed
//     greedily into runs of <= 128 slots, so every network runs nearly
//     full; buckets above the leaf bound are written out as they are and
//     re-queued for another finish round (the reference's "partition again"
//     branch);
//   * the whole range, now sorted, leaves with one coalesced store.
#pragma once

#include "bitonic.cuh"
#include "common.cuh"
#include "qsort.cuh"

namespace vx {

constexpr int kFinMaxSplit = 255;
constexpr int kFinMaxBkt = 2 * kFinMaxSplit + 1;
#ifndef VX_FIN_LUT_BITS
#define VX_FIN_LUT_BITS 10
#endif
#ifndef VX_FIN_GROUP
#define VX_FIN_GROUP 128
#endif
constexpr int kFinLutBits = VX_FIN_LUT_BITS;
constexpr unsigned kFinGroup = VX_FIN_GROUP;  // adjacent buckets are sorted together up to this many slots
constexpr int kFinMaxSample = 512;
constexpr unsigned kWarpSortMax = 256;

__device__ __forceinline__ unsigned pad32(unsigned i) { return i + (i >> 5); }
__device__ __forceinline__ unsigned wmax_of(unsigned leaf) { return leaf < kWarpSortMax ? leaf : kWarpSortMax; }

template <typename K, typename V>
struct FinSmem {
    static constexpr uint32_t CAP = FinCap<K, V>::value;
    static constexpr uint32_t PCAP = CAP + CAP / 32;
    using VS = typename std::conditional<HasVal<V>::value, V, char>::type;
    K b[PCAP];
    VS bv[HasVal<V>::value ? PCAP : 1];
    using U = typename OKey<K>::U;  // samples and pivots as order-preserving codes
    U samp[kFinMaxSample];
    U samp2[kFinMaxSample];
    CellTableT<U, kFinMaxSplit + 1, kFinLutBits> ct;  // pivots + 1024-cell lookup table
    unsigned next_bucket, next_big, ngrp;
    unsigned cnt[kFinMaxBkt + 1];
    unsigned loc[kFinMaxBkt + 2];
    unsigned short nxt[kFinMaxBkt + 1];  // greedy group successor of each bucket
    unsigned short grp[kFinMaxBkt + 2];  // group boundaries (bucket ids)
    unsigned scan[kFinNT / 32 + 1];
    U rmin[kFinNT / 32], rmax[kFinNT / 32];  // per-warp key-code range
};

template <typename U>
__device__ __forceinline__ U warp_min_u(U v) {
    if constexpr (sizeof(U) == 4) {
        return __reduce_min_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const U o = __shfl_xor_sync(0xffffffffu, v, d);
            v = o < v ? o : v;
        }
        return v;
    }
}
template <typename U>
__device__ __forceinline__ U warp_max_u(U v) {
    if constexpr (sizeof(U) == 4) {
        return __reduce_max_sync(0xffffffffu, v);
    } else {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const U o = __shfl_xor_sync(0xffffffffu, v, d);
            v = o > v ? o : v;
        }
        return v;
    }
}

// Sort P = 32*E padded-smem slots b[pad32(lo + q)], q < c, in place with one
// warp (blocked layout, sentinel padding by count).
template <typename K, typename V, int E>
__device__ __forceinline__ void warp_sort_smem_e(K* b, V* bv, unsigned lo, unsigned c) {
    constexpr bool KV = HasVal<V>::value;
    using R = KeyRep<K>;
    using I = typename R::I;
    const unsigned lane = threadIdx.x & 31;
    I k[E];
    V v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const unsigned q = lane * E + r;
        k[r] = q < c ? R::to(b[pad32(lo + q)]) : KeyTraits<I>::sentinel();
        if constexpr (KV) v[r] = q < c ? bv[pad32(lo + q)] : V();
    }
    WarpBitonic<I, V, E>::sort(k, v);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const unsigned q = lane * E + r;
        if (q < c) {
            b[pad32(lo + q)] = R::from(k[r]);
            if constexpr (KV) bv[pad32(lo + q)] = v[r];
        }
    }
    __syncwarp();
}

// Lane-group variant: every group of G lanes sorts its own run b[pad32(lo +
// q)], q < c <= G*E (lo, c uniform within the group; c = 0 sorts padding
// only and writes nothing).
template <typename K, typename V, int E, int G>
__device__ __forceinline__ void group_sort_smem(K* b, V* bv, unsigned lo, unsigned c) {
    constexpr bool KV = HasVal<V>::value;
    using R = KeyRep<K>;
    using I = typename R::I;
    const unsigned gl = threadIdx.x & (G - 1);
    I k[E];
    V v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const unsigned q = gl * E + r;
        k[r] = q < c ? R::to(b[pad32(lo + q)]) : KeyTraits<I>::sentinel();
        if constexpr (KV) v[r] = q < c ? bv[pad32(lo + q)] : V();
    }
    WarpBitonic<I, V, E, G>::sort(k, v);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const unsigned q = gl * E + r;
        if (q < c) {
            b[pad32(lo + q)] = R::from(k[r]);
            if constexpr (KV) bv[pad32(lo + q)] = v[r];
        }
    }
    __syncwarp();
}

// Group shape of the finish networks: 128 slots per group of G lanes -- 16
// lanes x 8 registers for 8-byte keys and pairs; 4-byte keys use whole-warp
// networks (G = 32: measured faster on B200 than 8 x 16 or 16 x 8 groups).
template <typename K, typename V>
struct FinGroupShape {
    static constexpr int BYTES = sizeof(K) + (HasVal<V>::value ? sizeof(V) : 0);
#ifndef VX_FIN_GLANES4
#define VX_FIN_GLANES4 32
#endif
#ifndef VX_FIN_GLANES8
#define VX_FIN_GLANES8 16
#endif
    static constexpr int G = BYTES <= 4 ? VX_FIN_GLANES4 : VX_FIN_GLANES8;
    static constexpr int E = 128 / G;
    static constexpr unsigned P = 128;
};

template <typename K, typename V>
__device__ __forceinline__ void warp_sort_smem(K* b, V* bv, unsigned lo, unsigned c) {
    if (c <= 32) warp_sort_smem_e<K, V, 1>(b, bv, lo, c);
    else if (c <= 64) warp_sort_smem_e<K, V, 2>(b, bv, lo, c);
    else if (c <= 128) warp_sort_smem_e<K, V, 4>(b, bv, lo, c);
    else warp_sort_smem_e<K, V, 8>(b, bv, lo, c);
    // callers never pass c > kWarpSortMax (256)
}

// sort the S (pow2, 32..512) samples of smem `s` ascending with one warp
template <typename K>
__device__ __forceinline__ void warp_sort_samples(K* s, unsigned S) {
    // samples live unpadded: reuse the padded helper on a tiny view is not
    // needed -- read blocked directly (S <= 512, a few bank conflicts)
    const unsigned lane = threadIdx.x & 31;
    auto run = [&](auto e_tag) {
        constexpr int E = decltype(e_tag)::value;
        K k[E];
        NoVal v[E];
#pragma unroll
        for (int r = 0; r < E; ++r) k[r] = s[lane * E + r];
        WarpBitonic<K, NoVal, E>::sort(k, v);
#pragma unroll
        for (int r = 0; r < E; ++r) s[lane * E + r] = k[r];
    };
    switch (S) {
        case 32: run(std::integral_constant<int, 1>{}); break;
        case 64: run(std::integral_constant<int, 2>{}); break;
        default: run(std::integral_constant<int, 4>{}); break;  // 128-sample chunks
    }
    __syncwarp();
}

template <typename K, typename V>
__device__ void fin_local(FinSmem<K, V>& sm, const K* __restrict__ src_k, const V* __restrict__ src_v,
                          K* __restrict__ dst_k, V* __restrict__ dst_v, uint64_t start, unsigned len, uint64_t seed,
                          unsigned leaf, Ctl* ctl, Ctl* ctl_next, Fin* fins_next, unsigned cap_fin) {
    constexpr bool KV = HasVal<V>::value;
    constexpr unsigned CAP = FinSmem<K, V>::CAP;
    constexpr int IPT = CAP / kFinNT;
    using U = typename OKey<K>::U;
    const unsigned tid = threadIdx.x, lane = tid & 31;

    // 1. stratified sample read straight from global, sorted by warp 0
    // mean fine-bucket size: small buckets packed into full networks pay off
    // when the network dominates (8-byte keys, pairs); for 4-byte keys the
    // extra pivots cost more than the padding they save
#ifndef VX_FIN_TARGET4
#define VX_FIN_TARGET4 112
#endif
#ifndef VX_FIN_TARGET8
#define VX_FIN_TARGET8 40
#endif
    constexpr bool kGroup = (sizeof(K) + (KV ? sizeof(V) : 0)) > 4;
    constexpr unsigned kTarget = kGroup ? VX_FIN_TARGET8 : VX_FIN_TARGET4;
    constexpr unsigned kSampleX = kGroup ? 3 : 6;  // samples per pivot (grouping tolerates uneven buckets)
    const unsigned target = max(2u, min(kTarget, leaf * 7 / 16));
    const unsigned mt = max(1u, min((unsigned)kFinMaxSplit, len / target));
    const unsigned S = max(32u, min((unsigned)kFinMaxSample, 2u << (31 - __clz(kSampleX * (mt + 1) - 1))));  // pow2 >= x(mt+1)
    // the range into registers first, striped and coalesced
    K x[IPT];
    V y[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const unsigned p = j * kFinNT + tid;
        if (p < len) {
            x[j] = ld_stream(src_k + start + p);
            if constexpr (KV) y[j] = ld_stream(src_v + start + p);
        }
    }
    // 2. interpolation buckets: nbl equal-width key-code intervals over the
    //    range's own [min, max] -- evenly spaced pivots, no sample.  Taken
    //    whenever every bucket fits one warp network; otherwise (skewed or
    //    clustered keys) the sampled pivots below decide.
    bool linear = false;
    unsigned nb = 0, m = 0;
    unsigned br[IPT];
#ifndef VX_FIN_LTARGET4
#define VX_FIN_LTARGET4 120
#endif
#ifndef VX_FIN_LTARGET8
#define VX_FIN_LTARGET8 40
#endif
    {
        constexpr unsigned kLTarget = kGroup ? VX_FIN_LTARGET8 : VX_FIN_LTARGET4;
        U lo = ~(U)0, hi = 0;
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (j * kFinNT + tid < len) {
                const U u = OKey<K>::of(x[j]);
                lo = u < lo ? u : lo;
                hi = u > hi ? u : hi;
            }
        }
        lo = warp_min_u(lo);
        hi = warp_max_u(hi);
        if (lane == 0) {
            sm.rmin[tid >> 5] = lo;
            sm.rmax[tid >> 5] = hi;
        }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kFinNT / 32; ++w) {
            lo = sm.rmin[w] < lo ? sm.rmin[w] : lo;
            hi = sm.rmax[w] > hi ? sm.rmax[w] : hi;
        }
        if (lo == hi) {  // every key equal: the range is sorted as it stands
            if (src_k != dst_k) {
#pragma unroll
                for (int j = 0; j < IPT; ++j) {
                    const unsigned p = j * kFinNT + tid;
                    if (p < len) {
                        dst_k[start + p] = x[j];
                        if constexpr (KV) dst_v[start + p] = y[j];
                    }
                }
            }
            __syncthreads();
            return;
        }
        const unsigned ltarget = max(2u, min(kLTarget, leaf * 7 / 16));
        unsigned nbl = min((unsigned)kFinMaxBkt, max(1u, (len + ltarget - 1) / ltarget));
        const U range = hi - lo;
        const unsigned bits = (unsigned)(8 * sizeof(U)) -
                              (sizeof(U) == 8 ? (unsigned)__clzll((long long)range) : (unsigned)__clz((int)range));
        const unsigned sh = bits > 32 ? bits - 32 : 0u;
        const uint32_t r32 = (uint32_t)(range >> sh);
        // bucket = floor(d * nbl / (r32 + 1)) as a high multiply; a range
        // narrower than nbl gets one bucket per value
        uint32_t mul;
        if ((uint64_t)r32 + 1 <= nbl) {
            nbl = r32 + 1;
            mul = 0;
        } else {
            mul = (uint32_t)(((uint64_t)nbl << 32) / ((uint64_t)r32 + 1));
        }
        if (tid < nbl) sm.cnt[tid] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            if (j * kFinNT + tid < len) {
                const uint32_t d = (uint32_t)((OKey<K>::of(x[j]) - lo) >> sh);
                const unsigned b = mul ? __umulhi(d, mul) : d;
                br[j] = (b << 16) | atomicAdd(&sm.cnt[b], 1u);
            }
        }
        __syncthreads();
        const bool over = __syncthreads_or(tid < nbl && sm.cnt[tid] > wmax_of(leaf));
        if (!over) {
            linear = true;
            nb = nbl;
        }
    }
    if (!linear) {
    if (tid < S) {
        const uint64_t h = mix64(seed ^ (start * 0x2545F4914F6CDD1DULL + tid));
        if (len >= 2 * kFinNT) {
            // sample from registers: column tid, a hashed row -> no extra reads
            const unsigned rows = (len + kFinNT - 1) / kFinNT;
            unsigned r = (unsigned)(h % rows);
            if (r * kFinNT + tid >= len) --r;
            K v = x[0];
#pragma unroll
            for (int j = 1; j < IPT; ++j)
                if ((unsigned)j == r) v = x[j];
            sm.samp[tid] = OKey<K>::of(v);
        } else {
            const unsigned stride = max(1u, len / S);
            const unsigned q = min(len - 1, (unsigned)(((uint64_t)tid * len) / S) + (unsigned)(h % stride));
            sm.samp[tid] = OKey<K>::of(src_k[start + q]);
        }
    }
    __syncthreads();
    // up to 4 warps sort 128-sample chunks in registers, then the chunks are
    // merged by rank (position = own index + ranks in the other chunks)
    const unsigned C = min(S, 128u), W = S / C;
    if ((tid >> 5) < W) warp_sort_samples<U>(sm.samp + (tid >> 5) * C, C);
    __syncthreads();
    if (W > 1) {
        if (tid < S) {
            const U v = sm.samp[tid];
            const unsigned c = tid / C;
            unsigned pos = tid % C;
            for (unsigned o = 0; o < W; ++o) {
                if (o == c) continue;
                const U* ch = sm.samp + o * C;
                unsigned lo = 0, hi = C;  // o < c: count(<= v); o > c: count(< v)
                while (lo < hi) {
                    const unsigned mid = (lo + hi) >> 1;
                    const bool before = o < c ? !(v < ch[mid]) : (ch[mid] < v);
                    if (before) lo = mid + 1; else hi = mid;
                }
                pos += lo;
            }
            sm.samp2[pos] = v;
        }
        __syncthreads();
    }
    const U* samp = W > 1 ? sm.samp2 : sm.samp;
    // 3. distinct pivots
    U cand = U();
    unsigned keep = 0;
    if (tid < mt) {
        const unsigned q = (unsigned)(((uint64_t)(tid + 1) * S) / (mt + 1));
        cand = samp[q];
        keep = tid == 0 ? 1u : (samp[(unsigned)(((uint64_t)tid * S) / (mt + 1))] < cand ? 1u : 0u);
    }
    const unsigned rank = block_excl_scan<kFinNT>(keep, sm.scan, &m);
    nb = 2 * m + 1;
    if (keep) sm.ct.spl[rank] = cand;
    if (tid < nb) sm.cnt[tid] = 0;
    __syncthreads();
    const CellParams<U> cp = ct_build<kFinNT, false>(sm.ct, m, sm.scan);  // code map (narrow ranges); ends with a barrier
    // 4. classify once, rank with smem atomics (bucket << 16 | rank)
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const unsigned p = j * kFinNT + tid;
        if (p < len) {
            const unsigned b = ct_classify(sm.ct, cp, x[j]);
            br[j] = (b << 16) | atomicAdd(&sm.cnt[b], 1u);
        }
    }
    }  // sampled pivots
    if (tid == 0) {
        sm.next_bucket = 0;
        sm.next_big = 0;
        sm.grp[0] = 0;
    }
    __syncthreads();
    {
        unsigned tot;
        const unsigned c = tid < nb ? sm.cnt[tid] : 0u;
        const unsigned ex = block_excl_scan<kFinNT>(c, sm.scan, &tot);
        if (tid < nb) sm.loc[tid] = ex;
        if (tid == 0) sm.loc[nb] = len;
    }
    __syncthreads();
    // 5. bucket-major into the padded smem buffer
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        const unsigned p = j * kFinNT + tid;
        if (p < len) {
            const unsigned slot = pad32(sm.loc[br[j] >> 16] + (br[j] & 0xffffu));
            sm.b[slot] = x[j];
            if constexpr (KV) sm.bv[slot] = y[j];
        }
    }
    __syncthreads();
    // 6. group adjacent buckets greedily into runs of <= G slots (fine
    //    buckets from many pivots, packed so every warp network runs nearly
    //    full); a bucket alone above G is sorted with a wider network, or --
    //    above the leaf bound -- re-queued (written out unsorted below);
    //    an equal-to-pivot bucket alone is final.
    const unsigned wmax = min(leaf, kWarpSortMax);
    unsigned ngrp = linear ? nb : m + 1;  // without grouping: the range buckets, one by one
    if constexpr (kGroup) {
        const unsigned G = min(wmax, kFinGroup);
        for (unsigned s = tid; s < nb; s += kFinNT) {
            // last e in [s+1, nb] with loc[e] - loc[s] <= G (loc is nondecreasing)
            const unsigned lim = sm.loc[s] + G;
            unsigned lo = s + 1, hi = nb + 1;
            while (lo < hi) {
                const unsigned mid = (lo + hi) >> 1;
                if (sm.loc[mid] <= lim) lo = mid + 1; else hi = mid;
            }
            sm.nxt[s] = (unsigned short)max(lo - 1, s + 1);
        }
        __syncthreads();
        if (tid == 0) {  // the greedy walk itself is serial (one short chain)
            unsigned s = 0, g = 0;
            while (s < nb) {
                s = sm.nxt[s];
                sm.grp[++g] = (unsigned short)s;
            }
            sm.ngrp = g;
        }
        __syncthreads();
        ngrp = sm.ngrp;
    }
    // 7a. runs of <= 128 slots: lane groups, 32/G runs per warp at a time
    //     (measured: 16-lane groups win for 8-byte keys and pairs; 4-byte
    //     keys keep one run per warp, 7b only)
    using GS = FinGroupShape<K, V>;
    constexpr unsigned NGW = 32 / GS::G;
    const unsigned gmax = GS::G == 32 ? 0u : min(wmax, GS::P);
    if constexpr (GS::G < 32) for (;;) {
        unsigned j0 = 0;
        if (lane == 0) j0 = atomicAdd(&sm.next_bucket, NGW);
        j0 = __shfl_sync(0xffffffffu, j0, 0);
        if (j0 >= ngrp) break;
        const unsigned j = j0 + lane / GS::G;
        unsigned lo = 0, c = 0;
        if (j < ngrp) {
            const unsigned s = kGroup ? sm.grp[j] : (linear ? j : 2 * j), e = kGroup ? sm.grp[j + 1] : s + 1;
            lo = sm.loc[s];
            c = sm.loc[e] - lo;
            if (c < 2 || c > gmax || (!linear && e == s + 1 && (s & 1u))) c = 0;  // none, too big, or final
        }
        if constexpr (KV) group_sort_smem<K, V, GS::E, GS::G>(sm.b, sm.bv, lo, c);
        else group_sort_smem<K, V, GS::E, GS::G>(sm.b, (V*)nullptr, lo, c);
    }
    // 7b. the rest (128 < c <= leaf bound) with whole-warp networks; above
    //     the leaf bound re-queued
    for (;;) {
        unsigned j = 0;
        if (lane == 0) j = atomicAdd(&sm.next_big, 1u);
        j = __shfl_sync(0xffffffffu, j, 0);
        if (j >= ngrp) break;
        const unsigned s = kGroup ? sm.grp[j] : (linear ? j : 2 * j), e = kGroup ? sm.grp[j + 1] : s + 1;
        const unsigned lo = sm.loc[s], c = sm.loc[e] - lo;
        if (c <= gmax || (!linear && e == s + 1 && (s & 1u))) continue;  // done above, or one equal-to-pivot bucket
        if (c <= wmax) {
            if constexpr (KV) warp_sort_smem<K, V>(sm.b, sm.bv, lo, c);
            else warp_sort_smem<K, V>(sm.b, (V*)nullptr, lo, c);
        } else if (lane == 0) {
            const unsigned f = atomicAdd(&ctl_next->fin_ctr, 1u);
            if (f < cap_fin) {
                fins_next[f].start = start + lo;
                fins_next[f].len = c;
                fins_next[f].flags = 0u;  // next round sorts it in place in `data`
            } else {
                atomicOr(&ctl->err, kErrCapacity);
            }
        }
    }
    __syncthreads();
    // 7. one coalesced store of the whole range
    for (unsigned i = tid; i < len; i += kFinNT) {
        dst_k[start + i] = sm.b[pad32(i)];
        if constexpr (KV) dst_v[start + i] = sm.bv[pad32(i)];
    }
    __syncthreads();
}

// One CTA per finish item (grid-stride).  Items: copy (flags bit1), direct
// warp bitonic (len <= leaf), or the CTA-local sort above.  Source is the
// scratch buffer when flags bit0 is set, else `data` (in place).
template <typename K, typename V>
__global__ void __launch_bounds__(kFinNT, 2) qs_finish_kernel(const Fin* __restrict__ fins, Ctl* __restrict__ ctl,
                                                           Ctl* __restrict__ ctl_next, Fin* __restrict__ fins_next,
                                                           unsigned cap_fin, K* __restrict__ data_k,
                                                           V* __restrict__ data_v, const K* __restrict__ scr_k,
                                                           const V* __restrict__ scr_v, uint64_t sort_seed,
                                                           const Ctl* __restrict__ tot, unsigned leaf) {
    constexpr bool KV = HasVal<V>::value;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FinSmem<K, V>& sm = *reinterpret_cast<FinSmem<K, V>*>(smem_raw);
    const unsigned nf = ctl->fin_ctr;
    const unsigned wmax = min(leaf, kWarpSortMax);
    const uint64_t seed = level_seed(sort_seed, tot);
    for (unsigned d = blockIdx.x; d < nf; d += gridDim.x) {
        const Fin f = fins[d];
        if (threadIdx.x == 0) atomicAdd(&ctl->fin_elems, (unsigned long long)f.len);
        const K* sk = (f.flags & 1u) ? scr_k : data_k;
        const V* sv = (f.flags & 1u) ? scr_v : data_v;
        if (f.flags & 2u) {
            cta_copy<K, kFinNT>(sk + f.start, data_k + f.start, f.len);
            if constexpr (KV) cta_copy<V, kFinNT>(sv + f.start, data_v + f.start, f.len);
        } else if (f.len <= min(wmax, 256u)) {
            if (threadIdx.x < 32) warp_sort_any2<K, V>(sk + f.start, sv ? sv + f.start : nullptr, data_k + f.start,
                                                       data_v ? data_v + f.start : nullptr, f.len);
        } else {
            fin_local<K, V>(sm, sk, sv, data_k, data_v, f.start, f.len, seed, leaf, ctl, ctl_next, fins_next,
                            cap_fin);
        }
    }
}

}  // namespace vx
