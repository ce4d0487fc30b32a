// local3.cuh -- CTA-local last partition level, one LANE per leaf bucket
// (north-star subsystems 2 + 3: the bottom of _kernels.quicksort,
// _kernels.py:396-423, and its bitonic small sort, _kernels.py:30-58).
//
// One CTA owns a leaf (~150 KB of keys) from partition to sorted output and
// builds the sorted leaf as an IMAGE in shared memory:
//   1. key-code range (the parent's pivots, or one pass for outer buckets);
//   2. count pass (the HBM read) into interpolation buckets of <= ~10 keys --
//      a whole number of rounds of kQlNT buckets, so no lane idles through a
//      partial last round; a bucket above 256 keys means skewed keys and
//      sends the leaf back to a sampled level;
//   3. one scan packs (image position << 16 | count) per bucket; the image
//      is UNPADDED -- bucket b sits exactly where it lands in the sorted
//      leaf -- so leaving it is one flat, coalesced copy.  Leaves larger
//      than the stage are cut into G groups of buckets (G = 1 as planned);
//   4. per group: a pass over the leaf (L2) drops every key at its bucket's
//      cursor in the image; then every lane sorts ONE bucket with the bitonic
//      network entirely in its registers: it loads the LE slots that start
//      at its bucket -- the slots past the bucket's end hold keys of LATER
//      buckets, all larger, so they are the network's sentinel padding for
//      free -- and stores back the bucket's own count.  No shuffles, no
//      padding tests, no bank conflicts by construction (mean bucket ~9.7
//      slots: an odd stride across the lanes; the load order is rotated by
//      the lane).  Buckets above LE keys (about 2 %) take the whole warp's
//      shuffle network in place;
//   5. the image goes to the output with 16-byte vector copies.
// DRAM traffic is the algorithmic read + write; the second read hits L2.
#pragma once

#include "bitonic.cuh"
#include "common.cuh"
#include "local.cuh"
#include "local2.cuh"
#include "qsort.cuh"
#include "tma.cuh"

namespace vx {

#ifndef VX_Q3_STAGE_BYTES
#define VX_Q3_STAGE_BYTES (176 * 1024)
#endif
#ifndef VX_Q3_TARGET_BYTES
#define VX_Q3_TARGET_BYTES (150 * 1024)
#endif
#ifndef VX_Q3_TARGET8_BYTES
#define VX_Q3_TARGET8_BYTES (150 * 1024)
#endif
#ifndef VX_Q3_TMIN_BYTES
#define VX_Q3_TMIN_BYTES (96 * 1024)
#endif
#ifndef VX_Q3_LT10
#define VX_Q3_LT10 97  // largest mean bucket x 10 for 16-slot lanes
#endif
#ifndef VX_Q3_NT
#define VX_Q3_NT kQlNT  // threads per CTA
#endif
#ifndef VX_Q3_CTAS
#define VX_Q3_CTAS 1  // resident CTAs per SM (the stage and table must fit that many times)
#endif
#ifndef VX_Q3_NB
#define VX_Q3_NB 12288  // bucket table capacity
#endif
constexpr unsigned kQ3NT = VX_Q3_NT;

template <typename K, typename V>
struct Q3Cfg {
    static constexpr bool KV = HasVal<V>::value;
    static constexpr unsigned BYTES = sizeof(K) + (KV ? sizeof(V) : 0);
    static constexpr int LE = BYTES <= 8 ? 16 : 8;  // slots a lane sorts in registers
    static constexpr unsigned LT10 = LE == 16 ? VX_Q3_LT10 : VX_Q3_LT10 / 2;
    static constexpr unsigned ROUND = kQ3NT;  // buckets per round: one per lane
    static constexpr unsigned NB = VX_Q3_NB;  // bucket table capacity (leaves up to ~2.8x the 4-byte target)
    static constexpr unsigned BPT = NB / kQ3NT;
    static constexpr unsigned TAIL = 256 + 16;  // sentinel slots after the image (the widest network + alignment)
    static constexpr unsigned SLOTS = VX_Q3_STAGE_BYTES / BYTES;
    static constexpr unsigned SCAP = SLOTS - TAIL - 16;  // largest image
    // the plan aims the leaves here (at most): reached at any n <= 2^32 by a
    // sampled level of 256 buckets, then an equal-width level of up to 511
    // (code space for 4-byte keys, value space for float64); just below 4
    // rounds of buckets for 4-byte keys
    static constexpr uint64_t TARGET = (sizeof(K) == 4 ? VX_Q3_TARGET_BYTES : VX_Q3_TARGET8_BYTES) / BYTES;
    static constexpr uint64_t TMIN = VX_Q3_TMIN_BYTES / BYTES;
    static constexpr uint64_t CAPB = (uint64_t)(NB - ROUND) * LT10 / 10;
    static constexpr uint64_t CAP = 3 * TARGET < CAPB ? 3 * TARGET : CAPB;  // largest leaf taken
    static constexpr unsigned MAXG = 8;
    static_assert(SLOTS < 65536, "image positions are 16-bit");
    static_assert(CAP / (SCAP - 256) + 1 <= MAXG, "too many bucket groups");
};

template <typename K, typename V>
struct Q3Smem {
    using C = Q3Cfg<K, V>;
    using VS = typename std::conditional<HasVal<V>::value, V, char>::type;
    alignas(16) K k[C::SLOTS];
    alignas(16) VS v[HasVal<V>::value ? C::SLOTS : 16];
    unsigned tab[C::NB];             // bucket counts; then image cursor << 16 | count
    unsigned gstart[C::MAXG + 1];    // offset in the sorted leaf where group g starts
    unsigned gfirst[C::MAXG + 1];    // first bucket of group g
    typename OKey<K>::U rmin[kQ3NT / 32], rmax[kQ3NT / 32];
    unsigned scan[kQ3NT / 32 + 1];
};

// One lane sorts the E consecutive image slots that start at its bucket and
// stores the bucket's own cb (<= E) back.  The slots past cb hold keys of
// later buckets (or the sentinel tail): every one of them is larger than the
// bucket's keys, so they pad the network.  The load order is rotated by the
// lane (any input order sorts), which keeps the lanes of a warp on different
// banks; cb = 0 idles the lane.
template <typename K, typename V, int E>
__device__ __forceinline__ void lane_sort(K* sk, V* sv, unsigned ps, unsigned cb) {
    constexpr bool KV = HasVal<V>::value;
    using R = KeyRep<K>;
    using I = typename R::I;
    const unsigned lane = threadIdx.x & 31;
    I k[E];
    V v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const unsigned q = ps + ((r + lane) & (E - 1));
        k[r] = R::to(sk[q]);
        if constexpr (KV) v[r] = sv[q];
    }
    WarpBitonic<I, V, E, 1, true>::sort(k, v);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        if (r < (int)cb) {
            sk[ps + r] = R::from(k[r]);
            if constexpr (KV) sv[ps + r] = v[r];
        }
    }
}

// int32 keys with a payload, in a leaf whose key codes span less than 2^27:
// the lane sorts ONE word per pair, (code - lo) << 4 | slot, with the
// keys-only network (min / max instead of a compare and four selects per
// comparator), then fetches each pair's payload from the slot the word
// names.  Equal keys come out in slot order (any order is allowed).
template <typename K, typename V, int E>
__device__ __forceinline__ void lane_sort_packed(K* sk, V* sv, unsigned ps, unsigned cb, uint32_t lo) {
    static_assert(E == 16 && sizeof(K) == 4, "4 slot bits next to a 27-bit key offset");
    const unsigned lane = threadIdx.x & 31;
    int32_t w[E];
    NoVal nv[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const unsigned q = (r + lane) & (E - 1);
        const uint32_t d = min(OKey<K>::of(sk[ps + q]) - lo, 0x07ffffffu);  // (the sentinel tail saturates)
        w[r] = (int32_t)((d << 4) | q);
    }
    WarpBitonic<int32_t, NoVal, E, 1, true>::sort(w, nv);
    V val[E];
#pragma unroll
    for (int r = 0; r < E; ++r)
        if (r < (int)cb) val[r] = sv[ps + ((unsigned)w[r] & 15u)];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        if (r < (int)cb) {
            sk[ps + r] = (K)((((uint32_t)w[r] >> 4) + lo) ^ 0x80000000u);
            sv[ps + r] = val[r];
        }
    }
}

// A bucket of cb <= 32 * E keys through the whole warp's shuffle network, in
// place in the image (later buckets' keys pad it, as above).
template <typename K, typename V, int E>
__device__ __forceinline__ void image_warp_sort_e(K* sk, V* sv, unsigned ps, unsigned cb) {
    constexpr bool KV = HasVal<V>::value;
    using R = KeyRep<K>;
    using I = typename R::I;
    const unsigned lane = threadIdx.x & 31;
    I k[E];
    V v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        k[r] = R::to(sk[ps + lane * E + r]);
        if constexpr (KV) v[r] = sv[ps + lane * E + r];
    }
    __syncwarp();
    WarpBitonic<I, V, E>::sort(k, v);
    __syncwarp();  // every lane has read its slots
#pragma unroll
    for (int r = 0; r < E; ++r) {
        if (lane * E + r < cb) {
            sk[ps + lane * E + r] = R::from(k[r]);
            if constexpr (KV) sv[ps + lane * E + r] = v[r];
        }
    }
    __syncwarp();
}

template <typename K, typename V>
__device__ __forceinline__ void image_warp_sort(K* sk, V* sv, unsigned ps, unsigned cb) {
    if (cb <= 32) image_warp_sort_e<K, V, 1>(sk, sv, ps, cb);
    else if (cb <= 64) image_warp_sort_e<K, V, 2>(sk, sv, ps, cb);
    else if (cb <= 128) image_warp_sort_e<K, V, 4>(sk, sv, ps, cb);
    else image_warp_sort_e<K, V, 8>(sk, sv, ps, cb);
}

// image[0, n) -> dst[0, n).  The image is placed at dst's 16-byte phase, so
// the body moves as aligned vectors (a payload array whose phase differs
// from its keys' falls back to element copies).
template <typename T, unsigned NT>
__device__ __forceinline__ void image_copy_out(const T* img, T* __restrict__ dst, unsigned n) {
    constexpr unsigned VE = 16 / sizeof(T);
    if (((reinterpret_cast<uintptr_t>(img) ^ reinterpret_cast<uintptr_t>(dst)) & 15) != 0) {
        for (unsigned i = threadIdx.x; i < n; i += NT) dst[i] = img[i];
        return;
    }
    const unsigned head = min(n, (unsigned)(((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) / sizeof(T)));
    const unsigned nv = (n - head) / VE;
    if (threadIdx.x < head) dst[threadIdx.x] = img[threadIdx.x];
    const uint4* s4 = reinterpret_cast<const uint4*>(img + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    for (unsigned j = threadIdx.x; j < nv; j += NT) d4[j] = s4[j];
    const unsigned t0 = head + nv * VE;
    if (t0 + threadIdx.x < n) dst[t0 + threadIdx.x] = img[t0 + threadIdx.x];
}

// The same, with the aligned body as ONE thread's bulk stores (TMA), which
// drain while the CTA goes on to the next leaf: the caller fences the async
// proxy + barriers before, and waits for the reads (bulk_wait_read) before
// the image is overwritten.
template <typename T, unsigned NT>
__device__ __forceinline__ void image_store_async(const T* img, T* __restrict__ dst, unsigned n) {
    constexpr unsigned VE = 16 / sizeof(T);
    if (((reinterpret_cast<uintptr_t>(img) ^ reinterpret_cast<uintptr_t>(dst)) & 15) != 0) {
        for (unsigned i = threadIdx.x; i < n; i += NT) dst[i] = img[i];
        return;
    }
    const unsigned head = min(n, (unsigned)(((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) / sizeof(T)));
    const unsigned nv = (n - head) / VE;
    if (threadIdx.x == 0) {
        constexpr unsigned CH = 32768;  // bytes per bulk store
        const char* s = reinterpret_cast<const char*>(img + head);
        char* d = reinterpret_cast<char*>(dst + head);
        for (unsigned o = 0; o < nv * 16; o += CH) bulk_s2g(d + o, s + o, min(CH, nv * 16 - o));
    }
    if (threadIdx.x >= 32 && threadIdx.x < 32 + head) dst[threadIdx.x - 32] = img[threadIdx.x - 32];
    const unsigned t0 = head + nv * VE;
    if (threadIdx.x >= 64 && t0 + threadIdx.x - 64 < n) dst[t0 + threadIdx.x - 64] = img[t0 + threadIdx.x - 64];
}

template <typename K, typename V>
__global__ void __launch_bounds__(kQ3NT, VX_Q3_CTAS) qs_local3_kernel(const QlItem* __restrict__ items, Ctl* __restrict__ ctl,
                                                             Ctl* __restrict__ ctl_next, Seg* __restrict__ next_segs,
                                                             unsigned cap_seg, const K* __restrict__ src_k,
                                                             const V* __restrict__ src_v, K* __restrict__ oth_k,
                                                             V* __restrict__ oth_v, K* __restrict__ out_k,
                                                             V* __restrict__ out_v, unsigned leaf) {
    using C = Q3Cfg<K, V>;
    using U = typename OKey<K>::U;
    constexpr bool KV = HasVal<V>::value;
    constexpr unsigned NT = kQ3NT, BPT = C::BPT;
    constexpr int LE = C::LE;
    constexpr unsigned VE = 16 / sizeof(K);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Q3Smem<K, V>& sm = *reinterpret_cast<Q3Smem<K, V>*>(smem_raw);
    V* const stv = KV ? reinterpret_cast<V*>(sm.v) : nullptr;
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned nitems = ctl->ql_ctr;
    const unsigned wmax = min(leaf, 256u);
    unsigned long long done = 0;
#ifdef VX_QL_PHASES
    long long tick = clock64();
#endif
    for (unsigned it = blockIdx.x; it < nitems; it += gridDim.x) {
        const uint64_t start = items[it].start;
        const unsigned len = (unsigned)items[it].len;
        const K* sk = src_k + start;
        // ---- 1. key-code range
        U lo = ~(U)0, hi = 0;
        if (items[it].lo <= items[it].hi) {
            lo = (U)items[it].lo;
            hi = (U)items[it].hi;
        } else {
            seg_for_each<K, NT>(sk, len, [&](K x) {
                const U u = OKey<K>::of(x);
                lo = ql_min(lo, u);
                hi = ql_max(hi, u);
            });
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
                lo = ql_min(lo, (U)__shfl_xor_sync(0xffffffffu, lo, d));
                hi = ql_max(hi, (U)__shfl_xor_sync(0xffffffffu, hi, d));
            }
            if (lane == 0) {
                sm.rmin[warp] = lo;
                sm.rmax[warp] = hi;
            }
            __syncthreads();
#pragma unroll
            for (int w = 0; w < (int)(NT / 32); ++w) {
                lo = ql_min(lo, sm.rmin[w]);
                hi = ql_max(hi, sm.rmax[w]);
            }
        }
        if (lo == hi) {  // one key value: already sorted
            if (sk != out_k + start)
                for (unsigned i = tid; i < len; i += NT) {
                    out_k[start + i] = sk[i];
                    if constexpr (KV) out_v[start + i] = src_v[start + i];
                }
            done += len;
            __syncthreads();
            continue;
        }
        VX_QL_TICK(0);
        // ---- 2. interpolation buckets: b = floor(d * nb / (range + 1)), a
        //      whole number of rounds of them
        unsigned nb = min(C::NB, (unsigned)(((uint64_t)len * 10 + C::ROUND * C::LT10 - 1) / (C::ROUND * C::LT10)) * C::ROUND);
        const U range = hi - lo;
        const unsigned bits = (unsigned)(8 * sizeof(U)) -
                              (sizeof(U) == 8 ? (unsigned)__clzll((long long)range) : (unsigned)__clz((int)range));
        const unsigned sh = bits > 32 ? bits - 32 : 0u;
        const uint32_t r32 = (uint32_t)(range >> sh);
        uint32_t mul = 0;
        if ((uint64_t)r32 + 1 <= nb) nb = r32 + 1;
        else mul = (uint32_t)(((uint64_t)nb << 32) / ((uint64_t)r32 + 1));
        auto bucket = [&](K key) -> unsigned {
            U u;
            if constexpr (sizeof(K) == 8) {
                // -0.0 joins +0.0's bucket (x + 0.0 is +0.0 for both): the
                // networks compare by value, so a later bucket may never hold
                // a key EQUAL to one of an earlier bucket (see lane_sort);
                // clamped, in case the parent's pivot fell between the two
                u = ql_min(OKey<K>::of(key + 0.0), hi);
            } else {
                u = OKey<K>::of(key);
            }
            VX_ASSERT(u >= lo && u <= hi);  // every key lies inside the leaf's bounds
            const uint32_t d = (uint32_t)((u - lo) >> sh);
            const unsigned bk = mul ? __umulhi(d, mul) : d;
            VX_ASSERT(bk < nb);
            return bk;
        };
        const unsigned nbt = (nb + BPT - 1) / BPT;  // threads that own buckets
        if (tid < nbt) {
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) sm.tab[tid * BPT + q] = 0;
        }
        __syncthreads();
        // (result unused: ATOMS.POPC.INC merges a warp's same-counter lanes)
        seg_for_each<K, NT>(sk, len, [&](K x) { atomicAdd(&sm.tab[bucket(x)], 1u); });
        __syncthreads();
        VX_QL_TICK(1);
        // ---- 3. image offsets
        unsigned c[BPT], sum = 0;
        bool over = false;
        if (tid < nbt) {
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) {
                c[q] = sm.tab[tid * BPT + q];
                sum += c[q];
                over |= c[q] > wmax;
            }
        } else {
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) c[q] = 0;
        }
        if (__syncthreads_or(over)) {
            // skewed keys: back to a sampled-pivot level (data stays in src)
            if (tid == 0) {
                const unsigned q = atomicAdd(&ctl_next->nseg, 1u);
                if (q >= cap_seg) {
                    atomicOr(&ctl->err, kErrCapacity);
                } else {
                    next_segs[q].start = start;
                    next_segs[q].len = len;
                    next_segs[q].lo = 1;  // skewed: sampled pivots next
                    next_segs[q].hi = 0;
                }
            }
            continue;  // the barrier above ends every use of the tables
        }
        unsigned tot;
        const unsigned ex0 = block_excl_scan<NT>(sum, sm.scan, &tot);  // tot == len
        VX_ASSERT(tot == len);
        const unsigned G = tot <= C::SCAP ? 1u : (tot + (C::SCAP - 256) - 1) / (C::SCAP - 256);
        const unsigned W = G == 1 ? 0xffffffffu : (tot + G - 1) / G;
        // a leaf sorted in place in G > 1 groups: the groups before the last
        // still have readers of the source, so their images detour through
        // the other buffer and come home after the last group's pass
        const bool detour = G > 1 && src_k == out_k;
        // group g's image starts at the 16-byte phase of its destination
        auto phase_of = [&](unsigned g, unsigned gs) -> unsigned {
            const K* d = (detour && g + 1 < G ? oth_k : out_k) + start + gs;
            return (unsigned)((reinterpret_cast<uintptr_t>(d) & 15) / sizeof(K));
        };
        if (G == 1) {
            if (tid < nbt) {
                unsigned ex = ex0 + phase_of(0, 0);
#pragma unroll
                for (unsigned q = 0; q < BPT; ++q) {
                    sm.tab[tid * BPT + q] = (ex << 16) | c[q];
                    ex += c[q];
                }
            }
            if (tid == 0) {
                sm.gstart[0] = 0;
                sm.gfirst[0] = 0;
                sm.gstart[1] = tot;
                sm.gfirst[1] = nb;
            }
        } else {
            if (tid < nbt) {
                // a bucket opens a group when its offset enters the group's window
                unsigned ex = ex0;
                unsigned prevo = tid > 0 ? ex0 - sm.tab[tid * BPT - 1] : 0u;
#pragma unroll
                for (unsigned q = 0; q < BPT; ++q) {
                    const unsigned b = tid * BPT + q;
                    // (empty buckets at the very end, offset == tot == G * W, stay in the last group)
                    const unsigned gq = min(ex / W, G - 1), gp = min(prevo / W, G - 1);
                    if (b < nb && (b == 0 || gp != gq)) {
                        sm.gstart[gq] = ex;
                        sm.gfirst[gq] = b;
                    }
                    prevo = ex;
                    ex += c[q];
                }
            }
            if (tid == 0) {
                sm.gstart[G] = tot;
                sm.gfirst[G] = nb;
            }
            __syncthreads();
            if (tid < nbt) {
                unsigned ex = ex0;
#pragma unroll
                for (unsigned q = 0; q < BPT; ++q) {
                    const unsigned g = min(ex / W, G - 1), gs = sm.gstart[g];
                    sm.tab[tid * BPT + q] = ((ex - gs + phase_of(g, gs)) << 16) | c[q];
                    ex += c[q];
                }
            }
        }
        // the previous leaf's image has left shared memory before anything
        // overwrites it
        if (tid == 0) bulk_wait_read();
        __syncthreads();
        VX_QL_TICK(2);
        for (unsigned g = 0; g < G; ++g) {
            const unsigned gs = sm.gstart[g], glen = sm.gstart[g + 1] - gs;
            const unsigned b_lo = sm.gfirst[g], nbg = sm.gfirst[g + 1] - b_lo;
            const unsigned ph = phase_of(g, gs);
            // sentinels behind the image: the padding of its last buckets
            if (tid < C::TAIL) sm.k[ph + glen + tid] = KeyTraits<K>::sentinel();
            // ---- 4a. every key of the group to its bucket's cursor in the image
            if (G == 1) {
                if constexpr (!KV) {
                    seg_for_each<K, NT>(sk, len, [&](K x) {
                        const unsigned p = atomicAdd(&sm.tab[bucket(x)], 0x10000u) >> 16;
                        VX_ASSERT(p >= ph && p < ph + glen);
                        sm.k[p] = x;
                    });
                } else {
                    const V* svp = src_v + start;
                    seg_for_each_idx<K, NT>(sk, len, [&](K x, unsigned i) {
                        const V y = svp[i];
                        const unsigned p = atomicAdd(&sm.tab[bucket(x)], 0x10000u) >> 16;
                        VX_ASSERT(p >= ph && p < ph + glen);
                        sm.k[p] = x;
                        stv[p] = y;
                    });
                }
            } else {
                const V* svp = KV ? src_v + start : nullptr;
                seg_for_each_idx<K, NT>(sk, len, [&](K x, unsigned i) {
                    const unsigned b = bucket(x);
                    if (b - b_lo < nbg) {
                        const unsigned p = atomicAdd(&sm.tab[b], 0x10000u) >> 16;
                        VX_ASSERT(p >= ph && p < ph + glen);
                        sm.k[p] = x;
                        if constexpr (KV) stv[p] = svp[i];
                    }
                });
            }
            __syncthreads();
            VX_QL_TICK(3);
            // the next leaf on its way into L2 while the networks run
            if (g + 1 == G && it + gridDim.x < nitems) {
                const QlItem nx = items[it + gridDim.x];
                const char* np = reinterpret_cast<const char*>(src_k + nx.start);
                const unsigned nbytes = (unsigned)nx.len * (unsigned)sizeof(K);
                for (unsigned o = tid * 128u; o < nbytes; o += NT * 128u)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(np + o));
                if constexpr (KV) {
                    const char* nv = reinterpret_cast<const char*>(src_v + nx.start);
                    for (unsigned o = tid * 128u; o < nbytes; o += NT * 128u)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(nv + o));
                }
            }
            // ---- 4b. one bucket per lane through the register network
            for (unsigned b0 = b_lo + warp * 32; b0 < b_lo + nbg; b0 += NT) {
                const unsigned b = b0 + lane;
                unsigned cb = 0, ps = ph;
                if (b < b_lo + nbg) {
                    const unsigned t = sm.tab[b];  // the cursor ended at the bucket's end
                    cb = t & 0xffffu;
                    ps = (t >> 16) - cb;
                    VX_ASSERT(ps >= ph && ps + cb <= ph + glen && ph + glen + C::TAIL <= C::SLOTS);
                }
                const bool big = cb > (unsigned)LE;
                if constexpr (KV && sizeof(K) == 4 && LE == 16) {
                    if (range < 0x07ffffffu) lane_sort_packed<K, V, LE>(sm.k, stv, ps, big ? 0u : cb, (uint32_t)lo);
                    else lane_sort<K, V, LE>(sm.k, stv, ps, big ? 0u : cb);
                } else {
                    lane_sort<K, V, LE>(sm.k, stv, ps, big ? 0u : cb);
                }
                // the few buckets above a lane's slots take the whole warp
                unsigned bm = __ballot_sync(0xffffffffu, big);
                while (bm) {
                    const int src = __ffs(bm) - 1;
                    bm &= bm - 1;
                    image_warp_sort<K, V>(sm.k, stv, __shfl_sync(0xffffffffu, ps, src),
                                          __shfl_sync(0xffffffffu, cb, src));
                }
            }
            if (G == 1) fence_async_smem();
            __syncthreads();
            VX_QL_TICK(4);
            // ---- 5. the image to the output
            if (G == 1) {
                image_store_async<K, NT>(sm.k + ph, out_k + start, glen);
                if constexpr (KV) image_store_async<V, NT>(stv + ph, out_v + start, glen);
                if (tid == 0) bulk_commit();
                // (no barrier: the next leaf's range / count / scan passes do
                // not touch the image; its scan waits for the store's reads)
            } else {
                const bool away = detour && g + 1 < G;
                image_copy_out<K, NT>(sm.k + ph, (away ? oth_k : out_k) + start + gs, glen);
                if constexpr (KV) image_copy_out<V, NT>(stv + ph, (away ? oth_v : out_v) + start + gs, glen);
                __syncthreads();
            }
            VX_QL_TICK(5);
        }
        if (detour) {
            const unsigned n1 = sm.gstart[G - 1];  // output offset of the last group
            for (unsigned i = tid; i < n1; i += NT) {
                out_k[start + i] = oth_k[start + i];
                if constexpr (KV) out_v[start + i] = oth_v[start + i];
            }
            __syncthreads();
        }
        done += len;
    }
    if (tid == 0) bulk_wait_read();  // the last image is still being read
    if (tid == 0 && done) atomicAdd(&ctl->loc_elems, done);
}

}  // namespace vx
