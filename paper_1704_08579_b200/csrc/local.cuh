// local.cuh -- CTA-local last partition level + bitonic leaves for medium
// segments (north-star subsystem 3, the bottom of _kernels.quicksort,
// _kernels.py:396-423).
//
// A segment of up to QlCfg::CAP keys (48-64 Ki int32 at the mean) is owned
// by one CTA from partition to sorted output, so its working set stays in L2:
//   1. the key-code range: the parent's pivots bound an inner bucket; the
//      two outer buckets of a segment take one pass for [min, max];
//   2. one pass (the HBM read) counting interpolation buckets of ~LT keys
//      over that range (equal-width code intervals = evenly spaced pivots);
//      if any bucket exceeds the leaf bound the keys are skewed and the
//      segment goes back to the sampled-pivot level queue instead;
//   3. one pass (from L2) that classifies again and places every key in its
//      bucket of the other buffer: keys only straight to the bucket's
//      shared-memory cursor, pairs staged per tile and written as runs;
//   4. warps take the buckets round-robin and sort each (<= leaf bound) with
//      the register bitonic network (bitonic.cuh) straight into the output.
// This replaces the last global level (plan + hist + scatter over the whole
// array) and the finish kernel's own partition for every segment it takes.
#pragma once

#include "bitonic.cuh"
#include "common.cuh"
#include "qsort.cuh"

namespace vx {

#ifndef VX_QL_NT
#define VX_QL_NT 1024
#endif
constexpr int kQlNT = VX_QL_NT;
#ifndef VX_QL_TARGET_BYTES
#define VX_QL_TARGET_BYTES (256 * 1024)
#endif
#ifndef VX_QL_LT
#define VX_QL_LT 110
#endif
constexpr unsigned kQlLeafTarget = VX_QL_LT;  // mean interpolation bucket (int32)

template <typename K, typename V>
struct QlCfg {
    static constexpr unsigned BYTES = sizeof(K) + (HasVal<V>::value ? sizeof(V) : 0);
    static constexpr uint64_t TARGET = VX_QL_TARGET_BYTES / BYTES;  // plan aims level leaves here (at most)
#ifndef VX_QL_TMIN_BYTES
#define VX_QL_TMIN_BYTES (192 * 1024)
#endif
    static constexpr uint64_t TMIN = VX_QL_TMIN_BYTES / BYTES;      // ... and at least here
    static constexpr uint64_t CAP = 3 * TARGET;                     // largest segment taken
    static constexpr unsigned IPT = 8;
    static constexpr unsigned TILE = kQlNT * IPT;
#ifndef VX_QL_LT8
#define VX_QL_LT8 55
#endif
    static constexpr unsigned LT = BYTES <= 4 ? kQlLeafTarget : VX_QL_LT8;  // mean bucket (8-byte elements: smaller)
    static constexpr unsigned NB = CAP / LT + 1 <= 2048 ? 2048 : 4096;     // bucket table capacity (>= CAP / LT)
    static constexpr unsigned BPT = NB / kQlNT;
    static_assert(CAP / LT + 1 <= NB, "bucket table too small");
};

using QlItem = QlItemT;

// Phase clocks of the CTA-local level (tuning builds only, -DVX_QL_PHASES):
// SM cycles summed over CTAs for range / count / scan / scatter / networks.
#ifdef VX_QL_PHASES
__device__ unsigned long long g_ql_phase[8];
#define VX_QL_TICK(i)                                                   \
    do {                                                                \
        if (threadIdx.x == 0) {                                         \
            const long long t_ = clock64();                             \
            atomicAdd(&g_ql_phase[i], (unsigned long long)(t_ - tick)); \
            tick = t_;                                                  \
        }                                                               \
    } while (0)
#else
#define VX_QL_TICK(i) \
    do {              \
    } while (0)
#endif

template <typename K, typename V>
struct QlSmem {
    using C = QlCfg<K, V>;
    using VS = typename std::conditional<HasVal<V>::value, V, char>::type;
    K k[C::TILE];
    VS v[HasVal<V>::value ? C::TILE : 1];
    unsigned short b[C::TILE];
    unsigned cnt[C::NB];    // bucket sizes of the segment
    unsigned off[C::NB];    // bucket start (segment-relative), then the fill cursor
    unsigned tcnt[C::NB];   // per-tile counts, then tile offsets
    unsigned delta[C::NB];  // per-tile: destination (segment-relative) of staged slot j = delta[b] + j
    typename OKey<K>::U rmin[kQlNT / 32], rmax[kQlNT / 32];
    unsigned scan[kQlNT / 32 + 1];
    unsigned next;
    unsigned tn;
};


// f(key) for every key of p[0, len): 16-byte vector loads for the aligned
// body, four vectors in flight per thread, scalar head and tail.
template <typename K, unsigned NT, typename F>
__device__ __forceinline__ void seg_for_each(const K* __restrict__ p, unsigned len, F&& f) {
    constexpr unsigned VE = 16 / sizeof(K);
    union Vec {
        uint4 v;
        K k[VE];
    };
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const unsigned head = min(len, (unsigned)(((16 - (a & 15)) & 15) / sizeof(K)));
    for (unsigned i = threadIdx.x; i < head; i += NT) f(p[i]);
    const unsigned nv = (len - head) / VE;
    const uint4* v = reinterpret_cast<const uint4*>(p + head);
    unsigned j = threadIdx.x;
    for (; j + 3 * NT < nv; j += 4 * NT) {
        Vec w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u].v = v[j + u * NT];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (unsigned r = 0; r < VE; ++r) f(w[u].k[r]);
    }
    for (; j < nv; j += NT) {
        Vec w;
        w.v = v[j];
#pragma unroll
        for (unsigned r = 0; r < VE; ++r) f(w.k[r]);
    }
    for (unsigned i = head + nv * VE + threadIdx.x; i < len; i += NT) f(p[i]);
}

// f(keys, count) for every 16-byte vector of p[0, len) (count = 16 /
// sizeof(K) consecutive keys; the unaligned head and tail come one key at a
// time): lets a pass aggregate a vector's keys that share a bucket.
template <typename K, unsigned NT, typename F>
__device__ __forceinline__ void seg_for_each_vec(const K* __restrict__ p, unsigned len, F&& f) {
    constexpr unsigned VE = 16 / sizeof(K);
    union Vec {
        uint4 v;
        K k[VE];
    };
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const unsigned head = min(len, (unsigned)(((16 - (a & 15)) & 15) / sizeof(K)));
    for (unsigned i = threadIdx.x; i < head; i += NT) f(&p[i], 1u);
    const unsigned nv = (len - head) / VE;
    const uint4* v = reinterpret_cast<const uint4*>(p + head);
    unsigned j = threadIdx.x;
    for (; j + 3 * NT < nv; j += 4 * NT) {
        Vec w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u].v = v[j + u * NT];
#pragma unroll
        for (int u = 0; u < 4; ++u) f(w[u].k, VE);
    }
    for (; j < nv; j += NT) {
        Vec w;
        w.v = v[j];
        f(w.k, VE);
    }
    for (unsigned i = head + nv * VE + threadIdx.x; i < len; i += NT) f(&p[i], 1u);
}

template <typename U>
__device__ __forceinline__ U ql_min(U a, U b) { return a < b ? a : b; }
template <typename U>
__device__ __forceinline__ U ql_max(U a, U b) { return a > b ? a : b; }

// Resident CTAs per SM: keys-only sorts run one 1024-thread CTA per SM (64
// registers, half the L2 footprint); pairs keep two (their tile-staged
// scatter hides more latency with the second CTA).  Measured on B200.
template <typename V>
struct QlMinBlocks {
    static constexpr int value = HasVal<V>::value ? 2048 / kQlNT : 1;
};
template <typename K, typename V>
__global__ void __launch_bounds__(kQlNT, QlMinBlocks<V>::value) qs_local_kernel(const QlItem* __restrict__ items, Ctl* __restrict__ ctl,
                                                            Ctl* __restrict__ ctl_next, Seg* __restrict__ next_segs,
                                                            unsigned cap_seg, const K* __restrict__ src_k,
                                                            const V* __restrict__ src_v, K* __restrict__ oth_k,
                                                            V* __restrict__ oth_v, K* __restrict__ out_k,
                                                            V* __restrict__ out_v, unsigned leaf) {
    using C = QlCfg<K, V>;
    using U = typename OKey<K>::U;
    constexpr bool KV = HasVal<V>::value;
    constexpr unsigned NT = kQlNT, IPT = C::IPT, TILE = C::TILE, BPT = C::BPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    QlSmem<K, V>& sm = *reinterpret_cast<QlSmem<K, V>*>(smem_raw);
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
        // ---- 1. key-code range: the parent's pivots bound an inner bucket;
        //      the two outer buckets of a segment are measured
        U lo = ~(U)0, hi = 0;
        const bool bounded = items[it].lo <= items[it].hi;
        if (bounded) {
            lo = (U)items[it].lo;
            hi = (U)items[it].hi;
        } else {
            unsigned i = tid;
            for (; i + 3 * NT < len; i += 4 * NT) {
                U u[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) u[r] = OKey<K>::of(sk[i + r * NT]);
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    lo = ql_min(lo, u[r]);
                    hi = ql_max(hi, u[r]);
                }
            }
            for (; i < len; i += NT) {
                const U u = OKey<K>::of(sk[i]);
                lo = ql_min(lo, u);
                hi = ql_max(hi, u);
            }
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
        // ---- 2. interpolation buckets: b = floor(d * nb / (range + 1))
        unsigned nb = min(C::NB, max(1u, (len + C::LT - 1) / C::LT));
        const U range = hi - lo;
        const unsigned bits = (unsigned)(8 * sizeof(U)) -
                              (sizeof(U) == 8 ? (unsigned)__clzll((long long)range) : (unsigned)__clz((int)range));
        const unsigned sh = bits > 32 ? bits - 32 : 0u;
        const uint32_t r32 = (uint32_t)(range >> sh);
        uint32_t mul = 0;
        if ((uint64_t)r32 + 1 <= nb) nb = r32 + 1;
        else mul = (uint32_t)(((uint64_t)nb << 32) / ((uint64_t)r32 + 1));
        auto bucket = [&](K key) -> unsigned {
#ifdef VX_CHECK
            // checked build: every key lies inside the segment's bounds
            if (OKey<K>::of(key) < lo || OKey<K>::of(key) > hi) __trap();
#endif
            const uint32_t d = (uint32_t)((OKey<K>::of(key) - lo) >> sh);
            return mul ? __umulhi(d, mul) : d;
        };
#pragma unroll
        for (unsigned q = 0; q < BPT; ++q) sm.cnt[tid * BPT + q] = 0;
        __syncthreads();
        // (result unused: ATOMS.POPC.INC merges a warp's same-counter lanes)
        seg_for_each<K, NT>(sk, len, [&](K x) { atomicAdd(&sm.cnt[bucket(x)], 1u); });
        __syncthreads();
        VX_QL_TICK(1);
        unsigned c[BPT], sum = 0;
        bool over = false;
#pragma unroll
        for (unsigned q = 0; q < BPT; ++q) {
            c[q] = sm.cnt[tid * BPT + q];
            sum += c[q];
            over |= c[q] > wmax;
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
        {
            unsigned tot;
            unsigned ex = block_excl_scan<NT>(sum, sm.scan, &tot);
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) {
                sm.off[tid * BPT + q] = ex;  // fill cursor, segment-relative
                ex += c[q];
            }
        }
        VX_QL_TICK(2);
        // ---- 3. scatter into the other buffer, bucket-major
        K* ok = oth_k + start;
        V* ov = KV ? oth_v + start : nullptr;
        // keys only: every element straight to its bucket's fill cursor (a
        // shared-memory atomic) -- order inside a bucket is irrelevant, the
        // network sorts it, and the scattered stores merge in L2, so there
        // are no tile barriers at all.  Pairs (two scattered stores per
        // element) are staged per tile and written as runs instead
        // (measured on B200: direct -4 % int32 keys, +26 % kv).
        if constexpr (!KV) {
        __syncthreads();  // cursors complete
        seg_for_each_vec<K, NT>(sk, len, [&](const K* x, unsigned c) {
            if (c == 1) {
                ok[atomicAdd(&sm.off[bucket(x[0])], 1u)] = x[0];
                return;
            }
            constexpr unsigned VE = 16 / sizeof(K);
            unsigned b[VE];
#pragma unroll
            for (unsigned r = 0; r < VE; ++r) b[r] = bucket(x[r]);
            bool run = true;
#pragma unroll
            for (unsigned r = 1; r < VE; ++r) run &= b[r] == b[0];
            if (run) {  // a sorted run inside one bucket: one reservation
                const unsigned p0 = atomicAdd(&sm.off[b[0]], VE);
#pragma unroll
                for (unsigned r = 0; r < VE; ++r) ok[p0 + r] = x[r];
                return;
            }
#pragma unroll
            for (unsigned r = 0; r < VE; ++r) ok[atomicAdd(&sm.off[b[r]], 1u)] = x[r];
        });
        } else {
        for (unsigned t0 = 0; t0 < len; t0 += TILE) {
            const unsigned tn = min(TILE, len - t0);
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) sm.tcnt[tid * BPT + q] = 0;
            __syncthreads();
            K x[IPT];
            V y[IPT];
            unsigned br[IPT];
#pragma unroll
            for (unsigned r = 0; r < IPT; ++r) {
                const unsigned i = r * NT + tid;
                if (i < tn) {
                    x[r] = sk[t0 + i];
                    if constexpr (KV) y[r] = src_v[start + t0 + i];
                    const unsigned b = bucket(x[r]);
                    br[r] = (b << 16) | atomicAdd(&sm.tcnt[b], 1u);
                }
            }
            __syncthreads();
            unsigned tc[BPT], ts = 0;
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) {
                tc[q] = sm.tcnt[tid * BPT + q];
                ts += tc[q];
            }
            unsigned tot;
            unsigned ex = block_excl_scan<NT>(ts, sm.scan, &tot);
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) {
                const unsigned b = tid * BPT + q;
                sm.tcnt[b] = ex;                       // tile offset of bucket b
                sm.delta[b] = sm.off[b] - ex;          // slot j of bucket b goes to delta[b] + j
                sm.off[b] += tc[q];
                ex += tc[q];
            }
            if (tid == 0) sm.tn = tn;
            __syncthreads();
#pragma unroll
            for (unsigned r = 0; r < IPT; ++r) {
                if (r * NT + tid < tn) {
                    const unsigned slot = sm.tcnt[br[r] >> 16] + (br[r] & 0xffffu);
                    sm.k[slot] = x[r];
                    if constexpr (KV) sm.v[slot] = y[r];
                    sm.b[slot] = (unsigned short)(br[r] >> 16);
                }
            }
            __syncthreads();
            for (unsigned j = tid; j < tn; j += NT) {
                const unsigned pos = sm.delta[sm.b[j]] + j;
                ok[pos] = sm.k[j];
                if constexpr (KV) ov[pos] = sm.v[j];
            }
        }
        }  // staged
        // ---- 4. every bucket through the bitonic network into the output
        if (tid == 0) sm.next = 0;
        __syncthreads();  // bucket runs written (CTA-scope visibility of global stores)
        VX_QL_TICK(3);
#ifndef VX_QL_DYNAMIC
        // buckets are near-equal (interpolation over a narrow range), so warps
        // take them round-robin: no shared counter between networks
        for (unsigned b0 = warp; b0 < nb; b0 += NT / 32) {
            const unsigned cb = sm.cnt[b0];
            if (cb == 0) continue;
            const unsigned bs = sm.off[b0] - cb;  // the cursor ended at the bucket's end
            warp_sort_any<K, V>(ok, ov, out_k + start, KV ? out_v + start : nullptr, bs, cb);
        }
#else
        for (;;) {
            unsigned b0 = 0;
            if (lane == 0) b0 = atomicAdd(&sm.next, 1u);
            b0 = __shfl_sync(0xffffffffu, b0, 0);
            if (b0 >= nb) break;
            const unsigned cb = sm.cnt[b0];
            if (cb == 0) continue;
            const unsigned bs = sm.off[b0] - cb;  // the cursor ended at the bucket's end
            warp_sort_any<K, V>(ok, ov, out_k + start, KV ? out_v + start : nullptr, bs, cb);
        }
#endif
        done += len;
        __syncthreads();
        VX_QL_TICK(4);
    }
    if (tid == 0 && done) atomicAdd(&ctl->loc_elems, done);
}

}  // namespace vx
