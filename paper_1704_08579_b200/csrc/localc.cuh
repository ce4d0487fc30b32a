// localc.cuh -- the CTA-local last partition level in DISTRIBUTED shared
// memory: a thread-block cluster of kQcC CTAs (one per SM) owns a medium
// segment from partition to sorted output (north-star subsystem 3, the
// bottom of _kernels.quicksort, _kernels.py:396-423).
//
// The segment (up to QlCfg::CAP keys, 768 KB of int32) is larger than one
// SM's shared memory but fits in the cluster's (4 x ~200 KB), so it is
// read from HBM once, partitioned straight into shared memory and written
// to HBM once -- one algorithmic pass, no intermediate copy in global
// memory (the single-CTA kernel in local.cuh wrote the bucket-major
// intermediate through L2 and read it back):
//   1. key-code range: the parent's pivots bound an inner bucket; outer
//      buckets reduce their quarters' [min, max] across the cluster;
//   2. every CTA counts its quarter of the segment into interpolation
//      buckets of ~LT keys (evenly spaced pivots, like local.cuh); a bucket
//      above the leaf bound means skewed keys: the segment goes back to the
//      sampled-pivot level queue (all CTAs see the same totals);
//   3. cluster-wide bucket starts (every CTA reads the others' counts over
//      DSMEM); the sorted segment is cut into C contiguous ranges at bucket
//      boundaries, range c owned by CTA c;
//   4. every CTA reads its quarter again (L2) and stores each key into the
//      OWNER's shared memory at its bucket cursor (st.shared::cluster);
//   5. after a cluster barrier each CTA sorts its buckets in place with the
//      warp bitonic network (bitonic.cuh, the reference's network) and
//      writes its whole range with coalesced stores.
#pragma once

#include <cooperative_groups.h>

#include "bitonic.cuh"
#include "common.cuh"
#include "finish.cuh"
#include "local.cuh"
#include "qsort.cuh"

namespace vx {

namespace cg = cooperative_groups;

constexpr int kQcC = 4;                  // CTAs per cluster
constexpr unsigned kQcSmemMax = 232448;  // B200 opt-in dynamic shared memory per CTA (227 KB)

template <typename K, typename V>
struct QcCfg {
    using Q = QlCfg<K, V>;
    static constexpr bool KV = HasVal<V>::value;
    static constexpr unsigned NB = Q::NB;  // bucket table entries (>= CAP / LT)
    static constexpr unsigned TABLES = 3 * NB * 4 + 2048;
    static constexpr unsigned PER = sizeof(K) + (KV ? sizeof(V) : 0);
    // receive slots per CTA (padded one word in 32 against bank conflicts)
    static constexpr unsigned PSLOTS = (kQcSmemMax - TABLES) / PER;
    static constexpr unsigned SLOTS = PSLOTS * 32 / 33 - 1;
    // a CTA owns a quarter of the segment plus at most one bucket (<= 256)
    static constexpr uint64_t CAP_CL = (uint64_t)(SLOTS - 256) * kQcC;
    static constexpr uint64_t CAP = Q::CAP < CAP_CL ? Q::CAP : CAP_CL;
};

template <typename K, typename V>
struct QcSmem {
    using C = QcCfg<K, V>;
    using U = typename OKey<K>::U;
    using VS = typename std::conditional<HasVal<V>::value, V, char>::type;
    K k[C::PSLOTS];
    VS v[HasVal<V>::value ? C::PSLOTS : 1];
    unsigned cnt[C::NB];  // this CTA's quarter: keys per bucket (read by the whole cluster)
    unsigned st[C::NB + 1];  // bucket start in the segment
    unsigned cur[C::NB];  // this CTA's write cursor per bucket: owner << 20 | owner-relative slot
    U rmin[kQlNT / 32], rmax[kQlNT / 32];
    U cmin, cmax;         // this CTA's quarter range (read by the cluster)
    unsigned first[kQcC + 1];   // owned range of CTA c: [first[c], first[c+1]) in the segment
    unsigned bfirst[kQcC + 1];  // first bucket owned by CTA c
    unsigned scan[kQlNT / 32 + 1];
};

template <typename K, typename V>
__global__ void __cluster_dims__(kQcC, 1, 1) __launch_bounds__(kQlNT, 1)
    qs_localc_kernel(const QlItem* __restrict__ items, Ctl* __restrict__ ctl, Ctl* __restrict__ ctl_next,
                     Seg* __restrict__ next_segs, unsigned cap_seg, const K* __restrict__ src_k,
                     const V* __restrict__ src_v, K* __restrict__ out_k, V* __restrict__ out_v, unsigned leaf) {
    using C = QcCfg<K, V>;
    using Q = QlCfg<K, V>;
    using U = typename OKey<K>::U;
    constexpr bool KV = HasVal<V>::value;
    constexpr unsigned NT = kQlNT, BPT = C::NB / kQlNT;
    static_assert(C::NB % kQlNT == 0, "buckets per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    QcSmem<K, V>& sm = *reinterpret_cast<QcSmem<K, V>*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned me = cluster.block_rank();
    const unsigned tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned nitems = ctl->ql_ctr;
    const unsigned ncl = gridDim.x / kQcC, cid = blockIdx.x / kQcC;
    const unsigned wmax = min(leaf, 256u);
    unsigned long long done = 0;
    for (unsigned it = cid; it < nitems; it += ncl) {
        const uint64_t start = items[it].start;
        const unsigned len = (unsigned)items[it].len;
        const unsigned q0 = (unsigned)((uint64_t)len * me / kQcC), q1 = (unsigned)((uint64_t)len * (me + 1) / kQcC);
        const K* sk = src_k + start;
        // ---- 1. key-code range
        U lo = ~(U)0, hi = 0;
        if (items[it].lo <= items[it].hi) {
            lo = (U)items[it].lo;
            hi = (U)items[it].hi;
        } else {
            seg_for_each<K, NT>(sk + q0, q1 - q0, [&](K x) {
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
            if (tid == 0) {
#pragma unroll 1
                for (int w = 0; w < (int)(NT / 32); ++w) {
                    lo = ql_min(lo, sm.rmin[w]);
                    hi = ql_max(hi, sm.rmax[w]);
                }
                sm.cmin = lo;
                sm.cmax = hi;
            }
            cluster.sync();
            lo = ~(U)0;
            hi = 0;
#pragma unroll
            for (int r = 0; r < kQcC; ++r) {
                lo = ql_min(lo, *cluster.map_shared_rank(&sm.cmin, r));
                hi = ql_max(hi, *cluster.map_shared_rank(&sm.cmax, r));
            }
        }
        if (lo == hi) {  // one key value: the segment is sorted as it stands
            if (sk != out_k + start)
                for (unsigned i = q0 + tid; i < q1; i += NT) {
                    out_k[start + i] = sk[i];
                    if constexpr (KV) out_v[start + i] = src_v[start + i];
                }
            if (me == 0) done += len;
            cluster.sync();  // the range words are read before the next item rewrites them
            continue;
        }
        // ---- 2. interpolation buckets: b = floor(d * nb / (range + 1))
        unsigned nb = min(C::NB, max(1u, (len + Q::LT - 1) / Q::LT));
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
            if (OKey<K>::of(key) < lo || OKey<K>::of(key) > hi) __trap();
#endif
            const uint32_t d = (uint32_t)((OKey<K>::of(key) - lo) >> sh);
            return mul ? __umulhi(d, mul) : d;
        };
#pragma unroll
        for (unsigned q = 0; q < BPT; ++q) sm.cnt[tid * BPT + q] = 0;
        __syncthreads();
        seg_for_each<K, NT>(sk + q0, q1 - q0, [&](K x) { atomicAdd(&sm.cnt[bucket(x)], 1u); });
        cluster.sync();  // every quarter counted, visible cluster-wide
        // ---- 3. cluster totals, bucket starts, owners, cursors
        unsigned tot[BPT], pre[BPT], sum = 0;
        bool over = false;
#pragma unroll
        for (unsigned q = 0; q < BPT; ++q) {
            const unsigned b = tid * BPT + q;
            tot[q] = 0;
            pre[q] = 0;
            if (b < nb) {
#pragma unroll
                for (int r = 0; r < kQcC; ++r) {
                    const unsigned c = cluster.map_shared_rank(sm.cnt, r)[b];
                    tot[q] += c;
                    pre[q] += (unsigned)r < me ? c : 0u;
                }
            }
            sum += tot[q];
            over |= tot[q] > wmax;
        }
        if (__syncthreads_or(over)) {
            // skewed keys: back to a sampled-pivot level (data stays in src);
            // every CTA saw the same totals
            if (me == 0 && tid == 0) {
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
            cluster.sync();  // the others are done reading this CTA's counts
            continue;
        }
        {
            unsigned total;
            unsigned ex = block_excl_scan<NT>(sum, sm.scan, &total);
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) {
                sm.st[tid * BPT + q] = ex;
                ex += tot[q];
            }
            if (tid == 0) sm.st[nb] = len;
        }
        __syncthreads();
        // owner(b) = thresholds T_c = ceil(c * len / C) (c = 1..C-1) at or
        // below the bucket's start; consecutive starts differ by <= 256 <
        // len / C, so owners step by at most one and every CTA owns a bucket
        auto owner_of = [&](unsigned s) -> unsigned {
            unsigned o = 0;
#pragma unroll
            for (int c = 1; c < kQcC; ++c) o += s * (uint64_t)kQcC >= (uint64_t)c * len ? 1u : 0u;
            return o;
        };
#pragma unroll
        for (unsigned q = 0; q < BPT; ++q) {
            const unsigned b = tid * BPT + q;
            if (b < nb) {
                const unsigned o = owner_of(sm.st[b]);
                if (b == 0 || owner_of(sm.st[b - 1]) != o) {
                    sm.first[o] = sm.st[b];
                    sm.bfirst[o] = b;
                }
            }
        }
        if (tid == 0) {
            sm.first[kQcC] = len;
            sm.bfirst[kQcC] = nb;
        }
        __syncthreads();
#pragma unroll
        for (unsigned q = 0; q < BPT; ++q) {
            const unsigned b = tid * BPT + q;
            if (b < nb) {
                const unsigned o = owner_of(sm.st[b]);
                sm.cur[b] = (o << 20) | (sm.st[b] - sm.first[o] + pre[q]);
            }
        }
        __syncthreads();
        // ---- 4. every key of this quarter into its owner's shared memory
        // (the owner's slot address: mapa of the local slot address)
        if constexpr (!KV) {
            seg_for_each_vec<K, NT>(sk + q0, q1 - q0, [&](const K* x, unsigned cn) {
                constexpr unsigned VE = 16 / sizeof(K);
                unsigned b[VE];
                bool run = cn == VE;
#pragma unroll
                for (unsigned r = 0; r < VE; ++r) {
                    b[r] = r < cn ? bucket(x[r]) : 0u;
                    run &= b[r] == b[0];
                }
                if (run) {  // a sorted run inside one bucket: one reservation
                    const unsigned c = atomicAdd(&sm.cur[b[0]], VE);
#pragma unroll
                    for (unsigned r = 0; r < VE; ++r)
                        *cluster.map_shared_rank(&sm.k[pad32((c & 0xfffffu) + r)], (int)(c >> 20)) = x[r];
                    return;
                }
                for (unsigned r = 0; r < cn; ++r) {
                    const unsigned c = atomicAdd(&sm.cur[b[r]], 1u);
                    *cluster.map_shared_rank(&sm.k[pad32(c & 0xfffffu)], (int)(c >> 20)) = x[r];
                }
            });
        } else {
            const V* sv = src_v + start;
            for (unsigned i = q0 + tid; i < q1; i += NT) {
                const K x = sk[i];
                const unsigned c = atomicAdd(&sm.cur[bucket(x)], 1u);
                const unsigned slot = pad32(c & 0xfffffu);
                *cluster.map_shared_rank(&sm.k[slot], (int)(c >> 20)) = x;
                *cluster.map_shared_rank(&sm.v[slot], (int)(c >> 20)) = sv[i];
            }
        }
        cluster.sync();  // every key landed in its owner's shared memory
        // ---- 5. sort the owned buckets in place, then one coalesced store
        const unsigned f0 = sm.first[me], b0 = sm.bfirst[me], b1 = sm.bfirst[me + 1];
        for (unsigned b = b0 + warp; b < b1; b += NT / 32) {
            const unsigned s0 = sm.st[b], cb = sm.st[b + 1] - s0;
            if (cb > 1) {
                if constexpr (KV) warp_sort_smem<K, V>(sm.k, reinterpret_cast<V*>(sm.v), s0 - f0, cb);
                else warp_sort_smem<K, V>(sm.k, (V*)nullptr, s0 - f0, cb);
            }
        }
        __syncthreads();
        const unsigned own = sm.first[me + 1] - f0;
        for (unsigned i = tid; i < own; i += NT) {
            out_k[start + f0 + i] = sm.k[pad32(i)];
            if constexpr (KV) out_v[start + f0 + i] = sm.v[pad32(i)];
        }
        if (me == 0) done += len;
        cluster.sync();  // nobody stores into this CTA's buffers before it is done
    }
    if (tid == 0 && done) atomicAdd(&ctl->loc_elems, done);
}

}  // namespace vx
