// local2.cuh -- CTA-local last partition level with the bucket-major
// intermediate STAGED IN SHARED MEMORY (north-star subsystem 3, the bottom
// of _kernels.quicksort, _kernels.py:396-423).
//
// local.cuh writes the bucket-major intermediate to the other global buffer
// (one scattered 4-byte store per key: one L1 wavefront per key, 2x the
// algorithmic DRAM writes) and reads it back for the networks.  Here the
// global levels aim the leaves at ~128 KB, so a whole leaf fits the SM's
// shared memory next to its bucket tables:
//   1. key-code range (parent's pivots, or one pass for the outer buckets);
//   2. count pass (the HBM read): interpolation buckets of ~LT keys; a bucket
//      above the leaf bound means skewed keys -> back to a sampled level;
//   3. one scan gives every bucket its output offset and its 16-byte aligned
//      stage offset; leaves larger than the stage are cut into G bucket
//      groups (G = 1 for the planned leaf size);
//   4. per group: one pass over the leaf (L2) drops every key of the group
//      at its bucket's cursor in SHARED memory; each warp then takes buckets
//      round-robin: aligned vector load from the stage, register bitonic
//      network (bitonic.cuh), sorted run back to the stage, coalesced store
//      to the output.
// DRAM traffic is the algorithmic read + write; the second read hits L2.
#pragma once

#include "bitonic.cuh"
#include "common.cuh"
#include "local.cuh"
#include "qsort.cuh"

namespace vx {

#ifndef VX_Q2_STAGE_BYTES
#define VX_Q2_STAGE_BYTES (184 * 1024)
#endif
#ifndef VX_Q2_TARGET_BYTES
#define VX_Q2_TARGET_BYTES (156 * 1024)
#endif
#ifndef VX_Q2_TARGET8_BYTES
#define VX_Q2_TARGET8_BYTES (256 * 1024)
#endif
#ifndef VX_Q2_TMIN_BYTES
#define VX_Q2_TMIN_BYTES (96 * 1024)
#endif

template <typename K, typename V>
struct Q2Cfg {
    static constexpr bool KV = HasVal<V>::value;
    static constexpr unsigned BYTES = sizeof(K) + (KV ? sizeof(V) : 0);
    // the plan aims the leaves here (at most).  4-byte keys reach it at any n
    // <= 2^32 (a sampled level of 256 buckets, then an equal-width level of
    // 511); 8-byte keys have sampled levels only (256 x 256), so their cap is
    // twice as large (two bucket groups per leaf at n = 2^31)
    static constexpr uint64_t TARGET = (sizeof(K) == 4 ? VX_Q2_TARGET_BYTES : VX_Q2_TARGET8_BYTES) / BYTES;
    static constexpr uint64_t TMIN = VX_Q2_TMIN_BYTES / BYTES;      // ... and at least here
    static constexpr unsigned SLACK = 256 + 32;                     // a group may overrun its width by one bucket (whole rows)
    static constexpr unsigned SCAP = VX_Q2_STAGE_BYTES / BYTES;     // stage slots
#ifndef VX_Q2_LT4
#define VX_Q2_LT4 107
#endif
#ifndef VX_Q2_LT8
#define VX_Q2_LT8 50
#endif
    // largest mean bucket: ~0.8 of the group network (128 slots for 4-byte
    // elements, 64 for larger ones), so few buckets overflow it.  A leaf takes
    // a whole number of ROUNDS of buckets (one bucket per lane group of the
    // CTA), so no warp idles through a partial last round; the plan's target
    // (3 rounds of 4-byte keys) sits just below a round boundary.
    static constexpr unsigned LT = BYTES <= 4 ? VX_Q2_LT4 : VX_Q2_LT8;
    static constexpr unsigned NB = 2048;                            // bucket table capacity
    static constexpr unsigned BPT = NB / kQlNT;
    static constexpr unsigned MAXG = 8;
    // network shape: GG lanes x GE registers sort one bucket of <= GP keys
    // (32 / GG buckets per warp side by side); larger buckets (<= 256) take
    // the whole warp
    static constexpr int GP = LT <= 64 ? 64 : 128;
    static constexpr int GE = BYTES <= 4 ? 16 : (BYTES <= 8 ? 8 : 4);
    static constexpr int GG = GP / GE;
    static constexpr unsigned ROUND = (kQlNT / 32) * (32 / GG);  // buckets per round
    // largest leaf taken: 3x the target, within the bucket table
    static constexpr uint64_t CAP = 3 * TARGET < (uint64_t)(NB - ROUND) * LT ? 3 * TARGET : (uint64_t)(NB - ROUND) * LT;
    // stage alignment of a bucket, in keys: one lane's slots, so a lane holds
    // either the bucket's keys (and the sentinels that fill the gap up to the
    // alignment) or nothing -- no per-slot padding tests in the networks
    static constexpr unsigned A = GE;
    static constexpr unsigned PSH = 17, PMASK = (1u << 17) - 1;  // packed scan: count in the low 17 bits, padding above
    static_assert(CAP / LT + ROUND <= NB, "bucket table too small");
    static_assert((CAP + (A - 1) * NB) / (SCAP - SLACK) + 1 <= MAXG, "too many bucket groups");
    static_assert(CAP < (1u << PSH) && (A - 1) * NB < (1u << (32 - PSH)), "packed scan fields");
};

template <typename K, typename V>
struct Q2Smem {
    using C = Q2Cfg<K, V>;
    using VS = typename std::conditional<HasVal<V>::value, V, char>::type;
    alignas(128) K k[C::SCAP + C::SLACK];
    alignas(128) VS v[HasVal<V>::value ? C::SCAP + C::SLACK : 16];
    unsigned cnt[C::NB];         // bucket sizes
    unsigned cur[C::NB];         // stage cursor: padded offset in the leaf, then the bucket's end
    unsigned short pad[C::NB];   // padded offset - output offset of the bucket
    unsigned gstart[C::MAXG + 1];  // padded offset where group g starts
    unsigned gfirst[C::MAXG + 1];  // first bucket of group g
    typename OKey<K>::U rmin[kQlNT / 32], rmax[kQlNT / 32];
    unsigned scan[kQlNT / 32 + 1];
};

// f(key, index) for every key of p[0, len): 16-byte vector loads for the
// aligned body, four vectors in flight per thread, scalar head and tail.
template <typename K, unsigned NT, typename F>
__device__ __forceinline__ void seg_for_each_idx(const K* __restrict__ p, unsigned len, F&& f) {
    constexpr unsigned VE = 16 / sizeof(K);
    union Vec {
        uint4 v;
        K k[VE];
    };
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const unsigned head = min(len, (unsigned)(((16 - (a & 15)) & 15) / sizeof(K)));
    for (unsigned i = threadIdx.x; i < head; i += NT) f(p[i], i);
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
            for (unsigned r = 0; r < VE; ++r) f(w[u].k[r], head + (j + u * NT) * VE + r);
    }
    for (; j < nv; j += NT) {
        Vec w;
        w.v = v[j];
#pragma unroll
        for (unsigned r = 0; r < VE; ++r) f(w.k[r], head + j * VE + r);
    }
    for (unsigned i = head + nv * VE + threadIdx.x; i < len; i += NT) f(p[i], i);
}

// Stage swizzle: the networks read a bucket blocked -- lane g of a group
// takes 64 consecutive bytes -- which would put the 8 lanes of one LDS.128
// phase on two 16-byte bank groups.  XOR-ing the 16-byte chunk index inside
// each 128-byte row with the row's low two bits spreads them over all eight.
template <typename K>
__device__ __forceinline__ unsigned q2_sw(unsigned p) {
    constexpr unsigned LA = sizeof(K) == 4 ? 2 : 1;  // log2(keys per 16-byte chunk)
    return p ^ (((p >> (LA + 3)) & 3u) << LA);
}
__device__ __forceinline__ unsigned q2_swc(unsigned c) { return c ^ ((c >> 3) & 3u); }  // chunk form

// The buckets of a warp's groups through G-lane register networks, in place
// in the (swizzled) stage: group lane gl holds slots gl*E .. gl*E+E-1 of its
// group's bucket at stage slot ps (16-byte aligned), cb <= G*E keys (cb = 0:
// the group idles).  Fewer lanes and more registers per network turn
// cross-lane rounds (a shuffle per slot) into in-register ones.
template <typename K, typename V, int E, int G, unsigned AL>
__device__ __forceinline__ void stage_sort_group(K* stage_k, V* stage_v, unsigned ps, unsigned cb) {
    constexpr bool KV = HasVal<V>::value;
    using R = KeyRep<K>;
    using I = typename R::I;
    constexpr int VE = 16 / sizeof(K);  // keys per 16-byte chunk
    constexpr int NV = E / VE;          // chunks per lane
    static_assert(E % VE == 0, "whole chunks per lane");
    const unsigned gl = threadIdx.x & (G - 1);
    struct alignas(16) KP { K x[VE]; };
    struct alignas(16) VP { typename std::conditional<KV, V, K>::type x[VE]; };
    const unsigned c0 = ps / VE + gl * NV;
    I k[E];
    V v[E];
    // the bucket's slots end at the next multiple of AL keys (sentinel-filled
    // past cb); lanes beyond hold sentinels only
#pragma unroll
    for (int r = 0; r < E; ++r) k[r] = KeyTraits<I>::sentinel();
    if (gl * E < (cb + AL - 1) / AL * AL) {
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            const unsigned pc = q2_swc(c0 + u);
            const KP t = reinterpret_cast<const KP*>(stage_k)[pc];
#pragma unroll
            for (int r = 0; r < VE; ++r) k[u * VE + r] = R::to(t.x[r]);
            if constexpr (KV) {
                const VP tv = reinterpret_cast<const VP*>(stage_v)[pc];
#pragma unroll
                for (int r = 0; r < VE; ++r) v[u * VE + r] = tv.x[r];
            }
        }
    }
    WarpBitonic<I, V, E, G, true>::sort(k, v);
    __syncwarp();  // every lane has read its slots
    // (chunks past the bucket's padded end belong to the next bucket)
#pragma unroll
    for (int u = 0; u < NV; ++u) {
        if (gl * E + u * VE < cb) {
            const unsigned pc = q2_swc(c0 + u);
            KP t;
#pragma unroll
            for (int r = 0; r < VE; ++r) t.x[r] = R::from(k[u * VE + r]);
            reinterpret_cast<KP*>(stage_k)[pc] = t;
            if constexpr (KV) {
                VP tv;
#pragma unroll
                for (int r = 0; r < VE; ++r) tv.x[r] = v[u * VE + r];
                reinterpret_cast<VP*>(stage_v)[pc] = tv;
            }
        }
    }
    __syncwarp();
}

// a sorted bucket from the stage to the output, consecutive lanes on
// consecutive elements
template <typename K, typename V>
__device__ __forceinline__ void stage_copy_out(const K* stage_k, const V* stage_v, unsigned ps, unsigned cb,
                                               K* __restrict__ ok, V* __restrict__ ov) {
    for (unsigned j = threadIdx.x & 31; j < cb; j += 32) {
        const unsigned p = q2_sw<K>(ps + j);
        ok[j] = stage_k[p];
        if constexpr (HasVal<V>::value) ov[j] = stage_v[p];
    }
}

template <typename K, typename V>
__global__ void __launch_bounds__(kQlNT, 1) qs_local2_kernel(const QlItem* __restrict__ items, Ctl* __restrict__ ctl,
                                                             Ctl* __restrict__ ctl_next, Seg* __restrict__ next_segs,
                                                             unsigned cap_seg, const K* __restrict__ src_k,
                                                             const V* __restrict__ src_v, K* __restrict__ oth_k,
                                                             V* __restrict__ oth_v, K* __restrict__ out_k,
                                                             V* __restrict__ out_v, unsigned leaf) {
    using C = Q2Cfg<K, V>;
    using U = typename OKey<K>::U;
    constexpr bool KV = HasVal<V>::value;
    constexpr unsigned NT = kQlNT, BPT = C::BPT, A = C::A;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Q2Smem<K, V>& sm = *reinterpret_cast<Q2Smem<K, V>*>(smem_raw);
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
        // ---- 2. interpolation buckets: b = floor(d * nb / (range + 1))
        unsigned nb = min(C::NB, (len + C::ROUND * C::LT - 1) / (C::ROUND * C::LT) * C::ROUND);
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
        // (result unused: ATOMS.POPC.INC merges a warp's same-counter lanes)
        seg_for_each<K, NT>(sk, len, [&](K x) { atomicAdd(&sm.cnt[bucket(x)], 1u); });
        __syncthreads();
        VX_QL_TICK(1);
        // ---- 3. offsets: one scan of (pad << C::PSH | count) per thread
        unsigned c[BPT], sum = 0;
        bool over = false;
#pragma unroll
        for (unsigned q = 0; q < BPT; ++q) {
            c[q] = sm.cnt[tid * BPT + q];
            sum += c[q] + ((((A - c[q] % A) % A)) << C::PSH);
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
        unsigned G, W;
        unsigned pbq[BPT];  // padded offsets of this thread's buckets
        {
            unsigned tot;
            unsigned ex = block_excl_scan<NT>(sum, sm.scan, &tot);
            const unsigned ptotal = (tot & C::PMASK) + (tot >> C::PSH);
            G = ptotal <= C::SCAP ? 1u : (ptotal + (C::SCAP - C::SLACK) - 1) / (C::SCAP - C::SLACK);
            W = G == 1 ? 0xffffffffu : ((ptotal + G - 1) / G + A - 1) / A * A;
            // the previous bucket's padded offset decides whether a bucket opens a group
            unsigned prevp = 0;
            if (tid > 0) {
                const unsigned cp = sm.cnt[tid * BPT - 1];
                prevp = (ex & C::PMASK) + (ex >> C::PSH) - (cp + (A - cp % A) % A);
            }
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) {
                const unsigned b = tid * BPT + q;
                const unsigned pb = (ex & C::PMASK) + (ex >> C::PSH);
                pbq[q] = pb;
                sm.cur[b] = pb;
                sm.pad[b] = (unsigned short)(ex >> C::PSH);
                if (b < nb && (b == 0 || prevp / W != pb / W)) {
                    sm.gstart[pb / W] = pb;
                    sm.gfirst[pb / W] = b;
                }
                prevp = pb;
                ex += c[q] + ((((A - c[q] % A) % A)) << C::PSH);
            }
            if (tid == 0) {
                sm.gstart[G] = ptotal;
                sm.gfirst[G] = nb;
            }
        }
        __syncthreads();
        VX_QL_TICK(2);
        // a leaf sorted in place in G > 1 groups: the groups before the last
        // still have readers of the source, so their runs detour through the
        // other buffer and come home after the last group's pass
        const bool detour = G > 1 && src_k == out_k;
        for (unsigned g = 0; g < G; ++g) {
            K* ok = (detour && g + 1 < G ? oth_k : out_k) + start;
            V* ov = KV ? (detour && g + 1 < G ? oth_v : out_v) + start : nullptr;
            const unsigned gs = sm.gstart[g], b_lo = sm.gfirst[g], nbg = sm.gfirst[g + 1] - b_lo;
            // sentinels into the gap between each bucket's end and its aligned end
#pragma unroll
            for (unsigned q = 0; q < BPT; ++q) {
                const unsigned b = tid * BPT + q;
                if (b - b_lo < nbg)
                    for (unsigned j = c[q]; j < (c[q] + A - 1) / A * A; ++j)
                        sm.k[q2_sw<K>(pbq[q] - gs + j)] = KeyTraits<K>::sentinel();
            }
            // ---- 4a. every key of the group to its bucket's cursor in the stage
            if (G == 1) {
                if constexpr (!KV) {
                    seg_for_each_vec<K, NT>(sk, len, [&](const K* x, unsigned n) {
                        if (n == 1) {
                            sm.k[q2_sw<K>(atomicAdd(&sm.cur[bucket(x[0])], 1u))] = x[0];
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
                            const unsigned p0 = atomicAdd(&sm.cur[b[0]], VE);
#pragma unroll
                            for (unsigned r = 0; r < VE; ++r) sm.k[q2_sw<K>(p0 + r)] = x[r];
                            return;
                        }
#pragma unroll
                        for (unsigned r = 0; r < VE; ++r) sm.k[q2_sw<K>(atomicAdd(&sm.cur[b[r]], 1u))] = x[r];
                    });
                } else {
                    const V* svp = src_v + start;
                    seg_for_each_idx<K, NT>(sk, len, [&](K x, unsigned i) {
                        const V y = svp[i];
                        const unsigned p = q2_sw<K>(atomicAdd(&sm.cur[bucket(x)], 1u));
                        sm.k[p] = x;
                        sm.v[p] = y;
                    });
                }
            } else {
                const V* svp = KV ? src_v + start : nullptr;
                seg_for_each_idx<K, NT>(sk, len, [&](K x, unsigned i) {
                    const unsigned b = bucket(x);
                    if (b - b_lo < nbg) {
                        const unsigned p = q2_sw<K>(atomicAdd(&sm.cur[b], 1u) - gs);
                        sm.k[p] = x;
                        if constexpr (KV) sm.v[p] = svp[i];
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
            // ---- 4b. every bucket of the group through the bitonic network
            {
                constexpr int GG = C::GG, GE = C::GE, NG = 32 / GG;
                V* stv = KV ? reinterpret_cast<V*>(sm.v) : nullptr;
                const unsigned grp = lane / GG;
                for (unsigned b0 = b_lo + warp * NG; b0 < b_lo + nbg; b0 += (NT / 32) * NG) {
                    const unsigned b = b0 + grp;
                    unsigned cb = 0, ps = 0, ob = 0;
                    if (b < b_lo + nbg) {
                        cb = sm.cnt[b];
                        const unsigned pend = sm.cur[b];  // the cursor ended at the bucket's end
                        ps = pend - cb - gs;              // its stage slot (16-byte aligned)
                        ob = pend - cb - sm.pad[b];       // its offset in the sorted leaf
                    }
                    const bool big = cb > (unsigned)C::GP;
                    stage_sort_group<K, V, GE, GG, C::A>(sm.k, stv, ps, big ? 0u : cb);
                    // the rare bucket above the group network takes the whole warp
                    unsigned bm = __ballot_sync(0xffffffffu, big && (lane % GG) == 0);
                    while (bm) {
                        const int src = __ffs(bm) - 1;
                        bm &= bm - 1;
                        const unsigned cbb = __shfl_sync(0xffffffffu, cb, src);
                        const unsigned psb = __shfl_sync(0xffffffffu, ps, src);
                        if (C::GP < 128 && cbb <= 128) stage_sort_group<K, V, 128 / 32, 32, C::A>(sm.k, stv, psb, cbb);
                        else stage_sort_group<K, V, 256 / 32, 32, C::A>(sm.k, stv, psb, cbb);
                    }
#pragma unroll
                    for (int i = 0; i < NG; ++i) {
                        const unsigned cbi = __shfl_sync(0xffffffffu, cb, i * GG);
                        const unsigned psi = __shfl_sync(0xffffffffu, ps, i * GG);
                        const unsigned obi = __shfl_sync(0xffffffffu, ob, i * GG);
                        stage_copy_out<K, V>(sm.k, stv, psi, cbi, ok + obi, KV ? ov + obi : nullptr);
                    }
                }
            }
            __syncthreads();
            VX_QL_TICK(4);
        }
        if (detour) {
            const unsigned bl = sm.gfirst[G - 1];
            const unsigned n1 = sm.gstart[G - 1] - sm.pad[bl];  // output offset of the last group
            for (unsigned i = tid; i < n1; i += NT) {
                out_k[start + i] = oth_k[start + i];
                if constexpr (KV) out_v[start + i] = oth_v[start + i];
            }
            __syncthreads();
        }
        done += len;
    }
    if (tid == 0 && done) atomicAdd(&ctl->loc_elems, done);
}

}  // namespace vx
