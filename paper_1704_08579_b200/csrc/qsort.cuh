// qsort.cuh -- device-side hybrid quicksort driver (north-star subsystem 3)
// and the k-way bucket partition (subsystem 4's partition step).
//
// Reference algorithm: _kernels.quicksort (_kernels.py:378-423) -- pick a
// pivot, partition, recurse on both sides, hand ranges <= sort_bound to the
// bitonic small sort.  The GPU keeps that structure but partitions each
// range around MANY sampled pivots at once (a multi-pivot quicksort / sample
// sort step) so the number of HBM passes is ~log_256(n) instead of log_2(n):
//
//   level loop (work queue of segments in device memory, ping-pong buffers)
//     qs_plan     one CTA per segment: sample, sort the sample in smem, pick
//                 up to 255 distinct pivots (= splitters), allocate bucket /
//                 tile slots with atomics
//     qs_hist     persistent CTAs over the level's tiles: classify each
//                 element into 2m+1 buckets (ranges + "equal to pivot"
//                 buckets), per-segment histograms
//     qs_emit     one CTA per segment: scan the histogram into bucket cursors
//                 and enqueue children: big -> next level, <= LOCAL_MAX ->
//                 finish queue, equal-to-pivot / singletons -> final
//     qs_scatter  persistent CTAs over tiles: classify again, rank inside the
//                 tile, reserve a run per bucket with one atomic, stage the
//                 tile in smem bucket-major and write runs coalesced
//     qs_finish   one CTA per finish item: CTA-local hybrid quicksort in
//                 shared memory (one more sampled multi-pivot partition, then
//                 the warp bitonic network on every range <= 256) straight
//                 into the output; or a chunked copy for final buckets that
//                 sit in the scratch buffer.
//
// The equal-to-pivot buckets are final (all keys equal), which removes the
// reference's quadratic behaviour on few-unique / sorted / reverse inputs
// (SURVEY.md section 0 finding 5) without changing the (unique) output.
#pragma once

#include "bitonic.cuh"
#include "common.cuh"

namespace vx {

constexpr int kMaxSplit = 255;                 // pivots per segment (level)
constexpr int kMaxBkt = 2 * kMaxSplit + 1;     // 511 buckets
#ifndef VX_QS_NT
#define VX_QS_NT 512
#endif
constexpr int kQsNT = VX_QS_NT;                // tile-kernel threads (tile = kQsNT * 8)
#ifndef VX_QS_SM_THREADS
#define VX_QS_SM_THREADS 1024
#endif
constexpr int kQsMinBlocks = VX_QS_SM_THREADS / kQsNT;  // resident tile-kernel threads per SM (register cap)
constexpr int kPlanNT = 512;                   // plan / emit threads
constexpr int kFinNT = 512;                    // finish-kernel threads
constexpr int kMaxSample = 4096;
constexpr int kFinSample = 1024;
constexpr uint32_t kCopyChunk = 16384;
// Bucket b of a segment counts (histogram) and reserves its runs (scatter)
// at bkt_pool[bkt_off + (b << cshift)].  Every tile of a level hits these
// cursors with one atomic per bucket, and L2 serialises atomics that share a
// 32-byte sector.  The equal-width ROOT level has a few hundred cursors side
// by side that every CTA of the GPU hammers: four per sector cost the 2^32
// int32 sort 7.7 ms (scatter 40.2 vs 32.5 ms), so they sit four slots apart,
// one per sector.  Later levels spread their atomics over hundreds of
// segments; spacing their cursors out only costs cache lines (measured: +1.1
// ms), and a sampled level's range buckets already sit two apart.
#ifndef VX_ROOT_CSHIFT
#define VX_ROOT_CSHIFT 2
#endif
constexpr unsigned kRootBktSlots = 512u << VX_ROOT_CSHIFT;  // pool slots the root level may take
constexpr int kMaxLevels = 48;
constexpr double kQlSlack = 2.0;  // global levels aim CTA-local leaves at <= this x the target

template <typename K>
#ifndef VX_QS_IPT
#define VX_QS_IPT 8
#endif
struct QsTile { static constexpr int IPT = VX_QS_IPT; };  // 4096-element tiles by default
template <typename K>
constexpr int qs_tile() { return kQsNT * QsTile<K>::IPT; }

// Elements a finish CTA sorts in shared memory (keys + payload, x2 buffers).
template <typename K, typename V>
struct FinCap {
    static constexpr uint32_t bytes_per = sizeof(K) + (HasVal<V>::value ? sizeof(V) : 0);
    // a multiple of the finish CTA (512 threads); sized so one partition
    // level of <= 255 pivots takes ~1M-element ranges below it
    static constexpr uint32_t value = bytes_per <= 4 ? 8192 : (bytes_per <= 8 ? 6144 : 3072);
};

// A level segment.  mode 0: partitioned around m sampled pivots into
// nb = 2m+1 buckets (ranges and equal-to-pivot buckets).  mode 1 (a segment
// whose key-code bounds [lo, hi] are known from its parent, 4-byte keys): nb
// equal-width buckets over [lo, hi], bucket = umulhi(code - lo, mul) with
// mul = floor(nb * 2^32 / (hi - lo + 1)) -- evenly spaced pivots, classified
// with a subtract and a high multiply (mul = 0: one code per bucket).
// mode 2 (the same for float64 keys): nb equal-width buckets in VALUE space,
// bucket = min(nb - 1, trunc((x - vlo) * vinv)) -- float64 codes change
// density at every binade, values of locally uniform keys do not.
struct Seg {
    unsigned long long start, len;
    unsigned spl_off, m, bkt_off, tile_base;
    unsigned long long lo, hi;  // key-code bounds (lo > hi: unknown)
    unsigned nb;
    unsigned direct;  // set by emit: every bucket is final, the scatter writes straight into the output
    unsigned mode, mul;
    double vlo, vinv;  // mode 2
    unsigned cshift;  // bucket b's counter / cursor is bkt_pool[bkt_off + (b << cshift)]
    unsigned open;    // root over the SAMPLE's extremes [lo, hi]: keys beyond them sit in the edge buckets
};
struct QlItemT {  // a segment for the CTA-local level (local.cuh)
    unsigned long long start, len;
    unsigned long long lo, hi;  // key-code bounds from the parent's pivots (lo > hi: unknown)
};
struct Fin {
    unsigned long long start;
    unsigned len, flags;  // bit0: source is the scratch buffer; bit1: copy only
};
// Per-level control record.  A sort keeps three in its workspace: the
// current level's, the next level's (its queue sizes, filled by this level's
// emit / finish / local kernels) and the running totals; qs_advance_kernel
// folds a finished level into the totals, clears its record for reuse two
// levels later and decides whether another level runs (tot.more).
struct Ctl {
    unsigned nseg;      // segments in this level's queue
    unsigned spl_ctr, bkt_ctr, tile_ctr, fin_ctr;
    unsigned err;
    unsigned long long scat_elems;  // elements moved by this level's scatter
    unsigned long long fin_elems;   // elements finished (sorted / copied) at this level
    unsigned long long loc_elems;   // elements sorted by the CTA-local level (local.cuh)
    unsigned ql_ctr;                // CTA-local segments queued by this level's emit
    unsigned level;                 // totals: levels completed (level seeds follow it)
    unsigned more;                  // totals: another level is needed
    unsigned launches;              // totals: kernels launched by the completed levels
};
static_assert(sizeof(Ctl) == 64, "Ctl is one 64-byte record");
enum : unsigned { kErrCapacity = 1, kErrTooLong = 2, kErrLevels = 4, kErrOffsets = 8 };

// ------------------------------------------------------------ classifiers
// ---------------------------------------------------- cell-table classifier
// Keys as order-preserving unsigned codes: int32 -> uint32 (sign bit
// flipped), float64 -> the uint64 code of KeyRep<double>.
template <typename K>
struct OKey;
template <>
struct OKey<int32_t> {
    using U = uint32_t;
    __device__ __forceinline__ static U of(int32_t k) { return (uint32_t)k ^ 0x80000000u; }
};
template <>
struct OKey<double> {
    using U = uint64_t;
    __device__ __forceinline__ static U of(double k) { return f64_to_ord(k); }
};

constexpr int kLutBits = 13;  // 8192 cells

// Per-segment classification table: the sorted splitters plus a 2^LB-cell
// lookup table over [lo, hi] (the smallest / largest splitter).  Cell c
// covers codes [lo + c<<shift, lo + (c+1)<<shift); lut[c] packs
// (#splitters below the cell) | (#splitters inside the cell) << 8, so a key
// is classified with one table load and, only when splitters share its
// cell, a compare or a short search over those few.  (Measured against a
// binary search over the sorted splitters -- every upper-level probe lands in
// the same shared-memory bank -- and an Eytzinger-order search; the table is
// fewer instructions and conflict-free.)
template <typename U, int NSPL, int LB>
struct CellTableT {
    static constexpr int kBits = LB;
    U spl[NSPL];
    unsigned short lut[1 << LB];
};
template <typename U>
using CellTable = CellTableT<U, 256, kLutBits>;
// Cell map: code-linear (cell = (code - lo) >> shift) or, for float64 keys
// whose splitters crowd a few code cells (e.g. uniform values spanning
// several binades), value-linear (cell = (v - vlo) * vscale).  Either map is
// monotone, which is all the table needs.
template <typename U>
struct CellParams {
    U lo, hi;
    unsigned shift, m, ncell, vmode;
    double vlo, vscale;
};

template <typename U>
__device__ __forceinline__ unsigned lower_bound_u(const U* a, unsigned lo, unsigned cnt, U x) {
    while (cnt > 0) {
        const unsigned half = cnt >> 1;
        if (a[lo + half] < x) {
            lo += half + 1;
            cnt -= half + 1;
        } else {
            cnt = half;
        }
    }
    return lo;
}

// Load m (>= 1) sorted splitters from the pool and build the table.  All
// threads of the CTA must call it; contains barriers.  `scan` is block-scan
// scratch (NT/32 + 1 words).
template <int NT, bool kTryValue = true, typename U, int NSPL, int LB>
__device__ CellParams<U> ct_build(CellTableT<U, NSPL, LB>& ct, unsigned m, unsigned* scan);

template <typename K, int NT>
__device__ CellParams<typename OKey<K>::U> ct_load(CellTable<typename OKey<K>::U>& ct, const K* spl_pool,
                                                   unsigned off, unsigned m, unsigned* scan) {
    for (unsigned i = threadIdx.x; i < m; i += NT) ct.spl[i] = OKey<K>::of(spl_pool[off + i]);
    __syncthreads();
    return ct_build<NT>(ct, m, scan);
}

template <typename U>
__device__ __forceinline__ unsigned cell_code(const CellParams<U>& p, U x) {
    const U d = x > p.lo ? x - p.lo : (U)0;
    const U c64 = d >> p.shift;
    return c64 < (U)p.ncell ? (unsigned)c64 : p.ncell - 1;
}
template <typename U>
__device__ __forceinline__ unsigned cell_val(const CellParams<U>& p, double v) {
    double t = (v - p.vlo) * p.vscale;  // NaN keys are unsupported (as in the reference)
    t = t > 0.0 ? t : 0.0;
    return t < (double)(p.ncell - 1) ? (unsigned)t : p.ncell - 1;
}

// Build the lookup table of a table whose m (1 <= m <= 255) sorted splitters
// are already in ct.spl (visible to all threads).  Counting construction:
// every splitter bumps its cell's count (16-bit halves of the table words),
// then one block scan over the cells turns counts into "#splitters below the
// cell" -- no per-cell search.  For 64-bit codes (float64 keys) a crowded
// code map (sum of squared cell counts well above m) is retried value-linear
// and the less crowded map is kept (kTryValue).  Ends with a barrier.
template <int NT, bool kTryValue, typename U, int NSPL, int LB>
__device__ CellParams<U> ct_build(CellTableT<U, NSPL, LB>& ct, unsigned m, unsigned* scan) {
    constexpr int NC = 1 << LB;
    static_assert(NC >= NT && NC % NT == 0, "cells must cover the CTA evenly");
    constexpr int CPT = NC / NT;
    CellParams<U> p;
    p.m = m;
    p.vmode = 0;
    p.vlo = 0.0;
    p.vscale = 0.0;
    p.lo = ct.spl[0];
    p.hi = ct.spl[m - 1];
    const U range = p.hi - p.lo;
    const unsigned bits = range == 0 ? 0u : (unsigned)(8 * sizeof(U)) - (sizeof(U) == 8 ? __clzll((long long)range)
                                                                                      : __clz((int)range));
    p.shift = bits > LB ? bits - LB : 0u;
    p.ncell = (unsigned)(range >> p.shift) + 1;
    unsigned* w = reinterpret_cast<unsigned*>(ct.lut);
    const unsigned c0 = threadIdx.x * CPT;
    unsigned cnt[CPT], sum = 0, sq = 0;
    auto count = [&]() {  // per-cell splitter counts of the current map into cnt[]
        for (unsigned i = threadIdx.x; i < NC / 2; i += NT) w[i] = 0u;
        __syncthreads();
        for (unsigned i = threadIdx.x; i < m; i += NT) {
            unsigned c;
            if constexpr (sizeof(U) == 8) c = p.vmode ? cell_val(p, ord_to_f64(ct.spl[i])) : cell_code(p, ct.spl[i]);
            else c = cell_code(p, ct.spl[i]);
            atomicAdd(&w[c >> 1], 1u << (16 * (c & 1u)));
        }
        __syncthreads();
        sum = 0;
        sq = 0;
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            cnt[j] = ct.lut[c0 + j];
            sum += cnt[j];
            sq += cnt[j] * cnt[j];
        }
    };
    count();
    if constexpr (sizeof(U) == 8 && kTryValue) {
        unsigned sq_code;
        block_excl_scan<NT>(sq, scan, &sq_code);
        const double vlo = ord_to_f64(p.lo), vhi = ord_to_f64(p.hi), span = vhi - vlo;
        if (sq_code > m + m / 8 && span > 0.0 && span <= 1.7e308) {
            const unsigned code_ncell = p.ncell;
            p.vmode = 1;
            p.vlo = vlo;
            p.vscale = (double)(NC - 1) / span;
            p.ncell = NC;
            p.ncell = cell_val(p, vhi) + 1;  // the last cell holds hi
            count();
            unsigned sq_val;
            block_excl_scan<NT>(sq, scan, &sq_val);
            if (sq_val >= sq_code) {  // no better: back to the code map
                p.vmode = 0;
                p.ncell = code_ncell;
                count();
            }
        }
    }
    unsigned tot;
    unsigned below = block_excl_scan<NT>(sum, scan, &tot);  // ends with a barrier
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        ct.lut[c0 + j] = (unsigned short)(below | (cnt[j] << 8));  // m <= 255: 8 | 8 bits
        below += cnt[j];
    }
    __syncthreads();
    return p;
}

// bucket = 2*lb + (x == spl[lb]), lb = #splitters < x (equality buckets odd)
// Keys below lo / above hi clamp into the first / last cell, whose splitter
// lists contain lo / hi, so no separate branches are needed.  With at most
// one splitter in the key's cell the answer is branch-free: s = spl[lbmin]
// is that splitter, or -- empty cell -- the first splitter above the cell,
// which is > x (every reachable empty cell lies below the last cell, so
// lbmin <= m-1 and s exists).  Only cells holding >= 2 splitters search.
template <typename U, int NSPL, int LB>
__device__ __forceinline__ unsigned ct_classify_cell(const CellTableT<U, NSPL, LB>& ct, const CellParams<U>& p, U x,
                                                     unsigned c) {
    const unsigned e = ct.lut[c];
    unsigned lb = e & 0xffu;
#ifdef VX_CLS_BRANCHY
    const unsigned cnt = e >> 8;
    if (cnt == 0) return 2 * lb;
    if (cnt == 1) {
        const U s = ct.spl[lb];
        return 2 * (lb + (unsigned)(s < x)) + (unsigned)(s == x);
    }
#else
    if (e < (2u << 8)) {
        const U s = ct.spl[lb];
        return 2 * (lb + (unsigned)(s < x)) + (unsigned)(s == x);
    }
#endif
    lb = lower_bound_u(ct.spl, lb, e >> 8, x);
    return 2 * lb + (unsigned)(lb < p.m && ct.spl[lb] == x);
}

// classify a key (int32 / float64) against a table built by ct_build
template <typename K, typename U, int NSPL, int LB>
__device__ __forceinline__ unsigned ct_classify(const CellTableT<U, NSPL, LB>& ct, const CellParams<U>& p, K key) {
    const U x = OKey<K>::of(key);
    if constexpr (sizeof(K) == 8) {
        const unsigned c = p.vmode ? cell_val(p, (double)key) : cell_code(p, x);
        return ct_classify_cell(ct, p, x, c);
    } else {
        return ct_classify_cell(ct, p, x, cell_code(p, x));
    }
}

// (key, global index) classifier for the sharded sort: bucket = number of
// splitters lexicographically below (x, gi); ties between equal keys are
// broken by global index, which keeps few-unique inputs balanced.
template <typename K>
__device__ __forceinline__ unsigned cls_idx(K x, uint64_t gi, const K* spk, const uint64_t* spi, unsigned m) {
    unsigned lo = 0, hi = m;
    while (lo < hi) {
        const unsigned mid = (lo + hi) >> 1;
        const bool below = (spk[mid] < x) || (!(x < spk[mid]) && spi[mid] < gi);
        if (below) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// --------------------------------------------------- smem bitonic (CTA-wide)
// Plain ascending bitonic sort of P (pow2) keys (+payload) in shared memory.
template <typename K, typename V, int NT>
__device__ __forceinline__ void cta_bitonic(K* a, V* av, unsigned P) {
    constexpr bool KV = HasVal<V>::value;
    for (unsigned k = 2; k <= P; k <<= 1) {
        for (unsigned j = k >> 1; j > 0; j >>= 1) {
            for (unsigned i = threadIdx.x; i < P; i += NT) {
                const unsigned ixj = i ^ j;
                if (ixj > i) {
                    const K x = a[i], y = a[ixj];
                    const bool asc = (i & k) == 0;
                    if (asc ? (y < x) : (x < y)) {
                        a[i] = y;
                        a[ixj] = x;
                        if constexpr (KV) {
                            V t = av[i];
                            av[i] = av[ixj];
                            av[ixj] = t;
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
}

#ifndef VX_PLAN_MERGE
#define VX_PLAN_MERGE 1
#endif
// Sort S (pow2, 256..4096) samples in shared memory with the CTA: each warp
// sorts a 256-sample chunk in registers (the warp bitonic network), then
// every sample's global rank is its position in its chunk plus its
// lower/upper bound in every other chunk (ties broken by chunk), and the
// samples move to their ranks.  One network pass and one merge instead of
// log^2(S) CTA-wide compare-exchange rounds.
template <typename K>
__device__ __forceinline__ void plan_sort_samples(K* s, unsigned S) {
    constexpr unsigned C = 256, E = C / 32, MAXW = kMaxSample / C;
    static_assert(kPlanNT / 32 >= MAXW, "one warp per chunk");
    const unsigned W = S / C, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < W) {
        K k[E];
        NoVal v[E];
#pragma unroll
        for (unsigned r = 0; r < E; ++r) k[r] = s[warp * C + lane * E + r];
        WarpBitonic<K, NoVal, E>::sort(k, v);
#pragma unroll
        for (unsigned r = 0; r < E; ++r) s[warp * C + lane * E + r] = k[r];
    }
    __syncthreads();
    if (W == 1) return;
#if VX_PLAN_MERGE
    // pairwise merges of sorted runs (256 -> 512 -> ... -> S), in place: each
    // sample's merged position is its index in its run plus its rank in the
    // partner run (lower run first on ties: count(< v) for a lower-run
    // sample, count(<= v) for an upper-run one), found by a fixed-step search
    // -- log2(run) steps per sample per round instead of 8 per other chunk
    constexpr unsigned PER = kMaxSample / kPlanNT;
    const unsigned per = (S + kPlanNT - 1) / kPlanNT;  // samples this thread really moves
    for (unsigned run = C; run < S; run *= 2) {
        K val[PER];
        unsigned dst[PER], lo[PER];
        const K* oth[PER];
        bool up[PER];
#pragma unroll
        for (unsigned q = 0; q < PER; ++q) {
            const unsigned i = min(q * kPlanNT + threadIdx.x, S - 1);
            const unsigned base = i & ~(2 * run - 1);
            up[q] = (i & run) != 0;
            val[q] = s[i];
            oth[q] = s + base + (up[q] ? 0u : run);
            dst[q] = base + (i & (run - 1));
            lo[q] = 0;
        }
        for (unsigned step = run / 2; step > 0; step >>= 1) {
#pragma unroll
            for (unsigned q = 0; q < PER; ++q) {
                if (q >= per) break;
                const K e = oth[q][lo[q] + step - 1];
                const bool before = up[q] ? !(val[q] < e) : (e < val[q]);
                lo[q] += before ? step : 0u;
            }
        }
#pragma unroll
        for (unsigned q = 0; q < PER; ++q) {
            if (q >= per) break;
            const K e = oth[q][lo[q]];  // lo <= run - 1 here
            const bool before = up[q] ? !(val[q] < e) : (e < val[q]);
            dst[q] += lo[q] + (before ? 1u : 0u);
        }
        __syncthreads();
#pragma unroll
        for (unsigned q = 0; q < PER; ++q)
            if (q * kPlanNT + threadIdx.x < S) s[dst[q]] = val[q];
        __syncthreads();
    }
#else
    // every thread ranks its PER samples in lockstep: fixed-step branch-free
    // searches, PER independent shared loads per step (the CTA is alone on
    // its SM at level 0, so latency is hidden by ILP, not by other warps)
    constexpr unsigned PER = kMaxSample / kPlanNT;
    const unsigned per = (S + kPlanNT - 1) / kPlanNT;  // samples this thread really ranks
    K val[PER];
    unsigned rk[PER], ch_of[PER];
#pragma unroll
    for (unsigned q = 0; q < PER; ++q) {
        const unsigned i = min(q * kPlanNT + threadIdx.x, S - 1);
        val[q] = s[i];
        ch_of[q] = i / C;
        rk[q] = i % C;
    }
    for (unsigned o = 0; o < W; ++o) {
        const K* ch = s + o * C;
        unsigned lo[PER];
#pragma unroll
        for (unsigned q = 0; q < PER; ++q) lo[q] = 0;
        // o < c: count(<= v); o > c: count(< v) -- ties ordered by chunk
#pragma unroll
        for (unsigned step = C / 2; step > 0; step >>= 1) {
#pragma unroll
            for (unsigned q = 0; q < PER; ++q) {
                if (q >= per) break;
                const K e = ch[lo[q] + step - 1];
                const bool before = o < ch_of[q] ? !(val[q] < e) : (e < val[q]);
                lo[q] += before ? step : 0u;
            }
        }
#pragma unroll
        for (unsigned q = 0; q < PER; ++q) {
            if (q >= per) break;
            const K e = ch[lo[q]];  // lo <= C - 1 here
            const bool before = o < ch_of[q] ? !(val[q] < e) : (e < val[q]);
            if (o != ch_of[q]) rk[q] += lo[q] + (before ? 1u : 0u);
        }
    }
    __syncthreads();
#pragma unroll
    for (unsigned q = 0; q < PER; ++q)
        if (q * kPlanNT + threadIdx.x < S) s[rk[q]] = val[q];
    __syncthreads();
#endif
}

// ------------------------------------------------------------ init
// Clears the three control records and queues the whole array: one level
// segment, or (n <= the finish capacity) one finish item whose source is the
// input (root_flags bit0).
__global__ void qs_init_kernel(Seg* segs, Ctl* ctl, Fin* fins, unsigned long long n, unsigned as_fin,
                               unsigned root_flags, unsigned* presort_flags) {
    unsigned* w = reinterpret_cast<unsigned*>(ctl);
    for (unsigned i = threadIdx.x; i < 3 * sizeof(Ctl) / 4; i += blockDim.x) w[i] = 0u;
    if (threadIdx.x < 2) presort_flags[threadIdx.x] = 0u;  // presort.cuh (the tile map's first words, free until the plan)
    __syncthreads();
    if (threadIdx.x == 0) {
        if (as_fin) {
            fins[0].start = 0;
            fins[0].len = (unsigned)n;
            fins[0].flags = root_flags;
            ctl[0].fin_ctr = 1;
        } else {
            segs[0].start = 0;
            segs[0].len = n;
            segs[0].lo = 1;
            segs[0].hi = 0;
            ctl[0].nseg = 1;
        }
    }
}

// Level seed: the sort's seed mixed with the number of completed levels.
__device__ __forceinline__ uint64_t level_seed(uint64_t seed, const Ctl* tot) {
    return mix64(seed + 0x51ED270B27AD1CULL * (tot->level + 1));
}

// After every kernel of a level: fold its record c into the totals, flag a
// level-count overflow, clear c (it serves as the "next" record two levels
// on) and decide whether another level is needed.  In a CUDA graph it also
// sets the level loop's condition (set_cond).
__global__ void qs_advance_kernel(Ctl* c, const Ctl* nx, Ctl* tot, unsigned kernels,
                                  cudaGraphConditionalHandle cond, int set_cond) {
    tot->scat_elems += c->scat_elems;
    tot->fin_elems += c->fin_elems;
    tot->loc_elems += c->loc_elems;
    tot->err |= c->err;
    tot->launches += kernels + 1;
    tot->level += 1;
    unsigned more = (tot->err == 0 && (nx->nseg > 0 || nx->fin_ctr > 0)) ? 1u : 0u;
    if (more && tot->level >= (unsigned)kMaxLevels) {
        tot->err |= kErrLevels;
        more = 0;
    }
    tot->more = more;
    *c = Ctl{};
    if (set_cond) cudaGraphSetConditional(cond, more);
}

// Body tail of the graph's level loop: continue while tot.more.
__global__ void qs_loopctl_kernel(const Ctl* tot, cudaGraphConditionalHandle cond) {
    cudaGraphSetConditional(cond, tot->more);
}

// ------------------------------------------------------------ plan
// Position (in [0, len)) of sample i of S for the sampled-pivot levels, by
// the reference's pivot_strategy (quicksort.py:55-74, _kernels.py:358-376).
// A level takes many pivots at once, so each strategy picks the level's
// SAMPLE the way the reference picks its one pivot index:
//   0 median3 (default): one sample per stratum [i*len/S, (i+1)*len/S) at a
//     hashed offset -- stratified, the low-variance robust default;
//   1 middle: the middle index of every stratum, (lo + hi) // 2 -- no
//     randomness, like the reference's middle pivot;
//   2 random: the reference's 64-bit MMIX LCG (quicksort.py:22-25) seeded
//     with pivot_seed, one draw per sample over the whole segment.
// The pivots only steer the work; the sorted output is unique.
constexpr uint64_t kLcgMul = 6364136223846793005ULL, kLcgAdd = 1442695040888963407ULL;
__device__ __forceinline__ uint64_t sample_pos(unsigned strategy, uint64_t seed, uint64_t start, uint64_t len,
                                               unsigned i, unsigned S) {
    if (strategy == 2) {
        const uint64_t lcg = (seed + start + i) * kLcgMul + kLcgAdd;
        return __umul64hi(lcg * kLcgMul + kLcgAdd, len);  // lo + lcg mod span, by a high multiply
    }
    const uint64_t lo = (uint64_t)i * len / S, hi = (uint64_t)(i + 1) * len / S;  // stratum [lo, hi)
    const uint64_t span = hi > lo ? hi - lo : 1;
    if (strategy == 1) return lo + (span - 1) / 2;
    const uint64_t h = mix64(seed ^ mix64(start * 0x9E3779B97F4A7C15ULL + i));
    const uint64_t p = lo + __umul64hi(h, span);
    return p < len ? p : len - 1;
}

template <typename K, typename V>
__global__ void __launch_bounds__(kPlanNT) qs_plan_kernel(const K* __restrict__ src, Seg* __restrict__ segs,
                                                          Ctl* __restrict__ ctl, K* __restrict__ spl_pool,
                                                          unsigned long long* __restrict__ bkt_pool,
                                                          unsigned* __restrict__ tile_owner, unsigned cap_spl,
                                                          unsigned cap_bkt, unsigned cap_tiles, uint64_t sort_seed,
                                                          const Ctl* __restrict__ tot, uint64_t ql_target,
                                                          unsigned strategy) {
    constexpr int TILE = qs_tile<K>();
    __shared__ K s_samp[kMaxSample];
    __shared__ unsigned s_scan[kPlanNT / 32 + 1];
    __shared__ unsigned s_off[3];
    const unsigned nseg = ctl->nseg;
    const uint64_t seed = level_seed(sort_seed, tot);
    for (unsigned s = blockIdx.x; s < nseg; s += gridDim.x) {
        const uint64_t start = segs[s].start, len = segs[s].len;
        using U = typename OKey<K>::U;
        const uint64_t slo = segs[s].lo, shi = segs[s].hi;
        // bounds known from the parent: equal-width buckets, in code space
        // for 4-byte keys and in value space for float64
#ifndef VX_NO_RADIX
        const bool radix = slo < shi;
#else
        const bool radix = false;
#endif
        unsigned mt, rb = 0;
        if (ql_target == 0 || len <= 3 * ql_target) {
            // aim the buckets at half the finish capacity
            const uint64_t mt64 = len / (FinCap<K, V>::value / 2);
            mt = (unsigned)max((uint64_t)2, min((uint64_t)kMaxSplit, mt64));
            rb = mt + 1;
        } else {
            // aim the leaves of the remaining levels at the CTA-local level's
            // target, fan-out balanced over them: L levels of r^(1/L) buckets,
            // r = len / target.  A sampled level has up to 256 range buckets
            // (plus the equal-to-pivot ones), an equal-width level up to 511.
            // L counts against TWICE the target (kQlSlack): the CTA-local
            // level takes up to 3x the target, so leaves up to 2x (x1.25
            // sampling spread) still fit.  Counting against the target itself
            // sent every level-0 bucket even slightly above fan-out x target
            // (half of them at n = 2^32) through two more levels.
            const double r = (double)len / (double)ql_target;
            const double F = radix ? (double)kMaxBkt : (double)(kMaxSplit + 1);
            const double L = ceil(log(r / kQlSlack) / log(F) - 1e-9);
            const double f = ceil(pow(r, 1.0 / (L < 1.0 ? 1.0 : L)) - 1e-9);
            mt = (unsigned)max(2.0, min((double)kMaxSplit, f - 1.0));
            rb = (unsigned)max(2.0, min((double)kMaxBkt, f));
        }
        // rb equal-width buckets over the code bounds [blo, bhi] -- no pivot table
        auto equal_width = [&](uint64_t blo, uint64_t bhi, unsigned cs, unsigned open) {
            const uint64_t range = (uint64_t)(U)(bhi - blo);
            unsigned nb = rb;
            unsigned mul = 0;
            double vlo = 0.0, vinv = 0.0;
            if constexpr (sizeof(K) == 4) {
                if (range + 1 <= (uint64_t)nb) nb = (unsigned)(range + 1);  // one code per bucket
                else mul = (unsigned)(((uint64_t)nb << 32) / (range + 1));
            } else {
                // value space: x in [vlo, vhi] -> trunc((x - vlo) * vinv) in [0, nb)
                vlo = ord_to_f64((uint64_t)blo);
                const double w = ord_to_f64((uint64_t)bhi) - vlo;  // > 0 (blo < bhi; -0.0 / +0.0 aside)
                vinv = w > 0.0 && w < 1.7e308 ? (double)nb * (1.0 - 1e-12) / w : 0.0;  // 0: everything in bucket 0
            }
            if (threadIdx.x == 0) {
                const unsigned ntiles = (unsigned)((len + TILE - 1) / TILE);
                unsigned bo = atomicAdd(&ctl->bkt_ctr, nb << cs);
                unsigned to = atomicAdd(&ctl->tile_ctr, ntiles);
                if (bo + (nb << cs) > cap_bkt || to + ntiles > cap_tiles) {
                    // capacity exceeded: flag it; hist / emit / scatter skip the
                    // level (they test ctl->err), so no pool slot is aliased
                    atomicOr(&ctl->err, kErrCapacity);
                    bo = to = 0;
                }
                s_off[1] = bo;
                s_off[2] = to;
                segs[s].spl_off = 0;
                segs[s].m = 0;
                segs[s].bkt_off = bo;
                segs[s].tile_base = to;
                segs[s].nb = nb;
                segs[s].direct = 0;
                segs[s].mul = mul;
                segs[s].mode = sizeof(K) == 4 ? 1 : 2;
                segs[s].vlo = vlo;
                segs[s].vinv = vinv;
                segs[s].lo = blo;
                segs[s].hi = bhi;
                segs[s].cshift = cs;
                segs[s].open = open;
            }
            __syncthreads();
            for (unsigned b = threadIdx.x; b < (nb << cs); b += kPlanNT) bkt_pool[s_off[1] + b] = 0;
            const unsigned ntiles = (unsigned)((len + TILE - 1) / TILE);
            for (unsigned t = threadIdx.x; t < ntiles; t += kPlanNT) tile_owner[s_off[2] + t] = s;
            __syncthreads();
        };
        if (radix) {
            // bounds known from the parent: no sample either
            equal_width(slo, shi, 0u, 0u);
            continue;
        }
        unsigned S = next_pow2_u32(16 * (mt + 1));
        S = S < 256 ? 256 : (S > kMaxSample ? kMaxSample : S);
#ifndef VX_NO_UNIFORM_ROOT
        // the whole array of a large sort: the full sample, so the uniformity
        // test below has its 4 sigma
        if (nseg == 1 && tot->level == 0 && len >= (1ull << 24)) S = kMaxSample;
#endif
#pragma unroll 4
        for (unsigned i = threadIdx.x; i < S; i += kPlanNT) {
            s_samp[i] = src[start + sample_pos(strategy, seed, start, len, i, S)];
        }
        __syncthreads();
#ifdef VX_PLAN_CTA_BITONIC
        cta_bitonic<K, NoVal, kPlanNT>(s_samp, nullptr, S);
#else
        plan_sort_samples<K>(s_samp, S);
#endif
#ifndef VX_NO_UNIFORM_ROOT
        if constexpr (sizeof(K) == 4) {
            // 4-byte keys spread evenly over the whole code range (hashes,
            // random ids, the C1 / C5 uniform inputs): equal-width buckets over
            // the type's bounds instead of sampled pivots -- the histogram pass
            // then classifies with a high multiply instead of the cell table
            // and a splitter compare (2^28: 0.52 -> 0.35 ms).  Decided on the
            // sorted sample: every 64th-quantile within 2^27 codes (3 % of the
            // range, 4 sigma of a 4096-key sample) of where a uniform
            // distribution puts it.  Anything else -- narrower ranges,
            // clusters, few distinct keys -- keeps the sampled pivots; a
            // distribution that passes and still fills some bucket beyond the
            // leaf capacity just costs that bucket one more level.
            bool uni = S == (unsigned)kMaxSample && rb >= 2;
            if (threadIdx.x >= 1 && threadIdx.x < 64) {
                const uint32_t got = (uint32_t)OKey<K>::of(s_samp[threadIdx.x * (S / 64)]);
                const uint32_t want = threadIdx.x << 26;
                const uint32_t dev = got > want ? got - want : want - got;
                uni = uni && dev <= (1u << 27);
            }
            if (__syncthreads_and(uni)) {
#ifndef VX_UNIFORM_ROOT_WIDE
                rb = min(rb, mt + 1);  // the fan-out the sampled level would have had
#endif
                equal_width(0ull, 0xffffffffull, (unsigned)VX_ROOT_CSHIFT, 0u);
                continue;
            }
            // the same test over the SAMPLE's extremes (keys uniform over part
            // of the range, e.g. C4's [0, 2^31)): the keys beyond them saturate
            // into the first and last bucket, whose children get no bounds
            const uint32_t smin = (uint32_t)OKey<K>::of(s_samp[0]), smax = (uint32_t)OKey<K>::of(s_samp[S - 1]);
            const uint32_t w = smax - smin;
            uni = S == (unsigned)kMaxSample && rb >= 2 && w >= (1u << 20);
            if (threadIdx.x >= 1 && threadIdx.x < 64) {
                const uint32_t got = (uint32_t)OKey<K>::of(s_samp[threadIdx.x * (S / 64)]);
                const uint32_t want = smin + (uint32_t)(((uint64_t)w * threadIdx.x) >> 6);
                const uint32_t dev = got > want ? got - want : want - got;
                uni = uni && dev <= (w >> 5);
            }
            if (__syncthreads_and(uni)) {
#ifndef VX_UNIFORM_ROOT_WIDE
                rb = min(rb, mt + 1);
#endif
                equal_width((uint64_t)smin, (uint64_t)smax, (unsigned)VX_ROOT_CSHIFT, 1u);
                continue;
            }
        } else {
            // float64: the same test in VALUE space over the sample's own
            // extremes (there is no meaningful type range).  The few keys
            // beyond them land in the first and last bucket -- the classifier
            // saturates on both sides -- whose children therefore get no
            // bounds (emit) and find their own.
            const double smin = (double)s_samp[0], smax = (double)s_samp[S - 1], w = smax - smin;
            bool uni = S == (unsigned)kMaxSample && rb >= 2 && w > 0.0 && w < 1.7e308;
            if (threadIdx.x >= 1 && threadIdx.x < 64) {
                const double got = (double)s_samp[threadIdx.x * (S / 64)];
                const double want = smin + w * ((double)threadIdx.x * (1.0 / 64.0));
                uni = uni && fabs(got - want) <= w * (1.0 / 32.0);
            }
            if (__syncthreads_and(uni)) {
#ifndef VX_UNIFORM_ROOT_WIDE
                rb = min(rb, mt + 1);
#endif
                equal_width((uint64_t)OKey<K>::of(s_samp[0]), (uint64_t)OKey<K>::of(s_samp[S - 1]),
                            (unsigned)VX_ROOT_CSHIFT, 1u);
                continue;
            }
        }
#endif
        // candidate j = sample at quantile (j+1)/(mt+1); keep distinct values
        K cand = K();
        unsigned keep = 0;
        if (threadIdx.x < mt) {
            const unsigned q = (unsigned)(((uint64_t)(threadIdx.x + 1) * S) / (mt + 1));
            cand = s_samp[q];
            if (threadIdx.x == 0) keep = 1;
            else {
                const unsigned qp = (unsigned)(((uint64_t)threadIdx.x * S) / (mt + 1));
                keep = (s_samp[qp] < cand) ? 1u : 0u;
            }
        }
        unsigned m;
        const unsigned rank = block_excl_scan<kPlanNT>(keep, s_scan, &m);
        if (threadIdx.x == 0) {
            const unsigned ntiles = (unsigned)((len + TILE - 1) / TILE);
            unsigned so = atomicAdd(&ctl->spl_ctr, m);
            constexpr unsigned cs = 0;
            unsigned bo = atomicAdd(&ctl->bkt_ctr, (2 * m + 1) << cs);
            unsigned to = atomicAdd(&ctl->tile_ctr, ntiles);
            if (so + m > cap_spl || bo + ((2 * m + 1) << cs) > cap_bkt || to + ntiles > cap_tiles) {
                atomicOr(&ctl->err, kErrCapacity);
                so = bo = to = 0;
            }
            s_off[0] = so;
            s_off[1] = bo;
            s_off[2] = to;
            segs[s].spl_off = so;
            segs[s].m = m;
            segs[s].bkt_off = bo;
            segs[s].tile_base = to;
            segs[s].nb = 2 * m + 1;
            segs[s].direct = 0;
            segs[s].mode = 0;
            segs[s].cshift = cs;
            segs[s].open = 0;
        }
        __syncthreads();
        if (keep) spl_pool[s_off[0] + rank] = cand;
        for (unsigned b = threadIdx.x; b < 2 * m + 1; b += kPlanNT) bkt_pool[s_off[1] + b] = 0;
        const unsigned ntiles = (unsigned)((len + TILE - 1) / TILE);
        for (unsigned t = threadIdx.x; t < ntiles; t += kPlanNT) tile_owner[s_off[2] + t] = s;
        __syncthreads();
    }
}

// ------------------------------------------------------------ tiles
struct TileGeo {
    uint64_t base;  // absolute index of the tile's first element
    unsigned tn;    // elements in the tile
    unsigned seg;   // owning segment
};

template <int TILE>
__device__ __forceinline__ TileGeo tile_geo(unsigned t, const unsigned* tile_owner, const Seg* segs) {
    TileGeo g;
    g.seg = tile_owner[t];
    const uint64_t start = segs[g.seg].start, len = segs[g.seg].len;
    const unsigned tb = segs[g.seg].tile_base;
    g.base = start + (uint64_t)(t - tb) * TILE;
    g.tn = (unsigned)min((uint64_t)TILE, start + len - g.base);
    return g;
}

// striped tile load: item i of thread tid is element i*NT + tid
template <typename T, int IPT>
__device__ __forceinline__ void load_tile(T (&x)[IPT], const T* src, const TileGeo& g) {
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        const unsigned idx = i * kQsNT + threadIdx.x;
        x[i] = idx < g.tn ? ld_stream(src + g.base + idx) : T();
    }
}

// ------------------------------------------------------------ emit
// Exclusive scan of one u64 per thread over a CTA.
template <int NT>
__device__ __forceinline__ unsigned long long block_excl_scan_u64(unsigned long long v, unsigned long long* sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = NT / 32;
    unsigned long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        unsigned long long t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < NW ? sm[lane] : 0ull, wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            unsigned long long t = __shfl_up_sync(0xffffffffu, wi, d);
            if (lane >= d) wi += t;
        }
        if (lane < NW) sm[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long r = sm[warp] + inc - v;
    __syncthreads();
    return r;
}

template <typename K, typename V>
__global__ void __launch_bounds__(kPlanNT) qs_emit_kernel(Seg* __restrict__ segs, Ctl* __restrict__ ctl,
                                                          Ctl* __restrict__ ctl_next, Seg* __restrict__ next_segs,
                                                          unsigned long long* __restrict__ bkt_pool,
                                                          Fin* __restrict__ fins, unsigned cap_seg, unsigned cap_fin,
                                                          int dst_is_scratch, const K* __restrict__ spl_pool,
                                                          QlItemT* __restrict__ qls,
                                                          uint64_t ql_cap, int direct_ok) {
    static_assert(kPlanNT >= kMaxBkt, "one thread per bucket");
    constexpr uint32_t LOCAL = FinCap<K, V>::value;
    __shared__ unsigned long long s_scan[kPlanNT / 32];
    if (ctl->err) return;  // the plan ran out of pool capacity: the level is void
    const unsigned nseg = ctl->nseg;
    for (unsigned s = blockIdx.x; s < nseg; s += gridDim.x) {
        const Seg sg = segs[s];
        const unsigned nb = sg.nb;
        const bool radix = sg.mode != 0;
        const unsigned b = threadIdx.x;
        const unsigned long long c = b < nb ? bkt_pool[sg.bkt_off + (b << sg.cshift)] : 0ull;
        const unsigned long long ex = block_excl_scan_u64<kPlanNT>(c, s_scan);
        // a bucket is final when it holds one key, one code (equal-width) or
        // the keys equal to a pivot.  If EVERY bucket of the segment is final
        // (few distinct keys) and the scatter may write the output (level 0 of
        // an out-of-place sort: direct_ok), it does so and nothing is copied
        // home afterwards.
        const bool final_b = c == 1 || (sg.mode == 1 ? (sg.mul == 0) : sg.mode == 0 && (b & 1u) != 0);
        const bool direct = !__syncthreads_or(b < nb && c > 0 && !final_b) && direct_ok != 0;
        if (direct && threadIdx.x == 0) segs[s].direct = 1u;
        if (b < nb) {
            const unsigned long long bstart = sg.start + ex;
            bkt_pool[sg.bkt_off + (b << sg.cshift)] = bstart;  // becomes the scatter cursor
            // the bucket's key-code bounds, for the child's own partition:
            // a range bucket 2j lies strictly between pivots j-1 and j; a
            // radix bucket spans its 2^shift codes.  A radix child holding
            // more than half its parent is skewed: it forgets its bounds
            // and is partitioned around sampled pivots.
            unsigned long long clo = 1, chi = 0;
            if (sg.mode == 2) {
                // value-space bucket b holds x with trunc((x - vlo) * vinv) == b:
                // bounds widened by 1/1000 of a bucket against rounding, kept
                // inside the parent's; a bucket too narrow for that margin to
                // dominate the rounding of vlo + offset leaves them unknown
                if constexpr (sizeof(K) == 8) {
                    if (sg.vinv > 0.0) {
                        const double w = 1.0 / sg.vinv;  // bucket width
                        const double lo_v = sg.vlo + ((double)b - 1e-3) * w, hi_v = sg.vlo + ((double)b + 1.001) * w;
                        const double mag = fmax(fabs(lo_v), fabs(hi_v));
                        if (w * 1e-3 > mag * 1e-15) {
                            const unsigned long long cl = f64_to_ord(lo_v), ch = f64_to_ord(hi_v);
                            clo = cl > sg.lo ? cl : sg.lo;
                            chi = ch < sg.hi ? ch : sg.hi;
                            if (b == 0) clo = sg.lo;
                            if (b + 1 == nb) chi = sg.hi;
                        }
                    }
                    if (sg.open && (b == 0 || b + 1 == nb)) {  // keys beyond the sample's extremes live here
                        clo = 1;
                        chi = 0;
                    }
                }
                if (2 * c > sg.len) {
                    clo = 1;
                    chi = 0;
                }
            } else if (radix) {
                // bucket b holds the offsets d with umulhi(d, mul) == b:
                // [ceil(b * 2^32 / mul), ceil((b + 1) * 2^32 / mul) - 1]
                auto dlo = [&](unsigned long long bb) -> unsigned long long {
                    return sg.mul ? ((bb << 32) + sg.mul - 1) / sg.mul : bb;
                };
                clo = sg.lo + dlo(b);
                chi = b + 1 < nb ? sg.lo + dlo(b + 1ull) - 1 : sg.hi;
                if (2 * c > sg.len || (sg.open && (b == 0 || b + 1 == nb))) {
                    clo = 1;
                    chi = 0;
                }
            } else if (!(b & 1u) && (b >> 1) > 0 && (b >> 1) < sg.m) {
                const unsigned j = b >> 1;
                clo = (unsigned long long)OKey<K>::of(spl_pool[sg.spl_off + j - 1]) + 1;
                chi = (unsigned long long)OKey<K>::of(spl_pool[sg.spl_off + j]) - 1;
            }
            if (c > 0) {
                const bool final_ = final_b;
                if (final_) {
                    if (dst_is_scratch && !direct) {  // final but parked in scratch: copy home in chunks
                        // (this thread writes every chunk record: at most ~1024 per bucket)
                        const unsigned long long chunk =
                            max((unsigned long long)kCopyChunk, ((c >> 10) + 4095ull) & ~4095ull);
                        const unsigned nch = (unsigned)((c + chunk - 1) / chunk);
                        unsigned f = atomicAdd(&ctl->fin_ctr, nch);
                        if (f + nch > cap_fin) {
                            atomicOr(&ctl->err, kErrCapacity);
                        } else {
                            for (unsigned i = 0; i < nch; ++i) {
                                const unsigned long long o = (unsigned long long)i * chunk;
                                fins[f + i].start = bstart + o;
                                fins[f + i].len = (unsigned)min(chunk, c - o);
                                fins[f + i].flags = 3u;
                            }
                        }
                    }
                } else if (c <= LOCAL) {
                    unsigned f = atomicAdd(&ctl->fin_ctr, 1u);
                    if (f >= cap_fin) {
                        atomicOr(&ctl->err, kErrCapacity);
                    } else {
                        fins[f].start = bstart;
                        fins[f].len = (unsigned)c;
                        fins[f].flags = dst_is_scratch ? 1u : 0u;
                    }
                } else if (c <= ql_cap) {
                    unsigned q = atomicAdd(&ctl->ql_ctr, 1u);
                    if (q >= cap_seg) {
                        atomicOr(&ctl->err, kErrCapacity);
                    } else {
                        qls[q].start = bstart;
                        qls[q].len = c;
                        qls[q].lo = clo;
                        qls[q].hi = chi;
                    }
                } else {
                    unsigned q = atomicAdd(&ctl_next->nseg, 1u);
                    if (q >= cap_seg) {
                        atomicOr(&ctl->err, kErrCapacity);
                    } else {
                        next_segs[q].start = bstart;
                        next_segs[q].len = c;
                        next_segs[q].lo = clo;
                        next_segs[q].hi = chi;
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ scatter
template <typename K, typename V>
struct ScatterSmem {
    static constexpr int TILE = qs_tile<K>();
    K k[TILE];
    typename std::conditional<HasVal<V>::value, V, char>::type v[HasVal<V>::value ? TILE : 1];
    unsigned short b[TILE];
    unsigned cnt[kMaxBkt + 1];
    unsigned loc[kMaxBkt + 1];
    unsigned long long gbase[kMaxBkt + 1];
    CellTable<typename OKey<K>::U> ct;  // splitters + cell lookup table
    typename KeyRep<K>::I spl[256];     // (key, index) splitters of the sharded bucket partition
    unsigned long long dstp[256];       // fused exchange: destination base pointer per bucket
    unsigned scan[kQsNT / 32 + 1];
};

// Rank IPT classified items of this thread inside the tile (smem atomics),
// scan the bucket counts, reserve global runs and stage bucket-major.
// Shared by the quicksort levels and the sharded bucket partition.
template <typename K, typename V, int IPT>
__device__ __forceinline__ void tile_scatter(ScatterSmem<K, V>& sm, const K (&k)[IPT], const V (&v)[IPT],
                                             const unsigned (&bk)[IPT], unsigned validmask, unsigned nb,
                                             unsigned long long* cursor, K* dst_k, V* dst_v, unsigned tn,
                                             bool per_bucket_dst = false) {
    constexpr bool KV = HasVal<V>::value;
    // rank inside the tile, packed next to the bucket id: (bucket << 16) | rank
    unsigned br[IPT];
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        br[i] = 0u;
        if ((validmask >> i) & 1u) br[i] = (bk[i] << 16) | atomicAdd(&sm.cnt[bk[i]], 1u);
    }
    __syncthreads();
    // exclusive scan of counts over nb (<= 2*NT) buckets: 2 per thread
    const unsigned b0 = 2 * threadIdx.x, b1 = b0 + 1;
    const unsigned c0 = b0 < nb ? sm.cnt[b0] : 0u, c1 = b1 < nb ? sm.cnt[b1] : 0u;
    unsigned tot;
    const unsigned ex = block_excl_scan<kQsNT>(c0 + c1, sm.scan, &tot);
    if (b0 < nb) {
        sm.loc[b0] = ex;
        if (c0) sm.gbase[b0] = atomicAdd(&cursor[b0], (unsigned long long)c0);
    }
    if (b1 < nb) {
        sm.loc[b1] = ex + c0;
        if (c1) sm.gbase[b1] = atomicAdd(&cursor[b1], (unsigned long long)c1);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < IPT; ++i) {
        if ((validmask >> i) & 1u) {
            const unsigned slot = sm.loc[br[i] >> 16] + (br[i] & 0xffffu);
            sm.k[slot] = k[i];
            if constexpr (KV) sm.v[slot] = v[i];
            sm.b[slot] = (unsigned short)(br[i] >> 16);
        }
    }
    __syncthreads();
    for (unsigned j = threadIdx.x; j < tn; j += kQsNT) {
        const unsigned b = sm.b[j];
        const unsigned long long pos = sm.gbase[b] + (j - sm.loc[b]);
        // fused exchange: bucket b's run goes straight into destination b's
        // buffer (a peer GPU's receive buffer mapped over NVLink)
        K* dk = per_bucket_dst ? reinterpret_cast<K*>(sm.dstp[b]) : dst_k;
        dk[pos] = sm.k[j];
        if constexpr (KV) dst_v[pos] = sm.v[j];
    }
}

// ------------------------------------------------------------ segments API
// Batched bitonic over CSR segments (config 2): one warp per segment,
// in place, lengths <= 256 (longer segments flag kErrTooLong, untouched;
// offsets outside [0, n] or decreasing flag kErrOffsets, untouched).
template <typename K, typename V>
__global__ void __launch_bounds__(256) segsort_kernel(K* __restrict__ k, V* __restrict__ v, uint64_t n,
                                                      const long long* __restrict__ offs, uint64_t nseg,
                                                      unsigned* __restrict__ err) {
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nseg; s += warps) {
        const long long lo = offs[s], hi = offs[s + 1];
        const long long len = hi - lo;
        if (lo < 0 || hi < lo || (unsigned long long)hi > n) {
            if ((threadIdx.x & 31) == 0) atomicOr(err, kErrOffsets);
            continue;
        }
        if (len < 2) continue;
        if (len > 256) {
            if ((threadIdx.x & 31) == 0) atomicOr(err, kErrTooLong);
            continue;
        }
        warp_sort_any2<K, V>(k + lo, v ? v + lo : nullptr, k + lo, v ? v + lo : nullptr, (unsigned)len);
    }
}

// ------------------------------------------------------------ bucket partition (sharded sort)
// k-way partition of one array around m (key, global-index) splitters into
// m+1 destination buckets.  Two kernels: histogram, then scatter; counts are
// exclusive-scanned in between by bp_scan_kernel.
template <typename K>
__global__ void __launch_bounds__(kQsNT) bp_hist_kernel(const K* __restrict__ src, uint64_t n, uint64_t gofs,
                                                        const K* __restrict__ spk, const uint64_t* __restrict__ spi,
                                                        unsigned m, unsigned long long* __restrict__ counts) {
    constexpr int IPT = QsTile<K>::IPT, TILE = kQsNT * IPT;
    __shared__ typename KeyRep<K>::I s_k[256];
    __shared__ uint64_t s_i[256];
    __shared__ unsigned s_hist[257];
    for (unsigned i = threadIdx.x; i < m; i += kQsNT) {
        s_k[i] = KeyRep<K>::to(spk[i]);
        s_i[i] = spi[i];
    }
    const uint64_t ntiles = (n + TILE - 1) / TILE;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        __syncthreads();
        for (unsigned b = threadIdx.x; b <= m; b += kQsNT) s_hist[b] = 0;
        __syncthreads();
        const uint64_t base = t * TILE;
        const unsigned tn = (unsigned)min((uint64_t)TILE, n - base);
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const unsigned idx = i * kQsNT + threadIdx.x;
            if (idx < tn) {
                const K x = ld_stream(src + base + idx);
                atomicAdd(&s_hist[cls_idx(KeyRep<K>::to(x), gofs + base + idx, s_k, s_i, m)], 1u);
            }
        }
        __syncthreads();
        for (unsigned b = threadIdx.x; b <= m; b += kQsNT)
            if (s_hist[b]) atomicAdd(&counts[b], (unsigned long long)s_hist[b]);
    }
}

// destination cursors = exclusive scan of the counts (nb <= 256, one CTA)
__global__ void __launch_bounds__(256) bp_scan_kernel(const unsigned long long* __restrict__ counts, unsigned nb,
                                                      unsigned long long* __restrict__ cursor) {
    __shared__ unsigned long long s_scan[256 / 32];
    const unsigned long long c = threadIdx.x < nb ? counts[threadIdx.x] : 0ull;
    const unsigned long long ex = block_excl_scan_u64<256>(c, s_scan);
    if (threadIdx.x < nb) cursor[threadIdx.x] = ex;
}

template <typename K, typename V>
__global__ void __launch_bounds__(kQsNT, kQsMinBlocks) bp_scatter_kernel(const K* __restrict__ src_k, const V* __restrict__ src_v,
                                                           K* __restrict__ dst_k, V* __restrict__ dst_v, uint64_t n,
                                                           uint64_t gofs, const K* __restrict__ spk,
                                                           const uint64_t* __restrict__ spi, unsigned m,
                                                           unsigned long long* __restrict__ cursor,
                                                           const unsigned long long* __restrict__ dst_ptrs) {
    constexpr bool KV = HasVal<V>::value;
    constexpr int IPT = QsTile<K>::IPT, TILE = kQsNT * IPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScatterSmem<K, V>& sm = *reinterpret_cast<ScatterSmem<K, V>*>(smem_raw);
    __shared__ uint64_t s_i[256];
    for (unsigned i = threadIdx.x; i < m; i += kQsNT) {
        sm.spl[i] = KeyRep<K>::to(spk[i]);
        s_i[i] = spi[i];
    }
    if (dst_ptrs)
        for (unsigned i = threadIdx.x; i <= m; i += kQsNT) sm.dstp[i] = dst_ptrs[i];
    const unsigned nb = m + 1;
    const uint64_t ntiles = (n + TILE - 1) / TILE;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        __syncthreads();
        for (unsigned b = threadIdx.x; b < nb; b += kQsNT) sm.cnt[b] = 0;
        __syncthreads();
        const uint64_t base = t * TILE;
        const unsigned tn = (unsigned)min((uint64_t)TILE, n - base);
        K k[IPT];
        V v[IPT];
        unsigned bk[IPT];
        unsigned valid = 0;
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            const unsigned idx = i * kQsNT + threadIdx.x;
            if (idx < tn) {
                k[i] = ld_stream(src_k + base + idx);
                if constexpr (KV) v[i] = ld_stream(src_v + base + idx);
                bk[i] = cls_idx(KeyRep<K>::to(k[i]), gofs + base + idx, sm.spl, s_i, m);
                valid |= 1u << i;
            }
        }
        tile_scatter<K, V, IPT>(sm, k, v, bk, valid, nb, cursor, dst_k, dst_v, tn, dst_ptrs != nullptr);
    }
}

// Splitter selection for the sharded sort: sort the gathered (key, index)
// samples lexicographically in smem and take nparts-1 evenly spaced ones.
template <typename K>
__global__ void __launch_bounds__(1024) select_splitters_kernel(const K* __restrict__ keys,
                                                                const uint64_t* __restrict__ idx, unsigned count,
                                                                unsigned nparts, K* __restrict__ out_k,
                                                                uint64_t* __restrict__ out_i) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned P = next_pow2_u32(count);
    K* sk = reinterpret_cast<K*>(smem_raw);
    uint64_t* si = reinterpret_cast<uint64_t*>(smem_raw + sizeof(K) * P);
    for (unsigned i = threadIdx.x; i < P; i += blockDim.x) {
        sk[i] = i < count ? keys[i] : KeyTraits<K>::sentinel();
        si[i] = i < count ? idx[i] : ~0ull;
    }
    __syncthreads();
    for (unsigned k = 2; k <= P; k <<= 1) {
        for (unsigned j = k >> 1; j > 0; j >>= 1) {
            for (unsigned i = threadIdx.x; i < P; i += blockDim.x) {
                const unsigned ixj = i ^ j;
                if (ixj > i) {
                    const K x = sk[i], y = sk[ixj];
                    const uint64_t xi = si[i], yi = si[ixj];
                    const bool y_lt_x = (y < x) || (!(x < y) && yi < xi);
                    const bool asc = (i & k) == 0;
                    if (asc ? y_lt_x : !y_lt_x) {
                        sk[i] = y; sk[ixj] = x;
                        si[i] = yi; si[ixj] = xi;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (unsigned r = threadIdx.x + 1; r < nparts; r += blockDim.x) {
        const unsigned q = (unsigned)(((uint64_t)r * count) / nparts);
        out_k[r - 1] = sk[q];
        out_i[r - 1] = si[q];
    }
}

}  // namespace vx
