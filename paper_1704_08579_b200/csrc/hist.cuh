// hist.cuh -- the partition level's histogram pass, TMA-pipelined.
//
// Persistent CTAs each own a contiguous chunk of the level's 4096-element
// tiles (consecutive tiles share a segment, so the segment's cell table is
// built once per CTA and segment).  Tiles stream into a shared memory ring
// (4 stages for int32) with 1-D bulk copies (cp.async.bulk, completion on an
// mbarrier) issued NS-1 tiles ahead by one thread, so HBM reads overlap the
// classification of the current tile without holding registers.  The copy
// takes the tile's 16-byte aligned window whenever it lies inside the array,
// so every element is read from shared memory with no edge tests.  Each
// element is classified into one of 2m+1 buckets (ranges and equal-to-pivot
// buckets) and counted in a shared histogram that is flushed to the
// segment's global histogram once per (CTA, segment).  The bucket id of every
// element is stored (u16, coalesced) for the scatter pass, which then ranks
// and moves elements without classifying them again -- except in equal-width
// segments of 4-byte keys, where the scatter recomputes it (a subtract and a
// high multiply) and this pass, DRAM-bound once its grid was chunked, writes
// nothing.
#pragma once

#include "common.cuh"
#include "qsort.cuh"
#include "tma.cuh"

namespace vx {

// TMA ring depth: 4 x 16 KB for int32 tiles, 2 x 32 KB for float64 (so two
// CTAs still fit on an SM)
#ifndef VX_HIST_STAGES4
#define VX_HIST_STAGES4 4
#endif
#ifndef VX_HIST_STAGES8
#define VX_HIST_STAGES8 2
#endif
template <typename K>
constexpr int hist_stages() { return sizeof(K) == 4 ? VX_HIST_STAGES4 : VX_HIST_STAGES8; }

template <typename K>
constexpr unsigned hist_stage_bytes() {
    return (unsigned)(qs_tile<K>() * sizeof(K) + 32);
}
template <typename K>
constexpr unsigned hist_smem_bytes() {
    return hist_stages<K>() * ((hist_stage_bytes<K>() + 127) / 128 * 128);
}

// Ring protocol: full[s] completes when the bulk copy into stage s landed;
// empty[s] (count = CTA size) when every thread has consumed it.  Thread 0
// refills a stage only after its empty phase, so warps drift freely within
// the ring instead of meeting at a CTA barrier every tile.
template <typename K>
__global__ void __launch_bounds__(kQsNT, kQsMinBlocks) qs_hist_kernel(const K* __restrict__ src, uint64_t n_all,
                                                        const Seg* __restrict__ segs,
                                                        const Ctl* __restrict__ ctl,
                                                        const unsigned* __restrict__ tile_owner,
                                                        const K* __restrict__ spl_pool,
                                                        unsigned long long* __restrict__ bkt_pool,
                                                        unsigned short* __restrict__ ids) {
    constexpr int IPT = QsTile<K>::IPT, TILE = kQsNT * IPT;
    constexpr unsigned BUF = (hist_stage_bytes<K>() + 127) / 128 * 128;
    constexpr int NS = hist_stages<K>();
    using U = typename OKey<K>::U;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ CellTable<U> s_ct;
    __shared__ unsigned s_hist[kMaxBkt + 1];
    __shared__ unsigned s_scan[kQsNT / 32 + 1];
    __shared__ __align__(8) uint64_t s_full[NS];
    __shared__ __align__(8) uint64_t s_empty[NS];
    __shared__ BulkTile s_meta[NS];

    if (ctl->err) return;  // the plan ran out of pool capacity: the level is void
    const unsigned ntiles = ctl->tile_ctr;
    const unsigned t0 = (unsigned)(((uint64_t)blockIdx.x * ntiles) / gridDim.x);
    const unsigned t1 = (unsigned)(((uint64_t)(blockIdx.x + 1) * ntiles) / gridDim.x);
    if (t0 >= t1) return;
    const unsigned tid = threadIdx.x;

    auto issue = [&](unsigned t, unsigned stage) {  // one thread
        const TileGeo g = tile_geo<TILE>(t, tile_owner, segs);
        BulkTile bt = plan_tile<K>(src, n_all, g.base, g.tn);
        bt.seg = g.seg;
        s_meta[stage] = bt;  // before the arrive (release): consumers read it after their acquire
        issue_planned(reinterpret_cast<char*>(smem_raw) + stage * BUF, bt, &s_full[stage]);
    };
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], kQsNT);
        }
        fence_mbar_init();
        for (unsigned j = 0; j + 1 < NS && t0 + j < t1; ++j) issue(t0 + j, j);
    }
    __syncthreads();

    unsigned cur = 0xffffffffu, bkt_off = 0, nb = 0, rsh = 0, cs = 0;
    bool radix = false, vmode = false;
    U rlo = 0;
    double vlo = 0.0, vinv = 0.0;
    CellParams<U> cp{};
    // equal-width segments: bucket = umulhi(code - lo, mul) (keys lie in
    // [lo, hi] by construction, so the bucket is < nb)
    auto classify = [&](K key) -> unsigned {
        if constexpr (sizeof(K) == 8) {
            // value-space equal-width buckets (mode 2)
            if (vmode) return min(nb - 1, (unsigned)__double2uint_rz(((double)key - vlo) * vinv));
        }
        if (radix) {
            // (saturating below: an open-ended root sees keys under its lower bound)
            const uint32_t d = (uint32_t)(max(OKey<K>::of(key), rlo) - rlo);
            return min(nb - 1, rsh ? __umulhi(d, rsh) : d);
        }
        return ct_classify(s_ct, cp, key);
    };
    unsigned stage = 0, par = 0;          // this tile's stage and phase parity
    unsigned pstage = NS - 1, ppar = 1;   // the previous tile's
    for (unsigned t = t0; t < t1; ++t) {
        if (tid == 0 && t + NS - 1 < t1) {
            // refill the previous tile's stage once everybody is done with it
            if (t > t0) mbar_wait(&s_empty[pstage], ppar);
            issue(t + NS - 1, pstage);
        }
        mbar_wait(&s_full[stage], par);
        const BulkTile bt = s_meta[stage];
        if (bt.seg != cur) {
            // flush the previous segment's counts, build the new table
            __syncthreads();
            if (cur != 0xffffffffu)
                for (unsigned b = tid; b < nb; b += kQsNT)
                    if (s_hist[b]) atomicAdd(&bkt_pool[bkt_off + (b << cs)], (unsigned long long)s_hist[b]);
            cur = bt.seg;
            const Seg sg = segs[bt.seg];
            bkt_off = sg.bkt_off;
            nb = sg.nb;
            cs = sg.cshift;
            radix = sg.mode == 1;
            vmode = sg.mode == 2;
            vlo = sg.vlo;
            vinv = sg.vinv;
            rlo = (U)sg.lo;
            rsh = sg.mul;
            if (!radix && !vmode) cp = ct_load<K, kQsNT>(s_ct, spl_pool, sg.spl_off, sg.m, s_scan);  // barriers inside
            for (unsigned b = tid; b < nb; b += kQsNT) s_hist[b] = 0;
            __syncthreads();
        }
        // (the scatter recomputes the bucket of a 4-byte key in an equal-width segment)
        const bool store_ids = sizeof(K) != 4 || !radix;
        const char* buf = reinterpret_cast<const char*>(smem_raw) + stage * BUF;
        if (bt.body == TILE) {  // the whole (full) tile is in shared memory
            const K* sb = reinterpret_cast<const K*>(buf + bt.shift);
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const unsigned b = classify(sb[i * kQsNT + tid]);
                VX_ASSERT(b < nb && bt.base + i * kQsNT + tid < n_all);
                // result unused: ATOMS.POPC.INC, which already merges the
                // lanes of a warp that hit one counter (sorted inputs)
                atomicAdd(&s_hist[b], 1u);
                if (store_ids) ids[bt.base + i * kQsNT + tid] = (unsigned short)b;
            }
        } else {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const unsigned idx = i * kQsNT + tid;
                if (idx < bt.tn) {
                    const K x = tile_get<K>(buf, bt, src, idx);
                    const unsigned b = classify(x);
                    VX_ASSERT(b < nb && bt.base + idx < n_all);
                    atomicAdd(&s_hist[b], 1u);
                    if (store_ids) ids[bt.base + idx] = (unsigned short)b;
                }
            }
        }
        mbar_arrive(&s_empty[stage]);
        pstage = stage;
        ppar = par;
        if (++stage == NS) {
            stage = 0;
            par ^= 1u;
        }
    }
    __syncthreads();
    for (unsigned b = tid; b < nb; b += kQsNT)
        if (s_hist[b]) atomicAdd(&bkt_pool[bkt_off + (b << cs)], (unsigned long long)s_hist[b]);
}

}  // namespace vx
