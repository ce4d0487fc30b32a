// scatter.cuh -- the partition level's scatter pass, software-pipelined.
//
// Per 4096-element tile: take every element's bucket (the id the histogram
// pass stored while classifying it), rank it inside its bucket with a shared
// memory atomic, reserve one run per non-empty bucket in the destination
// with a global atomic, stage the tile bucket-major in shared memory and
// write the runs with consecutive threads (coalesced).  The reservation is
// a round trip to L2 (~1 us); to keep it off the critical path the write-out
// of tile t-1 is done while tile t's reservations are in flight (two staging
// buffers), and tile t+1's loads are already in registers.
#pragma once

#include "common.cuh"
#include "qsort.cuh"

namespace vx {

template <typename K, typename V>
struct ScatterPipeSmem {
    static constexpr int TILE = qs_tile<K>();
    using VS = typename std::conditional<HasVal<V>::value, V, char>::type;
    struct Stage {
        K k[TILE];
        VS v[HasVal<V>::value ? TILE : 1];
        unsigned short b[TILE];
        unsigned long long delta[kMaxBkt + 1];  // destination of slot j in bucket b: delta[b] + j
        unsigned tn;
#ifdef VX_CHECK
        unsigned long long lo, hi;  // the owning segment's range in the destination
#endif
    };
    Stage st[2];
    unsigned cnt[2][kMaxBkt + 1];  // per-tile counts, then (in place) bucket offsets; double-buffered
    unsigned scan[kQsNT / 32 + 1];
};

template <typename K, typename V>
__device__ __forceinline__ void stage_writeout(const typename ScatterPipeSmem<K, V>::Stage& s, K* dst_k, V* dst_v) {
    constexpr bool KV = HasVal<V>::value;
    for (unsigned j = threadIdx.x; j < s.tn; j += kQsNT) {
        const unsigned long long pos = s.delta[s.b[j]] + j;
        VX_ASSERT(pos >= s.lo && pos < s.hi);  // inside the tile's segment
        dst_k[pos] = s.k[j];
        if constexpr (KV) dst_v[pos] = s.v[j];
    }
}

template <typename K, typename V>
__global__ void __launch_bounds__(kQsNT, kQsMinBlocks) qs_scatter_kernel(const K* __restrict__ src_k, const V* __restrict__ src_v,
                                                           const unsigned short* __restrict__ ids,
                                                           K* __restrict__ dst_k, V* __restrict__ dst_v, K* root_out_k, V* root_out_v,
                                                           const Seg* __restrict__ segs, Ctl* __restrict__ ctl,
                                                           const unsigned* __restrict__ tile_owner,
                                                           unsigned long long* __restrict__ bkt_pool) {
    constexpr bool KV = HasVal<V>::value;
    constexpr int IPT = QsTile<K>::IPT, TILE = kQsNT * IPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ScatterPipeSmem<K, V>& sm = *reinterpret_cast<ScatterPipeSmem<K, V>*>(smem_raw);
    if (ctl->err) return;  // the plan ran out of pool capacity: the level is void
    const unsigned ntiles = ctl->tile_ctr;
    const unsigned t0 = (unsigned)(((uint64_t)blockIdx.x * ntiles) / gridDim.x);
    const unsigned t1 = (unsigned)(((uint64_t)(blockIdx.x + 1) * ntiles) / gridDim.x);
    if (t0 >= t1) return;
    // level 0 of an out-of-place sort whose buckets are all final (emit set
    // Seg::direct on the one root segment): straight into the output
    if (root_out_k && segs[0].direct) {
        dst_k = root_out_k;
        dst_v = root_out_v;
    }
    const unsigned b0 = 2 * threadIdx.x, b1 = b0 + 1;  // the two buckets this thread scans / reserves
    const bool owner = b1 <= (unsigned)kMaxBkt;        // threads past the bucket range own none
    if (owner) sm.cnt[0][b0] = sm.cnt[0][b1] = sm.cnt[1][b0] = sm.cnt[1][b1] = 0u;
    unsigned cur = 0xffffffffu, bkt_off = 0, nb = 0, cs = 0;
    // equal-width segments of 4-byte keys (mode 1): the histogram pass stores
    // no ids for them; a key's bucket is a subtract and a high multiply away
    // (2 B/key less to write there and to read here)
    auto stored_ids = [&](unsigned seg) -> bool { return sizeof(K) != 4 || segs[seg].mode != 1; };
    unsigned ew = 0, ew_lo = 0, ew_mul = 0;
    TileGeo g = tile_geo<TILE>(t0, tile_owner, segs);
    K k[IPT];
    V v[IPT];
    unsigned short id[IPT];
    load_tile<K, IPT>(k, src_k, g);
    if (stored_ids(g.seg)) load_tile<unsigned short, IPT>(id, ids, g);
    if constexpr (KV) load_tile<V, IPT>(v, src_v, g);
    unsigned long long moved = 0;
    __syncthreads();
    for (unsigned t = t0; t < t1; ++t) {
        const int p = (t - t0) & 1;
        TileGeo gn{};
        K kn[IPT];
        V vn[IPT];
        unsigned short idn[IPT];
        if (t + 1 < t1) {
            gn = tile_geo<TILE>(t + 1, tile_owner, segs);
            load_tile<K, IPT>(kn, src_k, gn);
            if (stored_ids(gn.seg)) load_tile<unsigned short, IPT>(idn, ids, gn);
            if constexpr (KV) load_tile<V, IPT>(vn, src_v, gn);
        }
        if (g.seg != cur) {
            cur = g.seg;
            bkt_off = segs[g.seg].bkt_off;
            nb = segs[g.seg].nb;
            cs = segs[g.seg].cshift;
            if constexpr (sizeof(K) == 4) {
                ew = segs[g.seg].mode == 1 ? 1u : 0u;
                ew_lo = (unsigned)segs[g.seg].lo;
                ew_mul = segs[g.seg].mul;
            }
        }
        if constexpr (sizeof(K) == 4) {
            if (ew) {
#pragma unroll
                for (int i = 0; i < IPT; ++i) {
                    const uint32_t d = max((uint32_t)OKey<K>::of(k[i]), ew_lo) - ew_lo;
                    id[i] = (unsigned short)min(nb - 1, ew_mul ? __umulhi(d, ew_mul) : d);
                }
            }
        }
        unsigned* cnt = sm.cnt[p];
        moved += g.tn;
        // rank by the bucket id the histogram pass stored: (bucket << 16) | rank within the tile
        unsigned br[IPT];
        if (g.tn == TILE) {
            // a warp whose IPT x 32 keys share one bucket (sorted / reverse /
            // few-unique inputs) reserves their ranks with one atomic
            const unsigned b0 = __shfl_sync(0xffffffffu, (unsigned)id[0], 0);
            bool same = true;
#pragma unroll
            for (int i = 0; i < IPT; ++i) same &= id[i] == b0;
            if (__all_sync(0xffffffffu, same)) {
                unsigned base = 0;
                if ((threadIdx.x & 31) == 0) base = atomicAdd(&cnt[b0], 32u * IPT);
                base = __shfl_sync(0xffffffffu, base, 0) + (threadIdx.x & 31);
#pragma unroll
                for (int i = 0; i < IPT; ++i) br[i] = (b0 << 16) | (base + 32u * i);
            } else {
#pragma unroll
                for (int i = 0; i < IPT; ++i) br[i] = ((unsigned)id[i] << 16) | atomicAdd(&cnt[id[i]], 1u);
            }
        } else {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const unsigned b = id[i];
                br[i] = (i * kQsNT + threadIdx.x < g.tn) ? ((b << 16) | atomicAdd(&cnt[b], 1u)) : 0xffffffffu;
            }
        }
        __syncthreads();
        // bucket offsets in the tile (2 buckets per thread, in place) + run reservations
        typename ScatterPipeSmem<K, V>::Stage& S = sm.st[p];
        const unsigned c0 = b0 < nb ? cnt[b0] : 0u, c1 = b1 < nb ? cnt[b1] : 0u;
        unsigned tot;
        const unsigned ex = block_excl_scan<kQsNT>(c0 + c1, sm.scan, &tot);
        unsigned long long r0 = 0, r1 = 0;
        if (c0) r0 = atomicAdd(&bkt_pool[bkt_off + (b0 << cs)], (unsigned long long)c0);
        if (c1) r1 = atomicAdd(&bkt_pool[bkt_off + (b1 << cs)], (unsigned long long)c1);
        if (b0 < nb) cnt[b0] = ex;
        if (b1 < nb) cnt[b1] = ex + c0;
        if (threadIdx.x == 0) S.tn = g.tn;
#ifdef VX_CHECK
        if (threadIdx.x == 0) {
            S.lo = segs[g.seg].start;
            S.hi = segs[g.seg].start + segs[g.seg].len;
        }
#endif
        // overlap: write out the previous tile while the reservations fly
        if (t > t0) stage_writeout<K, V>(sm.st[p ^ 1], dst_k, dst_v);
        if (c0) S.delta[b0] = r0 - ex;
        if (c1) S.delta[b1] = r1 - (ex + c0);
        __syncthreads();  // offsets complete; previous stage written out
        unsigned* nxt = sm.cnt[p ^ 1];  // the previous tile's offsets are dead: clear for tile t+1
        if (owner) nxt[b0] = nxt[b1] = 0u;
        if (g.tn == TILE) {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                const unsigned slot = cnt[br[i] >> 16] + (br[i] & 0xffffu);
                VX_ASSERT(slot < (unsigned)TILE && (br[i] >> 16) < nb);
                S.k[slot] = k[i];
                if constexpr (KV) S.v[slot] = v[i];
                S.b[slot] = (unsigned short)(br[i] >> 16);
            }
        } else {
#pragma unroll
            for (int i = 0; i < IPT; ++i) {
                if (br[i] != 0xffffffffu) {
                    const unsigned slot = cnt[br[i] >> 16] + (br[i] & 0xffffu);
                    VX_ASSERT(slot < g.tn && (br[i] >> 16) < nb);
                    S.k[slot] = k[i];
                    if constexpr (KV) S.v[slot] = v[i];
                    S.b[slot] = (unsigned short)(br[i] >> 16);
                }
            }
        }
        __syncthreads();  // stage complete; counts for t+1 cleared
#pragma unroll
        for (int i = 0; i < IPT; ++i) {
            k[i] = kn[i];
            id[i] = idn[i];
            if constexpr (KV) v[i] = vn[i];
        }
        g = gn;
    }
    stage_writeout<K, V>(sm.st[(t1 - 1 - t0) & 1], dst_k, dst_v);
    if (threadIdx.x == 0) atomicAdd(&ctl->scat_elems, moved);
}

}  // namespace vx
