// bitonic.cuh -- warp-register bitonic sorting network (north-star subsystem 2).
//
// The network is the reference's same-direction bitonic network
// (_kernels.py:30-58, smallsort.py:88-117): for every block size s a
// *crossing* round compares slot i with slot (blk + s-1-k), i.e. partner
// i ^ (s-1), then *linear* rounds of halving distance d compare i with
// i ^ d.  Every comparator leaves the minimum at the lower index, so padding
// with the sentinel (INT32_MAX / +inf) at the end cannot change the written
// prefix (sentinel padding by count, _kernels.py:97-113).
//
// Key/value: a pair is swapped only on a strict key inversion (b < a),
// exactly as _kv_net (_kernels.py:60-95), so equal keys keep their values.
//
// Layout: one warp holds P = 32*E slots, slot q = lane*E + r lives in
// register r of `lane` (blocked).  Comparators whose XOR distance is < E are
// in-register; larger distances cross lanes with __shfl_xor_sync (lane mask
// = dist / E, register mask = dist % E).  Each side of a cross-lane pair
// computes its own half from the *old* values.
//
// Everything is branch-free: keys-only comparators are min/max (one
// VIMNMX / DMNMX each, the lane's side picked by a per-round predicate);
// key/value comparators use a strict-inversion predicate and selects.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace vx {

__device__ __forceinline__ int32_t kmin(int32_t a, int32_t b) { return min(a, b); }
__device__ __forceinline__ int32_t kmax(int32_t a, int32_t b) { return max(a, b); }
// plain ordered compares (NaN unsupported): DSETP + selects, no NaN fix-ups
__device__ __forceinline__ double kmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double kmax(double a, double b) { return b < a ? a : b; }
__device__ __forceinline__ uint32_t kmin(uint32_t a, uint32_t b) { return min(a, b); }
__device__ __forceinline__ uint32_t kmax(uint32_t a, uint32_t b) { return max(a, b); }
__device__ __forceinline__ uint64_t kmin(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t kmax(uint64_t a, uint64_t b) { return a < b ? b : a; }

// G (a power of two <= 32) lanes sort one network of P = G*E slots; a warp
// runs 32/G independent networks side by side (every shuffle stays inside
// its group of G lanes).  Fewer lanes and more registers per lane turn
// cross-lane rounds (shuffle + two selects per slot) into in-register
// rounds (one min/max per slot).
//
// MIX (int32 keys only): integer min / max issue on the half-rate ALU pipe,
// which bounds a keys-only network.  Two of every three in-register
// comparators compute the maximum as a + b - min(a, b) with two IMADs (the
// FMA pipe, idle otherwise; exact in two's complement), which balances the
// two pipes.  The multiplier is the launch's gridDim.y (= 1), opaque to
// ptxas, so the multiply-adds are not folded back into ALU adds.
template <typename K, typename V, int E, int G = 32, bool MIX = false>
struct WarpBitonic {
    static constexpr int P = G * E;
    static constexpr bool KV = HasVal<V>::value;
    static constexpr bool MIXED = MIX && !KV && std::is_same<K, int32_t>::value;

    // one comparator round with XOR distance MASK over all P slots
    template <int MASK>
    __device__ __forceinline__ static void round(K (&k)[E], V (&v)[E]) {
        if constexpr (MASK < E) {
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int r2 = r ^ MASK;
                if (r < r2) {  // slot r is the lower index: minimum stays at r
                    const K a = k[r], b = k[r2];
                    if constexpr (KV) {
                        const bool sw = b < a;  // strict inversion only
                        k[r] = sw ? b : a;
                        k[r2] = sw ? a : b;
                        const V x = v[r], y = v[r2];
                        v[r] = sw ? y : x;
                        v[r2] = sw ? x : y;
                    } else if constexpr (MIXED) {
                        if ((r + (r >> 2)) % 3 != 0) {
                            const int one = (int)gridDim.y;
                            const int mn = min((int)a, (int)b);
                            int t, mx;
                            asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(t) : "r"((int)a), "r"(one), "r"((int)b));
                            asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(mx) : "r"(mn), "r"(-one), "r"(t));
                            k[r] = (K)mn;
                            k[r2] = (K)mx;
                        } else {
                            k[r] = kmin(a, b);
                            k[r2] = kmax(a, b);
                        }
                    } else {
                        k[r] = kmin(a, b);
                        k[r2] = kmax(a, b);
                    }
                }
            }
        } else {
            constexpr int LM = MASK / E;  // lane xor mask
            constexpr int RM = MASK % E;  // register xor mask (E-1 on crossing rounds, else 0)
            constexpr int HB = 1 << (31 - __builtin_clz(LM));  // highest lane bit
            const int lane = threadIdx.x & 31;
            const bool low = (lane & HB) == 0;  // this lane holds the lower slots
            // slot r's partner value is the partner lane's register r ^ RM;
            // registers are updated pairwise {r, r ^ RM} from old values, so
            // at most two partner values are live at a time
            auto upd = [&](K& mk, V& mv, K pk, V pv) {
                if constexpr (KV) {
                    // low side takes the partner iff partner < mine, high side
                    // iff partner > mine: strict inversion, branch-free
                    const int lt = pk < mk, ne = pk != mk;
                    const int t = ne & (lt ^ (int)!low);
                    mk = t ? pk : mk;
                    mv = t ? pv : mv;
                } else {
                    if constexpr (std::is_floating_point<K>::value) {
                        // +0.0 and -0.0 compare equal but are different keys.
                        // min on the low lane and max on the high lane must
                        // resolve that tie the same way -- both lanes keep their
                        // own key -- or the high lane takes its partner's zero
                        // and the pair ends up holding the same zero twice.
                        // One ordered compare with the operands swapped on the
                        // high lane: exchange iff (high lane's key) < (low lane's).
                        const K hi_k = low ? pk : mk, lo_k = low ? mk : pk;
                        mk = hi_k < lo_k ? pk : mk;
                    } else {
                        mk = low ? kmin(mk, pk) : kmax(mk, pk);
                    }
                }
            };
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int r2 = r ^ RM;
                if (r2 < r) continue;  // handled with its pair
                const K pa = __shfl_xor_sync(0xffffffffu, k[r2], LM);
                V va{};
                if constexpr (KV) va = __shfl_xor_sync(0xffffffffu, v[r2], LM);
                if (r2 == r) {
                    upd(k[r], v[r], pa, va);
                } else {
                    const K pb = __shfl_xor_sync(0xffffffffu, k[r], LM);
                    V vb{};
                    if constexpr (KV) vb = __shfl_xor_sync(0xffffffffu, v[r], LM);
                    upd(k[r], v[r], pa, va);
                    upd(k[r2], v[r2], pb, vb);
                }
            }
        }
    }

    template <int S, int D>
    __device__ __forceinline__ static void linear(K (&k)[E], V (&v)[E]) {
        if constexpr (D >= 1) {
            round<D>(k, v);
            linear<S, D / 2>(k, v);
        }
    }

    template <int S>
    __device__ __forceinline__ static void stage(K (&k)[E], V (&v)[E]) {
        if constexpr (S <= P) {
            round<S - 1>(k, v);      // crossing round: partner i ^ (s-1)
            linear<S, S / 4>(k, v);  // linear rounds d = s/4 .. 1
            stage<S * 2>(k, v);
        }
    }

    __device__ __forceinline__ static void sort(K (&k)[E], V (&v)[E]) { stage<2>(k, v); }
};

// Sort one region of `len` (<= 32*E) elements: load blocked with sentinel
// padding by count, run the network, write back exactly `len` elements.
// src and dst may alias (in-place) -- every lane reads all its slots before
// any lane writes.
template <typename K, typename V, int E>
__device__ __forceinline__ void warp_sort_region(const K* src_k, const V* src_v, K* dst_k, V* dst_v,
                                                 uint64_t start, uint32_t len) {
    constexpr bool KV = HasVal<V>::value;
    using R = KeyRep<K>;
    using I = typename R::I;
    const int lane = threadIdx.x & 31;
    I k[E];
    V v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const uint32_t q = lane * E + r;
        k[r] = q < len ? R::to(src_k[start + q]) : KeyTraits<I>::sentinel();
        if constexpr (KV) v[r] = q < len ? src_v[start + q] : V();
    }
    __syncwarp();
    WarpBitonic<I, V, E>::sort(k, v);
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const uint32_t q = lane * E + r;
        if (q < len) {
            dst_k[start + q] = R::from(k[r]);
            if constexpr (KV) dst_v[start + q] = v[r];
        }
    }
}

// Dispatch on the padded size class (P = 32, 64, 128, 256).  Returns false
// if len exceeds 256.
template <typename K, typename V>
__device__ __forceinline__ bool warp_sort_any(const K* src_k, const V* src_v, K* dst_k, V* dst_v,
                                              uint64_t start, uint32_t len) {
    if (len <= 32) {
        warp_sort_region<K, V, 1>(src_k, src_v, dst_k, dst_v, start, len);
    } else if (len <= 64) {
        warp_sort_region<K, V, 2>(src_k, src_v, dst_k, dst_v, start, len);
    } else if (len <= 128) {
        warp_sort_region<K, V, 4>(src_k, src_v, dst_k, dst_v, start, len);
    } else if (len <= 256) {
        warp_sort_region<K, V, 8>(src_k, src_v, dst_k, dst_v, start, len);
    } else {
        return false;
    }
    return true;
}

// Pointer-offset form: sort src[0..len) into dst[0..len) (src may alias dst,
// and may live in shared memory).
template <typename K, typename V>
__device__ __forceinline__ bool warp_sort_any2(const K* src_k, const V* src_v, K* dst_k, V* dst_v, uint32_t len) {
    return warp_sort_any<K, V>(src_k, src_v, dst_k, dst_v, 0, len);
}

}  // namespace vx
