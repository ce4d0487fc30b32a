/*
 * vexsort_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's native region kernels
 * (/root/reference/pkg/src/vexsort/_kernels.py, numba-JIT'd Python) used as
 * the CPU checker for the B200 kernels.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library;
 * the product path (paper_1704_08579_b200/) never does.
 *
 * Every function follows the reference statement for statement so that the
 * *layouts* it produces (partitioned arrays, kv value order among equal keys)
 * are bit-identical to the reference's native backend; this is pinned against
 * fixtures generated from the reference itself (tests/golden/, made by
 * tests/golden/make_golden.py) in tests/test_oracle.py.
 *
 * Types: keys int32 ("i32") or float64 ("f64"); kv values have the key's
 * element width (int32 values for i32 keys, 64-bit values for f64 keys),
 * mirroring _check_kv (keyvalue.py:44-47).
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -shared -fPIC).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define LCG_MUL 6364136223846793005ULL /* _kernels.py:375 */
#define LCG_ADD 1442695040888963407ULL /* _kernels.py:376 */

int vxo_max_threads(void);

/* ------------------------------------------------------------------------ */
/* Key-only kernels, instantiated for int32 and double.                       */
/* ------------------------------------------------------------------------ */
#define DEFINE_KEY_KERNELS(SUF, T)                                             \
    /* _net (_kernels.py:30-58): same-direction bitonic network; one crossing  \
     * round per block size, then halving linear rounds; minima low. */        \
    static void net_##SUF(T *buf, int64_t base, int64_t n) {                   \
        for (int64_t s = 2; s <= n; s <<= 1) {                                 \
            int64_t half = s >> 1;                                             \
            for (int64_t blk = base; blk < base + n; blk += s)                 \
                for (int64_t k = 0; k < half; k++) {                           \
                    int64_t i = blk + k, j = blk + s - 1 - k;                  \
                    T a = buf[i], b = buf[j];                                  \
                    buf[i] = (a <= b) ? a : b;                                 \
                    buf[j] = (a <= b) ? b : a;                                 \
                }                                                              \
            for (int64_t d = s >> 2; d >= 1; d >>= 1) {                        \
                int64_t step = d << 1;                                         \
                for (int64_t blk = base; blk < base + n; blk += step)          \
                    for (int64_t k = 0; k < d; k++) {                          \
                        int64_t i = blk + k, j = i + d;                        \
                        T a = buf[i], b = buf[j];                              \
                        buf[i] = (a <= b) ? a : b;                             \
                        buf[j] = (a <= b) ? b : a;                             \
                    }                                                          \
            }                                                                  \
        }                                                                      \
    }                                                                          \
    /* _smallsort_impl (_kernels.py:97-113): pad to pow2 with the sentinel    \
     * in scratch, sort, write back `length` only. */                          \
    static void smallsort_impl_##SUF(T *arr, int64_t lo, int64_t length,       \
                                     T sentinel, T *scratch) {                 \
        if (length < 2) return;                                                \
        int64_t n = 2;                                                         \
        while (n < length) n <<= 1;                                            \
        if (n == length) { net_##SUF(arr, lo, n); return; }                    \
        for (int64_t i = 0; i < length; i++) scratch[i] = arr[lo + i];         \
        for (int64_t i = length; i < n; i++) scratch[i] = sentinel;            \
        net_##SUF(scratch, 0, n);                                              \
        for (int64_t i = 0; i < length; i++) arr[lo + i] = scratch[i];         \
    }                                                                          \
    /* smallsort_region (_kernels.py:115-126), uncapped length. */             \
    int vxo_smallsort_region_##SUF(T *arr, int64_t lo, int64_t length,        \
                                   T sentinel) {                               \
        if (length < 2) return 0;                                              \
        int64_t n = 2;                                                         \
        while (n < length) n <<= 1;                                            \
        if (n == length) { net_##SUF(arr, lo, n); return 0; }                  \
        T *scratch = (T *)malloc(sizeof(T) * (size_t)n);                       \
        if (!scratch) return -1;                                               \
        smallsort_impl_##SUF(arr, lo, length, sentinel, scratch);              \
        free(scratch);                                                         \
        return 0;                                                              \
    }                                                                          \
    /* scalar_partition (_kernels.py:162-171). */                              \
    static int64_t scalar_partition_##SUF(T *arr, int64_t lo, int64_t hi,     \
                                          T pivot) {                           \
        int64_t w = lo;                                                        \
        for (int64_t i = lo; i < hi; i++) {                                    \
            T v = arr[i];                                                      \
            if (v <= pivot) { arr[i] = arr[w]; arr[w] = v; w++; }              \
        }                                                                      \
        return w;                                                              \
    }                                                                          \
    /* _split_pack (_kernels.py:187-212). */                                   \
    static void split_pack_##SUF(T *arr, const T *val, int64_t nb, T pivot,    \
                                 int64_t *left_w, int64_t *right_w,            \
                                 int opt_a) {                                  \
        int64_t nb_low = 0;                                                    \
        for (int64_t k = 0; k < nb; k++) if (val[k] <= pivot) nb_low++;        \
        int64_t nb_high = nb - nb_low;                                         \
        int64_t li = *left_w, ri = *right_w - nb_high;                         \
        if (nb_low > 0 || !opt_a)                                              \
            for (int64_t k = 0; k < nb; k++) {                                 \
                T v = val[k];                                                  \
                if (v <= pivot) arr[li++] = v;                                 \
            }                                                                  \
        if (nb_high > 0 || !opt_a)                                             \
            for (int64_t k = 0; k < nb; k++) {                                 \
                T v = val[k];                                                  \
                if (!(v <= pivot)) arr[ri++] = v;                              \
            }                                                                  \
        *left_w += nb_low;                                                     \
        *right_w -= nb_high;                                                   \
    }                                                                          \
    /* _partition_impl (_kernels.py:214-255): two-cursor in-place partition; \
     * both extremity packs buffered, load from the side with less free      \
     * space, then remainder, left buffer, right buffer. */                    \
    static int64_t partition_impl_##SUF(T *arr, int64_t lo, int64_t hi,        \
                                        T pivot, int64_t lane, int opt_a,      \
                                        int opt_b, T *val, T *lbuf, T *rbuf) { \
        int64_t n = hi - lo;                                                   \
        if (n <= 2 * lane) return scalar_partition_##SUF(arr, lo, hi, pivot);  \
        int64_t left = lo, left_w = lo, right = hi - lane, right_w = hi;       \
        for (int64_t k = 0; k < lane; k++) {                                   \
            lbuf[k] = arr[lo + k];                                             \
            rbuf[k] = arr[right + k];                                          \
        }                                                                      \
        left += lane;                                                          \
        while (left + lane <= right) {                                         \
            int64_t off;                                                       \
            if (left - left_w <= right_w - right) {                            \
                off = left;                                                    \
                left += lane;                                                  \
                if (opt_b)                                                     \
                    for (int64_t k = 0; k < lane; k++) {                       \
                        val[k] = lbuf[k];                                      \
                        lbuf[k] = arr[off + k];                                \
                    }                                                          \
                else                                                           \
                    for (int64_t k = 0; k < lane; k++) val[k] = arr[off + k];  \
            } else {                                                           \
                right -= lane;                                                 \
                off = right;                                                   \
                if (opt_b)                                                     \
                    for (int64_t k = 0; k < lane; k++) {                       \
                        val[k] = rbuf[k];                                      \
                        rbuf[k] = arr[off + k];                                \
                    }                                                          \
                else                                                           \
                    for (int64_t k = 0; k < lane; k++) val[k] = arr[off + k];  \
            }                                                                  \
            split_pack_##SUF(arr, val, lane, pivot, &left_w, &right_w, opt_a); \
        }                                                                      \
        int64_t rem = right - left;                                            \
        for (int64_t k = 0; k < rem; k++) val[k] = arr[left + k];              \
        split_pack_##SUF(arr, val, rem, pivot, &left_w, &right_w, opt_a);      \
        split_pack_##SUF(arr, lbuf, lane, pivot, &left_w, &right_w, opt_a);    \
        split_pack_##SUF(arr, rbuf, lane, pivot, &left_w, &right_w, opt_a);    \
        return left_w;                                                         \
    }                                                                          \
    /* partition (_kernels.py:257-262).  lane <= 64. */                        \
    int64_t vxo_partition_##SUF(T *arr, int64_t lo, int64_t hi, T pivot,       \
                                int64_t lane, int opt_a, int opt_b) {          \
        T val[64], lbuf[64], rbuf[64];                                         \
        if (lane < 1 || lane > 64) return -1;                                  \
        return partition_impl_##SUF(arr, lo, hi, pivot, lane, opt_a, opt_b,    \
                                    val, lbuf, rbuf);                          \
    }                                                                          \
    int64_t vxo_scalar_partition_##SUF(T *arr, int64_t lo, int64_t hi,        \
                                       T pivot) {                              \
        return scalar_partition_##SUF(arr, lo, hi, pivot);                     \
    }                                                                          \
    /* _pivot_index (_kernels.py:358-373): 0 median3, 1 middle, 2 random. */  \
    static int64_t pivot_index_##SUF(const T *arr, int64_t lo, int64_t hi,     \
                                     int strategy, uint64_t lcg) {             \
        if (strategy == 1) return (lo + hi) / 2;                               \
        if (strategy == 2) {                                                   \
            uint64_t span = (uint64_t)(hi - lo + 1);                           \
            return lo + (int64_t)(lcg % span);                                 \
        }                                                                      \
        int64_t mid = (lo + hi) / 2;                                           \
        T a = arr[lo], b = arr[mid], c = arr[hi];                              \
        if ((b <= a && a <= c) || (c <= a && a <= b)) return lo;               \
        if ((a <= b && b <= c) || (c <= b && b <= a)) return mid;              \
        return hi;                                                             \
    }                                                                          \
    /* One quicksort work loop over the inclusive range [lo0, hi0]            \
     * (_kernels.py:378-423).  With par_min > 0 the deferred larger side is   \
     * spawned as an OpenMP task when it exceeds par_min elements (the        \
     * paper's future-work task parallelism); the sorted output \
     * is identical either way. */                                             \
    static void qs_loop_##SUF(T *arr, int64_t lo0, int64_t hi0, int64_t lane,  \
                              int64_t sort_bound, T sentinel, int strategy,    \
                              int opt_a, int opt_b, uint64_t lcg,              \
                              int64_t par_min) {                               \
        T scratch[16 * 64], val[64], lbuf[64], rbuf[64];                       \
        int64_t stack[96][2];                                                  \
        stack[0][0] = lo0;                                                     \
        stack[0][1] = hi0;                                                     \
        int top = 1;                                                           \
        while (top > 0) {                                                      \
            top--;                                                             \
            int64_t lo = stack[top][0], hi = stack[top][1];                    \
            while (hi - lo + 1 > sort_bound) {                                 \
                if (strategy == 2) lcg = lcg * LCG_MUL + LCG_ADD;              \
                int64_t pidx = pivot_index_##SUF(arr, lo, hi, strategy, lcg);  \
                T t = arr[pidx];                                               \
                arr[pidx] = arr[hi];                                           \
                arr[hi] = t;                                                   \
                T pivot = arr[hi];                                             \
                int64_t b = partition_impl_##SUF(arr, lo, hi, pivot, lane,     \
                                                 opt_a, opt_b, val, lbuf,      \
                                                 rbuf);                        \
                t = arr[b];                                                    \
                arr[b] = arr[hi];                                              \
                arr[hi] = t;                                                   \
                int64_t dlo, dhi; /* deferred larger side */                   \
                if (b - lo < hi - b) {                                         \
                    dlo = b + 1; dhi = hi; hi = b - 1;                         \
                } else {                                                       \
                    dlo = lo; dhi = b - 1; lo = b + 1;                         \
                }                                                              \
                if (dlo < dhi) {                                               \
                    if (par_min > 0 && dhi - dlo + 1 > par_min) {              \
                        uint64_t l2 = lcg;                                     \
                        _Pragma("omp task firstprivate(dlo, dhi, l2)")         \
                        qs_loop_##SUF(arr, dlo, dhi, lane, sort_bound,         \
                                      sentinel, strategy, opt_a, opt_b, l2,    \
                                      par_min);                                \
                    } else {                                                   \
                        stack[top][0] = dlo;                                   \
                        stack[top][1] = dhi;                                   \
                        top++;                                                 \
                    }                                                          \
                }                                                              \
            }                                                                  \
            if (hi - lo >= 1)                                                  \
                smallsort_impl_##SUF(arr, lo, hi - lo + 1, sentinel, scratch); \
        }                                                                      \
    }                                                                          \
    /* quicksort (_kernels.py:378-423).  sort_bound <= 16*lane, lane <= 64. */ \
    int vxo_quicksort_##SUF(T *arr, int64_t n, int64_t lane,                   \
                            int64_t sort_bound, T sentinel, int strategy,      \
                            int opt_a, int opt_b, uint64_t seed) {             \
        if (lane < 1 || lane > 64 || sort_bound < 1 || sort_bound > 16 * lane) \
            return -1;                                                         \
        if (n < 2) return 0;                                                   \
        uint64_t lcg = seed * LCG_MUL + LCG_ADD;                               \
        qs_loop_##SUF(arr, 0, n - 1, lane, sort_bound, sentinel, strategy,     \
                      opt_a, opt_b, lcg, 0);                                   \
        return 0;                                                              \
    }                                                                          \
    /* Task-parallel variant (same output); nthreads <= 0 uses all cores. */  \
    int vxo_quicksort_mt_##SUF(T *arr, int64_t n, int64_t lane,                \
                               int64_t sort_bound, T sentinel, int strategy,   \
                               int opt_a, int opt_b, uint64_t seed,            \
                               int nthreads) {                                 \
        if (lane < 1 || lane > 64 || sort_bound < 1 || sort_bound > 16 * lane) \
            return -1;                                                         \
        if (n < 2) return 0;                                                   \
        uint64_t lcg = seed * LCG_MUL + LCG_ADD;                               \
        int64_t par_min = 1 << 16;                                             \
        if (nthreads <= 0) nthreads = vxo_max_threads();                       \
        _Pragma("omp parallel num_threads(nthreads)")                          \
        _Pragma("omp single")                                                  \
        qs_loop_##SUF(arr, 0, n - 1, lane, sort_bound, sentinel, strategy,     \
                      opt_a, opt_b, lcg, par_min);                             \
        return 0;                                                              \
    }

/* ------------------------------------------------------------------------ */
/* Key/value kernels.                                                         */
/* ------------------------------------------------------------------------ */
#define DEFINE_KV_KERNELS(SUF, K, V)                                           \
    /* _kv_net (_kernels.py:60-95): swap a pair only on strict inversion. */  \
    static void kv_net_##SUF(K *kb, V *vb, int64_t base, int64_t n) {          \
        for (int64_t s = 2; s <= n; s <<= 1) {                                 \
            int64_t half = s >> 1;                                             \
            for (int64_t blk = base; blk < base + n; blk += s)                 \
                for (int64_t k = 0; k < half; k++) {                           \
                    int64_t i = blk + k, j = blk + s - 1 - k;                  \
                    K a = kb[i], b = kb[j];                                    \
                    if (b < a) {                                               \
                        kb[i] = b; kb[j] = a;                                  \
                        V x = vb[i]; vb[i] = vb[j]; vb[j] = x;                 \
                    }                                                          \
                }                                                              \
            for (int64_t d = s >> 2; d >= 1; d >>= 1) {                        \
                int64_t step = d << 1;                                         \
                for (int64_t blk = base; blk < base + n; blk += step)          \
                    for (int64_t k = 0; k < d; k++) {                          \
                        int64_t i = blk + k, j = i + d;                        \
                        K a = kb[i], b = kb[j];                                \
                        if (b < a) {                                           \
                            kb[i] = b; kb[j] = a;                              \
                            V x = vb[i]; vb[i] = vb[j]; vb[j] = x;             \
                        }                                                      \
                    }                                                          \
            }                                                                  \
        }                                                                      \
    }                                                                          \
    /* _kv_smallsort_impl (_kernels.py:128-146). */                            \
    static void kv_smallsort_impl_##SUF(K *keys, V *vals, int64_t lo,          \
                                        int64_t length, K sentinel,            \
                                        K *ks, V *vs) {                        \
        if (length < 2) return;                                                \
        int64_t n = 2;                                                         \
        while (n < length) n <<= 1;                                            \
        if (n == length) { kv_net_##SUF(keys, vals, lo, n); return; }          \
        for (int64_t i = 0; i < length; i++) {                                 \
            ks[i] = keys[lo + i];                                              \
            vs[i] = vals[lo + i];                                              \
        }                                                                      \
        /* padded value slots are left as-is, as in the reference (np.empty) */\
        for (int64_t i = length; i < n; i++) { ks[i] = sentinel; vs[i] = 0; }  \
        kv_net_##SUF(ks, vs, 0, n);                                            \
        for (int64_t i = 0; i < length; i++) {                                 \
            keys[lo + i] = ks[i];                                              \
            vals[lo + i] = vs[i];                                              \
        }                                                                      \
    }                                                                          \
    int vxo_kv_smallsort_region_##SUF(K *keys, V *vals, int64_t lo,            \
                                      int64_t length, K sentinel) {            \
        if (length < 2) return 0;                                              \
        int64_t n = 2;                                                         \
        while (n < length) n <<= 1;                                            \
        if (n == length) { kv_net_##SUF(keys, vals, lo, n); return 0; }        \
        K *ks = (K *)malloc(sizeof(K) * (size_t)n);                            \
        V *vs = (V *)malloc(sizeof(V) * (size_t)n);                            \
        if (!ks || !vs) { free(ks); free(vs); return -1; }                     \
        kv_smallsort_impl_##SUF(keys, vals, lo, length, sentinel, ks, vs);     \
        free(ks);                                                              \
        free(vs);                                                              \
        return 0;                                                              \
    }                                                                          \
    /* kv_scalar_partition (_kernels.py:173-185). */                           \
    static int64_t kv_scalar_partition_##SUF(K *keys, V *vals, int64_t lo,     \
                                             int64_t hi, K pivot) {            \
        int64_t w = lo;                                                        \
        for (int64_t i = lo; i < hi; i++) {                                    \
            K k = keys[i];                                                     \
            if (k <= pivot) {                                                  \
                keys[i] = keys[w]; keys[w] = k;                                \
                V x = vals[i]; vals[i] = vals[w]; vals[w] = x;                 \
                w++;                                                           \
            }                                                                  \
        }                                                                      \
        return w;                                                              \
    }                                                                          \
    int64_t vxo_kv_scalar_partition_##SUF(K *keys, V *vals, int64_t lo,        \
                                          int64_t hi, K pivot) {               \
        return kv_scalar_partition_##SUF(keys, vals, lo, hi, pivot);           \
    }                                                                          \
    /* _kv_split_pack (_kernels.py:264-288). */                                \
    static void kv_split_pack_##SUF(K *keys, V *vals, const K *kv_,            \
                                    const V *vv, int64_t nb, K pivot,          \
                                    int64_t *left_w, int64_t *right_w,         \
                                    int opt_a) {                               \
        int64_t nb_low = 0;                                                    \
        for (int64_t k = 0; k < nb; k++) if (kv_[k] <= pivot) nb_low++;        \
        int64_t nb_high = nb - nb_low;                                         \
        int64_t li = *left_w, ri = *right_w - nb_high;                         \
        if (nb_low > 0 || !opt_a)                                              \
            for (int64_t k = 0; k < nb; k++)                                   \
                if (kv_[k] <= pivot) { keys[li] = kv_[k]; vals[li] = vv[k];    \
                                       li++; }                                 \
        if (nb_high > 0 || !opt_a)                                             \
            for (int64_t k = 0; k < nb; k++)                                   \
                if (!(kv_[k] <= pivot)) { keys[ri] = kv_[k]; vals[ri] = vv[k]; \
                                          ri++; }                              \
        *left_w += nb_low;                                                     \
        *right_w -= nb_high;                                                   \
    }                                                                          \
    /* _kv_partition_impl (_kernels.py:290-345). */                            \
    static int64_t kv_partition_impl_##SUF(K *keys, V *vals, int64_t lo,       \
                                           int64_t hi, K pivot, int64_t lane,  \
                                           int opt_a, int opt_b) {             \
        K kval[64], klbuf[64], krbuf[64];                                      \
        V vval[64], vlbuf[64], vrbuf[64];                                      \
        int64_t n = hi - lo;                                                   \
        if (n <= 2 * lane)                                                     \
            return kv_scalar_partition_##SUF(keys, vals, lo, hi, pivot);       \
        int64_t left = lo, left_w = lo, right = hi - lane, right_w = hi;       \
        for (int64_t k = 0; k < lane; k++) {                                   \
            klbuf[k] = keys[lo + k]; vlbuf[k] = vals[lo + k];                  \
            krbuf[k] = keys[right + k]; vrbuf[k] = vals[right + k];            \
        }                                                                      \
        left += lane;                                                          \
        while (left + lane <= right) {                                         \
            int64_t off;                                                       \
            if (left - left_w <= right_w - right) {                            \
                off = left;                                                    \
                left += lane;                                                  \
                if (opt_b)                                                     \
                    for (int64_t k = 0; k < lane; k++) {                       \
                        kval[k] = klbuf[k]; vval[k] = vlbuf[k];                \
                        klbuf[k] = keys[off + k]; vlbuf[k] = vals[off + k];    \
                    }                                                          \
                else                                                           \
                    for (int64_t k = 0; k < lane; k++) {                       \
                        kval[k] = keys[off + k]; vval[k] = vals[off + k];      \
                    }                                                          \
            } else {                                                           \
                right -= lane;                                                 \
                off = right;                                                   \
                if (opt_b)                                                     \
                    for (int64_t k = 0; k < lane; k++) {                       \
                        kval[k] = krbuf[k]; vval[k] = vrbuf[k];                \
                        krbuf[k] = keys[off + k]; vrbuf[k] = vals[off + k];    \
                    }                                                          \
                else                                                           \
                    for (int64_t k = 0; k < lane; k++) {                       \
                        kval[k] = keys[off + k]; vval[k] = vals[off + k];      \
                    }                                                          \
            }                                                                  \
            kv_split_pack_##SUF(keys, vals, kval, vval, lane, pivot, &left_w,  \
                                &right_w, opt_a);                              \
        }                                                                      \
        int64_t rem = right - left;                                            \
        for (int64_t k = 0; k < rem; k++) {                                    \
            kval[k] = keys[left + k]; vval[k] = vals[left + k];                \
        }                                                                      \
        kv_split_pack_##SUF(keys, vals, kval, vval, rem, pivot, &left_w,       \
                            &right_w, opt_a);                                  \
        kv_split_pack_##SUF(keys, vals, klbuf, vlbuf, lane, pivot, &left_w,    \
                            &right_w, opt_a);                                  \
        kv_split_pack_##SUF(keys, vals, krbuf, vrbuf, lane, pivot, &left_w,    \
                            &right_w, opt_a);                                  \
        return left_w;                                                         \
    }                                                                          \
    int64_t vxo_kv_partition_##SUF(K *keys, V *vals, int64_t lo, int64_t hi,   \
                                   K pivot, int64_t lane, int opt_a,           \
                                   int opt_b) {                                \
        if (lane < 1 || lane > 64) return -1;                                  \
        return kv_partition_impl_##SUF(keys, vals, lo, hi, pivot, lane, opt_a, \
                                       opt_b);                                 \
    }                                                                          \
    /* kv_quicksort (_kernels.py:425-482). */                                  \
    static void kv_qs_loop_##SUF(K *keys, V *vals, int64_t lo0, int64_t hi0,   \
                                 int64_t lane, int64_t sort_bound, K sentinel, \
                                 int strategy, int opt_a, int opt_b,           \
                                 uint64_t lcg, int64_t par_min) {              \
        K ks[16 * 64];                                                         \
        V vs[16 * 64];                                                         \
        int64_t stack[96][2];                                                  \
        stack[0][0] = lo0;                                                     \
        stack[0][1] = hi0;                                                     \
        int top = 1;                                                           \
        while (top > 0) {                                                      \
            top--;                                                             \
            int64_t lo = stack[top][0], hi = stack[top][1];                    \
            while (hi - lo + 1 > sort_bound) {                                 \
                if (strategy == 2) lcg = lcg * LCG_MUL + LCG_ADD;              \
                int64_t pidx = kv_pivot_index_##SUF(keys, lo, hi, strategy,    \
                                                    lcg);                      \
                K t = keys[pidx]; keys[pidx] = keys[hi]; keys[hi] = t;         \
                V x = vals[pidx]; vals[pidx] = vals[hi]; vals[hi] = x;         \
                K pivot = keys[hi];                                            \
                int64_t b = kv_partition_impl_##SUF(keys, vals, lo, hi, pivot, \
                                                    lane, opt_a, opt_b);       \
                t = keys[b]; keys[b] = keys[hi]; keys[hi] = t;                 \
                x = vals[b]; vals[b] = vals[hi]; vals[hi] = x;                 \
                int64_t dlo, dhi;                                              \
                if (b - lo < hi - b) {                                         \
                    dlo = b + 1; dhi = hi; hi = b - 1;                         \
                } else {                                                       \
                    dlo = lo; dhi = b - 1; lo = b + 1;                         \
                }                                                              \
                if (dlo < dhi) {                                               \
                    if (par_min > 0 && dhi - dlo + 1 > par_min) {              \
                        uint64_t l2 = lcg;                                     \
                        _Pragma("omp task firstprivate(dlo, dhi, l2)")         \
                        kv_qs_loop_##SUF(keys, vals, dlo, dhi, lane,           \
                                         sort_bound, sentinel, strategy,       \
                                         opt_a, opt_b, l2, par_min);           \
                    } else {                                                   \
                        stack[top][0] = dlo;                                   \
                        stack[top][1] = dhi;                                   \
                        top++;                                                 \
                    }                                                          \
                }                                                              \
            }                                                                  \
            if (hi - lo >= 1)                                                  \
                kv_smallsort_impl_##SUF(keys, vals, lo, hi - lo + 1, sentinel, \
                                        ks, vs);                               \
        }                                                                      \
    }                                                                          \
    int vxo_kv_quicksort_##SUF(K *keys, V *vals, int64_t n, int64_t lane,      \
                               int64_t sort_bound, K sentinel, int strategy,   \
                               int opt_a, int opt_b, uint64_t seed,            \
                               int nthreads) {                                 \
        if (lane < 1 || lane > 64 || sort_bound < 1 || sort_bound > 16 * lane) \
            return -1;                                                         \
        if (n < 2) return 0;                                                   \
        uint64_t lcg = seed * LCG_MUL + LCG_ADD;                               \
        if (nthreads == 1) {                                                   \
            kv_qs_loop_##SUF(keys, vals, 0, n - 1, lane, sort_bound, sentinel, \
                             strategy, opt_a, opt_b, lcg, 0);                  \
            return 0;                                                          \
        }                                                                      \
        if (nthreads <= 0) nthreads = vxo_max_threads();                       \
        _Pragma("omp parallel num_threads(nthreads)")                          \
        _Pragma("omp single")                                                  \
        kv_qs_loop_##SUF(keys, vals, 0, n - 1, lane, sort_bound, sentinel,     \
                         strategy, opt_a, opt_b, lcg, (int64_t)1 << 16);       \
        return 0;                                                              \
    }

int vxo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

DEFINE_KEY_KERNELS(i32, int32_t)
DEFINE_KEY_KERNELS(f64, double)

/* the kv drivers pick the pivot from the keys with the same rule */
#define kv_pivot_index_kvi32 pivot_index_i32
#define kv_pivot_index_kvf64 pivot_index_f64
DEFINE_KV_KERNELS(kvi32, int32_t, int32_t)
DEFINE_KV_KERNELS(kvf64, double, int64_t)
