/*
 * vexsort_b200.h -- C ABI of the B200-native hybrid sort.
 *
 * Drop-in boundary for the hot path of the reference package `vexsort`
 * (arXiv 1704.08579).  The reference's plugin boundary is the numba kernel
 * module pkg/src/vexsort/_kernels.py, called from quicksort.py,
 * partition.py, smallsort.py and keyvalue.py whenever
 * `backend.uses_kernels` (lanes.py:297).  Two families of entry points:
 *
 *  1. vx_host_* -- HOST-buffer twins of the _kernels.py functions, same
 *     argument order and meaning, in-place on caller memory; the library
 *     copies to the B200, runs the kernels and copies back.  These are what
 *     a maintainer binds in place of `_kernels`.
 *  2. vx_* device API -- device pointers, caller-provided workspace, an
 *     explicit cudaStream_t, stream-ordered and CUDA-graph capturable, no
 *     allocation; used by the PyTorch-facing Python package and bench.py.
 *     Calls run on the CURRENT device, whose memory the pointers must be.
 *
 * Element kinds (lanes.py:50-63, kind_of lanes.py:502-507): VX_I32 = int32
 * keys, VX_F64 = float64 keys.  Key/value values must have the key's element
 * width (keyvalue.py:44-47): 32-bit values with int32 keys, 64-bit values
 * with float64 keys; their bits are moved, never interpreted.
 *
 * Every function returns 0 (or a non-negative index) on success and a
 * negative VX_E* code on failure; vx_last_error() returns a thread-local
 * message for the last failure.  NaN keys are unsupported, as in the
 * reference (quicksort.py:140-141).
 */
#ifndef VEXSORT_B200_H
#define VEXSORT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *vx_stream_t; /* == cudaStream_t */

enum { VX_I32 = 0, VX_F64 = 1 };
enum {
    VX_OK = 0,
    VX_EINVAL = -1,    /* bad argument (reference: AssertionError / ValueError) */
    VX_ETYPE = -2,     /* unsupported dtype (reference: TypeError, lanes.py:507) */
    VX_ECUDA = -3,     /* CUDA runtime / launch failure */
    VX_EWORKSPACE = -4,/* workspace too small */
    VX_ECAPACITY = -5, /* internal queue capacity exceeded */
    VX_ETOOLONG = -6   /* a small-sort segment exceeds 256 elements */
};

/* SortConfig (quicksort.py:28-46).  sort_bound <= 0 selects the default
 * 16*lanes (256 int32 / 128 float64); it is the largest range handed to the
 * bitonic network and must be <= 16*lanes (quicksort.py:49-52).
 * pivot_strategy (0 median3, 1 middle, 2 random; VX_EINVAL otherwise)
 * selects how the sampled-pivot levels draw their sample: stratified hashed
 * positions (default), stratum midpoints, or the reference's MMIX LCG seeded
 * by pivot_seed (see qsort.cuh sample_pos).  The output is the same for all
 * three.  The two partition flags are CPU store-pattern variants of the
 * reference partition and do not apply on the GPU (accepted, ignored). */
typedef struct {
    int64_t sort_bound;
    int32_t pivot_strategy;
    int32_t skip_empty_stores;
    int32_t swap_buffered;
    int32_t flags; /* VX_SORT_* bits (0 = default) */
    uint64_t pivot_seed;
} vx_sort_config;

/* vx_sort_config.flags.  A sort normally runs its level loop from the host
 * (one 64-byte status read per partition level) the first few times it sees
 * a set of buffers, and replays a cached CUDA graph -- no host
 * synchronisation at all -- once the same buffers keep coming back;
 * VX_SORT_GRAPH builds the graph on the first call (steady-state loops),
 * VX_SORT_EAGER never builds one.  Inside a caller's stream capture the sort
 * always records itself into the caller's graph. */
#define VX_SORT_GRAPH 1
#define VX_SORT_EAGER 2

const char *vx_last_error(void);
int vx_version(void);

/* ------------------------------------------------------------------ device API */

/* Full hybrid sort, in place on device keys[n] (values[n] optional, may be
 * NULL).  Replaces _kernels.quicksort / kv_quicksort (_kernels.py:378-482)
 * as called by sort_with_config (quicksort.py:115-134) and kv_sort
 * (keyvalue.py:228-252). */
/* Inputs that are already in order leave early: a sort of >= 2^24 keys first
 * tests 512 evenly spaced adjacent pairs and, only if all of them rise (or
 * all fall), every adjacent pair in one read pass; a non-decreasing array is
 * then copied (or left in place), a non-increasing one written reversed
 * (csrc/presort.cuh; environment VX_NO_PRESORT switches the test off,
 * VX_PRESORT_MIN_N moves the threshold).  The output is the same either way. */
size_t vx_sort_workspace_bytes(int dtype, int has_values, int64_t n);
int vx_sort(int dtype, void *keys, void *values, int64_t n, const vx_sort_config *cfg, void *ws,
            size_t ws_bytes, vx_stream_t stream);
/* Out-of-place twin: sorted copy of in[n] into out[n]; the input is only
 * read (by the first partition level), so it costs no extra traffic.
 * in == out is the in-place vx_sort. */
int vx_sort_into(int dtype, const void *in_keys, const void *in_values, void *out_keys, void *out_values,
                 int64_t n, const vx_sort_config *cfg, void *ws, size_t ws_bytes, vx_stream_t stream);

/* Sorts are stream-ordered: vx_sort / vx_sort_into never synchronise.
 * Without per-launch timing (vx_profile_enable) the level loop runs as a
 * CUDA graph with a device-side WHILE condition, so both calls may also be
 * captured into the caller's own CUDA graph.  Errors found on the device
 * (work-queue capacity, level limit) land in the workspace; vx_sort_status
 * synchronises `stream`, returns VX_OK or VX_ECAPACITY for the last sort
 * that used `ws`, and fills `stats` (may be NULL). */
typedef struct {
    uint32_t err;             /* device error bits (0 = ok) */
    uint32_t levels;          /* partition levels run */
    uint32_t launches;        /* kernels launched by those levels */
    uint32_t reserved;
    uint64_t scatter_elems;   /* elements moved by the global scatter passes */
    uint64_t finish_elems;    /* elements sorted / copied by the finish kernel */
    uint64_t local_elems;     /* elements sorted by the CTA-local level */
} vx_sort_stats;
int vx_sort_status(const void *ws, int64_t n, vx_stream_t stream, vx_sort_stats *stats);

/* Pivot partition, out of place: out[0:split) <= pivot < out[split:n).
 * *pivot points to a HOST scalar of the key type.  The split (= count of
 * keys <= pivot) is written to the DEVICE int64 *d_split.  Replaces
 * _kernels.partition / kv_partition / scalar_partition (_kernels.py:162-262,
 * 264-356) as called by partition_region (partition.py:115-145) and
 * kv_partition_region (keyvalue.py:138-161). */
size_t vx_partition_workspace_bytes(int dtype, int64_t n);
int vx_partition(int dtype, const void *in_keys, const void *in_values, void *out_keys, void *out_values,
                 int64_t n, const void *pivot, int64_t *d_split, void *ws, size_t ws_bytes,
                 vx_stream_t stream);

/* Batched small sort of CSR segments [offs[s], offs[s+1]) in place, every
 * segment <= 256 elements (config 2).  Replaces one _kernels.smallsort_region
 * call per segment (_kernels.py:115-126; sort_small_region,
 * smallsort.py:218-252).  n is the length of keys (and values): segments
 * outside [0, n] are flagged, never touched.  ws >= 4 bytes holds a device
 * error flag that vx_segments_status() reads back (synchronising). */
int vx_sort_segments(int dtype, void *keys, void *values, int64_t n, const int64_t *d_offsets, int64_t nseg,
                     void *ws, size_t ws_bytes, vx_stream_t stream);
int vx_segments_status(void *ws, vx_stream_t stream);

/* Sharded sample sort building blocks (no reference counterpart; BASELINE
 * config 5).  Splitters are (key, global index) pairs so equal keys are
 * split by position.  Buckets: dest(x at global index g) = number of
 * splitters lexicographically below (x, g).  out is grouped by destination;
 * d_counts[nsplit+1] receives per-destination counts. */
size_t vx_bucket_partition_workspace_bytes(int dtype, int nsplit);
int vx_bucket_partition(int dtype, const void *in_keys, void *out_keys, int64_t n, uint64_t global_offset,
                        const void *d_split_keys, const uint64_t *d_split_idx, int nsplit,
                        unsigned long long *d_counts, void *ws, size_t ws_bytes, vx_stream_t stream);
int vx_select_splitters(int dtype, const void *d_sample_keys, const uint64_t *d_sample_idx, int64_t count,
                        int nparts, void *d_out_keys, uint64_t *d_out_idx, vx_stream_t stream);

/* Fused exchange: the bucket partition writes each
 * destination's run STRAIGHT into that destination's buffer -- on a
 * multi-GPU box a peer GPU's receive buffer mapped with CUDA IPC, so the
 * partition's stores are the NVLink transfer and no all-to-all copy
 * follows.  vx_bucket_counts: per-destination counts only (histogram pass).
 * vx_bucket_scatter_to: destination b's keys land in
 * ((K*)d_dst_ptrs[b])[d_dst_offsets[b] ...] (both device arrays of
 * nsplit+1 uint64; ws as for vx_bucket_partition).  The caller orders the
 * kernel before any reader (stream sync + a host barrier across ranks). */
int vx_bucket_counts(int dtype, const void *in_keys, int64_t n, uint64_t global_offset, const void *d_split_keys,
                     const uint64_t *d_split_idx, int nsplit, unsigned long long *d_counts, vx_stream_t stream);
int vx_bucket_scatter_to(int dtype, const void *in_keys, int64_t n, uint64_t global_offset,
                         const void *d_split_keys, const uint64_t *d_split_idx, int nsplit,
                         const unsigned long long *d_dst_ptrs, const unsigned long long *d_dst_offsets, void *ws,
                         size_t ws_bytes, vx_stream_t stream);
/* Receive buffers shared across processes: a cudaMalloc'd buffer, its
 * 64-byte IPC handle, and mapping / unmapping a peer's handle (peer access
 * enabled lazily).  vx_sort_from_ptr: vx_sort_into from a raw device
 * address (e.g. the receive buffer) into out_keys. */
int vx_ipc_alloc(size_t bytes, void **dptr);
int vx_ipc_free(void *dptr);
int vx_ipc_handle(const void *dptr, void *handle64);
int vx_ipc_open(const void *handle64, void **dptr);
int vx_ipc_close(void *dptr);
int vx_sort_from_ptr(int dtype, uint64_t in_keys, void *out_keys, int64_t n, const vx_sort_config *cfg, void *ws,
                     size_t ws_bytes, vx_stream_t stream);

/* Seeded synthetic inputs generated on the device (bench only).
 * dist: 0 uniform (int32 full range / f64 [-1e6,1e6)), 1 sorted, 2 reverse,
 * 3 few-unique [0,16), 4 standard normal (f64), 5 uniform [0,2^31) int32,
 * 6 index (values = global index). */
int vx_generate(int dtype, int dist, void *out, int64_t n, uint64_t seed, uint64_t global_offset,
                int64_t global_n, vx_stream_t stream);

/* Output verification on the device (the bench's correctness gate, the
 * size-independent form of benchcli.py:398-427 "equals np.sort").  Writes 4
 * device uint64 to d_out: [0] sum and [1] xor of a per-element hash of the
 * key bits (folded with the value bits when values != NULL) -- an
 * order-independent multiset digest; [2] adjacent inversions k[i+1] < k[i]
 * (0 when check_order == 0; counted only inside each CSR segment when
 * d_offsets[nseg+1] is given); [3] an order-dependent positional digest
 * sum_i mix64(bits(k[i]) ^ mix64(i)).  Stream-ordered. */
int vx_verify(int dtype, const void *keys, const void *values, int64_t n, int check_order,
              const int64_t *d_offsets, int64_t nseg, uint64_t *d_out, vx_stream_t stream);

/* Instrumentation.  Kernel launches are always counted per class; with
 * profiling enabled every launch is also bracketed by CUDA events on its
 * stream (sorts then run their level loop eagerly, host-driven).
 * Classes: 0 plan, 1 hist, 2 emit, 3 scatter, 4 finish, 5 partition,
 * 6 segsort, 7 bucket-partition, 8 CTA-local level.  vx_profile_read fills up to
 * nclass entries (launch counts, summed device ms, elements processed) and
 * returns the number of classes. */
int vx_profile_enable(int on);
int vx_profile_reset(void);
int vx_profile_read(int64_t *launches, double *ms, uint64_t *elems, int nclass);

/* ------------------------------------------------------- host-buffer drop-in */
/* Same argument order as the _kernels.py functions they replace.  Arrays are
 * HOST memory (pinned or pageable), mutated in place; lo/hi are absolute.
 * `lane` and `sentinel` are validated against the element kind and otherwise
 * unused (the GPU has no 512-bit packs).  `pivot` points to a host scalar of
 * the key type.  Partition functions return the absolute boundary. */
int vx_host_quicksort(int dtype, void *arr, int64_t n, int64_t lane, int64_t sort_bound, int strategy,
                      int opt_a, int opt_b, uint64_t seed);                      /* _kernels.py:378 */
int vx_host_kv_quicksort(int dtype, void *keys, void *vals, int64_t n, int64_t lane, int64_t sort_bound,
                         int strategy, int opt_a, int opt_b, uint64_t seed);     /* _kernels.py:425 */
int64_t vx_host_partition(int dtype, void *arr, int64_t lo, int64_t hi, const void *pivot, int64_t lane,
                          int opt_a, int opt_b);                                 /* _kernels.py:257 */
int64_t vx_host_kv_partition(int dtype, void *keys, void *vals, int64_t lo, int64_t hi, const void *pivot,
                             int64_t lane, int opt_a, int opt_b);                /* _kernels.py:347 */
int64_t vx_host_scalar_partition(int dtype, void *arr, int64_t lo, int64_t hi, const void *pivot);
                                                                                 /* _kernels.py:162 */
int64_t vx_host_kv_scalar_partition(int dtype, void *keys, void *vals, int64_t lo, int64_t hi,
                                    const void *pivot);                          /* _kernels.py:173 */
int vx_host_smallsort_region(int dtype, void *arr, int64_t lo, int64_t length);  /* _kernels.py:115 */
int vx_host_kv_smallsort_region(int dtype, void *keys, void *vals, int64_t lo, int64_t length);
                                                                                 /* _kernels.py:148 */
/* Pipelined twins of vx_host_quicksort / vx_host_kv_quicksort for a STREAM of
 * sorts (quicksort.py:115-134 called once per array).  A single in-place
 * host sort is bound by PCIe one direction at a time (copy in, sort, copy
 * out); vx_host_sort_submit enqueues copy-in, sort and copy-out of
 * src -> dst (dst may equal src; vals NULL for keys only) on one of two
 * device slots and returns at once, so the copy-out of one sort overlaps the
 * copy-in of the next (full-duplex PCIe).  *ticket identifies the slot;
 * vx_host_sort_wait(ticket) blocks until that sort's dst is complete and
 * returns its status.  A third submit first waits for the oldest sort.
 * Overlap needs page-locked host memory (vx_host_pin / cudaHostRegister, or
 * a pinned allocator); pageable buffers are correct but serialise. */
int vx_host_sort_submit(int dtype, const void *src_keys, const void *src_vals, void *dst_keys, void *dst_vals,
                        int64_t n, int64_t lane, int64_t sort_bound, int strategy, uint64_t seed, int *ticket);
int vx_host_sort_wait(int ticket);
int vx_host_pin(void *p, size_t bytes);
int vx_host_unpin(void *p);
/* Free the device arenas the host functions keep between calls. */
int vx_host_release(void);

#ifdef __cplusplus
}
#endif
#endif /* VEXSORT_B200_H */
