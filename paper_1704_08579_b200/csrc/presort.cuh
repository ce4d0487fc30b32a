// presort.cuh -- already-ordered inputs leave the sort before its first level.
//
// The reference's median-of-3 quicksort is quadratic on sorted and reverse
// sorted input (finding 5); the partition levels here are
// not, but they still move every key three times to arrive where it started.
// Large sorts therefore first ask whether the input is monotone:
//   * qs_presort_check_kernel: every CTA tests 512 evenly spaced adjacent
//     pairs (a few microseconds; random data fails here with certainty
//     1 - 2^-512 and the kernel returns); if all of them rise (or all fall)
//     the CTAs test EVERY adjacent pair of their chunk of the array -- one
//     read pass, which an out-of-place sort also uses to write the copy (or
//     the reversed copy: pairs travel together and equal keys may take any
//     order, keyvalue.py:230) -- and raise a flag on the first
//     counter-example;
//   * qs_presort_apply_kernel: if no CTA objected, the level-0 segment is
//     withdrawn so every later kernel of the sort finds an empty queue (and
//     a falling array sorted in place is reversed).
// The output is the same sorted array either way.
#pragma once

#include "common.cuh"
#include "qsort.cuh"

namespace vx {

constexpr int kPreNT = 512;
constexpr unsigned kPreSample = 512;  // one pair per thread: a single round of loads

// 1: the sampled adjacent pairs never fall; 2: they never rise; 0: neither.
template <typename K>
__device__ __forceinline__ unsigned presort_sample_dir(const K* __restrict__ k, uint64_t n) {
    bool asc = true, desc = true;
    for (unsigned i = threadIdx.x; i < kPreSample; i += kPreNT) {
        const uint64_t p = (uint64_t)i * (n - 1) / kPreSample;  // n > kPreSample: p + 1 < n
        const K a = k[p], b = k[p + 1];
        asc &= !(b < a);
        desc &= !(a < b);
    }
    const int a = __syncthreads_and(asc), d = __syncthreads_and(desc);
    return a ? 1u : (d ? 2u : 0u);
}

// One adjacent pair against the direction.
template <typename K>
__device__ __forceinline__ bool presort_pair_ok(unsigned dir, K a, K b) {
    return dir == 1 ? !(b < a) : !(a < b);
}

// flags[0] <- direction (0 none), flags[1] |= 1 when some adjacent pair
// contradicts it (flags[1] is zero on entry: qs_init_kernel).  An
// out-of-place sort (out != in) writes the answer while it checks -- the
// copy for a rising input, the reversed copy for a falling one: nothing else
// touches the output before level 1, so a check that fails half way leaves
// only garbage the partition levels overwrite, and a check that passes has
// cost one read and one write of the array instead of a read, a read and a
// write.  Keys without a payload whose array is 16-byte aligned go through
// vector loads (four keys and their successor per thread and step).
template <typename K, typename V>
__global__ void __launch_bounds__(kPreNT) qs_presort_check_kernel(const K* __restrict__ in_k,
                                                                  const V* __restrict__ in_v, K* out_k, V* out_v,
                                                                  uint64_t n, unsigned* __restrict__ flags) {
    constexpr bool KV = HasVal<V>::value;
    constexpr unsigned VE = 16 / sizeof(K);
    const unsigned dir = presort_sample_dir(in_k, n);
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[0] = dir;
    if (!dir) return;
    const bool copy = in_k != out_k;
    volatile unsigned* bad = flags + 1;
    bool ok = true;
    unsigned round = 0;
    // stop as soon as anybody has found a counter-example (polled every 32 steps)
    auto give_up = [&]() -> bool {
        if ((++round & 31u) != 0u) return false;
        return !__syncthreads_and(ok && *bad == 0u);
    };
    bool vec = !KV && (reinterpret_cast<uintptr_t>(in_k) & 15) == 0;
    if (copy && dir == 1) vec = vec && (reinterpret_cast<uintptr_t>(out_k) & 15) == 0;
    if (vec) {
        union Vec {
            uint4 v;
            K k[VE];
        };
        const uint64_t nv = n / VE;  // whole vectors; block 0 takes the n % VE keys after them
        const uint64_t v0 = nv / gridDim.x * blockIdx.x + min((uint64_t)blockIdx.x, nv % gridDim.x);
        const uint64_t v1 = v0 + nv / gridDim.x + (blockIdx.x < nv % gridDim.x ? 1u : 0u);
        const uint4* in4 = reinterpret_cast<const uint4*>(in_k);
        uint4* out4 = reinterpret_cast<uint4*>(out_k);
        for (uint64_t base = v0; base < v1; base += 4ull * kPreNT) {
            Vec w[4];
            K nxt[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t q = base + (uint64_t)u * kPreNT + threadIdx.x;
                if (q < v1) {
                    w[u].v = __ldcs(in4 + q);
                    nxt[u] = (q + 1) * VE < n ? in_k[(q + 1) * VE] : w[u].k[VE - 1];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t q = base + (uint64_t)u * kPreNT + threadIdx.x;
                if (q < v1) {
#pragma unroll
                    for (unsigned r = 0; r + 1 < VE; ++r) ok &= presort_pair_ok(dir, w[u].k[r], w[u].k[r + 1]);
                    ok &= presort_pair_ok(dir, w[u].k[VE - 1], nxt[u]);
                    if (copy) {
                        if (dir == 1) {
                            out4[q] = w[u].v;
                        } else {
#pragma unroll
                            for (unsigned r = 0; r < VE; ++r) out_k[n - 1 - (q * VE + r)] = w[u].k[r];
                        }
                    }
                }
            }
            if (give_up()) {
                ok = false;
                break;
            }
        }
        if (blockIdx.x == 0) {
            for (uint64_t i = nv * VE + threadIdx.x; i < n; i += kPreNT) {
                const K a = in_k[i];
                if (i + 1 < n) ok &= presort_pair_ok(dir, a, in_k[i + 1]);
                if (copy) out_k[dir == 1 ? i : n - 1 - i] = a;
            }
        }
    } else {
        // element by element: key i (and its payload) with its successor
        const uint64_t p0 = n / gridDim.x * blockIdx.x + min((uint64_t)blockIdx.x, n % gridDim.x);
        const uint64_t p1 = p0 + n / gridDim.x + (blockIdx.x < n % gridDim.x ? 1u : 0u);
        for (uint64_t base = p0; base < p1; base += 4ull * kPreNT) {
            K a[4], b[4];
            V va[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = base + (uint64_t)u * kPreNT + threadIdx.x;
                if (i < p1) {
                    a[u] = ld_stream(in_k + i);
                    b[u] = i + 1 < n ? in_k[i + 1] : a[u];
                    if constexpr (KV) {
                        if (copy) va[u] = ld_stream(in_v + i);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = base + (uint64_t)u * kPreNT + threadIdx.x;
                if (i < p1) {
                    ok &= presort_pair_ok(dir, a[u], b[u]);
                    if (copy) {
                        const uint64_t o = dir == 1 ? i : n - 1 - i;
                        out_k[o] = a[u];
                        if constexpr (KV) out_v[o] = va[u];
                    }
                }
            }
            if (give_up()) {
                ok = false;
                break;
            }
        }
    }
    if (!__syncthreads_and(ok) && threadIdx.x == 0) atomicExch(flags + 1, 1u);
}

// If nobody objected the array is in order: withdraw the level-0 segment, so
// every later kernel of the sort finds an empty queue.  The output already
// holds the answer (written by the check, or the input itself when a rising
// array is sorted in place); a falling array sorted in place is reversed here
// (position i of the lower half swaps with n - 1 - i).
template <typename K, typename V>
__global__ void __launch_bounds__(kPreNT) qs_presort_apply_kernel(K* keys, V* vals, int inplace, uint64_t n,
                                                                  const unsigned* __restrict__ flags,
                                                                  Ctl* __restrict__ ctl) {
    constexpr bool KV = HasVal<V>::value;
    const unsigned dir = flags[0];
    if (!dir || flags[1]) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->nseg = 0;
        ctl->fin_elems += n;
    }
    if (dir == 1 || !inplace) return;
    const uint64_t m = n / 2;
    const uint64_t c0 = m / gridDim.x * blockIdx.x + min((uint64_t)blockIdx.x, m % gridDim.x);
    const uint64_t c1 = c0 + m / gridDim.x + (blockIdx.x < m % gridDim.x ? 1u : 0u);
    for (uint64_t base = c0; base < c1; base += 4ull * kPreNT) {
        K a[4], b[4];
        V va[4], vb[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t i = base + (uint64_t)u * kPreNT + threadIdx.x;
            if (i < c1) {
                a[u] = keys[i];
                b[u] = keys[n - 1 - i];
                if constexpr (KV) {
                    va[u] = vals[i];
                    vb[u] = vals[n - 1 - i];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t i = base + (uint64_t)u * kPreNT + threadIdx.x;
            if (i < c1) {
                keys[i] = b[u];
                keys[n - 1 - i] = a[u];
                if constexpr (KV) {
                    vals[i] = vb[u];
                    vals[n - 1 - i] = va[u];
                }
            }
        }
    }
}

}  // namespace vx
