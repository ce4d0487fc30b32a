// tma.cuh -- 1-D bulk copies (TMA, cp.async.bulk) global -> shared with
// mbarrier completion, for the streaming tile kernels.
//
// A tile is an arbitrary element range [base, base+tn) of a global array.
// The bulk engine needs 16-byte aligned addresses and sizes, so the tile is
// placed in shared memory at the byte offset (address mod 16) and only its
// aligned interior is bulk-copied; the at most 15 head/tail bytes are read
// from global by whichever thread needs them (see BulkTile::get).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace vx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Metadata of one staged tile.
struct BulkTile {
    uint64_t base;  // first element (absolute index)
    unsigned tn;    // elements
    unsigned seg;   // owning segment (tile kernels)
    unsigned shift; // byte offset of element 0 inside the stage buffer
    unsigned head;  // elements before the bulk-copied interior
    unsigned body;  // elements in the bulk-copied interior
};

// Issue (one thread) the copy of elements [base, base+tn) of `src` into the
// stage buffer `buf` (16-byte aligned, >= tn*sizeof(T) + 16 bytes) and arm
// `bar` for it.  Returns the metadata consumers need.
template <typename T>
__device__ __forceinline__ BulkTile issue_tile(char* buf, const T* src, uint64_t base, unsigned tn, uint64_t* bar) {
    BulkTile bt;
    bt.base = base;
    bt.tn = tn;
    bt.seg = 0;
    const uintptr_t p0 = reinterpret_cast<uintptr_t>(src + base);
    const uintptr_t p1 = reinterpret_cast<uintptr_t>(src + base + tn);
    const uintptr_t a0 = (p0 + 15) & ~(uintptr_t)15, a1 = p1 & ~(uintptr_t)15;
    bt.shift = (unsigned)(p0 & 15);
    if (a1 > a0) {
        bt.head = (unsigned)((a0 - p0) / sizeof(T));
        bt.body = (unsigned)((a1 - a0) / sizeof(T));
        mbar_arrive_expect_tx(bar, (unsigned)(a1 - a0));
        bulk_g2s(buf + bt.shift + (a0 - p0), reinterpret_cast<const void*>(a0), (unsigned)(a1 - a0), bar);
    } else {
        bt.head = tn;  // nothing bulk-copied: every element comes from global
        bt.body = 0;
        mbar_arrive(bar);
    }
    return bt;
}

// Window variant: when the 16-byte aligned window around the tile lies
// inside the array [src, src + n_all), copy the whole window so that every
// element of the tile is in shared memory (head = 0, body = tn); `buf` needs
// tn*sizeof(T) + 32 bytes.  Otherwise fall back to issue_tile (interior only).
template <typename T>
__device__ __forceinline__ BulkTile issue_tile_window(char* buf, const T* src, uint64_t n_all, uint64_t base,
                                                      unsigned tn, uint64_t* bar) {
    const uintptr_t p0 = reinterpret_cast<uintptr_t>(src + base);
    const uintptr_t p1 = reinterpret_cast<uintptr_t>(src + base + tn);
    const uintptr_t a0 = p0 & ~(uintptr_t)15, a1 = (p1 + 15) & ~(uintptr_t)15;
    if (tn == 0 || a0 < reinterpret_cast<uintptr_t>(src) || a1 > reinterpret_cast<uintptr_t>(src + n_all))
        return issue_tile<T>(buf, src, base, tn, bar);
    BulkTile bt;
    bt.base = base;
    bt.tn = tn;
    bt.seg = 0;
    bt.shift = (unsigned)(p0 - a0);
    bt.head = 0;
    bt.body = tn;
    mbar_arrive_expect_tx(bar, (unsigned)(a1 - a0));
    bulk_g2s(buf, reinterpret_cast<const void*>(a0), (unsigned)(a1 - a0), bar);
    return bt;
}

// Element i of a staged tile (after the stage's barrier phase completed).
template <typename T>
__device__ __forceinline__ T tile_get(const char* buf, const BulkTile& bt, const T* src, unsigned i) {
    if (i >= bt.head && i < bt.head + bt.body) return reinterpret_cast<const T*>(buf + bt.shift)[i];
    return src[bt.base + i];
}

}  // namespace vx
