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

// shared -> global bulk store (bulk async-group completion).  src / dst are
// 16-byte aligned, bytes a multiple of 16.  The threads that wrote the source
// fence the async proxy (fence_async_smem) before the barrier that precedes
// the issue; the issuing thread commits, and waits for the group's smem READS
// before the source is overwritten.
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
                 "r"(smem_u32(src_smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// Metadata of one staged tile.
struct BulkTile {
    uint64_t base;  // first element (absolute index)
    unsigned tn;    // elements
    unsigned seg;   // owning segment (tile kernels)
    unsigned shift; // byte offset of element 0 inside the stage buffer
    unsigned head;  // elements before the bulk-copied interior
    unsigned body;  // elements in the bulk-copied interior
    uintptr_t src;  // bulk copy: global source (16-byte aligned)
    unsigned dst;   // bulk copy: byte offset in the stage buffer
    unsigned bytes; // bulk copy: size (0: nothing to copy)
};

// Plan (no side effects) the copy of elements [base, base+tn) of `src` into
// a stage buffer (16-byte aligned, >= tn*sizeof(T) + 32 bytes).  When the
// 16-byte aligned window around the tile lies inside [src, src + n_all) the
// whole window is copied, so every element of the tile is in shared memory
// (head = 0, body = tn); otherwise only the aligned interior is.
template <typename T>
__device__ __forceinline__ BulkTile plan_tile(const T* src, uint64_t n_all, uint64_t base, unsigned tn) {
    BulkTile bt;
    bt.base = base;
    bt.tn = tn;
    bt.seg = 0;
    const uintptr_t p0 = reinterpret_cast<uintptr_t>(src + base);
    const uintptr_t p1 = reinterpret_cast<uintptr_t>(src + base + tn);
    const uintptr_t w0 = p0 & ~(uintptr_t)15, w1 = (p1 + 15) & ~(uintptr_t)15;
    if (tn > 0 && w0 >= reinterpret_cast<uintptr_t>(src) && w1 <= reinterpret_cast<uintptr_t>(src + n_all)) {
        bt.shift = (unsigned)(p0 - w0);
        bt.head = 0;
        bt.body = tn;
        bt.src = w0;
        bt.dst = 0;
        bt.bytes = (unsigned)(w1 - w0);
        return bt;
    }
    const uintptr_t a0 = (p0 + 15) & ~(uintptr_t)15, a1 = p1 & ~(uintptr_t)15;
    bt.shift = (unsigned)(p0 & 15);
    if (a1 > a0) {
        bt.head = (unsigned)((a0 - p0) / sizeof(T));
        bt.body = (unsigned)((a1 - a0) / sizeof(T));
        bt.src = a0;
        bt.dst = bt.shift + (unsigned)(a0 - p0);
        bt.bytes = (unsigned)(a1 - a0);
    } else {
        bt.head = tn;  // nothing bulk-copied: every element comes from global
        bt.body = 0;
        bt.src = 0;
        bt.dst = 0;
        bt.bytes = 0;
    }
    return bt;
}

// Issue (one thread) a planned copy and arm `bar` for it.  Everything the
// consumers read about the tile (its BulkTile, stored to shared memory) must
// be written BEFORE this call: the arrive is a release and the consumers'
// phase wait an acquire, which orders those stores.  (A copy of zero bytes
// completes the phase at the arrive itself.)
__device__ __forceinline__ void issue_planned(char* buf, const BulkTile& bt, uint64_t* bar) {
    if (bt.bytes) {
        mbar_arrive_expect_tx(bar, bt.bytes);
        bulk_g2s(buf + bt.dst, reinterpret_cast<const void*>(bt.src), bt.bytes, bar);
    } else {
        mbar_arrive(bar);
    }
}

// Element i of a staged tile (after the stage's barrier phase completed).
template <typename T>
__device__ __forceinline__ T tile_get(const char* buf, const BulkTile& bt, const T* src, unsigned i) {
    if (i >= bt.head && i < bt.head + bt.body) return reinterpret_cast<const T*>(buf + bt.shift)[i];
    return src[bt.base + i];
}

}  // namespace vx
