"""Sharded sample sort over 1-8 B200s (north-star subsystem 4, config 5).

No reference counterpart (the reference is single-core); this
is the data-parallel extension of its hybrid quicksort: the top partition
level runs across GPUs.  One process per GPU, torch.distributed over NCCL:

  1. every rank draws `s` samples of its shard with their GLOBAL indices;
  2. ``all_gather`` the (key, index) samples; pick P-1 splitters on the
     device (vx_select_splitters: smem bitonic over the gathered pairs);
  3. k-way bucket partition of the shard into P destination runs
     (vx_bucket_partition: the quicksort level's hist + scatter kernels with
     a (key, global index) classifier, so equal keys are split by position
     and few-unique inputs stay balanced);
  4. ``all_to_all_single`` of the per-destination counts, then of the
     payload with uneven splits (NCCL over NVLink 5 / NVSwitch);
  5. local hybrid quicksort of what arrived (vx_sort).

Rank r ends up with a contiguous slice of the global sorted order;
concatenating the ranks' outputs equals the sorted global input.  The
collective plumbing is written against an ``ops`` object so the host logic
can be exercised on CPU (gloo) with test doubles; the product ops are the
B200 kernels and there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes

from ._lib import SortConfigC, check, lib
from ._region import check_region, dev_ptr, on_device, stream_of, workspace
from .quicksort import SortConfig, sort_into, sort_with_config

__all__ = ["sharded_sort", "sample_positions", "B200Ops", "ExchangeStats"]


def sample_positions(n_local: int, s: int, rank: int, seed: int = 0):
    """Deterministic stratified sample positions of a shard: one position in
    each of s equal strata, jittered by a hash of (seed, rank, stratum)."""
    import torch

    if n_local == 0 or s == 0:
        return torch.zeros(0, dtype=torch.int64)
    s = min(s, n_local)
    j = torch.arange(s, dtype=torch.int64)
    lo = j * n_local // s
    hi = (j + 1) * n_local // s
    h = (j * 0x9E3779B1 + (seed * 1000003 + rank) * 0x85EBCA77) & 0x7FFFFFFF
    return lo + h % (hi - lo).clamp(min=1)


@dataclass
class ExchangeStats:
    n_local_in: int = 0
    n_local_out: int = 0
    send_counts: list | None = None
    recv_counts: list | None = None


class B200Ops:
    """Device kernels used by the exchange (the product path)."""

    def select_splitters(self, keys, gidx, nparts):
        import torch

        kind = check_region(keys)
        m = nparts - 1
        with on_device(keys):
            sk = torch.empty(max(m, 1), dtype=keys.dtype, device=keys.device)
            si = torch.empty(max(m, 1), dtype=torch.int64, device=keys.device)
            check(lib().vx_select_splitters(kind.code, dev_ptr(keys), dev_ptr(gidx), len(keys), nparts, dev_ptr(sk),
                                            dev_ptr(si), stream_of(keys)), "select_splitters")
        return sk[:m], si[:m]

    def bucket_partition(self, local, gofs, sk, si):
        import torch

        kind = check_region(local)
        m = len(sk)
        with on_device(local):
            out = torch.empty_like(local)
            counts = torch.empty(m + 1, dtype=torch.int64, device=local.device)
            L = lib()
            ws = workspace(L.vx_bucket_partition_workspace_bytes(kind.code, m), local.device)
            check(L.vx_bucket_partition(kind.code, dev_ptr(local), dev_ptr(out), len(local), int(gofs),
                                        dev_ptr(sk) if m else None, dev_ptr(si) if m else None, m, dev_ptr(counts),
                                        dev_ptr(ws), ws.numel(), stream_of(local)), "bucket_partition")
        return out, counts

    def bucket_counts(self, local, gofs, sk, si):
        import torch

        kind = check_region(local)
        m = len(sk)
        with on_device(local):
            counts = torch.empty(m + 1, dtype=torch.int64, device=local.device)
            check(lib().vx_bucket_counts(kind.code, dev_ptr(local), len(local), int(gofs), dev_ptr(sk) if m else None,
                                         dev_ptr(si) if m else None, m, dev_ptr(counts), stream_of(local)),
                  "bucket_counts")
        return counts

    def bucket_scatter_to(self, local, gofs, sk, si, dst_ptrs, dst_offsets):
        """Destination d's run of `local` goes to dst_ptrs[d] + dst_offsets[d]
        elements (device addresses; peers' receive buffers)."""
        import torch

        kind = check_region(local)
        m = len(sk)
        with on_device(local):
            L = lib()
            ptrs = torch.tensor(dst_ptrs, dtype=torch.int64).to(local.device)
            offs = torch.tensor(dst_offsets, dtype=torch.int64).to(local.device)
            ws = workspace(L.vx_bucket_partition_workspace_bytes(kind.code, m), local.device)
            check(L.vx_bucket_scatter_to(kind.code, dev_ptr(local), len(local), int(gofs), dev_ptr(sk) if m else None,
                                         dev_ptr(si) if m else None, m, dev_ptr(ptrs), dev_ptr(offs), dev_ptr(ws),
                                         ws.numel(), stream_of(local)), "bucket_scatter_to")
            torch.cuda.current_stream(local.device).synchronize()  # ptrs/offs/ws stay alive until done

    def recv_buffer(self, dev, nbytes):
        return _ipc_recv_buffer(dev, nbytes)

    def open_peer(self, rank, handle):
        return _ipc_open_peer(rank, handle)

    def local_sort_from(self, ptr, n, dtype, dev, seed):
        import torch

        out = torch.empty(n, dtype=dtype, device=dev)
        if n == 0:
            return out
        kind = check_region(out)
        L = lib()
        with on_device(out):
            ws = workspace(L.vx_sort_workspace_bytes(kind.code, 0, n), dev)
            cfg = SortConfigC(kind.lanes * 16, 0, 0, 0, 0, seed & ((1 << 64) - 1))
            check(L.vx_sort_from_ptr(kind.code, ptr, dev_ptr(out), n, ctypes.byref(cfg), dev_ptr(ws), ws.numel(),
                                     stream_of(out)), "sort")
            check(L.vx_sort_status(dev_ptr(ws), n, stream_of(out), None), "sort")
        return out

    def local_sort(self, x, seed):
        sort_with_config(x, SortConfig(pivot_seed=seed))
        return x

    def local_sort_into(self, x, seed):
        import torch

        return sort_into(x, torch.empty_like(x), SortConfig(pivot_seed=seed))


# ------------------------------------------------ fused exchange (IPC buffers)
# One receive buffer per device, exported with a CUDA IPC handle and grown on
# demand; peers' buffers are mapped once per (rank, handle).
_RECV = {}
_PEERS = {}


def _ipc_recv_buffer(dev, nbytes):
    """(device address, 64-byte handle) of this process's receive buffer on
    `dev`, at least nbytes long."""
    L = lib()
    key = dev.index
    b = _RECV.get(key)
    if b is None or b[1] < nbytes:
        with on_device_index(key):
            if b is not None:
                check(L.vx_ipc_free(ctypes.c_void_p(b[0])), "ipc_free")
            cap = max(int(nbytes * 1.25), 1 << 20)
            p = ctypes.c_void_p()
            check(L.vx_ipc_alloc(cap, ctypes.byref(p)), "ipc_alloc")
            h = ctypes.create_string_buffer(64)
            check(L.vx_ipc_handle(p, h), "ipc_handle")
            b = (p.value, cap, h.raw)
            _RECV[key] = b
    return b[0], b[2]


def _ipc_open_peer(rank, handle):
    """Device address of a peer's receive buffer (mapped once per handle;
    a peer that grew its buffer sends a new handle, the old mapping closes)."""
    L = lib()
    old = _PEERS.get(rank)
    if old is not None and old[0] == handle:
        return old[1]
    if old is not None:
        check(L.vx_ipc_close(ctypes.c_void_p(old[1])), "ipc_close")
    p = ctypes.c_void_p()
    check(L.vx_ipc_open(ctypes.create_string_buffer(handle, 64), ctypes.byref(p)), "ipc_open")
    _PEERS[rank] = (handle, p.value)
    return p.value


def on_device_index(idx):
    import torch

    return torch.cuda.device(idx)


def fused_offsets(cmat, r):
    """Where rank r's run for destination d starts inside d's receive buffer:
    after the runs of every lower rank (so each receive buffer holds its
    sources in rank order).  cmat[q][d] = elements rank q sends to d."""
    return [sum(cmat[q][d] for q in range(r)) for d in range(len(cmat[0]))]


class _Comm:
    """The collectives of the exchange on `group`.  NCCL moves CUDA tensors
    directly (NVLink / NVSwitch); other backends (gloo: CPU tests, one-GPU
    multi-process tests) get host-staged copies."""

    def __init__(self, group, dev):
        import torch.distributed as dist

        self.group = group
        self.dev = dev
        self.staged = dev.type == "cuda" and dist.get_backend(group) != "nccl"

    def _h(self, t):
        return t.cpu() if self.staged else t

    def _d(self, t):
        return t.to(self.dev) if self.staged else t

    def all_gather(self, t):
        import torch
        import torch.distributed as dist

        P = dist.get_world_size(self.group)
        src = self._h(t)
        out = torch.empty(P * len(src), dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.group)
        return self._d(out)

    def all_to_all(self, out_len, x, send, recv):
        import torch
        import torch.distributed as dist

        src = self._h(x)
        out = torch.empty(out_len, dtype=src.dtype, device=src.device)
        dist.all_to_all_single(out, src, output_split_sizes=recv, input_split_sizes=send, group=self.group)
        return self._d(out)


def sharded_sort(local, group=None, *, samples_per_rank: int = 1024, seed: int = 0, ops=None,
                 stats: ExchangeStats | None = None, exchange: str = "collective"):
    """Globally sort the distributed array whose shard on this rank is
    `local` (1-D, contiguous; global order = rank order).  Returns this
    rank's slice of the sorted result (a new tensor; size varies by rank).
    Raises RuntimeError if the exchange loses or duplicates elements.

    exchange="collective": bucket partition into a local buffer, then
    all_to_all_single (NCCL).  exchange="fused": the bucket
    partition stores every run straight into its destination's receive
    buffer (CUDA IPC mappings of the peers' buffers, NVLink stores on a
    multi-GPU box) -- the partition pass IS the transfer; then a barrier and
    the local sort.  Needs every rank's GPU in this node."""
    assert exchange in ("collective", "fused"), exchange
    import torch
    import torch.distributed as dist

    ops = ops or B200Ops()
    P = dist.get_world_size(group) if dist.is_initialized() else 1
    r = dist.get_rank(group) if dist.is_initialized() else 0
    n_local = len(local)
    if stats is not None:
        stats.n_local_in = n_local
    if P == 1:
        out = ops.local_sort_into(local, seed)
        if stats is not None:
            stats.n_local_out = n_local
            stats.send_counts = stats.recv_counts = [n_local]
        return out
    dev = local.device
    comm = _Comm(group, dev)
    # global offset of this shard
    sizes = comm.all_gather(torch.tensor([n_local], dtype=torch.int64, device=dev)).tolist()
    gofs = int(sum(sizes[:r]))
    n_total = int(sum(sizes))
    if n_total == 0:
        if stats is not None:
            stats.n_local_out = 0
            stats.send_counts = stats.recv_counts = [0] * P
        return local.clone()
    # samples with global indices; fixed count per rank (padded; the valid
    # count travels with them)
    s = max(1, min(samples_per_rank, 8192 // P))
    pos = sample_positions(n_local, s, r, seed).to(dev)
    cnt = torch.tensor([len(pos)], dtype=torch.int64, device=dev)
    skeys = torch.zeros(s, dtype=local.dtype, device=dev)
    sidx = torch.full((s,), -1, dtype=torch.int64, device=dev)
    if len(pos):
        skeys[: len(pos)] = local[pos]
        sidx[: len(pos)] = pos + gofs
    all_keys = comm.all_gather(skeys)
    all_idx = comm.all_gather(sidx)
    all_cnt = comm.all_gather(cnt)
    valid = torch.cat([torch.arange(r_ * s, r_ * s + int(c), device=dev) for r_, c in enumerate(all_cnt.tolist())])
    sk, si = ops.select_splitters(all_keys[valid].contiguous(), all_idx[valid].contiguous(), P)
    if exchange == "fused":
        return _fused_exchange(local, gofs, sk, si, ops, comm, P, r, n_total, seed, stats)
    parted, counts = ops.bucket_partition(local, gofs, sk, si)
    send = counts.tolist()
    # counts matrix: row q = what rank q sends to each rank
    cmat = comm.all_gather(counts).view(P, P).tolist()
    recv = [cmat[q][r] for q in range(P)]
    if sum(send) != n_local:
        raise RuntimeError(f"bucket partition lost elements on rank {r}: {sum(send)} != {n_local}")
    out = comm.all_to_all(int(sum(recv)), parted, send, recv)
    # post-exchange check: the global count is conserved and every rank got
    # what the counts matrix says
    got = comm.all_gather(torch.tensor([len(out)], dtype=torch.int64, device=dev)).tolist()
    want = [sum(cmat[q][d] for q in range(P)) for d in range(P)]
    if got != want or sum(got) != n_total:
        raise RuntimeError(f"exchange count mismatch: received {got}, expected {want} (total {n_total})")
    out = ops.local_sort(out, seed)
    if stats is not None:
        stats.n_local_out = len(out)
        stats.send_counts = send
        stats.recv_counts = recv
    return out


def _fused_exchange(local, gofs, sk, si, ops, comm, P, r, n_total, seed, stats):
    import torch.distributed as dist

    dev = local.device
    counts = ops.bucket_counts(local, gofs, sk, si)
    send = counts.tolist()
    if sum(send) != len(local):
        raise RuntimeError(f"bucket counts lost elements on rank {r}: {sum(send)} != {len(local)}")
    cmat = comm.all_gather(counts).view(P, P).tolist()
    recv = [cmat[q][r] for q in range(P)]
    n_recv = int(sum(recv))
    esz = local.element_size()
    ptr, handle = ops.recv_buffer(dev, max(n_recv, 1) * esz)
    handles = [None] * P
    dist.all_gather_object(handles, handle, group=comm.group)
    ptrs = [ptr if d == r else ops.open_peer(d, handles[d]) for d in range(P)]
    # every rank's buffer is (re)allocated and mapped before anyone stores
    dist.barrier(group=comm.group)
    ops.bucket_scatter_to(local, gofs, sk, si, ptrs, fused_offsets(cmat, r))
    # every peer's stores into this rank's buffer have completed
    dist.barrier(group=comm.group)
    want = [sum(cmat[q][d] for q in range(P)) for d in range(P)]
    if sum(want) != n_total or want[r] != n_recv:
        raise RuntimeError(f"exchange count mismatch: expected {want}, total {n_total}")
    out = ops.local_sort_from(ptr, n_recv, local.dtype, dev, seed)
    if stats is not None:
        stats.n_local_out = len(out)
        stats.send_counts = send
        stats.recv_counts = recv
    return out
