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

from ._lib import check, lib
from ._region import check_region, dev_ptr, stream_of, workspace
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
        sk = torch.empty(max(m, 1), dtype=keys.dtype, device=keys.device)
        si = torch.empty(max(m, 1), dtype=torch.int64, device=keys.device)
        check(lib().vx_select_splitters(kind.code, dev_ptr(keys), dev_ptr(gidx), len(keys), nparts, dev_ptr(sk),
                                        dev_ptr(si), stream_of(keys)), "select_splitters")
        return sk[:m], si[:m]

    def bucket_partition(self, local, gofs, sk, si):
        import torch

        kind = check_region(local)
        m = len(sk)
        out = torch.empty_like(local)
        counts = torch.empty(m + 1, dtype=torch.int64, device=local.device)
        L = lib()
        ws = workspace(L.vx_bucket_partition_workspace_bytes(kind.code, m), local.device)
        check(L.vx_bucket_partition(kind.code, dev_ptr(local), dev_ptr(out), len(local), int(gofs),
                                    dev_ptr(sk) if m else None, dev_ptr(si) if m else None, m, dev_ptr(counts),
                                    dev_ptr(ws), ws.numel(), stream_of(local)), "bucket_partition")
        return out, counts

    def local_sort(self, x, seed):
        sort_with_config(x, SortConfig(pivot_seed=seed))
        return x

    def local_sort_into(self, x, seed):
        import torch

        return sort_into(x, torch.empty_like(x), SortConfig(pivot_seed=seed))


def sharded_sort(local, group=None, *, samples_per_rank: int = 1024, seed: int = 0, ops=None,
                 stats: ExchangeStats | None = None):
    """Globally sort the distributed array whose shard on this rank is
    `local` (1-D, contiguous; global order = rank order).  Returns this
    rank's slice of the sorted result (a new tensor; size varies by rank)."""
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
    # global offset of this shard
    sizes = torch.zeros(P, dtype=torch.int64, device=dev)
    mine = torch.tensor([n_local], dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(sizes, mine, group=group)
    gofs = int(sizes[:r].sum().item())
    # samples with global indices; fixed count per rank (pad with the last
    # element of the shard, or a sentinel-free empty marker when empty)
    s = max(1, min(samples_per_rank, 8192 // P))
    pos = sample_positions(n_local, s, r, seed).to(dev)
    cnt = torch.tensor([len(pos)], dtype=torch.int64, device=dev)
    skeys = torch.zeros(s, dtype=local.dtype, device=dev)
    sidx = torch.full((s,), -1, dtype=torch.int64, device=dev)
    if len(pos):
        skeys[: len(pos)] = local[pos]
        sidx[: len(pos)] = pos + gofs
    all_keys = torch.empty(P * s, dtype=local.dtype, device=dev)
    all_idx = torch.empty(P * s, dtype=torch.int64, device=dev)
    all_cnt = torch.empty(P, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_keys, skeys, group=group)
    dist.all_gather_into_tensor(all_idx, sidx, group=group)
    dist.all_gather_into_tensor(all_cnt, cnt, group=group)
    valid = torch.cat([torch.arange(r_ * s, r_ * s + int(c), device=dev) for r_, c in enumerate(all_cnt.tolist())])
    sk, si = ops.select_splitters(all_keys[valid].contiguous(), all_idx[valid].contiguous(), P)
    parted, counts = ops.bucket_partition(local, gofs, sk, si)
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts, group=group)
    send = counts.tolist()
    recv = recv_counts.tolist()
    out = torch.empty(int(sum(recv)), dtype=local.dtype, device=dev)
    dist.all_to_all_single(out, parted, output_split_sizes=recv, input_split_sizes=send, group=group)
    out = ops.local_sort(out, seed)
    if stats is not None:
        stats.n_local_out = len(out)
        stats.send_counts = send
        stats.recv_counts = recv
    return out
