"""Multi-rank host logic of the sharded sample sort, on CPU with gloo
(world size 2 and 3).  The device kernels are replaced by numpy test doubles
with the same contracts (CpuModelOps, test-only), so this exercises exactly
the product's exchange plumbing in paper_1704_08579_b200/sharded.py:
global offsets, (key, global index) sampling, splitter selection, per
destination counts, the uneven all-to-all and the final local sort.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs


class CpuModelOps:
    """numpy models of the three device kernels (tests only)."""

    def select_splitters(self, keys, gidx, nparts):
        k, i = keys.numpy(), gidx.numpy()
        order = np.lexsort((i, k))
        q = [(r * len(k)) // nparts for r in range(1, nparts)]
        return torch.from_numpy(k[order][q].copy()), torch.from_numpy(i[order][q].copy())

    def bucket_partition(self, local, gofs, sk, si):
        x = local.numpy()
        g = np.arange(len(x), dtype=np.int64) + gofs
        dest = np.zeros(len(x), dtype=np.int64)
        for kk, ii in zip(sk.numpy(), si.numpy()):
            dest += (kk < x) | ((kk == x) & (ii < g))
        order = np.argsort(dest, kind="stable")
        counts = np.bincount(dest, minlength=len(sk) + 1).astype(np.int64)
        return torch.from_numpy(x[order].copy()), torch.from_numpy(counts)

    def local_sort(self, x, seed):
        x.copy_(torch.from_numpy(np.sort(x.numpy())))
        return x

    def local_sort_into(self, x, seed):
        return torch.from_numpy(np.sort(x.numpy()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dtype, dist_name, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1704_08579_b200.sharded import ExchangeStats, sharded_sort

        local = torch.from_numpy(inputs.c5_input(dtype, dist_name, n=n, rank=rank, world=world, nchunks=64))
        st = ExchangeStats()
        out = sharded_sort(local, samples_per_rank=256, ops=CpuModelOps(), stats=st)
        q.put((rank, out.numpy(), st.send_counts, st.recv_counts))
    finally:
        dist.destroy_process_group()


def _run(world, dtype, dist_name, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, dist_name, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("dist_name", ["uniform", "sorted", "reverse", "few"])
def test_sharded_sort_gloo(world, dist_name):
    n = 1 << 14
    dtype = np.int32
    res = _run(world, dtype, dist_name, n)
    glob = inputs.c5_input(dtype, dist_name, n=n)
    outs = [r[1] for r in res]
    assert np.array_equal(np.concatenate(outs), np.sort(glob))
    # counts: what rank r sent to s is what s received from r
    send = np.array([r[2] for r in res])
    recv = np.array([r[3] for r in res])
    assert np.array_equal(send, recv.T)
    assert send.sum() == n
    # (key, index) splitters keep even few-unique inputs balanced
    sizes = np.array([len(o) for o in outs])
    assert sizes.max() <= 1.5 * n / world, sizes
    if dist_name == "sorted":
        # already globally sorted: nothing crosses ranks except at the edges
        assert np.trace(send) >= 0.9 * n


def test_sharded_sort_f64_gloo():
    n = 1 << 13
    res = _run(2, np.float64, "uniform", n)
    glob = inputs.c5_input(np.float64, "uniform", n=n)
    assert np.array_equal(np.concatenate([r[1] for r in res]), np.sort(glob))


def test_sample_positions_are_in_range_and_stratified():
    from paper_1704_08579_b200.sharded import sample_positions

    for n, s in ((1000, 64), (10, 64), (1 << 20, 1024), (1, 5)):
        p = sample_positions(n, s, rank=3, seed=7).numpy()
        assert len(p) == min(n, s)
        assert p.min() >= 0 and p.max() < n
        assert np.all(np.diff(p) > 0)  # one per stratum, increasing


def test_fused_offsets_pack_sources_in_rank_order():
    from paper_1704_08579_b200.sharded import fused_offsets

    cm = [[3, 1, 4], [1, 5, 9], [2, 6, 5]]  # cm[q][d]: q sends to d
    assert fused_offsets(cm, 0) == [0, 0, 0]
    assert fused_offsets(cm, 1) == [3, 1, 4]
    assert fused_offsets(cm, 2) == [4, 6, 13]
    # the last source's run ends exactly at the receive size
    for d in range(3):
        assert fused_offsets(cm, 2)[d] + cm[2][d] == sum(cm[q][d] for q in range(3))
