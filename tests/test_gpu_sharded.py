"""The sharded sort's device path with more than one rank, on ONE GPU.

* The fused exchange's scatter (vx_bucket_scatter_to) with several
  destination buffers in one process: every destination receives exactly
  its bucket, at the offset the counts matrix assigns.
* Two processes sharing cuda:0 over a gloo process group run the REAL
  B200Ops end to end: the collective exchange (host-staged all_to_all, since
  gloo) and the fused exchange (each rank's bucket partition stores straight
  into the other process's receive buffer through a CUDA IPC mapping).  No
  kernel waits on another process: ordering is host barriers only, so
  sharing one GPU is sound (B200_PROFILING.md).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs

pytestmark = pytest.mark.gpu


def test_bucket_scatter_to_several_destinations():
    from paper_1704_08579_b200.sharded import B200Ops, fused_offsets

    ops = B200Ops()
    rng = np.random.default_rng(3)
    P = 4
    for n, dt in ((1 << 20, np.int32), (300001, np.float64), (1 << 16, np.int32)):
        x = inputs.c5_input(dt, "uniform", n=1 << 20)[:n]
        t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        gi = torch.arange(n, dtype=torch.int64, device="cuda")
        pos = torch.from_numpy(np.sort(rng.choice(n, 512, replace=False))).cuda()
        sk, si = ops.select_splitters(t[pos].contiguous(), gi[pos].contiguous(), P)
        counts = ops.bucket_counts(t, 0, sk, si)
        ref, ref_counts = ops.bucket_partition(t, 0, sk, si)
        assert counts.tolist() == ref_counts.tolist() and int(counts.sum()) == n
        # pretend to be rank 1 of 3 senders: lower ranks fill the front
        cm = [[5, 7, 11, 13], counts.tolist(), [2, 3, 4, 5]]
        offs = fused_offsets(cm, 1)
        bufs = [torch.full((offs[d] + cm[1][d] + cm[2][d],), -7, dtype=t.dtype, device="cuda") for d in range(P)]
        ops.bucket_scatter_to(t, 0, sk, si, [b.data_ptr() for b in bufs], offs)
        starts = np.concatenate([[0], np.cumsum(counts.cpu().numpy())])
        refn = ref.cpu().numpy()
        for d in range(P):
            b = bufs[d].cpu().numpy()
            got = b[offs[d]:offs[d] + cm[1][d]]
            assert np.array_equal(np.sort(got), np.sort(refn[starts[d]:starts[d + 1]]))
            assert np.all(b[:offs[d]] == -7) and np.all(b[offs[d] + cm[1][d]:] == -7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dtype, dist_name, n, exchange, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1704_08579_b200.sharded import ExchangeStats, sharded_sort

        local = torch.from_numpy(inputs.c5_input(dtype, dist_name, n=n, rank=rank, world=world, nchunks=64)).cuda()
        outs = []
        for rep in range(2):  # the second call reuses the receive buffers / peer mappings
            st = ExchangeStats()
            out = sharded_sort(local, samples_per_rank=512, seed=rep, stats=st, exchange=exchange)
            outs.append(out.cpu().numpy())
        q.put((rank, outs, st.send_counts, st.recv_counts, None))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["collective", "fused"])
@pytest.mark.parametrize("dtype,dist_name", [(np.int32, "uniform"), (np.int32, "few"), (np.int32, "reverse"),
                                             (np.float64, "uniform")])
def test_two_processes_one_gpu_real_kernels(exchange, dtype, dist_name):
    world, n = 2, 1 << 22
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, dist_name, n, exchange, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    errs = [r[4] for r in res if r[4]]
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
    glob = np.sort(inputs.c5_input(dtype, dist_name, n=n))
    for rep in range(2):
        assert np.array_equal(np.concatenate([r[1][rep] for r in res]), glob)
    send = np.array([r[2] for r in res])
    recv = np.array([r[3] for r in res])
    assert np.array_equal(send, recv.T) and send.sum() == n
