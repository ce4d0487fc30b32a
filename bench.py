"""Benchmark of the B200 hybrid sort (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c5_i32_uniform|...] [--n N_GLOBAL]

Default workload (the BASELINE.json metric "Gelements/s sorted (int32/f64/kv)
at 1-8 B200"): config 5, the sharded sort of n = 2^32 int32 i.i.d. uniform
over the full range, global n fixed across 1/2/4/8 ranks ("strong"); one
step = one complete sort of the global array (at N=1 the local hybrid
quicksort, at N>1 sample sort: splitters + bucket partition + NCCL
all-to-all + local sort).  Inputs are generated on the device from a seeded
counter hash and stay resident; every step sorts the same pristine input
out of place (16 GiB >> the 126 MB L2, so no L2 flush is needed).

Other workloads (--workload): sort_i32_2^28, sort_f64_2^28, c1 (int32 2^20),
c2_i32 / c2_f64 (2^20 CSR segments of U{1..256}), c3 (f64 2^28 N(0,1)
partition around median-of-3), c4 (kv 2^28), c5_{i32,f64}_{uniform,sorted,
reverse,few}.

value  = elements / max-over-ranks device time of the K timed steps.
e2e    = the same metric through the public API with HOST buffers: pinned
         host input -> device -> sort -> host, copies inside the timed region
         (N=1 sorts: the reference-facing C-ABI host entry vx_host_quicksort).
roofline = the dominant kernel class: algorithmic bytes (one read + one
         write of every element it processed) / its summed
         CUDA-event time, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline = the CPU oracle (C port of the reference's _kernels.py,
         OpenMP task-parallel variant, identical output) on a bounded sample,
         the same port on one thread, and -- when the copy of the reference
         package in baseline/_ref travels with the repo -- the reference's own
         numba backend on one pinned core.
--impl reference: only that CPU port, rank 0, same metric and unit.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import re
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

METRIC = "Gelements/s sorted (int32/f64/kv) at 1-8 B200; % of HBM/NVLink roofline"
PEAK_FALLBACK = 6650.0
NVL_GBS = 900.0  # per direction, spec (no measured all-to-all peak yet)

# generator dist codes of vx_generate
DIST = {"uniform": 0, "sorted": 1, "reverse": 2, "few": 3, "normal": 4, "u31": 5, "index": 6}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return PEAK_FALLBACK, "fallback (B200_PROFILING.md)"


def workload_spec(name: str, n_override: int | None):
    """-> dict(kind, dtype, n, ...)."""
    if name.startswith("c5_"):
        _, t, dist = name.split("_")
        n = n_override or (1 << 32 if t == "i32" else 1 << 31)
        return dict(kind="sharded", dtype=t, dist=dist, n=n, scaling="strong")
    if name.startswith("sort_"):
        t = name.split("_")[1]
        n = n_override or (1 << 28)
        return dict(kind="sort", dtype=t, dist="uniform", n=n, scaling="weak")
    if name == "c1":
        return dict(kind="sort", dtype="i32", dist="uniform", n=n_override or (1 << 20), scaling="weak")
    if name in ("c2_i32", "c2_f64"):
        return dict(kind="segments", dtype=name[3:], nseg=n_override or (1 << 20), scaling="weak")
    if name == "c3":
        return dict(kind="partition", dtype="f64", dist="normal", n=n_override or (1 << 28), scaling="weak")
    if name == "c4":
        return dict(kind="kv", dtype="i32", dist="u31", n=n_override or (1 << 28), scaling="weak")
    raise SystemExit(f"unknown workload {name}")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            cmd = ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "50", "-i",
                   str(self.idx)]
            if shutil.which("stdbuf"):  # line-buffer the pipe so short regions still yield samples
                cmd = ["stdbuf", "-oL"] + cmd
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.2)  # let the sampler start before the timed region
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[4:8]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        loaded = [r for r in rows if r[0] > 0.5 * r[1]] or rows
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


# --------------------------------------------------------------- utilities
def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus and world > 1:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    # VX_BENCH_SHARE_GPU=1 (with VX_BENCH_BACKEND=gloo): every rank on cuda:0 with
    # host-staged collectives -- a functional check of the N > 1 code path on a
    # one-GPU box (tests/test_gpu_sharded.py), never a measurement
    if os.environ.get("VX_BENCH_SHARE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import datetime

        backend = os.environ.get("VX_BENCH_BACKEND", "nccl")
        kw = {"device_id": torch.device("cuda", local)} if backend == "nccl" else {}
        # a hung peer fails the run within minutes instead of blocking forever
        dist.init_process_group(backend, timeout=datetime.timedelta(seconds=int(os.environ.get("VX_PG_TIMEOUT", "600"))),
                                **kw)
    return rank, world, local


def barrier():
    import torch.distributed as dist

    if dist.is_initialized():
        dist.barrier()


def allmax(x: float) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gen(L, dtype_code, dist_code, t, seed, gofs, gn):
    import torch

    L.vx_generate(dtype_code, dist_code, ctypes.c_void_p(t.data_ptr()), t.numel(), seed, gofs, gn,
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))


def prof_read(L):
    n = 9
    la = (ctypes.c_int64 * n)()
    ms = (ctypes.c_double * n)()
    el = (ctypes.c_uint64 * n)()
    L.vx_profile_read(la, ms, el, n)
    return list(la), list(ms), list(el)


CLASSES = ["qs_plan", "qs_hist", "qs_emit", "qs_scatter", "qs_finish", "partition2", "segsort", "bucket_partition",
           "qs_local"]
KERNEL_REGEX = {"qs_plan": "qs_plan_kernel", "qs_hist": "qs_hist_kernel", "qs_emit": "qs_emit_kernel",
                "qs_scatter": "qs_scatter_kernel", "qs_finish": "qs_finish_kernel",
                "partition2": "partition2_kernel", "segsort": "segsort_kernel",
                "bucket_partition": "bp_scatter_kernel", "qs_local": "qs_local_kernel"}


def ncu_traffic(workload, kernel_class):
    """DRAM bytes per launch of `kernel_class` in one step of `workload`, from
    the committed ncu --set full capture (tools/summarize_ncu.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        name = KERNEL_REGEX.get(kernel_class, kernel_class)
        w = d.get(workload, {})
        e = w.get(name)
        if e is None and kernel_class == "qs_local":  # the CTA-local level's kernel variants (local*.cuh)
            e = next((v for k, v in w.items() if re.fullmatch(r"qs_local\w*_kernel", k) and v["bytes_per_launch"] > 1e6),
                     None)
        return None if e is None else round(e["bytes_per_launch"])
    except Exception:
        return None


# ----------------------------------------------------------- our workloads
def make_step(spec, vx, L, dev, rank, world, seed):
    """Inputs resident in HBM and the step closure (stream-ordered: no host
    synchronisation inside a step).  Returns a dict with the pieces the
    verification gate needs."""
    import numpy as np
    import torch

    tdt = torch.int32 if spec["dtype"] == "i32" else torch.float64
    dcode = 0 if spec["dtype"] == "i32" else 1
    esz = 4 if dcode == 0 else 8
    kind = spec["kind"]
    w = {"kind": kind, "esz": esz, "dcode": dcode}
    if kind == "sharded":
        n = spec["n"]
        lo, hi = n * rank // world, n * (rank + 1) // world
        src = torch.empty(hi - lo, dtype=tdt, device=dev)
        gen(L, dcode, DIST[spec["dist"]], src, seed, lo, n)
        if world == 1:
            out = torch.empty_like(src)
            w["step"] = lambda: vx.sort_into(src, out, check=False)  # noqa: E731
        else:
            w["step"] = lambda: vx.sharded_sort(src, seed=seed, exchange=spec.get("exchange", "collective"))  # noqa: E731
        w.update(src=src, units=n, unit_bytes=2 * esz)
    elif kind == "sort":
        n = spec["n"]
        src = torch.empty(n, dtype=tdt, device=dev)
        gen(L, dcode, DIST[spec["dist"]], src, seed, 0, n)
        out = torch.empty_like(src)
        w.update(src=src, units=n * world, unit_bytes=2 * esz, step=lambda: vx.sort_into(src, out, check=False))
    elif kind == "kv":
        n = spec["n"]
        src = torch.empty(n, dtype=tdt, device=dev)
        vals = torch.empty(n, dtype=tdt, device=dev)
        gen(L, dcode, DIST["u31"], src, seed, 0, n)
        gen(L, dcode, DIST["index"], vals, seed, 0, n)
        out, outv = torch.empty_like(src), torch.empty_like(vals)
        w.update(src=src, vals=vals, units=n * world, unit_bytes=2 * 2 * esz,
                 step=lambda: (vx.sort_into(src, out, values=vals, out_values=outv, check=False), outv)[0])
        w["outv"] = outv
    elif kind == "partition":
        n = spec["n"]
        src = torch.empty(n, dtype=tdt, device=dev)
        gen(L, dcode, DIST["normal"], src, seed, 0, n)
        pivot = float(src[vx.select_pivot(src, 0, n - 1)].item())
        out = torch.empty_like(src)
        split = {}

        def pstep():
            split["b"] = vx.partition_region(src, pivot, out=out)
            return out

        w.update(src=src, units=n * world, unit_bytes=2 * esz, step=pstep, pivot=pivot, split=split)
    elif kind == "segments":
        import inputs

        nseg = spec["nseg"]
        offs_np, vals_np = inputs.c2_input(np.int32 if dcode == 0 else np.float64, nseg=nseg)
        offs = torch.from_numpy(offs_np).to(dev)
        src = torch.from_numpy(vals_np).to(dev)
        w.update(src=src, orig=src.clone(), offs=offs, offs_np=offs_np, units=len(vals_np) * world,
                 unit_bytes=2 * esz, step=lambda: (vx.sort_segments(src, offs, validate=False), src)[1])
    return w


def verify_output(w, out, vx, world):
    """The correctness gate (benchcli.py:398-427: output == np.sort(input),
    exit 1 otherwise), as size-independent device checks: ascending order plus
    an order-independent multiset digest against the input (pairs hashed
    together); across ranks, boundary order and the global multiset.
    Raises AssertionError on a mismatch."""
    import torch
    import torch.distributed as dist
    from paper_1704_08579_b200.verify import MASK64, digest, verify_sorted_permutation

    kind = w["kind"]
    if kind in ("sort", "kv") or (kind == "sharded" and world == 1):
        verify_sorted_permutation(w["src"], out, w.get("vals"), w.get("outv"))
        return "sorted + multiset digest == input" + (" (key/value pairs)" if kind == "kv" else "")
    if kind == "partition":
        b, p = w["split"]["b"], w["pivot"]
        assert b == int((w["src"] <= p).sum().item()), "split != count(x <= pivot)"
        assert bool((out[:b] <= p).all()) and bool((out[b:] > p).all()), "sides violate the pivot"
        assert digest(w["src"], order=False).multiset() == digest(out, order=False).multiset()
        return "split == count(<= pivot), sides respect the pivot, multiset digest == input"
    if kind == "segments":
        d_in = digest(w["orig"], order=False)
        d_out = digest(out, order=True, offsets=w["offs"])
        assert d_out.inversions == 0, f"{d_out.inversions} inversions inside segments"
        assert d_in.multiset() == d_out.multiset(), "output is not a permutation of the input"
        return "every segment ascending, multiset digest == input"
    # sharded over P ranks
    d_in = digest(w["src"], order=False)
    d_out = digest(out, order=True)
    assert d_out.inversions == 0, f"rank-local output not sorted ({d_out.inversions} inversions)"
    dt = out.dtype
    edge = torch.zeros(2, dtype=dt, device=out.device)
    if len(out):
        edge[0], edge[1] = out[0], out[-1]
    info = [None] * world
    dist.all_gather_object(info, {"in": (d_in.n, d_in.hsum, d_in.hxor), "out": (d_out.n, d_out.hsum, d_out.hxor),
                                  "edge": edge.cpu().tolist() if len(out) else None})
    tin = [0, 0, 0]
    tout = [0, 0, 0]
    last = None
    for r in info:
        tin = [tin[0] + r["in"][0], (tin[1] + r["in"][1]) & MASK64, tin[2] ^ r["in"][2]]
        tout = [tout[0] + r["out"][0], (tout[1] + r["out"][1]) & MASK64, tout[2] ^ r["out"][2]]
        if r["edge"] is not None:
            assert last is None or not (r["edge"][0] < last), "rank boundaries out of order"
            last = r["edge"][1]
    assert tin == tout, "global output is not a permutation of the global input"
    return f"rank-local sorted, rank boundaries ordered, global multiset digest == input over {world} ranks"


def run_ours(args, spec, rank, world, local):
    import torch

    import paper_1704_08579_b200 as vx
    from paper_1704_08579_b200 import _lib

    L = _lib.lib()
    dev = torch.device("cuda", local)
    seed = 1
    kind = spec["kind"]
    w = make_step(spec, vx, L, dev, rank, world, seed)
    step, units, unit_bytes, src, esz = w["step"], w["units"], w["unit_bytes"], w["src"], w["esz"]
    torch.cuda.synchronize()

    # ---------------------------------------------------------- warm-up
    for _ in range(args.warmup):
        r = step()
        del r
    torch.cuda.synchronize()
    barrier()

    # ---------------------------------------------------------- timed
    # the product path: stream-ordered steps (sorts as CUDA graphs), no host
    # synchronisation inside the region
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            r = step()
            del r
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1)
    ms_max = allmax(ms)
    value = units * args.steps / (ms_max / 1e3) / 1e9

    # ------------------------------------- one more step: gate + launch count
    stats = {}
    if kind in ("sort", "kv") or (kind == "sharded" and world == 1):
        # rerun the step synchronously with its device counters
        if kind == "kv":
            out = torch.empty_like(src)
            w["outv"] = torch.empty_like(w["vals"])
            vx.sort_into(src, out, values=w["vals"], out_values=w["outv"], stats=stats)
        else:
            out = torch.empty_like(src)
            vx.sort_into(src, out, stats=stats)
    else:
        out = step()
    torch.cuda.synchronize()
    try:
        verified = verify_output(w, out, vx, world)
        ok = True
    except AssertionError as e:
        verified, ok = f"FAILED: {e}", False
    if stats:
        # init + every level's kernels (counted on the device) + the loop
        # control kernel of each WHILE iteration
        per_step = 1 + stats["launches"] + (stats["levels"] // 2)
        launches_claim = per_step * args.steps
    else:
        launches_claim = None
    del out

    # ---------------------------------------------------------- profiled pass
    # per-kernel CUDA events need the eager (host-driven) level loop: the same
    # kernels, timed one by one on their stream
    psteps = max(1, min(args.steps, args.prof_steps))
    L.vx_profile_reset()
    L.vx_profile_enable(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(psteps):
        r = step()
        del r
    e1.record(stream)
    torch.cuda.synchronize()
    L.vx_profile_enable(0)
    prof_ms = e0.elapsed_time(e1) / psteps
    launches, kms, kel = prof_read(L)
    if launches_claim is None:
        launches_claim = int(sum(launches) / psteps * args.steps)

    # dominant kernel roofline
    peak, peak_src = peaks()
    dom = max(range(len(CLASSES)), key=lambda i: kms[i])
    alg_bytes = unit_bytes * kel[dom]
    if kind == "segments" and CLASSES[dom] == "segsort":
        alg_bytes = unit_bytes * len(src) * psteps + 8 * len(w["offs"]) * psteps
    achieved = alg_bytes / (kms[dom] / 1e3) / 1e9 if kms[dom] > 0 else 0.0
    traffic = ncu_traffic(args.workload, CLASSES[dom]) if args.n is None else None
    alg_per_launch = int(alg_bytes / max(launches[dom], 1))
    dom_name = CLASSES[dom]
    if alg_bytes == 0:
        # the longest kernel moves no elements (a small sort whose one-CTA plan
        # outlasts its data passes): the roofline is the whole sort's, one read
        # + one write of the array against the time of all its kernels
        alg_bytes = unit_bytes * len(src) * psteps
        tot_ms = sum(kms)
        achieved = alg_bytes / (tot_ms / 1e3) / 1e9 if tot_ms > 0 else 0.0
        alg_per_launch = int(alg_bytes / psteps)
        dom_name = "whole sort (latency-bound: longest kernel is " + CLASSES[dom] + ", which moves no elements)"
        traffic = None
    roof = {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "traffic_over_alg": round(traffic / alg_per_launch, 3) if traffic and alg_per_launch else None,
            "peak_source": peak_src, "alg_bytes_per_launch": alg_per_launch,
            "avg_launch_ms": round((kms[dom] / max(launches[dom], 1)) if alg_per_launch and dom_name == CLASSES[dom]
                                   else sum(kms) / psteps, 4),
            "timing": "CUDA events around every launch of the profiled pass (eager level loop, same kernels)"}
    # whole-step roofline: one read+write pass at HBM peak (+ NVLink term)
    step_bytes = unit_bytes * units / world
    t_roof = step_bytes / (peak * 1e9)
    if kind == "sharded" and world > 1:
        t_roof += (units / world * esz * (world - 1) / world) / (NVL_GBS * 1e9)
    kernels = {CLASSES[i]: {"launches": launches[i], "ms_per_step": round(kms[i] / psteps, 3),
                            "elems_per_step": kel[i] // psteps}
               for i in range(len(CLASSES)) if launches[i]}
    res = dict(value=value, ms=ms_max / args.steps, roofline=roof, kernels=kernels,
               step_roofline={"t_roof_ms": round(t_roof * 1e3, 4),
                              "frac": round(t_roof * 1e3 / (ms_max / args.steps), 4),
                              "passes_equiv": round((ms_max / args.steps) / (t_roof * 1e3), 2)},
               profiled_ms_per_step=round(prof_ms, 3), gpu_launches=launches_claim, clocks=clk.summary(),
               units=units, verified=ok, verification=verified)
    if stats:
        res["sort_stats"] = {k: stats[k] for k in ("levels", "launches", "scatter_elems", "local_elems",
                                                   "finish_elems")}
        res["sort_stats"]["scatter_levels_per_key"] = round(stats["scatter_elems"] / max(len(src), 1), 3)

    # ---------------------------------------------------------- e2e
    if not args.no_e2e:
        extra = {}
        if kind == "segments":
            extra["offs_host"] = torch.from_numpy(w["offs_np"]).pin_memory()
            src.copy_(w["orig"])
        res["e2e"] = run_e2e(args, spec, vx, L, src, w.get("vals"), dev, rank, world, units, extra)
    # ---------------------------------------------------------- cpu baseline
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_baseline(spec, args, src=src if kind != "segments" else None)
    return res


def run_e2e(args, spec, vx, L, src, vals, dev, rank, world, units, extra):
    """Host buffers in, host buffers out, copies inside the timed region."""
    import torch

    kind = spec["kind"]
    host = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
    hv = torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True) if (kind == "kv") else None
    code = 0 if src.dtype == torch.int32 else 1
    times = []
    h2d = src.numel() * src.element_size() * (2 if hv is not None else 1)
    if "offs_host" in extra:
        h2d += extra["offs_host"].numel() * 8
    d2h = h2d
    torch.cuda.empty_cache()
    for it in range(args.warmup + args.steps):
        host.copy_(src)  # restore pristine input (untimed)
        if hv is not None:
            hv.copy_(vals)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        if kind == "sort" and world == 1:
            # reference-facing C ABI, host buffers (twin of _kernels.quicksort)
            rc = L.vx_host_quicksort(code, ctypes.c_void_p(host.data_ptr()), host.numel(), 16 if code == 0 else 8,
                                     0, 0, 0, 0, 0)
            assert rc == 0, L.vx_last_error()
        elif kind == "kv" and world == 1:
            rc = L.vx_host_kv_quicksort(code, ctypes.c_void_p(host.data_ptr()), ctypes.c_void_p(hv.data_ptr()),
                                        host.numel(), 16 if code == 0 else 8, 0, 0, 0, 0, 0)
            assert rc == 0, L.vx_last_error()
        elif kind == "partition":
            pc = ctypes.c_double(float(src[vx.select_pivot(src, 0, src.numel() - 1)].item()))
            b = L.vx_host_partition(1, ctypes.c_void_p(host.data_ptr()), 0, host.numel(), ctypes.byref(pc), 8, 0, 0)
            assert b >= 0
        elif kind == "sharded" and world == 1:
            rc = L.vx_host_quicksort(code, ctypes.c_void_p(host.data_ptr()), host.numel(), 16 if code == 0 else 8,
                                     0, 0, 0, 0, 0)
            assert rc == 0, L.vx_last_error()
        else:
            # public Python API: pinned host -> device -> sort -> pinned host
            d = host.to(dev, non_blocking=True)
            if kind == "sharded":
                out = vx.sharded_sort(d)
                if "res_h" not in extra or extra["res_h"].numel() < out.numel():
                    torch.cuda.synchronize()  # (re)allocate outside the steady state
                    extra["res_h"] = torch.empty(2 * out.numel(), dtype=out.dtype, pin_memory=True)
                extra["res_h"][: out.numel()].copy_(out, non_blocking=True)
                d2h = out.numel() * out.element_size()
            else:  # segments, in place: offsets travel with the values
                offs = extra["offs_host"].to(dev, non_blocking=True)
                vx.sort_segments(d, offs, validate=False)
                host.copy_(d, non_blocking=True)
            torch.cuda.synchronize()
        t1 = time.perf_counter()
        if it >= args.warmup:
            times.append(t1 - t0)
    total = allmax(sum(times))
    L.vx_host_release()
    res = {"value": units * args.steps / total / 1e9, "unit": "Gelem/s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "ms_per_step": round(total / args.steps * 1e3, 3),
           "path": "vx_host_* C ABI (host buffers)" if world == 1 and kind != "segments" else
           "public API, pinned host tensors"}
    if world == 1 and kind in ("sort", "kv", "sharded") and not args.no_pipeline:
        pipe = run_e2e_pipelined(args, vx, L, src, vals if kind == "kv" else None, host, hv, code, units)
        if "value" in pipe:
            # the headline e2e is the throughput of a stream of sorts through the
            # pipelined boundary; the one-call-at-a-time figure stays beside it
            res = {**pipe, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                   "single_call": {"value": res["value"], "ms_per_step": res["ms_per_step"], "path": res["path"]}}
        else:
            res["pipelined"] = pipe
    return res


def run_e2e_pipelined(args, vx, L, src, vals, host, hv, code, units):
    """Throughput of a STREAM of host sorts: every step copies the pristine
    pinned input in, sorts, and copies the result out to pinned memory, but
    two steps are in flight (vx_host_sort_submit / vx_host_sort_wait), so one
    step's copy-out overlaps the next step's copy-in over full-duplex PCIe."""
    import torch

    try:
        outs = [torch.empty(src.shape, dtype=src.dtype, pin_memory=True) for _ in range(2)]
        outv = [torch.empty(vals.shape, dtype=vals.dtype, pin_memory=True) for _ in range(2)] if vals is not None \
            else [None, None]
    except RuntimeError as e:  # not enough page-locked host memory on this box
        return {"skipped": f"pinned output buffers: {e}"[:200]}
    host.copy_(src)  # pristine input, read by every step, never written
    if hv is not None:
        hv.copy_(vals)
    torch.cuda.synchronize()
    lane = 16 if code == 0 else 8
    n = host.numel()
    vp = ctypes.c_void_p

    def run(steps):
        tickets = []
        for i in range(steps):
            if len(tickets) == 2:
                rc = L.vx_host_sort_wait(tickets.pop(0))
                assert rc == 0, L.vx_last_error()
            t = ctypes.c_int(-1)
            rc = L.vx_host_sort_submit(code, vp(host.data_ptr()), vp(hv.data_ptr()) if hv is not None else None,
                                       vp(outs[i % 2].data_ptr()),
                                       vp(outv[i % 2].data_ptr()) if hv is not None else None,
                                       n, lane, 0, 0, 0, ctypes.byref(t))
            assert rc == 0, L.vx_last_error()
            tickets.append(t.value)
        for t in tickets:
            rc = L.vx_host_sort_wait(t)
            assert rc == 0, L.vx_last_error()

    run(max(2, args.warmup))  # both slots: arenas allocated, sort graphs built
    barrier()
    t0 = time.perf_counter()
    run(args.steps)
    total = allmax(time.perf_counter() - t0)
    L.vx_host_release()
    # gate: the last step's host output against the device sort of the same input
    last = (args.steps - 1) % 2
    want = torch.empty_like(src)
    if vals is not None:
        wantv = torch.empty_like(vals)
        vx.sort_into(src, want, values=vals, out_values=wantv)
        got = outs[last].to(src.device)
        ok = bool(torch.equal(got, want))
        gv = outv[last].to(src.device)
        ok = ok and bool(torch.equal(src[gv.long()], got))  # values still name their keys
        del wantv, gv
    else:
        vx.sort_into(src, want)
        got = outs[last].to(src.device)
        ok = bool(torch.equal(got, want))
    del got, want
    torch.cuda.empty_cache()
    if not ok:
        raise SystemExit("pipelined e2e output differs from the device sort")
    return {"value": units * args.steps / total / 1e9, "unit": "Gelem/s",
            "ms_per_step": round(total / args.steps * 1e3, 3), "verified": True,
            "path": "vx_host_sort_submit / vx_host_sort_wait C ABI (pinned host buffers, 2 sorts in flight: "
                    "copy-out of step i overlaps copy-in of step i+1)"}


# ------------------------------------------------------------ CPU baseline
def cpu_sample(spec, src=None, n_sample=None):
    """A bounded sample of the same workload on the host (numpy)."""
    import numpy as np

    import inputs

    kind = spec["kind"]
    if kind in ("sort", "sharded"):
        n = n_sample or (1 << 24)
        note = ""
        if spec.get("dist", "uniform") != "uniform":
            # the reference's median-of-3 quicksort is quadratic on sorted /
            # reverse / few-unique inputs (SURVEY.md section 0 finding 5):
            # only a small sample is feasible
            n = min(n, 1 << 16)
            note = " (reference is quadratic on this distribution; full n infeasible)"
        if src is not None:
            return src[:n].cpu().numpy().copy(), f"first 2^{n.bit_length()-1} elements of the device input{note}"
        dt = np.int32 if spec["dtype"] == "i32" else np.float64
        return inputs.c5_input(dt, spec["dist"], n=n), f"2^{n.bit_length()-1}-element C5 input{note}"
    if kind == "kv":
        n = n_sample or (1 << 22)
        k, v = inputs.c4_input(n=n)
        return (k, v), f"2^{n.bit_length()-1} C4 pairs"
    if kind == "partition":
        n = n_sample or (1 << 26)
        return inputs.c3_input(n=n), f"2^{n.bit_length()-1} C3 normals"
    if kind == "segments":
        nseg = n_sample or (1 << 16)
        dt = np.int32 if spec["dtype"] == "i32" else np.float64
        return inputs.c2_input(dt, nseg=nseg), f"2^{nseg.bit_length()-1} C2 segments"


def cpu_run_once(spec, sample, nthreads):
    """Run the oracle port once on a fresh copy; return (elements, seconds)."""
    import oracle

    kind = spec["kind"]
    if kind in ("sort", "sharded"):
        a = sample.copy()
        t0 = time.perf_counter()
        oracle.sort(a, nthreads=nthreads)
        return len(a), time.perf_counter() - t0
    if kind == "kv":
        k, v = sample[0].copy(), sample[1].copy()
        t0 = time.perf_counter()
        oracle.kv_sort(k, v, nthreads=nthreads)
        return len(k), time.perf_counter() - t0
    if kind == "partition":
        a = sample.copy()
        p = a[oracle.median3_index(a, 0, len(a) - 1)]
        t0 = time.perf_counter()
        oracle.partition_region(a, p)
        return len(a), time.perf_counter() - t0
    if kind == "segments":
        offs, vals = sample
        a = vals.copy()
        sent = oracle.sentinel_for(a)
        t0 = time.perf_counter()
        for s in range(len(offs) - 1):
            oracle.smallsort_region(a, int(offs[s]), int(offs[s + 1] - offs[s]), sent)
        return len(a), time.perf_counter() - t0


def cpu_threads(spec):
    import oracle

    # partition / small sorts are single-threaded in the reference and the port
    return oracle.max_threads() if spec["kind"] in ("sort", "sharded", "kv") else 1


def cpu_baseline(spec, args, src=None):
    sample, desc = cpu_sample(spec, src)
    nt = cpu_threads(spec)
    cpu_run_once(spec, sample, nt)  # warm (page faults, thread pool)
    n, sec = cpu_run_once(spec, sample, nt)
    out = {"value": n / sec / 1e9, "unit": "Gelem/s", "cores": nt, "kind": "port",
           "sample": f"{desc}; C port of _kernels.py (oracle/), "
                     f"{'OpenMP task-parallel quicksort' if nt > 1 else 'single thread'}, {sec:.2f} s"}
    if nt > 1:
        # BASELINE.md section 3 quotes the reference on ONE core: the same port, one thread
        n1, sec1 = cpu_run_once(spec, sample, 1)
        out["single_core"] = {"value": n1 / sec1 / 1e9, "unit": "Gelem/s", "cores": 1, "seconds": round(sec1, 2)}
    ref = numba_reference(spec, sample)
    if ref is not None:
        out["reference_numba"] = ref
    return out


def numba_reference(spec, sample):
    """BASELINE.md section 3's setting, when a copy of the reference package
    travels with the repo (baseline/_ref, made by tests/golden/make_golden.py):
    the reference's own numba backend through its public API, ONE pinned
    core, JIT call excluded, on a (smaller) prefix of the same sample.
    Returns None when the copy or numba is missing."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "vexsort")):
        return None
    try:
        if ref not in sys.path:
            sys.path.insert(0, ref)
        import numpy as np
        import vexsort

        if not vexsort.native_available():
            return None
    except Exception:  # noqa: BLE001  (numba missing / import error: no reference figure)
        return None
    kind = spec["kind"]
    old_aff = os.sched_getaffinity(0)
    core = min(old_aff)
    try:
        os.sched_setaffinity(0, {core})
        if kind in ("sort", "sharded"):
            a = sample[: 1 << 22].copy()
            vexsort.sort(a[: 1 << 12].copy())  # JIT
            t0 = time.perf_counter()
            vexsort.sort(a)
            sec, n, what = time.perf_counter() - t0, len(a), "vexsort.sort"
            ok = bool(np.all(a[1:] >= a[:-1]))
        elif kind == "kv":
            k, v = sample[0][: 1 << 21].copy(), sample[1][: 1 << 21].copy()
            vexsort.kv_sort(k[: 1 << 12].copy(), v[: 1 << 12].copy())
            t0 = time.perf_counter()
            vexsort.kv_sort(k, v)
            sec, n, what = time.perf_counter() - t0, len(k), "vexsort.kv_sort"
            ok = bool(np.all(k[1:] >= k[:-1]))
        elif kind == "partition":
            a = sample[: 1 << 24].copy()
            from vexsort.quicksort import select_pivot as ref_select_pivot

            piv = float(a[ref_select_pivot(a, 0, len(a) - 1)])
            vexsort.partition_region(a[: 1 << 12].copy(), piv)
            t0 = time.perf_counter()
            b = vexsort.partition_region(a, piv)
            sec, n, what = time.perf_counter() - t0, len(a), "vexsort.partition_region"
            ok = bool(np.all(a[:b] <= piv) and np.all(a[b:] > piv))
        else:  # segments: one small sort per segment, as BASELINE.md section 2 timed it
            from vexsort import _kernels

            offs, vals = sample
            nseg = min(len(offs) - 1, 1 << 13)
            a = vals[: int(offs[nseg])].copy()
            sent = np.iinfo(np.int32).max if a.dtype == np.int32 else np.inf
            _kernels.smallsort_region(a[:64].copy(), 0, 64, sent)
            t0 = time.perf_counter()
            for i in range(nseg):
                _kernels.smallsort_region(a, int(offs[i]), int(offs[i + 1] - offs[i]), sent)
            sec, n, what = time.perf_counter() - t0, len(a), f"_kernels.smallsort_region x {nseg} segments"
            ok = True
    except Exception as e:  # noqa: BLE001
        return {"unavailable": repr(e)[:160]}
    finally:
        os.sched_setaffinity(0, old_aff)
    return {"value": n / sec / 1e9, "unit": "Gelem/s", "cores": 1, "kind": "reference",
            "sample": f"{what} (numba backend, baseline/_ref copy of the reference), first {n} elements of the "
                      f"sample, pinned to core {core}, {sec:.2f} s, output ordered: {ok}"}


def run_reference(args, spec, rank):
    """--impl reference: the reference's CPU algorithm (oracle port) on the
    host cores, rank 0 only; each step one bounded sample."""
    if rank != 0:
        return None
    sample, desc = cpu_sample(spec)
    nt = cpu_threads(spec)
    for _ in range(args.warmup):
        cpu_run_once(spec, sample, nt)
    tot_n, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, s = cpu_run_once(spec, sample, nt)
        tot_n += n
        tot_s += s
    v = tot_n / tot_s / 1e9
    cb = {"value": v, "unit": "Gelem/s", "cores": nt, "kind": "port",
          "sample": f"{desc} per step; C port of _kernels.py (oracle/)"}
    ref = numba_reference(spec, sample)
    if ref is not None:
        cb["reference_numba"] = ref
    return {"value": v, "ms": tot_s / args.steps * 1e3,
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5_i32_uniform")
    ap.add_argument("--n", "--size", dest="n", type=lambda s: int(eval(s, {}, {})), default=None, help="global n (e.g. 2**28)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true", help="e2e: one synchronous host call per step only")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--prof-steps", type=int, default=2, help="steps of the per-kernel profiled pass")
    ap.add_argument("--exchange", default="collective", choices=["collective", "fused"],
                    help="sharded sort (N>1): NCCL all-to-all, or the fused partition+NVLink-store exchange")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    spec = workload_spec(args.workload, args.n)
    if spec["kind"] == "sharded":
        spec["exchange"] = args.exchange
    dtype = {"i32": "int32", "f64": "float64"}[spec["dtype"]]
    cfg = {"workload": args.workload, **{k: v for k, v in spec.items() if k not in ("kind", "scaling")}}
    base = {"metric": METRIC, "unit": "Gelem/s", "higher_is_better": True, "scaling": spec["scaling"],
            "vs_baseline": None, "dtype": dtype, "steps": args.steps, "warmup": args.warmup}

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        r = run_reference(args, spec, rank)
        if r is None:
            return
        cfg["sample"] = r["cpu_baseline"]["sample"]
        line = {**base, "impl": "reference", "value": r["value"], "n_gpus": args.gpus,
                "ms_per_step": r["ms"], "data": "synthetic (seeded numpy generators, tests/golden/inputs.py)",
                "config": cfg, "cpu_baseline": r["cpu_baseline"], "e2e": r["e2e"]}
        print(json.dumps(line))
        return

    rank, world, local = dist_setup(args.gpus)
    r = run_ours(args, spec, rank, world, local)
    xname = "NCCL all-to-all" if spec.get("exchange") != "fused" else "fused partition + IPC/NVLink stores"
    if os.environ.get("VX_BENCH_BACKEND", "nccl") != "nccl":
        xname += f"; {os.environ['VX_BENCH_BACKEND']} collectives, host-staged: a functional check, not a measurement"
    cfg["parallelism"] = ((f"sample sort over {world} ranks ({xname})" if world > 1 else
                           "single GPU (P=1 sample sort = the local hybrid sort; no exchange)")
                          if spec["kind"] == "sharded"
                          else ("replicas" if world > 1 else "single GPU"))
    cfg["l2"] = "inputs larger than the 126 MB L2 (no flush needed)" if r["units"] * 4 > (256 << 20) \
        else "input fits in L2; steps re-run on resident data"
    if rank == 0:
        line = {**base, "value": r["value"], "n_gpus": world, "ms_per_step": r["ms"],
                "data": "synthetic (device counter-hash generator, seed 1)", "config": cfg,
                "verified": r["verified"], "verification": r["verification"],
                "roofline": r["roofline"], "step_roofline": r["step_roofline"], "kernels": r["kernels"],
                "profiled_ms_per_step": r["profiled_ms_per_step"],
                "gpu_launches": r["gpu_launches"], "clocks": r["clocks"]}
        if "sort_stats" in r:
            line["sort_stats"] = r["sort_stats"]
        if "e2e" in r:
            line["e2e"] = r["e2e"]
        if "cpu_baseline" in r:
            line["cpu_baseline"] = r["cpu_baseline"]
        print(json.dumps(line))
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()
    if not r["verified"]:
        print(f"verification failed: {r['verification']}", file=sys.stderr)
        sys.exit(1)


if __name__ == "__main__":
    main()
