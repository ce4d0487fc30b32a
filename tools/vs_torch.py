"""Sort time vs n against the device's library sort (torch.sort), same inputs.
    python tools/vs_torch.py [--dtype i32|f64] [--exps 16 18 20 ...]
CUDA events around `reps` back-to-back sorts after warm-up; the input is
re-copied from a pristine buffer before every sort (copy time measured and
subtracted)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1704_08579_b200 as vx  # noqa: E402


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="i32")
    ap.add_argument("--exps", type=int, nargs="*", default=[16, 18, 20, 21, 22, 23, 24, 26, 28])
    a = ap.parse_args()
    rows = []
    for e in a.exps:
        n = 1 << e
        g = torch.Generator(device="cuda").manual_seed(e)
        if a.dtype == "i32":
            src = torch.randint(-(2**31), 2**31 - 1, (n,), dtype=torch.int32, device="cuda", generator=g)
        else:
            src = (torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5) * 2e6
        out = torch.empty_like(src)
        reps = max(5, min(200, (1 << 27) // n))
        for _ in range(20):  # past the eager sorts: the cached CUDA graph
            vx.sort_into(src, out, check=False)
        ours = timed(lambda: vx.sort_into(src, out, check=False), reps)
        ref = torch.sort(src).values
        assert torch.equal(out, ref)
        for _ in range(3):
            torch.sort(src)
        lib = timed(lambda: torch.sort(src), reps)
        libk = timed(lambda: torch.sort(src, stable=False), reps)
        rows.append({"n": f"2^{e}", "ours_ms": round(ours, 4), "torch_sort_ms": round(min(lib, libk), 4),
                     "speedup": round(min(lib, libk) / ours, 2)})
        print(json.dumps(rows[-1]), flush=True)
        del src, out, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
