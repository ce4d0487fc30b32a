"""Phase clocks of the CTA-local level (library built with -DVX_QL_PHASES).

    VEXSORT_B200_LIB=build/phases.so python tools/ql_phases.py [i32|f64|kv] [log2n]
"""
import ctypes
import sys

import torch

import paper_1704_08579_b200 as vx
from paper_1704_08579_b200._lib import lib
from paper_1704_08579_b200.verify import generate

kind = sys.argv[1] if len(sys.argv) > 1 else "i32"
n = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 28)
L = lib()
src = generate(torch.float64 if kind == "f64" else torch.int32, "uniform", n)
out = torch.empty_like(src)
vals = torch.arange(n, dtype=torch.int32, device="cuda") if kind == "kv" else None
ovals = torch.empty_like(vals) if vals is not None else None
names = ["range", "count", "scan", "scatter", "networks", "copyout"]
buf = (ctypes.c_ulonglong * 8)()
for it in range(3):
    vx.sort_into(src, out, values=vals, out_values=ovals)
    torch.cuda.synchronize()
    L.vx_debug_phases(buf)
    tot = sum(buf[:6]) or 1
    print(kind, n, " ".join(f"{nm}={buf[i] / tot:.3f}" for i, nm in enumerate(names)),
          f"cycles/key/SM={tot / n:.3f}")
