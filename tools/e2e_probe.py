"""Time the C2 e2e call (gfp_poly_mul_host2, pinned operands) under the current
environment; prints ms per call (median of 20)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_01490_b200 as gp  # noqa: E402
from paper_1811_01490_b200 import _lib  # noqa: E402

R8 = (1 << 59) + (1 << 16)
params = gp.GfpParams(R8, 8)
plan = gp.build_plan(gp.GfpFftField(params, backend="cuda"), 16, 4, gp.roots_for(params, 1 << 16))
nf = 1 << 15
f = torch.from_numpy(gp.vec.to_host(gp.vec.uniform(nf, params, seed=1))).pin_memory()
g = torch.from_numpy(gp.vec.to_host(gp.vec.uniform(nf, params, seed=2))).pin_memory()
o = torch.empty((2 * nf - 1, 8), dtype=torch.uint64).pin_memory()
lib = _lib.load()
sp = ctypes.c_void_p
st = sp(torch.cuda.current_stream().cuda_stream)


def call():
    _lib.check(lib.gfp_poly_mul_host2(plan.handle, sp(f.data_ptr()), nf, sp(g.data_ptr()), nf,
                                      sp(o.data_ptr()), 1, st))


for _ in range(5):
    call()
ts = []
for _ in range(20):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    call()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
h2d = torch.empty((nf, 8), dtype=torch.uint64, device="cuda")
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    h2d.copy_(f, non_blocking=True)
b.record()
torch.cuda.synchronize()
ms_copy = a.elapsed_time(b) / 10
print("e2e_ms %.4f  (GFP_ZERO_COPY=%s)  memcpy H2D 2 MiB: %.4f ms = %.1f GB/s" % (
    ts[len(ts) // 2], os.environ.get("GFP_ZERO_COPY", "1"), ms_copy, 2 * 2**20 / ms_copy / 1e6))
