"""C2 poly-multiply replayed from a CUDA graph (as bench.py times it), L2
flushed between steps: prints the median ms per step."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import setup_c2  # noqa: E402
from paper_1811_01490_b200 import _lib  # noqa: E402

gp, params, plan, f, g, N, k, K = setup_c2()
out = torch.empty_like(f)
lib = _lib.load()
work = torch.empty(int(lib.gfp_fft_workspace_words(plan.handle, 1)), dtype=torch.uint64,
                   device="cuda")
sp = ctypes.c_void_p


def direct():
    _lib.check(lib.gfp_poly_mul(plan.handle, sp(f.data_ptr()), sp(g.data_ptr()),
                                sp(out.data_ptr()), sp(work.data_ptr()), 1,
                                sp(torch.cuda.current_stream().cuda_stream)))


direct()
graph = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    direct()
    with torch.cuda.graph(graph, stream=s):
        direct()
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ts = []
for i in range(60):
    flush.zero_()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    graph.replay()
    b.record()
    torch.cuda.synchronize()
    if i >= 10:
        ts.append(a.elapsed_time(b))
ts.sort()
ref = out.clone()
direct()
torch.cuda.synchronize()
assert torch.equal(ref.view(torch.int64), out.view(torch.int64))
print("c2 graph ms %.4f  (GFP_PDL=%s)" % (ts[len(ts) // 2], os.environ.get("GFP_PDL", "1")))
