"""CTA timeline of the k = 8 TMA pass (a library built with -DP44T_TRACE=1):
GFPFFT_LIB=vlibs/trace.so python tools/trace_c2.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_01490_b200 as gp
from bench import R
p8 = gp.GfpParams(R[8], 8); f8 = gp.GfpFftField(p8, backend="cuda")
plan = gp.build_plan(f8, 16, 4, gp.roots_for(p8, 1 << 16))
f = gp.vec.uniform(1 << 16, p8, seed=1); g = gp.vec.uniform(1 << 16, p8, seed=2)
out = torch.empty_like(f)
for i in range(3):
    gp.poly_mul(f, g, plan, out=out)
    torch.cuda.synchronize()
    print("---- step", i, flush=True)
graph = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    gp.poly_mul(f, g, plan, out=out)
    with torch.cuda.graph(graph, stream=s):
        gp.poly_mul(f, g, plan, out=out)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
print("---- graph", flush=True)
for i in range(2):
    graph.replay(); torch.cuda.synchronize(); print("---- replay", i, flush=True)
