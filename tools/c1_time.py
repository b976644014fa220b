"""C1 forward+inverse timing (device, graph-free) for A/B runs: python tools/c1_time.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_01490_b200 as gp
from bench import R
p8 = gp.GfpParams(R[8], 8); f8 = gp.GfpFftField(p8, backend="cuda")
res = {}
for e in (3, 4):
    plan = gp.build_plan(f8, 16, e, gp.roots_for(p8, 16 ** e))
    x = gp.vec.uniform(16 ** e, p8, seed=1); y = torch.empty_like(x)
    def step():
        gp.fft_tensor(x, plan, out=y); gp.fft_tensor(y, plan, inverse=True, out=y)
    for _ in range(5): step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(50):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); step(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); res["fwd_inv_16^%d_ms" % e] = ts[len(ts) // 2]
print(os.environ.get("GFP_PASS44_GPC", "auto"), json.dumps(res))
