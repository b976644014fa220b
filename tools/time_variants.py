"""A/B timing of library builds: python tools/time_variants.py lib1.so lib2.so[:VAR=val,...] ...
Each library is timed in a fresh subprocess (GFPFFT_LIB) on C2 poly-mul
(graph replay, L2 flushed), C4 forward and C3 forward (8 transforms)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, torch
sys.path.insert(0, %r)
import paper_1811_01490_b200 as gp
from bench import R
res = {}
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
def timeit(fn, reps, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); means[0] = sum(ts[len(ts) // 10: -len(ts) // 10 or None]) / max(1, len(ts[len(ts) // 10: -len(ts) // 10 or None]))
    return ts[len(ts) // 2]
means = [0.0]
p8 = gp.GfpParams(R[8], 8); f8 = gp.GfpFftField(p8, backend="cuda")
plan2 = gp.build_plan(f8, 16, 4, gp.roots_for(p8, 1 << 16))
f = gp.vec.uniform(1 << 16, p8, seed=1); g = gp.vec.uniform(1 << 16, p8, seed=2)
out = torch.empty_like(f)
res["c2_polymul_ms"] = timeit(lambda: gp.poly_mul(f, g, plan2, out=out), 100)
import hashlib
dig = lambda t: hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:12]
res["c2_digest"] = dig(out)
# C2 as bench.py times it: the 8 pass launches replayed from a CUDA graph
graph = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    gp.poly_mul(f, g, plan2, out=out)
    with torch.cuda.graph(graph, stream=s):
        gp.poly_mul(f, g, plan2, out=out)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
res["c2_graph_ms"] = timeit(graph.replay, 300)
res["c2_graph_trimmed_mean_ms"] = round(means[0], 5)
def g20():
    for _ in range(20): graph.replay()
res["c2_graph_x20_warm_ms"] = round(timeit(g20, 30) / 20, 5)  # finer than one event pair resolves; L2-warm
plan1 = gp.build_plan(f8, 16, 3, gp.roots_for(p8, 4096))
x1 = gp.vec.uniform(4096, p8, seed=9); y1 = torch.empty_like(x1)
def c1():
    gp.fft_tensor(x1, plan1, out=y1); gp.fft_tensor(y1, plan1, inverse=True, out=y1)
res["c1_ms"] = timeit(c1, 100)
res["c1_trimmed_mean_ms"] = round(means[0], 5)
plan4 = gp.build_plan(f8, 16, 6, gp.roots_for(p8, 1 << 24))
x = gp.vec.uniform(1 << 24, p8, seed=4); y = torch.empty_like(x)
res["c4_fwd_ms"] = timeit(lambda: gp.fft_tensor(x, plan4, out=y), 10)
res["c4_digest"] = dig(y)
from paper_1811_01490_b200 import fft as F
res["c4_pass_ms"] = [round(ms, 4) for _, ms in F.pass_times(plan4, lambda: gp.fft_tensor(x, plan4, out=y))[1]]
del x, y
p16 = gp.GfpParams(R[16], 16); f16 = gp.GfpFftField(p16, backend="cuda")
plan3 = gp.build_plan(f16, 32, 4, gp.roots_for(p16, 1 << 20))
x = gp.vec.uniform(1 << 20, p16, seed=3, batch=8); y = torch.empty_like(x)
res["c3x8_fwd_ms"] = timeit(lambda: gp.fft_tensor(x, plan3, out=y), 10)
res["c3_digest"] = dig(y)
res["c3_pass_ms"] = [round(ms, 4) for _, ms in F.pass_times(plan3, lambda: gp.fft_tensor(x, plan3, out=y))[1]]
del x, y
p32 = gp.GfpParams(R[32], 32); f32 = gp.GfpFftField(p32, backend="cuda")
a = gp.vec.uniform(1 << 22, p32, seed=51); b = gp.vec.uniform(1 << 22, p32, seed=52)
res["c5_mul_ms"] = timeit(lambda: gp.vec.mul(a, b, p32), 5)
del a, b
plan5 = gp.build_plan(f32, 64, 3, gp.roots_for(p32, 1 << 18))
x = gp.vec.uniform(1 << 18, p32, seed=5); y = torch.empty_like(x)
res["c5_fwd_ms"] = timeit(lambda: gp.fft_tensor(x, plan5, out=y), 10)
res["c5_digest"] = dig(y)
print(json.dumps(res))
''' % ROOT

for spec in sys.argv[1:]:
    lib, _, envs = spec.partition(":")
    env = dict(os.environ, GFPFFT_LIB=os.path.abspath(lib))
    for kv in filter(None, envs.split(",")):
        kk, _, vv = kv.partition("=")
        env[kk] = vv
    outp = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = outp.stdout.strip().splitlines()[-1] if outp.stdout.strip() else outp.stderr[-500:]
    print(spec.replace(os.path.dirname(os.path.abspath(lib)) + '/', ''), line, flush=True)
