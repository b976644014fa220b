"""Word-prime NTT / convolution timing (8 x 2^20 over P1): python tools/word_time.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_01490_b200 as gp
q, n, B = gp.P1, 1 << 20, 8
plan = gp.conv_plan(gp.word_prime(q), n, False)
g = torch.Generator(device="cuda").manual_seed(11)
x = (torch.randint(0, 1 << 62, (B, n), device="cuda", generator=g) % q).view(torch.uint64)
y = (torch.randint(0, 1 << 62, (B, n), device="cuda", generator=g) % q).view(torch.uint64)
z = torch.empty_like(x)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); b.synchronize(); return a.elapsed_time(b) / reps
ntt = t(lambda: gp.word_ntt(x, plan, out=z))
conv = t(lambda: gp.word_convolve(x, y, plan, out=z))
print(json.dumps({"ntt_ms": ntt, "ntt_gbs": 5 * 16 * n * B / (ntt * 1e-3) / 1e9, "conv_ms": conv}))
