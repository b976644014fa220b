"""Sharded C4 forward (four-step 2^12 x 2^12, one rank, peer-store exchange
fused into the column DFTs' last pass) under the current library
(GFPFFT_LIB): prints the median ms of 10 (L2 flushed between runs)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_01490_b200 as gp  # noqa: E402
from paper_1811_01490_b200.sharded import GpuShardOps, ShardedFFT  # noqa: E402

R8 = (1 << 59) + (1 << 16)
N1 = N2 = 1 << 12
params = gp.GfpParams(R8, 8)
ops = GpuShardOps(gp.GfpFftField(params, backend="cuda"), 16, N1, N2,
                  gp.roots_for(params, N1 * N2))
sh = ShardedFFT(ops, 8, N1, N2).use_peer_exchange()
cols = gp.vec.uniform(N1, params, seed=400, batch=N2)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
ts = []
for i in range(13):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sh.forward(cols)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
ts.sort()
print("c4s fused-exchange forward ms %.4f  (%s)" % (ts[len(ts) // 2], os.environ.get("GFPFFT_LIB", "default")))
