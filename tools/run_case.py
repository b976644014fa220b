"""Run one BASELINE workload a few times (for ncu / compute-sanitizer).

    python tools/run_case.py c4 [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1811_01490_b200 as gp  # noqa: E402
from bench import R, WORKLOADS  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    if key == "c4s":  # sharded C4 (1 rank): fused exchange, then the standalone kernel
        from paper_1811_01490_b200.sharded import GpuShardOps, ShardedFFT
        N1 = N2 = 1 << 12
        params = gp.GfpParams(R[8], 8)
        field = gp.GfpFftField(params, backend="cuda")
        ops = GpuShardOps(field, 16, N1, N2, gp.roots_for(params, N1 * N2))
        sh = ShardedFFT(ops, 8, N1, N2).use_peer_exchange()
        cols = gp.vec.uniform(N1, params, seed=400, batch=N2)
        for _ in range(reps):
            sh.forward(cols)
        y = sh.forward_columns(cols)
        for _ in range(reps):
            sh.peer.transpose("rows", y, A=N2, B=N1)
        torch.cuda.synchronize()
        print("ok", key, reps)
        return
    wl = WORKLOADS[key]
    k, K, e, B = wl["k"], wl["K"], wl["e"], wl["batch"]
    if key == "c3" and len(sys.argv) > 3:
        B = int(sys.argv[3])
    N = K ** e
    params = gp.GfpParams(R[k], k)
    field = gp.GfpFftField(params, backend="cuda")
    plan = gp.build_plan(field, K, e, gp.roots_for(params, N))
    if key == "c5":
        n = 1 << 22
        a = gp.vec.uniform(n, params, seed=51)
        b = gp.vec.uniform(n, params, seed=52)
        for _ in range(reps):
            gp.vec.mul(a, b, params)
    x = gp.vec.uniform(N, params, seed=7, batch=B if B > 1 else None)
    y = torch.empty_like(x)
    for _ in range(reps):
        if wl["kind"] == "polymul":
            gp.poly_mul(x, x, plan, out=y)
        else:
            gp.fft_tensor(x, plan, out=y)
    torch.cuda.synchronize()
    print("ok", key, reps)


if __name__ == "__main__":
    main()
