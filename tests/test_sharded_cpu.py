"""The sharded four-step transform (paper_1811_01490_b200/sharded.py) run as
two gloo ranks on CPU with oracle-backed local steps: the orchestration
(layouts, permutes, the all-to-all exchange, twiddle exponents) must
reproduce the oracle's single-process DFT and invert exactly.  The GPU
kernels behind GpuShardOps are covered by tests/test_gpu_parity.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401  (sys.path)
from oracle import oracle as O

K, k = 16, 8
R8 = O.DEFAULT_RADIX[8]


class OracleShardOps:
    """Local steps on CPU with the oracle (test-only stand-in for GpuShardOps)."""

    def __init__(self, N1, N2, omega):
        N = N1 * N2
        self.N, self.M = N, N // K
        self.big = O.Plan(k, R8, K, _e(N), omega)
        self.tab = self.big.table()
        # sub-roots: w1 = omega^N2, w2 = omega^N1, via the oracle table/pow
        w1 = _pow(omega, N2, N)
        w2 = _pow(omega, N1, N)
        self.plans = {"N1": O.Plan(k, R8, K, _e(N1), w1), "N2": O.Plan(k, R8, K, _e(N2), w2)}

    def fft(self, x, which, inverse):
        a = _np(x)
        out = np.empty_like(a)
        for b in range(a.shape[0]):
            v = np.ascontiguousarray(a[b].T)
            p = self.plans[which]
            out[b] = (p.inverse(v) if inverse else p.forward(v)).T
        return torch.from_numpy(out.view(np.int64))

    def twiddle(self, x, row0, inverse):
        a = _np(x)
        B, kk, n = a.shape
        out = np.empty_like(a)
        for b in range(B):
            v = np.ascontiguousarray(a[b].T)
            E = ((row0 + b) * np.arange(n)) % self.N
            if inverse:
                E = np.where(E != 0, self.N - E, 0)
            j, sh = E % self.M, E // self.M
            w = np.ascontiguousarray(self.tab[j])
            y = O.mul(v, w, R8, backend="school")
            for s in np.unique(sh):
                sel = sh == s
                y[sel] = O.mul_pow_r(np.ascontiguousarray(y[sel]), R8, int(s))
            out[b] = y.T
        return torch.from_numpy(out.view(np.int64))


def _e(n):
    e = 0
    while n > 1:
        n //= K
        e += 1
    return e


def _pow(x, e, N):
    acc = np.zeros((1, k), dtype=np.uint64)
    acc[0, 0] = 1
    base = np.asarray(x, dtype=np.uint64).reshape(1, k).copy()
    while e:
        if e & 1:
            acc = O.mul(acc, base, R8, backend="school")
        base = O.mul(base, base, R8, backend="school")
        e >>= 1
    return acc[0]


def _np(t):
    a = t.numpy() if t.dtype == torch.int64 else t.view(torch.int64).numpy()
    return a.view(np.uint64)


def _worker(rank, world, port, N1, N2, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_01490_b200.sharded import ShardedFFT
        N = N1 * N2
        _, omega = O.gfp_root(k, R8, N)
        ops = OracleShardOps(N1, N2, omega)
        sh = ShardedFFT(ops, k, N1, N2, rank, world)
        x = O.random_elements(4, k, R8, N)                       # element-major [N, k]
        xd = torch.from_numpy(np.ascontiguousarray(x.T).view(np.int64))  # digit-major
        cols = sh.scatter_columns(xd)
        rows = sh.forward(cols)
        want = ops.big.forward(x)                                 # oracle single-process DFT
        idx = sh.gather_rows_index().numpy()
        got = _np(rows)                                           # [N1/G, k, N2]
        ok_fwd = np.array_equal(got.transpose(0, 2, 1).reshape(-1, k),
                                want[idx.reshape(-1)])
        back = sh.inverse(rows)
        ok_inv = np.array_equal(_np(back), _np(cols))
        q.put((rank, bool(ok_fwd), bool(ok_inv)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("N1,N2", [(16, 256), (256, 256)])
def test_sharded_two_ranks_gloo(N1, N2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N1, N2, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert res == [(0, True, True), (1, True, True)]


def test_sharded_single_rank_layouts():
    # world = 1: no exchange, same orchestration
    from paper_1811_01490_b200.sharded import ShardedFFT
    N1, N2 = 16, 256
    N = N1 * N2
    _, omega = O.gfp_root(k, R8, N)
    ops = OracleShardOps(N1, N2, omega)
    sh = ShardedFFT(ops, k, N1, N2)
    x = O.random_elements(11, k, R8, N)
    xd = torch.from_numpy(np.ascontiguousarray(x.T).view(np.int64))
    rows = sh.forward(sh.scatter_columns(xd))
    want = ops.big.forward(x)
    got = _np(rows).transpose(0, 2, 1).reshape(-1, k)
    assert np.array_equal(got, want[sh.gather_rows_index().numpy().reshape(-1)])
