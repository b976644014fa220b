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


class GlooPeer:
    """CPU stand-in for sharded.PeerExchange: the same receive buffers and
    the same store layout as gfp_exchange_transpose,
        dst_g[bl][d][rank A + a] = src[a][d][g b + bl],
    realised with a gloo all_to_all, so the peer-exchange branches of
    ShardedFFT (columns_to_rows / rows_to_columns) run as two real ranks.
    The kernel itself is checked against this layout on the GPU
    (test_exchange_transpose_layout)."""

    def __init__(self, shapes, rank, world):
        self.rank, self.world, self.fuse = rank, world, True
        self.recv = {n: torch.empty(sh, dtype=torch.int64) for n, sh in shapes.items()}
        self.barriers = 0

    def begin(self, name, fn):
        dist.barrier()
        return fn()

    def finish(self, name, res=True):
        if res is not False:
            dist.barrier()
        self.barriers += 1

    def consumed(self, name):
        pass

    def _store(self, name, src, A, B):
        G, b = self.world, B // self.world
        s = src.view(torch.int64) if src.dtype != torch.int64 else src
        kk = s.shape[1]

        def run():
            send = s.view(A, kk, G, b).permute(2, 0, 1, 3).contiguous()   # [g][a][d][bl]
            got = torch.empty_like(send)
            dist.all_to_all_single(got, send)                             # [src rank][a][d][bl]
            self.recv[name].view(b, kk, G, A)[:] = got.permute(3, 2, 0, 1)
        return run

    def transpose(self, name, src, A, B, wait=True):
        res = self.begin(name, self._store(name, src, A, B))
        if wait:
            self.finish(name, res)
        return self.recv[name]


def _flag_peer_class():
    from paper_1811_01490_b200.sharded import PeerExchange

    class CpuFlagPeer(PeerExchange):
        """sharded.PeerExchange in device-flag mode with the two flag
        kernels replaced by their host equivalents on flag arrays in shared
        CPU memory (one per rank, written by the peers): the protocol code
        itself -- begin / finish / consumed, epochs, slots -- is the
        product's, run by two real processes."""

        def __init__(self, shapes, rank, world, shared_flags, log):
            self.rank, self.world, self.group = rank, world, None
            self.fuse, self.local, self.mode = True, False, "flags"
            self.device_barrier = False
            self.epoch = {n: 0 for n in self.SLOTS}
            self.recv = {n: torch.empty(sh, dtype=torch.int64) for n, sh in shapes.items()}
            self.shared, self.log, self.barriers = shared_flags, log, 0
            self._opened = []

        def _signal(self, slot, epoch):  # gfp_flag_signal
            for g in range(self.world):
                self.shared[g][slot, self.rank] = epoch
            self.log.append(("signal", slot, epoch))

        def _wait(self, slot, epoch):    # gfp_flag_wait (bounded spin)
            import time
            t_end = time.monotonic() + 60
            while not bool((self.shared[self.rank][slot] >= epoch).all()):
                if time.monotonic() > t_end:
                    raise RuntimeError("flag wait timed out: slot %d epoch %d" % (slot, epoch))
                time.sleep(0.001)
            self.log.append(("wait", slot, epoch))

        def transpose(self, name, src, A, B, wait=True):
            res = self.begin(name, GlooPeer._store(self, name, src, A, B))
            if wait:
                self.finish(name, res)
            return self.recv[name]

    return CpuFlagPeer


def _peer_worker(rank, world, port, N1, N2, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_01490_b200.sharded import ShardedFFT
        N = N1 * N2
        _, omega = O.gfp_root(k, R8, N)
        ops = OracleShardOps(N1, N2, omega)
        sh = ShardedFFT(ops, k, N1, N2, rank, world)
        sh.peer = GlooPeer(sh.exchange_shapes(), rank, world)
        x = O.random_elements(5, k, R8, N)
        xd = torch.from_numpy(np.ascontiguousarray(x.T).view(np.int64))
        cols = sh.scatter_columns(xd)
        rows = sh.forward(cols)
        want = ops.big.forward(x)
        idx = sh.gather_rows_index().numpy()
        ok_fwd = np.array_equal(_np(rows).transpose(0, 2, 1).reshape(-1, k),
                                want[idx.reshape(-1)])
        ok_inv = np.array_equal(_np(sh.inverse(rows)), _np(cols))
        q.put((rank, bool(ok_fwd), bool(ok_inv), sh.peer.barriers))
    finally:
        dist.destroy_process_group()


def _flag_worker(rank, world, port, N1, N2, flags, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1811_01490_b200.sharded import ShardedFFT
        N = N1 * N2
        _, omega = O.gfp_root(k, R8, N)
        ops = OracleShardOps(N1, N2, omega)
        sh = ShardedFFT(ops, k, N1, N2, rank, world)
        log = []
        sh.peer = _flag_peer_class()(sh.exchange_shapes(), rank, world, flags, log)
        x = O.random_elements(6, k, R8, N)
        xd = torch.from_numpy(np.ascontiguousarray(x.T).view(np.int64))
        cols = sh.scatter_columns(xd)
        want = ops.big.forward(x)
        idx = sh.gather_rows_index().numpy()
        ok = []
        for _ in range(3):  # three round trips: epochs 1..3 on both exchanges
            rows = sh.forward(cols)
            ok.append(np.array_equal(_np(rows).transpose(0, 2, 1).reshape(-1, k),
                                     want[idx.reshape(-1)]))
            ok.append(np.array_equal(_np(sh.inverse(rows)), _np(cols)))
        q.put((rank, all(ok), dict(sh.peer.epoch), log))
    finally:
        dist.destroy_process_group()


def test_sharded_peer_exchange_device_flag_protocol_gloo():
    # the device-flag synchronisation of PeerExchange (begin / finish /
    # consumed with epochs) driving ShardedFFT's peer-exchange branches in two
    # real processes, the flag kernels emulated on shared CPU memory
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    flags = [torch.zeros((4, 2), dtype=torch.int64).share_memory_() for _ in range(2)]
    procs = [ctx.Process(target=_flag_worker, args=(r, 2, port, 16, 256, flags, q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted((q.get(timeout=5) for _ in range(2)), key=lambda t: t[0])
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok, epoch, log in res:
        assert ok and epoch == {"rows": 3, "cols": 3}
        # per exchange: wait(consumed, e-1), signal(ready, e), wait(ready, e),
        # then signal(consumed, e) after the reading DFTs
        assert log[:4] == [("wait", 2, 0), ("signal", 0, 1), ("wait", 0, 1), ("signal", 2, 1)]
        assert log[4:8] == [("wait", 3, 0), ("signal", 1, 1), ("wait", 1, 1), ("signal", 3, 1)]
        assert ("wait", 2, 2) in log and ("signal", 3, 3) in log
    # every flag ends at the last epoch
    assert all(int(f.min()) == 3 for f in flags)


def test_sharded_peer_exchange_two_ranks_gloo():
    # the peer-store exchange branches of ShardedFFT with two gloo ranks:
    # one bracketed transpose per direction, results equal the oracle DFT
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, 16, 256, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert res == [(0, True, True, 2), (1, True, True, 2)]
