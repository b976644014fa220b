"""One N = N1 * N2 point GF(p) transform sharded across ranks (four-step).

The reference has no distributed transform; this is the multi-GPU row of
SURVEY §8(e) (BASELINE.json config C4: N = 2^24 = 2^12 * 2^12 over 1-8
GPUs).  With n = N2 n1 + n2 and k = k1 + N1 k2:

    X[k1 + N1 k2] = sum_n2 w_N2^(n2 k2) [ w_N^(n2 k1) sum_n1 x[N2 n1 + n2] w_N1^(n1 k1) ]

  1. column DFTs of size N1 on the local columns n2 (batched k_pass kernels);
  2. the inter-stage twiddle w_N^(n2 k1) (gfp_fft_twiddle, the D_{N1,N2}
     stage of the reference's tensor formula, fft.py:62-103);
  3. the transpose: ONE all-to-all (torch.distributed.all_to_all_single,
     NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests), or -- with
     use_peer_exchange() -- direct stores into every rank's receive buffer
     over CUDA IPC peer pointers, fused into the column DFTs' last pass
     (PeerExchange: host barriers, NCCL barriers or device-side
     release/acquire completion flags between the ranks' kernels);
  4. row DFTs of size N2 on the local rows k1.

Layouts (digit-major, like every device vector of the package):
  columns  rank g holds n2 in [g N2/G, (g+1) N2/G) as [N2/G, k, N1]
           (cols[n2l, d, n1] = digit d of x[N2 n1 + n2]);
  rows     rank g holds k1 in [g N1/G, (g+1) N1/G) as [N1/G, k, N2]
           (rows[k1l, d, k2] = digit d of X[k1 + N1 k2]).
The inverse runs the same steps backwards (inverse row DFTs, all-to-all,
conjugate twiddle, inverse column DFTs; the two local N^-1 scales multiply
to 1/N), so forward followed by inverse returns the input columns.

The orchestration is backend-agnostic: `ops` supplies the three local
operations (GPU: GpuShardOps, libgfpfft kernels; the CPU tests plug in the
oracle), the permutes are torch views on int64, the exchange is
torch.distributed.
"""

import torch


def _i64(t):
    return t.view(torch.int64) if t.dtype == torch.uint64 else t


def _u64(t):
    return t.view(torch.uint64) if t.dtype == torch.int64 and t.is_cuda else t


class ShardedFFT:
    """One rank's share of an N1 N2-point transform (see the module
    docstring): forward(cols) -> rows, inverse(rows) -> cols; the exchange
    path in use is recorded in exchange_path."""

    def __init__(self, ops, k, N1, N2, rank=0, world=1, group=None):
        if N1 % world or N2 % world:
            raise ValueError("N1 and N2 must be divisible by the number of ranks")
        self.ops, self.k, self.N1, self.N2 = ops, k, N1, N2
        self.rank, self.world, self.group = rank, world, group
        self.c1 = N1 // world  # local rows
        self.c2 = N2 // world  # local columns
        self.peer = None       # PeerExchange: the transpose as peer stores
        self.exchange_path = "all_to_all_single" if world > 1 else "local"

    def exchange_shapes(self):
        return {"rows": (self.c1, self.k, self.N2), "cols": (self.c2, self.k, self.N1)}

    def use_peer_exchange(self, device=None, local_peers=None, fuse=True):
        """Switch the transpose from all_to_all_single to direct stores into
        every rank's receive buffer over CUDA IPC peer pointers: fused into
        the last pass of the preceding DFTs (gfp_fft_exec_exchange) when
        `fuse` and the pass kernel supports it, else one
        gfp_exchange_transpose kernel (instead of pack / all-to-all / unpack)."""
        try:
            self.peer = PeerExchange(self.exchange_shapes(), self.rank, self.world, self.group,
                                     device, local_peers)
        except PeerIPCError as exc:
            # every rank saw the same failure (PeerExchange agrees on it), so
            # every rank stays on the NCCL all-to-all path
            self.peer = None
            self.exchange_path = "all_to_all_single (peer IPC unavailable: %s)" % str(exc)[:200]
            return self
        self.peer.fuse = fuse
        self.exchange_path = "peer stores (%s)" % ("fused into the last pass" if fuse
                                                   else "gfp_exchange_transpose")
        return self

    # -- exchange ---------------------------------------------------------
    def _all_to_all(self, send):
        if self.world == 1:
            return send
        import torch.distributed as dist
        src = _i64(send).contiguous()
        recv = torch.empty_like(src)
        dist.all_to_all_single(recv, src, group=self.group)
        return recv.view(send.dtype) if send.dtype != recv.dtype else recv

    # -- forward ----------------------------------------------------------
    def forward_columns(self, cols):
        """Step 1 (+2): column DFTs [N2/G, k, N1] -> A[n2l, d, k1]."""
        if getattr(self.ops, "fused", False):  # lazy digits through the exchange
            return self.ops.fft_ex(cols, "N1", inverse=False, in_canon=True, out_canon=False)
        y = self.ops.fft(cols, "N1", inverse=False)
        return self.ops.twiddle(y, self.rank * self.c2, inverse=False)   # * w_N^(n2 k1)

    def forward_rows(self, rows):
        """Step 4: row DFTs [N1/G, k, N2] (+ the folded twiddle)."""
        if getattr(self.ops, "fused", False):  # * w_N^(k1 n2) on the row DFT's first pass
            return self.ops.fft_ex(_u64(rows), "N2", inverse=False, in_canon=False,
                                   out_canon=True, ft_row0=self.rank * self.c1)
        return self.ops.fft(_u64(rows), "N2", inverse=False)

    def columns_to_rows(self, cols, wait=True):
        """Steps 1-3: column DFTs, twiddle and the transpose; returns this
        rank's rows [N1/G, k, N2] (before the row DFTs).  wait=False (peer
        exchange, emulated ranks): return after publishing this rank's
        stores; peer.finish("rows") completes the exchange."""
        G, k, c1, c2 = self.world, self.k, self.c1, self.c2
        if self.peer is not None:
            if self.peer.fuse and getattr(self.ops, "fused", False):
                # the column DFTs' last pass stores straight into the owners'
                # row buffers (gfp_fft_exec_exchange)
                res = self.peer.begin("rows", lambda: self.ops.fft_exchange(
                    cols, "N1", False, True, False, self.peer.addrs["rows"], G, self.rank))
                if res:
                    if wait:
                        self.peer.finish("rows", res)
                    return self.peer.recv["rows"]
            y = self.forward_columns(cols)  # one kernel stores into every rank's buffer
            return self.peer.transpose("rows", y, A=c2, B=self.N1, wait=wait)
        y = self.forward_columns(cols)
        send = _i64(y).view(c2, k, G, c1).permute(2, 0, 1, 3).contiguous()
        recv = self._all_to_all(send)                                  # [g, n2l, d, k1l]
        return recv.permute(3, 2, 0, 1).reshape(c1, k, self.N2).contiguous()

    def forward(self, cols):
        """cols [N2/G, k, N1] (canonical) -> rows [N1/G, k, N2] (canonical)."""
        out = self.forward_rows(self.columns_to_rows(cols))
        if self.peer is not None:
            self.peer.consumed("rows")  # the row DFTs have read the receive buffer
        return out

    # -- inverse ----------------------------------------------------------
    def inverse_rows(self, rows):
        """Inverse row DFTs [N1/G, k, N2] -> B[k1l, d, n2]."""
        if getattr(self.ops, "fused", False):
            return self.ops.fft_ex(rows, "N2", inverse=True, in_canon=True, out_canon=False)
        return self.ops.fft(rows, "N2", inverse=True)

    def inverse_columns(self, cols):
        """Conjugate twiddle + inverse column DFTs [N2/G, k, N1]."""
        if getattr(self.ops, "fused", False):  # * w_N^-(n2 k1) on the first pass
            return self.ops.fft_ex(_u64(cols), "N1", inverse=True, in_canon=False,
                                   out_canon=True, ft_row0=self.rank * self.c2, ft_inverse=True)
        cols = self.ops.twiddle(_u64(cols), self.rank * self.c2, inverse=True)
        return self.ops.fft(cols, "N1", inverse=True)

    def rows_to_columns(self, rows, wait=True):
        """Inverse row DFTs and the transpose back; returns this rank's
        columns [N2/G, k, N1] (before the conjugate twiddle)."""
        G, k, c1, c2 = self.world, self.k, self.c1, self.c2
        if self.peer is not None:
            if self.peer.fuse and getattr(self.ops, "fused", False):
                res = self.peer.begin("cols", lambda: self.ops.fft_exchange(
                    rows, "N2", True, True, False, self.peer.addrs["cols"], G, self.rank))
                if res:
                    if wait:
                        self.peer.finish("cols", res)
                    return self.peer.recv["cols"]
            z = self.inverse_rows(rows)
            return self.peer.transpose("cols", z, A=c1, B=self.N2, wait=wait)
        z = self.inverse_rows(rows)
        send = _i64(z).view(c1, k, G, c2).permute(2, 0, 1, 3).contiguous()
        recv = self._all_to_all(send)                                  # [g, k1l, d, n2l]
        return recv.permute(3, 2, 0, 1).reshape(c2, k, self.N1).contiguous()

    def inverse(self, rows):
        """rows [N1/G, k, N2] -> cols [N2/G, k, N1]; inverse of forward()."""
        out = self.inverse_columns(self.rows_to_columns(rows))
        if self.peer is not None:
            self.peer.consumed("cols")
        return out

    # -- global <-> local layouts (tests and benchmark data placement) ----
    def scatter_columns(self, x):
        """Natural-order digit-major [k, N] -> this rank's columns."""
        k = self.k
        n2_0 = self.rank * self.c2
        v = _i64(x).view(k, self.N1, self.N2)[:, :, n2_0:n2_0 + self.c2]
        return _u64(v.permute(2, 0, 1).contiguous())

    def gather_rows_index(self):
        """Global output indices k1 + N1 k2 of this rank's rows, [N1/G, N2]."""
        k1 = torch.arange(self.rank * self.c1, (self.rank + 1) * self.c1).view(-1, 1)
        k2 = torch.arange(self.N2).view(1, -1)
        return k1 + self.N1 * k2


def _barrier(group):
    import torch.distributed as dist
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=group)


class PeerIPCError(RuntimeError):
    """CUDA IPC / peer access unavailable on some rank."""


class PeerExchange:
    """Receive buffers of the four-step transpose and every rank's address of
    them: CUDA IPC handles (gfp_ipc_get_handle / gfp_ipc_open) gathered once
    with all_gather_object, so each exchange is one kernel writing over NVLink
    into the owners' buffers (the fused XCH pass or gfp_exchange_transpose).

    Synchronisation of an exchange named n ("rows" / "cols"), three modes:
      host   (default) two host barriers: peers finished reading their
             buffers (previous exchange) before the stores start, and every
             store into this rank's buffer landed before it is read;
      nccl   the same two barriers as stream-ordered one-element NCCL
             all-reduces (use_device_barrier);
      flags  device-side completion flags, no host involvement
             (use_device_flags): per exchange an epoch e,
               wait  consumed[n][g] >= e - 1   (peer g read its previous buffer)
               the stores (fn)
               signal ready[n] = e into every peer   (st.release.sys)
               wait  ready[n][g] >= e            (every peer's stores landed)
             and after the kernel that reads recv[n], consumed(n) signals
             consumed[n] = e (gfp_flag_signal / gfp_flag_wait).
    begin(n, fn) / finish(n) split an exchange at the point where a rank
    waits for its peers (the emulated-ranks tests issue every rank's begin
    before any finish on one stream); bracket(fn, n) is both.

    ``local_peers`` (tests, one process): a list of G PeerExchange-like
    receive-buffer dicts on this device standing in for the peers (no
    barriers; the caller runs the ranks' stages in order)."""

    SLOTS = {"rows": (0, 2), "cols": (1, 3)}  # (ready, consumed) flag slots

    def __init__(self, shapes, rank, world, group=None, device=None, local_peers=None):
        import ctypes
        from . import _lib
        self.rank, self.world, self.group = rank, world, group
        self._opened = []
        self.addrs = {}
        self.fuse = True
        self.mode = "host"
        self.device_barrier = False
        self._flag = None
        self.max_spins = 1 << 24  # ~1 s of polling per wait before an error is recorded
        self.epoch = {n: 0 for n in self.SLOTS}
        self.local = local_peers is not None
        if self.local:
            mine = local_peers[rank]
            self.recv = {n: t for n, t in mine.items() if not n.startswith("__")}
            self.flags, self.err = mine["__flags"], mine["__err"]
            for n in shapes:
                self.addrs[n] = [p[n].data_ptr() for p in local_peers]
            self.flag_addrs = [p["__flags"].data_ptr() for p in local_peers]
            return
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.recv = {n: torch.empty(sh, dtype=torch.int64, device=dev).view(torch.uint64)
                     for n, sh in shapes.items()}
        self.flags = torch.zeros((4, world), dtype=torch.int64, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        if world == 1:
            self.addrs = {n: [t.data_ptr()] for n, t in self.recv.items()}
            self.flag_addrs = [self.flags.data_ptr()]
            return
        import torch.distributed as dist
        lib = _lib.load()
        shared = dict(self.recv, __flags=self.flags)
        mine, failure = {}, None
        try:
            for n, t in shared.items():
                h = ctypes.create_string_buffer(64)
                off = ctypes.c_int64(0)
                _lib.check(lib.gfp_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), h,
                                                  ctypes.byref(off)), "gfp_ipc_get_handle")
                mine[n] = (h.raw, off.value)
        except Exception as exc:  # reported to every rank below
            failure = "rank %d: %s" % (rank, exc)
        every = [None] * world
        dist.all_gather_object(every, (mine, failure), group=group)
        addrs = {n: [] for n in shared}
        try:
            bad = [f for _, f in every if f]
            if bad:
                raise PeerIPCError("; ".join(bad))
            for n, t in shared.items():
                for g in range(world):
                    if g == rank:
                        addrs[n].append(t.data_ptr())
                        continue
                    raw, off = every[g][0][n]
                    ptr = ctypes.c_void_p(0)
                    _lib.check(lib.gfp_ipc_open(raw, off, ctypes.byref(ptr)), "gfp_ipc_open")
                    addrs[n].append(ptr.value)
                    self._opened.append((ptr.value, off))
            failure = None
        except Exception as exc:
            failure = "rank %d: %s" % (rank, exc)
        # every rank agrees on the outcome before anyone uses a peer pointer
        outcome = [None] * world
        dist.all_gather_object(outcome, failure, group=group)
        bad = [f for f in outcome if f]
        if bad:
            self.close()
            raise PeerIPCError("; ".join(bad))
        self.flag_addrs = addrs.pop("__flags")
        self.addrs = addrs

    def use_device_barrier(self):
        """Replace the two host barriers by stream-ordered NCCL barriers (only
        with an NCCL group -- 'nccl' or a device-specific 'cuda:nccl' backend;
        a no-op otherwise)."""
        if self.world > 1 and not self.local:
            import torch.distributed as dist
            if "nccl" in str(dist.get_backend(self.group)):
                self.mode = "nccl"
                self.device_barrier = True
                self._flag = torch.zeros(1, dtype=torch.int32,
                                         device=next(iter(self.recv.values())).device)
        return self

    def use_device_flags(self, max_spins=None):
        """Device-side completion flags instead of barriers (see the class
        docstring): the host never blocks between the exchange's kernels."""
        self.mode = "flags"
        if max_spins is not None:
            self.max_spins = int(max_spins)
        return self

    @staticmethod
    def local_buffers(shapes, world, device="cuda"):
        """Receive buffers (and flag arrays) of `world` emulated ranks on one
        device."""
        out = []
        for _ in range(world):
            d = {n: torch.empty(sh, dtype=torch.int64, device=device).view(torch.uint64)
                 for n, sh in shapes.items()}
            d["__flags"] = torch.zeros((4, world), dtype=torch.int64, device=device)
            d["__err"] = torch.zeros(1, dtype=torch.int32, device=device)
            out.append(d)
        return out

    # -- the three synchronisation modes ------------------------------------
    def _sync(self):
        if self.device_barrier:
            # stream-ordered barrier: a one-element NCCL all-reduce on the
            # current stream (it starts after this rank's queued kernels and
            # completes when every rank reached it; the host never blocks)
            import torch.distributed as dist
            dist.all_reduce(self._flag, group=self.group)
        else:
            _barrier(self.group)

    def _stream(self):
        import ctypes
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def _signal(self, slot, epoch):
        import ctypes
        from . import _lib
        ptrs = (ctypes.c_uint64 * self.world)(*self.flag_addrs)
        _lib.check(_lib.load().gfp_flag_signal(ptrs, self.world, slot, self.rank, epoch,
                                               self._stream()), "gfp_flag_signal")

    def _wait(self, slot, epoch):
        import ctypes
        from . import _lib
        _lib.check(_lib.load().gfp_flag_wait(
            ctypes.c_void_p(self.flags.data_ptr()), self.world, slot, epoch, self.max_spins,
            ctypes.c_void_p(self.err.data_ptr()), self._stream()), "gfp_flag_wait")

    def _flags_on(self):
        return self.mode == "flags" and (self.world > 1 or self.local)

    def begin(self, name, fn):
        """The first half of an exchange: wait until the peers may be written
        (flags: their previous buffers consumed; barrier modes: a barrier),
        run fn (the stores into every rank's recv[name]; False = this route
        is unsupported and nothing was stored) and publish the stores."""
        if self._flags_on():
            ready, consumed = self.SLOTS[name]
            epoch = self.epoch[name] + 1
            self._wait(consumed, epoch - 1)
            res = fn()
            if res is not False:
                self._signal(ready, epoch)
                self.epoch[name] = epoch
            return res
        if self.world > 1 and not self.local:
            self._sync()
        return fn()

    def finish(self, name, res=True):
        """The second half: every peer's stores into recv[name] have landed."""
        if res is False:
            return
        if self._flags_on():
            self._wait(self.SLOTS[name][0], self.epoch[name])
        elif self.world > 1 and not self.local:
            self._sync()

    def bracket(self, fn, name="rows"):
        """begin + finish: run fn (stores into the peers' buffers) between the
        two synchronisation points; returns fn's result.  Every rank takes
        the same branch (the supported-or-not outcome of fn depends only on
        shapes)."""
        res = self.begin(name, fn)
        self.finish(name, res)
        return res

    def consumed(self, name):
        """After the kernel that read recv[name] (flags mode): tell every peer
        it may write the buffer again."""
        if self._flags_on():
            self._signal(self.SLOTS[name][1], self.epoch[name])

    def check(self):
        """Raise if a flag wait timed out (reads the device error word)."""
        e = int(self.err.item())
        if e:
            e -= 1
            raise RuntimeError("peer-exchange flag wait timed out: slot %d, rank %d"
                               % (e // 256, e % 256))

    def transpose(self, name, src, A, B, wait=True):
        """src [A, k, B] -> every rank's recv[name] (see gfp_exchange_transpose);
        returns this rank's receive buffer."""
        import ctypes
        from . import _lib
        src = _u64(src).contiguous()
        k = src.shape[1]
        ptrs = (ctypes.c_uint64 * self.world)(*self.addrs[name])

        def run():
            _lib.check(_lib.load().gfp_exchange_transpose(
                ctypes.c_void_p(src.data_ptr()), ptrs, self.world, self.rank, A, k, B,
                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
                "gfp_exchange_transpose")
        res = self.begin(name, run)
        if wait:
            self.finish(name, res)
        return self.recv[name]

    def close(self):
        import ctypes
        from . import _lib
        for ptr, off in self._opened:
            _lib.load().gfp_ipc_close(ctypes.c_void_p(ptr), off)
        self._opened = []


class GpuShardOps:
    """Local steps of ShardedFFT on the GPU (libgfpfft kernels)."""

    def __init__(self, field, K, N1, N2, omega_N):
        from . import fft as F
        params = field.params
        self.field = field
        N = N1 * N2
        e = lambda n: round(__import__("math").log(n, K))  # noqa: E731
        if K ** e(N1) != N1 or K ** e(N2) != N2:
            raise ValueError("N1 and N2 must be powers of K = 2k")
        self.plan_N = F.build_plan(field, K, e(N), omega_N)
        w1 = field.pow(omega_N, N2)  # N1-th root, w1^(N1/2k) = r
        w2 = field.pow(omega_N, N1)
        self.plans = {"N1": F.build_plan(field, K, e(N1), w1),
                      "N2": F.build_plan(field, K, e(N2), w2)}
        self.params = params
        # pass kernels that can fold the inter-stage twiddle into the next
        # transform's first pass (gfp_fft_exec_ex; k_pass44: k = 8 and a
        # radix with 4 lazy stages per normalisation) are used fused; the
        # library reports it per plan.  Others take the separate twiddle
        # kernel (and the standalone exchange kernel).
        from . import _lib
        lib = _lib.load()
        self.fused = all(lib.gfp_fft_plan_caps(p.handle) & _lib.GFP_CAP_FT
                         for p in self.plans.values())

    def fft(self, x, which, inverse):
        from .fft import fft
        return fft(x.contiguous(), self.plans[which], inverse=inverse)

    def fft_ex(self, x, which, inverse, in_canon, out_canon, ft_row0=None, ft_inverse=False):
        """Batched transform with chosen digit forms; ft_row0 folds the
        four-step twiddle w_N^(+-(ft_row0 + b) i) into the first pass."""
        import ctypes
        from . import _lib
        x = x.contiguous()
        plan = self.plans[which]
        B = x.shape[0]
        out = torch.empty_like(x)
        work = torch.empty(int(_lib.load().gfp_fft_workspace_words(plan.handle, B)),
                           dtype=torch.uint64, device=x.device)
        vp = ctypes.c_void_p
        _lib.check(_lib.load().gfp_fft_exec_ex(
            plan.handle, vp(x.data_ptr()), vp(out.data_ptr()), vp(work.data_ptr()), B,
            1 if inverse else 0, 1 if in_canon else 0, 1 if out_canon else 0,
            vp(self.plan_N.handle) if ft_row0 is not None else None,
            ft_row0 if ft_row0 is not None else 0, 1 if ft_inverse else 0,
            vp(torch.cuda.current_stream().cuda_stream)), "gfp_fft_exec_ex")
        return out

    def fft_exchange(self, x, which, inverse, in_canon, out_canon, dst_addrs, world, rank):
        """Batched transform whose last pass stores into the exchange buffers
        dst_addrs (gfp_fft_exec_exchange); False when the pass kernel cannot
        (the caller then transposes with gfp_exchange_transpose)."""
        import ctypes
        from . import _lib
        lib = _lib.load()
        x = x.contiguous()
        plan = self.plans[which]
        B = x.shape[0]
        scratch = torch.empty_like(x)
        work = torch.empty(int(lib.gfp_fft_workspace_words(plan.handle, B)),
                           dtype=torch.uint64, device=x.device)
        vp = ctypes.c_void_p
        ptrs = (ctypes.c_uint64 * world)(*dst_addrs)
        code = lib.gfp_fft_exec_exchange(
            plan.handle, vp(x.data_ptr()), vp(scratch.data_ptr()), vp(work.data_ptr()), B,
            1 if inverse else 0, 1 if in_canon else 0, 1 if out_canon else 0, ptrs, world, rank,
            vp(torch.cuda.current_stream().cuda_stream))
        if code == _lib.GFP_EUNSUPPORTED:
            return False
        _lib.check(code, "gfp_fft_exec_exchange")
        return True

    def twiddle(self, x, row0, inverse):
        import ctypes
        from . import _lib
        x = x.contiguous()
        out = torch.empty_like(x)
        B, k, n = x.shape
        _lib.check(_lib.load().gfp_fft_twiddle(
            self.plan_N.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            B, n, row0, 1 if inverse else 0,
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "gfp_fft_twiddle")
        return out
