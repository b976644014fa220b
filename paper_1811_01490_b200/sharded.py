"""One N = N1 * N2 point GF(p) transform sharded across ranks (four-step).

The reference has no distributed transform; this is the multi-GPU row of
SURVEY §8(e) (BASELINE.json config C4: N = 2^24 = 2^12 * 2^12 over 1-8
GPUs).  With n = N2 n1 + n2 and k = k1 + N1 k2:

    X[k1 + N1 k2] = sum_n2 w_N2^(n2 k2) [ w_N^(n2 k1) sum_n1 x[N2 n1 + n2] w_N1^(n1 k1) ]

  1. column DFTs of size N1 on the local columns n2 (batched k_pass kernels);
  2. the inter-stage twiddle w_N^(n2 k1) (gfp_fft_twiddle, the D_{N1,N2}
     stage of the reference's tensor formula, fft.py:62-103);
  3. the transpose as ONE all-to-all (torch.distributed.all_to_all_single,
     NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests);
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
    def __init__(self, ops, k, N1, N2, rank=0, world=1, group=None):
        if N1 % world or N2 % world:
            raise ValueError("N1 and N2 must be divisible by the number of ranks")
        self.ops, self.k, self.N1, self.N2 = ops, k, N1, N2
        self.rank, self.world, self.group = rank, world, group
        self.c1 = N1 // world  # local rows
        self.c2 = N2 // world  # local columns

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
    def forward(self, cols):
        """cols [N2/G, k, N1] (canonical) -> rows [N1/G, k, N2] (canonical)."""
        G, k, c1, c2 = self.world, self.k, self.c1, self.c2
        fused = getattr(self.ops, "fused", False)
        if fused:  # lazy digits through the exchange, twiddle folded into the row DFT
            y = self.ops.fft_ex(cols, "N1", inverse=False, in_canon=True, out_canon=False)
        else:
            y = self.ops.fft(cols, "N1", inverse=False)               # A[n2l, d, k1]
            y = self.ops.twiddle(y, self.rank * c2, inverse=False)    # * w_N^(n2 k1)
        send = _i64(y).view(c2, k, G, c1).permute(2, 0, 1, 3).contiguous()
        recv = self._all_to_all(send)                                  # [g, n2l, d, k1l]
        rows = recv.permute(3, 2, 0, 1).reshape(c1, k, self.N2).contiguous()
        if fused:  # * w_N^(k1 n2) on the row DFT's first pass
            return self.ops.fft_ex(_u64(rows), "N2", inverse=False, in_canon=False,
                                   out_canon=True, ft_row0=self.rank * c1)
        return self.ops.fft(_u64(rows), "N2", inverse=False)

    # -- inverse ----------------------------------------------------------
    def inverse(self, rows):
        """rows [N1/G, k, N2] -> cols [N2/G, k, N1]; inverse of forward()."""
        G, k, c1, c2 = self.world, self.k, self.c1, self.c2
        fused = getattr(self.ops, "fused", False)
        if fused:
            z = self.ops.fft_ex(rows, "N2", inverse=True, in_canon=True, out_canon=False)
        else:
            z = self.ops.fft(rows, "N2", inverse=True)               # B[k1l, d, n2]
        send = _i64(z).view(c1, k, G, c2).permute(2, 0, 1, 3).contiguous()
        recv = self._all_to_all(send)                                  # [g, k1l, d, n2l]
        cols = recv.permute(3, 2, 0, 1).reshape(c2, k, self.N1).contiguous()
        if fused:  # * w_N^-(n2 k1) on the column inverse DFT's first pass
            return self.ops.fft_ex(_u64(cols), "N1", inverse=True, in_canon=False,
                                   out_canon=True, ft_row0=self.rank * c2, ft_inverse=True)
        cols = self.ops.twiddle(_u64(cols), self.rank * c2, inverse=True)
        return self.ops.fft(cols, "N1", inverse=True)

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
        # the k_pass44 kernels fold the inter-stage twiddle into the next
        # transform's first pass (gfp_fft_exec_ex); other k use the
        # separate twiddle kernel
        self.fused = params.k == 8 and min(e(N1), e(N2)) >= 2  # (single-pass plans
        # would carry N^-1 and the twiddle in one pass: unfused)

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
