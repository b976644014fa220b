"""DFT of N = K^e points over GF(r^k + 1), K = 2k, on the GPU.

Mirrors gfpfft/fft.py's public surface (build_plan, FftPlan, dft_general,
dft_inverse, dft_base, stride_permutation, twiddle_apply) for the GFP field,
plus the tensor-level API the data-parallel path is built for:

  plan = build_plan(field, K, e, omega)       # fft.py:237-275
  y = fft(x, plan)                            # x: [k, N] or [B, k, N] uint64 CUDA
  x = fft(y, plan, inverse=True)              # includes the N^-1 scale
  h = poly_mul(f, g, plan)                    # IDFT(DFT(f) .* DFT(g))

The schedule is not the reference's (right-to-left stride permutations,
separate twiddle stages): each of the e passes is one Stockham radix-K
kernel (csrc/gfp_pass44.cuh k_pass44 for k = 8, csrc/gfp_pass.cuh k_pass
otherwise) that reads K elements at stride N/K, multiplies by omega^E (the r^a part of omega^E = r^a omega^b folded into a
digit rotation, the reference's cheap-twiddle split, fft.py:84-103),
runs the K-point DFT at root r with shift-only butterflies, and writes in
natural order.  The output is the unique canonical encoding of the DFT, so it
equals dft_general's bit for bit.
"""

import ctypes
import time

import numpy as np
import torch

from . import _lib, vec
from .gfp_field import gfp_encode

BASE_SIZES = (8, 16, 32, 64)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class FftPlan:
    """Device plan for a size K^e transform at root omega (fft.py:199-234).

    Holds the C plan (twiddle tables omega^j and omega^j N^-1 in HBM).
    Attributes follow the reference: K, e, N, omega, omega_base,
    shift_step, cheap_twiddle, threads.
    """

    def __init__(self, field, K, e, omega, handle, shift_step, threads=1):
        self.field = field
        self.params = field.params
        self.K = K
        self.e = e
        self.N = K ** e
        self.omega = tuple(omega)
        self.shift_step = shift_step
        self.omega_base = field.shift_root if shift_step > 0 else field.shift_root_inv
        self.cheap_twiddle = True
        self.threads = threads
        self.block = 4
        self._h = handle
        self._inverse = None
        self._n_inv = None
        self._table = None

    @property
    def handle(self):
        return self._h

    def inverse(self):
        """Plan at omega^(N-1) = omega^-1 (fft.py:221-229)."""
        if self._inverse is None:
            omega_inv = self.field.pow(self.omega, self.N - 1)
            self._inverse = build_plan(self.field, self.K, self.e, omega_inv,
                                       threads=self.threads)
        return self._inverse

    def n_inv(self):
        if self._n_inv is None:
            self._n_inv = self.field.inv_scalar(self.N)
        return self._n_inv

    @property
    def twiddle_table(self):
        """omega^j for j < K^(e-1) (fft.py:211-214), computed on the device."""
        if self._table is None:
            M = self.N // self.K
            base = vec.to_device([self.omega], self.params.k)
            ones = vec.to_device([(1,) + (0,) * (self.params.k - 1)] * M, self.params.k)
            # omega^j via device exponentiation of a broadcast base, one
            # exponent per chunk of bits: table[j] = prod_b omega^(2^b [bit b of j])
            out = ones
            j = torch.arange(M, device="cuda", dtype=torch.int64)
            sq = base
            bit = 0
            while (1 << bit) < M:
                mask = ((j >> bit) & 1).bool()
                prod = vec.mul(out, sq, self.params)
                out = torch.where(mask.unsqueeze(0), prod.view(torch.int64),
                                  out.view(torch.int64)).view(torch.uint64).contiguous()
                sq = vec.mul(sq, sq, self.params)
                bit += 1
            self._table = vec.to_tuples(out)
        return self._table

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().gfp_fft_plan_destroy(h)
            except Exception:
                pass
            self._h = None


def build_plan(field, K, e, omega, cheap_twiddle=None, threads=1):
    """Validate omega and build the device twiddle tables (fft.py:237-275).

    Raises ValueError when K is not a base size, e < 1, omega is not a
    primitive N-th root, K != 2k, or omega^(N/2k) is neither r nor 1/r --
    the reference's rejections, checked on the device.
    """
    from .word import build_word_plan
    # The reference accepts any object of its field protocol (fft.py:13-17).
    # The device transform is chosen by the field's structure, not its class,
    # so the reference's own field objects plug in too:
    #   word-prime fields (a Montgomery context .ctx with .q, like MontField,
    #   fft.py:376-421) -> the word-prime transform (csrc/gfp_word.cu);
    #   shift-capable GFP fields (.params with r, k, plus shift_root / two_k,
    #   like GfpFftField, gfp_mult.py:518-592) -> the GFP transform.
    ctx = getattr(field, "ctx", None)
    if ctx is not None and hasattr(ctx, "q") and hasattr(ctx, "one_mont"):
        return build_word_plan(field, K, e, omega)
    if K not in BASE_SIZES:
        raise ValueError("unsupported base-case size")
    if e < 1:
        raise ValueError("e must be at least 1")
    params = getattr(field, "params", None)
    if (params is None or not hasattr(params, "r") or not hasattr(params, "k")
            or not hasattr(field, "shift_root") or not hasattr(field, "two_k")):
        raise ValueError("no device transform for this field: the GPU path covers GF(r^k + 1) "
                         "fields (GfpFftField protocol) and word-prime Montgomery fields")
    if K != field.two_k:
        raise ValueError("base-case size must equal 2k for this field")
    k = params.k
    om = tuple(int(d) for d in omega)
    if len(om) != k:
        raise ValueError("omega must have k digits")
    from .gfp_field import is_canonical
    if not is_canonical(params, om):
        raise ValueError("omega is not a canonical element")
    arr = (ctypes.c_uint64 * k)(*om)
    h = ctypes.c_void_p()
    code = _lib.load().gfp_fft_plan_create(ctypes.byref(h), k, params.r, K, e, arr, _stream())
    if code == _lib.GFP_EINVAL:
        raise ValueError("omega is not a primitive N-th root with omega^(N/2k) in {r, 1/r}")
    _lib.check(code, "gfp_fft_plan_create")
    N = K ** e
    head = field.pow(om, N // field.two_k)
    shift_step = 1 if head == field.shift_root else -1
    return FftPlan(field, K, e, om, h.value, shift_step, threads)


def _as_batch(x, plan):
    k, N = plan.params.k, plan.N
    if x.dim() == 2:
        if tuple(x.shape) != (k, N):
            raise ValueError("vector length must equal K^e")
        return x.unsqueeze(0), True
    if x.dim() == 3 and tuple(x.shape[1:]) == (k, N):
        return x, False
    raise ValueError("expected [k, N] or [batch, k, N]")


def fft(x, plan, inverse=False, out=None):
    """Batched forward / inverse DFT of digit-major device tensors."""
    vec._require_cuda(x)
    xb, squeeze = _as_batch(x, plan)
    B = xb.shape[0]
    if out is None:
        out = torch.empty_like(xb)
    else:
        vec._require_cuda(out)
        out = out.view_as(xb)
    if B == 0:  # an empty batch: nothing to transform
        return out
    work = torch.empty(int(_lib.load().gfp_fft_workspace_words(plan.handle, B)),
                       dtype=torch.uint64, device=x.device)
    _lib.check(_lib.load().gfp_fft_exec(plan.handle, _ptr(xb), _ptr(out), _ptr(work), B,
                                       1 if inverse else 0, _stream()), "gfp_fft_exec")
    return out.squeeze(0) if squeeze else out


def poly_mul(f, g, plan, out=None):
    """Cyclic product IDFT(DFT(f) .* DFT(g)) of digit-major device tensors
    (the polynomial product when deg f + deg g < N)."""
    vec._require_cuda(f, g)
    fb, squeeze = _as_batch(f, plan)
    gb, _ = _as_batch(g, plan)
    if fb.shape != gb.shape:
        raise ValueError("shape mismatch")
    B = fb.shape[0]
    out = torch.empty_like(fb) if out is None else out.view_as(fb)
    work = torch.empty(int(_lib.load().gfp_fft_workspace_words(plan.handle, B)),
                       dtype=torch.uint64, device=f.device)
    _lib.check(_lib.load().gfp_poly_mul(plan.handle, _ptr(fb), _ptr(gb), _ptr(out), _ptr(work),
                                       B, _stream()), "gfp_poly_mul")
    return out.squeeze(0) if squeeze else out


def last_launches(plan):
    """Kernel launches of the last exec / poly_mul on this plan."""
    return int(_lib.load().gfp_fft_plan_last_launches(plan.handle))


# ---------------------------------------------------------------------------
# host-buffer entry points (the e2e path: H2D, transform, D2H in one C call)

def fft_host(v, plan, inverse=False, inplace=False):
    """Element-major host array [N, k] or [B, N, k] (uint64) -> new array, or
    v itself transformed in place (inplace=True: v must be a C-contiguous
    uint64 array; pinned memory is then read and written by the kernels
    directly)."""
    if inplace:
        if not (isinstance(v, np.ndarray) and v.dtype == np.uint64 and v.flags.c_contiguous):
            raise ValueError("inplace needs a C-contiguous uint64 array")
        a = v
    else:
        a = np.ascontiguousarray(np.asarray(v, dtype=np.uint64)).copy()
    B = a.size // (plan.N * plan.params.k)
    _lib.check(_lib.load().gfp_fft_exec_host(plan.handle, ctypes.c_void_p(a.ctypes.data), B,
                                            1 if inverse else 0, _stream()),
               "gfp_fft_exec_host")
    return a


def poly_mul_host(f, g, plan):
    """Product of host coefficient arrays [n, k] (or [B, n, k]) with n <= N:
    [min(nf + ng - 1, N), k] -- the linear product when it fits in N, else
    the cyclic one (N-length inputs give the length-N cyclic product)."""
    f = np.ascontiguousarray(np.asarray(f, dtype=np.uint64))
    g = np.ascontiguousarray(np.asarray(g, dtype=np.uint64))
    k = plan.params.k
    if f.ndim == 2:
        f, g, squeeze = f[None], g[None], True
    else:
        squeeze = False
    B, nf, ng = f.shape[0], f.shape[1], g.shape[1]
    if g.shape[0] != B or f.shape[2] != k or g.shape[2] != k:
        raise ValueError("operand shapes must be [n, k] (or [B, n, k]) with matching B")
    if not (1 <= nf <= plan.N and 1 <= ng <= plan.N):
        raise ValueError("polynomial lengths must be in [1, N]")
    n_out = min(nf + ng - 1, plan.N)
    out = np.empty((B, n_out, k), dtype=np.uint64)
    _lib.check(_lib.load().gfp_poly_mul_host2(plan.handle, ctypes.c_void_p(f.ctypes.data), nf,
                                             ctypes.c_void_p(g.ctypes.data), ng,
                                             ctypes.c_void_p(out.ctypes.data), B, _stream()),
               "gfp_poly_mul_host2")
    return out[0] if squeeze else out


# ---------------------------------------------------------------------------
# the reference's list-of-tuples API

def dft_general(v, plan, field=None, profile=None):
    """In-place DFT of K^e points (fft.py:298-360); returns v.

    profile, when given, accumulates seconds under the reference's phase
    keys "permutation", "basecase" and "twiddle" (see pass_profile).
    """
    from .word import WordPlan, dft_word
    if isinstance(plan, WordPlan):
        return dft_word(v, plan)
    if len(v) != plan.N:
        raise ValueError("vector length must equal K^e")
    _run_list(v, plan, False, profile)
    return v


def dft_inverse(v, plan, field=None, profile=None):
    """Inverse transform including the 1/N scale (fft.py:363-370)."""
    from .word import WordPlan, dft_word
    if isinstance(plan, WordPlan):
        return dft_word(v, plan, inverse=True)
    if len(v) != plan.N:
        raise ValueError("vector length must equal K^e")
    _run_list(v, plan, True, profile)
    return v


def pass_times(plan, fn):
    """Run fn() with per-pass device timing on plan; returns fn's result and
    [(pass index, ms)] of its pass launches (gfp_fft_plan_pass_times)."""
    lib = _lib.load()
    _lib.check(lib.gfp_fft_plan_set_timing(plan.handle, 1), "gfp_fft_plan_set_timing")
    try:
        res = fn()
        ms = (ctypes.c_float * 64)()
        idx = (ctypes.c_int * 64)()
        n = lib.gfp_fft_plan_pass_times(plan.handle, ms, idx, 64)
        if n < 0:
            _lib.check(-n, "gfp_fft_plan_pass_times")
    finally:
        lib.gfp_fft_plan_set_timing(plan.handle, 0)
    return res, [(int(idx[i]), float(ms[i])) for i in range(n)]


def pass_profile(passes, moved_seconds):
    """The reference's dft_general phases (fft.py:298-360) from the device
    passes.  The GPU fuses the phases: each Stockham pass applies one level's
    twiddles (none in the first pass) and one layer of K-point base cases,
    and the stride permutations are its load / store indexing.  So:
      basecase    = the first pass (base cases only, no twiddle);
      twiddle     = the later passes (each a level's twiddle multiplies --
                    the bulk of its instructions -- fused with its layer of
                    base cases; the inverse's N^-1 scale rides on the last);
      permutation = the data movement outside the passes (host list ->
                    device digit-major vectors and back)."""
    base = sum(ms for i, ms in passes if i == 0) * 1e-3
    tw = sum(ms for i, ms in passes if i > 0) * 1e-3
    return {"permutation": moved_seconds, "basecase": base, "twiddle": tw}


def _run_list(v, plan, inverse, profile):
    if profile is None:
        v[:] = vec.to_tuples(fft(vec.to_device(v, plan.params.k), plan, inverse=inverse))
        return
    t0 = time.perf_counter()
    x = vec.to_device(v, plan.params.k)
    torch.cuda.synchronize()
    moved = time.perf_counter() - t0
    y, passes = pass_times(plan, lambda: fft(x, plan, inverse=inverse))
    t0 = time.perf_counter()
    v[:] = vec.to_tuples(y)
    moved += time.perf_counter() - t0
    for key, sec in pass_profile(passes, moved).items():
        profile[key] = profile.get(key, 0.0) + sec


_base_plans = {}


def dft_base(v, omega_base, field, K=None, offset=0):
    """In-place K-point DFT at omega_base in {r, 1/r} (fft.py:186-193)."""
    if K is None:
        K = len(v)
    if K not in BASE_SIZES:
        raise ValueError("unsupported base-case size")
    key = (field.params, K, tuple(omega_base))
    plan = _base_plans.get(key)
    if plan is None:
        plan = build_plan(field, K, 1, omega_base)
        _base_plans[key] = plan
    block = list(v[offset:offset + K])
    dft_general(block, plan, field)
    v[offset:offset + K] = block
    return v


def stride_permutation(v, m, n, block=16, offset=0):
    """L_m^{mn}: element j*m + i -> i*n + j (fft.py:34-56).

    A host-side list permutation (no field arithmetic), kept for API
    compatibility; the device transform never materialises it -- its
    Stockham passes fold the permutations into their load/store indexing.
    """
    if len(v) < offset + m * n:
        raise ValueError("vector length must equal m*n")
    if m == 1 or n == 1:
        return v
    out = [None] * (m * n)
    for j in range(n):
        base = offset + j * m
        for i in range(m):
            out[i * n + j] = v[base + i]
    v[offset:offset + m * n] = out
    return v


def twiddle_apply(v, m, n, omega_i, field, offset=0):
    """v[j*m + i] *= omega_i^(i*j) for j < n, i < m (fft.py:62-81), with the
    multiplies batched on the device."""
    if m == 1:
        return v
    params = field.params
    k = params.k
    block = vec.to_device(v[offset:offset + m * n], k)          # [k, m*n]
    # row[j] = omega_i^j (j < n), then powers row[j]^i by running products
    w = vec.to_device([omega_i], k)
    rows = [vec.to_device([field.one()], k)]
    for _ in range(1, n):
        rows.append(vec.mul(rows[-1], w, params))
    i64 = torch.int64
    row = torch.cat([t.view(i64) for t in rows], dim=1).contiguous().view(torch.uint64)
    ones = vec.to_device([field.one()] * n, k)
    factors = [ones]
    for _ in range(1, m):
        factors.append(vec.mul(factors[-1], row, params))
    F = torch.stack([t.view(i64) for t in factors], dim=2).reshape(k, n * m)  # j*m + i
    res = vec.mul(block, F.contiguous().view(torch.uint64), params)
    v[offset:offset + m * n] = vec.to_tuples(res)
    return v


def poly_mul_list(f, g, plan):
    """Cyclic product of two length-N lists of elements (tuples)."""
    k = plan.params.k
    out = poly_mul(vec.to_device(f, k), vec.to_device(g, k), plan)
    return vec.to_tuples(out)


def roots_for(params, N):
    """The reference's root convention: bench_cli._gfp_root (bench_cli.py:398-402)."""
    from .gfp_field import gfp_find_nth_root, gfp_primitive_root
    g = gfp_find_nth_root(params, N, seed=0)
    return gfp_primitive_root(params, N, g)


def encode_many(params, ints):
    return [gfp_encode(params, n) for n in ints]
