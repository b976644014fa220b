"""The word-prime transform on the GPU: DFT over Z/qZ (q an odd prime below
2^63) on Montgomery residues, and the cyclic / negacyclic convolutions.

Mirrors the reference's word-prime layer:
  word_field.py:103-200   WordPrime / word_prime, mont_mul, mont_convert_in/out,
                          word_pow, mont_inv, word_primitive_root
  fft.py:376-421          MontField (the field dft_general runs on for q)
  gfp_mult.py:230-386     cyclic_convolution, negacyclic_convolution
The data-parallel work (transforms, convolutions, batched products) runs in
libgfpfft.so (csrc/gfp_word.cu); there is no CPU path for it.  The scalar
functions here are the plan-time constants and the field protocol's scalar
methods, computed with exact Python integers exactly as the reference
defines them (they are one multiply each; a device round trip per scalar
would only add latency).  Roots come from the reference's seeded search, so
plans and outputs are bit-identical to the reference's.
"""

import ctypes
import random
from dataclasses import dataclass
from functools import lru_cache

import numpy as np
import torch

from . import _lib

MASK64 = (1 << 64) - 1
BASE_SIZES = (8, 16, 32, 64)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


@dataclass(frozen=True)
class WordPrime:
    """An odd prime q < 2^63 with its Montgomery constants (R = 2^64)."""

    q: int
    q_neg_inv: int  # -q^-1 mod 2^64
    r2: int         # 2^128 mod q
    one_mont: int   # 2^64 mod q

    @classmethod
    def make(cls, q):
        """word_field.py:111-119 (constants from the C library's gfp_word_consts)."""
        if q < 3 or q % 2 == 0:
            raise ValueError("q must be an odd prime")
        if q >= 1 << 63:
            raise ValueError("q must be below 2^63")
        qinv, r2, one = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(_lib.load().gfp_word_consts(q, ctypes.byref(qinv), ctypes.byref(r2),
                                               ctypes.byref(one)), "gfp_word_consts")
        return cls(q, qinv.value, r2.value, one.value)


@lru_cache(maxsize=None)
def word_prime(q):
    """Shared WordPrime instance for q (word_field.py:125-130)."""
    return WordPrime.make(q)


def mont_mul(ctx, a, b):
    """REDC product a b 2^-64 mod q (word_field.py:133-140)."""
    c = a * b
    d = ((c & MASK64) * ctx.q_neg_inv) & MASK64
    c = (c + ctx.q * d) >> 64
    return c - ctx.q if c >= ctx.q else c


def mont_convert_in(ctx, a):
    if not 0 <= a < ctx.q:
        raise ValueError("input must be reduced")
    return mont_mul(ctx, a, ctx.r2)


def mont_convert_out(ctx, a):
    return mont_mul(ctx, a, 1)


def word_pow(ctx, a, e):
    """a^e in Montgomery form (word_field.py:153-164)."""
    if e < 0:
        raise ValueError("exponent must be non-negative")
    acc, base = ctx.one_mont, a
    while e:
        if e & 1:
            acc = mont_mul(ctx, base, acc)
        base = mont_mul(ctx, base, base)
        e >>= 1
    return acc


def mont_inv(ctx, a):
    if a == 0:
        raise ZeroDivisionError("zero has no inverse")
    return word_pow(ctx, a, ctx.q - 2)


def word_primitive_root(ctx, n, seed=0):
    """Seeded primitive n-th root in Montgomery form (word_field.py:174-200):
    candidates from random.Random(seed), the first whose (q-1)/n-th power has
    order n -- the reference's root, bit for bit."""
    if n < 1 or n & (n - 1):
        raise ValueError("n must be a power of two")
    if (ctx.q - 1) % n:
        raise ValueError("n does not divide q - 1")
    if n == 1:
        return ctx.one_mont
    minus_one = mont_convert_in(ctx, ctx.q - 1)
    rng = random.Random(seed)
    e = (ctx.q - 1) // n
    while True:
        c = rng.randrange(1, ctx.q)
        g = word_pow(ctx, mont_convert_in(ctx, c), e)
        if word_pow(ctx, g, n // 2) == minus_one:
            return g


class MontField:
    """Field view of Z/qZ on Montgomery residues (fft.py:376-421).  Transforms
    built on it (build_plan) run on the GPU; the scalar methods keep the
    reference's protocol for callers that use them directly."""

    def __init__(self, ctx):
        self.ctx = ctx
        self._tables = {}

    def add(self, a, b):
        c = a + b
        return c - self.ctx.q if c >= self.ctx.q else c

    def sub(self, a, b):
        c = a - b
        return c + self.ctx.q if c < 0 else c

    def mul(self, a, b):
        return mont_mul(self.ctx, a, b)

    def pow(self, a, e):
        return word_pow(self.ctx, a, e)

    def zero(self):
        return 0

    def one(self):
        return self.ctx.one_mont

    def inv_scalar(self, n):
        return mont_inv(self.ctx, mont_convert_in(self.ctx, n % self.ctx.q))

    def root_power_mul_factory(self, omega, count):
        key = (omega, count)
        table = self._tables.get(key)
        if table is None:
            table = [self.one()]
            for _ in range(count - 1):
                table.append(self.mul(table[-1], omega))
            self._tables[key] = table
        ctx = self.ctx
        return lambda x, t: mont_mul(ctx, x, table[t])


class WordPlan:
    """Device plan: n-point transforms at omega over q (and the convolution
    weights when built for one).  Mirrors FftPlan's attributes for
    MontField plans (fft.py:199-234)."""

    def __init__(self, ctx, n, omega, negacyclic=False, theta=0, K=None, e=None):
        self.ctx = ctx
        self.field = MontField(ctx)
        self.N = self.n = n
        self.K, self.e = K, e
        self.omega = omega
        self.negacyclic = negacyclic
        h = ctypes.c_void_p()
        code = _lib.load().gfp_word_plan_create(ctypes.byref(h), ctx.q, n, omega,
                                                1 if negacyclic else 0, theta, _stream())
        if code == _lib.GFP_EINVAL:
            raise ValueError("omega is not a primitive N-th root")
        _lib.check(code, "gfp_word_plan_create")
        self._h = h.value
        self._inverse = None

    @property
    def handle(self):
        return ctypes.c_void_p(self._h)

    def inverse(self):
        """Plan at omega^-1 (fft.py:221-229)."""
        if self._inverse is None:
            self._inverse = WordPlan(self.ctx, self.n, word_pow(self.ctx, self.omega, self.n - 1),
                                     K=self.K, e=self.e)
        return self._inverse

    def n_inv(self):
        return self.field.inv_scalar(self.n)

    def __del__(self):
        try:
            if self._h:
                _lib.load().gfp_word_plan_destroy(ctypes.c_void_p(self._h))
        except Exception:
            pass


def build_word_plan(field, K, e, omega):
    """build_plan for a MontField (fft.py:237-275): K a base size, e >= 1,
    omega a primitive K^e-th root (checked on the device)."""
    if K not in BASE_SIZES:
        raise ValueError("unsupported base-case size")
    if e < 1:
        raise ValueError("e must be at least 1")
    N = K ** e
    if not 0 <= omega < field.ctx.q:
        raise ValueError("omega is not a primitive N-th root")
    return WordPlan(field.ctx, N, omega, K=K, e=e)


def _as_batch(x, n):
    if not isinstance(x, torch.Tensor) or x.device.type != "cuda" or x.dtype != torch.uint64:
        raise ValueError("expected a uint64 CUDA tensor (the package has no CPU path)")
    if not x.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if x.dim() == 1 and x.shape[0] == n:
        return x.unsqueeze(0), True
    if x.dim() == 2 and x.shape[1] == n:
        return x, False
    raise ValueError("expected [n] or [batch, n]")


def word_ntt(x, plan, inverse=False, out=None):
    """Batched DFT of Montgomery residues on the device ([n] or [B, n]
    uint64); inverse includes the 1/n scale (dft_inverse)."""
    xb, squeeze = _as_batch(x, plan.n)
    out = torch.empty_like(xb) if out is None else out.view_as(xb)
    _lib.check(_lib.load().gfp_word_ntt_exec(plan.handle, _ptr(xb), _ptr(out), xb.shape[0],
                                            1 if inverse else 0, _stream()), "gfp_word_ntt_exec")
    return out.squeeze(0) if squeeze else out


def word_convolve(x, y, plan, out=None):
    """Batched convolution of standard-form residues on the device with a
    convolution plan (conv_plan): cyclic or negacyclic per the plan."""
    xb, squeeze = _as_batch(x, plan.n)
    yb, _ = _as_batch(y, plan.n)
    if xb.shape != yb.shape:
        raise ValueError("shape mismatch")
    out = torch.empty_like(xb) if out is None else out.view_as(xb)
    code = _lib.load().gfp_word_convolve(plan.handle, _ptr(xb), _ptr(yb), _ptr(out), xb.shape[0],
                                         _stream())
    if code == _lib.GFP_EINVAL:
        raise ValueError("inputs must be reduced mod q")
    _lib.check(code, "gfp_word_convolve")
    return out.squeeze(0) if squeeze else out


_conv_plans = {}


def conv_plan(ctx, n, negacyclic):
    """The reference's _cyclic_plan / _nega_plan (gfp_mult.py:280-322): roots
    from word_primitive_root (n-th for cyclic, 2n-th theta with omega =
    theta^2 for negacyclic)."""
    key = (ctx.q, n, bool(negacyclic))
    plan = _conv_plans.get(key)
    if plan is not None:
        return plan
    if n < 1 or n & (n - 1):
        raise ValueError("%s must be a power of 2" % ("k" if negacyclic else "n"))
    if negacyclic:
        if (ctx.q - 1) % (2 * n):
            raise ValueError("unsupported size: 2k does not divide q - 1")
        theta = word_primitive_root(ctx, 2 * n)
        plan = WordPlan(ctx, n, mont_mul(ctx, theta, theta), negacyclic=True, theta=theta)
    else:
        if (ctx.q - 1) % n:
            raise ValueError("unsupported size: n does not divide q - 1")
        plan = WordPlan(ctx, n, word_primitive_root(ctx, n))
    _conv_plans[key] = plan
    return plan


def _check_reduced(v, n, q):
    if len(v) != n:
        raise ValueError("vector length mismatch")
    for d in v:
        if not 0 <= d < q:
            raise ValueError("inputs must be reduced mod q")


def _run_conv(x, y, ctx, n, negacyclic):
    plan = conv_plan(ctx, n, negacyclic)
    _check_reduced(x, n, ctx.q)
    _check_reduced(y, n, ctx.q)
    a = torch.from_numpy(np.asarray(x, dtype=np.uint64).copy()).cuda()
    b = torch.from_numpy(np.asarray(y, dtype=np.uint64).copy()).cuda()
    return tuple(int(v) for v in word_convolve(a, b, plan).cpu().numpy())


def negacyclic_convolution(x, y, ctx, k):
    """Coefficients of f_x f_y mod (X^k + 1) mod q (gfp_mult.py:369-378)."""
    return _run_conv(x, y, ctx, k, True)


def cyclic_convolution(f, g, ctx, n):
    """Coefficients of f g mod (X^n - 1) mod q (gfp_mult.py:381-386)."""
    return _run_conv(f, g, ctx, n, False)


def dft_word(v, plan, inverse=False):
    """The list API of dft_general / dft_inverse for MontField plans: v is a
    list of Montgomery residues, transformed in place and returned."""
    if len(v) != plan.n:
        raise ValueError("vector length must equal K^e")
    for d in v:
        if not 0 <= d < plan.ctx.q:
            raise ValueError("residues must be reduced mod q")
    x = torch.from_numpy(np.asarray(v, dtype=np.uint64).copy()).cuda()
    y = word_ntt(x, plan, inverse=inverse)
    v[:] = [int(d) for d in y.cpu().numpy()]
    return v
