"""General GF(r^k + 1) multiplication and the GFP field adapter.

Mirrors gfpfft/gfp_mult.py's public surface for the hot path:

  gfp_mul_fft / gfp_mul_bigint (gfp_mult.py:416-512)  -> one device multiply
      (exact; limb-split IMAD.WIDE negacyclic convolution plus reduction mod
      r^k + 1 -- see csrc/gfp_fast.cuh and csrc/gfp_generic.cuh).
      gfp_mul_fft keeps the reference's ConfigurationError contract from
      check_prime_compat (gfp_mult.py:207-226, 395-402).
  GfpFftField (gfp_mult.py:518-592)                   -> the field protocol
      object the transform consumes; every method runs on the device.

The reference's CPU mechanism for the multiply (word-prime NTTs, CRT, LHC,
word_field Montgomery arithmetic) is not the product's mechanism; only the
configuration contract is kept (CrtParams / crt_default hold the prime pair
for check_prime_compat).
"""

from dataclasses import dataclass
from functools import lru_cache
from typing import NamedTuple

from . import _lib, vec
from .gfp_field import (GfpParams, gfp_encode, gfp_mul_pow_r, gfp_one, gfp_zero)

P1 = 4179340454199820289
P2 = 2485986994308513793


class ConfigurationError(ValueError):
    """A (field, prime pair) combination cannot be used (gfp_mult.py:35)."""


@dataclass(frozen=True)
class CrtParams:
    """The word-prime pair of the reference's FFT multiplier (gfp_mult.py:131-167)."""

    p1: int = P1
    p2: int = P2

    @property
    def p1_ctx(self):
        from .word import word_prime
        return word_prime(self.p1)

    @property
    def p2_ctx(self):
        from .word import word_prime
        return word_prime(self.p2)

    @classmethod
    def make(cls, q1=P1, q2=P2):
        from math import gcd
        if gcd(q1, q2) != 1:
            raise ValueError("primes must be coprime")
        return cls(q1, q2)


@lru_cache(maxsize=None)
def crt_default():
    return CrtParams()


class CompatReport(NamedTuple):
    passed: bool
    slack: int
    reasons: tuple


def check_prime_compat(params, crt):
    """k r^2 <= (p1 p2 - 1)/2 and 2k | p_i - 1 (gfp_mult.py:207-226)."""
    q1, q2 = crt.p1, crt.p2
    bound = params.k * params.r * params.r
    limit = (q1 * q2 - 1) // 2
    reasons = []
    if bound > limit:
        reasons.append("coefficient bound k*r^2 = %d exceeds usable range %d" % (bound, limit))
    two_k = 2 * params.k
    if (q1 - 1) % two_k:
        reasons.append("2k = %d does not divide p1 - 1" % two_k)
    if (q2 - 1) % two_k:
        reasons.append("2k = %d does not divide p2 - 1" % two_k)
    return CompatReport(not reasons, limit - bound, tuple(reasons))


_compat_ok = {}


def _require_compat(params, crt):
    key = (params.r, params.k, crt.p1, crt.p2)
    if _compat_ok.get(key):
        return
    report = check_prime_compat(params, crt)
    if not report.passed:
        raise ConfigurationError("; ".join(report.reasons))
    _compat_ok[key] = True


def add_step_profile(profile, cycles, seconds):
    """Accumulate `seconds` of device time into profile under the reference's
    step keys (gfp_mult.py:428-500), split by the measured per-step cycle
    shares of the instrumented mechanism kernel."""
    total = sum(cycles.values())
    for step in vec.MUL_STEPS:
        share = cycles[step] / total if total else 1.0 / len(vec.MUL_STEPS)
        profile[step] = profile.get(step, 0.0) + seconds * share


def _mul_device(params, x, y, profile=None, mechanism=False):
    if len(x) != params.k or len(y) != params.k:
        raise ValueError("element must have k digits")
    if profile is None and params.k <= 128:  # one staged call (gfp_scalar_op)
        from .gfp_field import OP_MUL, OP_MUL_CRT, scalar_op
        return scalar_op(OP_MUL_CRT if mechanism and params.k <= 64 else OP_MUL, params, x, y)
    a = vec.to_device([x], params.k)
    b = vec.to_device([y], params.k)
    # mechanism: the reference's two-prime convolution + CRT + LHC route
    # (gfp_vec_mul_crt); else the direct exact multiply the transforms use
    if mechanism and params.k <= 64:
        if profile is not None:
            # the instrumented mechanism kernel: per-step cycles, device time
            z, cycles, ms = vec.mul_crt_profile(a, b, params)
            add_step_profile(profile, cycles, ms * 1e-3)
        else:
            z = vec.mul_crt(a, b, params)
    else:
        z = vec.mul(a, b, params)
    return vec.to_tuples(z)[0]


def gfp_mul_fft(params, crt, x, y, profile=None):
    """x * y mod p through the reference's mechanism on the device; raises
    ConfigurationError like the reference when the prime pair cannot carry
    k r^2 (gfp_mult.py:416-422).  profile, when given, accumulates seconds
    under the reference's keys convert_in, convolution, convert_out, crt,
    lhc, final: the device time of the instrumented kernel split by its
    per-step cycle counts."""
    _require_compat(params, crt)
    return _mul_device(params, x, y, profile, mechanism=True)


def gfp_mul_bigint(params, x, y):
    """x * y mod p (gfp_mult.py:504-512)."""
    return _mul_device(params, x, y)


def gfp_mul_vec(params, x, y):
    """Batched product of device vectors [k, n] (the C5 multiply path)."""
    return vec.mul(x, y, params)


class GfpFftField:
    """The field protocol object for GF(r^k + 1) (gfp_mult.py:518-592).

    backend "fft" (default) keeps the reference's compat gate; "bigint" and
    "cuda" skip it.  All three compute on the device with the same exact
    multiply.  Transforms built on this field run entirely on the GPU
    (fft.build_plan).
    """

    def __init__(self, params, crt=None, backend="fft"):
        if backend not in ("fft", "bigint", "cuda"):
            raise ValueError("unknown backend")
        if backend == "fft":
            crt = crt if crt is not None else crt_default()
            _require_compat(params, crt)
        self.params = params
        self.crt = crt
        self.backend = backend
        self.two_k = 2 * params.k
        self.shift_root = gfp_encode(params, params.r)
        # r^(2k-1) = 1/r, the root inverse transforms align with
        self.shift_root_inv = self.shift(self.one(), self.two_k - 1)
        self._tables = {}

    def add(self, a, b):
        from .gfp_field import gfp_add
        return gfp_add(self.params, a, b)

    def sub(self, a, b):
        from .gfp_field import gfp_sub
        return gfp_sub(self.params, a, b)

    def mul(self, a, b):
        return _mul_device(self.params, a, b)

    def pow(self, a, e):
        from .gfp_field import gfp_pow
        if e < 0:
            raise ValueError("exponent must be non-negative")
        return gfp_pow(self.params, a, e)

    def zero(self):
        return gfp_zero(self.params)

    def one(self):
        return gfp_one(self.params)

    def inv_scalar(self, n):
        return gfp_encode(self.params, pow(n, -1, self.params.p))

    def shift(self, a, i):
        return gfp_mul_pow_r(self.params, a, i)

    def root_power_mul_factory(self, omega, count):
        """x * omega^t for t < count (gfp_mult.py:574-592)."""
        if omega == self.shift_root and count <= self.two_k:
            params = self.params
            return lambda a, t: gfp_mul_pow_r(params, a, t)
        if omega == self.shift_root_inv and count <= self.two_k:
            params = self.params
            two_k = self.two_k
            return lambda a, t: gfp_mul_pow_r(params, a, (two_k - t) % two_k)
        table = self._tables.get((omega, count))
        if table is None:
            table = [self.one()]
            for _ in range(count - 1):
                table.append(self.mul(table[-1], omega))
            self._tables[(omega, count)] = table

        def mul_pow(a, t):
            return self.mul(a, table[t])

        return mul_pow


__all__ = ["ConfigurationError", "CrtParams", "crt_default", "CompatReport",
           "check_prime_compat", "gfp_mul_fft", "gfp_mul_bigint", "gfp_mul_vec",
           "GfpFftField", "GfpParams", "P1", "P2"]

# the library must be loadable for this module to be usable at all
_lib.load()
