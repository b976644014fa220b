"""ctypes wrapper over the CPU oracle (oracle/gfp_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference leg.  The product
package never imports this module.

Arrays here are element-major numpy uint64 of shape [n, k] (the reference's
tuple order).  The CUDA product uses digit-major [k, n]; tests transpose.
"""

import ctypes
import hashlib
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgfp_oracle.so")

DEFAULT_RADIX = {
    8: (1 << 59) + (1 << 16),
    16: (1 << 58) + (1 << 10),
    32: (1 << 56) + (1 << 21),
    64: 284903849103190610,
}

_u64p = ctypes.POINTER(ctypes.c_uint64)
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, u64, c_int = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        L.orc_random_elements.argtypes = [u64, c_int, u64, i64, i64, _u64p]
        L.orc_gfp_add.argtypes = [_u64p, _u64p, _u64p, i64, c_int, u64]
        L.orc_gfp_sub.argtypes = [_u64p, _u64p, _u64p, i64, c_int, u64]
        L.orc_gfp_mul_pow_r.argtypes = [_u64p, _u64p, i64, c_int, u64, c_int]
        L.orc_gfp_mul.argtypes = [_u64p, _u64p, _u64p, i64, c_int, u64, c_int, c_int]
        L.orc_check_prime_compat.argtypes = [c_int, u64]
        L.orc_base_case_ops.argtypes = [c_int, ctypes.POINTER(ctypes.c_int32), c_int]
        L.orc_gfp_root.argtypes = [c_int, u64, i64, _u64p, _u64p]
        L.orc_plan_create.argtypes = [c_int, u64, c_int, c_int, _u64p, c_int,
                                      ctypes.POINTER(c_int)]
        L.orc_plan_create.restype = ctypes.c_void_p
        L.orc_plan_destroy.argtypes = [ctypes.c_void_p]
        L.orc_plan_exec.argtypes = [ctypes.c_void_p, _u64p, c_int, c_int]
        L.orc_plan_prepare_inverse.argtypes = [ctypes.c_void_p]
        L.orc_poly_mul.argtypes = [ctypes.c_void_p, _u64p, _u64p, _u64p, c_int]
        L.orc_is_canonical.argtypes = [_u64p, i64, c_int, u64,
                                       ctypes.POINTER(ctypes.c_uint8)]
        L.orc_plan_table.argtypes = [ctypes.c_void_p, _u64p, i64]
        _lib = L
    return _lib


def _p(a):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


def _check(rc, what):
    if rc != 0:
        raise ValueError("oracle %s failed with code %d" % (what, rc))


def digest(arr):
    """sha256 prefix over element-major little-endian u64 digits."""
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()[:16]


def random_elements(seed, k, r, n, skip=0):
    """The reference input convention: Random(seed).randrange(p), encoded."""
    out = np.zeros((n, k), dtype=np.uint64)
    _check(lib().orc_random_elements(seed, k, r, skip, n, _p(out)), "random")
    return out


def add(x, y, r):
    z = np.empty_like(x)
    _check(lib().orc_gfp_add(_p(x), _p(y), _p(z), x.shape[0], x.shape[1], r), "add")
    return z


def sub(x, y, r):
    z = np.empty_like(x)
    _check(lib().orc_gfp_sub(_p(x), _p(y), _p(z), x.shape[0], x.shape[1], r), "sub")
    return z


def mul_pow_r(x, r, i):
    z = np.empty_like(x)
    _check(lib().orc_gfp_mul_pow_r(_p(x), _p(z), x.shape[0], x.shape[1], r, i), "shift")
    return z


def mul(x, y, r, backend="fft", threads=1):
    """backend 'fft' restates gfp_mul_fft (paper Alg. 13); 'school' is an
    independent schoolbook second opinion."""
    z = np.empty_like(x)
    b = 0 if backend == "fft" else 1
    _check(lib().orc_gfp_mul(_p(x), _p(y), _p(z), x.shape[0], x.shape[1], r, b,
                             threads), "mul")
    return z


def check_prime_compat(k, r):
    return bool(lib().orc_check_prime_compat(k, r))


def base_case_ops(K):
    buf = (ctypes.c_int32 * (3 * 4096))()
    n = lib().orc_base_case_ops(K, buf, 3 * 4096)
    if n < 0:
        raise ValueError("unsupported base-case size")
    kinds = ("dft2", "tw", "swap")
    return tuple((kinds[buf[3 * i]], buf[3 * i + 1], buf[3 * i + 2]) for i in range(n))


def gfp_root(k, r, N):
    """(g, omega) of bench_cli._gfp_root (seed 0 root search + Alg. 1 lift)."""
    g = np.zeros((1, k), dtype=np.uint64)
    w = np.zeros((1, k), dtype=np.uint64)
    _check(lib().orc_gfp_root(k, r, N, _p(g), _p(w)), "root")
    return g[0], w[0]


def is_canonical(x, r):
    out = np.zeros(x.shape[0], dtype=np.uint8)
    lib().orc_is_canonical(_p(x), x.shape[0], x.shape[1], r,
                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    return out.astype(bool)


class Plan:
    """build_plan / dft_general / dft_inverse restated (fft.py:199-370)."""

    def __init__(self, k, r, K, e, omega, backend="fft"):
        self.k, self.r, self.K, self.e = k, r, K, e
        self.N = K ** e
        err = ctypes.c_int(0)
        om = np.ascontiguousarray(np.asarray(omega, dtype=np.uint64).reshape(1, k))
        b = 0 if backend == "fft" else 1
        self._h = lib().orc_plan_create(k, r, K, e, _p(om), b, ctypes.byref(err))
        if not self._h:
            raise ValueError("oracle build_plan rejected the parameters (code %d)"
                             % err.value)

    def table(self, n=None):
        """omega^j for j < n <= N/K (FftPlan.twiddle_table, fft.py:211-214)."""
        n = self.N // self.K if n is None else n
        out = np.zeros((n, self.k), dtype=np.uint64)
        _check(lib().orc_plan_table(self._h, _p(out), n), "plan table")
        return out

    def prepare_inverse(self):
        _check(lib().orc_plan_prepare_inverse(self._h), "inverse plan")

    def forward(self, v, threads=1):
        v = np.ascontiguousarray(v, dtype=np.uint64).copy()
        _check(lib().orc_plan_exec(self._h, _p(v), 0, threads), "dft_general")
        return v

    def inverse(self, v, threads=1):
        v = np.ascontiguousarray(v, dtype=np.uint64).copy()
        _check(lib().orc_plan_exec(self._h, _p(v), 1, threads), "dft_inverse")
        return v

    def poly_mul(self, f, g, threads=1):
        f = np.ascontiguousarray(f, dtype=np.uint64)
        g = np.ascontiguousarray(g, dtype=np.uint64)
        out = np.empty_like(f)
        _check(lib().orc_poly_mul(self._h, _p(f), _p(g), _p(out), threads), "poly_mul")
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_plan_destroy(self._h)
            self._h = None
