"""Device vectors of GF(r^k + 1) elements: torch uint64 tensors, digit-major.

A vector of n elements is a contiguous CUDA tensor of shape [k, n] (a batch
of transforms: [batch, k, N]); digit d of element i is t[d, i].  torch is
only the allocator and stream provider here -- every operation is a kernel
of libgfpfft.so called through its C-ABI on the current torch stream.
"""

import ctypes

import numpy as np
import torch

from . import _lib


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _require_cuda(*ts):
    for t in ts:
        if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
            raise ValueError("expected a CUDA tensor (the package has no CPU path)")
        if t.dtype != torch.uint64:
            raise ValueError("expected a uint64 tensor")
        if not t.is_contiguous():
            raise ValueError("expected a contiguous tensor")


def empty(k, n, device="cuda"):
    return torch.empty((k, n), dtype=torch.uint64, device=device)


def to_device(elements, k, device="cuda"):
    """Element-major host data (list of k-tuples or [n, k] array) -> [k, n]."""
    arr = np.ascontiguousarray(np.asarray(elements, dtype=np.uint64).reshape(-1, k))
    host = torch.from_numpy(arr.T.copy())
    return host.to(device)


def to_host(t):
    """[k, n] device tensor -> element-major numpy array [n, k]."""
    return np.ascontiguousarray(t.cpu().numpy().T)


def to_tuples(t):
    return [tuple(int(d) for d in row) for row in to_host(t)]


def add(x, y, params):
    _require_cuda(x, y)
    z = torch.empty_like(x)
    k, n = x.shape
    _lib.check(_lib.load().gfp_vec_add(_ptr(x), _ptr(y), _ptr(z), n, k, params.r, _stream()),
               "gfp_vec_add")
    return z


def sub(x, y, params):
    _require_cuda(x, y)
    z = torch.empty_like(x)
    k, n = x.shape
    _lib.check(_lib.load().gfp_vec_sub(_ptr(x), _ptr(y), _ptr(z), n, k, params.r, _stream()),
               "gfp_vec_sub")
    return z


def mul_pow_r(x, i, params):
    _require_cuda(x)
    z = torch.empty_like(x)
    k, n = x.shape
    _lib.check(_lib.load().gfp_vec_mul_pow_r(_ptr(x), _ptr(z), n, k, params.r, int(i),
                                            _stream()), "gfp_vec_mul_pow_r")
    return z


def mul(x, y, params):
    """Element-wise product; y may be a single element [k, 1] (broadcast)."""
    _require_cuda(x, y)
    z = torch.empty_like(x)
    k, n = x.shape
    y_inc = 0 if y.shape[1] == 1 and n != 1 else 1
    if y_inc and y.shape != x.shape:
        raise ValueError("shape mismatch")
    _lib.check(_lib.load().gfp_vec_mul(_ptr(x), _ptr(y), y_inc, _ptr(z), n, k, params.r,
                                      _stream()), "gfp_vec_mul")
    return z


def mul_host(x, y, params, out=None):
    """Element-wise product of element-major host arrays [n, k] (uint64) ->
    [n, k] array (gfp_vec_mul_host: the whole H2D / multiply / D2H); `out`
    (e.g. a pinned buffer) receives the product when given."""
    import ctypes as C
    x = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
    y = np.ascontiguousarray(np.asarray(y, dtype=np.uint64))
    if x.shape != y.shape or x.ndim != 2 or x.shape[1] != params.k:
        raise ValueError("operands must be [n, k] arrays of the same shape")
    if out is None:
        z = np.empty_like(x)
    else:
        z = out
        if not (isinstance(z, np.ndarray) and z.dtype == np.uint64 and z.shape == x.shape
                and z.flags.c_contiguous):
            raise ValueError("out must be a C-contiguous uint64 array shaped like x")
    _lib.check(_lib.load().gfp_vec_mul_host(C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data),
                                           C.c_void_p(z.ctypes.data), x.shape[0], params.k,
                                           params.r, _stream()), "gfp_vec_mul_host")
    return z


def mul_crt(x, y, params):
    """Element-wise product through the reference's own mechanism (two word-
    prime negacyclic convolutions, CRT, LHC: gfp_mul_fft, gfp_mult.py:416-501);
    the same canonical result as mul().  ConfigurationError when
    check_prime_compat fails."""
    _require_cuda(x, y)
    z = torch.empty_like(x)
    k, n = x.shape
    y_inc = 0 if y.shape[1] == 1 and n != 1 else 1
    if y_inc and y.shape != x.shape:
        raise ValueError("shape mismatch")
    _lib.check(_lib.load().gfp_vec_mul_crt(_ptr(x), _ptr(y), y_inc, _ptr(z), n, k, params.r,
                                          _stream()), "gfp_vec_mul_crt")
    return z


MUL_STEPS = ("convert_in", "convolution", "convert_out", "crt", "lhc", "final")


def mul_crt_profile(x, y, params):
    """mul_crt through the instrumented kernel: (product, {step: SM cycles},
    device ms) with the reference's step keys (gfp_mult.py:428-500)."""
    _require_cuda(x, y)
    z = torch.empty_like(x)
    k, n = x.shape
    y_inc = 0 if y.shape[1] == 1 and n != 1 else 1
    if y_inc and y.shape != x.shape:
        raise ValueError("shape mismatch")
    cyc = (ctypes.c_uint64 * 6)()
    ms = ctypes.c_float(0.0)
    _lib.check(_lib.load().gfp_vec_mul_crt_profile(_ptr(x), _ptr(y), y_inc, _ptr(z), n, k,
                                                  params.r, cyc, ctypes.byref(ms), _stream()),
               "gfp_vec_mul_crt_profile")
    return z, dict(zip(MUL_STEPS, (int(c) for c in cyc))), float(ms.value)


def pow(x, e, params):
    """x^e for a non-negative Python int exponent shared by all elements."""
    _require_cuda(x)
    if e < 0:
        raise ValueError("exponent must be non-negative")
    limbs = []
    while e:
        limbs.append(e & ((1 << 64) - 1))
        e >>= 64
    arr = (ctypes.c_uint64 * max(1, len(limbs)))(*limbs)
    z = torch.empty_like(x)
    k, n = x.shape
    _lib.check(_lib.load().gfp_vec_pow(_ptr(x), arr, len(limbs), _ptr(z), n, k, params.r,
                                      _stream()), "gfp_vec_pow")
    return z


def is_canonical(x, params):
    _require_cuda(x)
    k, n = x.shape
    out = torch.empty(n, dtype=torch.uint8, device=x.device)
    _lib.check(_lib.load().gfp_vec_is_canonical(_ptr(x), _ptr(out), n, k, params.r, _stream()),
               "gfp_vec_is_canonical")
    return out.bool()


def uniform(n, params, seed, device="cuda", batch=None):
    """Seeded synthetic canonical elements (digits uniform in [0, r))."""
    shape = (params.k, n) if batch is None else (batch, params.k, n)
    z = torch.empty(shape, dtype=torch.uint64, device=device)
    total = n if batch is None else n * batch
    _lib.check(_lib.load().gfp_vec_uniform(_ptr(z), total, params.k, params.r, seed, _stream()),
               "gfp_vec_uniform")
    return z


def to_digit_major(elem_major, k):
    """Device element-major [n, k] -> digit-major [k, n]."""
    _require_cuda(elem_major)
    n = elem_major.numel() // k
    z = torch.empty((k, n), dtype=torch.uint64, device=elem_major.device)
    _lib.check(_lib.load().gfp_to_digit_major(_ptr(elem_major), _ptr(z), n, k, _stream()),
               "gfp_to_digit_major")
    return z


def to_element_major(x):
    _require_cuda(x)
    k, n = x.shape
    z = torch.empty((n, k), dtype=torch.uint64, device=x.device)
    _lib.check(_lib.load().gfp_to_element_major(_ptr(x), _ptr(z), n, k, _stream()),
               "gfp_to_element_major")
    return z
