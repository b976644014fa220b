"""ctypes binding of libgfpfft.so (the C-ABI declared in include/gfpfft.h).

The CUDA library is the only compute path of this package: there is no CPU
fallback.  If the shared object is missing the import fails loudly; if no
GPU is present, every compute call raises RuntimeError from the CUDA error
code it returns.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GFPFFT_LIB", os.path.join(HERE, "libgfpfft.so"))

GFP_OK = 0
GFP_EINVAL = 1
GFP_ECONFIG = 2
GFP_ECUDA = 3
GFP_ENOMEM = 4
GFP_EUNSUPPORTED = 5
GFP_CAP_EM_IO = 1
GFP_CAP_FT = 2
GFP_CAP_XCH = 4

# every symbol include/gfpfft.h declares: (name, restype, argtypes)
_u64p = ctypes.c_void_p  # device or host pointers are passed as integers
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_vp = ctypes.c_void_p

SIGNATURES = {
    "gfp_strerror": (ctypes.c_char_p, [_int]),
    "gfp_version": (_int, []),
    "gfp_check_prime_compat": (_int, [_int, _u64]),
    "gfp_fast_path_ok": (_int, [_int, _u64]),
    "gfp_vec_add": (_int, [_u64p, _u64p, _u64p, _i64, _int, _u64, _vp]),
    "gfp_vec_sub": (_int, [_u64p, _u64p, _u64p, _i64, _int, _u64, _vp]),
    "gfp_vec_mul_pow_r": (_int, [_u64p, _u64p, _i64, _int, _u64, _int, _vp]),
    "gfp_vec_mul": (_int, [_u64p, _u64p, _i64, _u64p, _i64, _int, _u64, _vp]),
    "gfp_scalar_op": (_int, [_int, ctypes.POINTER(ctypes.c_uint64),
                             ctypes.POINTER(ctypes.c_uint64), _i64,
                             ctypes.POINTER(ctypes.c_uint64), _int, _u64, _vp]),
    "gfp_vec_mul_host": (_int, [_u64p, _u64p, _u64p, _i64, _int, _u64, _vp]),
    "gfp_vec_mul_crt": (_int, [_u64p, _u64p, _i64, _u64p, _i64, _int, _u64, _vp]),
    "gfp_vec_mul_crt_profile": (_int, [_u64p, _u64p, _i64, _u64p, _i64, _int, _u64,
                                       ctypes.POINTER(ctypes.c_uint64),
                                       ctypes.POINTER(ctypes.c_float), _vp]),
    "gfp_vec_pow": (_int, [_u64p, ctypes.POINTER(ctypes.c_uint64), _int, _u64p, _i64, _int,
                           _u64, _vp]),
    "gfp_vec_is_canonical": (_int, [_u64p, _vp, _i64, _int, _u64, _vp]),
    "gfp_vec_uniform": (_int, [_u64p, _i64, _int, _u64, _u64, _vp]),
    "gfp_to_digit_major": (_int, [_u64p, _u64p, _i64, _int, _vp]),
    "gfp_to_element_major": (_int, [_u64p, _u64p, _i64, _int, _vp]),
    "gfp_word_consts": (_int, [_u64, ctypes.POINTER(ctypes.c_uint64),
                               ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]),
    "gfp_word_vec_mont_mul": (_int, [_u64, _u64p, _u64p, _u64p, _i64, _vp]),
    "gfp_word_plan_create": (_int, [ctypes.POINTER(_vp), _u64, _i64, _u64, _int, _u64, _vp]),
    "gfp_word_plan_destroy": (_int, [_vp]),
    "gfp_word_ntt_exec": (_int, [_vp, _u64p, _u64p, _i64, _int, _vp]),
    "gfp_word_convolve": (_int, [_vp, _u64p, _u64p, _u64p, _i64, _vp]),
    "gfp_fft_plan_create": (_int, [ctypes.POINTER(_vp), _int, _u64, _int, _int,
                                   ctypes.POINTER(ctypes.c_uint64), _vp]),
    "gfp_fft_plan_destroy": (_int, [_vp]),
    "gfp_fft_plan_size": (_i64, [_vp]),
    "gfp_fft_workspace_words": (_i64, [_vp, _i64]),
    "gfp_fft_exec": (_int, [_vp, _u64p, _u64p, _u64p, _i64, _int, _vp]),
    "gfp_fft_exec_ex": (_int, [_vp, _u64p, _u64p, _u64p, _i64, _int, _int, _int, _vp, _i64,
                               _int, _vp]),
    "gfp_poly_mul": (_int, [_vp, _u64p, _u64p, _u64p, _u64p, _i64, _vp]),
    "gfp_fft_exec_host": (_int, [_vp, _u64p, _i64, _int, _vp]),
    "gfp_poly_mul_host": (_int, [_vp, _u64p, _u64p, _u64p, _i64, _vp]),
    "gfp_poly_mul_host2": (_int, [_vp, _u64p, _i64, _u64p, _i64, _u64p, _i64, _vp]),
    "gfp_fft_plan_last_launches": (_i64, [_vp]),
    "gfp_fft_plan_caps": (_int, [_vp]),
    "gfp_fft_plan_set_timing": (_int, [_vp, _int]),
    "gfp_fft_plan_pass_times": (_int, [_vp, ctypes.POINTER(ctypes.c_float),
                                       ctypes.POINTER(ctypes.c_int), _int]),
    "gfp_fft_twiddle": (_int, [_vp, _u64p, _u64p, _i64, _i64, _i64, _int, _vp]),
    "gfp_exchange_transpose": (_int, [_u64p, ctypes.POINTER(ctypes.c_uint64), _int, _int, _i64,
                                      _int, _i64, _vp]),
    "gfp_fft_exec_exchange": (_int, [_vp, _u64p, _u64p, _u64p, _i64, _int, _int, _int,
                                     ctypes.POINTER(ctypes.c_uint64), _int, _int, _vp]),
    "gfp_flag_signal": (_int, [ctypes.POINTER(ctypes.c_uint64), _int, _int, _int, _u64, _vp]),
    "gfp_flag_wait": (_int, [_u64p, _int, _int, _u64, _i64, _vp, _vp]),
    "gfp_ipc_get_handle": (_int, [_vp, ctypes.c_char_p, ctypes.POINTER(_i64)]),
    "gfp_ipc_open": (_int, [ctypes.c_char_p, _i64, ctypes.POINTER(_vp)]),
    "gfp_ipc_close": (_int, [_vp, _i64]),
    "gfp_radix_mode": (_int, [_int, _u64]),
    "gfp_tma_pass_launches": (_i64, []),
    "gfp_debug_build": (_int, []),
    "gfp_debug_selftest": (_int, [_vp]),
    "gfp_probe_imad_wide": (_int, [_i64, _int, _int, ctypes.POINTER(ctypes.c_float),
                                   ctypes.POINTER(ctypes.c_double), _vp]),
}


class GfpError(RuntimeError):
    pass


_lib = None


def load():
    """Load libgfpfft.so (raises ImportError when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            "libgfpfft.so not found at %s: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
            % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(code, what=""):
    """Map a C return code to the reference's exception types."""
    if code == GFP_OK:
        return
    msg = load().gfp_strerror(code).decode()
    if what:
        msg = "%s: %s" % (what, msg)
    if code == GFP_EINVAL:
        raise ValueError(msg)
    if code == GFP_ECONFIG:
        from .gfp_mult import ConfigurationError
        raise ConfigurationError(msg)
    if code == GFP_EUNSUPPORTED:
        raise ValueError(msg)
    raise GfpError(msg)
