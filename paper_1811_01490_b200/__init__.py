"""B200-native GF(r^k + 1) FFT and polynomial multiply (arXiv:1811.01490 path).

Drop-in for the hot path of the reference package `gfpfft`: the public names
below mirror gfpfft/__init__.py:9-38 for GFP element arithmetic, general
multiply and the transforms.  Every arithmetic operation is a CUDA kernel of
libgfpfft.so (sm_100a); there is no CPU fallback, and importing fails loudly
when the library has not been built.

Device-scale API: `vec` (digit-major uint64 tensors), `fft.fft`,
`fft.poly_mul`, `fft.fft_host` / `fft.poly_mul_host` (host buffers).
"""

from . import _lib

_lib.load()

from .gfp_field import (GfpParams, element_from_text, element_to_text,  # noqa: E402
                        gfp_add, gfp_decode, gfp_encode, gfp_find_nth_root,
                        gfp_mul_pow_r, gfp_one, gfp_pow, gfp_primitive_root, gfp_sub,
                        gfp_zero, is_canonical)
from .gfp_mult import (P1, P2, CompatReport, ConfigurationError,  # noqa: E402
                       CrtParams, GfpFftField, check_prime_compat, crt_default,
                       gfp_mul_bigint, gfp_mul_fft, gfp_mul_vec)
from .fft import (BASE_SIZES, FftPlan, build_plan, dft_base, dft_general,  # noqa: E402
                  dft_inverse, fft as fft_tensor, fft_host, poly_mul, poly_mul_host,
                  poly_mul_list, roots_for, stride_permutation, twiddle_apply)
from . import vec  # noqa: E402
from .word import (MontField, WordPlan, WordPrime, conv_plan,  # noqa: E402
                   cyclic_convolution, mont_convert_in, mont_convert_out, mont_inv, mont_mul,
                   negacyclic_convolution, word_convolve, word_ntt, word_pow, word_prime,
                   word_primitive_root)

DEFAULT_RADIX = {
    8: (1 << 59) + (1 << 16),
    16: (1 << 58) + (1 << 10),
    32: (1 << 56) + (1 << 21),
    64: 284903849103190610,
}

__version__ = "0.1.0"

__all__ = [
    "GfpParams", "gfp_add", "gfp_sub", "gfp_mul_pow_r", "gfp_pow",
    "gfp_encode", "gfp_decode", "gfp_primitive_root", "gfp_find_nth_root",
    "gfp_zero", "gfp_one", "is_canonical", "element_to_text", "element_from_text",
    "ConfigurationError", "CrtParams", "CompatReport", "GfpFftField",
    "check_prime_compat", "crt_default", "gfp_mul_bigint", "gfp_mul_fft", "gfp_mul_vec",
    "P1", "P2", "BASE_SIZES", "FftPlan", "build_plan", "dft_base", "dft_general",
    "dft_inverse", "stride_permutation", "twiddle_apply", "fft_tensor", "fft_host",
    "poly_mul", "poly_mul_host", "poly_mul_list", "roots_for", "vec", "DEFAULT_RADIX",
    "MontField", "WordPlan", "WordPrime", "conv_plan", "cyclic_convolution",
    "negacyclic_convolution", "mont_convert_in", "mont_convert_out", "mont_inv", "mont_mul",
    "word_convolve", "word_ntt", "word_pow", "word_prime", "word_primitive_root",
    "__version__",
]
