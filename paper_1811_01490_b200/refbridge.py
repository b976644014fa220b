"""The reference package's own CLI on the GPU path: a `gfp-cuda` backend for
gfpfft.bench_cli (the binding INTEGRATION.md section 2 describes, made real).

    import gfpfft.bench_cli as bench_cli
    from paper_1811_01490_b200 import refbridge
    refbridge.install(bench_cli)
    bench_cli.main(["bench-fft", "--K", "16", "--e", "3"])   # all backends, cross-checked

install() registers "gfp-cuda" in BACKENDS (bench_cli.py:43) and wraps two
module functions the reference's bench-fft calls by name:

  _fft_bench_setup (bench_cli.py:369-395)  for backend "gfp-cuda": the same
      radix / primality gate, the reference's own root routine _gfp_root
      (bench_cli.py:398-402) for omega, the same Random(seed).randrange(p)
      -> gfp_encode input convention; the plan and field are this package's
      (device twiddle tables, device multiply);
  dft_general (imported into bench_cli from fft.py:298-360)  plans of this
      package run on the GPU (fft.dft_general, profile keys permutation /
      basecase / twiddle as the reference's), any other plan goes to the
      reference's own function unchanged.

cmd_bench_fft then cross-checks the gfp-cuda digest against gfp-fft,
gfp-bigint and oracle-bigint before timing (bench_cli.py:437-448), exactly as
it does among its own backends.  Nothing else in the reference changes.
"""

import random

from . import fft as F
from .gfp_field import GfpParams
from .gfp_mult import GfpFftField

BACKEND = "gfp-cuda"


def install(bench_cli):
    """Register the gfp-cuda backend in the given gfpfft.bench_cli module
    (idempotent); returns the module."""
    if BACKEND in bench_cli.BACKENDS and getattr(bench_cli._fft_bench_setup, "_gfp_cuda", False):
        return bench_cli
    ref_setup = bench_cli._fft_bench_setup
    ref_dft = bench_cli.dft_general

    def setup(K, e, backend, r, threads, seed):
        if backend != BACKEND:
            return ref_setup(K, e, backend, r, threads, seed)
        k = K // 2
        if r is None:
            r = bench_cli.DEFAULT_RADIX.get(k)
            if r is None:
                raise ValueError("no default radix for K=%d, pass --r" % K)
        ref_params = bench_cli.GfpParams(r, k)
        if not bench_cli.oracle.oracle_is_probable_prime(ref_params.p, 40):
            raise ValueError("r^%d+1 is not prime for r=%d, transforms need a prime modulus"
                             % (k, r))
        N = K ** e
        omega = bench_cli._gfp_root(ref_params, N)
        field = GfpFftField(GfpParams(r, k), backend="cuda")
        plan = F.build_plan(field, K, e, omega, threads=threads)
        rng = random.Random(seed)

        def make():
            return [bench_cli.gfp_encode(ref_params, rng.randrange(ref_params.p))
                    for _ in range(N)]

        return field, plan, make, lambda v: bench_cli.gfp_decode(ref_params, v)

    def dft_general(v, plan, field, profile=None):
        if isinstance(plan, F.FftPlan):
            return F.dft_general(v, plan, field, profile=profile)
        return ref_dft(v, plan, field, profile=profile)

    setup._gfp_cuda = True
    if BACKEND not in bench_cli.BACKENDS:
        bench_cli.BACKENDS = tuple(bench_cli.BACKENDS) + (BACKEND,)
    bench_cli._fft_bench_setup = setup
    bench_cli.dft_general = dft_general
    return bench_cli
