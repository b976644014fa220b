"""The reference's profile= contracts on the GPU path: dft_general's phase
keys (fft.py:298-360; pinned by the reference's tests/test_fft.py:276-282),
gfp_mul_fft's step keys (gfp_mult.py:428-500; tests/test_gfp_mult.py:295-306),
the profile-mul CSV (bench_cli.py:470-494), and the per-pass timing and
capability queries behind them."""
import csv
import io
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

R8 = (1 << 59) + (1 << 16)
R16 = (1 << 58) + (1 << 10)


def _gp():
    import paper_1811_01490_b200 as gp
    return gp


def test_dft_general_profile_keys(cuda):
    gp = _gp()
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    plan = gp.build_plan(field, 16, 3, gp.roots_for(params, 4096))
    rng = random.Random(1)
    v = [gp.gfp_encode(params, rng.randrange(params.p)) for _ in range(4096)]
    want = gp.dft_general(list(v), plan, field)
    profile = {}
    got = gp.dft_general(list(v), plan, field, profile=profile)
    assert got == want
    assert set(profile) == {"permutation", "basecase", "twiddle"}
    assert all(t >= 0 for t in profile.values())
    assert profile["basecase"] > 0 and profile["twiddle"] > 0
    gp.dft_inverse(got, plan, field, profile=profile)
    assert got == v and set(profile) == {"permutation", "basecase", "twiddle"}


@pytest.mark.parametrize("k,r", [(8, R8), (16, R16), (32, (1 << 56) + (1 << 21))])
def test_mul_fft_profile_steps(k, r, cuda):
    gp = _gp()
    params = gp.GfpParams(r, k)
    crt = gp.crt_default()
    rng = random.Random(5)
    profile = {}
    for _ in range(3):
        a, b = rng.randrange(params.p), rng.randrange(params.p)
        z = gp.gfp_mul_fft(params, crt, gp.gfp_encode(params, a), gp.gfp_encode(params, b),
                           profile=profile)
        assert gp.gfp_decode(params, z) == a * b % params.p
    assert set(profile) == {"convert_in", "convolution", "convert_out", "crt", "lhc", "final"}
    assert all(t >= 0 for t in profile.values()) and sum(profile.values()) > 0


def test_mul_crt_profile_cycles_and_product(cuda):
    gp = _gp()
    from oracle import oracle as O
    params = gp.GfpParams(R8, 8)
    x = O.random_elements(3, 8, R8, 5000)
    y = O.random_elements(4, 8, R8, 5000)
    z, cycles, ms = gp.vec.mul_crt_profile(gp.vec.to_device(x, 8), gp.vec.to_device(y, 8),
                                           params)
    assert np.array_equal(gp.vec.to_host(z), O.mul(x, y, R8))
    assert set(cycles) == set(gp.vec.MUL_STEPS) and all(c > 0 for c in cycles.values())
    assert ms > 0


def test_profile_mul_cli(cuda):
    from paper_1811_01490_b200 import cli
    out = io.StringIO()
    args = cli.build_parser().parse_args(["profile-mul", "--k", "8,16,32", "--trials", "64"])
    assert cli.cmd_profile_mul(args, out) == 0
    rows = list(csv.reader(io.StringIO(out.getvalue())))
    assert rows[0] == ["k", "r", "convert_in_pct", "convolution_pct", "convert_out_pct",
                       "crt_pct", "lhc_pct", "final_pct"]
    assert [int(r[0]) for r in rows[1:]] == [8, 16, 32]
    for row in rows[1:]:
        pct = [float(c) for c in row[2:]]
        assert abs(sum(pct) - 100.0) < 0.1 and all(p >= 0 for p in pct)
    # the reference's exit-code contract for an incompatible radix
    assert cli.main(["profile-mul", "--k", "8", "--r", "2^63+2^34"]) == 2


def test_pass_times_and_caps(cuda):
    gp = _gp()
    from paper_1811_01490_b200 import _lib, fft as F
    lib = _lib.load()
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    plan = gp.build_plan(field, 16, 4, gp.roots_for(params, 1 << 16))
    assert lib.gfp_fft_plan_caps(plan.handle) == 7
    x = gp.vec.uniform(1 << 16, params, seed=1)
    y, passes = F.pass_times(plan, lambda: gp.fft_tensor(x, plan))
    assert [i for i, _ in passes] == [0, 1, 2, 3] and all(ms > 0 for _, ms in passes)
    _, passes = F.pass_times(plan, lambda: gp.poly_mul(x, x, plan))
    # forward passes 0-2 (both operands), the fused forward-last + pointwise
    # + inverse-first kernel (marked with the forward pass index 3), inverse
    # passes 1-3
    assert [i for i, _ in passes] == [0, 1, 2, 3, 1, 2, 3]
    # timing off again: no marks recorded
    gp.fft_tensor(x, plan)
    assert lib.gfp_fft_plan_pass_times(plan.handle, None, None, 0) == 0
    p16 = gp.GfpParams(R16, 16)
    f16 = gp.GfpFftField(p16, backend="cuda")
    plan16 = gp.build_plan(f16, 32, 2, gp.roots_for(p16, 1024))
    assert lib.gfp_fft_plan_caps(plan16.handle) == 0
    one = gp.build_plan(field, 16, 1, gp.roots_for(params, 16))
    assert lib.gfp_fft_plan_caps(one.handle) == _lib.GFP_CAP_EM_IO
