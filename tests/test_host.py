"""Host-side logic of the package (no GPU): parameter validation, encode /
decode, canonical checks, list utilities, compat reports."""
import random

import pytest

import paper_1811_01490_b200 as gp

R8 = (1 << 59) + (1 << 16)


def test_params_validation():
    # tests/test_gfp_field.py:38-50
    with pytest.raises(ValueError):
        gp.GfpParams(10, 3)
    with pytest.raises(ValueError):
        gp.GfpParams(10, 0)
    with pytest.raises(ValueError):
        gp.GfpParams(1, 8)
    with pytest.raises(ValueError):
        gp.GfpParams(1 << 64, 8)
    assert gp.GfpParams(10, 4).p == 10 ** 4 + 1


@pytest.mark.parametrize("k,r", [(8, R8), (16, (1 << 58) + (1 << 10)), (1, 4), (2, 6),
                                 (4, 10), (8, 2)])
def test_encode_decode_bijection(k, r):
    params = gp.GfpParams(r, k)
    rng = random.Random(7)
    vals = [0, 1, r - 1, r, params.p - 2, params.p - 1] + \
        [rng.randrange(params.p) for _ in range(200)]
    for v in vals:
        v %= params.p
        x = gp.gfp_encode(params, v)
        assert gp.is_canonical(params, x)
        assert gp.gfp_decode(params, x) == v
    assert gp.gfp_encode(params, params.p - 1) == (0,) * (k - 1) + (r,)


def test_canonical_rejects():
    params = gp.GfpParams(10, 4)
    assert not gp.is_canonical(params, (10, 0, 0, 0))
    assert not gp.is_canonical(params, (1, 0, 0, 10))
    assert not gp.is_canonical(params, (0, 0, 0))
    with pytest.raises(ValueError):
        gp.gfp_decode(params, (0, 11, 0, 0))


def test_text_roundtrip():
    params = gp.GfpParams(R8, 8)
    x = gp.gfp_encode(params, 123456789 ** 5)
    assert gp.element_from_text(params, gp.element_to_text(x)) == x
    with pytest.raises(ValueError):
        gp.element_from_text(params, "1,2")


def test_stride_permutation_example():
    # tests/test_fft.py:56-58
    assert gp.stride_permutation(list(range(8)), 2, 4) == [0, 2, 4, 6, 1, 3, 5, 7]
    v = list(range(24))
    gp.stride_permutation(v, 3, 4)
    gp.stride_permutation(v, 4, 3)
    assert v == list(range(24))


def test_compat_report():
    params = gp.GfpParams((1 << 63) + (1 << 34), 8)
    rep = gp.check_prime_compat(params, gp.crt_default())
    assert not rep.passed and rep.slack < 0
    ok = gp.check_prime_compat(gp.GfpParams(R8, 8), gp.crt_default())
    assert ok.passed and ok.slack > 0


def test_oracle_element_ops_property():
    # the CPU oracle's digit algorithms (gfp_field.py:82-161, gfp_mult.py)
    # against plain integer arithmetic mod p for random (k, r) and operands
    # (form B, zero and r - 1 digits included); the oracle is the checker of
    # every GPU parity test, so it is itself checked here beyond the goldens
    import numpy as np
    from oracle import oracle as O
    rng = random.Random(20261020)
    for _ in range(40):
        k = rng.choice([1, 2, 4, 8, 16, 32])
        r = rng.choice([2, 3, rng.randrange(2, 1 << 16), rng.randrange(1 << 40, 1 << 62),
                        rng.randrange(1 << 62, 1 << 64)])
        params = gp.GfpParams(r, k)
        p = params.p
        vals = [0, 1, p - 1, p - 2, r, r - 1] + [rng.randrange(p) for _ in range(10)]
        xs = [rng.choice(vals) for _ in range(24)]
        ys = [rng.choice(vals) for _ in range(24)]
        X = np.array([gp.gfp_encode(params, v) for v in xs], dtype=np.uint64)
        Y = np.array([gp.gfp_encode(params, v) for v in ys], dtype=np.uint64)
        dec = lambda A: [gp.gfp_decode(params, tuple(int(d) for d in row)) for row in A]  # noqa: E731
        assert dec(O.add(X, Y, r)) == [(a + b) % p for a, b in zip(xs, ys)]
        assert dec(O.sub(X, Y, r)) == [(a - b) % p for a, b in zip(xs, ys)]
        assert dec(O.mul(X, Y, r, backend="school")) == [a * b % p for a, b in zip(xs, ys)]
        i = rng.randrange(2 * k + 1)
        assert dec(O.mul_pow_r(X, r, i)) == [a * pow(r, i, p) % p for a in xs]


def test_radix_mode_host_bound_proofs():
    """gfp_radix_mode runs the host-side bound proofs (make_consts): the
    paper's radices (bench_cli.py:36-41) take the compile-time mode 3 -- which
    includes the proof of the rounding column quotient's bounds --, other
    r = 2^a + 2^b the run-time mode 2, a radix near 2^64 has no lazy-digit
    headroom (the generic canonical path), invalid (k, r) are rejected."""
    from paper_1811_01490_b200 import _lib
    lib = _lib.load()
    assert lib.gfp_radix_mode(8, (1 << 59) + (1 << 16)) == 3
    assert lib.gfp_radix_mode(16, (1 << 58) + (1 << 10)) == 3
    assert lib.gfp_radix_mode(32, (1 << 56) + (1 << 21)) == 3
    assert lib.gfp_radix_mode(8, (1 << 58) + (1 << 12)) == 2   # not the k = 8 radix
    assert lib.gfp_radix_mode(16, (1 << 59) + (1 << 16)) == -1  # k = 8's radix at k = 16: no headroom
    assert lib.gfp_radix_mode(8, (1 << 63) + (1 << 34)) == -1
    assert lib.gfp_radix_mode(4, (1 << 64) - (1 << 50)) == -1
    assert lib.gfp_radix_mode(8, 12345678901234567) == 0        # no sparse structure
    assert lib.gfp_radix_mode(3, 1000) == -2 and lib.gfp_radix_mode(8, 1) == -2
