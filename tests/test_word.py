"""The word-prime layer: Montgomery constants and seeded roots (CPU), the GPU
transform and cyclic / negacyclic convolutions against the reference's own
outputs (tests/golden/word.npz, make_golden.py task_word) -- bit-exact.

Mirrors the reference's tests/test_word_field.py (constants, REDC, roots) and
the convolution checks of tests/test_gfp_mult.py / bench_cli verify
(negacyclic_vs_schoolbook).
"""
import random

import numpy as np
import pytest

from conftest import load_npz

import paper_1811_01490_b200 as gp
from paper_1811_01490_b200 import word as W

P1, P2 = gp.P1, gp.P2


# ---------------------------------------------------------------------------
# CPU: constants and roots

@pytest.mark.parametrize("q", [P1, P2, 257, 65537, (1 << 61) - 1])
def test_word_prime_constants(q):
    ctx = W.word_prime(q)
    assert (q * ctx.q_neg_inv) & W.MASK64 == W.MASK64
    assert ctx.r2 == (1 << 128) % q and ctx.one_mont == (1 << 64) % q


@pytest.mark.parametrize("q", [1, 2, 4, 1 << 63, (1 << 63) + 1])
def test_word_prime_rejects(q):
    with pytest.raises(ValueError):
        W.WordPrime.make(q)


def test_mont_mul_and_conversions():
    ctx = W.word_prime(P1)
    rng = random.Random(5)
    for _ in range(200):
        a, b = rng.randrange(P1), rng.randrange(P1)
        am, bm = W.mont_convert_in(ctx, a), W.mont_convert_in(ctx, b)
        assert W.mont_convert_out(ctx, W.mont_mul(ctx, am, bm)) == a * b % P1
    assert W.mont_convert_out(ctx, W.mont_inv(ctx, W.mont_convert_in(ctx, 12345))) == \
        pow(12345, -1, P1)
    with pytest.raises(ZeroDivisionError):
        W.mont_inv(ctx, 0)


def test_roots_match_reference(golden):
    for q, K, e, om, tag in golden["word"]["transforms"]:
        assert W.word_primitive_root(W.word_prime(q), K ** e) == om, tag


def test_root_rejections():
    ctx = W.word_prime(P2)  # P2 - 1 = 69 * 2^55
    with pytest.raises(ValueError):
        W.word_primitive_root(ctx, 3 << 2)
    with pytest.raises(ValueError):
        W.word_primitive_root(ctx, 1 << 56)


# ---------------------------------------------------------------------------
# GPU: transforms and convolutions vs the reference



@pytest.mark.gpu
def test_word_dft_vs_reference(cuda, golden):
    z = load_npz("word.npz")
    for q, K, e, om, tag in golden["word"]["transforms"]:
        ctx = W.word_prime(q)
        field = gp.MontField(ctx)
        plan = gp.build_plan(field, K, e, om)
        v = [int(t) for t in z["dft_in_" + tag]]
        fwd = gp.dft_general(list(v), plan, field)
        assert fwd == [int(t) for t in z["dft_fwd_" + tag]], tag
        inv = gp.dft_inverse(list(v), plan, field)
        assert inv == [int(t) for t in z["dft_inv_" + tag]], tag
        assert gp.dft_inverse(list(fwd), plan, field) == v, tag


@pytest.mark.gpu
def test_word_ntt_batched_tensor(cuda, golden):
    import torch
    z = load_npz("word.npz")
    q, K, e, om, tag = golden["word"]["transforms"][-1]
    plan = gp.build_plan(gp.MontField(W.word_prime(q)), K, e, om)
    x = torch.from_numpy(np.stack([z["dft_in_" + tag]] * 3)).cuda()
    y = gp.word_ntt(x, plan)
    want = torch.from_numpy(np.stack([z["dft_fwd_" + tag]] * 3)).cuda()
    assert torch.equal(y.view(torch.int64), want.view(torch.int64))
    back = gp.word_ntt(y, plan, inverse=True)
    assert torch.equal(back.view(torch.int64), x.view(torch.int64))


@pytest.mark.gpu
def test_word_plan_rejections(cuda):
    ctx = W.word_prime(P1)
    field = gp.MontField(ctx)
    om = W.word_primitive_root(ctx, 256)
    with pytest.raises(ValueError):
        gp.build_plan(field, 16, 2, W.mont_mul(ctx, om, om))  # order 128, not 256
    with pytest.raises(ValueError):
        gp.build_plan(field, 12, 2, om)
    with pytest.raises(ValueError):
        gp.build_plan(field, 16, 0, om)
    plan = gp.build_plan(field, 16, 2, om)
    with pytest.raises(ValueError):
        gp.dft_general([0] * 255, plan, field)


@pytest.mark.gpu
def test_convolutions_vs_reference(cuda, golden):
    z = load_npz("word.npz")
    for q, n, tag in golden["word"]["cyclic"]:
        f = [int(t) for t in z["cyc_f_" + tag]]
        g = [int(t) for t in z["cyc_g_" + tag]]
        got = gp.cyclic_convolution(f, g, W.word_prime(q), n)
        assert list(got) == [int(t) for t in z["cyc_h_" + tag]], tag
    for q, k, tag in golden["word"]["negacyclic"]:
        x = [int(t) for t in z["neg_x_" + tag]]
        y = [int(t) for t in z["neg_y_" + tag]]
        got = gp.negacyclic_convolution(x, y, W.word_prime(q), k)
        assert list(got) == [int(t) for t in z["neg_h_" + tag]], tag


@pytest.mark.gpu
def test_negacyclic_vs_schoolbook(cuda):
    """bench_cli's negacyclic_vs_schoolbook check (bench_cli.py:185-194)."""
    rng = random.Random(9)
    for q in (P1, P2):
        ctx = W.word_prime(q)
        for k in (4, 16, 64):
            x = [rng.randrange(q) for _ in range(k)]
            y = [rng.randrange(q) for _ in range(k)]
            want = [0] * k
            for i in range(k):
                for j in range(k):
                    if i + j < k:
                        want[i + j] += x[i] * y[j]
                    else:
                        want[i + j - k] -= x[i] * y[j]
            assert list(gp.negacyclic_convolution(x, y, ctx, k)) == [w % q for w in want]


@pytest.mark.gpu
def test_convolution_rejections(cuda):
    ctx = W.word_prime(P1)
    with pytest.raises(ValueError):
        gp.cyclic_convolution([1, 2, 3], [1, 2, 3], ctx, 3)
    with pytest.raises(ValueError):
        gp.cyclic_convolution([P1, 0], [1, 0], ctx, 2)      # unreduced
    with pytest.raises(ValueError):
        gp.negacyclic_convolution([1, 2], [1, 2, 3, 4], ctx, 4)
    with pytest.raises(ValueError):
        gp.cyclic_convolution([0] * 4, [0] * 4, W.word_prime(7), 4)  # 4 does not divide 6


@pytest.mark.gpu
def test_large_batched_convolution_properties(cuda):
    """n = 2^16, batch 4: convolving with a unit impulse at position s
    rotates (cyclic) or rotates with sign (negacyclic); and linearity."""
    import torch
    n, s = 1 << 16, 12345
    for q in (P1, P2):
        ctx = W.word_prime(q)
        gen = torch.Generator().manual_seed(q % 1000)
        x = (torch.randint(0, 1 << 62, (4, n), generator=gen, dtype=torch.int64) % q)
        delta = torch.zeros((4, n), dtype=torch.int64)
        delta[:, s] = 1
        xd, dd = x.view(torch.uint64).cuda(), delta.view(torch.uint64).cuda()
        cyc = gp.word_convolve(xd, dd, gp.conv_plan(ctx, n, False)).view(torch.int64).cpu()
        assert torch.equal(cyc, torch.roll(x, s, dims=1))
        neg = gp.word_convolve(xd, dd, gp.conv_plan(ctx, n, True)).view(torch.int64).cpu()
        want = torch.roll(x, s, dims=1)
        want[:, :s] = (q - want[:, :s]) % q
        assert torch.equal(neg, want)
        y = (torch.randint(0, 1 << 62, (4, n), generator=gen, dtype=torch.int64) % q)
        yd = y.view(torch.uint64).cuda()
        plan = gp.conv_plan(ctx, n, False)
        a = gp.word_convolve(xd, yd, plan).view(torch.int64).cpu()
        b = gp.word_convolve(yd, xd, plan).view(torch.int64).cpu()
        assert torch.equal(a, b)
