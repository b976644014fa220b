"""Shape sweep of the transform kernels: batch sizes on both sides of every
CTA-shape threshold (k_pass44t NW = 16 / 8 / 4 by grid size, two vector sets
per launch, the fused poly-multiply middle with grid.y > 1, k_first16t), each
batched call compared row by row with the single-row call of the same
library, and sampled rows with the oracle (dft_general / dft_inverse,
fft.py:298-370; the poly-multiply composition of SURVEY 3.4)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

R8 = (1 << 59) + (1 << 16)
R16 = (1 << 58) + (1 << 10)


def _eq(a, b):
    import torch
    return a.shape == b.shape and torch.equal(a.view(torch.int64), b.view(torch.int64))


def _setup(k, r, K, e):
    import paper_1811_01490_b200 as gp
    from oracle import oracle as O
    params = gp.GfpParams(r, k)
    field = gp.GfpFftField(params, backend="cuda")
    omega = gp.roots_for(params, K ** e)
    plan = gp.build_plan(field, K, e, omega)
    return gp, O, params, plan, O.Plan(k, r, K, e, omega)


@pytest.mark.parametrize("e,batches", [(2, (1, 3, 40)), (3, (1, 7, 18, 19, 37, 73, 74, 75)),
                                       (4, (1, 2, 3, 5))],
                         ids=["n256", "n4096", "n65536"])
def test_k8_transform_batches(e, batches, cuda):
    gp, O, params, plan, oplan = _setup(8, R8, 16, e)
    N = 16 ** e
    for B in batches:
        x = gp.vec.uniform(N, params, seed=900 + B, batch=B) if B > 1 else \
            gp.vec.uniform(N, params, seed=900 + B).unsqueeze(0)
        y = gp.fft_tensor(x, plan)
        z = gp.fft_tensor(x, plan, inverse=True)
        for b in sorted({0, B // 2, B - 1}):
            assert _eq(gp.fft_tensor(x[b], plan), y[b]), (e, B, b)
            assert _eq(gp.fft_tensor(x[b], plan, inverse=True), z[b]), (e, B, b)
        xb = gp.vec.to_host(x[B - 1])
        assert np.array_equal(gp.vec.to_host(y[B - 1]), oplan.forward(xb)), (e, B)
        assert np.array_equal(gp.vec.to_host(z[B - 1]), oplan.inverse(xb)), (e, B)
        # round trip of the whole batch
        assert _eq(gp.fft_tensor(y, plan, inverse=True), x), (e, B)


@pytest.mark.parametrize("e,batches", [(2, (1, 5)), (3, (1, 2, 9, 37, 38)), (4, (1, 3))],
                         ids=["n256", "n4096", "n65536"])
def test_k8_poly_mul_batches(e, batches, cuda):
    """Batched poly-multiplies (the fused middle kernel with grid.y = batch for
    N >= 512, the two-kernel middle below) against the single product and the
    oracle."""
    gp, O, params, plan, oplan = _setup(8, R8, 16, e)
    N = 16 ** e
    for B in batches:
        import torch
        f = gp.vec.uniform(N, params, seed=1300 + B, batch=max(B, 2)).view(torch.int64)[:B] \
            .contiguous().view(torch.uint64)
        g = gp.vec.uniform(N, params, seed=1400 + B, batch=max(B, 2)).view(torch.int64)[:B] \
            .contiguous().view(torch.uint64)
        h = gp.poly_mul(f, g, plan)
        for b in sorted({0, B // 2, B - 1}):
            assert _eq(gp.poly_mul(f[b], g[b], plan), h[b]), (e, B, b)
        got = gp.vec.to_host(h[B - 1])
        want = oplan.poly_mul(gp.vec.to_host(f[B - 1]), gp.vec.to_host(g[B - 1]))
        assert np.array_equal(got, want), (e, B)
        # out aliasing an operand
        f2 = f.view(torch.int64).clone().view(torch.uint64)
        gp.poly_mul(f2, g, plan, out=f2)
        assert _eq(f2, h), (e, B)


@pytest.mark.parametrize("e,batches", [(2, (1, 3, 10)), (3, (1, 2, 5))], ids=["n1024", "n32768"])
def test_k16_transform_batches(e, batches, cuda):
    gp, O, params, plan, oplan = _setup(16, R16, 32, e)
    N = 32 ** e
    for B in batches:
        x = gp.vec.uniform(N, params, seed=1700 + B, batch=B) if B > 1 else \
            gp.vec.uniform(N, params, seed=1700 + B).unsqueeze(0)
        y = gp.fft_tensor(x, plan)
        z = gp.fft_tensor(x, plan, inverse=True)
        for b in sorted({0, B - 1}):
            assert _eq(gp.fft_tensor(x[b], plan), y[b]), (e, B, b)
        xb = gp.vec.to_host(x[B - 1])
        assert np.array_equal(gp.vec.to_host(y[B - 1]), oplan.forward(xb)), (e, B)
        assert np.array_equal(gp.vec.to_host(z[B - 1]), oplan.inverse(xb)), (e, B)
        assert _eq(gp.fft_tensor(y, plan, inverse=True), x), (e, B)
        h = gp.poly_mul(x, x, plan)
        assert np.array_equal(gp.vec.to_host(h[B - 1]), oplan.poly_mul(xb, xb)), (e, B)


# GFP primes p = r^8 + 1 outside the reference's list (found by a Miller-Rabin
# search over r = 2^a + 2^b and random even r): the run-time arithmetic modes
# of the fast path (gfp_radix_mode 1: sparse radix, 0: reciprocal quotient)
OTHER_R8 = [((1 << 56) + (1 << 28), 1), ((1 << 57) + (1 << 38), 0), (71234253391507836, 0),
            ((1 << 44) + (1 << 16), 1)]


@pytest.mark.parametrize("r,mode", OTHER_R8, ids=["2^56+2^28", "2^57+2^38", "random56", "2^44+2^16"])
def test_k8_other_prime_radices_run_time_modes(r, mode, cuda):
    """The reference's build_plan accepts any GFP prime (fft.py:237-275).  For
    k = 8 radices other than the paper's, the same pass kernels (k_pass44t,
    k_pmid44t, k_pass44) run in their run-time-radix instantiations: forward,
    inverse, batched, poly-multiply and the host entry against the oracle
    (schoolbook products)."""
    import torch
    import paper_1811_01490_b200 as gp
    from oracle import oracle as O
    from paper_1811_01490_b200 import _lib
    lib = _lib.load()
    assert lib.gfp_radix_mode(8, r) == mode
    k, K, e = 8, 16, 3
    N = K ** e
    params = gp.GfpParams(r, k)
    field = gp.GfpFftField(params, backend="cuda")
    omega = gp.roots_for(params, N)
    plan = gp.build_plan(field, K, e, omega)
    oplan = O.Plan(k, r, K, e, np.array(omega, dtype=np.uint64), backend="school")
    B = 20  # 160 CTAs: the NW = 8 shape; single rows take NW = 16
    x = O.random_elements(7000 + mode, k, r, B * N).reshape(B, N, k)
    xd = torch.stack([gp.vec.to_device(x[b], k) for b in range(B)])
    before = lib.gfp_tma_pass_launches()
    y = gp.fft_tensor(xd, plan)
    z = gp.fft_tensor(xd, plan, inverse=True)
    assert lib.gfp_tma_pass_launches() - before == 6
    for b in (0, B - 1):
        assert np.array_equal(gp.vec.to_host(y[b]), oplan.forward(x[b])), b
        assert np.array_equal(gp.vec.to_host(z[b]), oplan.inverse(x[b])), b
        assert _eq(gp.fft_tensor(xd[b], plan), y[b]), b
    assert _eq(gp.fft_tensor(y, plan, inverse=True), xd)
    f = np.zeros((N, k), dtype=np.uint64)
    g = f.copy()
    f[: N // 2] = x[0][: N // 2]
    g[: N // 3] = x[1][: N // 3]
    want = oplan.poly_mul(f, g)
    got = gp.vec.to_host(gp.poly_mul(gp.vec.to_device(f, k), gp.vec.to_device(g, k), plan))
    assert np.array_equal(got, want)
    assert np.array_equal(gp.poly_mul_host(f[: N // 2], g[: N // 3], plan),
                          want[: N // 2 + N // 3 - 1])
    # element-wise multiply in the same mode
    a, b2 = x[2][:1000], x[3][:1000]
    prod = gp.vec.to_host(gp.vec.mul(gp.vec.to_device(a, k), gp.vec.to_device(b2, k), params))
    assert np.array_equal(prod, O.mul(a, b2, r, backend="school"))


@pytest.mark.parametrize("r,mode", [((1 << 52) + (1 << 22), 1), ((1 << 52) + (1 << 34), 0)],
                         ids=["2^52+2^22", "2^52+2^34"])
def test_k16_other_prime_radices_run_time_modes(r, mode, cuda):
    """GFP primes p = r^16 + 1 outside the reference's list: k_pass<16> in its
    run-time-radix instantiations against the oracle (schoolbook products)."""
    import torch
    import paper_1811_01490_b200 as gp
    from oracle import oracle as O
    from paper_1811_01490_b200 import _lib
    assert _lib.load().gfp_radix_mode(16, r) == mode
    k, K, e = 16, 32, 2
    N = K ** e
    params = gp.GfpParams(r, k)
    field = gp.GfpFftField(params, backend="cuda")
    omega = gp.roots_for(params, N)
    plan = gp.build_plan(field, K, e, omega)
    oplan = O.Plan(k, r, K, e, np.array(omega, dtype=np.uint64), backend="school")
    x = O.random_elements(7100 + mode, k, r, 3 * N).reshape(3, N, k)
    xd = torch.stack([gp.vec.to_device(x[b], k) for b in range(3)])
    y = gp.fft_tensor(xd, plan)
    z = gp.fft_tensor(xd, plan, inverse=True)
    for b in range(3):
        assert np.array_equal(gp.vec.to_host(y[b]), oplan.forward(x[b])), b
        assert np.array_equal(gp.vec.to_host(z[b]), oplan.inverse(x[b])), b
    h = gp.poly_mul(xd[0], xd[1], plan)
    assert np.array_equal(gp.vec.to_host(h), oplan.poly_mul(x[0], x[1]))
    prod = gp.vec.to_host(gp.vec.mul(xd[0], xd[1], params))
    assert np.array_equal(prod, O.mul(x[0], x[1], r, backend="school"))


def test_k8_device_buffers_at_8_byte_offsets(cuda):
    """Device tensors whose base is only 8-byte aligned cannot be described to
    the TMA unit (tensor maps need 16 bytes): the same passes then run on the
    LDG form of the kernel and the poly-multiply keeps its two-kernel middle,
    with identical results."""
    import torch
    import paper_1811_01490_b200 as gp
    from paper_1811_01490_b200 import _lib
    lib = _lib.load()
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    N = 4096
    plan = gp.build_plan(field, 16, 3, gp.roots_for(params, N))

    def shifted(t):
        flat = torch.zeros(t.numel() + 1, dtype=torch.int64, device="cuda")
        v = flat[1:].view(t.shape)
        v.copy_(t.view(torch.int64))
        v = v.view(torch.uint64)
        assert v.data_ptr() % 16 == 8
        return v

    f = gp.vec.uniform(N, params, seed=31)
    g = gp.vec.uniform(N, params, seed=32)
    want_y = gp.fft_tensor(f, plan)
    want_h = gp.poly_mul(f, g, plan)
    fs, gs = shifted(f), shifted(g)
    before = lib.gfp_tma_pass_launches()
    out = shifted(torch.zeros_like(f.view(torch.int64)).view(torch.uint64))
    y = gp.fft_tensor(fs, plan, out=out)
    assert _eq(y, want_y)
    h = gp.poly_mul(fs, gs, plan, out=shifted(torch.zeros_like(f.view(torch.int64)).view(torch.uint64)))
    assert _eq(h, want_h)
    # aligned output, unaligned inputs: only the first pass falls back
    assert _eq(gp.fft_tensor(fs, plan), want_y)
    assert lib.gfp_tma_pass_launches() > before
