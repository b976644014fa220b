"""GPU parity of the drop-in API surface around the transform: the root
routine at every benchmark size, the field protocol object as the
reference's transform drives it, the public wrappers twiddle_apply /
dft_base / FftPlan.twiddle_table, the device canonical-form check's reject
path, and the sharded four-step output in natural order against the
reference's own digest.  Bit-exact throughout (integer work).
"""
import numpy as np
import pytest

from conftest import load_npz

pytestmark = pytest.mark.gpu

R8 = (1 << 59) + (1 << 16)


def _gp():
    import paper_1811_01490_b200 as gp
    return gp


def _O():
    from oracle import oracle as O
    return O


def _tuples(a):
    return [tuple(int(d) for d in row) for row in a]


# ---------------------------------------------------------------------------
# roots: bench_cli._gfp_root (bench_cli.py:398-402) at every golden size,
# through roots_for -- the routine bench.py builds its plans with

def test_roots_for_every_golden_size(golden, cuda):
    gp = _gp()
    keys = sorted(k for k in golden if k.startswith("root_"))
    assert {"root_k8_N65536", "root_k8_N16777216", "root_k16_N1048576",
            "root_k32_N262144"} <= set(keys)
    for key in keys:
        g = golden[key]
        params = gp.GfpParams(g["r"], g["k"])
        got_g = gp.gfp_find_nth_root(params, g["N"], seed=0)
        assert got_g == tuple(int(d) for d in g["g"]), key
        assert gp.roots_for(params, g["N"]) == tuple(int(d) for d in g["omega"]), key


# ---------------------------------------------------------------------------
# the field protocol (gfp_mult.py:518-592) driven by the reference's schedule

def test_field_protocol_drives_reference_schedule(golden, cuda):
    # oracle/protocol.py restates fft.py's dft_general / dft_inverse call
    # pattern (pinned on the CPU by test_protocol_driver.py); every add, sub,
    # shift, mul, pow, inv_scalar and root_power_mul_factory call here is a
    # device call on the product's GfpFftField
    from oracle import protocol as P
    gp = _gp()
    z = load_npz("fft_small.npz")
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    omega = tuple(int(d) for d in golden["root_k8_N256"]["omega"])
    plan = P.ProtocolPlan(field, 16, 2, omega)
    v = _tuples(z["x"][0])
    assert P.dft(list(v), plan) == _tuples(z["fwd"][0])
    assert P.dft_inverse(list(v), plan) == _tuples(z["inv"][0])


def test_field_protocol_methods_vs_oracle(cuda):
    gp, O = _gp(), _O()
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    xs = O.random_elements(11, 8, R8, 70)
    omega = tuple(int(d) for d in xs[0])
    # root_power_mul_factory, generic omega: the table path (gfp_mult.py:584-592)
    f = field.root_power_mul_factory(omega, 64)
    pw = [np.array([[1] + [0] * 7], dtype=np.uint64)]
    for _ in range(63):
        pw.append(O.mul(pw[-1], xs[:1].copy(), R8))
    for t in (0, 1, 2, 17, 63):
        x = tuple(int(d) for d in xs[t + 1 if t < 69 else 1])
        want = O.mul(np.array([x], dtype=np.uint64), pw[t], R8)
        assert f(x, t) == tuple(int(d) for d in want[0])
    # omega = r / 1/r: rotations (gfp_mult.py:574-583)
    fr = field.root_power_mul_factory(field.shift_root, 16)
    fi = field.root_power_mul_factory(field.shift_root_inv, 16)
    for t in range(16):
        x = xs[t + 2:t + 3].copy()
        assert fr(tuple(int(d) for d in x[0]), t) == tuple(int(d) for d in O.mul_pow_r(x, R8, t)[0])
        assert fi(tuple(int(d) for d in x[0]), t) == \
            tuple(int(d) for d in O.mul_pow_r(x, R8, (16 - t) % 16)[0])
    # inv_scalar (gfp_mult.py:562-563): n * n^-1 = 1 on the device multiply
    for n in (1, 2, 4096, 1 << 16, 1 << 24, 12345):
        inv = field.inv_scalar(n)
        assert field.mul(inv, gp.gfp_encode(params, n)) == field.one()
    # pow (gfp_mult.py:552-554) against repeated oracle multiplies
    x = xs[5:6].copy()
    acc = np.array([[1] + [0] * 7], dtype=np.uint64)
    for e in range(0, 40):
        assert field.pow(tuple(int(d) for d in x[0]), e) == tuple(int(d) for d in acc[0])
        acc = O.mul(acc, x, R8)
    big = (1 << 200) + 12345
    want = gp.gfp_encode(params, pow(gp.gfp_decode(params, tuple(int(d) for d in x[0])),
                                     big, params.p))
    assert field.pow(tuple(int(d) for d in x[0]), big) == want
    with pytest.raises(ValueError):
        field.pow(field.one(), -1)


# ---------------------------------------------------------------------------
# public wrappers

def test_twiddle_apply_diagonal_known_answer(cuda):
    # tests/test_fft.py:110-118: D_{2,4} over p = r^4 + 1, r = 2^64 - 2^50
    gp = _gp()
    params = gp.GfpParams((1 << 64) - (1 << 50), 4)
    field = gp.GfpFftField(params, backend="bigint")
    v = [field.one()] * 8
    gp.twiddle_apply(v, 4, 2, gp.gfp_encode(params, params.r), field)
    assert [gp.gfp_decode(params, x) for x in v] == \
        [1, 1, 1, 1, 1, params.r, params.r ** 2, params.r ** 3]


@pytest.mark.parametrize("m,n,off", [(4, 4, 0), (16, 16, 0), (8, 32, 5), (2, 3, 1)])
def test_twiddle_apply_vs_oracle(m, n, off, cuda):
    # v[off + j m + i] *= w^(i j) (fft.py:62-81), w the 256-th root
    gp, O = _gp(), _O()
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    w = gp.roots_for(params, 256)
    total = off + m * n + 3
    x = O.random_elements(21 + m, 8, R8, total)
    v = _tuples(x)
    gp.twiddle_apply(v, m, n, w, field, offset=off)
    wa = np.array([w], dtype=np.uint64)
    pw = [np.array([[1] + [0] * 7], dtype=np.uint64)]
    for _ in range(m * n):
        pw.append(O.mul(pw[-1], wa, R8))
    want = x.copy()
    for j in range(n):
        for i in range(m):
            want[off + j * m + i] = O.mul(x[off + j * m + i:off + j * m + i + 1].copy(),
                                          pw[i * j], R8)[0]
    assert v == _tuples(want)


@pytest.mark.parametrize("k,K", [(8, 16), (16, 32), (32, 64)])
def test_dft_base_at_r_and_inverse_r(k, K, cuda):
    # dft_base (fft.py:186-193) at omega_base = r and 1/r, against the
    # oracle's K-point plan at the same root; offset addressing as in _run_base
    gp, O = _gp(), _O()
    r = O.DEFAULT_RADIX[k]
    params = gp.GfpParams(r, k)
    field = gp.GfpFftField(params, backend="cuda")
    x = O.random_elements(31 + k, k, r, 2 * K + 3)
    for root, want_root in ((field.shift_root, field.shift_root),
                            (field.shift_root_inv, field.shift_root_inv)):
        v = _tuples(x)
        gp.dft_base(v, root, field, K=K, offset=K + 3)
        plan = O.Plan(k, r, K, 1, np.array(want_root, dtype=np.uint64))
        want = x.copy()
        want[K + 3:2 * K + 3] = plan.forward(x[K + 3:2 * K + 3].copy())
        assert v == _tuples(want)


def test_plan_twiddle_table_vs_oracle(golden, cuda):
    # FftPlan.twiddle_table = omega^j, j < K^(e-1) (fft.py:211-214)
    gp, O = _gp(), _O()
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    omega = tuple(int(d) for d in golden["root_k8_N4096"]["omega"])
    plan = gp.build_plan(field, 16, 3, omega)
    oplan = O.Plan(8, R8, 16, 3, np.array(omega, dtype=np.uint64))
    assert plan.twiddle_table == _tuples(oplan.table())


# ---------------------------------------------------------------------------
# is_canonical's reject path on the device (gfp_field.py:49-56;
# tests/test_gfp_field.py:73-83)

def test_device_is_canonical_rejects(cuda):
    gp, O = _gp(), _O()
    params = gp.GfpParams(10, 4)
    cases = [((10, 0, 0, 0), False), ((0, 0, 0, 11), False), ((1, 0, 0, 10), False),
             ((0, 0, 0, 10), True), ((9, 9, 9, 9), True), ((0, 10, 0, 0), False),
             ((0, 0, 0, 0), True), ((0, 0, 1, 10), False), ((2 ** 64 - 1, 0, 0, 0), False)]
    got = gp.vec.is_canonical(gp.vec.to_device([c for c, _ in cases], 4), params)
    assert [bool(b) for b in got.cpu().numpy()] == [w for _, w in cases]
    # k = 8, paper radix: random mixtures of digits < r, = r, > r and form B
    rng = np.random.default_rng(5)
    n = 4096
    x = O.random_elements(9, 8, R8, n)
    sel = rng.integers(0, 5, size=n)
    x[sel == 1, rng.integers(0, 8)] = R8                     # digit r somewhere
    x[sel == 2, 7] = R8                                      # top digit r (form B iff rest 0)
    x[sel == 3] = 0
    x[sel == 3, 7] = R8                                      # exact form B
    x[sel == 4, rng.integers(0, 8)] = R8 + 1 + rng.integers(0, 1 << 40)
    got = gp.vec.is_canonical(gp.vec.to_device(x, 8), params=gp.GfpParams(R8, 8))
    want = O.is_canonical(x, R8)
    assert np.array_equal(got.cpu().numpy().astype(bool), want)
    assert want.sum() not in (0, n)  # both outcomes exercised


# ---------------------------------------------------------------------------
# the sharded four-step C4 output, gathered to natural order, against the
# reference's digest of out[0:2^16] of the full 2^24-point forward

@pytest.mark.slow
def test_sharded_c4_natural_order_vs_reference(golden, cuda):
    import torch
    gp, O = _gp(), _O()
    from paper_1811_01490_b200.sharded import GpuShardOps, ShardedFFT
    if "c4_full" not in golden:
        pytest.skip("golden c4_full not generated")
    N1 = N2 = 4096
    N = N1 * N2
    params = gp.GfpParams(R8, 8)
    field = gp.GfpFftField(params, backend="cuda")
    omega = gp.roots_for(params, N)
    assert omega == tuple(int(d) for d in golden["root_k8_N16777216"]["omega"])
    x = O.random_elements(4, 8, R8, N)
    assert O.digest(x) == golden["c4_full"]["input"]
    xd = gp.vec.to_device(x, 8)
    del x
    ops = GpuShardOps(field, 16, N1, N2, omega)
    for peer in (False, True):
        sh = ShardedFFT(ops, 8, N1, N2)
        if peer:
            sh.use_peer_exchange()
        rows = sh.forward(sh.scatter_columns(xd))          # [k1, d, k2] = X[k1 + N1 k2]
        head = rows.view(torch.int64)[:, :, : (1 << 16) // N1]   # k2 < 16
        nat = head.permute(2, 0, 1).reshape(1 << 16, 8)    # i = k1 + N1 k2 -> [i, d]
        got = nat.contiguous().cpu().numpy().view(np.uint64)
        assert O.digest(got) == golden["c4_full"]["forward_slice_2_16"], peer
