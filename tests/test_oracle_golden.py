"""The oracle (oracle/gfp_oracle.c, a CPU restatement of the reference)
pinned against the reference's own outputs (tests/golden, produced by
tests/golden/make_golden.py running /root/reference).  CPU only."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_npz
from oracle import oracle as O

R8 = O.DEFAULT_RADIX[8]
R16 = O.DEFAULT_RADIX[16]
R32 = O.DEFAULT_RADIX[32]


def _configs():
    return sorted(glob.glob(os.path.join(GOLDEN, "elementwise_k*.npz")))


@pytest.mark.parametrize("path", _configs(), ids=lambda p: os.path.basename(p)[:-4])
def test_elementwise(path):
    z = np.load(path)
    k, r = int(z["k"]), int(z["r"])
    x, y = z["x"], z["y"]
    assert np.array_equal(O.add(x, y, r), z["add"])
    assert np.array_equal(O.sub(x, y, r), z["sub"])
    assert np.array_equal(O.mul(x, y, r, backend="school"), z["mul"])
    if O.check_prime_compat(k, r):
        assert np.array_equal(O.mul(x, y, r, backend="fft"), z["mul"])
    xs = np.ascontiguousarray(x[: z["shift"].shape[0]])
    for i in range(2 * k + 1):
        assert np.array_equal(O.mul_pow_r(xs, r, i), z["shift"][:, i, :])
    assert O.is_canonical(x, r).all()


def test_compat_matches_reference_table():
    # tests/test_acceptance.py:41-45, 259-261 and the by-design failure
    assert O.check_prime_compat(8, R8)
    assert O.check_prime_compat(16, R16)
    assert O.check_prime_compat(32, R32)
    assert not O.check_prime_compat(8, (1 << 63) + (1 << 34))


def test_base_case_ops(golden):
    # fft.base_case_ops for every base size; DFT8 transcript of tests/test_fft.py:25-32
    for K in (8, 16, 32, 64):
        assert [list(op) for op in O.base_case_ops(K)] == golden["base_case_ops"][str(K)]
    ops = O.base_case_ops(16)
    assert sum(1 for op in ops if op[0] == "tw") == 17


def test_roots(golden):
    for key, g in golden.items():
        if not key.startswith("root_"):
            continue
        if g["k"] not in (8, 16, 32) or g["N"] > (1 << 20):
            continue
        gg, w = O.gfp_root(g["k"], g["r"], g["N"])
        assert [str(int(d)) for d in gg] == g["g"], key
        assert [str(int(d)) for d in w] == g["omega"], key


def test_input_convention(golden):
    # Random(seed).randrange(p) + gfp_encode (bench_cli.py:383, 394)
    assert O.digest(O.random_elements(0, 8, R8, 4096)) == golden["c1"]["input"]
    assert O.digest(O.random_elements(4, 8, R8, 1 << 16)) == golden["c4_prefix"]["input"]


def test_small_fft(golden):
    z = load_npz("fft_small.npz")
    w = [int(d) for d in golden["root_k8_N256"]["omega"]]
    plan = O.Plan(8, R8, 16, 2, w)
    for b in range(z["x"].shape[0]):
        assert np.array_equal(plan.forward(z["x"][b]), z["fwd"][b])
        assert np.array_equal(plan.inverse(z["x"][b]), z["inv"][b])


def test_c1(golden):
    z = load_npz("c1.npz")
    w = [int(d) for d in golden["root_k8_N4096"]["omega"]]
    plan = O.Plan(8, R8, 16, 3, w)
    y = plan.forward(z["x"])
    assert np.array_equal(y, z["fwd"])
    assert O.digest(y) == golden["c1"]["forward"]
    assert np.array_equal(plan.inverse(y), z["x"])


def test_c2(golden):
    g = golden["c2"]
    N = 1 << 16
    f = np.zeros((N, 8), dtype=np.uint64)
    h = np.zeros((N, 8), dtype=np.uint64)
    f[: N // 2] = O.random_elements(1, 8, R8, N // 2)
    h[: N // 2] = O.random_elements(2, 8, R8, N // 2)
    w = [int(d) for d in golden["root_k8_N65536"]["omega"]]
    plan = O.Plan(8, R8, 16, 4, w)
    out = plan.poly_mul(f, h, threads=os.cpu_count() or 1)
    assert O.digest(out) == g["product"]


def test_c4_prefix(golden):
    g = golden["c4_prefix"]
    w = [int(d) for d in golden["root_k8_N65536"]["omega"]]
    plan = O.Plan(8, R8, 16, 4, w)
    x = O.random_elements(4, 8, R8, 1 << 16)
    assert O.digest(plan.forward(x, threads=os.cpu_count() or 1)) == g["forward"]


def test_c5_mul(golden):
    g = golden["c5_mul"]
    xy = O.random_elements(5, 32, R32, 2 * g["pairs"])
    x, y = np.ascontiguousarray(xy[0::2]), np.ascontiguousarray(xy[1::2])
    assert O.digest(O.mul(x, y, R32, backend="fft")) == g["products"]


def test_oracle_threads_match_serial(golden):
    # tests/test_fft.py:264-273
    w = [int(d) for d in golden["root_k8_N4096"]["omega"]]
    plan = O.Plan(8, R8, 16, 3, w)
    x = O.random_elements(9, 8, R8, 4096)
    assert np.array_equal(plan.forward(x, threads=1), plan.forward(x, threads=4))


def test_plan_rejections():
    w = [int(d) for d in O.gfp_root(8, R8, 256)[1]]
    with pytest.raises(ValueError):
        O.Plan(8, R8, 12, 2, w)
    with pytest.raises(ValueError):
        O.Plan(8, R8, 32, 2, w)
    with pytest.raises(ValueError):
        O.Plan(8, R8, 16, 2, [1] + [0] * 7)
