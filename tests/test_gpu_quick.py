"""First GPU parity checks: element-wise ops vs the reference goldens and a
small transform vs the oracle."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_npz

pytestmark = pytest.mark.gpu


def _configs():
    return sorted(glob.glob(os.path.join(GOLDEN, "elementwise_k*.npz")))


@pytest.mark.parametrize("path", _configs(), ids=lambda p: os.path.basename(p)[:-4])
def test_elementwise_vs_reference(path, cuda):
    import paper_1811_01490_b200 as gp
    z = np.load(path)
    k, r = int(z["k"]), int(z["r"])
    params = gp.GfpParams(r, k)
    x = gp.vec.to_device(z["x"], k)
    y = gp.vec.to_device(z["y"], k)
    assert np.array_equal(gp.vec.to_host(gp.vec.add(x, y, params)), z["add"])
    assert np.array_equal(gp.vec.to_host(gp.vec.sub(x, y, params)), z["sub"])
    assert np.array_equal(gp.vec.to_host(gp.vec.mul(x, y, params)), z["mul"])
    xs = gp.vec.to_device(z["x"][: z["shift"].shape[0]], k)
    for i in range(2 * k + 1):
        got = gp.vec.to_host(gp.vec.mul_pow_r(xs, i, params))
        assert np.array_equal(got, z["shift"][:, i, :]), "shift %d" % i


def test_small_fft_vs_reference(cuda):
    import paper_1811_01490_b200 as gp
    z = load_npz("fft_small.npz")
    k, K, e = 8, 16, 2
    r = gp.DEFAULT_RADIX[k]
    params = gp.GfpParams(r, k)
    field = gp.GfpFftField(params)
    omega = gp.roots_for(params, K ** e)
    plan = gp.build_plan(field, K, e, omega)
    for b in range(z["x"].shape[0]):
        x = gp.vec.to_device(z["x"][b], k)
        fwd = gp.vec.to_host(gp.fft_tensor(x, plan))
        assert np.array_equal(fwd, z["fwd"][b])
        inv = gp.vec.to_host(gp.fft_tensor(x, plan, inverse=True))
        assert np.array_equal(inv, z["inv"][b])
