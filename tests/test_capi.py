"""The C-ABI library loads and exports every symbol include/gfpfft.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "gfpfft.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gfp_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    from paper_1811_01490_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_library_exports_every_symbol():
    from paper_1811_01490_b200 import _lib
    checked = os.path.join(os.path.dirname(_lib.LIB_PATH), "libgfpfft_checked.so")
    for path in (_lib.LIB_PATH, checked):  # the product and the checked build
        lib = ctypes.CDLL(path)
        for name in _declared():
            assert hasattr(lib, name), (path, name)


def test_host_only_entry_points():
    from paper_1811_01490_b200 import _lib
    lib = _lib.load()
    assert lib.gfp_version() == 1
    assert lib.gfp_strerror(0) == b"ok"
    # check_prime_compat / fast-path eligibility are host-side decisions
    assert lib.gfp_check_prime_compat(8, (1 << 59) + (1 << 16)) == 1
    assert lib.gfp_check_prime_compat(8, (1 << 63) + (1 << 34)) == 0
    for k, r in [(8, (1 << 59) + (1 << 16)), (16, (1 << 58) + (1 << 10)),
                 (32, (1 << 56) + (1 << 21))]:
        assert lib.gfp_fast_path_ok(k, r) == 1
    assert lib.gfp_fast_path_ok(8, (1 << 63) + (1 << 34)) == 0
    assert lib.gfp_fast_path_ok(64, 284903849103190610) == 0


def test_invalid_arguments_rejected_before_device_work():
    from paper_1811_01490_b200 import _lib
    lib = _lib.load()
    # k not a power of two / r < 2 / shift out of range -> GFP_EINVAL
    assert lib.gfp_vec_add(None, None, None, 4, 3, 10, None) == _lib.GFP_EINVAL
    assert lib.gfp_vec_add(None, None, None, 4, 8, 1, None) == _lib.GFP_EINVAL
    assert lib.gfp_vec_mul_pow_r(None, None, 4, 8, 10, 17, None) == _lib.GFP_EINVAL
    h = ctypes.c_void_p()
    om = (ctypes.c_uint64 * 8)()
    assert lib.gfp_fft_plan_create(ctypes.byref(h), 8, 10, 12, 2, om, None) == _lib.GFP_EINVAL
    assert lib.gfp_fft_plan_create(ctypes.byref(h), 8, 10, 32, 2, om, None) == _lib.GFP_EINVAL


def test_missing_library_fails_loudly(tmp_path):
    # no CPU fallback: importing the package without its CUDA library raises
    import subprocess
    import sys
    env = dict(os.environ, GFPFFT_LIB=str(tmp_path / "missing" / "libgfpfft.so"))
    code = "import paper_1811_01490_b200"
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode != 0
    assert "ImportError" in p.stderr and "no CPU fallback" in p.stderr
