"""The checked build (libgfpfft_checked.so, GFP_DEBUG=1) as the stand-in for
compute-sanitizer, which the GPU pool does not offer: every kernel family
runs small cases under index guards and per-warp timing jitter
(tools/checked_cases.py), every result is compared with the oracle, and no
guard may fire.  The self-test proves the guards are live."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

CHECKED = os.path.join(ROOT, "paper_1811_01490_b200", "libgfpfft_checked.so")


def _run(code_or_script, timeout=900):
    if not os.path.exists(CHECKED):
        pytest.fail("checked build missing: make -C paper_1811_01490_b200/csrc checked")
    env = dict(os.environ, GFPFFT_LIB=CHECKED)
    args = [sys.executable] + (["-c", code_or_script] if "\n" in code_or_script
                               else [code_or_script])
    return subprocess.run(args, env=env, capture_output=True, text=True, timeout=timeout,
                          cwd=ROOT)


def test_checked_build_exports_debug_flag():
    import ctypes
    lib = ctypes.CDLL(CHECKED)
    assert lib.gfp_debug_build() == 1
    from paper_1811_01490_b200 import _lib
    assert _lib.load().gfp_debug_build() == 0  # the product build has no guards


@pytest.mark.gpu
def test_checked_build_guards_fire(cuda):
    res = _run("""
import sys; sys.path.insert(0, %r)
from paper_1811_01490_b200 import _lib
import torch
torch.cuda.set_device(0)
assert _lib.load().gfp_debug_selftest(None) == 0
print("selftest done")
""" % ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "GFP_CHECK" in res.stdout and "selftest done" in res.stdout


@pytest.mark.gpu
@pytest.mark.slow
def test_checked_build_all_kernel_families(cuda):
    res = _run(os.path.join(ROOT, "tools", "checked_cases.py"))
    out = res.stdout + res.stderr
    assert res.returncode == 0, out[-3000:]
    assert "GFP_CHECK" not in out, [ln for ln in out.splitlines() if "GFP_CHECK" in ln][:20]
    assert "checked build: 1" in out and "all cases ok" in out
