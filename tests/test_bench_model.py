"""bench.py's algorithmic work model (no GPU): the general-multiply counts it
divides by equal the reference's own counts of the cheap-twiddle split
(from fft.py:84-103), pass by pass and per transform."""
import os
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("N,K,want", [(4096, 16, 7136), (1 << 16, 16, 175584),
                                      (1 << 20, 32, 2962864), (1 << 24, 16, 76406240),
                                      (1 << 18, 64, 503616)])
def test_mults_per_transform_matches_reference_count(N, K, want):
    assert bench.mults_per_transform(N, K) == want
    assert sum(bench.mults_in_pass(N, K, p) for p in range(bench.passes(N, K))) == want


def test_mults_model_by_brute_force():
    # the per-pass count against a direct enumeration of the Stockham twiddles
    # omega^E, E = t (j mod Ns)(M / Ns): a general multiply iff E mod M != 0
    for N, K in [(256, 16), (4096, 16), (1024, 32), (512, 8)]:
        M = N // K
        for p in range(bench.passes(N, K)):
            Ns = K ** p
            direct = sum(1 for j in range(M) for t in range(K)
                         if ((t * (j % Ns) * (M // Ns)) % M) != 0)
            assert bench.mults_in_pass(N, K, p) == direct, (N, K, p)
            # the inverse's last pass multiplies every element by N^-1, a fused
            # pointwise operand every element of pass 0
            e = bench.passes(N, K)
            if p == e - 1:
                assert bench.mults_in_pass(N, K, p, inverse=True) == N
            if p == 0:
                assert bench.mults_in_pass(N, K, p, pre=True) == direct + N


def test_cpu_model_string():
    assert isinstance(bench.cpu_model(), str) and bench.cpu_model()
