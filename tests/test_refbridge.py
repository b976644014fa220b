"""The reference's own CLI (gfpfft.bench_cli) with the gfp-cuda backend
registered by paper_1811_01490_b200.refbridge.

The reference package is imported from baseline/_ref (a pip install of
/root/reference into the repo, git-ignored; it travels to the GPU box with
the snapshot).  When it is absent the tests skip."""
import csv
import io
import os
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")


def _bench_cli():
    if not os.path.isdir(os.path.join(REF, "gfpfft")):
        pytest.skip("reference package not installed under baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import importlib
    import gfpfft.bench_cli as bc
    importlib.reload(bc)  # a fresh module: install() patches module globals
    return bc


def _run(bc, argv):
    out = io.StringIO()
    old = sys.stdout
    cpus = os.sched_getaffinity(0)  # the reference's bench pins to one CPU
    sys.stdout = out
    try:
        rc = bc.main(argv)
    finally:
        sys.stdout = old
        os.sched_setaffinity(0, cpus)
    return rc, list(csv.reader(io.StringIO(out.getvalue())))


def test_install_registers_backend_and_keeps_reference_backends():
    from paper_1811_01490_b200 import refbridge
    bc = _bench_cli()
    refbridge.install(bc)
    refbridge.install(bc)  # idempotent
    assert bc.BACKENDS.count("gfp-cuda") == 1
    assert set(bc.BACKENDS) >= {"gfp-fft", "gfp-bigint", "oracle-bigint", "gfp-cuda"}
    # the parser takes the new backend name
    args = bc.build_parser().parse_args(["bench-fft", "--backend", "gfp-cuda"])
    assert args.backend == "gfp-cuda"
    # the reference's own backends still run through the wrapped dft_general
    rc, rows = _run(bc, ["bench-fft", "--K", "16", "--e", "1", "--backend", "gfp-bigint"])
    assert rc == 0 and rows[1][2] == "gfp-bigint"


@pytest.mark.gpu
@pytest.mark.parametrize("e", [2, 3])
def test_reference_bench_fft_cross_checks_gfp_cuda(e, cuda):
    # cmd_bench_fft (bench_cli.py:417-467) computes every backend's digest on
    # the same seeded vector and aborts on any mismatch before timing: with
    # all four backends, "verified" = yes on every row means gfp-cuda's
    # transform equals gfp-fft's, gfp-bigint's and oracle-bigint's
    from paper_1811_01490_b200 import refbridge
    bc = refbridge.install(_bench_cli())
    rc, rows = _run(bc, ["bench-fft", "--K", "16", "--e", str(e), "--seed", "3"])
    assert rc == 0
    assert rows[0] == ["K", "e", "backend", "total_seconds", "permutation_seconds",
                       "basecase_seconds", "twiddle_seconds", "avg_mult_seconds", "verified"]
    got = {row[2]: row for row in rows[1:]}
    assert set(got) == {"gfp-fft", "gfp-bigint", "oracle-bigint", "gfp-cuda"}
    assert all(row[8] == "yes" for row in got.values())
    cuda_row = got["gfp-cuda"]
    assert float(cuda_row[3]) > 0 and all(float(c) >= 0 for c in cuda_row[4:7])
