"""The CLI front end (paper_1811_01490_b200/cli.py): radix syntax and GFPV
files on the CPU, the gfp-cuda commands on the GPU.

Mirrors the reference's tests/test_bench_cli.py (radix forms and rejections,
GFPV round trip / corruption cases, verify determinism and exit codes).  The
GFPV interop fixtures tests/golden/fft256_{in,fwd}.gfpv were written by the
reference's own bench_cli.write_gfpv (tests/golden/make_golden.py task_gfpv).
"""
import csv
import io
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN

from paper_1811_01490_b200 import cli
from paper_1811_01490_b200.cli import (GfpvFormatError, main, parse_radix, read_gfpv,
                                       read_gfpv_array, write_gfpv)

R8 = (1 << 59) + (1 << 16)


# ---------------------------------------------------------------------------
# radix syntax (reference tests/test_bench_cli.py:19-41)

def test_parse_radix_forms():
    assert parse_radix("2^59+2^16") == R8
    assert parse_radix("2^64-2^50") == (1 << 64) - (1 << 50)
    assert parse_radix("2^62") == 1 << 62
    assert parse_radix("12345") == 12345
    assert parse_radix(" 2^59 + 2^16 ") == R8


@pytest.mark.parametrize("text", ["2^64", "2^65", "2^1+2^64", "1", "0", "abc", "3^4",
                                  "2^a+2^b", "2^-3", ""])
def test_parse_radix_rejects(text):
    with pytest.raises(ValueError):
        parse_radix(text)


# ---------------------------------------------------------------------------
# GFPV files (reference tests/test_bench_cli.py:47-87)

def test_gfpv_roundtrip(tmp_path):
    rng = random.Random(0x3C11)
    vecs = [tuple(rng.randrange(R8) for _ in range(8)) for _ in range(5)]
    path = tmp_path / "sample.gfpv"
    write_gfpv(path, 8, R8, vecs)
    assert read_gfpv(path) == (8, R8, vecs)
    k, r, arr = read_gfpv_array(path)
    assert (k, r) == (8, R8) and arr.dtype == np.uint64 and arr.shape == (5, 8)
    write_gfpv(tmp_path / "again.gfpv", 8, R8, arr)
    assert (tmp_path / "again.gfpv").read_bytes() == path.read_bytes()


def test_gfpv_empty_and_bad_rows(tmp_path):
    path = tmp_path / "empty.gfpv"
    write_gfpv(path, 16, 1 << 62, [])
    assert read_gfpv(path) == (16, 1 << 62, [])
    with pytest.raises(ValueError):
        write_gfpv(tmp_path / "bad.gfpv", 8, 1 << 62, [(1, 2, 3)])


def test_gfpv_read_errors(tmp_path):
    good = tmp_path / "good.gfpv"
    write_gfpv(good, 8, 1 << 62, [(0,) * 8])
    raw = good.read_bytes()

    def bad(data, name):
        p = tmp_path / name
        p.write_bytes(data)
        return p

    with pytest.raises(GfpvFormatError, match="bad magic"):
        read_gfpv(bad(b"NOPE" + raw[4:], "magic.gfpv"))
    with pytest.raises(GfpvFormatError, match="unsupported version"):
        read_gfpv(bad(raw[:4] + b"\x02" + raw[5:], "ver.gfpv"))
    with pytest.raises(GfpvFormatError, match="truncated header"):
        read_gfpv(bad(raw[:10], "header.gfpv"))
    with pytest.raises(GfpvFormatError, match="truncated payload"):
        read_gfpv(bad(raw[:-8], "payload.gfpv"))


def test_gfpv_reads_reference_files_byte_exact(tmp_path, golden):
    """Files written by the reference's write_gfpv parse, and re-writing
    them reproduces the same bytes."""
    g = golden["gfpv"]
    for name in ("fft256_in.gfpv", "fft256_fwd.gfpv"):
        src = os.path.join(GOLDEN, name)
        k, r, arr = read_gfpv_array(src)
        assert (k, r, arr.shape) == (8, R8, (256, 8))
        out = tmp_path / name
        write_gfpv(out, k, r, arr)
        assert out.read_bytes() == open(src, "rb").read()
    from oracle import oracle as O
    assert O.digest(read_gfpv_array(os.path.join(GOLDEN, "fft256_in.gfpv"))[2]) == g["in"]


def test_mult_count_matches_reference_formula():
    # bench_cli._mult_count values computed with the reference (K, e) -> count
    assert cli._mult_count(16, 2) == 16 * 17 * 2 + 15 * 15
    for K in (8, 16, 32, 64):
        base = {8: 5, 16: 17, 32: 49, 64: 129}[K]
        assert cli._mult_count(K, 1) == base


def test_parser_and_usage_errors(capsys):
    ap = cli.build_parser()
    a = ap.parse_args(["bench-fft", "--K", "16,32", "--e", "2,3", "--backend", "gfp-cuda"])
    assert a.K_list == [16, 32] and a.e_list == [2, 3]
    a = ap.parse_args(["bench-mul", "--k", "8,16"])
    assert a.k_list == [8, 16]
    # a bad radix is a usage error (exit code 2), reported before any GPU work
    assert main(["verify", "--k", "8", "--r", "2^a"]) == 2
    assert "bad radix syntax" in capsys.readouterr().err
    assert main(["bench-fft", "--backend", "gfp-fft"]) == 2


# ---------------------------------------------------------------------------
# the gfp-cuda commands

@pytest.mark.gpu
def test_verify_passes_and_is_deterministic(cuda, capsys):
    argv = ["verify", "--k", "8", "--r", "2^59+2^16", "--seed", "7", "--trials", "40"]
    assert main(argv) == 0
    first = capsys.readouterr().out
    assert first.count("PASS") == 8 and "FAIL" not in first
    assert "all checks passed" in first
    assert main(argv) == 0
    assert capsys.readouterr().out == first


@pytest.mark.gpu
@pytest.mark.parametrize("k", [16, 32])
def test_verify_other_k(cuda, capsys, k):
    assert main(["verify", "--k", str(k), "--trials", "16"]) == 0
    assert "all checks passed" in capsys.readouterr().out


@pytest.mark.gpu
def test_verify_rejects_oversized_radix(cuda, capsys):
    assert main(["verify", "--k", "8", "--r", "2^62", "--trials", "5"]) == 2
    assert "configuration error" in capsys.readouterr().err


@pytest.mark.gpu
def test_verify_failure_writes_counterexample(cuda, tmp_path, capsys, monkeypatch):
    import paper_1811_01490_b200 as gp
    bad = gp.gfp_encode(gp.GfpParams(R8, 8), 12345)

    def fake_checks(k, r, seed, samples):
        yield ("prime_compat", True, "forced", None)
        yield ("mul_vs_integers", False, "forced mismatch", (bad, bad))

    monkeypatch.setattr(cli, "_verify_checks", fake_checks)
    out = tmp_path / "cex.gfpv"
    assert main(["verify", "--out", str(out)]) == 1
    assert "FAIL mul_vs_integers" in capsys.readouterr().out
    assert read_gfpv(out) == (8, R8, [bad, bad])


@pytest.mark.gpu
def test_bench_fft_row(cuda):
    buf = io.StringIO()
    args = cli.build_parser().parse_args(["bench-fft", "--K", "16", "--e", "2",
                                          "--backend", "gfp-cuda", "--trials", "2"])
    assert cli.cmd_bench_fft(args, buf) == 0
    rows = list(csv.DictReader(io.StringIO(buf.getvalue())))
    assert len(rows) == 1
    row = rows[0]
    assert (row["K"], row["e"], row["backend"], row["verified"]) == ("16", "2", "gfp-cuda",
                                                                    "roundtrip")
    assert float(row["total_seconds"]) > 0 and float(row["device_seconds"]) > 0


@pytest.mark.gpu
def test_bench_mul_row(cuda):
    buf = io.StringIO()
    args = cli.build_parser().parse_args(["bench-mul", "--k", "8,32", "--trials", "4",
                                          "--batch", "4096"])
    assert cli.cmd_bench_mul(args, buf) == 0
    rows = list(csv.DictReader(io.StringIO(buf.getvalue())))
    assert [r["k"] for r in rows] == ["8", "32"]
    assert all(r["verified"] == "yes" for r in rows)


@pytest.mark.gpu
def test_fft_command_matches_reference_file(cuda, tmp_path, capsys):
    """GFPV in (written by the reference) -> forward -> GFPV out: the bytes
    equal the reference's own forward file; the inverse restores the input."""
    src = os.path.join(GOLDEN, "fft256_in.gfpv")
    want = open(os.path.join(GOLDEN, "fft256_fwd.gfpv"), "rb").read()
    out = tmp_path / "fwd.gfpv"
    assert main(["fft", "--in", src, "--out", str(out)]) == 0
    assert out.read_bytes() == want
    back = tmp_path / "back.gfpv"
    assert main(["fft", "--in", str(out), "--out", str(back), "--inverse"]) == 0
    assert back.read_bytes() == open(src, "rb").read()


@pytest.mark.gpu
def test_fft_command_rejects_bad_input(cuda, tmp_path, capsys):
    p = tmp_path / "bad.gfpv"
    write_gfpv(p, 8, R8, [(R8,) + (0,) * 7] * 256)  # digit r in form A position
    assert main(["fft", "--in", str(p), "--out", str(tmp_path / "o.gfpv")]) == 2
    assert "non-canonical" in capsys.readouterr().err
    write_gfpv(p, 8, R8, [(0,) * 8] * 100)  # not a power of K
    assert main(["fft", "--in", str(p), "--out", str(tmp_path / "o.gfpv")]) == 2


@pytest.mark.gpu
def test_polymul_command_vs_schoolbook(cuda, tmp_path):
    import paper_1811_01490_b200 as gp
    params = gp.GfpParams(R8, 8)
    p = params.p
    rng = random.Random(11)
    f = [rng.randrange(p) for _ in range(40)]
    g = [rng.randrange(p) for _ in range(25)]
    write_gfpv(tmp_path / "f.gfpv", 8, R8, [gp.gfp_encode(params, c) for c in f])
    write_gfpv(tmp_path / "g.gfpv", 8, R8, [gp.gfp_encode(params, c) for c in g])
    out = tmp_path / "h.gfpv"
    assert main(["polymul", "--in", str(tmp_path / "f.gfpv"), "--in2", str(tmp_path / "g.gfpv"),
                 "--out", str(out)]) == 0
    k, r, h = read_gfpv(out)
    want = [0] * (len(f) + len(g) - 1)
    for i, a in enumerate(f):
        for j, b in enumerate(g):
            want[i + j] = (want[i + j] + a * b) % p
    assert [gp.gfp_decode(params, t) for t in h] == want
