"""Command-line front end for the GPU path: the reference CLI's commands
(gfpfft/bench_cli.py) on the `gfp-cuda` backend, plus GFPV vector files.

    python -m paper_1811_01490_b200 bench-fft --K 16 --e 3 [--trials T] [--seed S] [--r R]
    python -m paper_1811_01490_b200 bench-mul --k 8,16,32 [--trials T]
    python -m paper_1811_01490_b200 profile-mul --k 8,16,32 [--trials T]
    python -m paper_1811_01490_b200 verify --k 8 [--trials T] [--out cex.gfpv]
    python -m paper_1811_01490_b200 fft --in x.gfpv --out y.gfpv [--inverse]
    python -m paper_1811_01490_b200 polymul --in f.gfpv --in2 g.gfpv --out h.gfpv

Same argument names, radix syntax (`2^a+2^b`), seeds, input convention
(random.Random(seed).randrange(p) then gfp_encode, bench_cli.py:369-395),
CSV headers and exit codes (2 for ValueError / ConfigurationError,
bench_cli.py:541-566) as the reference, so its bench scripts can switch the
backend string.  `verify` checks the device results against Python
integers (the reference's property suite, bench_cli.py:126-234, restricted
to the operations this package implements).  GFPV files
(bench_cli.py:88-116: magic "GFPV", u32 version 1, u64 k, u64 r, u64 count,
count x k little-endian u64 digits, element-major) are read and written
byte-compatibly, so vectors move between the two implementations.
"""

import argparse
import csv
import random
import statistics
import struct
import sys
import time

import numpy as np

DEFAULT_RADIX = {
    8: (1 << 59) + (1 << 16),
    16: (1 << 58) + (1 << 10),
    32: (1 << 56) + (1 << 21),
    64: 284903849103190610,
}

BACKENDS = ("gfp-cuda",)

_GFPV_HEADER = struct.Struct("<IQQQ")


class GfpvFormatError(ValueError):
    """Bad magic, version, or truncated GFPV payload (bench_cli.py:46-47)."""


# ---------------------------------------------------------------------------
# radix syntax (bench_cli.parse_radix, bench_cli.py:53-82)

def parse_radix(text):
    """`2^a+2^b`, `2^a-2^b`, `2^a` or a decimal integer; 2 <= r < 2^64."""
    s = text.strip().replace(" ", "")
    try:
        if "^" in s:
            if not s.startswith("2^"):
                raise ValueError
            rest = s[2:]
            for sign in ("+", "-"):
                if sign in rest:
                    a, b = rest.split(sign, 1)
                    if not b.startswith("2^"):
                        raise ValueError
                    hi, lo = 1 << int(a), 1 << int(b[2:])
                    val = hi + lo if sign == "+" else hi - lo
                    break
            else:
                val = 1 << int(rest)
        else:
            val = int(s)
    except (ValueError, IndexError):
        raise ValueError("bad radix syntax: %r" % text) from None
    if not 2 <= val < 1 << 64:
        raise ValueError("radix out of word range: %r" % text)
    return val


# ---------------------------------------------------------------------------
# GFPV files (bench_cli.py:88-116)

def write_gfpv(path, k, r, vectors):
    """Write `vectors` (k-tuples, or a uint64 array [count, k])."""
    arr = np.asarray(vectors, dtype=np.uint64) if len(vectors) else np.zeros((0, k), np.uint64)
    if arr.ndim != 2 or arr.shape[1] != k:
        raise ValueError("vector length mismatch")
    with open(path, "wb") as fh:
        fh.write(b"GFPV")
        fh.write(_GFPV_HEADER.pack(1, k, r, arr.shape[0]))
        fh.write(np.ascontiguousarray(arr).astype("<u8", copy=False).tobytes())


def read_gfpv_array(path):
    """(k, r, uint64 array [count, k]) -- the bulk form of read_gfpv."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != b"GFPV":
        raise GfpvFormatError("bad magic")
    if len(data) < 4 + _GFPV_HEADER.size:
        raise GfpvFormatError("truncated header")
    version, k, r, count = _GFPV_HEADER.unpack_from(data, 4)
    if version != 1:
        raise GfpvFormatError("unsupported version %d" % version)
    need = 4 + _GFPV_HEADER.size + count * k * 8
    if len(data) != need:
        raise GfpvFormatError("truncated payload: %d != %d bytes" % (len(data), need))
    arr = np.frombuffer(data, dtype="<u8", offset=4 + _GFPV_HEADER.size).astype(np.uint64)
    return k, r, arr.reshape(count, k)


def read_gfpv(path):
    """(k, r, list of k-tuples), like bench_cli.read_gfpv."""
    k, r, arr = read_gfpv_array(path)
    return k, r, [tuple(int(d) for d in row) for row in arr]


# ---------------------------------------------------------------------------
# helpers

def _gp():
    import paper_1811_01490_b200 as gp  # the CUDA library loads here
    return gp


def _is_probable_prime(n, rounds=40):
    """Miller-Rabin with random.Random(0) bases: the root search over a
    composite modulus never terminates (bench_cli.py:377-381)."""
    if n < 2:
        return False
    for sp in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % sp == 0:
            return n == sp
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    rng = random.Random(0)
    for _ in range(rounds):
        x = pow(rng.randrange(2, n - 1), d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _radix_for(args, k):
    r = parse_radix(args.r) if args.r else DEFAULT_RADIX.get(k)
    if r is None:
        raise ValueError("no default radix for k=%d, pass --r" % k)
    return r


def _plan_for(k, r, K, e):
    gp = _gp()
    params = gp.GfpParams(r, k)
    if not _is_probable_prime(params.p):
        raise ValueError("r^%d+1 is not prime for r=%d, transforms need a prime modulus" % (k, r))
    field = gp.GfpFftField(params, backend="cuda")
    plan = gp.build_plan(field, K, e, gp.roots_for(params, K ** e))
    return params, field, plan


def _mult_count(K, e):
    """The reference's multiplications per K^e transform (bench_cli.py:405-414):
    the r^t shifts of the unrolled base cases (base_case_ops(K) holds
    log2(K) K/2 - (K - 1) of them: 5, 17, 49, 129 for K = 8 .. 64) plus the
    general twiddle stages (unit factors skipped)."""
    base_tw = (K.bit_length() - 1) * K // 2 - (K - 1)
    N = K ** e
    total = e * (N // K) * base_tw
    for i in range(e - 1):
        m = K ** (e - i - 1)
        total += K ** i * (m - 1) * (K - 1)
    return total


def _check_canonical(arr, r):
    """Form A (all digits < r) or form B (0, ..., 0, r) per row."""
    form_a = (arr < np.uint64(r)).all(axis=1)
    form_b = (arr[:, -1] == np.uint64(r)) & (arr[:, :-1] == 0).all(axis=1)
    if not (form_a | form_b).all():
        raise ValueError("input holds a non-canonical element")


def _device_seconds(fn, reps):
    import torch
    fn()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        fn()
    t1.record()
    t1.synchronize()
    return t0.elapsed_time(t1) / 1e3 / reps


# ---------------------------------------------------------------------------
# bench-fft (bench_cli.cmd_bench_fft, bench_cli.py:417-467)

def cmd_bench_fft(args, out=None):
    out = sys.stdout if out is None else out
    gp = _gp()
    Ks = args.K_list or [16]
    es = args.e_list or [2]
    if args.backend and args.backend not in BACKENDS:
        raise ValueError("backend %r is not available here (gfp-cuda only)" % args.backend)
    trials = args.trials or 1
    w = csv.writer(out, lineterminator="\n")
    # the reference's columns (phases per fft.pass_profile), then the
    # device-resident transform time
    w.writerow(["K", "e", "backend", "total_seconds", "permutation_seconds",
                "basecase_seconds", "twiddle_seconds", "avg_mult_seconds", "verified",
                "device_seconds"])
    for K in Ks:
        for e in es:
            k = K // 2
            r = parse_radix(args.r) if args.r else DEFAULT_RADIX.get(k)
            if r is None:
                raise ValueError("no default radix for K=%d, pass --r" % K)
            params, field, plan = _plan_for(k, r, K, e)
            N = K ** e
            rng = random.Random(args.seed)
            v0 = [gp.gfp_encode(params, rng.randrange(params.p)) for _ in range(N)]
            # round trip through the drop-in API before timing
            chk = gp.dft_inverse(gp.dft_general(list(v0), plan, field), plan, field)
            verified = "roundtrip" if chk == v0 else "FAILED"
            if verified != "roundtrip":
                raise SystemExit("round trip mismatch at K=%d e=%d" % (K, e))
            total, prof = 0.0, {}
            for _ in range(trials):
                v = list(v0)
                t0 = time.perf_counter()
                gp.dft_general(v, plan, field, profile=prof)
                total += time.perf_counter() - t0
            total /= trials
            x = gp.vec.to_device(v0, k)
            y = gp.vec.empty(k, N)
            dev = _device_seconds(lambda: gp.fft_tensor(x, plan, out=y), max(3, trials))
            w.writerow([K, e, "gfp-cuda", "%.6f" % total,
                        "%.6f" % (prof.get("permutation", 0.0) / trials),
                        "%.6f" % (prof.get("basecase", 0.0) / trials),
                        "%.6f" % (prof.get("twiddle", 0.0) / trials),
                        "%.9f" % (total / _mult_count(K, e)), verified, "%.6f" % dev])
    return 0


# ---------------------------------------------------------------------------
# bench-mul (bench_cli.cmd_bench_mul, bench_cli.py:282-324)

def cmd_bench_mul(args, out=None):
    out = sys.stdout if out is None else out
    gp = _gp()
    ks = args.k_list or [8, 16, 32]
    trials = args.trials or 50
    batch = args.batch or (1 << 20)
    rng = random.Random(args.seed)
    w = csv.writer(out, lineterminator="\n")
    w.writerow(["k", "r", "cuda_call_ns", "cuda_call_median_ns", "cuda_batched_ns_per_mul",
                "batch", "verified"])
    for k in ks:
        r = _radix_for(args, k)
        params = gp.GfpParams(r, k)
        crt = gp.crt_default()
        p = params.p
        pairs = [(rng.randrange(p), rng.randrange(p)) for _ in range(trials)]
        elems = [(gp.gfp_encode(params, a), gp.gfp_encode(params, b)) for a, b in pairs]
        # cross-verify against integers before timing (bench_cli.py:301-305)
        for (a, b), (x, y) in zip(pairs, elems):
            if gp.gfp_decode(params, gp.gfp_mul_fft(params, crt, x, y)) != a * b % p:
                raise SystemExit("backend mismatch at k=%d a=%d b=%d" % (k, a, b))
        times = []
        for x, y in elems:
            t0 = time.perf_counter()
            gp.gfp_mul_fft(params, crt, x, y)
            times.append(time.perf_counter() - t0)
        xs = gp.vec.uniform(batch, params, seed=args.seed * 2 + 1)
        ys = gp.vec.uniform(batch, params, seed=args.seed * 2 + 2)
        dev = _device_seconds(lambda: gp.vec.mul(xs, ys, params), 5)
        w.writerow([k, r, round(statistics.mean(times) * 1e9),
                    round(statistics.median(times) * 1e9), "%.3f" % (dev / batch * 1e9), batch,
                    "yes"])
    return 0


# ---------------------------------------------------------------------------
# profile-mul (bench_cli.cmd_profile_mul, bench_cli.py:470-494)

def cmd_profile_mul(args, out=None):
    """Per-step percentages of the reference's multiply mechanism
    (convert_in, convolution, convert_out, crt, lhc, final), measured on the
    device: `trials` random pairs multiplied by the instrumented mechanism
    kernel in one launch (gfp_vec_mul_crt_profile: SM cycles per step),
    after a check against Python integers.  Same CSV as the reference."""
    out = sys.stdout if out is None else out
    gp = _gp()
    ks = args.k_list or [8, 16, 32, 64]
    trials = args.trials or 50
    rng = random.Random(args.seed)
    steps = gp.vec.MUL_STEPS
    w = csv.writer(out, lineterminator="\n")
    w.writerow(["k", "r"] + ["%s_pct" % s for s in steps])
    for k in ks:
        r = _radix_for(args, k)
        params = gp.GfpParams(r, k)
        gp.gfp_mult._require_compat(params, gp.crt_default())
        p = params.p
        pairs = [(rng.randrange(p), rng.randrange(p)) for _ in range(trials)]
        x = gp.vec.to_device([gp.gfp_encode(params, a) for a, _ in pairs], k)
        y = gp.vec.to_device([gp.gfp_encode(params, b) for _, b in pairs], k)
        z, cycles, _ = gp.vec.mul_crt_profile(x, y, params)
        for (a, b), t in zip(pairs, gp.vec.to_tuples(z)):
            if gp.gfp_decode(params, t) != a * b % p:
                raise SystemExit("backend mismatch at k=%d a=%d b=%d" % (k, a, b))
        total = sum(cycles.values()) or 1
        w.writerow([k, r] + ["%.2f" % (100.0 * cycles[s] / total) for s in steps])
    return 0


# ---------------------------------------------------------------------------
# verify (bench_cli._verify_checks / cmd_verify, bench_cli.py:126-234)

def _verify_checks(k, r, seed, samples):
    """Yields (name, ok, detail[, counterexample]) like the reference."""
    gp = _gp()
    rng = random.Random(seed)
    params = gp.GfpParams(r, k)
    p = params.p
    crt = gp.crt_default()
    report = gp.check_prime_compat(params, crt)
    if not report.passed:
        raise gp.ConfigurationError("; ".join(report.reasons))
    yield "prime_compat", True, "slack=%d" % report.slack

    enc = lambda n: gp.gfp_encode(params, n)  # noqa: E731
    dec = lambda x: gp.gfp_decode(params, x)  # noqa: E731
    A = [rng.randrange(p) for _ in range(samples)]
    B = [rng.randrange(p) for _ in range(samples)]
    X, Y = gp.vec.to_device([enc(a) for a in A], k), gp.vec.to_device([enc(b) for b in B], k)

    def first_bad(got, want):
        for i, (g, v) in enumerate(zip(gp.vec.to_tuples(got), want)):
            if dec(g) != v:
                return i
        return None

    i = first_bad(gp.vec.add(X, Y, params), [(a + b) % p for a, b in zip(A, B)])
    j = first_bad(gp.vec.sub(X, Y, params), [(a - b) % p for a, b in zip(A, B)])
    bad = i if i is not None else j
    yield ("add_sub_vs_integers", bad is None,
           "" if bad is None else "%s counterexample a=%d b=%d" % (
               "add" if i is not None else "sub", A[bad], B[bad]))

    ok, detail = True, ""
    for s in range(2 * k + 1):
        bad = first_bad(gp.vec.mul_pow_r(X, s, params), [a * pow(r, s, p) % p for a in A])
        if bad is not None:
            ok, detail = False, "shift counterexample a=%d i=%d" % (A[bad], s)
            break
    yield "cyclic_shift_vs_integers", ok, detail

    bad = first_bad(gp.vec.mul(X, Y, params), [a * b % p for a, b in zip(A, B)])
    yield ("mul_vs_integers", bad is None,
           "" if bad is None else "mul counterexample a=%d b=%d" % (A[bad], B[bad]),
           None if bad is None else (enc(A[bad]), enc(B[bad])))

    # the word-prime layer (gfp_mult.negacyclic_convolution over the prime
    # pair, bench_cli.py:185-194), on the device
    ok, detail = True, ""
    for ctx in (crt.p1_ctx, crt.p2_ctx):
        for _ in range(max(1, samples // 8)):
            xs = [rng.randrange(ctx.q) for _ in range(k)]
            ys = [rng.randrange(ctx.q) for _ in range(k)]
            want = [0] * k
            for i in range(k):
                for jj in range(k):
                    if i + jj < k:
                        want[i + jj] += xs[i] * ys[jj]
                    else:
                        want[i + jj - k] -= xs[i] * ys[jj]
            if list(gp.negacyclic_convolution(xs, ys, ctx, k)) != [w % ctx.q for w in want]:
                ok, detail = False, "negacyclic counterexample q=%d" % ctx.q
                break
        if not ok:
            break
    yield "negacyclic_vs_schoolbook", ok, detail

    K, e = 2 * k, 2
    N = K ** e
    _, field, plan = _plan_for(k, r, K, e)
    omega = dec(plan.omega)
    v = [rng.randrange(p) for _ in range(N)]
    got = gp.dft_general([enc(t) for t in v], plan, field)
    ok, detail = True, ""
    # X_j = sum_i v_i omega^(ij), checked on a sample of outputs (Horner)
    for jj in sorted({0, 1, N // 2, N - 1} | {rng.randrange(N) for _ in range(8)}):
        wj, acc = pow(omega, jj, p), 0
        for t in reversed(v):
            acc = (acc * wj + t) % p
        if dec(got[jj]) != acc:
            ok, detail = False, "dft counterexample N=%d j=%d" % (N, jj)
            break
    yield "dft_vs_definition", ok, detail

    back = gp.dft_inverse(list(got), plan, field)
    yield ("dft_roundtrip", [dec(t) for t in back] == v,
           "" if [dec(t) for t in back] == v else "inverse(forward(v)) != v, N=%d" % N)

    n = N // 2
    f = [rng.randrange(p) for _ in range(n)]
    g = [rng.randrange(p) for _ in range(n)]
    zero = gp.gfp_zero(params)
    prod = gp.poly_mul_list([enc(c) for c in f] + [zero] * (N - n),
                            [enc(c) for c in g] + [zero] * (N - n), plan)
    ok, detail = True, ""
    for m in sorted({0, 1, n - 1, 2 * n - 2, N - 1} | {rng.randrange(N) for _ in range(8)}):
        want = sum(f[i] * g[m - i] for i in range(max(0, m - n + 1), min(m, n - 1) + 1)) % p
        if dec(prod[m]) != want:
            ok, detail = False, "poly_mul counterexample N=%d m=%d" % (N, m)
            break
    yield "poly_mul_vs_schoolbook", ok, detail


def cmd_verify(args, out=None):
    out = sys.stdout if out is None else out
    k = args.k or 8
    r = _radix_for(args, k)
    failed, cex = 0, None
    for item in _verify_checks(k, r, args.seed, args.trials or 200):
        name, ok, detail = item[0], item[1], item[2]
        line = "%s %s" % ("PASS" if ok else "FAIL", name)
        if detail:
            line += " (%s)" % detail
        print(line, file=out)
        if not ok:
            failed += 1
            if len(item) > 3 and item[3] and cex is None:
                cex = item[3]
    print("verify: k=%d r=%d seed=%d: %s" % (
        k, r, args.seed, "all checks passed" if not failed else "%d check(s) failed" % failed),
        file=out)
    if failed and cex and args.out:
        write_gfpv(args.out, k, r, list(cex))
        print("counterexample written to %s" % args.out, file=out)
    return 1 if failed else 0


# ---------------------------------------------------------------------------
# GFPV in -> transform / product -> GFPV out (the data path either side of
# dft_general: vectors written by the reference's write_gfpv or by this CLI)

def _k_e_for(count, k, K):
    K = K or 2 * k
    e, n = 0, 1
    while n < count:
        n *= K
        e += 1
    if n != count or e < 1:
        raise ValueError("vector length %d is not a power of K=%d" % (count, K))
    return K, e


def cmd_fft(args, out=None):
    gp = _gp()
    k, r, arr = read_gfpv_array(args.inp)
    K, e = _k_e_for(arr.shape[0], k, args.K)
    params, field, plan = _plan_for(k, r, K, e)
    _check_canonical(arr, r)
    y = gp.fft_host(arr, plan, inverse=args.inverse)
    write_gfpv(args.out, k, r, y)
    print("%s: %s %d-point transform (K=%d, e=%d) -> %s" % (
        args.inp, "inverse" if args.inverse else "forward", arr.shape[0], K, e, args.out),
        file=out or sys.stdout)
    return 0


def cmd_polymul(args, out=None):
    gp = _gp()
    k, r, f = read_gfpv_array(args.inp)
    k2, r2, g = read_gfpv_array(args.inp2)
    if (k, r) != (k2, r2):
        raise ValueError("operands are over different fields")
    _check_canonical(f, r)
    _check_canonical(g, r)
    n = f.shape[0] + g.shape[0] - 1
    K = args.K or 2 * k
    N = K
    while N < n:
        N *= K
    _, e = _k_e_for(N, k, K)
    params, field, plan = _plan_for(k, r, K, e)
    h = gp.poly_mul_host(f, g, plan)
    write_gfpv(args.out, k, r, h)
    print("product of degrees %d and %d (N=%d) -> %s" % (
        f.shape[0] - 1, g.shape[0] - 1, N, args.out), file=out or sys.stdout)
    return 0


# ---------------------------------------------------------------------------
# argument plumbing (bench_cli.build_parser / main, bench_cli.py:500-566)

def _int_list(text):
    return [int(t) for t in text.split(",") if t]


def build_parser():
    ap = argparse.ArgumentParser(prog="paper_1811_01490_b200",
                                 description="GF(r^k+1) FFT on B200 (gfp-cuda backend)")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p, k_list=False):
        if k_list:
            p.add_argument("--k", dest="k_list", type=_int_list, default=None)
        else:
            p.add_argument("--k", type=int, default=None)
        p.add_argument("--r", default=None, help="radix, sparse syntax 2^a+2^b accepted")
        p.add_argument("--trials", type=int, default=None)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--out", default=None, help="output path")

    common(sub.add_parser("verify", help="property suite on the GPU path"))
    p = sub.add_parser("bench-mul", help="time the general multiply")
    common(p, k_list=True)
    p.add_argument("--batch", type=int, default=None, help="batched-throughput size")
    common(sub.add_parser("profile-mul", help="per-step multiplication profile"), k_list=True)
    p = sub.add_parser("bench-fft", help="time a K^e DFT")
    common(p)
    p.add_argument("--K", dest="K_list", type=_int_list, default=None)
    p.add_argument("--e", dest="e_list", type=_int_list, default=None)
    p.add_argument("--backend", default=None, help="gfp-cuda (the only backend here)")
    p = sub.add_parser("fft", help="transform a GFPV vector file")
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--K", type=int, default=None, help="base size (default 2k)")
    p.add_argument("--inverse", action="store_true")
    p = sub.add_parser("polymul", help="multiply two GFPV coefficient files")
    p.add_argument("--in", dest="inp", required=True)
    p.add_argument("--in2", dest="inp2", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--K", type=int, default=None)
    return ap


def main(argv=None):
    args = build_parser().parse_args(argv)
    out, opened = sys.stdout, None
    if args.command in ("bench-mul", "bench-fft", "profile-mul") and args.out:
        opened = open(args.out, "w", newline="")
        out = opened
    try:
        fn = {"verify": cmd_verify, "bench-mul": cmd_bench_mul, "bench-fft": cmd_bench_fft,
              "profile-mul": cmd_profile_mul, "fft": cmd_fft,
              "polymul": cmd_polymul}[args.command]
        return fn(args, out)
    except ValueError as exc:  # ConfigurationError and GfpvFormatError included
        kind = "configuration error" if type(exc).__name__ == "ConfigurationError" else "error"
        print("%s: %s" % (kind, exc), file=sys.stderr)
        return 2
    finally:
        if opened:
            opened.close()


if __name__ == "__main__":
    sys.exit(main())
