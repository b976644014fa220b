"""Generate the golden fixtures by running the reference `gfpfft` package.

Run in the build container only (the reference lives at /root/reference and
does not travel to the GPU box):

    python tests/golden/make_golden.py [--big]

Everything written here comes from the reference's own public functions on
its own input convention (`random.Random(seed).randrange(p)` then
`gfp_encode`, as in bench_cli._fft_bench_setup, bench_cli.py:369-395) and
its own root routine (`bench_cli._gfp_root`, bench_cli.py:398-402).  The
"bigint" field backend is used for speed; the reference's own tests pin it
equal to the "fft" backend (tests/test_gfp_mult.py:249-261,
tests/test_acceptance.py:69-101).

Outputs (all under tests/golden/):
  elementwise_k{k}.npz   add/sub/mul/shift vectors per (k, r) config
  fft_small.npz          k=8 K=16 e=2 (N=256) forward + inverse vectors
  c1.npz                 C1: seed 0, k=8, N=4096 input and forward output
  fft256_{in,fwd}.gfpv   GFPV files from the reference's write_gfpv (CLI interop)
  word.npz               word-prime transforms and cyclic / negacyclic convolutions
  golden.json            roots, base-case op lists, digests of the large
                         configs (C2..C5), element-major sha256 prefixes
"""

import argparse
import hashlib
import json
import os
import random
import sys
import time
from multiprocessing import Pool

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("GFPFFT_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from gfpfft import bench_cli, fft, gfp_field, gfp_mult  # noqa: E402
from gfpfft.gfp_field import GfpParams, gfp_encode  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

DEFAULT_RADIX = bench_cli.DEFAULT_RADIX
# tests/test_gfp_field.py:15-24 (TABLE_CONFIGS + SMALL_CONFIGS) plus k=64
ELEMENTWISE_CONFIGS = [
    (8, (1 << 59) + (1 << 16)),
    (16, (1 << 58) + (1 << 10)),
    (32, (1 << 56) + (1 << 21)),
    (64, DEFAULT_RADIX[64]),
    (8, (1 << 63) + (1 << 34)),
    (4, (1 << 64) - (1 << 50)),
    (1, 4), (2, 6), (4, 10), (8, 2),
]


def digest(vec):
    """sha256 prefix over element-major little-endian u64 digits."""
    h = hashlib.sha256()
    arr = np.asarray(vec, dtype=np.uint64)
    h.update(arr.astype("<u8").tobytes())
    return h.hexdigest()[:16]


def as_array(vec, k):
    return np.array(vec, dtype=np.uint64).reshape(len(vec), k)


def draws(params, seed, n, rng=None):
    rng = rng or random.Random(seed)
    return [gfp_encode(params, rng.randrange(params.p)) for _ in range(n)]


def field_plan(k, N):
    params = GfpParams(DEFAULT_RADIX[k], k)
    field = gfp_mult.GfpFftField(params, backend="bigint")
    omega = bench_cli._gfp_root(params, N)
    plan = fft.build_plan(field, 2 * k, _log(N, 2 * k), omega)
    return params, field, plan


def _log(N, K):
    e = 0
    while N > 1:
        assert N % K == 0
        N //= K
        e += 1
    return e


# ---------------------------------------------------------------------------
# tasks (each returns (name, payload dict))

def task_elementwise(cfg):
    k, r = cfg
    params = GfpParams(r, k)
    rng = random.Random(0xE1E7 ^ k ^ (r & 0xFFFF))
    p = params.p
    vals = [0, 1, r - 1, r, p - 2, p - 1]
    vals = [v % p for v in vals]
    xs, ys = [], []
    for a in vals:
        for b in vals:
            xs.append(a)
            ys.append(b)
    n_rand = 1024 if k <= 16 else 256
    for _ in range(n_rand):
        xs.append(rng.randrange(p))
        ys.append(rng.randrange(p))
    X = [gfp_encode(params, a) for a in xs]
    Y = [gfp_encode(params, b) for b in ys]
    add = [gfp_field.gfp_add(params, x, y) for x, y in zip(X, Y)]
    sub = [gfp_field.gfp_sub(params, x, y) for x, y in zip(X, Y)]
    mul = [gfp_mult.gfp_mul_bigint(params, x, y) for x, y in zip(X, Y)]
    n_shift = min(len(X), 48)
    shifts = [[gfp_field.gfp_mul_pow_r(params, X[j], i) for i in range(2 * k + 1)]
              for j in range(n_shift)]
    out = {
        "k": np.uint64(k), "r": np.uint64(r),
        "x": as_array(X, k), "y": as_array(Y, k),
        "add": as_array(add, k), "sub": as_array(sub, k),
        "mul": as_array(mul, k),
        "shift": np.array(shifts, dtype=np.uint64).reshape(n_shift, 2 * k + 1, k),
    }
    # pow: x^e for a few exponents, reference gfp_pow with the bigint backend
    exps = [0, 1, 2, 3, 65537, (p - 1) // 2 if p > 3 else 1]
    pw = [[gfp_field.gfp_pow(params, X[j], e, gfp_mult.gfp_mul_bigint)
           for e in exps] for j in range(min(8, len(X)))]
    out["pow_exps"] = np.array([e % (1 << 64) for e in exps], dtype=np.uint64)
    out["pow_exps_text"] = np.array([str(e) for e in exps])
    out["pow"] = np.array(pw, dtype=np.uint64).reshape(len(pw), len(exps), k)
    np.savez_compressed(os.path.join(HERE, "elementwise_k%d_r%d.npz" % (k, r)), **out)
    return "elementwise_k%d_r%d" % (k, r), {"n": len(X)}


def task_roots(item):
    k, N = item
    params = GfpParams(DEFAULT_RADIX[k], k)
    g = gfp_field.gfp_find_nth_root(params, N, seed=0)
    omega = bench_cli._gfp_root(params, N)
    return "root_k%d_N%d" % (k, N), {"k": k, "N": N, "r": DEFAULT_RADIX[k],
                                       "g": [str(d) for d in g],
                                       "omega": [str(d) for d in omega],
                                       "omega_digest": digest([omega])}


def task_fft_small(_):
    params, field, plan = field_plan(8, 256)
    rng = random.Random(0xF1F0)
    vecs_in, vecs_fwd, vecs_inv = [], [], []
    for _ in range(3):
        v = draws(params, None, 256, rng)
        w = fft.dft_general(list(v), plan, field)
        u = fft.dft_inverse(list(v), plan, field)  # inverse transform of the input
        vecs_in.append(v)
        vecs_fwd.append(w)
        vecs_inv.append(u)
    np.savez_compressed(os.path.join(HERE, "fft_small.npz"),
                        x=np.array(vecs_in, dtype=np.uint64),
                        fwd=np.array(vecs_fwd, dtype=np.uint64),
                        inv=np.array(vecs_inv, dtype=np.uint64))
    return "fft_small", {"k": 8, "K": 16, "e": 2, "N": 256, "seed": 0xF1F0,
                         "count": 3}


def task_gfpv(_):
    """GFPV files written by the reference's own bench_cli.write_gfpv
    (bench_cli.py:88-97): a seed-0 k=8 K=16 e=2 input (the bench-fft input
    convention, bench_cli.py:383-394) and its forward transform -- the
    byte-level interop fixture for the CLI's `fft` command."""
    params, field, plan = field_plan(8, 256)
    v = draws(params, 0, 256)
    w = fft.dft_general(list(v), plan, field)
    bench_cli.write_gfpv(os.path.join(HERE, "fft256_in.gfpv"), 8, params.r, v)
    bench_cli.write_gfpv(os.path.join(HERE, "fft256_fwd.gfpv"), 8, params.r, w)
    return "gfpv", {"k": 8, "K": 16, "e": 2, "N": 256, "seed": 0,
                    "in": digest(v), "fwd": digest(w)}


def task_word(_):
    """The word-prime layer (word_field.py, fft.py MontField, gfp_mult.py
    convolutions) over the default prime pair: dft_general / dft_inverse on
    MontField plans at the reference's word_primitive_root, and
    cyclic / negacyclic convolutions of seeded standard-form vectors."""
    from gfpfft import word_field as W
    from gfpfft.fft import MontField
    out, meta = {}, {"transforms": [], "cyclic": [], "negacyclic": []}
    rng = random.Random(0x3D)
    for q in (W.P1, W.P2):
        ctx = W.word_prime(q)
        field = MontField(ctx)
        for K, e in [(8, 1), (8, 2), (16, 2), (32, 2), (64, 2), (8, 3), (16, 3)]:
            N = K ** e
            om = W.word_primitive_root(ctx, N)
            plan = fft.build_plan(field, K, e, om)
            v = [rng.randrange(q) for _ in range(N)]
            tag = "%d_%d_%d" % (q % 1000, K, e)
            out["dft_in_" + tag] = np.array(v, dtype=np.uint64)
            out["dft_fwd_" + tag] = np.array(fft.dft_general(list(v), plan, field), dtype=np.uint64)
            out["dft_inv_" + tag] = np.array(fft.dft_inverse(list(v), plan, field), dtype=np.uint64)
            meta["transforms"].append([q, K, e, om, tag])
        for n in (1, 2, 4, 8, 64, 128, 256, 1024, 4096):
            f = [rng.randrange(q) for _ in range(n)]
            g = [rng.randrange(q) for _ in range(n)]
            tag = "%d_%d" % (q % 1000, n)
            out["cyc_f_" + tag] = np.array(f, dtype=np.uint64)
            out["cyc_g_" + tag] = np.array(g, dtype=np.uint64)
            out["cyc_h_" + tag] = np.array(gfp_mult.cyclic_convolution(f, g, ctx, n),
                                           dtype=np.uint64)
            meta["cyclic"].append([q, n, tag])
        for k in (1, 2, 4, 8, 16, 32, 64, 128, 512):
            x = [rng.randrange(q) for _ in range(k)]
            y = [rng.randrange(q) for _ in range(k)]
            tag = "%d_%d" % (q % 1000, k)
            out["neg_x_" + tag] = np.array(x, dtype=np.uint64)
            out["neg_y_" + tag] = np.array(y, dtype=np.uint64)
            out["neg_h_" + tag] = np.array(gfp_mult.negacyclic_convolution(x, y, ctx, k),
                                           dtype=np.uint64)
            meta["negacyclic"].append([q, k, tag])
    np.savez_compressed(os.path.join(HERE, "word.npz"), **out)
    return "word", meta


def task_c1(_):
    params, field, plan = field_plan(8, 4096)
    v = draws(params, 0, 4096)
    w = fft.dft_general(list(v), plan, field)
    back = fft.dft_inverse(list(w), plan, field)
    assert back == v
    np.savez_compressed(os.path.join(HERE, "c1.npz"),
                        x=as_array(v, 8), fwd=as_array(w, 8))
    return "c1", {"k": 8, "N": 4096, "seed": 0, "input": digest(v),
                  "forward": digest(w), "roundtrip": True}


def task_c2(_):
    N = 1 << 16
    params, field, plan = field_plan(8, N)
    zero = (0,) * 8
    f = draws(params, 1, N // 2) + [zero] * (N // 2)
    g = draws(params, 2, N // 2) + [zero] * (N // 2)
    F = fft.dft_general(list(f), plan, field)
    G = fft.dft_general(list(g), plan, field)
    H = [field.mul(a, b) for a, b in zip(F, G)]
    h = fft.dft_inverse(H, plan, field)
    assert h[N - 1] == zero
    np.savez_compressed(os.path.join(HERE, "c2_head.npz"),
                        product_head=as_array(h[:256], 8),
                        product_tail=as_array(h[-256:], 8),
                        F_head=as_array(F[:256], 8))
    return "c2", {"k": 8, "N": N, "seeds": [1, 2], "f": digest(f[:N // 2]),
                  "g": digest(g[:N // 2]), "f_padded": digest(f),
                  "F": digest(F), "G": digest(G), "product": digest(h)}


def task_c3_idx0(_):
    N = 1 << 20
    params, field, plan = field_plan(16, N)
    v = draws(params, 3, N)
    t0 = time.time()
    w = fft.dft_general(list(v), plan, field)
    return "c3_idx0", {"k": 16, "N": N, "seed": 3, "batch_index": 0,
                       "input": digest(v), "forward": digest(w),
                       "forward_head": [[str(d) for d in e] for e in w[:4]],
                       "seconds": time.time() - t0}


def task_c3_idx63(_):
    # the last transform of the C3 batch: draws [63 * 2^20, 64 * 2^20) of one
    # Random(3) stream (bench_cli._fft_bench_setup convention, one stream)
    N = 1 << 20
    params, field, plan = field_plan(16, N)
    rng = random.Random(3)
    for _ in range(63 * N):
        rng.randrange(params.p)
    v = draws(params, 3, N, rng=rng)
    t0 = time.time()
    w = fft.dft_general(list(v), plan, field)
    return "c3_idx63", {"k": 16, "N": N, "seed": 3, "batch_index": 63,
                        "input": digest(v), "forward": digest(w),
                        "seconds": time.time() - t0}


def task_c3_idx(b):
    # transform b of the C3 batch: draws [b 2^20, (b + 1) 2^20) of one
    # Random(3) stream, forward by the reference's dft_general
    N = 1 << 20
    params, field, plan = field_plan(16, N)
    rng = random.Random(3)
    for _ in range(b * N):
        rng.randrange(params.p)
    v = draws(params, 3, N, rng=rng)
    t0 = time.time()
    w = fft.dft_general(list(v), plan, field)
    return "c3_idx%d" % b, {"k": 16, "N": N, "seed": 3, "batch_index": b,
                            "input": digest(v), "forward": digest(w),
                            "seconds": time.time() - t0}


def task_c4_prefix(_):
    N = 1 << 16
    params, field, plan = field_plan(8, N)
    v = draws(params, 4, N)
    w = fft.dft_general(list(v), plan, field)
    return "c4_prefix", {"k": 8, "N": N, "seed": 4, "input": digest(v),
                         "forward": digest(w)}


def task_c4_full(_):
    N = 1 << 24
    params, field, plan = field_plan(8, N)
    v = draws(params, 4, N)
    din = digest(v)
    t0 = time.time()
    w = fft.dft_general(v, plan, field)
    slice_ = w[: 1 << 16]
    np.savez_compressed(os.path.join(HERE, "c4_slice.npz"),
                        forward_slice=as_array(slice_[:1024], 8))
    return "c4_full", {"k": 8, "N": N, "seed": 4, "input": din,
                       "forward": digest(w), "forward_slice_2_16": digest(slice_),
                       "seconds": time.time() - t0}


def task_c5(_):
    k = 32
    params = GfpParams(DEFAULT_RADIX[k], k)
    rng = random.Random(5)
    n_pairs = 1 << 14
    xs, ys, zs = [], [], []
    for _ in range(n_pairs):
        a, b = rng.randrange(params.p), rng.randrange(params.p)
        x, y = gfp_encode(params, a), gfp_encode(params, b)
        xs.append(x)
        ys.append(y)
        zs.append(gfp_mult.gfp_mul_bigint(params, x, y))
    np.savez_compressed(os.path.join(HERE, "c5_mul_head.npz"),
                        x=as_array(xs[:64], k), y=as_array(ys[:64], k),
                        z=as_array(zs[:64], k))
    return "c5_mul", {"k": k, "pairs": n_pairs, "seed": 5, "x": digest(xs),
                      "y": digest(ys), "products": digest(zs)}


def task_c5_full(_):
    # all 2^22 C5 pairs through the reference's gfp_mul_bigint (gfp_mult.py:504-512)
    k = 32
    params = GfpParams(DEFAULT_RADIX[k], k)
    rng = random.Random(5)
    n_pairs = 1 << 22
    h = hashlib.sha256()
    t0 = time.time()
    for _ in range(n_pairs):
        a, b = rng.randrange(params.p), rng.randrange(params.p)
        z = gfp_mult.gfp_mul_bigint(params, gfp_encode(params, a), gfp_encode(params, b))
        h.update(np.asarray(z, dtype=np.uint64).astype("<u8").tobytes())
    return "c5_mul_full", {"k": k, "pairs": n_pairs, "seed": 5,
                           "products": h.hexdigest()[:16], "seconds": time.time() - t0}


def task_c5_fft(_):
    N = 1 << 18
    params, field, plan = field_plan(32, N)
    v = draws(params, 5, N)
    w = fft.dft_general(list(v), plan, field)
    return "c5_fft", {"k": 32, "N": N, "seed": 5, "input": digest(v),
                      "forward": digest(w)}


def task_ops(_):
    ops = {str(K): [list(op) for op in fft.base_case_ops(K)]
           for K in fft.BASE_SIZES}
    return "base_case_ops", ops


def run(task):
    fn, arg = task
    t0 = time.time()
    name, payload = fn(arg)
    print("done %-28s %.1fs" % (name, time.time() - t0), flush=True)
    return name, payload


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true",
                    help="also run C3[0], C5-FFT and the full C4 forward")
    ap.add_argument("--only", default="")
    ap.add_argument("--jobs", type=int, default=os.cpu_count())
    ap.add_argument("--c3", default="", help="extra C3 batch indices, comma-separated")
    args = ap.parse_args()
    tasks = [(task_ops, None), (task_fft_small, None), (task_gfpv, None), (task_word, None),
             (task_c1, None),
             (task_c2, None), (task_c4_prefix, None), (task_c5, None)]
    tasks += [(task_elementwise, c) for c in ELEMENTWISE_CONFIGS]
    roots = [(8, 256), (8, 4096), (8, 1 << 16), (8, 1 << 24), (16, 1 << 10),
             (16, 1 << 20), (32, 1 << 12), (32, 1 << 18), (8, 16), (16, 32),
             (32, 64), (64, 128)]
    tasks += [(task_roots, it) for it in roots]
    if args.big:
        tasks = [(task_c4_full, None), (task_c3_idx0, None), (task_c3_idx63, None),
                 (task_c5_full, None), (task_c5_fft, None)] + tasks
    if args.c3:
        tasks = [(task_c3_idx, int(b)) for b in args.c3.split(",")] + tasks
    if args.only:
        keep = set(args.only.split(","))
        tasks = [t for t in tasks if t[0].__name__ in keep]
    path = os.path.join(HERE, "golden.json")
    existing = {}
    if os.path.exists(path):
        with open(path) as fh:
            existing = json.load(fh)
    with Pool(min(args.jobs, len(tasks))) as pool:
        for name, payload in pool.imap_unordered(run, tasks):
            existing[name] = payload
            with open(path, "w") as fh:
                json.dump(existing, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
