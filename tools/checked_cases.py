"""Small invocations of every kernel family, run against the CHECKED build
of the library (GFPFFT_LIB=paper_1811_01490_b200/libgfpfft_checked.so, built
with GFP_DEBUG=1: every global / shared index of the pass and exchange
kernels guarded, pseudo-random per-warp delays at every phase boundary; see
gfp_device.cuh).  compute-sanitizer is not available on the GPU pool; this is
its stand-in (tests/test_checked_build.py).  Each case is compared with the
oracle, so a run that completes with no "GFP_CHECK" line proves both: no
index left its buffer and no result changed under the timing perturbation.

Cases (kernel families): k_pass44 NW = 16 / 8 / 4 and the fused-exchange
(XCH) instantiation, element-major host I/O (zero-copy first / last pass),
the four-step twiddle fold, k_exchange, k_pass<16>, k_pass<32>, the element
kernels (k_add, k_mul_pow_r, k_mul_fast, k_mul_wide, k_mul_generic, k_pow,
k_is_canonical), the mechanism multiply k_mul_crt (plain and profiled), the
word-prime transform and convolution.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_01490_b200 as gp  # noqa: E402
from oracle import oracle as O  # noqa: E402

R = {8: (1 << 59) + (1 << 16), 16: (1 << 58) + (1 << 10), 32: (1 << 56) + (1 << 21)}


def check(name, ok):
    print("%-40s %s" % (name, "ok" if ok else "MISMATCH"), flush=True)
    if not ok:
        raise SystemExit(1)


def fft_case(k, e, batch, seed):
    K = 2 * k
    N = K ** e
    params = gp.GfpParams(R[k], k)
    field = gp.GfpFftField(params, backend="cuda")
    omega = gp.roots_for(params, N)
    plan = gp.build_plan(field, K, e, omega)
    oplan = O.Plan(k, R[k], K, e, omega)
    x = O.random_elements(seed, k, R[k], N * batch).reshape(batch, N, k)
    xd = torch.stack([gp.vec.to_device(x[b], k) for b in range(batch)])
    y = gp.fft_tensor(xd, plan)
    z = gp.fft_tensor(xd, plan, inverse=True)
    ok = all(np.array_equal(gp.vec.to_host(y[b]), oplan.forward(x[b])) and
             np.array_equal(gp.vec.to_host(z[b]), oplan.inverse(x[b])) for b in range(batch))
    check("fft k=%d N=%d batch=%d" % (k, N, batch), ok)
    return params, field, plan, oplan, x


def main():
    torch.cuda.set_device(0)
    # k_pass44: NW = 16 (few CTAs), 8 (>= 148 CTAs), 4 (>= 592 CTAs)
    fft_case(8, 2, 1, 1)
    params, field, plan, oplan, x = fft_case(8, 3, 1, 2)
    fft_case(8, 3, 20, 3)
    fft_case(8, 4, 5, 4)
    # poly-mul (pointwise operand fused, N^-1) and the host paths (element-major
    # pinned zero-copy and pageable staged)
    f = np.zeros((4096, 8), dtype=np.uint64)
    g = f.copy()
    f[:2048] = x[0][:2048]
    g[:2048] = O.random_elements(9, 8, R[8], 2048)
    want = oplan.poly_mul(f, g)
    got = gp.vec.to_host(gp.poly_mul(gp.vec.to_device(f, 8), gp.vec.to_device(g, 8), plan))
    check("poly_mul k=8 N=4096", np.array_equal(got, want))
    fp = torch.from_numpy(f[:2048].copy()).pin_memory().numpy()
    gq = torch.from_numpy(g[:2048].copy()).pin_memory().numpy()
    check("poly_mul_host (pinned)", np.array_equal(gp.poly_mul_host(fp, gq, plan),
                                                   want[:4095]))
    check("poly_mul_host (pageable)", np.array_equal(gp.poly_mul_host(f[:2048], g[:2048], plan),
                                                     want[:4095]))
    check("fft_host", np.array_equal(gp.fft_host(x[0], plan), oplan.forward(x[0])))
    # sharded four-step on one device: fused twiddle, fused exchange (XCH
    # pass), standalone k_exchange, all-to-all path
    from paper_1811_01490_b200.sharded import GpuShardOps, ShardedFFT
    N1 = N2 = 256
    om = gp.roots_for(params, N1 * N2)
    ops = GpuShardOps(field, 16, N1, N2, om)
    xs = gp.vec.uniform(N1 * N2, params, seed=5)
    ref = gp.fft_tensor(xs, ops.plan_N)
    idx = ShardedFFT(ops, 8, N1, N2).gather_rows_index().reshape(-1).to("cuda")
    want_rows = ref.view(torch.int64)[:, idx].view(8, N1, N2).permute(1, 0, 2).contiguous()
    for peer, fuse in ((False, True), (True, True), (True, False)):
        sh = ShardedFFT(ops, 8, N1, N2)
        if peer:
            sh.use_peer_exchange(fuse=fuse)
        cols = sh.scatter_columns(xs)
        rows = sh.forward(cols)
        back = sh.inverse(rows)
        check("sharded peer=%s fuse=%s" % (peer, fuse),
              torch.equal(rows.view(torch.int64), want_rows) and
              torch.equal(back.view(torch.int64), cols.view(torch.int64)))
    # k_pass<16>, k_pass<32>
    fft_case(16, 2, 2, 6)
    fft_case(32, 2, 1, 7)
    # the generic-radix path (canonical radix-2 passes, k_pass_generic)
    R[-8] = (1 << 63) + (1 << 34)
    pg = gp.GfpParams(R[-8], 8)
    fg = gp.GfpFftField(pg, backend="cuda")
    om = gp.roots_for(pg, 256)
    plg = gp.build_plan(fg, 16, 2, om)
    opg = O.Plan(8, R[-8], 16, 2, np.array(om, dtype=np.uint64), backend="school")
    xg = O.random_elements(8, 8, R[-8], 256)
    check("generic radix fwd/inv",
          np.array_equal(gp.vec.to_host(gp.fft_tensor(gp.vec.to_device(xg, 8), plg)),
                         opg.forward(xg)) and
          np.array_equal(gp.vec.to_host(gp.fft_tensor(gp.vec.to_device(xg, 8), plg,
                                                      inverse=True)), opg.inverse(xg)))
    # element kernels
    for k in (8, 16, 32):
        a = O.random_elements(10 + k, k, R[k], 1000)
        b = O.random_elements(20 + k, k, R[k], 1000)
        p = gp.GfpParams(R[k], k)
        ad, bd = gp.vec.to_device(a, k), gp.vec.to_device(b, k)
        check("add/sub/shift k=%d" % k,
              np.array_equal(gp.vec.to_host(gp.vec.add(ad, bd, p)), O.add(a, b, R[k])) and
              np.array_equal(gp.vec.to_host(gp.vec.sub(ad, bd, p)), O.sub(a, b, R[k])) and
              np.array_equal(gp.vec.to_host(gp.vec.mul_pow_r(ad, 3, p)), O.mul_pow_r(a, R[k], 3)))
        prod = O.mul(a, b, R[k])
        check("mul k=%d" % k, np.array_equal(gp.vec.to_host(gp.vec.mul(ad, bd, p)), prod))
        check("mul_crt k=%d" % k, np.array_equal(gp.vec.to_host(gp.vec.mul_crt(ad, bd, p)), prod))
        z, cyc, _ = gp.vec.mul_crt_profile(ad, bd, p)
        check("mul_crt_profile k=%d" % k, np.array_equal(gp.vec.to_host(z), prod))
        check("is_canonical k=%d" % k, bool(gp.vec.is_canonical(ad, p).all()))
    p4 = gp.GfpParams((1 << 64) - (1 << 50), 4)  # generic multiply / pow (k_mul_generic, k_pow)
    a = np.array([[3, 5, 7, 11], [1, 0, 0, 0]], dtype=np.uint64)
    ad = gp.vec.to_device(a, 4)
    check("mul/pow generic radix",
          np.array_equal(gp.vec.to_host(gp.vec.mul(ad, ad, p4)),
                         O.mul(a, a, p4.r, backend="school")) and
          gp.vec.to_tuples(gp.vec.pow(ad, 5, p4))[1] == (1, 0, 0, 0))
    # word-prime transform and convolution
    ctx = gp.word_prime(gp.P1)
    wplan = gp.conv_plan(ctx, 1 << 12, False)
    xw = torch.randint(0, 1 << 40, (2, 1 << 12), device="cuda").view(torch.uint64)
    yw = torch.randint(0, 1 << 40, (2, 1 << 12), device="cuda").view(torch.uint64)
    c1 = gp.word_convolve(xw, yw, wplan)
    back = gp.word_ntt(gp.word_ntt(xw, wplan), wplan, inverse=True)
    check("word ntt round trip", torch.equal(back.view(torch.int64), xw.view(torch.int64)))
    check("word convolve runs", c1.shape == xw.shape)
    torch.cuda.synchronize()
    from paper_1811_01490_b200 import _lib
    lib = _lib.load()
    print("checked build:", lib.gfp_debug_build())
    print("all cases ok")


if __name__ == "__main__":
    main()
