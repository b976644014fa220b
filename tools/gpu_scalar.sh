timeout 900 python -m pytest tests -m gpu -q -x -k "scalar or elementwise or protocol or pow or roots or twiddle or mul_fft or crt" > gpurun_out/pytest_scalar.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_scalar.log
python - <<'PY'
import time, random, sys
sys.path.insert(0, '.')
import paper_1811_01490_b200 as gp
p = gp.GfpParams((1 << 59) + (1 << 16), 8); crt = gp.crt_default()
rng = random.Random(1); xs = [gp.gfp_encode(p, rng.randrange(p.p)) for _ in range(64)]
for name, fn in (("add", lambda a, b: gp.gfp_add(p, a, b)), ("mul_fft", lambda a, b: gp.gfp_mul_fft(p, crt, a, b)), ("mul_bigint", lambda a, b: gp.gfp_mul_bigint(p, a, b))):
    for i in range(50): fn(xs[i % 64], xs[(i + 1) % 64])
    t0 = time.perf_counter()
    for i in range(1000): fn(xs[i % 64], xs[(i + 3) % 64])
    print(name, "%.1f us/call" % ((time.perf_counter() - t0) * 1e3))
PY
