"""Field-protocol driver: the reference's transform schedule, run through
an arbitrary field object's methods.

TEST INFRASTRUCTURE ONLY (never imported by the product package).  The
reference's fft.py consumes its coefficient field through a duck-typed
protocol (fft.py:13-17): add, sub, mul, pow, zero, one, inv_scalar,
root_power_mul_factory, plus the shift-capable extras shift / shift_root /
shift_root_inv / two_k (fft.py:84-103, 237-275).  This module restates the
schedule that drives those calls so a test can hand it the product's
GfpFftField and check that the object behaves, call for call, the way the
reference's transform needs -- every arithmetic call then runs on the GPU.

Schedule restated (reference file:line):
  * plan constants: omega_base = omega^(K^(e-1)), twiddle table omega^j,
    j < K^(e-1), by sequential field.mul (FftPlan.__init__, fft.py:199-214);
    shift direction from omega^(N/2k) in {shift_root, shift_root_inv}
    (build_plan, fft.py:254-267);
  * stride permutation L_m^(mn): element j*m + i -> i*n + j (fft.py:34-56);
  * base pass: the unrolled K-point step list (base_case_ops, fft.py:138-168,
    taken from the pinned C oracle) over each K-block, twiddle steps through
    root_power_mul_factory(omega_base, K) (_run_base / _base_pass,
    fft.py:171-183, 278-295);
  * level twiddles split r^a * omega^b with (a, b) = divmod(i j, m)
    (_twiddle_level_cheap, fft.py:84-103);
  * dft_general's permutation / base / twiddle cascade (fft.py:298-360) and
    dft_inverse's N^-1 scale through inv_scalar + mul (fft.py:363-370).
"""

from . import oracle as O


def permute(v, m, n, off=0):
    """L_m^(mn) on v[off : off + m n] (fft.py:34-56)."""
    if m == 1 or n == 1:
        return
    seg = v[off:off + m * n]
    out = [None] * (m * n)
    for src, x in enumerate(seg):
        j, i = divmod(src, m)
        out[i * n + j] = x
    v[off:off + m * n] = out


class ProtocolPlan:
    """Plan constants computed through the field protocol only."""

    def __init__(self, field, K, e, omega):
        self.field, self.K, self.e, self.N = field, K, e, K ** e
        self.omega = omega
        self.omega_base = field.pow(omega, K ** (e - 1))
        head = field.pow(omega, self.N // field.two_k)
        if head == field.shift_root:
            self.forward_shift = True
        elif head == field.shift_root_inv:
            self.forward_shift = False
        else:
            raise ValueError("omega^(N/2k) is neither r nor 1/r")
        table = [field.one()]
        for _ in range(K ** (e - 1) - 1):
            table.append(field.mul(table[-1], omega))
        self.table = table
        self.ops = O.base_case_ops(K)


def _base_pass(v, plan):
    f, K = plan.field, plan.K
    mul_pow = f.root_power_mul_factory(plan.omega_base, K)
    for off in range(0, plan.N, K):
        for kind, a, b in plan.ops:
            if kind == "dft2":
                x, y = v[off + a], v[off + b]
                v[off + a], v[off + b] = f.add(x, y), f.sub(x, y)
            elif kind == "tw":
                v[off + a] = mul_pow(v[off + a], b)
            else:
                v[off + a], v[off + b] = v[off + b], v[off + a]


def _level_twiddle(v, off, m, plan, stride):
    f = plan.field
    for j in range(1, plan.K):
        for i in range(1, m):
            a, b = divmod(i * j, m)
            x = v[off + j * m + i]
            if a:
                x = f.shift(x, a if plan.forward_shift else f.two_k - a)
            if b:
                x = f.mul(x, plan.table[b * stride])
            v[off + j * m + i] = x


def dft(v, plan):
    """In-place DFT of K^e points through the field protocol (fft.py:298-360)."""
    K, e, N = plan.K, plan.e, plan.N
    if len(v) != N:
        raise ValueError("vector length must equal K^e")
    for lev in range(e - 1):
        size = K ** (e - lev)
        for off in range(0, N, size):
            permute(v, K, size // K, off)
    _base_pass(v, plan)
    for lev in range(e - 2, -1, -1):
        size, m, stride = K ** (e - lev), K ** (e - lev - 1), K ** lev
        for off in range(0, N, size):
            _level_twiddle(v, off, m, plan, stride)
        for off in range(0, N, size):
            permute(v, m, K, off)
        _base_pass(v, plan)
        for off in range(0, N, size):
            permute(v, K, m, off)
    return v


def dft_inverse(v, plan):
    """DFT at omega^(N-1), then * N^-1 (fft.py:363-370)."""
    f = plan.field
    inv = ProtocolPlan(f, plan.K, plan.e, f.pow(plan.omega, plan.N - 1))
    dft(v, inv)
    n_inv = f.inv_scalar(plan.N)
    for i in range(len(v)):
        v[i] = f.mul(v[i], n_inv)
    return v
