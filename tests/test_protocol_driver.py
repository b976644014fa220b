"""The field-protocol driver (oracle/protocol.py) pinned on the CPU: driven by
a field object whose methods are the oracle's element functions, it must
reproduce the reference's own transform vectors (tests/golden/fft_small.npz,
written by running fft.dft_general / dft_inverse).  The GPU test
(test_gpu_protocol.py) then hands the same driver the product's
GfpFftField."""
import numpy as np

from conftest import load_npz
from oracle import oracle as O
from oracle import protocol as P

R8 = (1 << 59) + (1 << 16)


class OracleField:
    """The reference's field protocol (fft.py:13-17) over the C oracle."""

    def __init__(self, k, r):
        self.k, self.r, self.p = k, r, r ** k + 1
        self.calls = {}
        self.two_k = 2 * k
        self.shift_root = self.encode(r)
        self.shift_root_inv = self.shift(self.one(), self.two_k - 1)

    def _count(self, name):
        self.calls[name] = self.calls.get(name, 0) + 1

    def encode(self, n):
        n %= self.p
        if n == self.p - 1:
            return (0,) * (self.k - 1) + (self.r,)
        out = []
        for _ in range(self.k):
            n, d = divmod(n, self.r)
            out.append(d)
        return tuple(out)

    @staticmethod
    def _a(x):
        return np.array([x], dtype=np.uint64)

    @staticmethod
    def _t(a):
        return tuple(int(d) for d in a[0])

    def add(self, x, y):
        self._count("add")
        return self._t(O.add(self._a(x), self._a(y), self.r))

    def sub(self, x, y):
        self._count("sub")
        return self._t(O.sub(self._a(x), self._a(y), self.r))

    def mul(self, x, y):
        self._count("mul")
        return self._t(O.mul(self._a(x), self._a(y), self.r, backend="school"))

    def shift(self, x, i):
        self._count("shift")
        return self._t(O.mul_pow_r(self._a(x), self.r, i))

    def pow(self, x, e):
        acc, base = self.one(), x
        while e:
            if e & 1:
                acc = self.mul(acc, base)
            e >>= 1
            if e:
                base = self.mul(base, base)
        return acc

    def zero(self):
        return (0,) * self.k

    def one(self):
        return (1,) + (0,) * (self.k - 1)

    def inv_scalar(self, n):
        return self.encode(pow(n, -1, self.p))

    def root_power_mul_factory(self, omega, count):
        if omega == self.shift_root and count <= self.two_k:
            return lambda a, t: self.shift(a, t)
        if omega == self.shift_root_inv and count <= self.two_k:
            return lambda a, t: self.shift(a, (self.two_k - t) % self.two_k)
        table = [self.one()]
        for _ in range(count - 1):
            table.append(self.mul(table[-1], omega))
        return lambda a, t: self.mul(a, table[t])


def test_protocol_driver_reproduces_reference_vectors(golden):
    z = load_npz("fft_small.npz")
    f = OracleField(8, R8)
    omega = tuple(int(d) for d in golden["root_k8_N256"]["omega"])
    plan = P.ProtocolPlan(f, 16, 2, omega)
    assert plan.forward_shift
    for b in range(2):
        v = [tuple(int(d) for d in row) for row in z["x"][b]]
        assert P.dft(list(v), plan) == [tuple(int(d) for d in row) for row in z["fwd"][b]]
        assert P.dft_inverse(list(v), plan) == \
            [tuple(int(d) for d in row) for row in z["inv"][b]]
    # the schedule went through every protocol method the reference uses
    assert {"add", "sub", "mul", "shift"} <= set(f.calls)


def test_protocol_permutation_known_answer():
    # tests/test_fft.py:56-58
    v = list(range(8))
    P.permute(v, 2, 4)
    assert v == [0, 2, 4, 6, 1, 3, 5, 7]
