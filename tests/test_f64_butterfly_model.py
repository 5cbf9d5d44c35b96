"""CPU model of the FP64-pipe NTT butterflies (csrc/ntt.cuh,
unit_butterflies_f64 / unit_butterflies_f64_inv / f64_enter / f64_leave),
checked against exact integer transforms.

Every double operation of the device code is emulated with IEEE round-to-
nearest-even semantics (Python float arithmetic for mul/add/sub, an exact
rational FMA rounded once), in the device's order, and the model asserts the
invariants the exactness argument in ntt.cuh rests on: every rint argument
below 2^51 (the 1.5*2^52 magic-constant range), every value an integer far
below 2^53, and the stage bound 1.89q.  Inputs cover the loaders' full
forward range [0, 4q) (random and constant 4q-1) for a prime at the top of
the FP64 range (q <= 2^50 + 2^40).
"""

from fractions import Fraction

import numpy as np
import pytest

MAGIC = 6755399441055744.0          # 1.5 * 2^52
F64_MAX_Q = (1 << 50) + (1 << 40)


def fma(a: float, b: float, c: float) -> float:
    return float(Fraction(a) * Fraction(b) + Fraction(c))      # exact, rounded once (RNE)


def rint_mul(a: float, b: float) -> float:
    y = Fraction(a) * Fraction(b)
    assert abs(y) < 2 ** 51, "rint argument outside the magic-constant range"
    r = fma(a, b, MAGIC) - MAGIC
    assert r == int(r)
    return r


def reduce(x: float, q: float, qinv: float) -> float:
    return fma(-rint_mul(x, qinv), q, x)


def mulmod(a: float, w: float, wq: float, q: float) -> float:
    hi = a * w
    lo = fma(a, w, -hi)
    Q = rint_mul(a, wq)
    r = fma(-Q, q, hi)
    t = r + lo
    # exactness: t is the integer a*w - Q*q
    assert Fraction(t) == Fraction(a) * Fraction(w) - Fraction(Q) * Fraction(q)
    return t


def is_prime(x: int) -> bool:
    if x < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if x % p == 0:
            return x == p
    d, s = x - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(s - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


def ntt_prime(n: int) -> int:
    q = F64_MAX_Q - (F64_MAX_Q - 1) % (2 * n)          # largest q = 1 mod 2n below the bound
    while not is_prime(q):
        q -= 2 * n
    return q


def psi_of(q: int, n: int) -> int:
    for g in range(2, 1000):
        psi = pow(g, (q - 1) // (2 * n), q)
        if pow(psi, n, q) == q - 1:
            return psi
    raise AssertionError("no root")


def brev(i: int, bits: int) -> int:
    return int(format(i, f"0{bits}b")[::-1], 2) if bits else 0


def exact_ntt(a, q, roots):
    a = list(a)
    n = len(a)
    m, t = 1, n
    while m < n:
        t //= 2
        for i in range(m):
            w = roots[m + i]
            for j in range(2 * i * t, 2 * i * t + t):
                u, v = a[j], a[j + t] * w % q
                a[j], a[j + t] = (u + v) % q, (u - v) % q
        m *= 2
    return a


def model_ntt(a, q, roots):
    """The device's FP64 forward path (first pass enter .. last pass leave),
    stages in the reference loop order (any schedule of the same butterflies
    computes the same values)."""
    qd = float(q)
    qinv = float(Fraction(1, q))                          # __drcp_rn(q)
    x = [reduce(float(v), qd, qinv) for v in a]           # f64_enter: I2F exact (< 2^53)
    n = len(x)
    bound = 0.0
    m, t, s = 1, n, 0
    while m < n:
        t //= 2
        for i in range(m):
            w = roots[m + i]
            wd, wq = float(w), float(w) / qd              # twd table {w, RN(w / q)}
            for j in range(2 * i * t, 2 * i * t + t):
                u = x[j]
                if s & 1:                                 # f64_reduce_at: odd global stages
                    u = reduce(u, qd, qinv)
                v = mulmod(x[j + t], wd, wq, qd)
                x[j], x[j + t] = u + v, u - v
                bound = max(bound, abs(x[j]), abs(x[j + t]))
        m *= 2
        s += 1
    assert bound <= 1.9 * q, bound / q
    out = []
    for v in x:                                           # f64_leave
        r = reduce(v, qd, qinv) + (qd + 2.0 ** 52)
        assert 2.0 ** 52 <= r < 2.0 ** 53
        u = int(r) - 2 ** 52
        assert q // 2 - 2 <= u <= 3 * q // 2 + 2          # [q/2, 3q/2] handed to the epilogue
        out.append(u % q)
    return out


def exact_gs(a, q, iroots):
    """Gentleman-Sande stages of the inverse NTT (without the n^-1 factor,
    which the device applies in the job's epilogue)."""
    a = list(a)
    n = len(a)
    t, m = 1, n
    while m > 1:
        h = m // 2
        j1 = 0
        for i in range(h):
            w = iroots[h + i]
            for j in range(j1, j1 + t):
                u, v = a[j], a[j + t]
                a[j], a[j + t] = (u + v) % q, (u - v) * w % q
            j1 += 2 * t
        t *= 2
        m = h
    return a


def model_gs(a, q, iroots):
    """unit_butterflies_f64_inv: x' = reduce(x + y), y' = (x - y) w mod q."""
    qd = float(q)
    qinv = float(Fraction(1, q))
    x = [reduce(float(v), qd, qinv) for v in a]
    n = len(x)
    bound = 0.0
    t, m = 1, n
    while m > 1:
        h = m // 2
        j1 = 0
        for i in range(h):
            w = iroots[h + i]
            wd, wq = float(w), float(w) / qd
            for j in range(j1, j1 + t):
                u, v = x[j], x[j + t]
                x[j] = reduce(u + v, qd, qinv)
                x[j + t] = mulmod(u - v, wd, wq, qd)
                bound = max(bound, abs(x[j]), abs(x[j + t]))
            j1 += 2 * t
        t *= 2
        m = h
    assert bound <= 0.7 * q, bound / q
    out = []
    for v in x:
        r = reduce(v, qd, qinv) + (qd + 2.0 ** 52)
        u = int(r) - 2 ** 52
        assert q // 2 - 2 <= u <= 3 * q // 2 + 2
        out.append(u % q)
    return out


@pytest.mark.parametrize("kind", ["random", "max", "alternating"])
def test_f64_inverse_gs_model_is_exact(kind):
    n, logn = 2048, 11
    q = ntt_prime(n)
    ipsi = pow(psi_of(q, n), q - 2, q)
    ipw = [pow(ipsi, k, q) for k in range(n)]
    iroots = [ipw[brev(i, logn)] for i in range(n)]
    rng = np.random.default_rng(11)
    if kind == "random":
        a = [int(v) for v in rng.integers(0, 4 * q, n, dtype=np.uint64)]
    elif kind == "max":
        a = [4 * q - 1] * n
    else:
        a = [(4 * q - 1) if k & 1 else 0 for k in range(n)]
    assert model_gs(a, q, iroots) == exact_gs([v % q for v in a], q, iroots)


@pytest.mark.parametrize("kind", ["random", "max", "alternating"])
def test_f64_forward_ntt_model_is_exact(kind):
    n, logn = 2048, 11
    q = ntt_prime(n)
    assert q <= F64_MAX_Q and q > 2 ** 50
    psi = psi_of(q, n)
    pw = [pow(psi, k, q) for k in range(n)]
    roots = [pw[brev(i, logn)] for i in range(n)]
    rng = np.random.default_rng(7)
    if kind == "random":
        a = [int(v) for v in rng.integers(0, 4 * q, n, dtype=np.uint64)]    # forward loaders: [0, 4q)
    elif kind == "max":
        a = [4 * q - 1] * n
    else:
        a = [(4 * q - 1) if k & 1 else 0 for k in range(n)]
    assert model_ntt(a, q, roots) == exact_ntt([v % q for v in a], q, roots)
