"""CPU ORACLE for the encrypted SpMSpM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import this module.  The
product package (``paper_2604_11659_b200``) never imports it and never falls
back to it.

What it is: a restatement of the reference package ``hespmm`` for the CSR/C
path.  The limb arithmetic and every evaluation primitive live in C
(``hs_oracle.c``, loaded through ctypes); this module restates the host-side
pieces that manufacture the path's inputs (parameter chain, key generation,
encoding, encryption, decryption/decoding, masks, the pair planner) with the
same numpy RNG consumption order and float expression order as the reference,
so both paths see bit-identical inputs.

Pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors that ``tests/golden/make_golden.py`` produced by running the real
reference (``/root/reference/pkg``) in the build container.

Citations are ``file:line`` relative to ``/root/reference/pkg/src/hespmm/``.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

u64p = ctypes.POINTER(ctypes.c_uint64)


def build() -> str:
    """Compile hs_oracle.c into oracle/liboracle.so (gcc + OpenMP)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_ctx_create.restype = ctypes.c_void_p
        L.or_ctx_create.argtypes = [ctypes.c_uint, ctypes.c_uint, u64p, ctypes.c_uint64]
        L.or_ctx_destroy.argtypes = [ctypes.c_void_p]
        for name in ("or_ctx_digit_factor", "or_ctx_aux_inv", "or_ctx_n_inv", "or_ctx_mu"):
            getattr(L, name).restype = ctypes.c_uint64
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_uint]
        L.or_ctx_qlast_inv.restype = ctypes.c_uint64
        L.or_ctx_qlast_inv.argtypes = [ctypes.c_void_p, ctypes.c_uint, ctypes.c_uint]
        for name in ("or_ctx_roots", "or_ctx_roots_sh", "or_ctx_iroots", "or_ctx_iroots_sh"):
            getattr(L, name).restype = u64p
            getattr(L, name).argtypes = [ctypes.c_void_p, ctypes.c_uint]
        L.or_ctx_ntt.argtypes = [ctypes.c_void_p, u64p, ctypes.c_uint]
        L.or_ctx_intt.argtypes = [ctypes.c_void_p, u64p, ctypes.c_uint]
        L.or_find_psi.restype = ctypes.c_uint64
        L.or_find_psi.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.or_ntt.argtypes = [u64p, ctypes.c_uint, ctypes.c_uint64, u64p, u64p]
        L.or_intt.argtypes = [u64p, ctypes.c_uint, ctypes.c_uint64, u64p, u64p, ctypes.c_uint64]
        L.or_add_mod.argtypes = [u64p, u64p, u64p, ctypes.c_uint, ctypes.c_uint64]
        L.or_sub_mod.argtypes = [u64p, u64p, u64p, ctypes.c_uint, ctypes.c_uint64]
        L.or_neg_mod.argtypes = [u64p, u64p, ctypes.c_uint, ctypes.c_uint64]
        L.or_mul_mod.argtypes = [u64p, u64p, u64p, ctypes.c_uint, ctypes.c_uint64, ctypes.c_uint64]
        L.or_scalar_mul_mod.argtypes = [u64p, ctypes.c_uint64, u64p, ctypes.c_uint, ctypes.c_uint64]
        L.or_fma_mod.argtypes = [u64p, u64p, u64p, ctypes.c_uint, ctypes.c_uint64, ctypes.c_uint64]
        L.or_extend_mod.argtypes = [u64p, u64p, ctypes.c_uint, ctypes.c_uint64, ctypes.c_uint64]
        L.or_key_switch.argtypes = [ctypes.c_void_p, u64p, u64p, ctypes.c_uint, u64p, u64p]
        L.or_eval_add.argtypes = [ctypes.c_void_p, u64p, u64p, u64p, ctypes.c_uint]
        L.or_eval_mult_ct.argtypes = [ctypes.c_void_p, u64p, u64p, u64p, ctypes.c_uint]
        L.or_eval_mult_pt.argtypes = [ctypes.c_void_p, u64p, u64p, u64p, ctypes.c_uint, ctypes.c_uint]
        L.or_relinearize.argtypes = [ctypes.c_void_p, u64p, u64p, u64p, ctypes.c_uint]
        L.or_rescale.restype = ctypes.c_int
        L.or_rescale.argtypes = [ctypes.c_void_p, u64p, u64p, ctypes.c_uint, ctypes.c_uint]
        L.or_eval_rotate.argtypes = [ctypes.c_void_p, u64p, ctypes.c_uint, u64p, u64p, ctypes.c_uint]
        L.or_decrypt.argtypes = [ctypes.c_void_p, u64p, u64p, u64p, ctypes.c_uint]
        L.or_spmspm.restype = ctypes.c_int
        L.or_spmspm.argtypes = [ctypes.c_void_p, u64p, u64p, ctypes.POINTER(ctypes.c_longlong),
                                ctypes.c_longlong, ctypes.c_uint, ctypes.POINTER(u64p), u64p,
                                ctypes.POINTER(u64p), u64p, ctypes.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(u64p)


# ------------------------------------------------------------- the 9 kernels
# Same contracts as the reference seam (_kernels/__init__.py:20-28).

def ntt(a, q, roots, roots_sh):
    out = np.array(a, dtype=np.uint64, copy=True)
    lib().or_ntt(_p(out), out.shape[0], int(q), _p(np.ascontiguousarray(roots)),
                 _p(np.ascontiguousarray(roots_sh)))
    return out


def intt(a, q, iroots, iroots_sh, n_inv):
    out = np.array(a, dtype=np.uint64, copy=True)
    lib().or_intt(_p(out), out.shape[0], int(q), _p(np.ascontiguousarray(iroots)),
                  _p(np.ascontiguousarray(iroots_sh)), int(n_inv))
    return out


def _binop(fn, a, b, *extra):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.empty_like(a)
    fn(_p(a), _p(b), _p(out), a.shape[0], *extra)
    return out


def add_mod(a, b, q):
    return _binop(lib().or_add_mod, a, b, int(q))


def sub_mod(a, b, q):
    return _binop(lib().or_sub_mod, a, b, int(q))


def neg_mod(a, q):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    lib().or_neg_mod(_p(a), _p(out), a.shape[0], int(q))
    return out


def mul_mod(a, b, q, mu):
    return _binop(lib().or_mul_mod, a, b, int(q), int(mu))


def scalar_mul_mod(a, s, q):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    lib().or_scalar_mul_mod(_p(a), int(s) % int(q), _p(out), a.shape[0], int(q))
    return out


def fma_mod(acc, a, b, q, mu):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    lib().or_fma_mod(_p(acc), _p(a), _p(b), a.shape[0], int(q), int(mu))


def extend_mod(a, q_src, q_dst):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    out = np.empty_like(a)
    lib().or_extend_mod(_p(a), _p(out), a.shape[0], int(q_src), int(q_dst))
    return out


# --------------------------------------------------------------- parameters
# Restates params.py:28-205 (deterministic prime chain).

_MR = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(x: int) -> bool:
    if x < 2:
        return False
    for p in _MR:
        if x % p == 0:
            return x == p
    d, r = x - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _MR:
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(r - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


def _scan(start, step, modulus, lo, hi, exclude):
    q = start - (start - 1) % modulus
    if step > 0 and q < start:
        q += modulus
    while lo <= q <= hi:
        if q not in exclude and is_prime(q):
            return q
        q += step * modulus
    raise ValueError("no NTT-friendly prime")


@dataclass(frozen=True)
class Params:
    ring_degree: int
    modulus_chain: tuple
    scale_bits: int
    aux_prime: int
    seed: int

    @property
    def levels(self):
        return len(self.modulus_chain) - 1

    @property
    def slots(self):
        return self.ring_degree // 2

    @property
    def scale(self):
        return float(1 << self.scale_bits)


def build_params(ring_degree, scale_bits, levels, seed=2024) -> Params:
    """params.py:170-205: 60-bit base, alternating scaling primes, 60-bit aux."""
    m = 2 * ring_degree
    ex = set()
    base = _scan((1 << 60) - 1, -1, m, 1 << 59, 1 << 60, ex)
    ex.add(base)
    target = 1 << scale_bits
    chain = [base]
    for i in range(levels):
        if i % 2 == 0:
            q = _scan(target + 1, 1, m, target // 2, target * 2, ex)
        else:
            q = _scan(target - 1, -1, m, target // 2, target * 2, ex)
        ex.add(q)
        chain.append(q)
    aux = _scan((1 << 60) - 1, -1, m, 1 << 59, 1 << 60, ex)
    return Params(ring_degree, tuple(chain), scale_bits, aux, seed)


# ------------------------------------------------------------------ context

@dataclass
class Keys:
    secret: np.ndarray          # int8 coefficients
    sk_ntt: np.ndarray          # [(L+2), n] NTT of secret over chain + aux
    pk_b: np.ndarray            # [(L+1), n]
    pk_a: np.ndarray
    relin: np.ndarray           # [2, L+1, L+2, n]
    galois: dict                # normalised step -> [2, L+1, L+2, n]


class OracleContext:
    """C-backed restatement of CkksContext (context.py:23-498)."""

    SIGMA = 3.2                 # context.py:18
    HW = 32                     # context.py:19

    def __init__(self, params: Params):
        self.params = params
        n = params.ring_degree
        self.n = n
        self.L = params.levels
        self.chain = list(params.modulus_chain)
        self.aux = params.aux_prime
        self.primes = self.chain + [self.aux]
        arr = np.array(self.chain, dtype=np.uint64)
        self._h = lib().or_ctx_create(n, self.L, _p(arr), self.aux)
        if not self._h:
            raise ValueError("oracle context creation failed")
        big_q = math.prod(self.chain)
        self.big_q = big_q
        self.ksk_factor = [[(self.aux * (big_q // qi)) % qm for qm in self.chain]
                           for qi in self.chain]                     # context.py:45-48
        idx = np.arange(n)
        self._twist = np.exp(1j * np.pi * idx / n)                   # context.py:62
        exps = np.array([pow(5, j, 2 * n) for j in range(n // 2)], dtype=np.int64)
        self._slot_pos = (exps - 1) // 2
        self._conj_pos = (2 * n - exps - 1) // 2
        self._enc_rng = np.random.default_rng(
            np.random.SeedSequence(entropy=(params.seed, 0xEC)))     # context.py:68-69

    def __del__(self):
        try:
            if self._h:
                lib().or_ctx_destroy(self._h)
        except Exception:
            pass

    # ---- tables and constants
    def tables(self, p):
        n = self.n
        L = lib()
        get = lambda f: np.ctypeslib.as_array(f(self._h, p), shape=(n,)).copy()
        return dict(q=self.primes[p], roots=get(L.or_ctx_roots), roots_sh=get(L.or_ctx_roots_sh),
                    iroots=get(L.or_ctx_iroots), iroots_sh=get(L.or_ctx_iroots_sh),
                    n_inv=L.or_ctx_n_inv(self._h, p), mu=L.or_ctx_mu(self._h, p))

    def digit_factor(self, i):
        return lib().or_ctx_digit_factor(self._h, i)

    def ntt_limb(self, limb, p):
        out = np.array(limb, dtype=np.uint64, copy=True)
        lib().or_ctx_ntt(self._h, _p(out), p)
        return out

    def intt_limb(self, limb, p):
        out = np.array(limb, dtype=np.uint64, copy=True)
        lib().or_ctx_intt(self._h, _p(out), p)
        return out

    def _coeffs_to_ntt(self, coeffs, nlimbs, primes=None):
        primes = self.primes if primes is None else primes
        out = np.empty((nlimbs, self.n), dtype=np.uint64)
        for i in range(nlimbs):
            out[i] = self.ntt_limb((coeffs % self.primes[i]).astype(np.uint64), i)
        return out

    # ---- sampling (context.py:106-116)
    def _ternary(self, rng):
        h = min(self.HW, self.n // 4)
        c = np.zeros(self.n, dtype=np.int64)
        pos = rng.choice(self.n, size=h, replace=False)
        c[pos] = rng.integers(0, 2, size=h, dtype=np.int64) * 2 - 1
        return c

    def _gauss(self, rng):
        return np.rint(rng.normal(0.0, self.SIGMA, self.n)).astype(np.int64)

    # ---- keys (context.py:120-200)
    def _make_ksk(self, rng, target, sk):
        """target/sk: [(L+2), n] NTT-form; returns [2, L+1, L+2, n]."""
        L, n = self.L, self.n
        out = np.empty((2, L + 1, L + 2, n), dtype=np.uint64)
        for i in range(L + 1):
            a = np.stack([rng.integers(0, q, size=n, dtype=np.uint64) for q in self.primes])
            e = self._gauss(rng)
            for m, qm in enumerate(self.primes):
                acc = self.ntt_limb((e % qm).astype(np.uint64), m)
                if m <= L:
                    acc = add_mod(acc, scalar_mul_mod(target[m], self.ksk_factor[i][m], qm), qm)
                mu = lib().or_ctx_mu(self._h, m)
                acc = sub_mod(acc, mul_mod(a[m], sk[m], qm, mu), qm)
                out[0, i, m] = acc
            out[1, i] = a
        return out

    def keygen(self) -> Keys:
        rng = np.random.default_rng(self.params.seed)
        secret = self._ternary(rng)
        pk_a = np.stack([rng.integers(0, q, size=self.n, dtype=np.uint64) for q in self.chain])
        pk_e = self._gauss(rng)
        sk = self._coeffs_to_ntt(secret, self.L + 2)
        pk_b = np.empty_like(pk_a)
        for i, q in enumerate(self.chain):
            mu = lib().or_ctx_mu(self._h, i)
            pk_b[i] = sub_mod(self.ntt_limb((pk_e % q).astype(np.uint64), i),
                              mul_mod(pk_a[i], sk[i], q, mu), q)
        sk2 = np.stack([mul_mod(sk[p], sk[p], q, lib().or_ctx_mu(self._h, p))
                        for p, q in enumerate(self.primes)])
        relin = self._make_ksk(rng, sk2, sk)
        return Keys(secret.astype(np.int8), sk, pk_b, pk_a, relin, {})

    def perm_tables(self, g):
        n = self.n
        i = np.arange(n, dtype=np.int64)
        t = (i * g) % (2 * n)
        src = np.empty(n, dtype=np.int64)
        neg = np.empty(n, dtype=bool)
        lo = t < n
        src[t[lo]] = i[lo]
        neg[t[lo]] = False
        src[t[~lo] - n] = i[~lo]
        neg[t[~lo] - n] = True
        return src, neg

    def gen_galois_keys(self, steps, keys: Keys):
        slots = self.params.slots
        for step in steps:
            if step == 0 or abs(step) >= slots:
                raise ValueError(f"rotation step {step} out of range")
            r = step % slots
            if r in keys.galois:
                continue
            rng = np.random.default_rng(np.random.SeedSequence(entropy=(self.params.seed, 0x90, r)))
            src, neg = self.perm_tables(pow(5, r, 2 * self.n))
            sk = keys.secret.astype(np.int64)
            rotated = sk[src] * np.where(neg, -1, 1)
            target = self._coeffs_to_ntt(rotated, self.L + 2)
            keys.galois[r] = self._make_ksk(rng, target, keys.sk_ntt)
        return keys

    # ---- encode / encrypt / decrypt / decode (context.py:204-313)
    def encode_coeffs(self, values, scale=None):
        values = np.asarray(values, dtype=np.float64)
        if values.ndim != 1:
            values = values.reshape(-1)
        if scale is None:
            scale = self.params.scale
        n = self.n
        full = np.zeros(n, dtype=np.complex128)
        padded = np.zeros(self.params.slots, dtype=np.float64)
        padded[: len(values)] = values
        full[self._slot_pos] = padded * scale
        full[self._conj_pos] = padded * scale
        b = np.fft.fft(full) / n
        coeffs = np.real(b * np.conj(self._twist))
        return np.rint(coeffs).astype(np.int64)

    def encode(self, values, scale=None, level=None):
        level = self.L if level is None else level
        scale = self.params.scale if scale is None else scale
        return self._coeffs_to_ntt(self.encode_coeffs(values, scale), level + 1), float(scale), level

    def encrypt(self, pt, keys: Keys):
        limbs, scale, level = pt
        rng = self._enc_rng
        v = self._ternary(rng)
        e0 = self._gauss(rng)
        e1 = self._gauss(rng)
        nl = level + 1
        ct = np.empty((2, nl, self.n), dtype=np.uint64)
        for i in range(nl):
            q = self.chain[i]
            mu = lib().or_ctx_mu(self._h, i)
            vl = self.ntt_limb((v % q).astype(np.uint64), i)
            c0 = add_mod(mul_mod(vl, keys.pk_b[i], q, mu),
                         self.ntt_limb((e0 % q).astype(np.uint64), i), q)
            ct[0, i] = add_mod(c0, limbs[i], q)
            ct[1, i] = add_mod(mul_mod(vl, keys.pk_a[i], q, mu),
                               self.ntt_limb((e1 % q).astype(np.uint64), i), q)
        return ct, scale, level

    def decrypt(self, ct, keys: Keys, level):
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        lib().or_decrypt(self._h, _p(np.ascontiguousarray(ct)), _p(keys.sk_ntt), _p(out), level)
        return out

    def crt_to_int(self, limbs):
        """Exact centred CRT lift (context.py:244-279) as Python ints."""
        nl = len(limbs)
        coeff = [self.intt_limb(limbs[i], i) for i in range(nl)]
        qs = self.chain[:nl]
        big = math.prod(qs)
        half = big // 2
        terms = []
        for i, q in enumerate(qs):
            m = big // q
            terms.append((m * pow(m % q, -1, q), coeff[i].tolist()))
        vals = []
        for c in range(self.n):
            x = sum(t * lst[c] for t, lst in terms) % big
            vals.append(x - big if x > half else x)
        return vals

    def decode(self, limbs, scale):
        nl = len(limbs)
        if nl == 1:
            q = self.chain[0]
            v = self.intt_limb(limbs[0], 0).astype(np.int64)
            coeffs = np.where(v > q // 2, v - q, v).astype(np.float64)
        else:
            coeffs = np.array([float(x) for x in self.crt_to_int(limbs)])
        b = coeffs * self._twist
        full = np.fft.ifft(b) * self.n
        return np.real(full[self._slot_pos]) / scale

    # ---- evaluation primitives (C)
    def key_switch(self, digits, ksk, level):
        nl = level + 1
        ob = np.empty((nl, self.n), dtype=np.uint64)
        oa = np.empty_like(ob)
        lib().or_key_switch(self._h, _p(np.ascontiguousarray(digits)), _p(np.ascontiguousarray(ksk)),
                            level, _p(ob), _p(oa))
        return ob, oa

    def eval_add(self, a, b, level):
        out = np.empty((2, level + 1, self.n), dtype=np.uint64)
        lib().or_eval_add(self._h, _p(np.ascontiguousarray(a)), _p(np.ascontiguousarray(b)), _p(out), level)
        return out

    def eval_mult_ct(self, a, b, level):
        out = np.empty((3, level + 1, self.n), dtype=np.uint64)
        lib().or_eval_mult_ct(self._h, _p(np.ascontiguousarray(a)), _p(np.ascontiguousarray(b)), _p(out), level)
        return out

    def eval_mult_pt(self, ct, pt, level):
        npoly = ct.shape[0]
        out = np.empty((npoly, level + 1, self.n), dtype=np.uint64)
        lib().or_eval_mult_pt(self._h, _p(np.ascontiguousarray(ct)), _p(np.ascontiguousarray(pt)),
                              _p(out), npoly, level)
        return out

    def relinearize(self, ct3, relin, level):
        out = np.empty((2, level + 1, self.n), dtype=np.uint64)
        lib().or_relinearize(self._h, _p(np.ascontiguousarray(ct3)), _p(np.ascontiguousarray(relin)),
                             _p(out), level)
        return out

    def rescale(self, ct, level):
        npoly = ct.shape[0]
        out = np.empty((npoly, level, self.n), dtype=np.uint64)
        rc = lib().or_rescale(self._h, _p(np.ascontiguousarray(ct)), _p(out), npoly, level)
        if rc:
            raise ValueError("modulus chain exhausted: cannot rescale at level 0")
        return out

    def eval_rotate(self, ct, steps, gk_by_step, level):
        r = steps % self.params.slots
        if r == 0:
            return np.array(ct, copy=True)
        out = np.empty((2, level + 1, self.n), dtype=np.uint64)
        lib().or_eval_rotate(self._h, _p(np.ascontiguousarray(ct)), r,
                             _p(np.ascontiguousarray(gk_by_step[r])), _p(out), level)
        return out

    def spmspm(self, ct_a, ct_b, pairs, dim, masks_by_pos, keys: Keys, nthreads=0):
        """Run Algorithm 1 over ``pairs`` ((i, j, a_pos, b_pos) rows).

        Returns the result ct [2, L-1, n] or None when there are no pairs
        (engine.py:162-164)."""
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int64).reshape(-1, 4))
        npairs = pairs.shape[0]
        if npairs == 0:
            return None
        L = self.L
        mask_arrs = [np.ascontiguousarray(masks_by_pos[int(min(p[2], p[3]))]) for p in pairs]
        mask_ptrs = (u64p * npairs)(*[_p(m) for m in mask_arrs])
        slots = self.params.slots
        gal = (u64p * slots)()
        keep = []
        for r, k in keys.galois.items():
            k = np.ascontiguousarray(k)
            keep.append(k)
            gal[r] = _p(k)
        out = np.empty((2, L - 1, self.n), dtype=np.uint64)
        rc = lib().or_spmspm(self._h, _p(np.ascontiguousarray(ct_a)), _p(np.ascontiguousarray(ct_b)),
                             pairs.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), npairs, dim,
                             mask_ptrs, _p(np.ascontiguousarray(keys.relin)), gal, _p(out), nthreads)
        if rc == -2:
            raise KeyError("missing Galois key")
        if rc:
            raise ValueError(f"or_spmspm failed: {rc}")
        return out


# ------------------------------------------------------ plaintext structure
# Restates formats.py:214-233 and encmat.py:86-124, 150-186, 232-251.

def generate_random_sparse(dim, sparsity, seed):
    rng = np.random.default_rng(seed)
    vals = rng.uniform(-1.0, 1.0, size=dim * dim)
    while np.any(vals == 0.0):
        hole = vals == 0.0
        vals[hole] = rng.uniform(-1.0, 1.0, size=int(hole.sum()))
    zeros = int(math.floor(sparsity * dim * dim + 0.5))
    if zeros:
        pos = rng.choice(dim * dim, size=zeros, replace=False)
        vals[pos] = 0.0
    return vals.reshape(dim, dim)


def csr_pack(m):
    """(offsets, indices, values) of the row-wise packing (formats.dense_to_csr)."""
    rows, cols = np.nonzero(m)
    offsets = np.zeros(m.shape[0] + 1, dtype=np.int64)
    np.add.at(offsets, rows + 1, 1)
    return np.cumsum(offsets), cols.astype(np.int64), m[rows, cols]


def csc_pack(m):
    off, idx, vals = csr_pack(np.ascontiguousarray(m.T))
    return off, idx, vals


def pair_schedule_csr_csc(off_a, idx_a, off_b, idx_b, dim):
    """Two-pointer intersection per output cell, row-major (encmat.py:170-186)."""
    out = []
    for i in range(dim):
        ia = idx_a[off_a[i]:off_a[i + 1]]
        for j in range(dim):
            ib = idx_b[off_b[j]:off_b[j + 1]]
            x = y = 0
            while x < len(ia) and y < len(ib):
                if ia[x] == ib[y]:
                    out.append((i, j, int(off_a[i] + x), int(off_b[j] + y)))
                    x += 1
                    y += 1
                elif ia[x] < ib[y]:
                    x += 1
                else:
                    y += 1
    return out


def rotation_steps(pairs, dim):
    steps = set()
    for i, j, ap, bp in pairs:
        if ap != bp:
            steps.add(abs(ap - bp))
        r = min(ap, bp) - (i * dim + j)
        if r:
            steps.add(r)
    return steps


def plain_matmul(a, b):
    """Triple loop in the reference's accumulation order (oracle.py:19-33)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = a.shape[0]
    out = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            acc = 0.0
            for k in range(n):
                acc += a[i, k] * b[k, j]
            out[i, j] = acc
    return out


def frobenius_error(a, b):
    d = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    return float(np.sqrt(np.sum(d * d)))
