"""CkksContext: the reference evaluator's API over the B200 engine.

Same constructor, methods, exceptions and float bookkeeping as the
reference ``CkksContext`` (ckks/context.py:23-498).  Division of labour:

* host (numpy): every random draw, in the reference's exact consumption
  order (keygen context.py:120-148, _make_ksk :150-174, gen_galois_keys
  :176-200, encrypt :281-301), and the float canonical-embedding FFT of
  encode/decode (:204-279) -- these produce the inputs that bit-exactness
  is judged on, so they are restated draw for draw;
* device (libhespmm_b200.so, sm_100a): all limb arithmetic -- NTTs, key
  assembly, encryption/decryption products and every eval_* primitive.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import device as D
from ._lib import check, lib
from .errors import CapacityError, EvalError, KeyMissingError, ParameterError
from .params import CkksParams
from .types import Ciphertext, KeyBundle, KeySwitchKey, Plaintext

NOISE_SIGMA = 3.2
SECRET_HAMMING_WEIGHT = 32
_SCALE_MATCH_RTOL = 1e-9

# seam op codes (include/hespmm_b200.h hs_seam_op)
_ADD, _SUB, _NEG, _MUL, _SCALAR, _FMA, _EXTEND = range(7)


class CkksContext:
    """Parameters, device tables and the evaluation primitives."""

    def __init__(self, params: CkksParams, device_index: int | None = None):
        self.params = params
        n = params.ring_degree
        self._n = n
        self._chain = list(params.modulus_chain)
        self._aux = params.aux_prime
        self._L = params.levels
        if device_index is not None:
            D.set_device(device_index)
        dev = D.device()
        h = ctypes.c_void_p()
        chain = (ctypes.c_uint64 * len(self._chain))(*self._chain)
        check(lib().hs_ctx_create(ctypes.byref(h), dev.index, n, self._L, chain, self._aux))
        self._h = h
        big_q = math.prod(self._chain)
        self._big_q = big_q
        # canonical embedding tables (context.py:60-65)
        idx = np.arange(n)
        self._twist = np.exp(1j * np.pi * idx / n)
        exps = np.array([pow(5, j, 2 * n) for j in range(n // 2)], dtype=np.int64)
        self._slot_pos = (exps - 1) // 2
        self._conj_pos = (2 * n - exps - 1) // 2
        self._enc_rng = np.random.default_rng(np.random.SeedSequence(entropy=(params.seed, 0xEC)))
        self.relin_noops = 0

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().hs_ctx_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # ------------------------------------------------------------ helpers

    def _signed_ntt(self, coeffs: np.ndarray, nlimbs: int, first: int = 0) -> torch.Tensor:
        c = D.to_dev(np.ascontiguousarray(coeffs, dtype=np.int64), dtype=torch.int64)
        out = D.empty((nlimbs, self._n))
        check(lib().hs_signed_to_ntt(self._h, D.ptr(c), nlimbs, first, D.ptr(out), D.stream()))
        return out

    def _prime(self, p: int) -> int:
        return self._chain[p] if p <= self._L else self._aux

    def _limbwise(self, op: int, a: torch.Tensor, b: torch.Tensor | None, out: torch.Tensor,
                  first: int = 0) -> torch.Tensor:
        n = self._n
        for i in range(a.shape[0]):
            check(lib().hs_seam_op(op, n, D.ptr(a[i]), D.ptr(b[i]) if b is not None else None,
                                   D.ptr(out[i]), self._prime(first + i), 0, 0, D.stream()))
        return out

    def _sk_ntt(self, keys: KeyBundle) -> torch.Tensor:
        sk = keys._sk_ntt_cache.get("all")
        if sk is None:
            sk = self._signed_ntt(keys.secret.astype(np.int64), self._L + 2)
            keys._sk_ntt_cache["all"] = sk
        return sk

    def _download_key(self, kind: int, step: int) -> np.ndarray:
        L, n = self._L, self._n
        out = D.empty((2, L + 1, L + 2, n))
        lazy = kind == 1 and step in getattr(self, "_lazy_steps", ()) and \
            not lib().hs_key_has(self._h, 1, step)
        if lazy:        # materialise a lazily registered key just for the copy
            from .rng import galois_states
            st = np.ascontiguousarray(galois_states(self.params.seed, [step]))
            check(lib().hs_key_generate_galois(self._h, (ctypes.c_uint32 * 1)(step),
                                               st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                               1, D.stream()))
        check(lib().hs_key_download(self._h, kind, step, D.ptr(out), D.stream()))
        host = D.to_host(out)
        if lazy:
            check(lib().hs_key_drop(self._h, 1, step))
        return host

    def upload_key(self, kind: int, step: int, key: np.ndarray) -> KeySwitchKey:
        """Install a standard-form key [2][L+1][L+2][n] (e.g. made elsewhere)."""
        k = D.to_dev(np.ascontiguousarray(key, dtype=np.uint64))
        check(lib().hs_key_upload(self._h, kind, step, D.ptr(k), 0, D.stream()))
        D.sync()
        return KeySwitchKey(self, kind, step)

    # ------------------------------------------------------------ sampling
    # context.py:106-116

    def _sample_ternary(self, rng) -> np.ndarray:
        h = min(SECRET_HAMMING_WEIGHT, self._n // 4)
        coeffs = np.zeros(self._n, dtype=np.int64)
        pos = rng.choice(self._n, size=h, replace=False)
        coeffs[pos] = rng.integers(0, 2, size=h, dtype=np.int64) * 2 - 1
        return coeffs

    def _sample_gaussian(self, rng) -> np.ndarray:
        return np.rint(rng.normal(0.0, NOISE_SIGMA, self._n)).astype(np.int64)

    def _draw_ksk_randomness(self, rng):
        """a limbs [L+1][L+2][n] and e [L+1][n], in _make_ksk's draw order."""
        L, n = self._L, self._n
        primes = (*self._chain, self._aux)
        a = np.empty((L + 1, L + 2, n), dtype=np.uint64)
        e = np.empty((L + 1, n), dtype=np.int64)
        for i in range(L + 1):
            for m, q in enumerate(primes):
                a[i, m] = rng.integers(0, q, size=n, dtype=np.uint64)
            e[i] = self._sample_gaussian(rng)
        return a, e

    def _make_ksk(self, kind: int, step: int, rng, target: torch.Tensor,
                  sk: torch.Tensor) -> KeySwitchKey:
        a, e = self._draw_ksk_randomness(rng)
        da = D.to_dev(a)
        de = D.to_dev(e, dtype=torch.int64)
        check(lib().hs_key_generate(self._h, kind, step, D.ptr(da), D.ptr(de), D.ptr(target),
                                    D.ptr(sk), D.stream()))
        return KeySwitchKey(self, kind, step)

    # -------------------------------------------------------------- keygen

    def keygen(self) -> KeyBundle:
        """Deterministic key generation from ``params.seed`` (context.py:120-148)."""
        if self.params.levels < 2:
            raise ParameterError("insufficient depth: need at least 2 levels")
        L, n = self._L, self._n
        rng = np.random.default_rng(self.params.seed)
        secret = self._sample_ternary(rng)
        pk_a_h = np.stack([rng.integers(0, q, size=n, dtype=np.uint64) for q in self._chain])
        pk_e = self._sample_gaussian(rng)
        sk = self._signed_ntt(secret, L + 2)
        pk_a = D.to_dev(pk_a_h)
        e_ntt = self._signed_ntt(pk_e, L + 1)
        prod = self._limbwise(_MUL, pk_a, sk[: L + 1], D.empty((L + 1, n)))
        pk_b = self._limbwise(_SUB, e_ntt, prod, D.empty((L + 1, n)))
        sk2 = self._limbwise(_MUL, sk, sk, D.empty((L + 2, n)))
        relin = self._make_ksk(0, 0, rng, sk2, sk)
        bundle = KeyBundle(secret=secret.astype(np.int8), public=(pk_b, pk_a), relin=relin)
        bundle._sk_ntt_cache["all"] = sk
        return bundle

    def _perm_tables(self, g: int):
        """Coefficient automorphism X -> X^g as (src, neg) (context.py:429-445)."""
        n = self._n
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

    def _ensure_device_keygen(self, keys: KeyBundle) -> None:
        if getattr(self, "_keygen_secret", None) is keys.secret:
            return
        from .rng import ziggurat_tables
        wi, fi, ki = ziggurat_tables()
        check(lib().hs_keygen_set_tables(
            self._h, wi.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            fi.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
            ki.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
        check(lib().hs_keygen_set_secret(self._h, D.ptr(self._sk_ntt(keys)), D.stream()))
        self._keygen_secret = keys.secret

    def gen_galois_keys(self, steps, keys: KeyBundle, device=False) -> KeyBundle:
        """Rotation keys for ``steps``; per-step seeded, so order-independent
        (context.py:176-200).

        ``device=False`` draws the numpy stream on the host (the reference's
        own calls) and assembles on the GPU; ``device=True`` replays each
        step's stream on the GPU (csrc/keygen.cu, bit-identical keys);
        ``device="lazy"`` only registers the steps -- the runner generates
        each key on the GPU when it needs it and frees it afterwards (keys
        that do not fit in HBM, e.g. 8.8 TB at N=2^16, L=24).
        """
        slots = self.params.slots
        extra = {}
        todo = []
        for step in steps:
            if step == 0 or abs(step) >= slots:
                raise ParameterError(f"rotation step {step} out of range")
            r = step % slots
            if r in keys.galois or r in extra or r in todo:
                continue
            todo.append(r)
        if device and todo and min(int(q) for q in (*self.params.modulus_chain,
                                                    self.params.aux_prime)) <= 0xFFFFFFFF:
            # numpy's integers(0, q) takes its buffered 32-bit Lemire path
            # when q - 1 fits 32 bits; keygen.cu replays the 64-bit path only,
            # so such chains draw on the host (bit-identical, just slower)
            device = False
        if device and todo:
            from .rng import galois_states
            self._ensure_device_keygen(keys)
            st = np.ascontiguousarray(galois_states(self.params.seed, todo))
            arr = (ctypes.c_uint32 * len(todo))(*todo)
            stp = st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
            if device == "lazy":
                check(lib().hs_keygen_register(self._h, arr, stp, len(todo)))
                self._lazy_steps = getattr(self, "_lazy_steps", set()) | set(todo)
            else:
                check(lib().hs_key_generate_galois(self._h, arr, stp, len(todo), D.stream()))
            return keys.with_galois({r: KeySwitchKey(self, 1, r) for r in todo})
        sk = self._sk_ntt(keys)
        secret = keys.secret.astype(np.int64)
        for r in todo:
            rng = np.random.default_rng(np.random.SeedSequence(entropy=(self.params.seed, 0x90, r)))
            src, neg = self._perm_tables(pow(5, r, 2 * self._n))
            rotated = secret[src] * np.where(neg, -1, 1)
            target = self._signed_ntt(rotated, self._L + 2)
            extra[r] = self._make_ksk(1, r, rng, target, sk)
        return keys.with_galois(extra)

    # ----------------------------------------------------- encode / crypt

    def encode_coeffs(self, values, scale: float | None = None) -> np.ndarray:
        """Integer coefficients of the canonical-embedding encoding
        (context.py:222-233), float ops in the reference's order."""
        values = np.asarray(values, dtype=np.float64)
        if values.ndim != 1:
            values = values.reshape(-1)
        if len(values) > self.params.slots:
            raise CapacityError(f"{len(values)} values exceed {self.params.slots} slots")
        if scale is None:
            scale = self.params.scale
        if scale <= 0:
            raise ParameterError("encoding scale must be positive")
        n = self._n
        full = np.zeros(n, dtype=np.complex128)
        padded = np.zeros(self.params.slots, dtype=np.float64)
        padded[: len(values)] = values
        full[self._slot_pos] = padded * scale
        full[self._conj_pos] = padded * scale
        b = np.fft.fft(full) / n
        coeffs = np.real(b * np.conj(self._twist))
        peak = np.max(np.abs(coeffs)) if n else 0.0
        if peak >= 2 ** 62:
            raise CapacityError("encoded coefficients overflow 62 bits; lower the scale")
        return np.rint(coeffs).astype(np.int64)

    def encode(self, values, scale: float | None = None, level: int | None = None) -> Plaintext:
        if scale is None:
            scale = self.params.scale
        if level is None:
            level = self.params.levels
        if not 0 <= level <= self.params.levels:
            raise ParameterError(f"level {level} outside chain bounds")
        coeffs = self.encode_coeffs(values, scale)
        return Plaintext(self._signed_ntt(coeffs, level + 1), float(scale), level)

    def _intt_copy(self, data: torch.Tensor, nlimbs: int) -> torch.Tensor:
        out = data[:nlimbs].clone()
        check(lib().hs_ntt(self._h, D.ptr(out), 1, nlimbs, 0, 1, D.stream()))
        return out

    def _crt_to_float(self, limbs: torch.Tensor) -> np.ndarray:
        """Exact centred CRT lift of the coefficients, as float64 (context.py:244-279),
        on the device (csrc/decode.cu: Garner + round-half-even, bit-equal to
        the reference's Python big-int path kept below as ``_crt_to_float_host``)."""
        nl = limbs.shape[0]
        coeff = self._intt_copy(limbs, nl)
        out = torch.empty(self._n, dtype=torch.float64, device=coeff.device)
        check(lib().hs_crt_decode(self._h, D.ptr(coeff), nl, out.data_ptr(), D.stream()))
        return out.cpu().numpy()

    def _crt_to_float_host(self, limbs: torch.Tensor) -> np.ndarray:
        """The reference's big-integer decode restated on the host (test oracle)."""
        nl = limbs.shape[0]
        coeff = D.to_host(self._intt_copy(limbs, nl))
        if nl == 1:
            q = self._chain[0]
            vals = coeff[0].astype(np.int64)
            vals = np.where(vals > q // 2, vals - q, vals)
            return vals.astype(np.float64)
        qs = self._chain[:nl]
        big = math.prod(qs)
        acc = np.zeros(self._n, dtype=object)
        for i, q in enumerate(qs):
            m = big // q
            acc = acc + coeff[i].astype(object) * (m * pow(m % q, -1, q))
        acc = acc % big
        acc = np.where(acc > big // 2, acc - big, acc)
        return np.array([float(x) for x in acc], dtype=np.float64)

    def decode(self, pt: Plaintext) -> np.ndarray:
        coeffs = self._crt_to_float(self._std_data(pt))
        b = coeffs * self._twist
        full = np.fft.ifft(b) * self._n
        return np.real(full[self._slot_pos]) / pt.scale

    def _std_data(self, pt: Plaintext) -> torch.Tensor:
        if not pt.mont:
            return pt.data
        out = pt.data.clone()
        check(lib().hs_to_montgomery(self._h, D.ptr(out), 1, pt.level + 1, 0, 1, D.stream()))
        return out

    def encrypt(self, pt: Plaintext, keys: KeyBundle) -> Ciphertext:
        """Public-key encryption with fresh noise per call (context.py:281-301)."""
        rng = self._enc_rng
        v = self._sample_ternary(rng)
        e0 = self._sample_gaussian(rng)
        e1 = self._sample_gaussian(rng)
        noise = D.to_dev(np.stack([v, e0, e1]), dtype=torch.int64)
        pk_b, pk_a = keys.public
        ct = D.empty((2, pt.level + 1, self._n))
        check(lib().hs_encrypt(self._h, D.ptr(noise[0]), D.ptr(noise[1]), D.ptr(noise[2]),
                               D.ptr(pk_b), D.ptr(pk_a), D.ptr(self._std_data(pt)), pt.level,
                               D.ptr(ct), D.stream()))
        return Ciphertext(ct, pt.scale, pt.level)

    def decrypt(self, ct: Ciphertext, keys: KeyBundle) -> Plaintext:
        if ct.degree != 1:
            raise EvalError("relinearize first: cannot decrypt a degree-2 ciphertext")
        out = D.empty((ct.level + 1, self._n))
        check(lib().hs_decrypt(self._h, D.ptr(ct.data), D.ptr(self._sk_ntt(keys)), ct.level,
                               D.ptr(out), D.stream()))
        return Plaintext(out, ct.scale, ct.level)

    # ---------------------------------------------------------- arithmetic
    # context.py:317-425

    def _check_same_level(self, a, b):
        if a.level != b.level:
            raise EvalError(f"level mismatch: {a.level} != {b.level}")

    def eval_add(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        self._check_same_level(a, b)
        if abs(a.scale - b.scale) / a.scale >= _SCALE_MATCH_RTOL:
            raise EvalError(f"scale mismatch: {a.scale} vs {b.scale}")
        if a.degree != 1 or b.degree != 1:
            raise EvalError("eval_add expects degree-1 ciphertexts")
        out = D.empty((2, a.level + 1, self._n))
        check(lib().hs_eval_add(self._h, D.ptr(a.data), D.ptr(b.data), D.ptr(out), a.level,
                                D.stream()))
        return Ciphertext(out, a.scale, a.level)

    def eval_mult_ct(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        self._check_same_level(a, b)
        if a.degree != 1 or b.degree != 1:
            raise EvalError("eval_mult_ct expects degree-1 ciphertexts")
        out = D.empty((3, a.level + 1, self._n))
        check(lib().hs_eval_mult_ct(self._h, D.ptr(a.data), D.ptr(b.data), D.ptr(out), a.level,
                                    D.stream()))
        return Ciphertext(out, a.scale * b.scale, a.level)

    def eval_mult_pt(self, ct: Ciphertext, pt: Plaintext) -> Ciphertext:
        self._check_same_level(ct, pt)
        npoly = ct.degree + 1
        out = D.empty((npoly, ct.level + 1, self._n))
        check(lib().hs_eval_mult_pt(self._h, D.ptr(ct.data), D.ptr(pt.data), D.ptr(out), npoly,
                                    ct.level, 1 if pt.mont else 0, D.stream()))
        return Ciphertext(out, ct.scale * pt.scale, ct.level)

    def relinearize(self, ct: Ciphertext, keys: KeyBundle) -> Ciphertext:
        if ct.degree == 1:
            self.relin_noops += 1
            return ct
        if keys.relin is None:
            raise KeyMissingError("no relinearization key in bundle")
        out = D.empty((2, ct.level + 1, self._n))
        check(lib().hs_relinearize(self._h, D.ptr(ct.data), D.ptr(out), ct.level, D.stream()))
        return Ciphertext(out, ct.scale, ct.level)

    def rescale(self, ct: Ciphertext) -> Ciphertext:
        if ct.level == 0:
            raise EvalError("modulus chain exhausted: cannot rescale at level 0")
        lvl = ct.level
        npoly = ct.degree + 1
        out = D.empty((npoly, lvl, self._n))
        check(lib().hs_rescale(self._h, D.ptr(ct.data), D.ptr(out), npoly, lvl, D.stream()))
        return Ciphertext(out, ct.scale / self._chain[lvl], lvl - 1)

    def eval_rotate(self, ct: Ciphertext, steps: int, keys: KeyBundle) -> Ciphertext:
        """Cyclic slot rotation: output slot s holds input slot (s + steps)."""
        if ct.degree != 1:
            raise EvalError("eval_rotate expects a degree-1 ciphertext")
        r = steps % self.params.slots
        if r == 0:
            return ct
        if keys.galois.get(r) is None:
            raise KeyMissingError(f"missing Galois key for step {steps}")
        out = D.empty((2, ct.level + 1, self._n))
        made = self._materialise_lazy([r])
        try:
            check(lib().hs_eval_rotate(self._h, D.ptr(ct.data), D.ptr(out), ct.level, r, D.stream()))
        finally:
            self._drop_materialised(made)
        return Ciphertext(out, ct.scale, ct.level)

    def _materialise_lazy(self, steps) -> list:
        """Generate lazily registered Galois keys (gen_galois_keys(device=
        "lazy")) that a single eval_rotate needs; returns the steps made."""
        lazy = getattr(self, "_lazy_steps", ())
        todo = sorted({r for r in steps if r in lazy and not lib().hs_key_has(self._h, 1, r)})
        if todo:
            from .rng import galois_states
            st = np.ascontiguousarray(galois_states(self.params.seed, todo))
            check(lib().hs_key_generate_galois(self._h, (ctypes.c_uint32 * len(todo))(*todo),
                                               st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                               len(todo), D.stream()))
        return todo

    def _drop_materialised(self, steps) -> None:
        for r in steps:
            check(lib().hs_key_drop(self._h, 1, r))

    def eval_rotate_hoisted(self, ct: Ciphertext, steps, keys: KeyBundle) -> list:
        """Several rotations of one ciphertext sharing one decomposition/ModUp
        (bit-identical to repeated eval_rotate)."""
        slots = self.params.slots
        rs = [s % slots for s in steps]
        outs = []
        todo = []
        for s, r in zip(steps, rs):
            if r == 0:
                outs.append(ct)
                continue
            if keys.galois.get(r) is None:
                raise KeyMissingError(f"missing Galois key for step {s}")
            o = D.empty((2, ct.level + 1, self._n))
            outs.append(Ciphertext(o, ct.scale, ct.level))
            todo.append((r, o))
        if todo:
            ptrs = (ctypes.c_void_p * len(todo))(*[o.data_ptr() for _, o in todo])
            st = (ctypes.c_uint32 * len(todo))(*[r for r, _ in todo])
            made = self._materialise_lazy([r for r, _ in todo])
            try:
                check(lib().hs_eval_rotate_hoisted(self._h, D.ptr(ct.data), ptrs, st, len(todo),
                                                   ct.level, D.stream()))
            finally:
                self._drop_materialised(made)
        return outs


def keygen(params: CkksParams) -> KeyBundle:
    return CkksContext(params).keygen()
