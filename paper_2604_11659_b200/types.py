"""Value types: plaintexts, ciphertexts and key material, resident in HBM.

Mirrors the reference's ckks/types.py:15-84 (same constructor arguments and
properties), but the limbs live in one contiguous device tensor per object:

    Plaintext.data   uint64 [level+1][n]            (NTT form)
    Ciphertext.data  uint64 [npoly][level+1][n]     (npoly 2, or 3 before relin)

``.limbs`` / ``.polys`` return the reference's tuple-of-numpy-limbs view
(a device-to-host copy) so parity checks read like the reference tests.
A ciphertext may also be built from host arrays; it is then uploaded on
first use (the end-to-end path copies host -> device inside the timed call).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as D


def _as_tensor(x) -> torch.Tensor | np.ndarray:
    if isinstance(x, torch.Tensor):
        return x
    if isinstance(x, np.ndarray):
        return x
    # tuple of limbs / tuple of tuple of limbs
    return np.ascontiguousarray(np.array(x, dtype=np.uint64))


class Plaintext:
    __slots__ = ("_data", "scale", "level", "mont", "_ctx")

    def __init__(self, limbs, scale: float, level: int, mont: bool = False, ctx=None):
        data = _as_tensor(limbs)
        if scale <= 0:
            raise ValueError("plaintext scale must be positive")
        if level < 0 or data.shape[0] != level + 1:
            raise ValueError("plaintext limbs inconsistent with level")
        self._data = data
        self.scale = float(scale)
        self.level = int(level)
        self.mont = mont          # device copy kept in Montgomery form (masks)
        self._ctx = ctx           # needed to convert a Montgomery-form copy back

    @property
    def data(self) -> torch.Tensor:
        if not isinstance(self._data, torch.Tensor) or not self._data.is_cuda:
            self._data = D.to_dev(self._data)
        return self._data

    @property
    def limbs(self) -> tuple:
        if self.mont:
            arr = D.to_host(self._ctx._std_data(self))
        else:
            arr = self._data if isinstance(self._data, np.ndarray) else D.to_host(self._data)
        return tuple(arr[i] for i in range(arr.shape[0]))


class Ciphertext:
    """2 or 3 RNS polynomials plus exact scale/level bookkeeping."""

    __slots__ = ("_data", "scale", "level")

    def __init__(self, polys, scale: float, level: int):
        data = _as_tensor(polys)
        if data.ndim != 3 or data.shape[0] not in (2, 3):
            raise ValueError("ciphertext must hold 2 or 3 polynomials")
        if scale <= 0:
            raise ValueError("ciphertext scale must be positive")
        if level < 0:
            raise ValueError("ciphertext level is negative")
        self._data = data
        self.scale = float(scale)
        self.level = int(level)

    @property
    def data(self) -> torch.Tensor:
        """Device tensor [npoly][level+1][n] (uploads host-built ciphertexts)."""
        if not isinstance(self._data, torch.Tensor) or not self._data.is_cuda:
            self._data = D.to_dev(self._data)
        return self._data

    @property
    def on_device(self) -> bool:
        return isinstance(self._data, torch.Tensor) and self._data.is_cuda

    @property
    def degree(self) -> int:
        return self._data.shape[0] - 1

    def host(self) -> np.ndarray:
        d = self._data
        if isinstance(d, torch.Tensor):
            return D.to_host(d)
        return np.asarray(d)

    @property
    def polys(self) -> tuple:
        arr = self.host()
        return tuple(tuple(arr[p, i] for i in range(arr.shape[1])) for p in range(arr.shape[0]))


class KeySwitchKey:
    """Handle of a key switching key held by the CUDA context.

    ``b[i][m]`` / ``a[i][m]`` (reference ckks/types.py:53-62) download a
    standard-form copy on demand.
    """

    __slots__ = ("_ctx", "kind", "step", "_cache")

    def __init__(self, ctx, kind: int, step: int):
        self._ctx = ctx
        self.kind = kind
        self.step = step
        self._cache = None

    def array(self) -> np.ndarray:
        """[2][L+1][L+2][n] standard form (host copy)."""
        if self._cache is None:
            self._cache = self._ctx._download_key(self.kind, self.step)
        return self._cache

    @property
    def b(self):
        a = self.array()
        return tuple(tuple(a[0, i, m] for m in range(a.shape[2])) for i in range(a.shape[1]))

    @property
    def a(self):
        a = self.array()
        return tuple(tuple(a[1, i, m] for m in range(a.shape[2])) for i in range(a.shape[1]))


@dataclass(frozen=True)
class KeyBundle:
    """Secret/public/relinearisation keys plus generated rotation keys
    (reference ckks/types.py:65-84)."""

    secret: np.ndarray                       # int8 coefficients in {-1, 0, 1}
    public: tuple                            # (pk_b, pk_a) device tensors [L+1][n]
    relin: KeySwitchKey | None
    galois: dict = field(default_factory=dict)
    _sk_ntt_cache: dict = field(default_factory=dict, repr=False, compare=False)

    def with_galois(self, extra: dict) -> "KeyBundle":
        merged = dict(self.galois)
        merged.update(extra)
        return KeyBundle(self.secret, self.public, self.relin, merged, self._sk_ntt_cache)
