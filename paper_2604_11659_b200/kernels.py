"""The reference's kernel seam (``hespmm._kernels``, _kernels/__init__.py:20-28)
served by the sm_100a kernels.

Same nine functions, same signatures and contracts: 1-D uint64 arrays of
canonical residues, a new array returned (``fma_mod`` updates ``acc`` in
place).  Each call is one device round trip, so this seam exists for API
compatibility and per-kernel parity tests; the hot path never goes through
it (~2,800 seam calls per key switch is too fine-grained for
a GPU) -- it calls the fused batched kernels of the C-ABI instead.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as D
from ._lib import check, lib

BACKEND = "cuda-sm_100a"

_ADD, _SUB, _NEG, _MUL, _SCALAR, _FMA, _EXTEND = range(7)


def _dev(a) -> torch.Tensor:
    return D.to_dev(np.ascontiguousarray(a, dtype=np.uint64))


def _op(op, a, b, q, s=0, q_src=0):
    da = _dev(a)
    db = _dev(b) if b is not None else None
    out = torch.empty_like(da)
    check(lib().hs_seam_op(op, da.numel(), D.ptr(da), D.ptr(db), D.ptr(out), int(q), int(s),
                           int(q_src), D.stream()))
    return D.to_host(out)


def ntt(a, q, roots, roots_sh):
    """Forward negacyclic NTT, natural-order input, bit-reversed output."""
    d = _dev(a)
    r, rs = _dev(roots), _dev(roots_sh)
    check(lib().hs_seam_ntt(D.ptr(d), d.numel(), int(q), D.ptr(r), D.ptr(rs), 0, 0, D.stream()))
    return D.to_host(d)


def intt(a, q, iroots, iroots_sh, n_inv):
    d = _dev(a)
    r, rs = _dev(iroots), _dev(iroots_sh)
    check(lib().hs_seam_ntt(D.ptr(d), d.numel(), int(q), D.ptr(r), D.ptr(rs), int(n_inv), 1,
                            D.stream()))
    return D.to_host(d)


def add_mod(a, b, q):
    return _op(_ADD, a, b, q)


def sub_mod(a, b, q):
    return _op(_SUB, a, b, q)


def neg_mod(a, q):
    return _op(_NEG, a, None, q)


def mul_mod(a, b, q, mu):
    return _op(_MUL, a, b, q)


def scalar_mul_mod(a, s, q):
    return _op(_SCALAR, a, None, q, s=int(s) % int(q))


def fma_mod(acc, a, b, q, mu):
    """In-place ``acc = (acc + a*b) mod q``."""
    dacc = _dev(acc)
    da, db = _dev(a), _dev(b)
    check(lib().hs_seam_op(_FMA, da.numel(), D.ptr(da), D.ptr(db), D.ptr(dacc), int(q), 0, 0,
                           D.stream()))
    acc[:] = D.to_host(dacc)


def extend_mod(a, q_src, q_dst):
    """Centred lift of residues mod q_src into q_dst."""
    return _op(_EXTEND, a, None, q_dst, q_src=q_src)


def get_backend() -> str:
    return BACKEND
