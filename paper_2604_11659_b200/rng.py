"""Host side of the on-device key generation: numpy stream states and tables.

The reference derives every Galois key from its own numpy stream
``default_rng(SeedSequence(entropy=(seed, 0x90, r)))`` (ckks/context.py:190-191).
The device replays that stream (csrc/keygen.cu); the host supplies

* the PCG64 state *before the first draw* for each step -- taken from numpy
  itself (``PCG64(SeedSequence(...)).state``), so SeedSequence hashing is
  numpy's own;
* numpy's ziggurat tables (``wi``, ``fi``, ``ki`` of random_standard_normal),
  read from the installed numpy binary (the constants are not exposed in
  Python) and validated here by replaying numpy draws before use.
"""

from __future__ import annotations

import glob
import math
import os
import struct
from functools import lru_cache

import numpy as np

from .errors import ParameterError

_MASK64 = (1 << 64) - 1
_PCG_MULT = (2549297995355413924 << 64) + 4865540595714422341


def pcg_state(entropy) -> tuple:
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy's PCG64 for a SeedSequence."""
    st = np.random.PCG64(np.random.SeedSequence(entropy=entropy)).state["state"]
    s, inc = st["state"], st["inc"]
    return (s >> 64, s & _MASK64, inc >> 64, inc & _MASK64)


def galois_states(seed: int, steps) -> np.ndarray:
    """[len(steps), 4] uint64 start states of the per-step key streams."""
    out = np.empty((len(steps), 4), dtype=np.uint64)
    for k, r in enumerate(steps):
        out[k] = pcg_state((seed, 0x90, int(r)))
    return out


# ------------------------------------------------------------- ziggurat

_ZIG_R = 3.6541528853610088
_ZIG_INV_R = 0.27366123732975828


def _pcg_next(st):
    st[0] = (st[0] * _PCG_MULT + st[1]) & ((1 << 128) - 1)
    s = st[0]
    hi, lo = s >> 64, s & _MASK64
    x, rot = hi ^ lo, hi >> 58
    return ((x >> rot) | (x << ((64 - rot) & 63))) & _MASK64


def _replay_normal(st, wi, fi, ki):
    """One random_standard_normal draw (numpy distributions.c), pure Python."""
    while True:
        r = _pcg_next(st)
        idx = r & 0xFF
        r >>= 8
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if r & 1:
            x = -x
        if rabs < ki[idx]:
            return x
        if idx == 0:
            while True:
                xx = -_ZIG_INV_R * math.log1p(-((_pcg_next(st) >> 11) / 9007199254740992.0))
                yy = -math.log1p(-((_pcg_next(st) >> 11) / 9007199254740992.0))
                if yy + yy > xx * xx:
                    return -(_ZIG_R + xx) if (rabs >> 8) & 1 else _ZIG_R + xx
        elif (fi[idx - 1] - fi[idx]) * ((_pcg_next(st) >> 11) / 9007199254740992.0) + fi[idx] < \
                math.exp(-0.5 * x * x):
            return x


@lru_cache(maxsize=1)
def ziggurat_tables():
    """(wi, fi, ki) as float64/float64/uint64 arrays of 256, validated."""
    d = os.path.dirname(np.random.__file__)
    cands = glob.glob(os.path.join(d, "_generator*.so")) + glob.glob(os.path.join(d, "_generator*.pyd"))
    if not cands:
        raise ParameterError("numpy.random._generator binary not found")
    blob = open(cands[0], "rb").read()
    # ki[0] and the first entries of wi/fi are fixed constants of the
    # 256-layer ziggurat (numpy ziggurat_constants.h); locate the arrays.
    ki_off = blob.find(struct.pack("<Q", 0x000EF33D8025EF6A))
    wi_off = blob.find(struct.pack("<d", 8.68362706080130616677e-16))
    fi_off = blob.find(struct.pack("<d", 1.0) + struct.pack("<d", 9.77101701267671596263e-01))
    if min(ki_off, wi_off, fi_off) < 0:
        raise ParameterError("ziggurat tables not found in the numpy binary")
    wi = np.frombuffer(blob[wi_off:wi_off + 2048], dtype="<f8").copy()
    fi = np.frombuffer(blob[fi_off:fi_off + 2048], dtype="<f8").copy()
    ki = np.frombuffer(blob[ki_off:ki_off + 2048], dtype="<u8").copy()
    # validate: replay numpy's normal() for a stream long enough to hit slow paths
    g = np.random.default_rng(np.random.SeedSequence(entropy=(12345, 0x21)))
    want = g.normal(0.0, 3.2, 4000)
    s = np.random.PCG64(np.random.SeedSequence(entropy=(12345, 0x21))).state["state"]
    st = [s["state"], s["inc"]]
    wl, fl, kl = wi.tolist(), fi.tolist(), [int(x) for x in ki]
    got = np.array([0.0 + 3.2 * _replay_normal(st, wl, fl, kl) for _ in range(4000)])
    if not np.array_equal(want, got):
        raise ParameterError("extracted ziggurat tables do not reproduce numpy's normal()")
    return wi, fi, ki
