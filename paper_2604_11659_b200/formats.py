"""Plaintext sparse structure feeding the encrypted path.

Only what the hot path consumes: the layouts' traversal order (which fixes
the packed positions, encmat.py:86-124 of the reference) and the synthetic
matrix generator used by the benchmark (formats.py:209-233).  Values are
float64; structure is int64.
"""

from __future__ import annotations

import math

import numpy as np

from .errors import ParameterError

DEFAULT_SLICE_HEIGHT = 4


def as_dense(m) -> np.ndarray:
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ParameterError(f"expected a square matrix, got shape {m.shape}")
    return m


def default_slice_height(dim: int) -> int:
    return math.gcd(dim, DEFAULT_SLICE_HEIGHT)


def zero_count(dim: int, sparsity: float) -> int:
    """Zero entries for a sparsity fraction, round half up."""
    return int(math.floor(sparsity * dim * dim + 0.5))


def generate_random_sparse(dim: int, sparsity: float, seed) -> np.ndarray:
    """Uniform [-1, 1) entries (exact zeros redrawn), then ``zero_count``
    uniformly placed zeros -- the reference's draw sequence."""
    if dim < 1:
        raise ParameterError("dimension must be >= 1")
    if not 0.0 <= sparsity <= 1.0:
        raise ParameterError(f"sparsity {sparsity} outside [0, 1]")
    rng = np.random.default_rng(seed)
    vals = rng.uniform(-1.0, 1.0, size=dim * dim)
    while np.any(vals == 0.0):
        hole = vals == 0.0
        vals[hole] = rng.uniform(-1.0, 1.0, size=int(hole.sum()))
    zeros = zero_count(dim, sparsity)
    if zeros:
        vals[rng.choice(dim * dim, size=zeros, replace=False)] = 0.0
    return vals.reshape(dim, dim)


def compressed_rows(m: np.ndarray):
    """(offsets, indices, values) of the row-major nonzero traversal."""
    rows, cols = np.nonzero(m)
    offsets = np.searchsorted(rows, np.arange(m.shape[0] + 1)).astype(np.int64)
    return offsets, cols.astype(np.int64), m[rows, cols]


def vertical_entries(m: np.ndarray, g: int, by_rows: bool):
    """Slice traversal of the vertical layouts: row slices ordered (col, row)
    for VCSR, column slices ordered (row, col) for VCSC."""
    n = m.shape[0]
    if g < 1 or n % g:
        raise ParameterError(f"slice height {g} must divide the dimension {n}")
    offsets = [0]
    rr, cc = [], []
    for s in range(n // g):
        lo, hi = s * g, (s + 1) * g
        if by_rows:
            c, r = np.nonzero(m[lo:hi, :].T)
            r = r + lo
        else:
            r, c = np.nonzero(m[:, lo:hi])
            c = c + lo
        rr.append(r)
        cc.append(c)
        offsets.append(offsets[-1] + len(r))
    rows = np.concatenate(rr).astype(np.int64) if rr else np.empty(0, np.int64)
    cols = np.concatenate(cc).astype(np.int64) if cc else np.empty(0, np.int64)
    return np.array(offsets, dtype=np.int64), rows, cols, m[rows, cols]
