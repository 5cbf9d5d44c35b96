"""Shared helpers for the parity tests."""
import hashlib

import numpy as np


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def parse_key(key: str):
    n, sb, L, seed = (int(x) for x in key.split("_"))
    return n, sb, L, seed


def kernel_inputs(q, n, pi):
    """Inputs of make_golden.py's kernel section for prime index pi."""
    rng = np.random.default_rng(1000 + pi)
    a = rng.integers(0, q, n, dtype=np.uint64)
    b = rng.integers(0, q, n, dtype=np.uint64)
    acc = rng.integers(0, q, n, dtype=np.uint64)
    s = int(rng.integers(0, 2**62))
    return a, b, acc, s


def runner_cases(golden):
    out = []
    for key, rec in golden["runner"].items():
        n, sb, L, seed = rec["params"]
        out.append((key, n, sb, L, seed, rec["dim"], rec["sparsity"], rec["mseed"]))
    return out
