"""Multi-GPU SpMSpM: one process per GPU, pairs sharded, one collective.

Every pair's contribution is independent given the two operands and the
keys, and the final accumulation is a modular sum (order-free).
So each rank runs a contiguous share of the step-sorted pair list
(hs_spmspm_* with shard=(rank, world)) against its full key replica and
produces a partial result ciphertext; the only exchange is one integer SUM
of those partials followed by a mod-q kernel.  world * q < 2^63 (P6), so an
int64 SUM is exact (as uint64 bits; checked: world * max q < 2^64); NCCL over NVLink moves 2(L-1) limbs per rank.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import device as D
from ._lib import check, lib
from .encmat import EncryptedResult
from .errors import ParameterError
from .engine import MaskCache, OpCounter, run_pairs
from .types import Ciphertext


def reduce_partials(partial: torch.Tensor, moduli, group=None) -> torch.Tensor:
    """Sum shard partials [2][nl][n] across ranks and reduce limb m mod q_m.

    Backend-agnostic (NCCL on GPUs, gloo in the CPU tests): the SUM runs on
    an int64 view, the reduction mod q is applied by ``mod_fn``.
    """
    flat = partial.view(torch.int64) if partial.dtype == torch.uint64 else partial
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


def host_mod(summed: np.ndarray, moduli) -> np.ndarray:
    """Reference reduction used by the CPU (gloo) tests."""
    out = summed.astype(np.uint64).copy()
    for m in range(out.shape[1]):
        out[:, m] %= np.uint64(moduli[m])
    return out


def spmm_csr_csc_distributed(enc_a, enc_b, ctx, keys, counter: OpCounter | None = None,
                             mask_cache: MaskCache | None = None, group=None) -> EncryptedResult:
    """spmm_csr_csc over all ranks of the default process group; every rank
    returns the full (bit-identical) result."""
    counter = counter if counter is not None else OpCounter()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    qmax = max(int(q) for q in ctx.params.modulus_chain)
    if world * qmax >= 1 << 64:
        # the int64 SUM of canonical partials is exact only while world*q < 2^64
        raise ParameterError(f"{world} ranks x {qmax.bit_length()}-bit moduli overflow the "
                             "64-bit partial sum")
    res = run_pairs(enc_a, enc_b, ctx, keys, counter, mask_cache, None, shard=(rank, world))
    if res.ctxt is None:
        return res
    part = res.ctxt.data
    summed = reduce_partials(part, None, group)
    L = ctx.params.levels
    check(lib().hs_reduce_mod(ctx.handle, D.ptr(summed), 2, L - 1, D.stream()))
    return EncryptedResult(Ciphertext(summed.view(torch.uint64), res.ctxt.scale, res.ctxt.level),
                           res.dim)
