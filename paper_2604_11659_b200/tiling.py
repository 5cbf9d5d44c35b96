"""Multi-ciphertext tiling: encrypted SpMSpM beyond one ciphertext's slots.

SURVEY.md §8(f) rank 3.  The reference packs a whole N x N matrix into one
ciphertext and raises ``CapacityError`` when the packing needs more than
``slots`` positions (hespmm/encmat.py:131-133, hespmm/engine.py:93-96), so
BASELINE configs[3] (256 x 256 at N = 2^16, 32,768 slots) and configs[4]
(512 x 512 at N = 2^17) do not run there.  Here the matrix is cut into a
T x T grid of b x b blocks (b = ceil(N / T), the smallest T with b^2 <= slots,
zero padding at the edges); every structurally non-empty block is its own
CSR (left operand) or CSC (right operand) ciphertext, and

    C[I][J] = sum_K A[I][K] B[K][J]

is evaluated block by block: each block product is an ordinary CSR/C
SpMSpM of dimension b on the engine (``engine.spmm_csr_csc``, bit-identical
to the untiled runner on that block pair), and the partial products of one
output block are added with ``eval_add``.  Empty blocks are skipped: the
sparsity structure is public metadata, as it is in the reference
(``SparseMeta`` offsets/indices travel in the clear).

Beyond the reference's capacity, so parity is against the plaintext product
(decrypted Frobenius error), plus bit-equality of each block product with a
direct ``spmm_csr_csc`` call on the same block ciphertexts
(tests/test_gpu_tiling.py).  Multi-GPU: pass ``spmm=dist.spmm_csr_csc_distributed``
to shard every block product's pairs across ranks.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import formats
from .encmat import EncryptedResult, Layout, decrypt_result, encrypt_sparse, required_rotation_steps
from .errors import ParameterError


def tile_grid(n: int, slots: int) -> tuple[int, int]:
    """(T, b): the fewest blocks per side whose b x b packing fits ``slots``."""
    if n <= 0:
        raise ParameterError("matrix dimension must be positive")
    T = 1
    while True:
        b = -(-n // T)
        if b * b <= slots:
            return T, b
        T += 1


def split_blocks(m, T: int) -> tuple[dict, int]:
    """{(I, K): b x b dense block} of the non-empty blocks, and b."""
    m = formats.as_dense(m)
    n = m.shape[0]
    if m.shape != (n, n):
        raise ParameterError("square matrices only")
    b = -(-n // T)
    pad = np.zeros((T * b, T * b), dtype=np.float64)
    pad[:n, :n] = m
    blocks = {}
    for I in range(T):
        for K in range(T):
            blk = pad[I * b:(I + 1) * b, K * b:(K + 1) * b]
            if np.count_nonzero(blk):
                blocks[(I, K)] = np.ascontiguousarray(blk)
    return blocks, b


@dataclass
class TiledMatrix:
    """An N x N matrix as a T x T grid of encrypted b x b blocks."""

    n: int
    T: int
    b: int
    layout: Layout
    tiles: dict = field(default_factory=dict)      # (I, K) -> EncryptedSparseMatrix


@dataclass
class TiledResult:
    n: int
    T: int
    b: int
    tiles: dict = field(default_factory=dict)      # (I, J) -> EncryptedResult


def encrypt_tiled(m, layout: Layout, ctx, keys, T: int | None = None) -> TiledMatrix:
    """Encrypt every non-empty block (CSR for the left operand, CSC for the
    right one), in row-major block order."""
    if layout not in (Layout.CSR, Layout.CSC):
        raise ParameterError("tiling supports the CSR/C method (CSR x CSC)")
    m = formats.as_dense(m)
    n = m.shape[0]
    if T is None:
        T, _ = tile_grid(n, ctx.params.slots)
    blocks, b = split_blocks(m, T)
    if b * b > ctx.params.slots:
        raise ParameterError(f"block side {b} needs {b * b} slots, only {ctx.params.slots}")
    out = TiledMatrix(n=n, T=T, b=b, layout=layout)
    for key in sorted(blocks):
        out.tiles[key] = encrypt_sparse(blocks[key], layout, ctx, keys)
    return out


def block_products(ta: TiledMatrix, tb: TiledMatrix):
    """(I, K, J) triples whose block product is structurally non-empty."""
    if (ta.n, ta.T, ta.b) != (tb.n, tb.T, tb.b):
        raise ParameterError("operand tilings differ")
    out = []
    for (I, K) in sorted(ta.tiles):
        for J in range(tb.T):
            if (K, J) in tb.tiles:
                out.append((I, K, J))
    return out


def required_rotation_steps_tiled(ta: TiledMatrix, tb: TiledMatrix) -> set:
    steps = set()
    for I, K, J in block_products(ta, tb):
        steps |= required_rotation_steps(ta.tiles[(I, K)].meta, tb.tiles[(K, J)].meta)
    return steps


def spmm_tiled(ta: TiledMatrix, tb: TiledMatrix, ctx, keys, counter=None, mask_cache=None,
               spmm=None) -> TiledResult:
    """Block SpMSpM.  Default: ONE runner call for every output block
    C[I][J] and all its products A[I][K] x B[K][J] (engine.run_blocks:
    hs_spmspm_multi schedules all pairs together, so a Galois key is
    generated once per step for the whole product, and each block's sum is
    the runner's own modular accumulation).  With ``spmm`` given (e.g. the
    multi-GPU runner), every non-empty product runs on it and the partial
    products of a block are joined with eval_add.  Both are bit-identical,
    with the same logical counters (the joins count as adds)."""
    from .engine import MaskCache, OpCounter, run_blocks
    if ta.layout is not Layout.CSR or tb.layout is not Layout.CSC:
        raise ParameterError("tiled product needs CSR x CSC operands")
    counter = counter if counter is not None else OpCounter()
    mask_cache = mask_cache if mask_cache is not None else MaskCache(ctx, ta.b)
    res = TiledResult(n=ta.n, T=ta.T, b=ta.b)
    if spmm is None:
        blocks: dict = {}
        for I, K, J in block_products(ta, tb):
            blocks.setdefault((I, J), []).append((ta.tiles[(I, K)], tb.tiles[(K, J)]))
        for key, part in run_blocks(blocks, ctx, keys, counter, mask_cache).items():
            if part.ctxt is not None:
                res.tiles[key] = part
        return res
    for I, K, J in block_products(ta, tb):
        part = spmm(ta.tiles[(I, K)], tb.tiles[(K, J)], ctx, keys, counter, mask_cache)
        if part.ctxt is None:
            continue
        prev = res.tiles.get((I, J))
        if prev is None:
            res.tiles[(I, J)] = part
        else:
            res.tiles[(I, J)] = EncryptedResult(ctx.eval_add(prev.ctxt, part.ctxt), ta.b)
            counter.adds += 1
    return res


def decrypt_tiled(res: TiledResult, ctx, keys) -> np.ndarray:
    """Dense N x N plaintext of a tiled result (empty blocks are zero)."""
    T, b = res.T, res.b
    out = np.zeros((T * b, T * b))
    for (I, J), r in res.tiles.items():
        out[I * b:(I + 1) * b, J * b:(J + 1) * b] = decrypt_result(r, ctx, keys)
    return out[:res.n, :res.n]


def tiled_pair_count(a, b_mat, T: int) -> int:
    """Pairs the tiled product executes (sum over block products) -- the
    work measure for the bench line; equals the untiled schedule's count."""
    from .encmat import meta_and_values, pair_array
    ba, bs = split_blocks(a, T)
    bb, _ = split_blocks(b_mat, T)
    total = 0
    for (I, K), blk in ba.items():
        ma, _ = meta_and_values(blk, Layout.CSR)
        for J in range(T):
            if (K, J) in bb:
                mb, _ = meta_and_values(bb[(K, J)], Layout.CSC)
                total += len(pair_array(ma, mb))
    return total


def grid_for(n: int, ring_degree: int) -> tuple[int, int]:
    return tile_grid(n, ring_degree // 2)


__all__ = ["TiledMatrix", "TiledResult", "tile_grid", "split_blocks", "encrypt_tiled",
           "block_products", "required_rotation_steps_tiled", "spmm_tiled", "decrypt_tiled",
           "tiled_pair_count", "grid_for"]
