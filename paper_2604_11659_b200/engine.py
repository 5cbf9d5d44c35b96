"""The encrypted matmul runners (reference engine.py) on the B200 engine.

``spmm_csr_csc`` is the drop-in for the reference hot path: same signature,
same exceptions, same logical ``OpCounter`` tallies, same output ciphertext
bits and float scale.  The whole schedule -- planning included, as in the
reference's timed region (engine.py:176-184) -- runs inside one C-ABI call
(``hs_spmspm_csr_csc``) that batches every pair on the device.  The other
three runners differ only in their schedule (engine.py:187-225) and use the
same executor through ``hs_spmspm_pairs``.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import device as D
from ._lib import HsCounters, c_i64p, check, lib
from .encmat import EncryptedResult, EncryptedSparseMatrix, Layout, pair_array, plan_csr_csc
from .errors import EvalError, ParameterError
from .types import Ciphertext, Plaintext


class MatmulMethod(str, Enum):
    NAIVE_DENSE = "naive_dense"
    NAIVE_SPARSE = "naive_sparse"
    CSR_C = "csr_c"
    VCSR_C = "vcsr_c"


@dataclass
class OpCounter:
    """Tally of homomorphic primitives (reference engine.py:29-58).

    Logical counts equal the reference's exactly.  ``physical_alignment``
    records how many alignment rotations were actually executed after
    deduplication by (operand, step); ``plan_ms`` the host planning time.
    """

    ct_ct_mults: int = 0
    pt_mults: int = 0
    rotations: int = 0
    relins: int = 0
    relin_noops: int = 0
    rescales: int = 0
    adds: int = 0
    alignment_rotations: int = 0
    accumulation_rotations: int = 0
    wall_time: float = 0.0
    physical_alignment: int = 0
    plan_ms: float = 0.0
    ranges: int = 0                 # most pair ranges one call needed (aligned operands vs HBM)

    def as_dict(self) -> dict:
        return {"ct_ct_mults": self.ct_ct_mults, "pt_mults": self.pt_mults,
                "rotations": self.rotations, "relins": self.relins,
                "relin_noops": self.relin_noops, "rescales": self.rescales, "adds": self.adds}

    def ct_ops(self) -> int:
        """Logical ct-ops of the north-star metric (relin no-ops excluded)."""
        return (self.ct_ct_mults + self.pt_mults + self.rotations + self.relins + self.rescales
                + self.adds)


class MaskCache:
    """Slot-isolation plaintexts, one per target position (engine.py:61-96).

    Device-resident, kept in Montgomery form so the runner's fused
    rescale-times-mask epilogue needs a single REDC.  ``misses`` counts
    encodes after :meth:`prewarm`.
    """

    def __init__(self, ctx, dim: int):
        lvl = ctx.params.levels - 1
        self._ctx = ctx
        self._size = dim * dim
        self._level = lvl
        self._scale = float(ctx.params.modulus_chain[lvl])
        self._masks: dict[int, Plaintext] = {}
        self._table = None
        self.misses = 0

    def get(self, position: int) -> Plaintext:
        pt = self._masks.get(position)
        if pt is None:
            self.misses += 1
            pt = self._encode(position)
            self._masks[position] = pt
            self._table = None
        return pt

    def prewarm(self, positions) -> None:
        for p in positions:
            p = int(p)
            if p not in self._masks:
                self._masks[p] = self._encode(p)
                self._table = None
        self.misses = 0

    def _encode(self, position: int) -> Plaintext:
        ctx = self._ctx
        vec = np.zeros(self._size)
        vec[position] = 1.0
        coeffs = ctx.encode_coeffs(vec, self._scale)
        limbs = ctx._signed_ntt(coeffs, self._level + 1)
        check(lib().hs_to_montgomery(ctx.handle, D.ptr(limbs), 1, self._level + 1, 0, 0, D.stream()))
        return Plaintext(limbs, self._scale, self._level, mont=True, ctx=ctx)

    def table(self):
        """(ctypes array of device pointers indexed by position, length)."""
        if self._table is None:
            n = max(self._masks) + 1 if self._masks else 1
            arr = (ctypes.c_void_p * n)()
            for p, pt in self._masks.items():
                arr[p] = pt.data.data_ptr()
            self._table = (arr, n)
        return self._table


def _counter_update(counter: OpCounter, c: HsCounters) -> None:
    for name in ("ct_ct_mults", "pt_mults", "rotations", "relins", "relin_noops", "rescales",
                 "adds", "alignment_rotations", "accumulation_rotations", "physical_alignment"):
        setattr(counter, name, getattr(counter, name) + getattr(c, name))
    counter.plan_ms += c.plan_ms
    counter.ranges = max(counter.ranges, int(c.ranges))


def _result_scale(ctx, sa: float, sb: float) -> float:
    """Float scale ledger of one pair, in the reference's expression order:
    mult_ct (context.py:351), rescale (:399), mult_pt (:361), rescale."""
    chain = ctx.params.modulus_chain
    L = ctx.params.levels
    s = sa * sb
    s = s / chain[L]
    s = s * float(chain[L - 1])
    return s / chain[L - 1]


def run_pairs(enc_a: EncryptedSparseMatrix, enc_b: EncryptedSparseMatrix, ctx, keys,
              counter: OpCounter, mask_cache: MaskCache | None, pairs: np.ndarray | None,
              shard: tuple = (0, 1)) -> EncryptedResult:
    """Execute a schedule on the device.  ``pairs`` None = CSR x CSC planned
    in C++ inside the call; otherwise an explicit (P, 4) int64 pair array.
    ``shard`` = (index, count): this call runs one contiguous share of the
    step-sorted pairs and returns that share's partial sum (dist.py)."""
    dim = enc_a.dim
    params = ctx.params
    L = params.levels
    if mask_cache is None:
        mask_cache = MaskCache(ctx, dim)
    if keys.relin is None:
        from .errors import KeyMissingError
        raise KeyMissingError("no relinearization key in bundle")
    start = time.perf_counter()
    ca, cb = enc_a.ctxt, enc_b.ctxt
    if ca.level != cb.level:
        raise EvalError(f"level mismatch: {ca.level} != {cb.level}")
    if ca.level != L:
        raise EvalError(f"level mismatch: {ca.level} != {L}")
    if ca.degree != 1 or cb.degree != 1:
        raise EvalError("eval_mult_ct expects degree-1 ciphertexts")
    da, db = ca.data, cb.data                 # host-built cts are uploaded here
    out = D.empty((2, L - 1, params.ring_degree))
    cnt = HsCounters()
    meta_a, meta_b = enc_a.meta, enc_b.meta
    for attempt in range(2):
        mt, nm = mask_cache.table()
        if pairs is None:
            oa = np.ascontiguousarray(meta_a.offsets, dtype=np.int64)
            ia = np.ascontiguousarray(meta_a.indices, dtype=np.int64)
            ob = np.ascontiguousarray(meta_b.offsets, dtype=np.int64)
            ib = np.ascontiguousarray(meta_b.indices, dtype=np.int64)
            st = lib().hs_spmspm_csr_csc(
                ctx.handle, dim, oa.ctypes.data_as(c_i64p), ia.ctypes.data_as(c_i64p),
                ob.ctypes.data_as(c_i64p), ib.ctypes.data_as(c_i64p), D.ptr(da), D.ptr(db), mt, nm,
                D.ptr(out), ctypes.byref(cnt), shard[0], shard[1], D.stream())
        else:
            pl = np.ascontiguousarray(pairs, dtype=np.int64)
            st = lib().hs_spmspm_pairs(ctx.handle, dim, pl.ctypes.data_as(c_i64p), len(pl),
                                       D.ptr(da), D.ptr(db), mt, nm, D.ptr(out), ctypes.byref(cnt),
                                       shard[0], shard[1], D.stream())
        if st == 4 and attempt == 0 and "not prewarmed" in lib().hs_last_error().decode():
            # encode the missing masks (counted as misses, like MaskCache.get)
            p = pair_array(meta_a, meta_b) if pairs is None else pairs
            for pos in np.unique(np.minimum(p[:, 2], p[:, 3])):
                mask_cache.get(int(pos))
            continue
        check(st)
        break
    D.sync()
    _counter_update(counter, cnt)
    ctx.relin_noops += cnt.relin_noops
    counter.wall_time += time.perf_counter() - start
    if not cnt.has_result:
        return EncryptedResult(ctxt=None, dim=dim)
    return EncryptedResult(ctxt=Ciphertext(out, _result_scale(ctx, ca.scale, cb.scale), L - 2),
                           dim=dim)


def run_blocks(blocks: dict, ctx, keys, counter: OpCounter, mask_cache: MaskCache | None,
               shard: tuple = (0, 1)) -> dict:
    """Output blocks of a tiled product, ``{key: [(enc_a, enc_b), ...]}``
    (C[I][J] = sum_K A[I][K] B[K][J]), in ONE runner call (hs_spmspm_multi):
    the pairs of every product and block are scheduled together, sorted by
    accumulation step, so each Galois key is generated once for the whole
    product and each (operand, step) alignment is rotated once.  Every
    block's result is bit-identical to running its products one by one and
    joining them with eval_add (a modular sum), and the logical counters are
    the same as well.  Returns ``{key: EncryptedResult}``."""
    keys_order = sorted(blocks)
    prods, rows = [], []
    dim = 0
    for o, key in enumerate(keys_order):
        for ea, eb in blocks[key]:
            dim = ea.dim
            p = plan_csr_csc(ea.meta, eb.meta)
            if len(p):
                k = len(prods)
                prods.append((ea, eb, o))
                rows.append(np.concatenate([p, np.full((len(p), 1), k, dtype=np.int64),
                                            np.full((len(p), 1), o, dtype=np.int64)], axis=1))
    out = {key: EncryptedResult(ctxt=None, dim=dim) for key in keys_order}
    if not prods:
        return out
    params = ctx.params
    L = params.levels
    if mask_cache is None:
        mask_cache = MaskCache(ctx, dim)
    if keys.relin is None:
        from .errors import KeyMissingError
        raise KeyMissingError("no relinearization key in bundle")
    start = time.perf_counter()
    scale = {}
    for ea, eb, o in prods:
        ca, cb = ea.ctxt, eb.ctxt
        if ca.level != L or cb.level != L:
            raise EvalError(f"level mismatch: {ca.level}/{cb.level} != {L}")
        if ca.degree != 1 or cb.degree != 1:
            raise EvalError("eval_mult_ct expects degree-1 ciphertexts")
        s_k = _result_scale(ctx, ca.scale, cb.scale)
        if o not in scale:
            scale[o] = s_k
        elif abs(s_k - scale[o]) > 1e-9 * max(abs(scale[o]), abs(s_k)):
            raise EvalError("scale mismatch between block products")   # eval_add's check
    pl = np.ascontiguousarray(np.concatenate(rows), dtype=np.int64)
    outs = [D.empty((2, L - 1, params.ring_degree)) for _ in keys_order]
    cnt = HsCounters()
    cta = [ea.ctxt.data for ea, _, _ in prods]
    ctb = [eb.ctxt.data for _, eb, _ in prods]
    pa = (ctypes.c_void_p * len(prods))(*[D.ptr(t) for t in cta])
    pb = (ctypes.c_void_p * len(prods))(*[D.ptr(t) for t in ctb])
    po = (ctypes.c_void_p * len(outs))(*[D.ptr(t) for t in outs])
    for attempt in range(2):
        mt, nm = mask_cache.table()
        st = lib().hs_spmspm_multi(ctx.handle, dim, pl.ctypes.data_as(c_i64p), len(pl), pa, pb, len(prods),
                                   mt, nm, po, len(outs), ctypes.byref(cnt), shard[0], shard[1],
                                   D.stream())
        if st == 4 and attempt == 0 and "not prewarmed" in lib().hs_last_error().decode():
            for pos in np.unique(np.minimum(pl[:, 2], pl[:, 3])):
                mask_cache.get(int(pos))
            continue
        check(st)
        break
    D.sync()
    _counter_update(counter, cnt)
    ctx.relin_noops += cnt.relin_noops
    counter.wall_time += time.perf_counter() - start
    for o, key in enumerate(keys_order):
        if o in scale:
            out[key] = EncryptedResult(ctxt=Ciphertext(outs[o], scale[o], L - 2), dim=dim)
    return out


def run_products(products, ctx, keys, counter: OpCounter, mask_cache: MaskCache | None,
                 shard: tuple = (0, 1)) -> EncryptedResult:
    """Several CSR x CSC products summed into ONE output (one block)."""
    return run_blocks({0: list(products)}, ctx, keys, counter, mask_cache, shard)[0]


def _require_layouts(enc_a, enc_b, layout_a: Layout, layout_b: Layout):
    if enc_a.meta.layout is not layout_a or enc_b.meta.layout is not layout_b:
        raise ParameterError(
            f"layout mismatch: need {layout_a.value} x {layout_b.value}, got "
            f"{enc_a.meta.layout.value} x {enc_b.meta.layout.value}")
    if enc_a.dim != enc_b.dim:
        raise ParameterError("matrix dimensions differ")


def spmm_csr_csc(enc_a, enc_b, ctx, keys, counter: OpCounter | None = None,
                 mask_cache: MaskCache | None = None) -> EncryptedResult:
    """Sorted-index intersection over a row-wise x column-wise packing."""
    _require_layouts(enc_a, enc_b, Layout.CSR, Layout.CSC)
    counter = counter if counter is not None else OpCounter()
    return run_pairs(enc_a, enc_b, ctx, keys, counter, mask_cache, None)


def spmm_vcsr(enc_a, enc_b, ctx, keys, counter: OpCounter | None = None,
              mask_cache: MaskCache | None = None) -> EncryptedResult:
    _require_layouts(enc_a, enc_b, Layout.VCSR, Layout.VCSC)
    counter = counter if counter is not None else OpCounter()
    return run_pairs(enc_a, enc_b, ctx, keys, counter, mask_cache,
                     pair_array(enc_a.meta, enc_b.meta))


def matmul_naive_dense(enc_a, enc_b, ctx, keys, counter: OpCounter | None = None,
                       mask_cache: MaskCache | None = None) -> EncryptedResult:
    _require_layouts(enc_a, enc_b, Layout.DENSE_ROW_MAJOR, Layout.DENSE_COL_MAJOR)
    counter = counter if counter is not None else OpCounter()
    return run_pairs(enc_a, enc_b, ctx, keys, counter, mask_cache,
                     pair_array(enc_a.meta, enc_b.meta))


def matmul_naive_sparse(enc_a, enc_b, ctx, keys, counter: OpCounter | None = None,
                        mask_cache: MaskCache | None = None,
                        skip_both_zero_only: bool = False) -> EncryptedResult:
    _require_layouts(enc_a, enc_b, Layout.DENSE_ROW_MAJOR, Layout.DENSE_COL_MAJOR)
    counter = counter if counter is not None else OpCounter()
    skip = "both" if skip_both_zero_only else "either"
    return run_pairs(enc_a, enc_b, ctx, keys, counter, mask_cache,
                     pair_array(enc_a.meta, enc_b.meta, skip=skip))


def fhe_spmspm_step(v_a: Ciphertext, v_b: Ciphertext, min_pos: int, i: int, j: int, dim: int,
                    accumulator: EncryptedResult | None, ctx, keys, counter: OpCounter,
                    mask_cache: MaskCache) -> EncryptedResult:
    """One aligned scalar product folded into the accumulator (engine.py:99-133),
    primitive by primitive on the device."""
    dot = ctx.eval_mult_ct(v_a, v_b)
    counter.ct_ct_mults += 1
    dot = ctx.relinearize(dot, keys)
    counter.relins += 1
    dot = ctx.rescale(dot)
    counter.rescales += 1
    dot = ctx.eval_mult_pt(dot, mask_cache.get(min_pos))
    counter.pt_mults += 1
    dot = ctx.relinearize(dot, keys)
    counter.relin_noops += 1
    dot = ctx.rescale(dot)
    counter.rescales += 1
    rot_idx = min_pos - (i * dim + j)
    if rot_idx != 0:
        dot = ctx.eval_rotate(dot, rot_idx, keys)
        counter.rotations += 1
        counter.accumulation_rotations += 1
    if accumulator is None or accumulator.ctxt is None:
        return EncryptedResult(ctxt=dot, dim=dim)
    merged = ctx.eval_add(accumulator.ctxt, dot)
    counter.adds += 1
    return EncryptedResult(ctxt=merged, dim=dim)


METHOD_RUNNERS = {
    MatmulMethod.NAIVE_DENSE: matmul_naive_dense,
    MatmulMethod.NAIVE_SPARSE: matmul_naive_sparse,
    MatmulMethod.CSR_C: spmm_csr_csc,
    MatmulMethod.VCSR_C: spmm_vcsr,
}

METHOD_LAYOUTS = {
    MatmulMethod.NAIVE_DENSE: (Layout.DENSE_ROW_MAJOR, Layout.DENSE_COL_MAJOR),
    MatmulMethod.NAIVE_SPARSE: (Layout.DENSE_ROW_MAJOR, Layout.DENSE_COL_MAJOR),
    MatmulMethod.CSR_C: (Layout.CSR, Layout.CSC),
    MatmulMethod.VCSR_C: (Layout.VCSR, Layout.VCSC),
}
