"""Bridge: run the REFERENCE package's own objects through the B200 runner.

A ``hespmm`` maintainer registers the B200 engine behind the reference's own
operator API (engine.py:228-233) without touching any other code:

    from paper_2604_11659_b200.refadapter import ReferenceBridge
    bridge = ReferenceBridge(ctx)                       # ctx: hespmm CkksContext
    hespmm.engine.METHOD_RUNNERS[MatmulMethod.CSR_C] = bridge.spmm_csr_csc

The bridge reads only the attributes the reference runner reads (SURVEY.md
§8b "duck-typed inputs"): ``enc.ctxt.polys/.scale/.level``, ``enc.meta``
(CSR/CSC offsets/indices), ``keys.relin.{b,a}``, ``keys.galois[step]``,
``ctx.params``, ``mask_cache.get(pos).limbs`` -- and returns the reference's
own result types (``type(enc_a.ctxt)`` / the encmat module's
``EncryptedResult``), with the reference's logical counter increments,
``ctx.relin_noops`` and ``counter.wall_time``.
"""

from __future__ import annotations

import ctypes
import sys
import time

import numpy as np

from . import device as D
from ._lib import HsCounters, c_i64p, check, lib
from .context import CkksContext
from .errors import KeyMissingError
from .params import CkksParams


def _key_array(ksk) -> np.ndarray:
    """Reference KeySwitchKey (b[i][m], a[i][m] tuples) -> [2][L+1][L+2][n]."""
    return np.ascontiguousarray(np.array([[np.stack(d) for d in ksk.b],
                                          [np.stack(d) for d in ksk.a]], dtype=np.uint64))


class ReferenceBridge:
    def __init__(self, ref_ctx, device_index: int | None = None):
        p = ref_ctx.params
        self.params = CkksParams(ring_degree=p.ring_degree, modulus_chain=tuple(p.modulus_chain),
                                 scale_bits=p.scale_bits, aux_prime=p.aux_prime, seed=p.seed)
        self.ctx = CkksContext(self.params, device_index)
        self._uploaded = set()          # ("relin", id) / ("galois", step)
        self._masks = {}                # (id(mask_cache), pos) -> device tensor (Montgomery)

    # -- key material: uploaded once per key, converted to Montgomery form on device
    def _sync_keys(self, keys, steps) -> None:
        if keys.relin is None:
            raise KeyMissingError("no relinearization key in bundle")
        if ("relin", id(keys.relin)) not in self._uploaded:
            self.ctx.upload_key(0, 0, _key_array(keys.relin))
            self._uploaded.add(("relin", id(keys.relin)))
        for r in steps:
            if ("galois", r) in self._uploaded:
                continue
            gk = keys.galois.get(r)
            if gk is None:
                raise KeyMissingError(f"missing Galois key for step {r}")
            self.ctx.upload_key(1, r, _key_array(gk))
            self._uploaded.add(("galois", r))

    def _mask_table(self, mask_cache, positions):
        L = self.params.levels
        n = self.params.ring_degree
        for pos in positions:
            key = (id(mask_cache), int(pos))
            if key in self._masks:
                continue
            pt = mask_cache.get(int(pos))
            t = D.to_dev(np.ascontiguousarray(np.stack(pt.limbs), dtype=np.uint64))
            check(lib().hs_to_montgomery(self.ctx.handle, D.ptr(t), 1, L, 0, 0, D.stream()))
            self._masks[key] = t
        npos = int(max(positions)) + 1 if len(positions) else 1
        arr = (ctypes.c_void_p * npos)()
        for pos in positions:
            arr[int(pos)] = self._masks[(id(mask_cache), int(pos))].data_ptr()
        del n
        return arr, npos

    def spmm_csr_csc(self, enc_a, enc_b, ctx, keys, counter=None, mask_cache=None):
        ref_engine = sys.modules[type(counter).__module__] if counter is not None else None
        ref_encmat = sys.modules[type(enc_a).__module__]
        if enc_a.meta.layout.value != "csr" or enc_b.meta.layout.value != "csc":
            raise ref_encmat.ParameterError(
                f"layout mismatch: need csr x csc, got {enc_a.meta.layout.value} x "
                f"{enc_b.meta.layout.value}")
        dim = enc_a.dim
        if counter is None:
            counter = sys.modules[ref_encmat.__name__.replace("encmat", "engine")].OpCounter()
        if mask_cache is None:
            mask_cache = sys.modules[ref_encmat.__name__.replace("encmat", "engine")].MaskCache(ctx, dim)
        start = time.perf_counter()
        from .encmat import plan_csr_csc
        pairs = plan_csr_csc(enc_a.meta, enc_b.meta)
        slots = self.params.slots
        L = self.params.levels
        steps = set()
        if len(pairs):
            ap, bp = pairs[:, 2], pairs[:, 3]
            al = np.abs(ap - bp)
            rot = np.minimum(ap, bp) - (pairs[:, 0] * dim + pairs[:, 1])
            steps = {int(x) % slots for x in np.unique(np.concatenate([al[al != 0], rot[rot != 0]]))}
        self._sync_keys(keys, sorted(steps))
        positions = np.unique(np.minimum(pairs[:, 2], pairs[:, 3])) if len(pairs) else []
        table, npos = self._mask_table(mask_cache, positions)
        ca = D.to_dev(np.ascontiguousarray(np.array(enc_a.ctxt.polys, dtype=np.uint64)))
        cb = D.to_dev(np.ascontiguousarray(np.array(enc_b.ctxt.polys, dtype=np.uint64)))
        out = D.empty((2, L - 1, self.params.ring_degree))
        cnt = HsCounters()
        pl = np.ascontiguousarray(pairs, dtype=np.int64)
        check(lib().hs_spmspm_pairs(self.ctx.handle, dim, pl.ctypes.data_as(c_i64p), len(pl),
                                    D.ptr(ca), D.ptr(cb), table, npos, D.ptr(out),
                                    ctypes.byref(cnt), 0, 1, D.stream()))
        res_np = D.to_host(out)
        for name in ("ct_ct_mults", "pt_mults", "rotations", "relins", "relin_noops", "rescales",
                     "adds", "alignment_rotations", "accumulation_rotations"):
            setattr(counter, name, getattr(counter, name) + getattr(cnt, name))
        ctx.relin_noops += cnt.relin_noops
        counter.wall_time += time.perf_counter() - start
        del ref_engine
        if not cnt.has_result:
            return ref_encmat.EncryptedResult(ctxt=None, dim=dim)
        chain = self.params.modulus_chain
        scale = ((enc_a.ctxt.scale * enc_b.ctxt.scale) / chain[L] * float(chain[L - 1])) / chain[L - 1]
        ct_type = type(enc_a.ctxt)
        polys = tuple(tuple(res_np[p, i] for i in range(L - 1)) for p in range(2))
        return ref_encmat.EncryptedResult(ctxt=ct_type(polys, scale, L - 2), dim=dim)
