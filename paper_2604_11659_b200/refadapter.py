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
        self._device_index = device_index
        self._ctx = None                # the device context, created on first execute
        self._uploaded = set()          # ("relin", id) / ("galois", step)
        self._masks = {}                # (id(mask_cache), pos) -> device tensor (Montgomery)

    @property
    def ctx(self) -> CkksContext:
        if self._ctx is None:
            self._ctx = CkksContext(self.params, self._device_index)
        return self._ctx

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

    # -- the three halves of one call (extract and wrap are pure host code,
    # tested with the genuine reference objects in tests/test_bridge_reference.py)
    def extract(self, enc_a, enc_b, ctx, counter=None, mask_cache=None) -> dict:
        """Read the reference objects: layout check (engine.py:167-173), the
        CSR x CSC schedule (C++ planner), the Galois steps it needs, the mask
        limbs of its slots and both ciphertexts as uint64 arrays."""
        ref_encmat = sys.modules[type(enc_a).__module__]
        if enc_a.meta.layout.value != "csr" or enc_b.meta.layout.value != "csc":
            raise ref_encmat.ParameterError(
                f"layout mismatch: need csr x csc, got {enc_a.meta.layout.value} x "
                f"{enc_b.meta.layout.value}")
        dim = enc_a.dim
        ref_engine = sys.modules[ref_encmat.__name__.replace("encmat", "engine")]
        if counter is None:
            counter = ref_engine.OpCounter()
        if mask_cache is None:
            mask_cache = ref_engine.MaskCache(ctx, dim)
        from .encmat import plan_csr_csc
        pairs = np.ascontiguousarray(plan_csr_csc(enc_a.meta, enc_b.meta), dtype=np.int64).reshape(-1, 4)
        slots = self.params.slots
        steps = set()
        if len(pairs):
            ap, bp = pairs[:, 2], pairs[:, 3]
            al = np.abs(ap - bp)
            rot = np.minimum(ap, bp) - (pairs[:, 0] * dim + pairs[:, 1])
            steps = {int(x) % slots for x in np.unique(np.concatenate([al[al != 0], rot[rot != 0]]))}
        positions = np.unique(np.minimum(pairs[:, 2], pairs[:, 3])) if len(pairs) else np.zeros(0, np.int64)
        masks = {int(p): np.ascontiguousarray(np.stack(mask_cache.get(int(p)).limbs), dtype=np.uint64)
                 for p in positions}
        return {"dim": dim, "pairs": pairs, "steps": sorted(steps), "masks": masks,
                "ct_a": np.ascontiguousarray(np.array(enc_a.ctxt.polys, dtype=np.uint64)),
                "ct_b": np.ascontiguousarray(np.array(enc_b.ctxt.polys, dtype=np.uint64)),
                "counter": counter, "mask_cache": mask_cache, "encmat": ref_encmat}

    def wrap(self, x: dict, enc_a, enc_b, ctx, res: np.ndarray | None, counts: dict, seconds: float):
        """The reference's own result types, counter increments,
        ctx.relin_noops and counter.wall_time (engine.py:136-184)."""
        counter, ref_encmat = x["counter"], x["encmat"]
        for name in ("ct_ct_mults", "pt_mults", "rotations", "relins", "relin_noops", "rescales",
                     "adds", "alignment_rotations", "accumulation_rotations"):
            setattr(counter, name, getattr(counter, name) + int(counts[name]))
        ctx.relin_noops += int(counts["relin_noops"])
        counter.wall_time += seconds
        dim = x["dim"]
        if res is None:
            return ref_encmat.EncryptedResult(ctxt=None, dim=dim)
        L = self.params.levels
        chain = self.params.modulus_chain
        scale = ((enc_a.ctxt.scale * enc_b.ctxt.scale) / chain[L] * float(chain[L - 1])) / chain[L - 1]
        polys = tuple(tuple(res[p, i] for i in range(L - 1)) for p in range(2))
        return ref_encmat.EncryptedResult(ctxt=type(enc_a.ctxt)(polys, scale, L - 2), dim=dim)

    def execute(self, x: dict, keys):
        """Device half: keys and masks uploaded once, the runner over the
        extracted schedule.  Returns (result [2][L-1][n] or None, counts)."""
        self._sync_keys(keys, x["steps"])
        positions = list(x["masks"])
        for pos in positions:
            key = (id(x["mask_cache"]), pos)
            if key not in self._masks:
                t = D.to_dev(x["masks"][pos])
                check(lib().hs_to_montgomery(self.ctx.handle, D.ptr(t), 1, self.params.levels, 0, 0,
                                             D.stream()))
                self._masks[key] = t
        npos = max(positions) + 1 if positions else 1
        table = (ctypes.c_void_p * npos)()
        for pos in positions:
            table[pos] = self._masks[(id(x["mask_cache"]), pos)].data_ptr()
        L = self.params.levels
        ca, cb = D.to_dev(x["ct_a"]), D.to_dev(x["ct_b"])
        out = D.empty((2, L - 1, self.params.ring_degree))
        cnt = HsCounters()
        pl = x["pairs"]
        check(lib().hs_spmspm_pairs(self.ctx.handle, x["dim"], pl.ctypes.data_as(c_i64p), len(pl),
                                    D.ptr(ca), D.ptr(cb), table, npos, D.ptr(out),
                                    ctypes.byref(cnt), 0, 1, D.stream()))
        counts = {name: getattr(cnt, name) for name, _ in HsCounters._fields_}
        return (D.to_host(out) if cnt.has_result else None), counts

    def spmm_csr_csc(self, enc_a, enc_b, ctx, keys, counter=None, mask_cache=None):
        start = time.perf_counter()
        x = self.extract(enc_a, enc_b, ctx, counter, mask_cache)
        res, counts = self.execute(x, keys)
        return self.wrap(x, enc_a, enc_b, ctx, res, counts, time.perf_counter() - start)
