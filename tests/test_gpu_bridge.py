"""The reference-object bridge (refadapter.ReferenceBridge) on the GPU.

The real reference package cannot travel to the GPU box, so reference-typed
objects are built here with the same attribute surface (SURVEY.md §8b
"duck-typed inputs") from CPU-oracle data, in a module named like the
reference's (`<pkg>.encmat` / `<pkg>.engine`).  The bridge must return the
oracle's result bit for bit, in the reference's own result types.  The host
halves of the bridge (extract / wrap) are checked against the GENUINE
reference objects and the reference's own runner in the build container
(tests/test_bridge_reference.py).
"""

import sys
import types
from dataclasses import dataclass, field

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _fake_reference_modules():
    enc = types.ModuleType("fakeref.encmat")
    eng = types.ModuleType("fakeref.engine")

    class ParameterError(ValueError):
        pass

    @dataclass(frozen=True)
    class Ciphertext:
        polys: tuple
        scale: float
        level: int

    @dataclass(frozen=True)
    class EncryptedSparseMatrix:
        ctxt: object
        meta: object

        @property
        def dim(self):
            return self.meta.dim

    @dataclass(frozen=True)
    class EncryptedResult:
        ctxt: object
        dim: int

    @dataclass
    class OpCounter:
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

    for cls in (Ciphertext, EncryptedSparseMatrix, EncryptedResult):
        cls.__module__ = enc.__name__
        setattr(enc, cls.__name__, cls)
    enc.ParameterError = ParameterError
    OpCounter.__module__ = eng.__name__
    eng.OpCounter = OpCounter
    sys.modules[enc.__name__] = enc
    sys.modules[eng.__name__] = eng
    return enc, eng


class _Layout:
    def __init__(self, v):
        self.value = v


@dataclass
class _Meta:
    dim: int
    layout: object
    offsets: np.ndarray
    indices: np.ndarray


@dataclass
class _KSK:
    b: tuple
    a: tuple


@dataclass
class _Keys:
    relin: object
    galois: dict = field(default_factory=dict)


class _Pt:
    def __init__(self, limbs):
        self.limbs = tuple(limbs)


class _Masks:
    def __init__(self, by_pos):
        self._m = by_pos
        self.misses = 0

    def get(self, pos):
        return _Pt(self._m[pos])


def _ksk(arr):
    return _KSK(b=tuple(tuple(arr[0, i, m] for m in range(arr.shape[2])) for i in range(arr.shape[1])),
                a=tuple(tuple(arr[1, i, m] for m in range(arr.shape[2])) for i in range(arr.shape[1])))


@pytest.mark.parametrize("n,sb,L,dim,sp", [(1024, 45, 2, 16, 0.5), (4096, 40, 3, 8, 0.6)])
def test_bridge_runs_reference_objects_bit_exact(oracle_mod, n, sb, L, dim, sp):
    import torch
    assert torch.cuda.is_available()
    from paper_2604_11659_b200.refadapter import ReferenceBridge
    O = oracle_mod
    enc_mod, eng_mod = _fake_reference_modules()
    P = O.build_params(n, sb, L, 2024)
    octx = O.OracleContext(P)
    okeys = octx.keygen()
    a = O.generate_random_sparse(dim, sp, (11, 0))
    b = O.generate_random_sparse(dim, sp, (11, 1))
    oa, ia, va = O.csr_pack(a)
    ob, ib, vb = O.csc_pack(b)
    ca = octx.encrypt(octx.encode(va), okeys)
    cb = octx.encrypt(octx.encode(vb), okeys)
    pairs = O.pair_schedule_csr_csc(oa, ia, ob, ib, dim)
    octx.gen_galois_keys(O.rotation_steps(pairs, dim), okeys)
    masks = {p: octx.encode(np.eye(1, dim * dim, p).ravel(), scale=float(P.modulus_chain[L - 1]),
                            level=L - 1)[0] for p in {min(x[2], x[3]) for x in pairs}}
    want = octx.spmspm(ca[0], cb[0], pairs, dim, masks, okeys)

    class RefCtx:
        params = P
        relin_noops = 0

    ref_ctx = RefCtx()
    keys = _Keys(relin=_ksk(okeys.relin), galois={r: _ksk(k) for r, k in okeys.galois.items()})
    C = enc_mod.Ciphertext
    ea = enc_mod.EncryptedSparseMatrix(C(tuple(tuple(ca[0][p]) for p in range(2)), ca[1], ca[2]),
                                       _Meta(dim, _Layout("csr"), oa, ia))
    eb = enc_mod.EncryptedSparseMatrix(C(tuple(tuple(cb[0][p]) for p in range(2)), cb[1], cb[2]),
                                       _Meta(dim, _Layout("csc"), ob, ib))
    bridge = ReferenceBridge(ref_ctx)
    counter = eng_mod.OpCounter()
    res = bridge.spmm_csr_csc(ea, eb, ref_ctx, keys, counter, _Masks(masks))
    assert isinstance(res, enc_mod.EncryptedResult)
    assert isinstance(res.ctxt, enc_mod.Ciphertext)
    assert np.array_equal(np.array(res.ctxt.polys), want)
    assert res.ctxt.level == L - 2
    assert counter.ct_ct_mults == len(pairs) and ref_ctx.relin_noops == len(pairs)
    assert counter.adds == len(pairs) - 1 and counter.wall_time > 0
    # second call reuses uploaded keys and masks
    res2 = bridge.spmm_csr_csc(ea, eb, ref_ctx, keys, eng_mod.OpCounter(), _Masks(masks))
    assert np.array_equal(np.array(res2.ctxt.polys), want)
