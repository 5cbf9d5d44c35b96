"""ReferenceBridge's host halves against the GENUINE reference objects.

The real reference (``hespmm``, built from /root/reference like
tests/golden/make_golden.py does) exists only in the build container, and
this container has no GPU; the GPU box has a GPU but no reference.  So the
bridge is checked in two halves:

* here: ``extract`` reads genuine ``hespmm`` objects (EncryptedSparseMatrix,
  KeyBundle, MaskCache, OpCounter, CkksContext), the CPU oracle stands in for
  the device half on the extracted arrays, and ``wrap`` must rebuild the
  reference's own result -- the same ``hespmm.encmat.EncryptedResult`` /
  ``hespmm.ckks.types.Ciphertext`` types, bit-identical limbs, float scale,
  level, OpCounter increments, ``ctx.relin_noops`` -- as the reference's
  ``spmm_csr_csc`` run on the same objects, and raise its ParameterError;
* on the GPU (tests/test_gpu_bridge.py): ``execute`` on the device, through
  reference-shaped objects.

Skipped where /root/reference is absent (the GPU box).
"""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

pytestmark = pytest.mark.skipif(not os.path.isdir("/root/reference/pkg"),
                                reason="the reference package is only in the build container")


@pytest.fixture(scope="module")
def hespmm():
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden import ref_import
    return ref_import()


def _counts(pairs: np.ndarray, dim: int) -> dict:
    """The runner's logical counts of a schedule (engine.py:99-160)."""
    P = len(pairs)
    al = int(np.count_nonzero(pairs[:, 2] != pairs[:, 3])) if P else 0
    acc = int(np.count_nonzero(np.minimum(pairs[:, 2], pairs[:, 3]) != pairs[:, 0] * dim + pairs[:, 1])) if P else 0
    return {"ct_ct_mults": P, "pt_mults": P, "relins": P, "relin_noops": P, "rescales": 2 * P,
            "adds": max(P - 1, 0), "alignment_rotations": al, "accumulation_rotations": acc,
            "rotations": al + acc, "has_result": int(P > 0)}


@pytest.mark.parametrize("n,sb,L,dim,sp,mseed", [(1024, 45, 2, 8, 0.5, 3), (64, 40, 3, 4, 0.4, 41),
                                                  (64, 40, 2, 4, 1.0, 51)])
def test_bridge_host_halves_with_genuine_reference_objects(hespmm, oracle_mod, n, sb, L, dim, sp, mseed):
    from hespmm.ckks import CkksContext, build_params
    from hespmm.encmat import Layout, encrypt_sparse, pair_schedule, required_rotation_steps
    from hespmm.engine import MaskCache, OpCounter, spmm_csr_csc
    from hespmm.formats import generate_random_sparse
    from paper_2604_11659_b200.refadapter import ReferenceBridge, _key_array
    O = oracle_mod
    P = build_params(n, sb, L, 2024)
    ctx = CkksContext(P)
    keys = ctx.keygen()
    a = generate_random_sparse(dim, sp, (mseed, 0))
    b = generate_random_sparse(dim, sp, (mseed, 1))
    ea = encrypt_sparse(a, Layout.CSR, ctx, keys)
    eb = encrypt_sparse(b, Layout.CSC, ctx, keys)
    steps = required_rotation_steps(ea.meta, eb.meta)
    keys = ctx.gen_galois_keys(steps, keys) if steps else keys
    mc = MaskCache(ctx, dim)
    mc.prewarm(min(ap, bp) for _, _, ap, bp in pair_schedule(ea.meta, eb.meta))

    ref_counter = OpCounter()
    noops0 = ctx.relin_noops
    want = spmm_csr_csc(ea, eb, ctx, keys, ref_counter, mc)
    ref_noops = ctx.relin_noops - noops0

    bridge = ReferenceBridge(ctx)            # no device context until execute()
    counter = OpCounter()
    x = bridge.extract(ea, eb, ctx, counter, mc)
    assert x["encmat"] is sys.modules["hespmm.encmat"]
    assert sorted(map(tuple, x["pairs"].tolist())) == sorted(pair_schedule(ea.meta, eb.meta))
    # the device half, done by the CPU oracle on the extracted arrays
    octx = O.OracleContext(O.build_params(n, sb, L, 2024))
    okeys = O.Keys(None, None, None, None, _key_array(keys.relin),
                   {r: _key_array(keys.galois[r]) for r in x["steps"]})
    res = octx.spmspm(x["ct_a"], x["ct_b"], x["pairs"], dim, x["masks"], okeys)
    noops0 = ctx.relin_noops
    got = bridge.wrap(x, ea, eb, ctx, res, _counts(x["pairs"], dim), 0.0)
    assert ctx.relin_noops - noops0 == ref_noops
    assert type(got) is type(want)
    for f in ("ct_ct_mults", "pt_mults", "rotations", "relins", "relin_noops", "rescales", "adds",
              "alignment_rotations", "accumulation_rotations"):
        assert getattr(counter, f) == getattr(ref_counter, f), f
    if want.ctxt is None:
        assert got.ctxt is None
        return
    assert type(got.ctxt) is type(want.ctxt)
    assert got.ctxt.level == want.ctxt.level and got.ctxt.scale == want.ctxt.scale
    assert np.array_equal(np.array(got.ctxt.polys, dtype=np.uint64), np.array(want.ctxt.polys, dtype=np.uint64))


def test_bridge_layout_error_is_the_references(hespmm):
    from hespmm.ckks import CkksContext, build_params
    from hespmm.encmat import Layout, encrypt_sparse
    from hespmm.errors import ParameterError
    from hespmm.formats import generate_random_sparse
    from paper_2604_11659_b200.refadapter import ReferenceBridge
    ctx = CkksContext(build_params(64, 40, 2, 7))
    keys = ctx.keygen()
    m = generate_random_sparse(4, 0.3, 1)
    ea = encrypt_sparse(m, Layout.CSR, ctx, keys)
    eb = encrypt_sparse(m, Layout.CSC, ctx, keys)
    with pytest.raises(ParameterError, match="layout mismatch"):
        ReferenceBridge(ctx).extract(eb, ea, ctx)
