"""Multi-ciphertext tiling on the GPU (beyond the
reference's one-ciphertext capacity): a 40 x 40 product at N = 2^10
(512 slots, so the untiled packing would raise CapacityError) as 2 x 2
blocks of 20 x 20.  Parity: decrypted result vs the plaintext product, and
every block product bit-identical to the CPU oracle's CSR/C runner on the
same block ciphertexts, accumulated exactly like eval_add."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    assert torch.cuda.is_available()
    import paper_2604_11659_b200 as P
    from paper_2604_11659_b200 import formats, tiling
    from paper_2604_11659_b200.encmat import Layout
    n, sb, L, seed, dim = 1024, 45, 2, 2024, 40
    params = P.build_params(n, sb, L, seed)
    ctx = P.CkksContext(params)
    keys = ctx.keygen()
    a = formats.generate_random_sparse(dim, 0.6, (21, 0))
    b = formats.generate_random_sparse(dim, 0.6, (21, 1))
    ta = tiling.encrypt_tiled(a, Layout.CSR, ctx, keys)
    tb = tiling.encrypt_tiled(b, Layout.CSC, ctx, keys)
    keys = ctx.gen_galois_keys(tiling.required_rotation_steps_tiled(ta, tb), keys, device=True)
    return P, ctx, keys, a, b, ta, tb, (n, sb, L, seed)


def test_untiled_packing_exceeds_capacity(setup):
    P, ctx, keys, a, *_ = setup
    from paper_2604_11659_b200 import encmat
    with pytest.raises(P.CapacityError):
        encmat.encrypt_sparse(a, encmat.Layout.CSR, ctx, keys)


def test_tiled_product_matches_plaintext(setup, oracle_mod):
    P, ctx, keys, a, b, ta, tb, _ = setup
    from paper_2604_11659_b200 import engine, tiling
    assert (ta.T, ta.b) == (2, 20)
    counter = engine.OpCounter()
    res = tiling.spmm_tiled(ta, tb, ctx, keys, counter)
    out = tiling.decrypt_tiled(res, ctx, keys)
    err = oracle_mod.frobenius_error(out, oracle_mod.plain_matmul(a, b))
    assert err < 1e-5, err
    prods = tiling.block_products(ta, tb)
    assert counter.ct_ct_mults == tiling.tiled_pair_count(a, b, ta.T)
    assert counter.adds >= len(prods) - len(res.tiles)


def test_block_products_bit_exact_vs_oracle(setup, oracle_mod):
    P, ctx, keys, a, b, ta, tb, prm = setup
    from paper_2604_11659_b200 import engine, encmat, tiling
    O = oracle_mod
    n, sb, L, seed = prm
    octx = O.OracleContext(O.build_params(n, sb, L, seed))
    okeys = octx.keygen()
    mc = engine.MaskCache(ctx, ta.b)
    res = tiling.spmm_tiled(ta, tb, ctx, keys, None, mc)
    steps = set()
    want = {}
    for I, K, J in tiling.block_products(ta, tb):
        ea, eb = ta.tiles[(I, K)], tb.tiles[(K, J)]
        pairs = encmat.pair_array(ea.meta, eb.meta)
        if len(pairs) == 0:
            continue
        octx.gen_galois_keys(O.rotation_steps(pairs.tolist(), ta.b), okeys)
        pos = np.unique(np.minimum(pairs[:, 2], pairs[:, 3]))
        mc.prewarm(pos)
        masks = {int(p): np.stack(mc.get(int(p)).limbs) for p in pos}
        part = octx.spmspm(ea.ctxt.host(), eb.ctxt.host(), pairs, ta.b, masks, okeys)
        if (I, J) in want:       # eval_add: limb-wise sum mod q
            qs = np.array(ctx.params.modulus_chain[:L - 1], dtype=object)
            s = want[(I, J)].astype(object) + part.astype(object)
            want[(I, J)] = (s % qs[None, :, None]).astype(np.uint64)
        else:
            want[(I, J)] = part
    assert set(want) == set(res.tiles)
    for key, w in want.items():
        assert np.array_equal(res.tiles[key].ctxt.host(), w), key


def test_block_runner_equals_per_product_runs(setup):
    """One hs_spmspm_multi call per output block (the default) == every
    product on the plain runner joined with eval_add: same limbs, scale,
    level and logical counters."""
    P, ctx, keys, a, b, ta, tb, _ = setup
    from paper_2604_11659_b200 import engine, tiling
    c1, c2 = engine.OpCounter(), engine.OpCounter()
    fused = tiling.spmm_tiled(ta, tb, ctx, keys, c1)
    plain = tiling.spmm_tiled(ta, tb, ctx, keys, c2, spmm=engine.spmm_csr_csc)
    assert sorted(fused.tiles) == sorted(plain.tiles)
    for k in fused.tiles:
        f, p = fused.tiles[k].ctxt, plain.tiles[k].ctxt
        assert np.array_equal(f.host(), p.host()), k
        assert f.scale == p.scale and f.level == p.level
    for name in ("ct_ct_mults", "pt_mults", "rotations", "relins", "relin_noops", "rescales", "adds",
                 "alignment_rotations", "accumulation_rotations"):
        assert getattr(c1, name) == getattr(c2, name), name
