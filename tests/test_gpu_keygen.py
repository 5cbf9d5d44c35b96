"""On-device Galois key generation is bit-exact with the reference's numpy
stream (ckks/context.py:176-200): raw draws vs numpy itself, whole keys vs
the host-drawn path and the golden digests, and lazily generated keys inside
the runner vs resident keys."""

import ctypes

import numpy as np
import pytest

from helpers import digest, parse_key

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    assert torch.cuda.is_available()
    import paper_2604_11659_b200 as P
    return P


def _numpy_draws(params, seed, r):
    rng = np.random.default_rng(np.random.SeedSequence(entropy=(seed, 0x90, r)))
    L, n = params.levels, params.ring_degree
    primes = (*params.modulus_chain, params.aux_prime)
    a = np.empty((L + 1, L + 2, n), dtype=np.uint64)
    e = np.empty((L + 1, n), dtype=np.int64)
    for i in range(L + 1):
        for m, q in enumerate(primes):
            a[i, m] = rng.integers(0, q, size=n, dtype=np.uint64)
        e[i] = np.rint(rng.normal(0.0, 3.2, n)).astype(np.int64)
    return a, e


# the last set is the north-star ring at L = 24: 6 keys x 25 digits x 65,536
# normals (~9.8 M ziggurat draws, ~120 K slow-path exp / log1p evaluations) and
# 6 x 650 uniform segments, raw draws compared with numpy itself
@pytest.mark.parametrize("n,sb,L,nkeys", [(64, 40, 2, 5), (1024, 45, 2, 5), (16384, 50, 2, 5), (8192, 40, 4, 5),
                                          (4096, 50, 6, 24), (65536, 50, 24, 6)])
def test_device_stream_replays_numpy(pkg, n, sb, L, nkeys):
    from paper_2604_11659_b200 import device as D
    from paper_2604_11659_b200._lib import check, lib
    from paper_2604_11659_b200.rng import galois_states, ziggurat_tables
    params = pkg.build_params(n, sb, L, 2024)
    ctx = pkg.CkksContext(params)
    wi, fi, ki = ziggurat_tables()
    check(lib().hs_keygen_set_tables(ctx.handle, wi.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     fi.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     ki.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    steps = ([1, 3, n // 2 - 1, 7, 11] + list(range(13, 13 + 2 * nkeys, 2)))[:nkeys]
    st = np.ascontiguousarray(galois_states(2024, steps))
    K = len(steps)
    a = D.empty((K, L + 1, L + 2, n))
    e = D.to_dev(np.zeros((K, L + 1, n), dtype=np.int64))
    check(lib().hs_keygen_streams(ctx.handle, st.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), K,
                                  D.ptr(a), D.ptr(e), D.stream()))
    ah, eh = D.to_host(a), D.to_host(e)
    for k, r in enumerate(steps):
        wa, we = _numpy_draws(params, 2024, r)
        assert np.array_equal(ah[k], wa), r
        assert np.array_equal(eh[k], we), r


@pytest.mark.parametrize("key", ["64_40_2_7", "1024_45_2_2024", "16384_50_2_2024"])
def test_device_keys_match_reference_digests(pkg, golden, key):
    rec = golden["ops"][key]
    n, sb, L, seed = parse_key(key)
    params = pkg.build_params(n, sb, L, seed)
    ctx = pkg.CkksContext(params)
    keys = ctx.keygen()
    keys = ctx.gen_galois_keys([1, 3, params.slots - 1, -2, 5], keys, device=True)
    for r, (hb, ha) in rec["galois"].items():
        arr = keys.galois[int(r)].array()
        assert digest(arr[0]) == hb and digest(arr[1]) == ha, r


def test_lazy_keys_inside_runner_match_resident_keys(pkg):
    """cfg1 shape: every Galois key generated on demand inside the runner."""
    from paper_2604_11659_b200 import encmat, engine, formats
    from paper_2604_11659_b200._lib import lib
    params = pkg.build_params(1024, 45, 2, 2024)
    res = {}
    for mode in (False, "lazy"):
        ctx = pkg.CkksContext(params)
        keys = ctx.keygen()
        seed = 1 * 1_000_003 + 16 * 1_009
        a = formats.generate_random_sparse(16, 0.5, (seed, 0))
        b = formats.generate_random_sparse(16, 0.5, (seed, 1))
        ea = encmat.encrypt_sparse(a, encmat.Layout.CSR, ctx, keys)
        eb = encmat.encrypt_sparse(b, encmat.Layout.CSC, ctx, keys)
        keys = ctx.gen_galois_keys(encmat.required_rotation_steps(ea.meta, eb.meta), keys, device=mode)
        mc = engine.MaskCache(ctx, 16)
        p = encmat.pair_array(ea.meta, eb.meta)
        mc.prewarm(np.unique(np.minimum(p[:, 2], p[:, 3])))
        from paper_2604_11659_b200._lib import lib as L_
        L_().hs_set_batch_bytes(ctx.handle, 64 << 20)      # force many small batches
        r = engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
        res[mode] = r.ctxt.host()
        if mode == "lazy":
            assert lib().hs_keys_generated(ctx.handle) >= len(keys.galois)
            assert lib().hs_key_count(ctx.handle) == 1     # only the relin key stays resident
    assert np.array_equal(res[False], res["lazy"])


def test_runner_n65536_lazy_keys_matches_oracle(pkg, oracle_mod):
    """N = 2^16 (the north-star ring degree), L = 3, keys generated on demand."""
    from paper_2604_11659_b200 import encmat, engine, formats
    O = oracle_mod
    n, sb, L, seed, dim = 1 << 16, 50, 3, 2024, 6
    params = pkg.build_params(n, sb, L, seed)
    ctx = pkg.CkksContext(params)
    keys = ctx.keygen()
    a = formats.generate_random_sparse(dim, 0.6, (17, 0))
    b = formats.generate_random_sparse(dim, 0.6, (17, 1))
    ea = encmat.encrypt_sparse(a, encmat.Layout.CSR, ctx, keys)
    eb = encmat.encrypt_sparse(b, encmat.Layout.CSC, ctx, keys)
    steps = encmat.required_rotation_steps(ea.meta, eb.meta)
    keys = ctx.gen_galois_keys(steps, keys, device="lazy")
    pairs = encmat.pair_array(ea.meta, eb.meta)
    mc = engine.MaskCache(ctx, dim)
    mc.prewarm(np.unique(np.minimum(pairs[:, 2], pairs[:, 3])))
    res = engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
    octx = O.OracleContext(O.build_params(n, sb, L, seed))
    okeys = octx.keygen()
    octx.gen_galois_keys(O.rotation_steps(pairs.tolist(), dim), okeys)
    masks = {int(p): np.stack(mc.get(int(p)).limbs) for p in np.unique(np.minimum(pairs[:, 2], pairs[:, 3]))}
    want = octx.spmspm(ea.ctxt.host(), eb.ctxt.host(), pairs, dim, masks, okeys)
    assert np.array_equal(res.ctxt.host(), want)
    err = O.frobenius_error(encmat.decrypt_result(res, ctx, keys), O.plain_matmul(a, b))
    assert err < 1e-6, err
