"""Bit-exact parity of the CUDA path (through the C-ABI) with the reference.

Every test compares device results either with the golden vectors recorded
from the real reference (tests/golden) or with the CPU oracle (oracle/) on
identical seeded inputs.  Integer work, so the bar is bit equality.
"""

import numpy as np
import pytest

from helpers import digest, kernel_inputs, parse_key

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2604_11659_b200 as P
    from paper_2604_11659_b200 import _lib
    _lib.lib()
    return P


# ----------------------------------------------------------- limb kernels

@pytest.mark.parametrize("key", ["64_35_2_3", "1024_45_2_2024", "16384_50_2_2024",
                                 "65536_50_2_2024"])
def test_seam_kernels_match_reference(pkg, golden, oracle_mod, key):
    from paper_2604_11659_b200 import kernels as K
    O = oracle_mod
    n, sb, L, seed = parse_key(key)
    octx = O.OracleContext(O.build_params(n, sb, L, seed))
    for pi_s, rec in golden["kernels"][key].items():
        pi = int(pi_s)
        q = rec["q"]
        t = octx.tables(pi)
        a, b, acc, s = kernel_inputs(q, n, pi)
        dg = rec["digests"]
        assert digest(K.ntt(a, q, t["roots"], t["roots_sh"])) == dg["ntt"]
        assert digest(K.intt(a, q, t["iroots"], t["iroots_sh"], t["n_inv"])) == dg["intt"]
        assert digest(K.add_mod(a, b, q)) == dg["add"]
        assert digest(K.sub_mod(a, b, q)) == dg["sub"]
        assert digest(K.neg_mod(a, q)) == dg["neg"]
        assert digest(K.mul_mod(a, b, q, t["mu"])) == dg["mul"]
        assert digest(K.scalar_mul_mod(a, s, q)) == dg["scalar"]
        assert digest(K.extend_mod(a, q, rec["q_dst"])) == dg["extend"]
        f = acc.copy()
        K.fma_mod(f, a, b, q, t["mu"])
        assert digest(f) == dg["fma"]


@pytest.mark.parametrize("log_n", list(range(3, 18)))
def test_batched_ntt_every_ring_degree(pkg, oracle_mod, log_n):
    """hs_ntt over all chain+aux primes, n = 2^3 .. 2^17, vs the oracle."""
    import torch
    from paper_2604_11659_b200 import device as D
    from paper_2604_11659_b200._lib import check, lib
    O = oracle_mod
    n = 1 << log_n
    params = pkg.build_params(n, 50 if log_n >= 12 else 40, 3, 2024)
    ctx = pkg.CkksContext(params)
    octx = O.OracleContext(O.build_params(n, params.scale_bits, 3, 2024))
    P = params.levels + 2
    rng = np.random.default_rng(log_n)
    primes = [*params.modulus_chain, params.aux_prime]
    host = np.stack([np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in primes])
                     for _ in range(3)])
    d = D.to_dev(host)
    check(lib().hs_ntt(ctx.handle, D.ptr(d), 3, P, 0, 0, D.stream()))
    fwd = D.to_host(d)
    for it in range(3):
        for p in range(P):
            assert np.array_equal(fwd[it, p], octx.ntt_limb(host[it, p], p)), (it, p)
    check(lib().hs_ntt(ctx.handle, D.ptr(d), 3, P, 0, 1, D.stream()))
    assert np.array_equal(D.to_host(d), host)
    # canonical outputs
    assert all((fwd[:, p] < primes[p]).all() for p in range(P))
    del torch


def test_ntt_extreme_inputs(pkg, oracle_mod):
    """Forward/inverse NTT of constant q-1, (q-1)/2, alternating 0/q-1 and
    one-hot limbs at N=2^16 (FP64-pipe butterflies on the ~50-bit primes,
    integer ones on the 60-bit primes) vs the oracle: the bound analysis of
    ntt.cuh unit_butterflies_f64 exercised at its largest magnitudes."""
    from paper_2604_11659_b200 import device as D
    from paper_2604_11659_b200._lib import check, lib
    O = oracle_mod
    n = 1 << 16
    params = pkg.build_params(n, 50, 3, 2024)
    ctx = pkg.CkksContext(params)
    octx = O.OracleContext(O.build_params(n, 50, 3, 2024))
    primes = [*params.modulus_chain, params.aux_prime]
    P = len(primes)
    pats = []
    for q in [np.uint64(x) for x in primes]:
        alt = np.zeros(n, dtype=np.uint64)
        alt[1::2] = q - np.uint64(1)
        one = np.zeros(n, dtype=np.uint64)
        one[n - 1] = q - np.uint64(1)
        pats.append([np.full(n, q - np.uint64(1)), np.full(n, (q - np.uint64(1)) // np.uint64(2)), alt, one])
    host = np.stack([np.stack([pats[p][k] for p in range(P)]) for k in range(4)])
    d = D.to_dev(host)
    check(lib().hs_ntt(ctx.handle, D.ptr(d), 4, P, 0, 0, D.stream()))
    fwd = D.to_host(d)
    for k in range(4):
        for p in range(P):
            assert np.array_equal(fwd[k, p], octx.ntt_limb(host[k, p], p)), (k, p)
    check(lib().hs_ntt(ctx.handle, D.ptr(d), 4, P, 0, 1, D.stream()))
    assert np.array_equal(D.to_host(d), host)


# ------------------------------------------------------- CKKS primitives

def _product_ops_pipeline(P, key):
    n, sb, L, seed = parse_key(key)
    params = P.build_params(n, sb, L, seed)
    ctx = P.CkksContext(params)
    keys = ctx.keygen()
    slots = params.slots
    rng = np.random.default_rng(77)
    va = rng.uniform(-1, 1, min(slots, 16))
    vb = rng.uniform(-1, 1, min(slots, 16))
    ct_a = ctx.encrypt(ctx.encode(va), keys)
    ct_b = ctx.encrypt(ctx.encode(vb), keys)
    keys = ctx.gen_galois_keys([1, 3, slots - 1, -2, 5], keys)
    return params, ctx, keys, ct_a, ct_b


def _arr(ct):
    return ct.host()


@pytest.mark.parametrize("key", ["64_40_2_7", "64_40_3_7", "1024_45_2_2024", "16384_50_2_2024"])
def test_keys_and_encryption_match_reference(pkg, golden, key):
    rec = golden["ops"][key]
    params, ctx, keys, ca, cb = _product_ops_pipeline(pkg, key)
    assert digest(keys.secret.astype(np.uint64) & np.uint64(0xFF)) == rec["secret"]
    assert digest(keys.public[0].cpu().numpy()) == rec["pk_b"]
    assert digest(keys.public[1].cpu().numpy()) == rec["pk_a"]
    rk = keys.relin.array()
    assert digest(rk[0]) == rec["relin_b"] and digest(rk[1]) == rec["relin_a"]
    for r, (hb, ha) in rec["galois"].items():
        gk = keys.galois[int(r)].array()
        assert digest(gk[0]) == hb and digest(gk[1]) == ha, r
    assert digest(_arr(ca)) == rec["digests"]["ct_a"]
    assert digest(_arr(cb)) == rec["digests"]["ct_b"]
    assert ca.scale == rec["scale_a"] and cb.scale == rec["scale_b"]


@pytest.mark.parametrize("key", ["64_40_2_7", "64_40_3_7", "1024_45_2_2024", "16384_50_2_2024"])
def test_primitives_match_reference(pkg, golden, key):
    rec = golden["ops"][key]
    dg = rec["digests"]
    params, ctx, keys, ca, cb = _product_ops_pipeline(pkg, key)
    L, slots = params.levels, params.slots
    m3 = ctx.eval_mult_ct(ca, cb)
    assert digest(_arr(m3)) == dg["mult_ct"]
    r1 = ctx.relinearize(m3, keys)
    assert digest(_arr(r1)) == dg["relin"]
    s1 = ctx.rescale(r1)
    assert digest(_arr(s1)) == dg["rescale"]
    mask = ctx.encode(np.eye(1, min(slots, 16), 2).ravel(), scale=float(params.modulus_chain[L - 1]),
                      level=L - 1)
    assert digest(np.stack(mask.limbs)) == dg["mask"]
    mp = ctx.eval_mult_pt(s1, mask)
    assert digest(_arr(mp)) == dg["mult_pt"]
    s2 = ctx.rescale(mp)
    assert digest(_arr(s2)) == dg["rescale2"]
    assert digest(_arr(ctx.eval_add(ca, cb))) == dg["add"]
    for r in (1, 3, slots - 1, slots - 2, 5):
        assert digest(_arr(ctx.eval_rotate(ca, r, keys))) == dg[f"rot_L_{r}"], r
        assert digest(_arr(ctx.eval_rotate(s2, r, keys))) == dg[f"rot_low_{r}"], r
    sc = rec["scales"]
    assert (m3.scale, s1.scale, mp.scale, s2.scale) == (sc["mult_ct"], sc["rescale"],
                                                        sc["mult_pt"], sc["rescale2"])
    dec = ctx.decode(ctx.decrypt(s2, keys))
    assert [float(x) for x in dec[:16]] == rec["decoded_rescale2_first16"]
    assert ctx.relinearize(s2, keys) is s2 and ctx.relin_noops == 1


@pytest.mark.parametrize("key", ["64_40_3_7", "1024_45_2_2024", "16384_50_2_2024"])
def test_hoisted_rotations_equal_single_rotations(pkg, key):
    params, ctx, keys, ca, cb = _product_ops_pipeline(pkg, key)
    slots = params.slots
    steps = [1, 3, slots - 1, -2, 5]
    outs = ctx.eval_rotate_hoisted(ca, steps, keys)
    for s, o in zip(steps, outs):
        assert np.array_equal(_arr(o), _arr(ctx.eval_rotate(ca, s, keys))), s


def test_errors_map_to_reference_exceptions(pkg):
    from paper_2604_11659_b200.errors import EvalError, KeyMissingError
    params, ctx, keys, ca, cb = _product_ops_pipeline(pkg, "64_40_2_7")
    with pytest.raises(KeyMissingError, match="missing Galois key for step 7"):
        ctx.eval_rotate(ca, 7, keys)
    low = ctx.rescale(ctx.rescale(ctx.relinearize(ctx.eval_mult_ct(ca, cb), keys)))
    with pytest.raises(EvalError, match="chain exhausted"):
        ctx.rescale(low)
    with pytest.raises(EvalError, match="level mismatch"):
        ctx.eval_add(ca, low)
    with pytest.raises(EvalError, match="degree-2"):
        ctx.decrypt(ctx.eval_mult_ct(ca, cb), keys)


# ------------------------------------------------------------------ runner

def product_runner_case(P, n, sb, L, seed, dim, sparsity, mseed, method="csr_c"):
    from paper_2604_11659_b200 import engine, encmat, formats
    params = P.build_params(n, sb, L, seed)
    ctx = P.CkksContext(params)
    keys = ctx.keygen()
    a = formats.generate_random_sparse(dim, sparsity, (mseed, 0))
    b = formats.generate_random_sparse(dim, sparsity, (mseed, 1))
    m = engine.MatmulMethod(method)
    la, lb = engine.METHOD_LAYOUTS[m]
    ea = encmat.encrypt_sparse(a, la, ctx, keys)
    eb = encmat.encrypt_sparse(b, lb, ctx, keys)
    skip = "either" if m is engine.MatmulMethod.NAIVE_SPARSE else None
    steps = encmat.required_rotation_steps(ea.meta, eb.meta, skip=skip)
    keys = ctx.gen_galois_keys(steps, keys) if steps else keys
    mc = engine.MaskCache(ctx, dim)
    mc.prewarm(min(ap, bp) for _, _, ap, bp in encmat.pair_schedule(ea.meta, eb.meta, skip=skip))
    counter = engine.OpCounter()
    res = engine.METHOD_RUNNERS[m](ea, eb, ctx, keys, counter, mc)
    return params, ctx, keys, a, b, ea, eb, res, counter, mc


def test_runner_matches_reference(pkg, golden, oracle_mod):
    from paper_2604_11659_b200 import encmat
    O = oracle_mod
    for key, rec in golden["runner"].items():
        n, sb, L, seed = rec["params"]
        params, ctx, keys, a, b, ea, eb, res, counter, mc = product_runner_case(
            pkg, n, sb, L, seed, rec["dim"], rec["sparsity"], rec["mseed"])
        assert digest(_arr(ea.ctxt)) == rec["ct_a"] and digest(_arr(eb.ctxt)) == rec["ct_b"], key
        assert counter.as_dict() == rec["counters"], key
        assert counter.alignment_rotations == rec["alignment_rotations"]
        assert counter.accumulation_rotations == rec["accumulation_rotations"]
        assert ctx.relin_noops == rec["relin_noops_ctx"]
        assert mc.misses == 0
        if rec["result"] is None:
            assert res.ctxt is None
            assert np.all(encmat.decrypt_result(res, ctx, keys) == 0.0)
            continue
        assert digest(_arr(res.ctxt)) == rec["result"], key
        assert res.ctxt.scale == rec["scale"] and res.ctxt.level == rec["level"]
        out = encmat.decrypt_result(res, ctx, keys)
        assert repr(O.frobenius_error(out, O.plain_matmul(a, b))) == rec["frobenius"], key
        assert digest(out.view(np.uint64)) == rec["decoded"], key


@pytest.mark.parametrize("method", ["csr_c", "vcsr_c", "naive_sparse", "naive_dense"])
def test_all_runners_match_oracle(pkg, oracle_mod, method):
    """Same executor, different schedules (engine.py:187-225), vs the oracle
    running the product's own schedule."""
    from paper_2604_11659_b200 import encmat
    O = oracle_mod
    n, sb, L, seed, dim = 256, 40, 2, 7, 4
    params, ctx, keys, a, b, ea, eb, res, counter, mc = product_runner_case(
        pkg, n, sb, L, seed, dim, 0.4, 99, method)
    skip = "either" if method == "naive_sparse" else None
    pairs = encmat.pair_array(ea.meta, eb.meta, skip)
    octx = O.OracleContext(O.build_params(n, sb, L, seed))
    okeys = octx.keygen()
    octx.gen_galois_keys(O.rotation_steps(pairs.tolist(), dim), okeys)
    masks = {p: np.stack(mc.get(p).limbs) for p in {int(min(r[2], r[3])) for r in pairs}}
    want = octx.spmspm(_arr(ea.ctxt), _arr(eb.ctxt), pairs, dim, masks, okeys)
    assert np.array_equal(_arr(res.ctxt), want)
    assert counter.ct_ct_mults == len(pairs)
    assert O.frobenius_error(encmat.decrypt_result(res, ctx, keys), O.plain_matmul(a, b)) < 1e-6


def test_runner_matches_oracle_deeper_chain(pkg, oracle_mod):
    """n = 2^13, L = 4 (the reference default shape), 12x12 @ 60%."""
    from paper_2604_11659_b200 import encmat
    O = oracle_mod
    n, sb, L, seed, dim = 8192, 45, 4, 2024, 12
    params, ctx, keys, a, b, ea, eb, res, counter, mc = product_runner_case(
        pkg, n, sb, L, seed, dim, 0.6, 5)
    pairs = encmat.pair_array(ea.meta, eb.meta)
    octx = O.OracleContext(O.build_params(n, sb, L, seed))
    okeys = octx.keygen()
    octx.gen_galois_keys(O.rotation_steps(pairs.tolist(), dim), okeys)
    masks = {p: np.stack(mc.get(p).limbs) for p in {int(min(r[2], r[3])) for r in pairs}}
    want = octx.spmspm(_arr(ea.ctxt), _arr(eb.ctxt), pairs, dim, masks, okeys)
    assert np.array_equal(_arr(res.ctxt), want)
    assert O.frobenius_error(encmat.decrypt_result(res, ctx, keys), O.plain_matmul(a, b)) < 1e-6


def test_sharded_runner_sums_to_full_result(pkg):
    """Shards of the step-sorted pair list summed mod q == the 1-shard result
    (the multi-GPU combine)."""
    import torch
    from paper_2604_11659_b200 import device as D
    from paper_2604_11659_b200 import engine
    from paper_2604_11659_b200._lib import check, lib
    params, ctx, keys, a, b, ea, eb, full, counter, mc = product_runner_case(
        pkg, 1024, 45, 2, 2024, 16, 0.5, 1 * 1_000_003 + 16 * 1_009)
    for world in (2, 3, 8):
        parts = []
        for r in range(world):
            res = engine.run_pairs(ea, eb, ctx, keys, engine.OpCounter(), mc, None, shard=(r, world))
            parts.append(res.ctxt.data.view(torch.int64).clone())
        summed = torch.stack(parts).sum(0)
        check(lib().hs_reduce_mod(ctx.handle, D.ptr(summed), 2, params.levels - 1, D.stream()))
        assert np.array_equal(D.to_host(summed.view(torch.uint64)), _arr(full.ctxt)), world


def test_runner_end_to_end_from_host_buffers(pkg):
    """Host-resident ciphertexts (the e2e path) give the identical result."""
    from paper_2604_11659_b200 import engine, encmat
    from paper_2604_11659_b200.types import Ciphertext
    params, ctx, keys, a, b, ea, eb, res, counter, mc = product_runner_case(
        pkg, 1024, 45, 2, 2024, 8, 0.5, 3)
    ha = encmat.EncryptedSparseMatrix(Ciphertext(_arr(ea.ctxt), ea.ctxt.scale, ea.ctxt.level), ea.meta)
    hb = encmat.EncryptedSparseMatrix(Ciphertext(_arr(eb.ctxt), eb.ctxt.scale, eb.ctxt.level), eb.meta)
    res2 = engine.spmm_csr_csc(ha, hb, ctx, keys, engine.OpCounter(), mc)
    assert np.array_equal(_arr(res2.ctxt), _arr(res.ctxt))


def test_runner_missing_key_and_layout_errors(pkg):
    from paper_2604_11659_b200 import encmat, engine, formats
    from paper_2604_11659_b200.errors import KeyMissingError, ParameterError
    params = pkg.build_params(64, 40, 2, 7)
    ctx = pkg.CkksContext(params)
    keys = ctx.keygen()
    a = formats.generate_random_sparse(4, 0.3, 1)
    ea = encmat.encrypt_sparse(a, encmat.Layout.CSR, ctx, keys)
    eb = encmat.encrypt_sparse(a, encmat.Layout.CSC, ctx, keys)
    with pytest.raises(KeyMissingError):
        engine.spmm_csr_csc(ea, eb, ctx, keys)
    with pytest.raises(ParameterError, match="layout mismatch"):
        engine.spmm_csr_csc(eb, ea, ctx, keys)


def test_bench_workload_full_size(pkg, oracle_mod):
    """The bench workload itself (BASELINE configs[1]: N = 2^14, L = 2,
    64 x 64 @ 75%, 16,434 pairs, 4,773 device-generated keys): the full product
    decrypts to the plaintext product, a sampled sub-schedule is bit-identical
    to the CPU oracle, and disjoint shards of the full schedule sum to the
    full result (size-independent properties at full size)."""
    import torch
    import bench
    from paper_2604_11659_b200 import device as D
    from paper_2604_11659_b200 import encmat, engine
    from paper_2604_11659_b200._lib import check, lib
    O = oracle_mod
    wl = dict(bench.WORKLOADS["cfg2"])
    params = pkg.build_params(wl["ring_degree"], wl["scale_bits"], wl["levels"], wl["seed"])
    ctx = pkg.CkksContext(params)
    keys = ctx.keygen()
    from paper_2604_11659_b200 import formats
    seed = bench.cell_seed(wl["dim"])
    a = formats.generate_random_sparse(wl["dim"], wl["sparsity"], (seed, 0))
    b = formats.generate_random_sparse(wl["dim"], wl["sparsity"], (seed, 1))
    ea = encmat.encrypt_sparse(a, encmat.Layout.CSR, ctx, keys)
    eb = encmat.encrypt_sparse(b, encmat.Layout.CSC, ctx, keys)
    keys = ctx.gen_galois_keys(encmat.required_rotation_steps(ea.meta, eb.meta), keys, device=True)
    pairs = encmat.pair_array(ea.meta, eb.meta)
    assert len(pairs) == 16434
    mc = engine.MaskCache(ctx, wl["dim"])
    mc.prewarm(np.unique(np.minimum(pairs[:, 2], pairs[:, 3])))
    full = engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
    err = O.frobenius_error(encmat.decrypt_result(full, ctx, keys), O.plain_matmul(a, b))
    assert err < 1e-6, err
    # shards of the full schedule sum to the full result
    parts = []
    for r in range(3):
        res = engine.run_pairs(ea, eb, ctx, keys, engine.OpCounter(), mc, None, shard=(r, 3))
        parts.append(res.ctxt.data.view(torch.int64).clone())
    summed = torch.stack(parts).sum(0)
    check(lib().hs_reduce_mod(ctx.handle, D.ptr(summed), 2, params.levels - 1, D.stream()))
    assert np.array_equal(D.to_host(summed.view(torch.uint64)), _arr(full.ctxt))
    # a sampled sub-schedule vs the oracle on identical inputs
    sub = pairs[:: len(pairs) // 48][:48]
    res = engine.run_pairs(ea, eb, ctx, keys, engine.OpCounter(), mc, sub)
    octx = O.OracleContext(O.build_params(wl["ring_degree"], wl["scale_bits"], wl["levels"], wl["seed"]))
    okeys = octx.keygen()
    octx.gen_galois_keys(O.rotation_steps(sub.tolist(), wl["dim"]), okeys)
    masks = {int(p): np.stack(mc.get(int(p)).limbs) for p in np.unique(np.minimum(sub[:, 2], sub[:, 3]))}
    want = octx.spmspm(_arr(ea.ctxt), _arr(eb.ctxt), sub, wl["dim"], masks, okeys)
    assert np.array_equal(_arr(res.ctxt), want)


@pytest.mark.parametrize("n,sb,L", [(1024, 45, 2), (16384, 50, 2), (8192, 45, 4), (65536, 50, 24)])
def test_device_crt_decode_bit_equal_to_big_int(pkg, n, sb, L):
    """csrc/decode.cu vs the reference's big-integer decode restated on the
    host, on random limbs at every level (incl. values near +-Q/2)."""
    import torch
    from paper_2604_11659_b200 import device as D
    params = pkg.build_params(n, sb, L, 2024)
    ctx = pkg.CkksContext(params)
    rng = np.random.default_rng(n + L)
    import random
    pyr = random.Random(n + L)
    for nl in sorted({1, 2, L + 1}):
        qs = [int(q) for q in params.modulus_chain[:nl]]
        Q = 1
        for q in qs:
            Q *= q
        # signed values up to 2^min(bits(Q)-2, 1000) (float() of larger ones overflows
        # in the reference too), plus the centring boundary when Q is small enough
        bits = min(Q.bit_length() - 2, 1000)
        xs = [pyr.randrange(-(1 << bits), 1 << bits) >> pyr.randrange(0, bits) for _ in range(n)]
        if Q.bit_length() < 1020:
            xs[:5] = [(Q - 1) // 2, -((Q - 1) // 2), 0, -1, 1]
        limbs = np.array([[x % q for x in xs] for q in qs], dtype=np.uint64)
        t = D.to_dev(limbs)
        # both paths INTT internally: feed NTT-domain limbs
        from paper_2604_11659_b200._lib import check, lib
        check(lib().hs_ntt(ctx.handle, D.ptr(t), 1, nl, 0, 0, D.stream()))
        got = ctx._crt_to_float(t)
        want = ctx._crt_to_float_host(t)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), nl


def test_distributed_path_single_rank_nccl(pkg):
    """The multi-GPU code path (dist.spmm_csr_csc_distributed: shard, NCCL
    int64 SUM, mod-q kernel) on a one-rank NCCL group equals the runner."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2604_11659_b200 import dist as hdist
    from paper_2604_11659_b200 import engine
    params, ctx, keys, a, b, ea, eb, full, counter, mc = product_runner_case(
        pkg, 1024, 45, 2, 2024, 8, 0.5, 3)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        res = hdist.spmm_csr_csc_distributed(ea, eb, ctx, keys, engine.OpCounter(), mc)
        assert np.array_equal(_arr(res.ctxt), _arr(full.ctxt))
        assert res.ctxt.scale == full.ctxt.scale and res.ctxt.level == full.ctxt.level
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_owned_alignments_across_simulated_ranks(pkg, world):
    """dist.py's multi-GPU plan on one GPU, ranks simulated in turn: each
    rank's owned alignments computed once (hs_align_compute), handed to the
    ranks that need them (hs_align_provide, no recomputation: the runner
    reports 0 physical alignments), shard partials summed mod q == the
    single-process result."""
    import ctypes
    import torch
    from paper_2604_11659_b200 import device as D
    from paper_2604_11659_b200 import dist as hdist
    from paper_2604_11659_b200 import engine
    from paper_2604_11659_b200._lib import check, lib
    params, ctx, keys, a, b, ea, eb, full, counter, mc = product_runner_case(
        pkg, 1024, 45, 2, 2024, 16, 0.5, 1 * 1_000_003 + 16 * 1_009)
    L, n = params.levels, params.ring_degree
    pairs = hdist._plan_pairs(ea, eb)
    plan = hdist.plan_shards(pairs, 16, n // 2, world)
    A = len(plan["align"])
    aligned = D.empty((A, 2, L + 1, n))
    for r in range(world):
        mine = [x for x in range(A) if plan["owner"][x] == r]
        srcs = (ctypes.c_int32 * len(mine))(*[plan["align"][x][0] for x in mine])
        steps = (ctypes.c_uint32 * len(mine))(*[plan["align"][x][1] for x in mine])
        outs = (ctypes.c_void_p * len(mine))(*[aligned[x].data_ptr() for x in mine])
        check(lib().hs_align_compute(ctx.handle, D.ptr(ea.ctxt.data), D.ptr(eb.ctxt.data), srcs, steps,
                                     len(mine), outs, D.stream()))
    parts = []
    for r in range(world):
        ids = plan["need"][r]
        srcs = (ctypes.c_int32 * len(ids))(*[plan["align"][x][0] for x in ids])
        steps = (ctypes.c_uint32 * len(ids))(*[plan["align"][x][1] for x in ids])
        ptrs = (ctypes.c_void_p * len(ids))(*[aligned[x].data_ptr() for x in ids])
        check(lib().hs_align_provide(ctx.handle, srcs, steps, ptrs, len(ids)))
        c = engine.OpCounter()
        res = engine.run_pairs(ea, eb, ctx, keys, c, mc, pairs, shard=(r, world))
        lib().hs_align_clear(ctx.handle)
        assert c.physical_alignment == 0          # nothing recomputed
        parts.append(res.ctxt.data.view(torch.int64).clone())
    summed = torch.stack(parts).sum(0)
    check(lib().hs_reduce_mod(ctx.handle, D.ptr(summed), 2, L - 1, D.stream()))
    assert np.array_equal(D.to_host(summed.view(torch.uint64)), _arr(full.ctxt))


def _dist_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_11659_b200 as P
        from paper_2604_11659_b200 import dist as hdist
        from paper_2604_11659_b200 import engine
        out = product_runner_case(P, 1024, 45, 2, 2024, 16, 0.5, 1 * 1_000_003 + 16 * 1_009)
        ea, eb, ctx, keys, mc = out[5], out[6], out[1], out[2], out[9]
        c = engine.OpCounter()
        res = hdist.spmm_csr_csc_distributed(ea, eb, ctx, keys, c, mc)
        q.put((rank, res.ctxt.host().tobytes(), c.physical_alignment, c.ct_ct_mults))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_runner_multiprocess(pkg, world):
    """The whole multi-GPU path (dist.spmm_csr_csc_distributed: shard plan,
    owned alignments computed once, point-to-point exchange, shard runs, SUM
    all-reduce, mod-q) in `world` processes -- on one GPU, so the collectives
    run over gloo (device tensors staged through host memory) -- equals the
    single-process runner bit for bit, and no alignment is computed twice."""
    import socket
    import torch.multiprocessing as mp
    from paper_2604_11659_b200 import dist as hdist
    params, ctx, keys, a, b, ea, eb, full, counter, mc = product_runner_case(
        pkg, 1024, 45, 2, 2024, 16, 0.5, 1 * 1_000_003 + 16 * 1_009)
    plan = hdist.plan_shards(hdist._plan_pairs(ea, eb), 16, params.slots, world)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    procs = [ctx_mp.Process(target=_dist_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = _arr(full.ctxt)
    for rank, blob, phys, mults in got:
        assert np.array_equal(np.frombuffer(blob, dtype=np.uint64).reshape(want.shape), want), rank
        assert mults == counter.ct_ct_mults
    # every rank computed exactly the alignments it owns (the runner recomputed none)
    owned = np.bincount(plan["owner"], minlength=world)
    assert {g[0]: g[2] for g in got} == {r: int(owned[r]) for r in range(world)}
