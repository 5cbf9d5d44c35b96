"""Bit-exact parity at the north-star parameters (N = 2^16, L = 24) and at
configs[4]'s (N = 2^17, L = 35), against golden vectors recorded from the
REAL reference (tests/golden/make_golden_big.py -> golden_big.json).

Covered at L = 24: the 26 limb-kernel digests, keygen (secret, public key,
relin key = the 25-digit x 26-modulus KSK of context.py:150-174), five Galois
keys (context.py:176-200) drawn on the host, replayed on the device and
generated lazily, encryption, mult_ct, the relinearisation key switch
(context.py:462-498), rescale 24 -> 23 -> 22 (context.py:382-399), mask,
mult_pt, add, rotations at L and L-2, the float scale ledger, decoded values,
and one complete CSR/C runner case (4x4 @50%, 16 pairs, 15 Galois keys) with
resident keys, lazily generated keys, and lazily generated keys through a
pool small enough to force evictions and regeneration.  The (2^10, Δ=2^30)
set has scaling primes < 2^32 (numpy's 32-bit Lemire path).
"""

import json
import os

import numpy as np
import pytest

from helpers import digest, parse_key

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def big():
    with open(os.path.join(HERE, "golden", "golden_big.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def pkg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2604_11659_b200 as P
    from paper_2604_11659_b200 import _lib
    _lib.lib()
    return P


OPS_KEYS = ["1024_30_2_2024", "65536_50_24_2024", "131072_50_35_2024"]


def _skip_missing(big, section, key):
    if key not in big[section]:
        pytest.skip(f"{key} not recorded in golden_big.json")


def test_kernels_every_prime_L24(pkg, big):
    from paper_2604_11659_b200 import kernels as K
    from paper_2604_11659_b200.params import prime_tables
    from helpers import kernel_inputs
    key = "65536_50_24_2024"
    n = parse_key(key)[0]
    for pi_s, rec in big["kernels"][key].items():
        q = rec["q"]
        t = prime_tables(q, n)
        a, b, acc, _ = kernel_inputs(q, n, int(pi_s))
        dg = rec["digests"]
        assert digest(K.ntt(a, q, t.roots, t.roots_sh)) == dg["ntt"], pi_s
        assert digest(K.intt(a, q, t.iroots, t.iroots_sh, t.n_inv)) == dg["intt"], pi_s
        assert digest(K.mul_mod(a, b, q, t.mu)) == dg["mul"], pi_s
        assert digest(K.extend_mod(a, q, rec["q_dst"])) == dg["extend"], pi_s
        f = acc.copy()
        K.fma_mod(f, a, b, q, t.mu)
        assert digest(f) == dg["fma"], pi_s


def _setup(P, key, device=False):
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
    keys = ctx.gen_galois_keys([1, 3, slots - 1, -2, 5], keys, device=device)
    return params, ctx, keys, ct_a, ct_b


@pytest.mark.parametrize("key", OPS_KEYS)
def test_keys_and_primitives_match_reference(pkg, big, key):
    _skip_missing(big, "ops", key)
    rec = big["ops"][key]
    dg = rec["digests"]
    params, ctx, keys, ca, cb = _setup(pkg, key)
    L, slots = params.levels, params.slots
    assert digest(keys.secret.astype(np.uint64) & np.uint64(0xFF)) == rec["secret"]
    assert digest(keys.public[0].cpu().numpy()) == rec["pk_b"]
    assert digest(keys.public[1].cpu().numpy()) == rec["pk_a"]
    rk = keys.relin.array()
    assert digest(rk[0]) == rec["relin_b"] and digest(rk[1]) == rec["relin_a"]
    del rk
    for r, (hb, ha) in rec["galois"].items():
        gk = keys.galois[int(r)].array()
        assert digest(gk[0]) == hb and digest(gk[1]) == ha, r
    assert digest(ca.host()) == dg["ct_a"] and digest(cb.host()) == dg["ct_b"]
    assert ca.scale == rec["scale_a"] and cb.scale == rec["scale_b"]
    m3 = ctx.eval_mult_ct(ca, cb)
    assert digest(m3.host()) == dg["mult_ct"]
    r1 = ctx.relinearize(m3, keys)
    assert digest(r1.host()) == dg["relin"]
    s1 = ctx.rescale(r1)
    assert digest(s1.host()) == dg["rescale"]
    mask = ctx.encode(np.eye(1, min(slots, 16), 2).ravel(), scale=float(params.modulus_chain[L - 1]),
                      level=L - 1)
    assert digest(np.stack(mask.limbs)) == dg["mask"]
    mp = ctx.eval_mult_pt(s1, mask)
    assert digest(mp.host()) == dg["mult_pt"]
    s2 = ctx.rescale(mp)
    assert digest(s2.host()) == dg["rescale2"]
    assert digest(ctx.eval_add(ca, cb).host()) == dg["add"]
    for r in (1, 3, slots - 1, slots - 2, 5):
        assert digest(ctx.eval_rotate(ca, r, keys).host()) == dg[f"rot_L_{r}"], r
        assert digest(ctx.eval_rotate(s2, r, keys).host()) == dg[f"rot_low_{r}"], r
    sc = rec["scales"]
    assert (m3.scale, s1.scale, mp.scale, s2.scale) == (sc["mult_ct"], sc["rescale"],
                                                        sc["mult_pt"], sc["rescale2"])
    dec = ctx.decode(ctx.decrypt(s2, keys))
    assert [float(x) for x in dec[:16]] == rec["decoded_rescale2_first16"]


@pytest.mark.parametrize("key", OPS_KEYS)
def test_device_galois_keys_match_reference(pkg, big, key):
    """device=True: each step's numpy stream replayed on the GPU (keygen.cu)."""
    _skip_missing(big, "ops", key)
    rec = big["ops"][key]
    n, sb, L, seed = parse_key(key)
    params = pkg.build_params(n, sb, L, seed)
    ctx = pkg.CkksContext(params)
    keys = ctx.keygen()
    keys = ctx.gen_galois_keys([1, 3, params.slots - 1, -2, 5], keys, device=True)
    for r, (hb, ha) in rec["galois"].items():
        arr = keys.galois[int(r)].array()
        assert digest(arr[0]) == hb and digest(arr[1]) == ha, r


@pytest.mark.parametrize("key", OPS_KEYS)
def test_lazy_rotations_match_reference(pkg, big, key):
    """device="lazy": eval_rotate generates the registered key on demand."""
    _skip_missing(big, "ops", key)
    dg = big["ops"][key]["digests"]
    params, ctx, keys, ca, cb = _setup(pkg, key, device="lazy")
    for r in (1, 3, params.slots - 1):
        assert digest(ctx.eval_rotate(ca, r, keys).host()) == dg[f"rot_L_{r}"], r
    outs = ctx.eval_rotate_hoisted(ca, [params.slots - 2, 5], keys)
    assert digest(outs[0].host()) == dg[f"rot_L_{params.slots - 2}"]
    assert digest(outs[1].host()) == dg["rot_L_5"]


def _runner(P, rec, device, batch_bytes=None):
    from paper_2604_11659_b200 import encmat, engine, formats
    from paper_2604_11659_b200._lib import lib
    n, sb, L, seed = rec["params"]
    params = P.build_params(n, sb, L, seed)
    ctx = P.CkksContext(params)
    keys = ctx.keygen()
    a = formats.generate_random_sparse(rec["dim"], rec["sparsity"], (rec["mseed"], 0))
    b = formats.generate_random_sparse(rec["dim"], rec["sparsity"], (rec["mseed"], 1))
    ea = encmat.encrypt_sparse(a, encmat.Layout.CSR, ctx, keys)
    eb = encmat.encrypt_sparse(b, encmat.Layout.CSC, ctx, keys)
    steps = encmat.required_rotation_steps(ea.meta, eb.meta)
    assert sorted(int(s) for s in steps) == rec["steps"]
    keys = ctx.gen_galois_keys(steps, keys, device=device)
    if batch_bytes:
        lib().hs_set_batch_bytes(ctx.handle, int(batch_bytes))
    mc = engine.MaskCache(ctx, rec["dim"])
    mc.prewarm(min(ap, bp) for _, _, ap, bp in encmat.pair_schedule(ea.meta, eb.meta))
    counter = engine.OpCounter()
    res = engine.spmm_csr_csc(ea, eb, ctx, keys, counter, mc)
    return params, ctx, keys, a, b, ea, eb, res, counter


RUNNER_MODES = [("65536_50_24_2024_4_0.5_1004039", False, None),
                ("65536_50_24_2024_4_0.5_1004039", "lazy", None),
                # two keys per batch -> a 4-key pool for 15 steps: evicts and regenerates
                ("65536_50_24_2024_4_0.5_1004039", "lazy", 1400 << 20),
                ("1024_30_2_2024_8_0.5_1008075", False, None),
                ("1024_30_2_2024_8_0.5_1008075", "lazy", 1 << 20)]


@pytest.mark.parametrize("case,device,batch_bytes", RUNNER_MODES)
def test_runner_matches_reference(pkg, big, oracle_mod, case, device, batch_bytes):
    from paper_2604_11659_b200 import encmat
    from paper_2604_11659_b200._lib import lib
    _skip_missing(big, "runner", case)
    rec = big["runner"][case]
    params, ctx, keys, a, b, ea, eb, res, counter = _runner(pkg, rec, device, batch_bytes)
    assert digest(ea.ctxt.host()) == rec["ct_a"] and digest(eb.ctxt.host()) == rec["ct_b"]
    assert counter.as_dict() == rec["counters"]
    assert counter.alignment_rotations == rec["alignment_rotations"]
    assert counter.accumulation_rotations == rec["accumulation_rotations"]
    assert ctx.relin_noops == rec["relin_noops_ctx"]
    assert digest(res.ctxt.host()) == rec["result"]
    assert res.ctxt.scale == rec["scale"] and res.ctxt.level == rec["level"]
    if device == "lazy":
        if min(params.modulus_chain) < 1 << 32:
            # numpy's 32-bit Lemire path: drawn on the host, kept resident
            assert lib().hs_key_count(ctx.handle) == 1 + rec["nsteps"]
        else:
            # every key generated on the device (with a small pool: some twice)
            assert lib().hs_keys_generated(ctx.handle) >= rec["nsteps"]
    out = encmat.decrypt_result(res, ctx, keys)
    O = oracle_mod
    assert repr(O.frobenius_error(out, O.plain_matmul(a, b))) == rec["frobenius"]
    assert digest(out.view(np.uint64)) == rec["decoded"]
