"""Golden vectors at the north-star parameters, from the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_big.py            # all sets
    python tests/golden/make_golden_big.py 65536_50_24_2024

Same recipe as make_golden.py (the reference is copied to /tmp and its Cython
kernels built there; nothing is written under /root/reference), at the sizes
BASELINE.json's north star names:

* (2^16, Δ=2^50, L=24): keygen, relin key, 5 Galois keys, encryption, every
  primitive (mult_ct, relin = the 25-digit x 26-modulus key switch of
  context.py:462-498, rescale 24->23->22 with the constants of :382-399, mask,
  mult_pt, add, rotations at L and L-2 with Galois keys of :176-200), the float
  scale ledger, the decoded values, plus the limb-kernel digests of all 26
  primes and one complete CSR/C runner case (4x4 @50%);
* (2^17, Δ=2^50, L=35): the same primitive set (configs[4]'s parameters);
* (2^10, Δ=2^30, L=2): a chain whose scaling primes are < 2^32, where numpy's
  ``integers(0, q)`` takes its buffered 32-bit Lemire path.

Output: tests/golden/golden_big.json (digests only; inputs are re-created from
the recorded seeds).  Existing entries for other keys are kept.
"""

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import ct_arr, h, ref_import  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "golden_big.json")

OPS_SETS = [(1024, 30, 2, 2024), (65536, 50, 24, 2024), (131072, 50, 35, 2024)]
KERNEL_SETS = [(65536, 50, 24, 2024)]
RUNNER_CASES = [(65536, 50, 24, 2024, 4, 0.5, 1 * 1_000_003 + 4 * 1_009 + 0),
                (1024, 30, 2, 2024, 8, 0.5, 1 * 1_000_003 + 8 * 1_009 + 0)]


def record_kernels(hespmm, n, sb, L, seed):
    from hespmm import _kernels as K
    from hespmm.ckks import build_params
    from hespmm.ckks.params import prime_tables
    P = build_params(n, sb, L, seed)
    primes = [*P.modulus_chain, P.aux_prime]
    rec = {}
    for pi, q in enumerate(primes):
        t = prime_tables(q, n)
        rng = np.random.default_rng(1000 + pi)
        a = rng.integers(0, q, n, dtype=np.uint64)
        b = rng.integers(0, q, n, dtype=np.uint64)
        acc = rng.integers(0, q, n, dtype=np.uint64)
        s = int(rng.integers(0, 2**62))
        q_dst = primes[(pi + 1) % len(primes)]
        outs = {"ntt": K.ntt(a, q, t.roots, t.roots_sh),
                "intt": K.intt(a, q, t.iroots, t.iroots_sh, t.n_inv),
                "mul": K.mul_mod(a, b, q, t.mu), "extend": K.extend_mod(a, q, q_dst)}
        f = acc.copy()
        K.fma_mod(f, a, b, q, t.mu)
        outs["fma"] = f
        rec[str(pi)] = {"q": int(q), "q_dst": int(q_dst),
                        "digests": {k: h(v) for k, v in outs.items()}}
    return rec


def record_ops(hespmm, n, sb, L, seed):
    """Same pipeline and record format as make_golden.py section 3."""
    from hespmm.ckks import CkksContext, build_params
    t0 = time.time()
    P = build_params(n, sb, L, seed)
    ctx = CkksContext(P)
    keys = ctx.keygen()
    slots = P.slots
    rng = np.random.default_rng(77)
    va = rng.uniform(-1, 1, min(slots, 16))
    vb = rng.uniform(-1, 1, min(slots, 16))
    ct_a = ctx.encrypt(ctx.encode(va), keys)
    ct_b = ctx.encrypt(ctx.encode(vb), keys)
    keys = ctx.gen_galois_keys([1, 3, slots - 1, -2, 5], keys)
    print("  keys", f"{time.time() - t0:.1f}s", flush=True)
    rec = {"secret": h(keys.secret.astype(np.uint64) & np.uint64(0xFF)),
           "pk_b": h(np.stack(keys.public[0])), "pk_a": h(np.stack(keys.public[1])),
           "relin_b": h(np.array(keys.relin.b)), "relin_a": h(np.array(keys.relin.a)),
           "galois": {str(r): [h(np.array(k.b)), h(np.array(k.a))] for r, k in keys.galois.items()},
           "scale_a": ct_a.scale, "scale_b": ct_b.scale}
    dg = {"ct_a": h(ct_arr(ct_a)), "ct_b": h(ct_arr(ct_b))}
    rec["ct_a"], rec["ct_b"] = dg["ct_a"], dg["ct_b"]
    m3 = ctx.eval_mult_ct(ct_a, ct_b)
    dg["mult_ct"] = h(ct_arr(m3))
    r1 = ctx.relinearize(m3, keys)
    dg["relin"] = h(ct_arr(r1))
    s1 = ctx.rescale(r1)
    dg["rescale"] = h(ct_arr(s1))
    mask = ctx.encode(np.eye(1, min(slots, 16), 2).ravel(),
                      scale=float(P.modulus_chain[L - 1]), level=L - 1)
    dg["mask"] = h(np.stack(mask.limbs))
    mp = ctx.eval_mult_pt(s1, mask)
    dg["mult_pt"] = h(ct_arr(mp))
    s2 = ctx.rescale(mp)
    dg["rescale2"] = h(ct_arr(s2))
    dg["add"] = h(ct_arr(ctx.eval_add(ct_a, ct_b)))
    for r in (1, 3, slots - 1, slots - 2, 5):
        dg[f"rot_L_{r}"] = h(ct_arr(ctx.eval_rotate(ct_a, r, keys)))
        dg[f"rot_low_{r}"] = h(ct_arr(ctx.eval_rotate(s2, r, keys)))
    dec = ctx.decode(ctx.decrypt(s2, keys))
    rec["scales"] = {"mult_ct": m3.scale, "rescale": s1.scale, "mult_pt": mp.scale,
                     "rescale2": s2.scale}
    rec["decoded_rescale2_first16"] = [float(x) for x in dec[:16]]
    rec["digests"] = dg
    rec["enc_values"] = {"va_seed": 77}
    print("  ops", f"{time.time() - t0:.1f}s", flush=True)
    return rec


def record_runner(hespmm, n, sb, L, seed, dim, sparsity, mseed):
    """Same record format as make_golden.py section 4."""
    from hespmm.ckks import CkksContext, build_params
    from hespmm.encmat import (Layout, decrypt_result, encrypt_sparse, pair_schedule,
                               required_rotation_steps)
    from hespmm.engine import MaskCache, OpCounter, spmm_csr_csc
    from hespmm.formats import generate_random_sparse
    from hespmm.oracle import frobenius_error, plain_matmul
    t0 = time.time()
    P = build_params(n, sb, L, seed)
    ctx = CkksContext(P)
    keys = ctx.keygen()
    a = generate_random_sparse(dim, sparsity, (mseed, 0))
    b = generate_random_sparse(dim, sparsity, (mseed, 1))
    ea = encrypt_sparse(a, Layout.CSR, ctx, keys)
    eb = encrypt_sparse(b, Layout.CSC, ctx, keys)
    steps = required_rotation_steps(ea.meta, eb.meta)
    keys = ctx.gen_galois_keys(steps, keys) if steps else keys
    mc = MaskCache(ctx, dim)
    mc.prewarm(min(ap, bp) for _, _, ap, bp in pair_schedule(ea.meta, eb.meta))
    counter = OpCounter()
    res = spmm_csr_csc(ea, eb, ctx, keys, counter, mc)
    out = decrypt_result(res, ctx, keys)
    err = frobenius_error(out, plain_matmul(a, b))
    rec = {"params": [n, sb, L, seed], "dim": dim, "sparsity": sparsity, "mseed": mseed,
           "counters": counter.as_dict(),
           "alignment_rotations": counter.alignment_rotations,
           "accumulation_rotations": counter.accumulation_rotations,
           "relin_noops_ctx": ctx.relin_noops,
           "ct_a": h(ct_arr(ea.ctxt)), "ct_b": h(ct_arr(eb.ctxt)),
           "steps": sorted(int(s) for s in steps),
           "nsteps": len(steps), "frobenius": repr(err),
           "galois": {str(r): [h(np.array(k.b)), h(np.array(k.a))]
                      for r, k in sorted(keys.galois.items())[:3]},
           "decoded": h(out.view(np.uint64)) if out.size else None}
    if res.ctxt is None:
        rec["result"] = None
    else:
        rec["result"] = h(ct_arr(res.ctxt))
        rec["scale"] = res.ctxt.scale
        rec["level"] = res.ctxt.level
    print("  runner", n, dim, sparsity, counter.as_dict(), f"{time.time() - t0:.1f}s", flush=True)
    return rec


def main(only=None):
    hespmm = ref_import()
    meta = {"generator": "tests/golden/make_golden_big.py", "numpy": np.__version__,
            "reference_backend": hespmm.get_backend(), "kernels": {}, "ops": {}, "runner": {}}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            meta.update(json.load(fh))

    def save():
        with open(OUT, "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)

    def want(key):
        return only is None or key.startswith(only)

    for s in KERNEL_SETS:
        key = "_".join(map(str, s))
        if want(key):
            print("kernels", key, flush=True)
            meta["kernels"][key] = record_kernels(hespmm, *s)
            save()
    for s in OPS_SETS:
        key = "_".join(map(str, s))
        if want(key):
            print("ops", key, flush=True)
            meta["ops"][key] = record_ops(hespmm, *s)
            save()
    for c in RUNNER_CASES:
        key = "_".join(str(x) for x in c)
        if want(key):
            print("runner", key, flush=True)
            meta["runner"][key] = record_runner(hespmm, *c)
            save()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
