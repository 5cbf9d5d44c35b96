"""Generate golden vectors by running the REAL reference package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch dir, builds the reference's Cython
kernels there (setup.py build_ext --inplace, nothing is written under
/root/reference), imports ``hespmm`` from that copy and records inputs and
outputs of the hot-path primitives and the CSR/C runner.  Large arrays are
stored as SHA-256 digests of their little-endian uint64 bytes; inputs are
re-created from the seeds recorded alongside, so the fixtures stay small.

Outputs: tests/golden/golden_small.npz (full arrays, n <= 1024) and
tests/golden/golden.json (chains, digests, counters, scales).
"""

import hashlib
import json
import os
import shutil
import subprocess
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SCRATCH = "/tmp/hespmm_ref_golden"


def ref_import():
    if not os.path.exists(os.path.join(SCRATCH, "src/hespmm/_kernels")):
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", SCRATCH)
        subprocess.run(["chmod", "-R", "u+w", SCRATCH], check=True)
    env = dict(os.environ)
    if os.path.exists("/usr/bin/gcc"):
        env["CC"] = "/usr/bin/gcc"
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                   check=True, capture_output=True, env=env)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import hespmm
    assert hespmm.get_backend() == "cython"
    return hespmm


def h(a) -> str:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return hashlib.sha256(a.astype("<u8").tobytes()).hexdigest()


def ct_arr(ct):
    return np.array([np.stack(p) for p in ct.polys], dtype=np.uint64)


def main():
    hespmm = ref_import()
    from hespmm import _kernels as K
    from hespmm.ckks import CkksContext, build_params
    from hespmm.ckks.params import prime_tables
    from hespmm.encmat import (Layout, decrypt_result, encrypt_sparse, pair_schedule,
                               required_rotation_steps)
    from hespmm.engine import MaskCache, OpCounter, spmm_csr_csc
    from hespmm.formats import generate_random_sparse
    from hespmm.oracle import frobenius_error, plain_matmul

    small = {}
    meta = {"generator": "tests/golden/make_golden.py", "reference_backend": hespmm.get_backend(),
            "numpy": np.__version__, "chains": {}, "kernels": {}, "ops": {}, "runner": {}}

    # 1. parameter chains (params.py:170-205)
    for (n, sb, L, seed) in [(64, 40, 2, 7), (64, 40, 3, 7), (64, 35, 2, 3), (1024, 45, 2, 2024),
                             (8192, 40, 4, 2024), (16384, 50, 2, 2024), (16384, 40, 2, 2024),
                             (65536, 50, 24, 2024), (131072, 50, 35, 2024)]:
        P = build_params(n, sb, L, seed)
        meta["chains"][f"{n}_{sb}_{L}_{seed}"] = {"chain": [int(q) for q in P.modulus_chain],
                                                 "aux": int(P.aux_prime)}

    # 2. limb kernels (_fast.pyx) -- inputs from default_rng(seed)
    for (n, sb, L, seed) in [(64, 35, 2, 3), (1024, 45, 2, 2024), (16384, 50, 2, 2024),
                             (65536, 50, 2, 2024)]:
        P = build_params(n, sb, L, seed)
        primes = [*P.modulus_chain, P.aux_prime]
        key = f"{n}_{sb}_{L}_{seed}"
        rec = {}
        for pi, q in enumerate(primes):
            t = prime_tables(q, n)
            rng = np.random.default_rng(1000 + pi)
            a = rng.integers(0, q, n, dtype=np.uint64)
            b = rng.integers(0, q, n, dtype=np.uint64)
            acc = rng.integers(0, q, n, dtype=np.uint64)
            s = int(rng.integers(0, 2**62))
            q_dst = primes[(pi + 1) % len(primes)]
            outs = {
                "roots": t.roots, "roots_sh": t.roots_sh, "iroots": t.iroots,
                "iroots_sh": t.iroots_sh,
                "ntt": K.ntt(a, q, t.roots, t.roots_sh),
                "intt": K.intt(a, q, t.iroots, t.iroots_sh, t.n_inv),
                "add": K.add_mod(a, b, q), "sub": K.sub_mod(a, b, q), "neg": K.neg_mod(a, q),
                "mul": K.mul_mod(a, b, q, t.mu), "scalar": K.scalar_mul_mod(a, s, q),
                "extend": K.extend_mod(a, q, q_dst),
            }
            f = acc.copy()
            K.fma_mod(f, a, b, q, t.mu)
            outs["fma"] = f
            rec[str(pi)] = {"q": int(q), "mu": int(t.mu), "n_inv": int(t.n_inv), "s": s,
                            "q_dst": int(q_dst), "digests": {k: h(v) for k, v in outs.items()}}
            if n <= 1024:
                for k, v in outs.items():
                    small[f"k_{key}_{pi}_{k}"] = np.asarray(v, dtype=np.uint64)
        meta["kernels"][key] = rec

    # 3. CKKS primitives on identical inputs (context.py:317-498)
    for (n, sb, L, seed) in [(64, 40, 2, 7), (64, 40, 3, 7), (1024, 45, 2, 2024),
                             (16384, 50, 2, 2024)]:
        t0 = time.time()
        P = build_params(n, sb, L, seed)
        ctx = CkksContext(P)
        keys = ctx.keygen()
        key = f"{n}_{sb}_{L}_{seed}"
        slots = P.slots
        rng = np.random.default_rng(77)
        va = rng.uniform(-1, 1, min(slots, 16))
        vb = rng.uniform(-1, 1, min(slots, 16))
        ct_a = ctx.encrypt(ctx.encode(va), keys)
        ct_b = ctx.encrypt(ctx.encode(vb), keys)
        steps = [1, 3, slots - 1, -2, 5]
        keys = ctx.gen_galois_keys(steps, keys)
        rec = {"secret": h(keys.secret.astype(np.uint64) & np.uint64(0xFF)),
               "pk_b": h(np.stack(keys.public[0])), "pk_a": h(np.stack(keys.public[1])),
               "relin_b": h(np.array(keys.relin.b)), "relin_a": h(np.array(keys.relin.a)),
               "galois": {str(r): [h(np.array(k.b)), h(np.array(k.a))] for r, k in keys.galois.items()},
               "ct_a": h(ct_arr(ct_a)), "ct_b": h(ct_arr(ct_b)),
               "scale_a": ct_a.scale, "scale_b": ct_b.scale}
        arrs = {"ct_a": ct_arr(ct_a), "ct_b": ct_arr(ct_b)}
        m3 = ctx.eval_mult_ct(ct_a, ct_b)
        arrs["mult_ct"] = ct_arr(m3)
        r1 = ctx.relinearize(m3, keys)
        arrs["relin"] = ct_arr(r1)
        s1 = ctx.rescale(r1)
        arrs["rescale"] = ct_arr(s1)
        mask = ctx.encode(np.eye(1, min(slots, 16), 2).ravel(),
                          scale=float(P.modulus_chain[L - 1]), level=L - 1)
        arrs["mask"] = np.stack(mask.limbs)
        mp = ctx.eval_mult_pt(s1, mask)
        arrs["mult_pt"] = ct_arr(mp)
        s2 = ctx.rescale(mp)
        arrs["rescale2"] = ct_arr(s2)
        arrs["add"] = ct_arr(ctx.eval_add(ct_a, ct_b))
        for r in (1, 3, slots - 1, slots - 2, 5):
            arrs[f"rot_L_{r}"] = ct_arr(ctx.eval_rotate(ct_a, r, keys))
            arrs[f"rot_low_{r}"] = ct_arr(ctx.eval_rotate(s2, r, keys))
        dec = ctx.decode(ctx.decrypt(s2, keys))
        rec["scales"] = {"mult_ct": m3.scale, "rescale": s1.scale, "mult_pt": mp.scale,
                         "rescale2": s2.scale}
        rec["decoded_rescale2_first16"] = [float(x) for x in dec[:16]]
        rec["digests"] = {k: h(v) for k, v in arrs.items()}
        rec["enc_values"] = {"va_seed": 77}
        if n <= 64:
            for k, v in arrs.items():
                small[f"o_{key}_{k}"] = v
            small[f"o_{key}_relin_key"] = np.array([np.array(keys.relin.b), np.array(keys.relin.a)])
            for r, k in keys.galois.items():
                small[f"o_{key}_gk_{r}"] = np.array([np.array(k.b), np.array(k.a)])
        meta["ops"][key] = rec
        print("ops", key, f"{time.time() - t0:.1f}s")

    # 4. the CSR/C runner (engine.py:176-184), harness-style cells
    def run_case(n, sb, L, seed, dim, sparsity, mseed):
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
               "nsteps": len(steps), "frobenius": repr(err),
               "decoded": h(out.view(np.uint64)) if out.size else None}
        if res.ctxt is None:
            rec["result"] = None
        else:
            rec["result"] = h(ct_arr(res.ctxt))
            rec["scale"] = res.ctxt.scale
            rec["level"] = res.ctxt.level
            if n <= 1024:
                small[f"r_{n}_{dim}_{sparsity}_{mseed}"] = ct_arr(res.ctxt)
        print("runner", n, dim, sparsity, counter.as_dict(), f"{time.time() - t0:.1f}s")
        return rec

    cases = [(64, 40, 2, 7, 4, 0.0, 31), (64, 40, 2, 7, 4, 0.4, 41), (64, 40, 2, 7, 4, 1.0, 51),
             (64, 40, 3, 7, 4, 0.5, 61),
             # cfg1: desk-small params, 16x16 @50%, harness cell seed (bench.py:93-96)
             (1024, 45, 2, 2024, 16, 0.5, 1 * 1_000_003 + 16 * 1_009 + 0),
             (1024, 45, 2, 2024, 8, 0.9, 1 * 1_000_003 + 8 * 1_009 + 0),
             (16384, 50, 2, 2024, 8, 0.75, 1 * 1_000_003 + 8 * 1_009 + 0)]
    for c in cases:
        meta["runner"]["_".join(str(x) for x in c)] = run_case(*c)

    # 5. plaintext schedules of all four runners (encmat.py:150-251) + predicted counts
    from hespmm.encmat import meta_and_values
    from hespmm.engine import MatmulMethod as MM
    from hespmm.oracle import predicted_op_counts
    meta["schedules"] = {}
    for dim, sp, mseed in [(4, 0.3, 51), (8, 0.5, 4), (12, 0.75, 9), (16, 0.9, 2)]:
        a = generate_random_sparse(dim, sp, (mseed, 0))
        b = generate_random_sparse(dim, sp, (mseed, 1))
        for method, la, lb, skip in [(MM.CSR_C, Layout.CSR, Layout.CSC, None),
                                     (MM.VCSR_C, Layout.VCSR, Layout.VCSC, None),
                                     (MM.NAIVE_DENSE, Layout.DENSE_ROW_MAJOR, Layout.DENSE_COL_MAJOR, None),
                                     (MM.NAIVE_SPARSE, Layout.DENSE_ROW_MAJOR, Layout.DENSE_COL_MAJOR, "either")]:
            ma, va = meta_and_values(a, la)
            mb, vb = meta_and_values(b, lb)
            pairs = np.array(list(pair_schedule(ma, mb, skip=skip)), dtype=np.int64).reshape(-1, 4)
            pred = predicted_op_counts(a, b, method)
            meta["schedules"][f"{dim}_{sp}_{mseed}_{method.value}"] = {
                "pairs": h(pairs.astype(np.uint64)), "npairs": len(pairs),
                "steps": sorted(required_rotation_steps(ma, mb, skip=skip)),
                "values_a": h(np.asarray(va).view(np.uint64)), "values_b": h(np.asarray(vb).view(np.uint64)),
                "pred": [pred.matching_pairs, pred.alignment_rotations, pred.accumulation_rotations]}

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **small)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(small), "arrays")


if __name__ == "__main__":
    main()
