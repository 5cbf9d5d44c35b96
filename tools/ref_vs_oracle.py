"""Time the REAL reference (hespmm, Cython backend, built from /root/reference
like tests/golden/make_golden.py) against the CPU oracle (oracle/hs_oracle.c,
one thread) on the same CSR/C pairs, and check they agree bit for bit.
Build container only (the reference cannot travel to the GPU box).

    python tools/ref_vs_oracle.py [n log2] [L] [pairs]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def main(logn=14, L=2, npairs=24):
    from make_golden import ref_import
    ref_import()
    from hespmm.ckks import CkksContext, build_params
    from hespmm.encmat import Layout, encrypt_sparse, pair_schedule
    from hespmm.engine import MaskCache, OpCounter, _run_schedule
    from hespmm.formats import generate_random_sparse
    from oracle import oracle as O
    from paper_2604_11659_b200.refadapter import _key_array
    n, sb, dim = 1 << logn, 50, 64
    P = build_params(n, sb, L, 2024)
    ctx = CkksContext(P)
    keys = ctx.keygen()
    seed = 1 * 1_000_003 + dim * 1_009
    a = generate_random_sparse(dim, 0.75, (seed, 0))
    b = generate_random_sparse(dim, 0.75, (seed, 1))
    ea = encrypt_sparse(a, Layout.CSR, ctx, keys)
    eb = encrypt_sparse(b, Layout.CSC, ctx, keys)
    pairs = list(pair_schedule(ea.meta, eb.meta))[:npairs]
    steps = set()
    for i, j, ap, bp in pairs:
        if ap != bp:
            steps.add(abs(ap - bp))
        mn = min(ap, bp)
        if mn != i * dim + j:
            steps.add(mn - (i * dim + j))
    keys = ctx.gen_galois_keys(sorted(steps), keys)
    mc = MaskCache(ctx, dim)
    mc.prewarm(min(ap, bp) for _, _, ap, bp in pairs)
    t0 = time.perf_counter()
    res = _run_schedule(ea, eb, iter(pairs), ctx, keys, OpCounter(), mc)
    t_ref = time.perf_counter() - t0
    octx = O.OracleContext(O.build_params(n, sb, L, 2024))
    slots = n // 2
    okeys = O.Keys(None, None, None, None, _key_array(keys.relin),
                   {r % slots: _key_array(keys.galois[r % slots]) for r in steps})
    masks = {int(min(p[2], p[3])): np.stack(mc.get(int(min(p[2], p[3]))).limbs) for p in pairs}
    ca = np.array(ea.ctxt.polys, dtype=np.uint64)
    cb = np.array(eb.ctxt.polys, dtype=np.uint64)
    t0 = time.perf_counter()
    got = octx.spmspm(ca, cb, np.array(pairs, dtype=np.int64), dim, masks, okeys, nthreads=1)
    t_or = time.perf_counter() - t0
    same = np.array_equal(got, np.array(res.ctxt.polys, dtype=np.uint64))
    print(f"n=2^{logn} L={L}: {len(pairs)} pairs; reference (hespmm {__import__('hespmm').get_backend()}, "
          f"1 thread) {t_ref / len(pairs) * 1e3:.1f} ms/pair; oracle (1 thread) "
          f"{t_or / len(pairs) * 1e3:.1f} ms/pair; bit-identical: {same}")


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
