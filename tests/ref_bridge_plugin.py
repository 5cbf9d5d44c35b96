"""pytest plugin (test infrastructure): the REFERENCE's own test suite with
its CSR/C runner replaced by ``ReferenceBridge`` (the drop-in a hespmm
maintainer registers).  The bridge's device half
is swapped for the CPU oracle here (the build container has no GPU): what
this exercises is the bridge's reference-facing surface -- reading genuine
hespmm objects, the C++ planner, counters, wall time, relin no-ops, result
types and errors -- under the reference's own assertions.  Loaded by
tests/test_reference_suite.py with ``-p ref_bridge_plugin``.
"""
import numpy as np
import pytest


def _counts(pairs, dim):
    P = len(pairs)
    al = int(np.count_nonzero(pairs[:, 2] != pairs[:, 3])) if P else 0
    acc = int(np.count_nonzero(np.minimum(pairs[:, 2], pairs[:, 3]) != pairs[:, 0] * dim + pairs[:, 1])) if P else 0
    return {"ct_ct_mults": P, "pt_mults": P, "relins": P, "relin_noops": P, "rescales": 2 * P,
            "adds": max(P - 1, 0), "alignment_rotations": al, "accumulation_rotations": acc,
            "rotations": al + acc}


@pytest.hookimpl(tryfirst=True)
def pytest_configure(config):
    import hespmm.engine as E
    from oracle import oracle as O
    from paper_2604_11659_b200.refadapter import ReferenceBridge, _key_array

    class OracleBackedBridge(ReferenceBridge):
        def execute(self, x, keys):
            p = self.params
            octx = O.OracleContext(O.build_params(p.ring_degree, p.scale_bits, p.levels, p.seed))
            okeys = O.Keys(None, None, None, None, _key_array(keys.relin),
                           {r: _key_array(keys.galois[r]) for r in x["steps"]})
            res = octx.spmspm(x["ct_a"], x["ct_b"], x["pairs"], x["dim"], x["masks"], okeys)
            return res, _counts(x["pairs"], x["dim"])

        def _sync_keys(self, keys, steps):       # what the device half would check
            from hespmm.errors import KeyMissingError
            if keys.relin is None:
                raise KeyMissingError("no relinearization key in bundle")
            for r in steps:
                if keys.galois.get(r) is None:
                    raise KeyMissingError(f"missing Galois key for step {r}")

    bridges = {}
    calls = config._ref_bridge_calls = [0]

    def csr_c_runner(enc_a, enc_b, ctx, keys, counter=None, mask_cache=None):
        calls[0] += 1
        b = bridges.get(id(ctx))
        if b is None:
            b = bridges[id(ctx)] = OracleBackedBridge(ctx)
        x = b.extract(enc_a, enc_b, ctx, counter, mask_cache)
        b._sync_keys(keys, x["steps"])
        import time
        t0 = time.perf_counter()
        res, counts = b.execute(x, keys)
        return b.wrap(x, enc_a, enc_b, ctx, res, counts, time.perf_counter() - t0 + 1e-9)

    E.METHOD_RUNNERS[E.MatmulMethod.CSR_C] = csr_c_runner
    E.spmm_csr_csc = csr_c_runner
    config._ref_bridge_installed = True


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    terminalreporter.write_line(f"REF_BRIDGE_CALLS {config._ref_bridge_calls[0]}")
