"""The C-ABI library loads on a CPU-only host and exports every declared symbol.

No compute calls here (no GPU in the build container); only the host-side
planner, which is plain C++, is exercised.
"""
import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hespmm_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_header_symbols():
    from paper_2604_11659_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes binding covers exactly the header
    assert set(_lib.EXPORTS) == set(syms)


def test_binding_loads_and_reports_version():
    from paper_2604_11659_b200 import _lib
    L = _lib.lib()
    assert b"sm_100a" in L.hs_version()


def test_sm100a_cubin_in_library():
    """The fatbinary carries sm_100a SASS (cross-compiled here)."""
    from paper_2604_11659_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_planner_matches_oracle_pair_schedule(oracle_mod):
    """hs_plan_csr_csc (host C++) == the reference two-pointer merge."""
    O = oracle_mod
    from paper_2604_11659_b200.encmat import Layout, meta_and_values, plan_csr_csc
    for dim, sp, seed in [(4, 0.0, 1), (8, 0.5, 2), (16, 0.75, 3), (32, 0.9, 4), (5, 1.0, 5)]:
        a = O.generate_random_sparse(dim, sp, (seed, 0))
        b = O.generate_random_sparse(dim, sp, (seed, 1))
        ma, _ = meta_and_values(a, Layout.CSR)
        mb, _ = meta_and_values(b, Layout.CSC)
        got = plan_csr_csc(ma, mb)
        oa, ia, _ = O.csr_pack(a)
        ob, ib, _ = O.csc_pack(b)
        want = np.array(O.pair_schedule_csr_csc(oa, ia, ob, ib, dim), dtype=np.int64).reshape(-1, 4)
        assert np.array_equal(got, want)
