"""Host-side logic of the drop-in API against the reference's golden schedules.

Plaintext packing (traversal order), pair schedules of all four runners, the
rotation-step sets and the count predictor -- the parts of the path that run
on the host (the CSR x CSC planner is the C++ one inside libhespmm_b200.so,
callable without a GPU).
"""

import numpy as np
import pytest

from helpers import digest


def _schedule_cases(golden):
    for key, rec in golden["schedules"].items():
        dim, sp, mseed, method = key.split("_", 3)
        yield key, int(dim), float(sp), int(mseed), method, rec


def test_schedules_match_reference(golden):
    from paper_2604_11659_b200 import encmat, formats
    from paper_2604_11659_b200.engine import METHOD_LAYOUTS, MatmulMethod
    for key, dim, sp, mseed, method, rec in _schedule_cases(golden):
        a = formats.generate_random_sparse(dim, sp, (mseed, 0))
        b = formats.generate_random_sparse(dim, sp, (mseed, 1))
        m = MatmulMethod(method)
        la, lb = METHOD_LAYOUTS[m]
        ma, va = encmat.meta_and_values(a, la)
        mb, vb = encmat.meta_and_values(b, lb)
        assert digest(np.asarray(va).view(np.uint64)) == rec["values_a"], key
        assert digest(np.asarray(vb).view(np.uint64)) == rec["values_b"], key
        skip = "either" if m is MatmulMethod.NAIVE_SPARSE else None
        pairs = encmat.pair_array(ma, mb, skip)
        assert len(pairs) == rec["npairs"], key
        assert digest(pairs.astype(np.uint64)) == rec["pairs"], key
        assert sorted(encmat.required_rotation_steps(ma, mb, skip=skip)) == rec["steps"], key
        # the logical counts the runner reports = the reference predictor
        align = int(np.count_nonzero(pairs[:, 2] != pairs[:, 3])) if len(pairs) else 0
        accum = int(np.count_nonzero(np.minimum(pairs[:, 2], pairs[:, 3])
                                     != pairs[:, 0] * dim + pairs[:, 1])) if len(pairs) else 0
        assert [len(pairs), align, accum] == rec["pred"], key
        # and pair_schedule iterates the same tuples
        assert list(encmat.pair_schedule(ma, mb, skip)) == [tuple(r) for r in pairs.tolist()]


def test_oracle_csr_schedule_matches_reference(golden, oracle_mod):
    O = oracle_mod
    for key, dim, sp, mseed, method, rec in _schedule_cases(golden):
        if method != "csr_c":
            continue
        a = O.generate_random_sparse(dim, sp, (mseed, 0))
        b = O.generate_random_sparse(dim, sp, (mseed, 1))
        oa, ia, _ = O.csr_pack(a)
        ob, ib, _ = O.csc_pack(b)
        pairs = np.array(O.pair_schedule_csr_csc(oa, ia, ob, ib, dim), dtype=np.int64).reshape(-1, 4)
        assert digest(pairs.astype(np.uint64)) == rec["pairs"], key
        assert sorted(O.rotation_steps(pairs.tolist(), dim)) == rec["steps"]


def test_generate_random_sparse_matches_oracle(oracle_mod):
    from paper_2604_11659_b200 import formats
    for dim, sp, seed in [(1, 0.0, 1), (7, 0.5, (3, 1)), (64, 0.75, (1_064_579, 0)), (5, 1.0, 2)]:
        assert np.array_equal(formats.generate_random_sparse(dim, sp, seed),
                              oracle_mod.generate_random_sparse(dim, sp, seed))


def test_layout_and_capacity_errors():
    from paper_2604_11659_b200 import encmat
    from paper_2604_11659_b200.errors import ParameterError
    ma, _ = encmat.meta_and_values(np.eye(2), encmat.Layout.CSR)
    mb, _ = encmat.meta_and_values(np.eye(2), encmat.Layout.CSR)
    with pytest.raises(ParameterError, match="unsupported layout pair"):
        encmat.pair_array(ma, mb)
    mc, _ = encmat.meta_and_values(np.eye(3), encmat.Layout.CSC)
    with pytest.raises(ParameterError, match="dimensions"):
        encmat.pair_array(ma, mc)
    with pytest.raises(ParameterError, match="square"):
        encmat.meta_and_values(np.ones((2, 3)), encmat.Layout.CSR)


def test_params_validation():
    from paper_2604_11659_b200.errors import ParameterError
    from paper_2604_11659_b200.params import CkksParams, build_params
    with pytest.raises(ParameterError):
        build_params(ring_degree=12)
    p = build_params(64, 40, 2, 7)
    with pytest.raises(ParameterError, match="duplicate"):
        CkksParams(64, (p.modulus_chain[0], p.modulus_chain[0]), 40, p.aux_prime)
    assert p.slots == 32 and p.levels == 2 and p.max_matrix_dim() == 5


def test_shard_plan_owns_each_alignment_once_and_balances():
    """dist.plan_shards on the bench workloads' real schedules (configs[1],
    configs[2]): every distinct alignment rotation has exactly one owner,
    owners carry at most ~1.1x (asserted: 1.3x) the ideal share, every rank's
    needed set is covered, and the pair ranges match the runner's shard rule."""
    import bench
    from paper_2604_11659_b200 import dist, encmat, formats
    from paper_2604_11659_b200.encmat import Layout, meta_and_values
    for wl, dim, n in (("cfg2", 64, 1 << 14), ("cfg3", 128, 1 << 16)):
        seed = bench.cell_seed(dim)
        sp = bench.WORKLOADS[wl]["sparsity"]
        a = formats.generate_random_sparse(dim, sp, (seed, 0))
        b = formats.generate_random_sparse(dim, sp, (seed, 1))
        ma, _ = meta_and_values(a, Layout.CSR)
        mb, _ = meta_and_values(b, Layout.CSC)
        pairs = encmat.pair_array(ma, mb)
        for world in (2, 4, 8):
            pl = dist.plan_shards(pairs, dim, n // 2, world)
            A = len(pl["align"])
            own = np.bincount(pl["owner"], minlength=world)
            assert own.sum() == A and own.max() <= 1.3 * A / world, (wl, world, own.max(), A)
            for r, (lo, hi) in enumerate(pl["ranges"]):
                used = {int(pl["pair_align"][p]) for p in pl["order"][lo:hi] if pl["pair_align"][p] >= 0}
                assert sorted(used) == pl["need"][r]
            assert sum(hi - lo for lo, hi in pl["ranges"]) == len(pairs)


def test_shard_plan_edge_cases():
    """More ranks than pairs, no alignment at all, a single rank."""
    from paper_2604_11659_b200 import dist
    pairs = np.array([[0, 0, 0, 0], [0, 1, 1, 1]], dtype=np.int64)          # no alignment rotations
    pl = dist.plan_shards(pairs, 4, 32, 5)
    assert len(pl["align"]) == 0 and all(n == [] for n in pl["need"])
    assert sum(hi - lo for lo, hi in pl["ranges"]) == 2
    pairs = np.array([[0, 0, 0, 3], [1, 0, 2, 5], [0, 1, 4, 3]], dtype=np.int64)
    pl = dist.plan_shards(pairs, 4, 32, 1)
    assert list(pl["owner"]) == [0] * len(pl["align"])
    assert pl["need"][0] == list(range(len(pl["align"])))
    pl = dist.plan_shards(np.zeros((0, 4), dtype=np.int64), 4, 32, 3)
    assert pl["ranges"] == [(0, 0)] * 3 and len(pl["align"]) == 0
