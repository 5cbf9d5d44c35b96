"""Multi-process (world_size 2 and 3, gloo, CPU) coverage of the multi-GPU path.

On GPUs (paper_2604_11659_b200/dist.py) every rank runs the product's shard
plan (``plan_shards``): one contiguous share of the step-sorted pair list,
and ownership of a balanced subset of the distinct alignment rotations;
owners compute their aligned operands and ``exchange_aligned`` ships them
point-to-point to the ranks that need them; partial result ciphertexts are
summed with one integer all-reduce (``reduce_partials``) and a mod-q pass.
Here the same planner, exchange and all-reduce run over gloo; the CPU oracle
(the checker) supplies the rotations and partial products, so every received
aligned operand and the combined result must match the single-process
oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _shard(pairs, dim, slots, rank, world):
    """The runner's shard rule: stable sort by accumulation step, then
    contiguous ranges np*r/world (paper_2604_11659_b200/csrc/runner.cu)."""
    mn = np.minimum(pairs[:, 2], pairs[:, 3])
    acc = (mn - (pairs[:, 0] * dim + pairs[:, 1])) % slots
    order = np.argsort(acc, kind="stable")
    n = len(pairs)
    return pairs[order[n * rank // world: n * (rank + 1) // world]]


def _case():
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import oracle as O
    P = O.build_params(256, 40, 2, 7)
    ctx = O.OracleContext(P)
    keys = ctx.keygen()
    dim = 8
    a = O.generate_random_sparse(dim, 0.5, (3, 0))
    b = O.generate_random_sparse(dim, 0.5, (3, 1))
    oa, ia, va = O.csr_pack(a)
    ob, ib, vb = O.csc_pack(b)
    ca = ctx.encrypt(ctx.encode(va), keys)
    cb = ctx.encrypt(ctx.encode(vb), keys)
    pairs = np.array(O.pair_schedule_csr_csc(oa, ia, ob, ib, dim), dtype=np.int64)
    ctx.gen_galois_keys(O.rotation_steps(pairs.tolist(), dim), keys)
    L = P.levels
    masks = {p: ctx.encode(np.eye(1, dim * dim, p).ravel(), scale=float(P.modulus_chain[L - 1]),
                           level=L - 1)[0] for p in set(np.minimum(pairs[:, 2], pairs[:, 3]).tolist())}
    return P, ctx, keys, ca[0], cb[0], pairs, dim, masks


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_11659_b200.dist import host_mod, reduce_partials
    P, ctx, keys, ca, cb, pairs, dim, masks = _case()
    mine = _shard(pairs, dim, P.slots, rank, world)
    part = ctx.spmspm(ca, cb, mine, dim, masks, keys) if len(mine) else None
    if part is None:
        part = np.zeros((2, P.levels - 1, P.ring_degree), dtype=np.uint64)
    t = torch.from_numpy(part.view(np.int64).copy())
    reduce_partials(t, None)
    full = host_mod(t.numpy().view(np.uint64), P.modulus_chain)
    out_q.put((rank, full.tobytes(), len(mine)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_partials_allreduce_to_single_process_result(world):
    P, ctx, keys, ca, cb, pairs, dim, masks = _case()
    want = ctx.spmspm(ca, cb, pairs, dim, masks, keys)
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(g[2] for g in got) == len(pairs)
    for rank, blob, _ in got:
        arr = np.frombuffer(blob, dtype=np.uint64).reshape(want.shape)
        assert np.array_equal(arr, want), rank


def _worker_owned(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_11659_b200.dist import exchange_aligned, host_mod, plan_shards, reduce_partials
    P, ctx, keys, ca, cb, pairs, dim, masks = _case()
    L = P.levels
    plan = plan_shards(pairs, dim, P.slots, world)
    src_ct = (ca, cb)

    def rotated(a):
        s, r = plan["align"][a]
        return torch.from_numpy(ctx.eval_rotate(src_ct[s], r, keys.galois, L).view(np.int64).copy())

    owned = {a: rotated(a) for a in range(len(plan["align"])) if plan["owner"][a] == rank}
    got = exchange_aligned(plan, rank, world, owned,
                           lambda: torch.zeros((2, L + 1, P.ring_degree), dtype=torch.int64))
    ok = sorted(got) == plan["need"][rank] and all(torch.equal(got[a], rotated(a)) for a in got)
    lo, hi = plan["ranges"][rank]
    mine = pairs[plan["order"][lo:hi]]
    part = ctx.spmspm(ca, cb, mine, dim, masks, keys) if len(mine) else None
    if part is None:
        part = np.zeros((2, L - 1, P.ring_degree), dtype=np.uint64)
    t = torch.from_numpy(part.view(np.int64).copy())
    reduce_partials(t, None)
    full = host_mod(t.numpy().view(np.uint64), P.modulus_chain)
    out_q.put((rank, full.tobytes(), len(mine), ok, len(owned),
               sum(1 for a in got if plan["owner"][a] != rank)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_owned_alignments_exchanged_and_partials_combine(world):
    """The product's shard planner + point-to-point exchange of owned
    aligned operands + SUM all-reduce, world 2 and 3 over gloo."""
    from paper_2604_11659_b200.dist import plan_shards
    P, ctx, keys, ca, cb, pairs, dim, masks = _case()
    want = ctx.spmspm(ca, cb, pairs, dim, masks, keys)
    plan = plan_shards(pairs, dim, P.slots, world)
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker_owned, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(g[2] for g in got) == len(pairs)
    assert sum(g[4] for g in got) == len(plan["align"])      # each alignment computed once
    assert any(g[5] for g in got)                              # something was actually exchanged
    for rank, blob, _, ok, _, _ in got:
        assert ok, rank
        arr = np.frombuffer(blob, dtype=np.uint64).reshape(want.shape)
        assert np.array_equal(arr, want), rank


def test_shard_rule_partitions_pairs():
    rng = np.random.default_rng(0)
    pairs = np.stack([rng.integers(0, 8, 50), rng.integers(0, 8, 50), rng.integers(0, 30, 50),
                      rng.integers(0, 30, 50)], axis=1)
    for world in (1, 2, 3, 8):
        parts = [_shard(pairs, 8, 128, r, world) for r in range(world)]
        assert sum(len(p) for p in parts) == len(pairs)
        merged = np.concatenate(parts)
        assert sorted(map(tuple, merged.tolist())) == sorted(map(tuple, pairs.tolist()))
