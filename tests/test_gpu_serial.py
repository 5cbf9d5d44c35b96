"""HESP containers straight into HBM (paper_2604_11659_b200.serial): a
container written by the REAL reference is loaded with one raw-byte copy per
key switching key and a device gather (hs_key_upload_hesp); the keys equal
the reference's golden digests, drive the primitives to the golden results,
and ``dumps`` writes the byte-identical container back."""
import os

import numpy as np
import pytest

from helpers import digest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "keys_64_40_2_7.hesp")


def test_load_container_to_device_and_round_trip(golden):
    import torch
    assert torch.cuda.is_available()
    from paper_2604_11659_b200 import serial
    ctx, keys = serial.load_to_device(FIX)
    rec = golden["ops"]["64_40_2_7"]
    rk = keys.relin.array()
    assert digest(rk[0]) == rec["relin_b"] and digest(rk[1]) == rec["relin_a"]
    for r, (hb, ha) in rec["galois"].items():
        k = keys.galois[int(r)].array()
        assert digest(k[0]) == hb and digest(k[1]) == ha, r
    assert digest(keys.public[0].cpu().numpy()) == rec["pk_b"]
    assert digest(keys.public[1].cpu().numpy()) == rec["pk_a"]
    assert digest(keys.secret.astype(np.uint64) & np.uint64(0xFF)) == rec["secret"]
    # the loaded keys drive the primitives to the reference's results
    P = ctx.params
    rng = np.random.default_rng(77)
    va = rng.uniform(-1, 1, 16)
    vb = rng.uniform(-1, 1, 16)
    ca = ctx.encrypt(ctx.encode(va), keys)
    cb = ctx.encrypt(ctx.encode(vb), keys)
    dg = rec["digests"]
    assert digest(ca.host()) == dg["ct_a"]
    assert digest(ctx.relinearize(ctx.eval_mult_ct(ca, cb), keys).host()) == dg["relin"]
    assert digest(ctx.eval_rotate(ca, 3, keys).host()) == dg["rot_L_3"]
    # byte-identical container back
    assert serial.dumps(P, keys) == open(FIX, "rb").read()
