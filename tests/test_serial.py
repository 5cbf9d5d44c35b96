"""The HESP key container (reference ckks/serial.py) on the host side:
paper_2604_11659_b200.serial indexes a container WRITTEN BY THE REFERENCE
(tests/golden/keys_64_40_2_7.hesp, tests/golden/make_hesp.py) by record
arithmetic, and the key limbs found at those offsets reproduce the
reference's golden key digests (golden.json ops["64_40_2_7"])."""
import os
import struct

import numpy as np
import pytest

from helpers import digest

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "keys_64_40_2_7.hesp")


def _ksk_host(buf, off, n, L):
    """Host unpacking of one KSK record (test oracle for the device gather)."""
    key = np.empty((2, L + 1, L + 2, n), dtype=np.uint64)
    o = off + 4
    for i in range(L + 1):
        for c in range(2):
            (cnt,) = struct.unpack_from("<I", buf, o)
            o += 4
            for m in range(cnt):
                o += 4
                key[c, i, m] = np.frombuffer(buf[o:o + 8 * n], dtype="<u8")
                o += 8 * n
    return key


def test_index_reference_container(golden):
    from paper_2604_11659_b200 import serial
    from paper_2604_11659_b200.params import build_params
    buf = open(FIX, "rb").read()
    idx = serial.index(buf)
    P = idx["params"]
    assert P == build_params(64, 40, 2, 7)
    rec = golden["ops"]["64_40_2_7"]
    n, L = P.ring_degree, P.levels
    relin = _ksk_host(buf, idx["relin"], n, L)
    assert digest(relin[0]) == rec["relin_b"] and digest(relin[1]) == rec["relin_a"]
    assert sorted(idx["galois"]) == sorted(int(r) for r in rec["galois"])
    for r, (hb, ha) in rec["galois"].items():
        k = _ksk_host(buf, idx["galois"][int(r)], n, L)
        assert digest(k[0]) == hb and digest(k[1]) == ha, r
    assert idx["ksk_bytes"] == serial.ksk_record_bytes(n, L)


def test_index_rejects_bad_containers():
    from paper_2604_11659_b200 import serial
    buf = bytearray(open(FIX, "rb").read())
    with pytest.raises(ValueError, match="bad magic"):
        serial.index(b"XXXX" + bytes(buf[4:]))
    with pytest.raises(ValueError, match="trailing"):
        serial.index(bytes(buf) + b"\0")
    bad = bytearray(buf)
    struct.pack_into("<H", bad, 4, 2)
    with pytest.raises(ValueError, match="version"):
        serial.index(bytes(bad))
