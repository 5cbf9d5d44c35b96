"""A small HESP key container written by the REAL reference (serial.save),
for tests/test_serial.py / test_gpu_serial.py: parameters (64, 40, 2, 7),
keygen, Galois keys for steps [1, 3, slots-1, -2, 5] -- the key set whose
digests golden.json records under ops["64_40_2_7"].

    python tests/golden/make_hesp.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def main():
    from make_golden import ref_import
    ref_import()
    from hespmm.ckks import CkksContext, build_params
    from hespmm.ckks import serial
    P = build_params(64, 40, 2, 7)
    ctx = CkksContext(P)
    keys = ctx.keygen()
    keys = ctx.gen_galois_keys([1, 3, P.slots - 1, -2, 5], keys)
    serial.save(os.path.join(HERE, "keys_64_40_2_7.hesp"), P, keys)


if __name__ == "__main__":
    main()
