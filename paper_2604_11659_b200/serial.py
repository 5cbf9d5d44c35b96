"""The reference's HESP key container, read straight into HBM.

Format (reference ckks/serial.py:1-134): ``b"HESP"``, u16 version (1), u16
has_keys, then u64 ring degree, u32 scale bits, u32 chain length, the chain
(u64 each), u64 aux prime, i64 seed; with keys: the secret (n int8), the
public key's two polys, the relinearisation KSK, u32 Galois key count and
per key u32 step + KSK.  A poly is a u32 limb count followed by (u32 byte
size, little-endian uint64 limb) records; a KSK is a u32 digit count
followed by the b and a polys of each digit.

``load_to_device`` never unpacks the per-limb records on the host: every
KSK record has a fixed size for given (n, L), so the file is indexed by
arithmetic, each record's bytes go file -> pinned buffer -> HBM as one copy,
and ``hs_key_upload_hesp`` gathers the limbs into the key on the device.
``dumps`` writes a container the reference's ``loads`` reads back
bit-exactly (keys downloaded from the device).
"""

from __future__ import annotations

import mmap
import struct

import numpy as np
import torch

from . import device as D
from ._lib import check, lib
from .params import CkksParams
from .types import KeyBundle, KeySwitchKey

MAGIC = b"HESP"
VERSION = 1


def _poly_bytes(nlimbs: int, n: int) -> int:
    return 4 + nlimbs * (4 + 8 * n)


def ksk_record_bytes(n: int, L: int) -> int:
    """Bytes of one KSK record: (L+1) digits x 2 polys of L+2 limbs."""
    return 4 + (L + 1) * 2 * _poly_bytes(L + 2, n)


def read_params(buf) -> tuple[CkksParams, bool, int]:
    """(params, has_keys, offset after the header) -- reference serial.py:83-104."""
    mv = memoryview(buf)
    if bytes(mv[:4]) != MAGIC:
        raise ValueError("not a hespmm key container (bad magic)")
    version, has_keys = struct.unpack_from("<HH", mv, 4)
    if version != VERSION:
        raise ValueError(f"unsupported container version {version}")
    off = 8
    n, scale_bits, chain_len = struct.unpack_from("<QII", mv, off)
    off += 16
    chain = struct.unpack_from(f"<{chain_len}Q", mv, off)
    off += 8 * chain_len
    aux, seed = struct.unpack_from("<Qq", mv, off)
    off += 16
    params = CkksParams(ring_degree=int(n), modulus_chain=tuple(int(q) for q in chain),
                        scale_bits=int(scale_bits), aux_prime=int(aux), seed=int(seed))
    return params, bool(has_keys), off


def index(buf) -> dict:
    """Byte offsets of every object in the container, by arithmetic on the
    fixed record sizes (the counts and sizes met on the way are checked)."""
    params, has_keys, off = read_params(buf)
    out = {"params": params, "has_keys": has_keys}
    if not has_keys:
        return out
    mv = memoryview(buf)
    n, L = params.ring_degree, params.levels
    out["secret"] = off
    off += n
    polys = []
    for _ in range(2):
        (cnt,) = struct.unpack_from("<I", mv, off)
        if cnt != L + 1:
            raise ValueError(f"public key poly has {cnt} limbs, expected {L + 1}")
        polys.append(off)
        off += _poly_bytes(cnt, n)
    out["public"] = polys
    rec = ksk_record_bytes(n, L)

    def ksk_at(o):
        (digits,) = struct.unpack_from("<I", mv, o)
        (cnt,) = struct.unpack_from("<I", mv, o + 4)
        (size,) = struct.unpack_from("<I", mv, o + 8)
        if digits != L + 1 or cnt != L + 2 or size != 8 * n:
            raise ValueError("KSK record shape does not match the parameters")
        return o

    out["relin"] = ksk_at(off)
    off += rec
    (ng,) = struct.unpack_from("<I", mv, off)
    off += 4
    galois = {}
    for _ in range(ng):
        (step,) = struct.unpack_from("<I", mv, off)
        galois[int(step)] = ksk_at(off + 4)
        off += 4 + rec
    out["galois"] = galois
    out["ksk_bytes"] = rec
    if off != len(mv):
        raise ValueError(f"trailing bytes in the container ({len(mv) - off})")
    return out


def _poly_array(mv, off: int, n: int) -> np.ndarray:
    (cnt,) = struct.unpack_from("<I", mv, off)
    a = np.empty((cnt, n), dtype=np.uint64)
    o = off + 4
    for k in range(cnt):
        a[k] = np.frombuffer(mv[o + 4: o + 4 + 8 * n], dtype="<u8")
        o += 4 + 8 * n
    return a


def load_to_device(path, ctx=None):
    """``(ctx, keys)`` from a reference HESP file, keys resident in HBM.

    ``ctx`` (a :class:`CkksContext` for the container's parameters) is
    created when not given; the secret and public key (small) are read on
    the host, every key switching key is copied as raw bytes to the device
    and gathered there (hs_key_upload_hesp)."""
    from .context import CkksContext
    with open(path, "rb") as fh:
        mm = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)
    try:
        idx = index(mm)
        params = idx["params"]
        if ctx is None:
            ctx = CkksContext(params)
        elif ctx.params.modulus_chain != params.modulus_chain or ctx.params.ring_degree != params.ring_degree:
            raise ValueError("container parameters differ from the context's")
        if not idx["has_keys"]:
            return ctx, None
        n = params.ring_degree
        mv = memoryview(mm)
        secret = np.frombuffer(mv[idx["secret"]: idx["secret"] + n], dtype="<i1").astype(np.int8)
        pk_b = D.to_dev(_poly_array(mv, idx["public"][0], n))
        pk_a = D.to_dev(_poly_array(mv, idx["public"][1], n))
        rec = idx["ksk_bytes"]
        host = torch.empty(rec, dtype=torch.uint8).pin_memory()
        dev = torch.empty(rec, dtype=torch.uint8, device=D.device())
        hv = host.numpy()

        def upload(kind, step, off):
            torch.cuda.current_stream().synchronize()       # the staging buffers are reused
            hv[:] = np.frombuffer(mv[off: off + rec], dtype=np.uint8)
            dev.copy_(host, non_blocking=True)
            check(lib().hs_key_upload_hesp(ctx.handle, kind, step, D.ptr(dev), rec, D.stream()))
            return KeySwitchKey(ctx, kind, step)

        relin = upload(0, 0, idx["relin"])
        galois = {r: upload(1, r, off) for r, off in idx["galois"].items()}
        torch.cuda.current_stream().synchronize()
        del mv
        return ctx, KeyBundle(secret=secret, public=(pk_b, pk_a), relin=relin, galois=galois)
    finally:
        mm.close()


def _write_poly(out: list, arr: np.ndarray) -> None:
    out.append(struct.pack("<I", arr.shape[0]))
    for limb in arr:
        data = np.ascontiguousarray(limb, dtype="<u8").tobytes()
        out.append(struct.pack("<I", len(data)))
        out.append(data)


def _write_ksk(out: list, key: np.ndarray) -> None:
    out.append(struct.pack("<I", key.shape[1]))
    for i in range(key.shape[1]):
        _write_poly(out, key[0, i])
        _write_poly(out, key[1, i])


def dumps(params: CkksParams, keys: KeyBundle | None = None) -> bytes:
    """A container the reference's ``serial.loads`` reads (serial.py:69-80)."""
    out = [MAGIC, struct.pack("<HH", VERSION, 1 if keys else 0),
           struct.pack("<QII", params.ring_degree, params.scale_bits, len(params.modulus_chain))]
    out += [struct.pack("<Q", q) for q in params.modulus_chain]
    out.append(struct.pack("<Qq", params.aux_prime, params.seed))
    if keys is not None:
        out.append(np.asarray(keys.secret, dtype="<i1").tobytes())
        for p in keys.public:
            _write_poly(out, p.cpu().numpy() if isinstance(p, torch.Tensor) else np.asarray(p))
        _write_ksk(out, keys.relin.array())
        out.append(struct.pack("<I", len(keys.galois)))
        for step in sorted(keys.galois):
            out.append(struct.pack("<I", step))
            _write_ksk(out, keys.galois[step].array())
    return b"".join(out)


def save(path, params: CkksParams, keys: KeyBundle | None = None) -> None:
    with open(path, "wb") as fh:
        fh.write(dumps(params, keys))


__all__ = ["MAGIC", "VERSION", "read_params", "index", "ksk_record_bytes", "load_to_device", "dumps",
           "save"]
