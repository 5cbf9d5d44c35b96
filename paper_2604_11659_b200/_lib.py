"""ctypes binding of libhespmm_b200.so (include/hespmm_b200.h).

The library is the only compute path of this package: there is no CPU
fallback.  If the shared object is missing or cannot be loaded, every entry
point raises ``RuntimeError`` loudly (``build()`` in ``__graft_entry__`` or
``make -C paper_2604_11659_b200/csrc`` produces it).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import CapacityError, EvalError, KeyMissingError, ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HS_LIB_PATH") or os.path.join(_HERE, "lib", "libhespmm_b200.so")  # override: A/B tools
CSRC = os.path.join(_HERE, "csrc")

c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_vp = ctypes.c_void_p


class HsCounters(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "ct_ct_mults", "pt_mults", "rotations", "relins", "relin_noops", "rescales", "adds",
        "alignment_rotations", "accumulation_rotations", "pairs", "physical_alignment",
        "has_result")] + [("plan_ms", ctypes.c_double), ("ranges", ctypes.c_int64)]


# name -> (restype, argtypes)
_SIGS = {
    "hs_last_error": (ctypes.c_char_p, []),
    "hs_version": (ctypes.c_char_p, []),
    "hs_launch_count": (ctypes.c_int64, []),
    "hs_probe_arm": (ctypes.c_int, [ctypes.c_int32]),
    "hs_probe_read": (ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(ctypes.c_double)]),
    "hs_int_peak": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_double), c_vp]),
    "hs_f64_peak": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(ctypes.c_double), c_vp]),
    "hs_ctx_create": (ctypes.c_int, [ctypes.POINTER(c_vp), ctypes.c_int, ctypes.c_uint32,
                                     ctypes.c_uint32, c_u64p, ctypes.c_uint64]),
    "hs_ctx_destroy": (None, [c_vp]),
    "hs_ctx_tables": (ctypes.c_int, [c_vp, ctypes.c_uint32, c_u64p, c_u64p, c_u64p, c_u64p,
                                     c_u64p, c_u64p]),
    "hs_key_upload": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_uint32, c_vp, ctypes.c_int, c_vp]),
    "hs_key_generate": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_uint32, c_vp, c_vp, c_vp, c_vp,
                                       c_vp]),
    "hs_key_download": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_uint32, c_vp, c_vp]),
    "hs_key_upload_hesp": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_uint32, c_vp, ctypes.c_int64, c_vp]),
    "hs_keygen_set_tables": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_double), c_u64p]),
    "hs_keygen_set_secret": (ctypes.c_int, [c_vp, c_vp, c_vp]),
    "hs_crt_decode": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int32, c_vp, c_vp]),
    "hs_key_generate_galois": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_uint32), c_u64p,
                                              ctypes.c_int32, c_vp]),
    "hs_keygen_register": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_uint32), c_u64p,
                                          ctypes.c_int32]),
    "hs_keygen_streams": (ctypes.c_int, [c_vp, c_u64p, ctypes.c_int32, c_vp, c_vp, c_vp]),
    "hs_keys_generated": (ctypes.c_int64, [c_vp]),
    "hs_key_has": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_uint32]),
    "hs_key_drop": (ctypes.c_int, [c_vp, ctypes.c_int, ctypes.c_uint32]),
    "hs_key_count": (ctypes.c_int64, [c_vp]),
    "hs_ntt": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                              ctypes.c_int32, c_vp]),
    "hs_signed_to_ntt": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int32, ctypes.c_int32, c_vp, c_vp]),
    "hs_seam_op": (ctypes.c_int, [ctypes.c_int32, ctypes.c_uint64, c_vp, c_vp, c_vp, ctypes.c_uint64,
                                  ctypes.c_uint64, ctypes.c_uint64, c_vp]),
    "hs_seam_ntt": (ctypes.c_int, [c_vp, ctypes.c_uint32, ctypes.c_uint64, c_vp, c_vp,
                                   ctypes.c_uint64, ctypes.c_int32, c_vp]),
    "hs_eval_add": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_uint32, c_vp]),
    "hs_eval_mult_ct": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_uint32, c_vp]),
    "hs_eval_mult_pt": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_int32, c_vp]),
    "hs_relinearize": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_uint32, c_vp]),
    "hs_rescale": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_uint32, ctypes.c_uint32, c_vp]),
    "hs_eval_rotate": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_uint32, ctypes.c_uint32, c_vp]),
    "hs_eval_rotate_hoisted": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(c_vp),
                                              ctypes.POINTER(ctypes.c_uint32), ctypes.c_int32,
                                              ctypes.c_uint32, c_vp]),
    "hs_encrypt": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.c_uint32, c_vp,
                                  c_vp]),
    "hs_decrypt": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.c_uint32, c_vp, c_vp]),
    "hs_to_montgomery": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int32, c_vp]),
    "hs_plan_csr_csc": (ctypes.c_int, [ctypes.c_int32, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p,
                                       ctypes.c_int64, c_i64p]),
    "hs_spmspm_csr_csc": (ctypes.c_int, [c_vp, ctypes.c_int32, c_i64p, c_i64p, c_i64p, c_i64p, c_vp,
                                         c_vp, ctypes.POINTER(c_vp), ctypes.c_int64, c_vp,
                                         ctypes.POINTER(HsCounters), ctypes.c_int32,
                                         ctypes.c_int32, c_vp]),
    "hs_spmspm_pairs": (ctypes.c_int, [c_vp, ctypes.c_int32, c_i64p, ctypes.c_int64, c_vp, c_vp,
                                       ctypes.POINTER(c_vp), ctypes.c_int64, c_vp,
                                       ctypes.POINTER(HsCounters), ctypes.c_int32, ctypes.c_int32,
                                       c_vp]),
    "hs_spmspm_multi": (ctypes.c_int, [c_vp, ctypes.c_int32, c_i64p, ctypes.c_int64, ctypes.POINTER(c_vp),
                                       ctypes.POINTER(c_vp), ctypes.c_int32, ctypes.POINTER(c_vp),
                                       ctypes.c_int64, ctypes.POINTER(c_vp), ctypes.c_int32,
                                       ctypes.POINTER(HsCounters), ctypes.c_int32, ctypes.c_int32, c_vp]),
    "hs_reduce_mod": (ctypes.c_int, [c_vp, c_vp, ctypes.c_int32, ctypes.c_int32, c_vp]),
    "hs_set_batch_bytes": (None, [c_vp, ctypes.c_uint64]),
    "hs_align_compute": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(ctypes.c_int32),
                                        ctypes.POINTER(ctypes.c_uint32), ctypes.c_int64,
                                        ctypes.POINTER(c_vp), c_vp]),
    "hs_align_provide": (ctypes.c_int, [c_vp, ctypes.POINTER(ctypes.c_int32),
                                        ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(c_vp),
                                        ctypes.c_int64]),
    "hs_align_clear": (None, [c_vp]),
}

EXPORTS = tuple(_SIGS)

_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-j4", "-C", CSRC], check=True)
    else:
        subprocess.run(["make", "-s", "-j4", "-C", CSRC], check=True)
    return LIB_PATH


def lib():
    """The loaded library; raises if it is absent (no silent fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libhespmm_b200.so not found at {LIB_PATH}; build it with "
                "`make -C paper_2604_11659_b200/csrc` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


_EXC = {1: ParameterError, 2: CapacityError, 3: KeyMissingError, 4: EvalError}


def check(status: int) -> None:
    """Map a C-ABI status onto the reference exception types (errors.py:4-17)."""
    if status == 0:
        return
    msg = lib().hs_last_error().decode()
    exc = _EXC.get(status)
    if exc is not None:
        raise exc(msg)
    if status == 6:
        raise MemoryError(msg)
    raise RuntimeError(f"hespmm_b200 CUDA failure ({status}): {msg}")
