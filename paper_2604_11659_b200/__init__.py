"""B200-native engine for encrypted sparse x sparse matrix multiplication.

Drop-in for the hot path of the reference package ``hespmm`` (arXiv
2604.11659): CKKS ciphertext x ciphertext SpMSpM, method CSR/C.  The public
API mirrors the reference's (``CkksContext``, ``build_params``,
``encrypt_sparse``, ``spmm_csr_csc``, ``decrypt_result`` ...); all limb
arithmetic runs in hand-written sm_100a kernels behind the C-ABI of
``lib/libhespmm_b200.so`` (include/hespmm_b200.h).  There is no CPU
fallback: without the library (or a GPU) the compute entry points raise.
"""

from .errors import CapacityError, EvalError, KeyMissingError, ParameterError
from .params import CkksParams, build_params, default_params, is_prime

__version__ = "0.1.0"

__all__ = [
    "CapacityError", "EvalError", "KeyMissingError", "ParameterError",
    "CkksParams", "build_params", "default_params", "is_prime",
    "get_backend", "__version__",
]


def get_backend() -> str:
    """Name of the compute backend (the reference reports "cython"/"python")."""
    return "cuda-sm_100a"


def __getattr__(name):
    # Lazy imports keep `import paper_2604_11659_b200` torch/CUDA-free for
    # host-only tooling; the compute API loads the library on first use.
    if name in ("CkksContext", "keygen"):
        from . import context
        return getattr(context, name)
    if name in ("Ciphertext", "Plaintext", "KeyBundle", "KeySwitchKey"):
        from . import types
        return getattr(types, name)
    if name in ("Layout", "SparseMeta", "EncryptedSparseMatrix", "EncryptedResult",
                "encrypt_sparse", "decrypt_result", "pair_schedule", "required_rotation_steps"):
        from . import encmat
        return getattr(encmat, name)
    if name in ("MatmulMethod", "OpCounter", "MaskCache", "spmm_csr_csc", "spmm_vcsr",
                "matmul_naive_dense", "matmul_naive_sparse", "METHOD_RUNNERS", "METHOD_LAYOUTS",
                "fhe_spmspm_step"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
