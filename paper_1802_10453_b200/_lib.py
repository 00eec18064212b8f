"""ctypes loader for libffldl_b200.so (the C-ABI in include/ffldl_b200.h).

The library is built in-tree (paper_1802_10453_b200/build.py).  There is no
fallback: if the shared library is missing or fails to load, importing the
package raises, and every compute call needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libffldl_b200.so")

_lib = None

# Every symbol declared in include/ffldl_b200.h (checked by tests/test_capi.py).
EXPORTS = [
    "ffb_version", "ffb_status_string", "ffb_last_error", "ffb_create", "ffb_destroy",
    "ffb_stream", "ffb_launch_count", "ffb_sync_count", "ffb_profile_enable", "ffb_profile_read",
    "ffb_ldlt", "ffb_ldlt_compact", "ffb_ldlt_zero_leading",
    "ffb_ldlt_device", "ffb_plduq", "ffb_trssyr2k", "ffb_gemm_sub", "ffb_trmm_sub",
    "ffb_trsm_inplace", "ffb_syrdk_sub", "ffb_syrdk_sub_diag", "ffb_syr2k_sub", "ffb_strictify",
    "ffb_strictify_device", "ffb_matrix_read", "ffb_matrix_write", "ffb_factorization_read",
    "ffb_factorization_write", "ffb_gemm_device", "ffb_generate_host",
    "ffb_generate_device", "ffb_config5_partners", "ffb_verify_device", "ffb_pivoting_partners_device",
]

P = C.c_void_p
SZ = C.c_size_t
U64 = C.c_uint64
I = C.c_int

_SIGS = {
    "ffb_version": (I, []),
    "ffb_status_string": (C.c_char_p, [I]),
    "ffb_last_error": (C.c_char_p, []),
    "ffb_create": (I, [C.POINTER(P), I]),
    "ffb_destroy": (I, [P]),
    "ffb_stream": (P, [P]),
    "ffb_launch_count": (U64, [P]),
    "ffb_sync_count": (U64, [P]),
    "ffb_profile_enable": (I, [P, I]),
    "ffb_profile_read": (I, [P, I, C.POINTER(U64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                             C.POINTER(C.c_double)]),
    "ffb_ldlt": (I, [P, U64, SZ, SZ, P, I, SZ, P, P, P, P, P, C.POINTER(SZ)]),
    "ffb_ldlt_compact": (I, [P, U64, SZ, P, I, I, SZ, P, P, I, P, P, P, C.POINTER(SZ)]),
    "ffb_ldlt_zero_leading": (I, [P, U64, SZ, SZ, P, SZ, P, I, SZ, P, P, P, P, P, C.POINTER(SZ)]),
    "ffb_ldlt_device": (I, [P, U64, SZ, P, SZ, I, SZ, P, P, SZ, P, P, P, C.POINTER(SZ)]),
    "ffb_plduq": (I, [P, U64, SZ, SZ, P, P, P, P, P, P, C.POINTER(SZ)]),
    "ffb_trssyr2k": (I, [P, U64, SZ, P, P, P]),
    "ffb_gemm_sub": (I, [P, U64, SZ, SZ, SZ, P, P, P]),
    "ffb_trmm_sub": (I, [P, U64, SZ, SZ, P, P, I, I, I, P]),
    "ffb_trsm_inplace": (I, [P, U64, SZ, SZ, P, I, I, I, P]),
    "ffb_syrdk_sub": (I, [P, U64, SZ, SZ, P, P, P, P, P]),
    "ffb_syr2k_sub": (I, [P, U64, SZ, SZ, P, P, P]),
    "ffb_syrdk_sub_diag": (I, [P, U64, SZ, SZ, P, P, P]),
    "ffb_matrix_read": (I, [C.c_char_p, C.POINTER(U64), C.POINTER(U64), C.POINTER(U64), C.POINTER(I), P, I]),
    "ffb_matrix_write": (I, [C.c_char_p, I, U64, U64, U64, I, P, I]),
    "ffb_factorization_read": (I, [C.c_char_p, C.POINTER(U64), C.POINTER(U64), C.POINTER(U64), P, P, I, P, P,
                                   P]),
    "ffb_factorization_write": (I, [C.c_char_p, I, U64, U64, U64, P, P, I, P, P, P]),
    "ffb_strictify": (I, [P, U64, SZ, SZ, P, P, P, P, P, C.POINTER(U64), C.POINTER(U64)]),
    "ffb_strictify_device": (I, [P, U64, SZ, SZ, P, P, SZ, P, P, P, C.POINTER(U64), C.POINTER(U64)]),
    "ffb_gemm_device": (I, [P, U64, I, SZ, SZ, SZ, P, SZ, P, SZ, I, P, SZ, I]),
    "ffb_generate_host": (I, [I, SZ, SZ, U64, U64, P]),
    "ffb_generate_device": (I, [P, I, SZ, SZ, U64, U64, P]),
    "ffb_config5_partners": (I, [SZ, SZ, U64, P]),
    "ffb_verify_device": (I, [P, U64, SZ, P, SZ, P, P, SZ, P, P, P, SZ, C.POINTER(U64)]),
    "ffb_pivoting_partners_device": (I, [P, SZ, P, P, SZ, P]),
}


def lib():
    """The loaded engine library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1802_10453_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
