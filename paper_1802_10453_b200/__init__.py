"""B200-native rank-profile-revealing PLDL^TP^T over GF(p) (arXiv 1802.10453).

Drop-in for the reference's hot path ``ffldl::ldlt``: the host recursion is
C++ (csrc/ffb_engine.cu), the node arithmetic runs in hand-written sm_100a
kernels behind the C-ABI of include/ffldl_b200.h, and this package mirrors the
reference's C++ API in Python (ffldl.py).
"""
from .ffldl import (AntiDiagBlock, AntiTriBlock, BadBlockSizes, BlockDiag, CharTwoDivision,
                    CharTwoNonzeroDiagonal, Context, CudaError, DimensionMismatch, Error,
                    Factorization, NoMemory, NonUnitTriangular, NotPrime, NotSymmetric,
                    Permutation, PlduqFactorization, PrimeField, ScalarBlock, SingularTriangular,
                    StrictifyStats, SytrfConfig, Unsupported, Uplo, Variant, ZeroInverse, default_context,
                    gemm_sub, ldlt, ldlt_zero_leading, plduq, syr2k_sub, syrdk_sub, trmm_sub,
                    trsm_inplace, trssyr2k, strictify, WrongCharacteristic, ParseError,
                    read_factorization, read_matrix, write_factorization, write_matrix)

__all__ = [n for n in dir() if not n.startswith("_")]
