"""Python mirror of the reference C++ API (proj/include/ffldl/) over the B200 engine.

Names, argument meaning and error behaviour follow the reference so that code
written against ``ffldl`` reads the same:

    ffldl::PrimeField            -> PrimeField              (field.hpp:73)
    ffldl::Variant / SytrfConfig -> Variant / SytrfConfig   (sytrf.hpp:8-17)
    ffldl::ScalarBlock ...       -> ScalarBlock, AntiDiagBlock, AntiTriBlock, BlockDiag
                                                            (blockdiag.hpp:20-144)
    ffldl::Permutation           -> Permutation             (permutation.hpp:20)
    ffldl::Factorization         -> Factorization           (blockdiag.hpp:153)
    ffldl::ldlt                  -> ldlt                    (sytrf.hpp:30)
    ffldl::ldlt_zero_leading     -> ldlt_zero_leading       (sytrf.hpp:41)
    ffldl::plduq                 -> plduq                   (plduq.hpp:42)
    ffldl::trssyr2k              -> trssyr2k                (trssyr2k.hpp:17)
    gemm_sub/trmm_sub/trsm_inplace/syrdk_sub/syr2k_sub      (kernels.hpp:13-32)
    the exception tree           -> Error and subclasses    (errors.hpp:9-55)

Matrices are numpy arrays of canonical residues (any unsigned dtype; uint64
is the reference's FieldElement).  Every compute call runs on the GPU through
libffldl_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field as dfield
from typing import List, Optional, Sequence, Union

import numpy as np

from ._lib import lib

# ---------------------------------------------------------------------------
# Errors (errors.hpp:9-55) + the two device-side additions.
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    pass


class NotPrime(Error): pass
class ZeroInverse(Error): pass
class CharTwoDivision(Error): pass
class DimensionMismatch(Error): pass
class BadBlockSizes(Error): pass
class NotSymmetric(Error): pass
class NonUnitTriangular(Error): pass
class SingularTriangular(Error): pass
class CharTwoNonzeroDiagonal(Error): pass
class NoMemory(Error): pass
class CudaError(Error): pass
class Unsupported(Error): pass
class WrongCharacteristic(Error): pass
class ParseError(Error): pass


_STATUS = {
    1: DimensionMismatch, 2: NotSymmetric, 3: NotPrime, 4: ZeroInverse, 5: CharTwoDivision,
    6: NonUnitTriangular, 7: SingularTriangular, 8: CharTwoNonzeroDiagonal, 9: BadBlockSizes,
    10: Error, 11: NoMemory, 12: CudaError, 13: Unsupported, 14: WrongCharacteristic,
    15: ParseError,
}


def _check(status: int) -> None:
    if status != 0:
        msg = lib().ffb_last_error().decode() or lib().ffb_status_string(status).decode()
        raise _STATUS.get(status, Error)(msg)


# ---------------------------------------------------------------------------
# Field, config, D blocks, permutations, factorization.
# ---------------------------------------------------------------------------


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    bases = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for q in bases:
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in bases:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


class PrimeField:
    """Z/pZ handle (field.hpp:73-134); p must be a prime below 2^62."""

    max_modulus = (1 << 62) - 1

    def __init__(self, p: int):
        p = int(p)
        if p < 2 or p > self.max_modulus or not _is_prime(p):
            raise NotPrime(f"modulus {p} is not a prime below 2^62")
        self.p = p

    def modulus(self) -> int:
        return self.p

    def is_char_two(self) -> bool:
        return self.p == 2

    def __eq__(self, other) -> bool:
        return isinstance(other, PrimeField) and other.p == self.p

    def __repr__(self) -> str:
        return f"PrimeField({self.p})"


class Variant(enum.IntEnum):
    Recursive = 0
    Crout = 1
    Cascade = 2


@dataclass
class SytrfConfig:
    variant: Variant = Variant.Cascade
    base_case_threshold: int = 64


@dataclass(frozen=True)
class ScalarBlock:
    d: int


@dataclass(frozen=True)
class AntiDiagBlock:
    x: int


@dataclass(frozen=True)
class AntiTriBlock:
    c: int
    d: int


DiagBlock = Union[ScalarBlock, AntiDiagBlock, AntiTriBlock]


def block_order(b: DiagBlock) -> int:
    return 1 if isinstance(b, ScalarBlock) else 2


class BlockDiag:
    """Block diagonal D (blockdiag.hpp:39-144)."""

    def __init__(self, blocks: Sequence[DiagBlock] = ()):
        self._blocks: List[DiagBlock] = []
        self._offsets: List[int] = []
        self._order = 0
        for b in blocks:
            self.push(b)

    def push(self, b: DiagBlock) -> None:
        self._offsets.append(self._order)
        self._order += block_order(b)
        self._blocks.append(b)

    def append(self, other: "BlockDiag") -> None:
        for b in other._blocks:
            self.push(b)

    def block_count(self) -> int:
        return len(self._blocks)

    def order(self) -> int:
        return self._order

    def block(self, k: int) -> DiagBlock:
        return self._blocks[k]

    def offset(self, k: int) -> int:
        return self._offsets[k]

    def has_antitriangular(self) -> bool:
        return any(isinstance(b, AntiTriBlock) for b in self._blocks)

    def to_dense(self, p: int) -> np.ndarray:
        m = np.zeros((self._order, self._order), dtype=np.uint64)
        for t, b in zip(self._offsets, self._blocks):
            if isinstance(b, ScalarBlock):
                m[t, t] = b.d
            elif isinstance(b, AntiDiagBlock):
                m[t, t + 1] = m[t + 1, t] = b.x
            else:
                m[t, t + 1] = m[t + 1, t] = b.c
                m[t + 1, t + 1] = b.d
        return m

    def support(self):
        s = []
        for t, b in zip(self._offsets, self._blocks):
            if isinstance(b, ScalarBlock):
                s.append((t, t))
            else:
                s += [(t, t + 1), (t + 1, t)]
        return s

    def columns(self):
        """Per-pivot-column encoding (kind, val, val2) used by the C-ABI."""
        r = self._order
        kind = np.zeros(r, np.int32)
        val = np.zeros(r, np.uint64)
        val2 = np.zeros(r, np.uint64)
        for t, b in zip(self._offsets, self._blocks):
            if isinstance(b, ScalarBlock):
                kind[t], val[t] = 0, b.d
            elif isinstance(b, AntiDiagBlock):
                kind[t], kind[t + 1] = 1, 2
                val[t] = val[t + 1] = b.x
            else:
                kind[t], kind[t + 1] = 3, 4
                val[t] = val[t + 1] = b.c
                val2[t] = val2[t + 1] = b.d
        return kind, val, val2

    @staticmethod
    def from_columns(kind, val, val2) -> "BlockDiag":
        d = BlockDiag()
        t, r = 0, len(kind)
        while t < r:
            k = int(kind[t])
            if k == 0:
                d.push(ScalarBlock(int(val[t])))
                t += 1
            elif k == 1:
                d.push(AntiDiagBlock(int(val[t])))
                t += 2
            else:
                d.push(AntiTriBlock(int(val[t]), int(val2[t])))
                t += 2
        return d

    def __eq__(self, other) -> bool:
        return isinstance(other, BlockDiag) and self._blocks == other._blocks


class Permutation:
    """Image-array permutation (permutation.hpp:20): image(i) = j moves row i to j."""

    def __init__(self, n_or_image: Union[int, Sequence[int], np.ndarray]):
        if isinstance(n_or_image, (int, np.integer)):
            self._image = np.arange(int(n_or_image), dtype=np.int64)
        else:
            img = np.asarray(n_or_image, dtype=np.int64)
            seen = np.zeros(img.shape[0], bool)
            if img.size and (img.min() < 0 or img.max() >= img.shape[0]):
                raise BadBlockSizes("image array is not a bijection")
            seen[img] = True
            if not seen.all():
                raise BadBlockSizes("image array is not a bijection")
            self._image = img

    @staticmethod
    def from_image(image) -> "Permutation":
        return Permutation(image)

    def size(self) -> int:
        return int(self._image.shape[0])

    def image(self, i: int) -> int:
        return int(self._image[i])

    def image_array(self) -> np.ndarray:
        return self._image

    def is_identity(self) -> bool:
        return bool(np.array_equal(self._image, np.arange(self.size())))

    def inverse(self) -> "Permutation":
        inv = np.empty_like(self._image)
        inv[self._image] = np.arange(self.size())
        return Permutation(inv)

    def __eq__(self, other) -> bool:
        return isinstance(other, Permutation) and np.array_equal(self._image, other._image)


@dataclass
class Factorization:
    """A = dense(P) [L;0] D [L;0]^T dense(P)^T (blockdiag.hpp:153-183)."""

    perm: Permutation
    lower: np.ndarray  # n x r, uint64
    diag: BlockDiag
    rank: int
    p: int = 0

    def dimension(self) -> int:
        return int(self.lower.shape[0])

    def reconstruct(self) -> np.ndarray:
        """Naive P L D L^T P^T (verification only, python ints; small n)."""
        p, n, r = self.p, self.dimension(), self.rank
        L = self.lower.astype(object)
        D = self.diag.to_dense(p).astype(object)
        m = (L.dot(D).dot(L.T)) % p if r else np.zeros((n, n), dtype=object)
        out = np.zeros((n, n), dtype=np.uint64)
        img = self.perm.image_array()
        out[np.ix_(img, img)] = m.astype(np.uint64)
        return out

    def pivoting_matrix(self) -> np.ndarray:
        """Pi = P support(D) P^T (rpmtools.cpp:61-68)."""
        n = self.dimension()
        pi = np.zeros((n, n), np.uint8)
        img = self.perm.image_array()
        for a, b in self.diag.support():
            pi[img[a], img[b]] = 1
        return pi


@dataclass
class PlduqFactorization:
    """B = P [L1;M1] diag(d) [U1 V1] Q^T (plduq.hpp:24-40)."""

    row_perm: Permutation
    col_perm: Permutation
    lower: np.ndarray
    diag: np.ndarray
    upper: np.ndarray
    rank: int

    def l1(self): return self.lower[: self.rank, : self.rank]
    def m1(self): return self.lower[self.rank:, : self.rank]
    def u1(self): return self.upper[:, : self.rank]
    def v1(self): return self.upper[:, self.rank:]


# ---------------------------------------------------------------------------
# Context (one per device and thread).
# ---------------------------------------------------------------------------


class Context:
    """One device, one CUDA stream, one cached workspace (ffb_context)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib().ffb_create(C.byref(h), int(device)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            lib().ffb_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().ffb_stream(self.handle) or 0

    def launch_count(self) -> int:
        return int(lib().ffb_launch_count(self.handle))

    def sync_count(self) -> int:
        return int(lib().ffb_sync_count(self.handle))

    KERNEL_CLASSES = ("gemm", "leaf", "plduq_rowdetect_seq", "trsm", "move", "other", "plduq_sketch",
                      "plduq_crp", "plduq_pair", "ldu", "pack", "plduq_rowelim")

    def profile(self, enable: bool = True) -> None:
        """Per-kernel-class CUDA-event timing of subsequent calls (resets totals)."""
        _check(lib().ffb_profile_enable(self.handle, int(enable)))

    def profile_read(self) -> dict:
        out = {}
        for k, name in enumerate(self.KERNEL_CLASSES):
            n, ms, ops, by = C.c_uint64(), C.c_double(), C.c_double(), C.c_double()
            _check(lib().ffb_profile_read(self.handle, k, C.byref(n), C.byref(ms), C.byref(ops),
                                          C.byref(by)))
            out[name] = dict(launches=n.value, ms=ms.value, ops=ops.value, bytes=by.value)
        return out


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


# ---------------------------------------------------------------------------
# Entry points.
# ---------------------------------------------------------------------------

FieldLike = Union[PrimeField, int]


def _p(field: FieldLike) -> int:
    return field.p if isinstance(field, PrimeField) else PrimeField(int(field)).p


def _u64(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype != np.uint64:
        a = a.astype(np.uint64)
    return np.ascontiguousarray(a)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _fact_outputs(n: int):
    return (np.zeros(max(n, 1), np.int64), np.zeros(max(n * n, 1), np.uint64),
            np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.uint64),
            np.zeros(max(n, 1), np.uint64))


def _make_fact(n, p, perm, lower, dkind, dval, dval2, r) -> Factorization:
    return Factorization(Permutation(perm[:n].copy()), lower[: n * r].reshape(n, r).copy(),
                         BlockDiag.from_columns(dkind[:r], dval[:r], dval2[:r]), r, p)


def ldlt(a, field: FieldLike, config: Optional[SytrfConfig] = None,
         ctx: Optional[Context] = None) -> Factorization:
    """Symmetric indefinite PLDL^TP^T revealing the rank profile matrix (sytrf.hpp:30)."""
    config = config or SytrfConfig()
    p = _p(field)
    a = _u64(a)
    if a.ndim != 2:
        raise DimensionMismatch("ldlt: matrix must be square")
    rows, cols = a.shape
    ctx = ctx or default_context()
    perm, lower, dkind, dval, dval2 = _fact_outputs(rows)
    rank = C.c_size_t(0)
    _check(lib().ffb_ldlt(ctx.handle, p, rows, cols, _ptr(a), int(config.variant),
                          int(config.base_case_threshold), _ptr(perm), _ptr(lower), _ptr(dkind),
                          _ptr(dval), _ptr(dval2), C.byref(rank)))
    return _make_fact(rows, p, perm, lower, dkind, dval, dval2, rank.value)


def ldlt_zero_leading(y, z, field: FieldLike, config: Optional[SytrfConfig] = None,
                      ctx: Optional[Context] = None) -> Factorization:
    """Factorization of [[0, Y], [Y^T, Z]] (sytrf.hpp:41)."""
    config = config or SytrfConfig()
    p = _p(field)
    y = _u64(y)
    z = _u64(z)
    if z.ndim != 2 or z.shape[0] != z.shape[1]:
        raise DimensionMismatch("ldlt_zero_leading: Z must be square")
    m, ny = y.shape if y.ndim == 2 else (0, 0)
    nz = z.shape[0]
    if y.ndim != 2:
        raise DimensionMismatch("ldlt_zero_leading: Y must be a matrix")
    n = m + nz
    ctx = ctx or default_context()
    perm, lower, dkind, dval, dval2 = _fact_outputs(n)
    rank = C.c_size_t(0)
    _check(lib().ffb_ldlt_zero_leading(ctx.handle, p, m, ny, _ptr(y), nz, _ptr(z),
                                       int(config.variant), int(config.base_case_threshold),
                                       _ptr(perm), _ptr(lower), _ptr(dkind), _ptr(dval),
                                       _ptr(dval2), C.byref(rank)))
    return _make_fact(n, p, perm, lower, dkind, dval, dval2, rank.value)


def plduq(b, field: FieldLike, ctx: Optional[Context] = None) -> PlduqFactorization:
    """Rank-profile-revealing PLDUQ (plduq.hpp:42)."""
    p = _p(field)
    b = _u64(b)
    m, n = b.shape
    mn = min(m, n)
    ri = np.zeros(max(m, 1), np.int64)
    ci = np.zeros(max(n, 1), np.int64)
    lo = np.zeros(max(m * mn, 1), np.uint64)
    dg = np.zeros(max(mn, 1), np.uint64)
    up = np.zeros(max(mn * n, 1), np.uint64)
    rank = C.c_size_t(0)
    ctx = ctx or default_context()
    _check(lib().ffb_plduq(ctx.handle, p, m, n, _ptr(b), _ptr(ri), _ptr(ci), _ptr(lo), _ptr(dg),
                           _ptr(up), C.byref(rank)))
    r = rank.value
    return PlduqFactorization(Permutation(ri[:m].copy()), Permutation(ci[:n].copy()),
                              lo[: m * r].reshape(m, r).copy(), dg[:r].copy(),
                              up[: r * n].reshape(r, n).copy(), r)


def trssyr2k(u, c, field: FieldLike, ctx: Optional[Context] = None) -> np.ndarray:
    """Upper triangular X with X^T U + U^T X = C (trssyr2k.hpp:17)."""
    p = _p(field)
    u = _u64(u)
    c = _u64(c)
    if u.shape[0] != u.shape[1] or c.shape[0] != c.shape[1] or u.shape[0] != c.shape[0]:
        raise DimensionMismatch("trssyr2k: operands must be square of equal order")
    n = u.shape[0]
    x = np.zeros((n, n), np.uint64)
    ctx = ctx or default_context()
    _check(lib().ffb_trssyr2k(ctx.handle, p, n, _ptr(u), _ptr(c), _ptr(x)))
    return x


class Uplo(enum.IntEnum):
    Lower = 0
    Upper = 1


def gemm_sub(c, a, b, field: FieldLike, ctx: Optional[Context] = None) -> np.ndarray:
    """C - A*B (kernels.hpp:13); returns the updated C."""
    p = _p(field)
    c, a, b = _u64(c).copy(), _u64(a), _u64(b)
    if a.shape[0] != c.shape[0] or b.shape[1] != c.shape[1] or a.shape[1] != b.shape[0]:
        raise DimensionMismatch("gemm_sub: incompatible shapes")
    ctx = ctx or default_context()
    _check(lib().ffb_gemm_sub(ctx.handle, p, c.shape[0], c.shape[1], a.shape[1], _ptr(c), _ptr(a),
                              _ptr(b)))
    return c


def trmm_sub(c, t, uplo: Uplo, trans: bool, unit: bool, b, field: FieldLike,
             ctx: Optional[Context] = None) -> np.ndarray:
    """C - op(T)*B (kernels.hpp:19)."""
    p = _p(field)
    c, t, b = _u64(c).copy(), _u64(t), _u64(b)
    if t.shape[0] != t.shape[1] or t.shape[1] != b.shape[0] or c.shape != b.shape:
        raise DimensionMismatch("trmm_sub: incompatible shapes")
    ctx = ctx or default_context()
    _check(lib().ffb_trmm_sub(ctx.handle, p, c.shape[0], c.shape[1], _ptr(c), _ptr(t), int(uplo),
                              int(trans), int(unit), _ptr(b)))
    return c


def trsm_inplace(t, uplo: Uplo, trans: bool, unit: bool, b, field: FieldLike,
                 ctx: Optional[Context] = None) -> np.ndarray:
    """op(T)^-1 B (kernels.hpp:22); returns the solution."""
    p = _p(field)
    t, b = _u64(t), _u64(b).copy()
    if t.shape[0] != t.shape[1] or t.shape[1] != b.shape[0]:
        raise DimensionMismatch("trsm_inplace: incompatible shapes")
    ctx = ctx or default_context()
    _check(lib().ffb_trsm_inplace(ctx.handle, p, b.shape[0], b.shape[1], _ptr(t), int(uplo),
                                  int(trans), int(unit), _ptr(b)))
    return b


def syrdk_sub(c, g, d, field: FieldLike, ctx: Optional[Context] = None) -> np.ndarray:
    """C - G*D*G^T with D a BlockDiag (kernels.hpp:26) or a sequence of field elements
    (the std::span overload, kernels.hpp:29, kernels.cpp:108-119)."""
    p = _p(field)
    c, g = _u64(c).copy(), _u64(g)
    ctx = ctx or default_context()
    if isinstance(d, BlockDiag):
        if c.shape[0] != c.shape[1] or g.shape[0] != c.shape[0] or g.shape[1] != d.order():
            raise DimensionMismatch("syrdk_sub: incompatible shapes")
        kind, val, val2 = d.columns()
        _check(lib().ffb_syrdk_sub(ctx.handle, p, c.shape[0], g.shape[1], _ptr(c), _ptr(g),
                                   _ptr(kind), _ptr(val), _ptr(val2)))
        return c
    dv = _u64(np.asarray(d, dtype=np.uint64).reshape(-1))
    if c.shape[0] != c.shape[1] or g.shape[0] != c.shape[0] or g.shape[1] != dv.shape[0]:
        raise DimensionMismatch("syrdk_sub: incompatible shapes")
    _check(lib().ffb_syrdk_sub_diag(ctx.handle, p, c.shape[0], g.shape[1], _ptr(c), _ptr(g), _ptr(dv)))
    return c


@dataclass
class StrictifyStats:
    """rpmtools.hpp:27-30."""
    blocks_converted: int = 0
    entries_touched: int = 0


def strictify(f: Factorization, stats: Optional[StrictifyStats] = None,
              ctx: Optional[Context] = None) -> Factorization:
    """Rewrite every characteristic-2 AntiTri block of f into two scalar pivots, in place
    (rpmtools.hpp:39, rpmtools.cpp:74-132); the arithmetic runs on the device.  Returns f."""
    ctx = ctx or default_context()
    n, r = f.dimension(), f.rank
    perm = np.ascontiguousarray(f.perm.image_array(), np.int64)
    lower = _u64(f.lower[:, :r]).copy()
    kind, val, val2 = f.diag.columns()
    kind = np.ascontiguousarray(kind, np.int32).copy()
    val, val2 = _u64(val).copy(), _u64(val2).copy()
    bc, et = C.c_uint64(0), C.c_uint64(0)
    _check(lib().ffb_strictify(ctx.handle, f.p, n, r, _ptr(perm), _ptr(lower), _ptr(kind),
                               _ptr(val), _ptr(val2), C.byref(bc), C.byref(et)))
    f.perm = Permutation.from_image(perm)
    f.lower = lower
    f.diag = BlockDiag.from_columns(kind, val, val2)
    if stats is not None:
        stats.blocks_converted, stats.entries_touched = int(bc.value), int(et.value)
    return f


def syr2k_sub(c, a, b, field: FieldLike, ctx: Optional[Context] = None) -> np.ndarray:
    """C - A^T B - B^T A (kernels.hpp:32)."""
    p = _p(field)
    c, a, b = _u64(c).copy(), _u64(a), _u64(b)
    if c.shape[0] != c.shape[1] or a.shape[1] != c.shape[0] or b.shape != a.shape:
        raise DimensionMismatch("syr2k_sub: incompatible shapes")
    ctx = ctx or default_context()
    _check(lib().ffb_syr2k_sub(ctx.handle, p, c.shape[0], a.shape[0], _ptr(c), _ptr(a), _ptr(b)))
    return c


# ---------------------------------------------------------------------------
# Files: MatrixFile / FactorizationFile (io.hpp:22-62), text format byte-compatible with the
# reference, plus a checksummed binary format (csrc/ffb_io.cu).  Host-side only.
# ---------------------------------------------------------------------------


def write_matrix(path: str, a, field: FieldLike, symmetric: bool = True, binary: bool = False) -> None:
    """MatrixFile::from(a, symmetric).emit (io.cpp:70-95), or the binary form."""
    a = _u64(a)
    if a.ndim != 2:
        raise DimensionMismatch("write_matrix: a matrix is required")
    _check(lib().ffb_matrix_write(path.encode(), int(binary), a.shape[0], a.shape[1], _p(field),
                                  int(symmetric), _ptr(a), 8))


def read_matrix(path: str):
    """MatrixFile::parse (io.cpp:39-67) of a text or binary file -> (values uint64 array,
    modulus, symmetric)."""
    r, c, m, sym = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0), C.c_int(0)
    _check(lib().ffb_matrix_read(path.encode(), C.byref(r), C.byref(c), C.byref(m), C.byref(sym), None, 8))
    out = np.zeros((r.value, c.value), np.uint64)
    _check(lib().ffb_matrix_read(path.encode(), C.byref(r), C.byref(c), C.byref(m), C.byref(sym),
                                 _ptr(out), 8))
    return out, int(m.value), bool(sym.value)


def write_factorization(path: str, f: Factorization, binary: bool = False) -> None:
    """FactorizationFile::from(f).emit (io.cpp:149-198), or the binary form."""
    n, r = f.dimension(), f.rank
    perm = np.ascontiguousarray(f.perm.image_array(), np.int64)
    lower = _u64(f.lower[:, :r])
    kind, val, val2 = f.diag.columns()
    kind = np.ascontiguousarray(kind, np.int32)
    _check(lib().ffb_factorization_write(path.encode(), int(binary), n, f.p, r, _ptr(perm), _ptr(lower), 8,
                                         _ptr(kind), _ptr(_u64(val)), _ptr(_u64(val2))))


def read_factorization(path: str) -> Factorization:
    """FactorizationFile::parse + bind (io.cpp:104-146,200-222) of a text or binary file."""
    n, m, r = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    _check(lib().ffb_factorization_read(path.encode(), C.byref(n), C.byref(m), C.byref(r), None, None, 8,
                                        None, None, None))
    N, R = n.value, r.value
    perm = np.zeros(max(N, 1), np.int64)
    lower = np.zeros(max(N * R, 1), np.uint64)
    kind = np.zeros(max(R, 1), np.int32)
    val = np.zeros(max(R, 1), np.uint64)
    val2 = np.zeros(max(R, 1), np.uint64)
    _check(lib().ffb_factorization_read(path.encode(), C.byref(n), C.byref(m), C.byref(r), _ptr(perm),
                                        _ptr(lower), 8, _ptr(kind), _ptr(val), _ptr(val2)))
    return _make_fact(N, int(m.value), perm, lower, kind, val, val2, R)
