"""oracle/bind.py -- TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers built by oracle/Makefile:

* ``Checker("oracle")`` -> oracle/_build/liboracle.so, the plain-C
  restatement of the reference algorithm (oracle/ldlt_oracle.c);
* ``Checker("ref")``    -> oracle/_ref/libffldl_ref.so, the UNMODIFIED
  reference sources (/root/reference/proj/src) behind oracle/ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module.  Layout conventions are documented in oracle/oracle_api.h.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "oracle": os.path.join(HERE, "_build", "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libffldl_ref.so"),
}
PREFIX = {"oracle": "orc_", "ref": "ref_"}

STATUS_NAMES = {
    0: "OK", 1: "DimensionMismatch", 2: "NotSymmetric", 3: "NotPrime", 4: "ZeroInverse",
    5: "CharTwoDivision", 6: "NonUnitTriangular", 7: "SingularTriangular",
    8: "CharTwoNonzeroDiagonal", 9: "BadBlockSizes", 10: "Error", 11: "NoMemory",
}

VARIANTS = {"recursive": 0, "crout": 1, "cascade": 2}


class CheckerError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(STATUS_NAMES.get(code, f"status {code}"))
        self.code = code
        self.name = STATUS_NAMES.get(code, "Error")


def build() -> None:
    """Compile the checkers (the reference part only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


@dataclass
class Fact:
    """Flat view of ffldl::Factorization (proj/include/ffldl/blockdiag.hpp:153)."""
    perm: np.ndarray   # int64[n], image(pos) = original row
    lower: np.ndarray  # uint64[n, r]
    dkind: np.ndarray  # int32[r]
    dval: np.ndarray   # uint64[r]
    dval2: np.ndarray  # uint64[r]
    rank: int

    def same_as(self, other: "Fact") -> bool:
        return (self.rank == other.rank and np.array_equal(self.perm, other.perm)
                and np.array_equal(self.lower, other.lower)
                and np.array_equal(self.dkind, other.dkind)
                and np.array_equal(self.dval, other.dval)
                and np.array_equal(self.dval2, other.dval2))


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Checker:
    def __init__(self, which: str = "oracle"):
        path = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle`")
        self.which = which
        self.lib = C.CDLL(path)
        self.pre = PREFIX[which]

    def _fn(self, name):
        f = getattr(self.lib, self.pre + name)
        f.restype = C.c_int
        return f

    @staticmethod
    def _check(code: int):
        if code != 0:
            raise CheckerError(code)

    def _fact_call(self, name, dim, args):
        perm = np.zeros(max(dim, 1), np.int64)
        lower = np.zeros(max(dim * dim, 1), np.uint64)
        dkind = np.zeros(max(dim, 1), np.int32)
        dval = np.zeros(max(dim, 1), np.uint64)
        dval2 = np.zeros(max(dim, 1), np.uint64)
        rank = C.c_size_t(0)
        self._check(self._fn(name)(*args, _ptr(perm), _ptr(lower), _ptr(dkind), _ptr(dval),
                                   _ptr(dval2), C.byref(rank)))
        r = rank.value
        return Fact(perm[:dim].copy(), lower[: dim * r].reshape(dim, r).copy(), dkind[:r].copy(),
                    dval[:r].copy(), dval2[:r].copy(), r)

    def ldlt(self, p: int, a, variant: str = "cascade", threshold: int = 64) -> Fact:
        a = _u64(a)
        rows, cols = a.shape
        return self._fact_call("ldlt", rows, (C.c_uint64(p), C.c_size_t(rows), C.c_size_t(cols),
                                              _ptr(a), C.c_int(VARIANTS[variant]),
                                              C.c_size_t(threshold)))

    def ldlt_zero_leading(self, p: int, y, z, variant: str = "cascade", threshold: int = 64) -> Fact:
        y = _u64(y)
        z = _u64(z)
        m, ny = y.shape
        nz = z.shape[0]
        return self._fact_call("ldlt_zero_leading", m + nz,
                               (C.c_uint64(p), C.c_size_t(m), C.c_size_t(ny), _ptr(y),
                                C.c_size_t(nz), _ptr(z), C.c_int(VARIANTS[variant]),
                                C.c_size_t(threshold)))

    def plduq(self, p: int, b):
        b = _u64(b)
        m, n = b.shape
        rowi = np.zeros(max(m, 1), np.int64)
        coli = np.zeros(max(n, 1), np.int64)
        lower = np.zeros(max(m * min(m, n), 1), np.uint64)
        diag = np.zeros(max(min(m, n), 1), np.uint64)
        upper = np.zeros(max(min(m, n) * n, 1), np.uint64)
        rank = C.c_size_t(0)
        self._check(self._fn("plduq")(C.c_uint64(p), C.c_size_t(m), C.c_size_t(n), _ptr(b),
                                      _ptr(rowi), _ptr(coli), _ptr(lower), _ptr(diag),
                                      _ptr(upper), C.byref(rank)))
        r = rank.value
        return dict(row_image=rowi[:m].copy(), col_image=coli[:n].copy(),
                    lower=lower[: m * r].reshape(m, r).copy(), diag=diag[:r].copy(),
                    upper=upper[: r * n].reshape(r, n).copy(), rank=r)

    def trssyr2k(self, p: int, u, c) -> np.ndarray:
        u = _u64(u)
        c = _u64(c)
        n = u.shape[0]
        x = np.zeros((n, n), np.uint64)
        self._check(self._fn("trssyr2k")(C.c_uint64(p), C.c_size_t(n), _ptr(u), _ptr(c), _ptr(x)))
        return x

    def gemm_sub(self, p, c, a, b):
        c = _u64(c).copy()
        a = _u64(a)
        b = _u64(b)
        m, k = a.shape
        n = b.shape[1]
        self._check(self._fn("gemm_sub")(C.c_uint64(p), C.c_size_t(m), C.c_size_t(n),
                                         C.c_size_t(k), _ptr(c), _ptr(a), _ptr(b)))
        return c

    def trsm_inplace(self, p, t, upper: bool, trans: bool, unit: bool, b):
        t = _u64(t)
        b = _u64(b).copy()
        n, nc = b.shape
        self._check(self._fn("trsm_inplace")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(nc), _ptr(t),
                                             C.c_int(int(upper)), C.c_int(int(trans)),
                                             C.c_int(int(unit)), _ptr(b)))
        return b

    def trmm_sub(self, p, c, t, upper: bool, trans: bool, unit: bool, b):
        c = _u64(c).copy()
        t = _u64(t)
        b = _u64(b)
        n, nc = c.shape
        self._check(self._fn("trmm_sub")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(nc), _ptr(c),
                                         _ptr(t), C.c_int(int(upper)), C.c_int(int(trans)),
                                         C.c_int(int(unit)), _ptr(b)))
        return c

    def syrdk_sub(self, p, c, g, dkind, dval, dval2):
        c = _u64(c).copy()
        g = _u64(g)
        n, k = g.shape
        dkind = np.ascontiguousarray(dkind, np.int32)
        dval = _u64(dval)
        dval2 = _u64(dval2)
        self._check(self._fn("syrdk_sub")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(k), _ptr(c),
                                          _ptr(g), _ptr(dkind), _ptr(dval), _ptr(dval2)))
        return c

    def syrdk_sub_diag(self, p, c, g, d):
        c = _u64(c).copy()
        g = _u64(g)
        n, k = g.shape
        d = _u64(d)
        self._check(self._fn("syrdk_sub_diag")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(k), _ptr(c),
                                               _ptr(g), _ptr(d)))
        return c

    def strictify(self, p, f: "Fact"):
        """strictify (rpmtools.cpp:74-132) of a copy of f; returns (Fact, (blocks, touched))."""
        n, r = f.perm.shape[0], f.rank
        perm = np.ascontiguousarray(f.perm, np.int64).copy()
        lower = _u64(f.lower).copy()
        dkind = np.ascontiguousarray(f.dkind, np.int32).copy()
        dval, dval2 = _u64(f.dval).copy(), _u64(f.dval2).copy()
        stats = np.zeros(2, np.uint64)
        self._check(self._fn("strictify")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(r), _ptr(perm),
                                          _ptr(lower), _ptr(dkind), _ptr(dval), _ptr(dval2),
                                          _ptr(stats)))
        return Fact(perm, lower, dkind, dval, dval2, r), (int(stats[0]), int(stats[1]))

    def syr2k_sub(self, p, c, a, b):
        c = _u64(c).copy()
        a = _u64(a)
        b = _u64(b)
        k, n = a.shape
        self._check(self._fn("syr2k_sub")(C.c_uint64(p), C.c_size_t(n), C.c_size_t(k), _ptr(c),
                                          _ptr(a), _ptr(b)))
        return c

    def generate(self, config: int, n: int, r: int, p: int, seed: int) -> np.ndarray:
        """Benchmark input of configuration `config` (oracle/gen_oracle.c; oracle only)."""
        out = np.zeros((n, n), np.uint64)
        self._check(self._fn("generate")(C.c_int(config), C.c_size_t(n), C.c_size_t(r),
                                         C.c_uint64(p), C.c_uint64(seed), _ptr(out)))
        return out

    def config5_partners(self, n: int, r: int, seed: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.int64)
        self._check(self._fn("config5_partners")(C.c_size_t(n), C.c_size_t(r), C.c_uint64(seed),
                                                 _ptr(out)))
        return out[:n]

    def file_reemit(self, kind: int, src: str, dst: str) -> None:
        """Reference only: parse `src` (0 MatrixFile, 1 FactorizationFile) and emit to dst."""
        self._check(self._fn("file_reemit")(C.c_int(kind), src.encode(), dst.encode()))

    def factorization_emit(self, p, f: "Fact", dst: str) -> None:
        """Reference only: FactorizationFile::from(f).emit into dst."""
        n = f.perm.shape[0]
        self._check(self._fn("factorization_emit")(
            C.c_uint64(p), C.c_size_t(n), C.c_size_t(f.rank), _ptr(np.ascontiguousarray(f.perm, np.int64)),
            _ptr(_u64(f.lower)), _ptr(np.ascontiguousarray(f.dkind, np.int32)), _ptr(_u64(f.dval)),
            _ptr(_u64(f.dval2)), dst.encode()))

    def rank_profile(self, p, a) -> np.ndarray:
        """Brute-force RPM (reference only: rpmtools.cpp:43-59)."""
        a = _u64(a)
        m, n = a.shape
        out = np.zeros((m, n), np.uint64)
        self._check(self._fn("rank_profile")(C.c_uint64(p), C.c_size_t(m), C.c_size_t(n), _ptr(a),
                                             _ptr(out)))
        return out


def pivoting_matrix(f: Fact) -> np.ndarray:
    """Pi = P * support(D) * P^T (restates rpmtools.cpp:61-68 + blockdiag.hpp:89-101)."""
    n = f.perm.shape[0]
    pi = np.zeros((n, n), np.uint8)
    t = 0
    while t < f.rank:
        if f.dkind[t] == 0:
            pi[f.perm[t], f.perm[t]] = 1
            t += 1
        else:
            pi[f.perm[t], f.perm[t + 1]] = 1
            pi[f.perm[t + 1], f.perm[t]] = 1
            t += 2
    return pi


def dense_d(f: Fact, p: int) -> np.ndarray:
    r = f.rank
    d = np.zeros((r, r), dtype=object)
    t = 0
    while t < r:
        if f.dkind[t] == 0:
            d[t, t] = int(f.dval[t])
            t += 1
        else:
            d[t, t + 1] = d[t + 1, t] = int(f.dval[t])
            if f.dkind[t] == 3:
                d[t + 1, t + 1] = int(f.dval2[t])
            t += 2
    return d


def reconstruct(f: Fact, p: int) -> np.ndarray:
    """P L D L^T P^T with python-int arithmetic (small n only)."""
    n = f.perm.shape[0]
    L = f.lower.astype(object)
    d = dense_d(f, p)
    m = (L.dot(d).dot(L.T)) % p if f.rank else np.zeros((n, n), dtype=object)
    a = np.zeros((n, n), dtype=object)
    perm = f.perm
    for i in range(n):
        for j in range(n):
            a[perm[i], perm[j]] = m[i, j]
    return a.astype(np.uint64)
