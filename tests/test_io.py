"""Matrix and factorization files (io.hpp:22-62, io.cpp:39-222).

CPU tests (host-side code of libffldl_b200.so, no device calls):
  * the text writer is byte-identical to the reference's FactorizationFile/MatrixFile emit,
    and the reference's parser re-emits our files unchanged (oracle/_ref);
  * the reference's known answer (test_io.cpp:103-113) and parse failures (:116-141);
  * binary round trips, checksum and truncation detection.
"""
import os

import numpy as np
import pytest

from helpers import hollow, rand_rook_rpm, rand_sym

BAD_FACTORIZATIONS = [  # test_io.cpp:120-134 (+ the bind-time duplicate image :136-139)
    "Fact 2 7\n",
    "Factorization 2 7\nrank 3\n",
    "Factorization 2 7\nrank 1\nP 1 2\nL\n1\n0\nD\nS 3\n",
    "Factorization 2 7\nrank 1\nP 1 0\nL\n1\n9\nD\nS 3\n",
    "Factorization 2 7\nrank 1\nP 1 0\nL\n1\n0\nD\nQ 3\n",
    "Factorization 2 7\nrank 1\nP 1 0\nL\n1\n0\nD\nS 0\n",
    "Factorization 2 7\nrank 1\nP 1 0\nL\n1\n0\nD\nA 3\n",
    "Factorization 2 7\nrank 1\nP 1 0\nL\n1\n0\nD\n",
    "Factorization 2 7\nrank 1\nP 1 1\nL\n1\n0\nD\nS 3\n",
]
BAD_MATRICES = ["Sym 2 7\n0 0\n0 0\n", "SymMat 2 1\n0 0\n0 0\n", "SymMat 2 7\n0 1\n0 0\n",
                "Mat 2 2 7\n0 7\n0 0\n", "SymMat 2 7\n0 0\n0\n"]


def _fact(o, p):
    import paper_1802_10453_b200 as ffb
    n = o.perm.shape[0]
    return ffb.ffldl._make_fact(n, p, o.perm, o.lower.reshape(-1), o.dkind, o.dval, o.dval2, o.rank)


def _cases(oracle):
    rng = np.random.default_rng(3)
    for p in (2, 7, 131, 8388593):
        for n in (1, 9, 40):
            for a in (rand_sym(rng, p, n), hollow(rng, p, n), rand_rook_rpm(rng, p, n, n // 2)):
                yield p, a, oracle.ldlt(p, a)


def test_text_matches_reference_emit(oracle, ref, tmp_path):
    import paper_1802_10453_b200 as ffb
    for k, (p, a, o) in enumerate(_cases(oracle)):
        ours, theirs, back = (str(tmp_path / f"{x}{k}") for x in "otb")
        ffb.write_factorization(ours, _fact(o, p))
        ref.factorization_emit(p, o, theirs)
        assert open(ours, "rb").read() == open(theirs, "rb").read(), (p, a.shape)
        ref.file_reemit(1, ours, back)
        assert open(back, "rb").read() == open(ours, "rb").read()
        ffb.write_matrix(ours + "m", a, p)
        ref.file_reemit(0, ours + "m", back + "m")
        assert open(back + "m", "rb").read() == open(ours + "m", "rb").read()
        g = ffb.read_factorization(theirs)
        assert g.rank == o.rank and np.array_equal(g.lower, o.lower)
        assert np.array_equal(g.perm.image_array(), o.perm)
        m, pp, sym = ffb.read_matrix(back + "m")
        assert np.array_equal(m, a) and pp == p and sym


def test_known_answer_and_parse_failures(ref, tmp_path):
    import paper_1802_10453_b200 as ffb
    from oracle.bind import CheckerError
    f = ffb.ffldl._make_fact(2, 7, np.array([1, 0]), np.array([1, 0], np.uint64),
                             np.array([0], np.int32), np.array([3], np.uint64), np.array([0], np.uint64), 1)
    path = str(tmp_path / "ka")
    ffb.write_factorization(path, f)
    assert open(path).read() == "Factorization 2 7\nrank 1\nP 1 0\nL\n1\n0\nD\nS 3\n"
    for k, text in enumerate(BAD_FACTORIZATIONS):
        bad = str(tmp_path / f"bad{k}")
        with open(bad, "w") as fh:
            fh.write(text)
        with pytest.raises(ffb.ParseError):
            ffb.read_factorization(bad)
        if k < len(BAD_FACTORIZATIONS) - 1:  # the duplicate image fails only at bind time there
            with pytest.raises(CheckerError):
                ref.file_reemit(1, bad, bad + ".out")
    for k, text in enumerate(BAD_MATRICES):
        bad = str(tmp_path / f"badm{k}")
        with open(bad, "w") as fh:
            fh.write(text)
        with pytest.raises(ffb.ParseError):
            ffb.read_matrix(bad)
        with pytest.raises(CheckerError):
            ref.file_reemit(0, bad, bad + ".out")
    with pytest.raises(ffb.ParseError):
        ffb.read_matrix(str(tmp_path / "missing"))


def test_binary_round_trip_and_integrity(oracle, tmp_path):
    import paper_1802_10453_b200 as ffb
    for k, (p, a, o) in enumerate(_cases(oracle)):
        f = _fact(o, p)
        path = str(tmp_path / f"b{k}")
        ffb.write_factorization(path, f, binary=True)
        g = ffb.read_factorization(path)
        assert g.rank == f.rank and g.p == p and g.diag == f.diag
        assert np.array_equal(g.lower, f.lower) and np.array_equal(g.perm.image_array(), f.perm.image_array())
        ffb.write_matrix(path + "m", a, p, binary=True)
        m, pp, sym = ffb.read_matrix(path + "m")
        assert np.array_equal(m, a) and pp == p and sym
    n = 300
    a = rand_sym(np.random.default_rng(1), 131, n)
    f = _fact(oracle.ldlt(131, a), 131)
    path = str(tmp_path / "big")
    ffb.write_factorization(path, f, binary=True)
    text = str(tmp_path / "big.txt")
    ffb.write_factorization(text, f)
    assert os.path.getsize(path) < os.path.getsize(text) / 2  # 1-byte residues at p = 131
    raw = bytearray(open(path, "rb").read())
    raw[len(raw) // 2] ^= 1
    with open(path + "x", "wb") as fh:
        fh.write(raw)
    with pytest.raises(ffb.ParseError):
        ffb.read_factorization(path + "x")
    with open(path + "t", "wb") as fh:
        fh.write(bytes(raw[: len(raw) - 100]))
    with pytest.raises(ffb.ParseError):
        ffb.read_factorization(path + "t")
    with pytest.raises(ffb.NotSymmetric):
        b = a.copy()
        b[0, 1] = (b[1, 0] + 1) % 131
        ffb.write_matrix(path + "s", b, 131)
