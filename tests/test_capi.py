"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/ffldl_b200.h declares, and its host-only logic
(generators, status strings) behaves.  No GPU needed."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ffldl_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ffb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1802_10453_b200._lib import EXPORTS, lib
    L = lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(EXPORTS) == syms


def test_status_strings_mirror_reference_exceptions():
    from paper_1802_10453_b200._lib import lib
    L = lib()
    names = {i: L.ffb_status_string(i).decode() for i in range(14)}
    assert names[0] == "OK"
    assert names[1] == "DimensionMismatch" and names[2] == "NotSymmetric"
    assert names[3] == "NotPrime" and names[8] == "CharTwoNonzeroDiagonal"
    assert L.ffb_version() >= 1


def test_python_mirror_validation_without_gpu():
    import paper_1802_10453_b200 as ffb
    with pytest.raises(ffb.NotPrime):
        ffb.PrimeField(8)
    with pytest.raises(ffb.NotPrime):
        ffb.PrimeField(1)
    assert ffb.PrimeField(8388593).modulus() == 8388593
    p = ffb.Permutation([1, 0, 2])
    assert p.inverse().image(0) == 1 and not p.is_identity()
    with pytest.raises(ffb.BadBlockSizes):
        ffb.Permutation([0, 0])
    d = ffb.BlockDiag([ffb.ScalarBlock(3), ffb.AntiDiagBlock(2), ffb.AntiTriBlock(1, 1)])
    assert d.order() == 5 and d.offset(2) == 3 and d.has_antitriangular()
    k, v, v2 = d.columns()
    assert ffb.BlockDiag.from_columns(k, v, v2) == d


def test_host_generator_deterministic_and_symmetric():
    from paper_1802_10453_b200 import configs
    for c in (1, 2, 3, 4, 5):
        w = configs.CONFIGS[c].scaled(96)
        a = configs.generate(w)
        b = configs.generate(w)
        assert np.array_equal(a, b) and np.array_equal(a, a.T)
        assert a.max() < w.p
        if c == 4:
            assert not a.diagonal().any()
    w = configs.CONFIGS[5].scaled(96)
    pt = configs.config5_partners(w)
    used = pt >= 0
    assert used.sum() == w.r
    assert all(pt[pt[i]] == i for i in np.nonzero(used)[0])


def test_config5_rank_profile_matches_generator(oracle):
    """The oracle reveals exactly R for configuration 5 (the construction's promise)."""
    from oracle.bind import pivoting_matrix
    from paper_1802_10453_b200 import configs
    w = configs.CONFIGS[5].scaled(320)
    f = oracle.ldlt(w.p, configs.generate(w))
    R = np.zeros((w.n, w.n), np.uint8)
    for i, j in enumerate(configs.config5_partners(w)):
        if j >= 0:
            R[i, j] = 1
    assert f.rank == w.r
    assert np.array_equal(pivoting_matrix(f), R)
