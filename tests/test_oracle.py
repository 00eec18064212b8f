"""Pin the CPU oracle (C restatement) before trusting it as the GPU checker.

(a) against the known-answer vectors stated in the reference's own tests and
    spec (tests/golden/known_answers.json);
(b) against the UNMODIFIED reference's outputs pinned in
    tests/golden/ref_outputs.npz (tests/golden/make_golden.py);
(c) live against oracle/_ref (when built) on seeded random inputs, including
    the reference's exhaustive sweeps (test_sytrf.cpp:124-156,
    test_plduq.cpp:89-110).
"""
import hashlib
import itertools
import json
import os

import numpy as np
import pytest

from helpers import hollow, rand_low_rank, rand_rook_rpm, rand_sym
from oracle.bind import CheckerError, pivoting_matrix, reconstruct

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KIND = {"S": 0, "A": 1, "T": 3}


def d_columns(blocks):
    kind, val, val2 = [], [], []
    for tag, a, b in blocks:
        if tag == "S":
            kind += [0]; val += [a]; val2 += [0]
        else:
            kind += [KIND[tag], KIND[tag] + 1]; val += [a, a]; val2 += [b, b]
    return kind, val, val2


def known():
    with open(os.path.join(GOLDEN, "known_answers.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("case", known()["ldlt"], ids=lambda c: c["src"])
def test_oracle_ldlt_known_answers(oracle, case):
    f = oracle.ldlt(case["p"], np.array(case["a"], np.uint64))
    kind, val, val2 = d_columns(case["D"])
    assert f.rank == case["rank"]
    assert f.perm.tolist() == case["perm"]
    assert f.lower.reshape(len(case["perm"]), -1).tolist() == [row for row in case["lower"]] or f.rank == 0
    assert f.dkind.tolist() == kind and f.dval.tolist() == val and f.dval2.tolist() == val2


@pytest.mark.parametrize("case", known()["ldlt_zero_leading"], ids=lambda c: c["src"])
def test_oracle_zero_leading_known_answers(oracle, case):
    f = oracle.ldlt_zero_leading(case["p"], np.array(case["y"], np.uint64), np.array(case["z"], np.uint64))
    kind, val, _ = d_columns(case["D"])
    assert f.rank == case["rank"] and f.perm.tolist() == case["perm"]
    assert f.lower.tolist() == case["lower"]
    assert f.dkind.tolist() == kind and f.dval.tolist() == val


def test_oracle_plduq_known_answer(oracle):
    c = known()["plduq"][0]
    r = oracle.plduq(c["p"], np.array(c["b"], np.uint64))
    assert r["rank"] == c["rank"] and r["row_image"].tolist() == c["row_image"]
    assert r["col_image"].tolist() == c["col_image"] and r["diag"].tolist() == c["diag"]


def test_oracle_trssyr2k_known_answer(oracle):
    c = known()["trssyr2k"][0]
    x = oracle.trssyr2k(c["p"], np.array(c["u"], np.uint64), np.array(c["c"], np.uint64))
    assert x.tolist() == c["x"]
    e = known()["trssyr2k_errors"][0]
    with pytest.raises(CheckerError) as ei:
        oracle.trssyr2k(e["p"], np.array(e["u"], np.uint64), np.array(e["c"], np.uint64))
    assert ei.value.name == e["error"]


def test_oracle_regression_f2(oracle, ref):
    a = np.array(known()["regressions"][0]["a"], np.uint64)
    for v, t in (("recursive", 64), ("crout", 64), ("cascade", 2), ("cascade", 4)):
        f = oracle.ldlt(2, a, v, t)
        assert np.array_equal(reconstruct(f, 2), a)
        assert np.array_equal(pivoting_matrix(f), ref.rank_profile(2, a).astype(np.uint8))
        assert f.same_as(ref.ldlt(2, a, v, t))


def test_oracle_matches_pinned_reference_outputs(oracle):
    from golden_cases import golden_cases
    z = np.load(os.path.join(GOLDEN, "ref_outputs.npz"))
    n_cases = 0
    for name, p, a, variant, T in golden_cases():
        assert bytes(z[f"{name}/sha"]) == hashlib.sha256(a.tobytes()).digest(), name
        f = oracle.ldlt(p, a, variant, T)
        assert f.rank == int(z[f"{name}/rank"][0]), name
        assert np.array_equal(f.perm, z[f"{name}/perm"]), name
        assert np.array_equal(f.lower, z[f"{name}/lower"].astype(np.uint64)), name
        assert np.array_equal(f.dkind, z[f"{name}/dkind"].astype(np.int32)), name
        assert np.array_equal(f.dval, z[f"{name}/dval"].astype(np.uint64)), name
        assert np.array_equal(f.dval2, z[f"{name}/dval2"].astype(np.uint64)), name
        n_cases += 1
    assert n_cases > 150


@pytest.mark.parametrize("p", [2, 3])
def test_oracle_exhaustive_3x3(oracle, ref, p):
    """Every symmetric 3x3 over F2/F3, every variant (test_sytrf.cpp:124-141)."""
    for code in range(p ** 6):
        a = np.zeros((3, 3), np.uint64)
        v = code
        for i in range(3):
            for j in range(i + 1):
                a[i, j] = a[j, i] = v % p
                v //= p
        for var, t in (("recursive", 64), ("crout", 64), ("cascade", 2), ("cascade", 4)):
            assert oracle.ldlt(p, a, var, t).same_as(ref.ldlt(p, a, var, t))


def test_oracle_exhaustive_4x4_f2(oracle, ref):
    """Every symmetric 4x4 over F2 (test_sytrf.cpp:143-156)."""
    for code in range(1 << 10):
        a = np.zeros((4, 4), np.uint64)
        v = code
        for i in range(4):
            for j in range(i + 1):
                a[i, j] = a[j, i] = v & 1
                v >>= 1
        assert oracle.ldlt(2, a).same_as(ref.ldlt(2, a))


def test_oracle_plduq_exhaustive(oracle, ref):
    """All 2x2 and 3x3 matrices mod 2 and 3 (test_plduq.cpp:89-110)."""
    for p in (2, 3):
        for n in (2, 3):
            for code in range(p ** (n * n)):
                b = np.array([(code // p ** k) % p for k in range(n * n)], np.uint64).reshape(n, n)
                x, y = oracle.plduq(p, b), ref.plduq(p, b)
                for k in x:
                    assert np.array_equal(np.asarray(x[k]), np.asarray(y[k])), (p, n, code, k)


@pytest.mark.parametrize("p", [2, 3, 7, 11, 131, 8388593])
def test_oracle_random_vs_reference(oracle, ref, p):
    rng = np.random.default_rng(p)
    for n in (1, 2, 3, 4, 7, 12, 33, 70):
        for a in (rand_sym(rng, p, n), rand_low_rank(rng, p, n, n // 2), hollow(rng, p, n),
                  rand_rook_rpm(rng, p, n, n // 2)):
            for v, t in (("cascade", 64), ("recursive", 64), ("cascade", 5)):
                assert oracle.ldlt(p, a, v, t).same_as(ref.ldlt(p, a, v, t))
        m = max(1, n // 3)
        y = rng.integers(0, p, (m, n), dtype=np.uint64)
        z = rand_sym(rng, p, n)
        assert oracle.ldlt_zero_leading(p, y, z, "cascade", 4).same_as(ref.ldlt_zero_leading(p, y, z, "cascade", 4))


def test_oracle_kernels_vs_reference(oracle, ref):
    rng = np.random.default_rng(5)
    for p in (2, 7, 8388593):
        m, n, k = 9, 11, 13
        c = rng.integers(0, p, (m, n), dtype=np.uint64)
        a = rng.integers(0, p, (m, k), dtype=np.uint64)
        b = rng.integers(0, p, (k, n), dtype=np.uint64)
        assert np.array_equal(oracle.gemm_sub(p, c, a, b), ref.gemm_sub(p, c, a, b))
        t = rng.integers(0, p, (n, n), dtype=np.uint64)
        t[np.diag_indices(n)] = rng.integers(1, p, n).astype(np.uint64)
        bb = rng.integers(0, p, (n, 5), dtype=np.uint64)
        cc = rng.integers(0, p, (n, 5), dtype=np.uint64)
        for up, tr, un in itertools.product((0, 1), repeat=3):
            assert np.array_equal(oracle.trsm_inplace(p, t, up, tr, un, bb), ref.trsm_inplace(p, t, up, tr, un, bb))
            assert np.array_equal(oracle.trmm_sub(p, cc, t, up, tr, un, bb), ref.trmm_sub(p, cc, t, up, tr, un, bb))
        g = rng.integers(0, p, (n, 6), dtype=np.uint64)
        cs = rand_sym(rng, p, n)
        kinds = np.array([0, 1, 2, 0, 3 if p == 2 else 1, 4 if p == 2 else 2], np.int32)
        dv = rng.integers(1, p, 6).astype(np.uint64)
        dv[2] = dv[1]; dv[5] = dv[4]
        d2 = np.zeros(6, np.uint64)
        if p == 2:
            d2[4] = d2[5] = 1
        assert np.array_equal(oracle.syrdk_sub(p, cs, g, kinds, dv, d2), ref.syrdk_sub(p, cs, g, kinds, dv, d2))
        a2 = rng.integers(0, p, (4, n), dtype=np.uint64)
        b2 = rng.integers(0, p, (4, n), dtype=np.uint64)
        assert np.array_equal(oracle.syr2k_sub(p, cs, a2, b2), ref.syr2k_sub(p, cs, a2, b2))


def test_oracle_config_families(oracle, ref):
    """The five benchmark families at small n: restatement == reference."""
    from paper_1802_10453_b200 import configs
    for c in (1, 2, 3, 4, 5):
        w = configs.CONFIGS[c].scaled(192)
        a = configs.generate(w)
        assert oracle.ldlt(w.p, a).same_as(ref.ldlt(w.p, a)), c


def test_oracle_errors(oracle):
    with pytest.raises(CheckerError) as e:
        oracle.ldlt(7, np.zeros((2, 3), np.uint64))
    assert e.value.name == "DimensionMismatch"
    a = np.zeros((2, 2), np.uint64)
    a[0, 1] = 1
    with pytest.raises(CheckerError) as e:
        oracle.ldlt(7, a)
    assert e.value.name == "NotSymmetric"
    with pytest.raises(CheckerError) as e:
        oracle.ldlt(8, np.zeros((2, 2), np.uint64))
    assert e.value.name == "NotPrime"


def test_oracle_generators_match_product(oracle):
    """oracle/gen_oracle.c (used by bench.py's CPU legs instead of the product library)
    builds the same inputs as ffb_generate_host, element for element."""
    from paper_1802_10453_b200 import configs
    for c in (1, 2, 3, 4, 5):
        for n in (1, 37, 300):
            w = configs.CONFIGS[c].scaled(n)
            want = configs.generate(w)
            got = oracle.generate(c, w.n, w.r, w.p, w.seed)
            assert np.array_equal(got, want), (c, n)
    w = configs.CONFIGS[5].scaled(1000)
    assert np.array_equal(oracle.config5_partners(w.n, w.r, w.seed), configs.config5_partners(w))


def test_fullsize_golden_small_configs(oracle):
    """tests/golden/fullsize.json (make_fullsize.py) re-derived for the configurations the
    oracle factors in seconds (1: n=1024, 2: n=4096); the larger ones are checked on the
    GPU against the same file (test_fullsize_gpu.py)."""
    import sys
    sys.path.insert(0, GOLDEN)
    from make_fullsize import digest
    with open(os.path.join(GOLDEN, "fullsize.json")) as fh:
        gold = json.load(fh)
    from paper_1802_10453_b200 import configs
    for c in (1, 2):
        w = configs.CONFIGS[c]
        g = gold[str(c)]
        assert (g["n"], g["p"], g["seed"], g["rank_param"]) == (w.n, w.p, w.seed, w.r)
        o = oracle.ldlt(w.p, oracle.generate(c, w.n, w.r, w.p, w.seed))
        d = digest(o.perm, o.lower, o.dkind, o.dval, o.dval2, o.rank)
        for k in ("rank", "perm", "lower_blocks", "dkind", "dval", "dval2"):
            assert d[k] == g[k], (c, k)
    for c in (1, 2, 3, 4, 5):
        assert str(c) in gold, f"config {c} missing from fullsize.json"


def test_oracle_strictify_and_syrdk_diag_vs_reference(oracle, ref):
    """strictify (rpmtools.cpp:74-132) and syrdk_sub(span) (kernels.cpp:108-119): the C
    restatement equals the unmodified reference, including its StrictifyStats and the
    WrongCharacteristic refusal over odd p."""
    rng = np.random.default_rng(71)
    hits = 0
    for n in (2, 5, 16, 40, 97):
        for a in (hollow(rng, 2, n), rand_sym(rng, 2, n), rand_rook_rpm(rng, 2, n, n // 2)):
            f = oracle.ldlt(2, a)
            hits += int(np.any(f.dkind == 3))
            go, so = oracle.strictify(2, f)
            gr, sr = ref.strictify(2, f)
            assert go.same_as(gr) and so == sr, n
    assert hits > 3
    f = oracle.ldlt(3, hollow(rng, 3, 30))
    assert oracle.strictify(3, f)[1][0] == 0
    g = oracle.ldlt(2, hollow(rng, 2, 30))
    bad = type(g)(g.perm, g.lower, g.dkind, g.dval, g.dval2, g.rank)
    if np.any(g.dkind == 3):
        with pytest.raises(CheckerError) as e:
            oracle.strictify(3, bad)
        assert e.value.name == "WrongCharacteristic"
        with pytest.raises(CheckerError):
            ref.strictify(3, bad)
    for p in (2, 131, 8388593):
        for n, k in ((1, 1), (7, 3), (40, 33)):
            c = rand_sym(rng, p, n)
            g = rng.integers(0, p, (n, k), dtype=np.uint64)
            d = rng.integers(0, p, k, dtype=np.uint64)
            assert np.array_equal(oracle.syrdk_sub_diag(p, c, g, d), ref.syrdk_sub_diag(p, c, g, d))
