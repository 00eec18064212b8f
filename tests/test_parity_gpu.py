"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bit-exact on P, L, D and rank for every case (integer arithmetic: no
tolerance).  Covers the reference's own known answers, its exhaustive sweeps,
random inputs over p in {2,3,7,11,131,8388593}, every variant, the bordered
entry point, PLDUQ, TRSSYR2K, the BLAS3 kernels, error behaviour, and the five
benchmark families."""
import itertools
import json
import os

import numpy as np
import pytest

from helpers import describe_diff, fact_equal, hollow, rand_low_rank, rand_rook_rpm, rand_sym

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = [("cascade", 64), ("recursive", 64), ("crout", 64), ("cascade", 2), ("cascade", 4),
            ("cascade", 8)]


def cfg(v, t):
    import paper_1802_10453_b200 as ffb
    return ffb.SytrfConfig({"cascade": ffb.Variant.Cascade, "recursive": ffb.Variant.Recursive,
                            "crout": ffb.Variant.Crout}[v], t)


def check(gpu, oracle, p, a, v="cascade", t=64):
    import paper_1802_10453_b200 as ffb
    g = ffb.ldlt(a, p, cfg(v, t), ctx=gpu)
    o = oracle.ldlt(p, a, v, t)
    assert fact_equal(g, o), f"p={p} n={a.shape[0]} {v}{t}: {describe_diff(g, o)}"
    return g


def test_known_answers(gpu, oracle):
    import paper_1802_10453_b200 as ffb
    with open(os.path.join(GOLDEN, "known_answers.json")) as fh:
        k = json.load(fh)
    for case in k["ldlt"]:
        g = check(gpu, oracle, case["p"], np.array(case["a"], np.uint64))
        assert g.rank == case["rank"] and g.perm.image_array().tolist() == case["perm"]
    for case in k["ldlt_zero_leading"]:
        y, z = np.array(case["y"], np.uint64), np.array(case["z"], np.uint64)
        g = ffb.ldlt_zero_leading(y, z, case["p"], ctx=gpu)
        o = oracle.ldlt_zero_leading(case["p"], y, z)
        assert fact_equal(g, o) and g.lower.tolist() == case["lower"]
    c = k["trssyr2k"][0]
    x = ffb.trssyr2k(np.array(c["u"]), np.array(c["c"]), c["p"], ctx=gpu)
    assert x.tolist() == c["x"]
    e = k["trssyr2k_errors"][0]
    with pytest.raises(ffb.CharTwoNonzeroDiagonal):
        ffb.trssyr2k(np.array(e["u"]), np.array(e["c"]), e["p"], ctx=gpu)
    c = k["plduq"][0]
    pf = ffb.plduq(np.array(c["b"]), c["p"], ctx=gpu)
    assert pf.rank == 2 and pf.col_perm.image_array().tolist() == c["col_image"]
    assert pf.diag.tolist() == c["diag"]


def test_regression_f2(gpu, oracle):
    with open(os.path.join(GOLDEN, "known_answers.json")) as fh:
        a = np.array(json.load(fh)["regressions"][0]["a"], np.uint64)
    for v, t in VARIANTS:
        check(gpu, oracle, 2, a, v, t)


def test_degenerate_inputs(gpu, oracle):
    for a in (np.zeros((0, 0), np.uint64), np.zeros((5, 5), np.uint64), np.eye(6, dtype=np.uint64),
              np.array([[3]], np.uint64), np.zeros((1, 1), np.uint64)):
        for v, t in VARIANTS:
            check(gpu, oracle, 7, a, v, t)


@pytest.mark.parametrize("p", [2, 3])
def test_exhaustive_3x3(gpu, oracle, p):
    for code in range(p ** 6):
        a = np.zeros((3, 3), np.uint64)
        v = code
        for i in range(3):
            for j in range(i + 1):
                a[i, j] = a[j, i] = v % p
                v //= p
        for var, t in VARIANTS[:5]:
            check(gpu, oracle, p, a, var, t)


def test_exhaustive_4x4_f2(gpu, oracle):
    for code in range(1 << 10):
        a = np.zeros((4, 4), np.uint64)
        v = code
        for i in range(4):
            for j in range(i + 1):
                a[i, j] = a[j, i] = v & 1
                v >>= 1
        check(gpu, oracle, 2, a)


@pytest.mark.parametrize("p", [2, 3, 7, 11, 131, 8388593])
def test_random_small(gpu, oracle, p):
    rng = np.random.default_rng(10 + p)
    for n in (1, 2, 3, 5, 9, 16, 31, 64, 65, 100):
        for a in (rand_sym(rng, p, n), rand_low_rank(rng, p, n, n // 2), hollow(rng, p, n),
                  rand_rook_rpm(rng, p, n, n // 2)):
            for v, t in VARIANTS:
                if v == "crout" and n > 64:
                    continue
                check(gpu, oracle, p, a, v, t)


@pytest.mark.parametrize("p", [3, 131, 8388593])
def test_random_medium(gpu, oracle, p):
    rng = np.random.default_rng(20 + p)
    for n in (129, 200, 257, 400):
        for a in (rand_sym(rng, p, n), rand_rook_rpm(rng, p, n, n // 2), rand_low_rank(rng, p, n, n // 3)):
            check(gpu, oracle, p, a)
            check(gpu, oracle, p, a, "cascade", 16)


def test_zero_leading_entry(gpu, oracle):
    import paper_1802_10453_b200 as ffb
    for p in (2, 7, 8388593):
        rng = np.random.default_rng(p + 111)
        for m, n in [(1, 1), (2, 3), (3, 2), (4, 4), (0, 3), (3, 0), (5, 2), (20, 33), (40, 70)]:
            y = rng.integers(0, p, (m, n), dtype=np.uint64)
            z = rand_sym(rng, p, n)
            for v, t in VARIANTS[:5]:
                g = ffb.ldlt_zero_leading(y, z, p, cfg(v, t), ctx=gpu)
                o = oracle.ldlt_zero_leading(p, y, z, v, t)
                assert fact_equal(g, o), (p, m, n, v, t, describe_diff(g, o))
        # Y = 0 and Z = 0 (test_sytrf.cpp:187-210)
        y0 = np.zeros((3, 4), np.uint64)
        z = rand_sym(rng, p, 4)
        assert fact_equal(ffb.ldlt_zero_leading(y0, z, p, ctx=gpu), oracle.ldlt_zero_leading(p, y0, z))
        y = rng.integers(0, p, (3, 4), dtype=np.uint64)
        z0 = np.zeros((4, 4), np.uint64)
        assert fact_equal(ffb.ldlt_zero_leading(y, z0, p, ctx=gpu), oracle.ldlt_zero_leading(p, y, z0))


def test_plduq(gpu, oracle):
    import paper_1802_10453_b200 as ffb
    for p in (2, 3, 7, 11, 131, 8388593):
        rng = np.random.default_rng(p + 3)
        for m, n in [(1, 1), (1, 5), (5, 1), (3, 7), (7, 3), (10, 10), (40, 70), (130, 90)]:
            for b in (rng.integers(0, p, (m, n), dtype=np.uint64),
                      (rng.integers(0, p, (m, 2)).astype(object).dot(rng.integers(0, p, (2, n))) % p).astype(np.uint64)):
                g = ffb.plduq(b, p, ctx=gpu)
                o = oracle.plduq(p, b)
                assert g.rank == o["rank"]
                assert np.array_equal(g.row_perm.image_array(), o["row_image"])
                assert np.array_equal(g.col_perm.image_array(), o["col_image"])
                assert np.array_equal(g.lower, o["lower"]) and np.array_equal(g.upper, o["upper"])
                assert np.array_equal(g.diag, o["diag"])


def test_trssyr2k(gpu, oracle):
    import paper_1802_10453_b200 as ffb
    for p in (3, 7, 131, 8388593):
        rng = np.random.default_rng(p * 17 + 1)
        for n in (1, 2, 3, 5, 8, 16, 33, 64, 65, 150):
            u = np.triu(rng.integers(0, p, (n, n), dtype=np.uint64), 1) + np.eye(n, dtype=np.uint64)
            c = rand_sym(rng, p, n)
            assert np.array_equal(ffb.trssyr2k(u, c, p, ctx=gpu), oracle.trssyr2k(p, u, c))
    rng = np.random.default_rng(99)
    for n in (1, 2, 3, 6, 17):  # characteristic 2 with zero-diagonal right-hand sides
        u = np.triu(rng.integers(0, 2, (n, n), dtype=np.uint64), 1) + np.eye(n, dtype=np.uint64)
        c = rand_sym(rng, 2, n)
        np.fill_diagonal(c, 0)
        assert np.array_equal(ffb.trssyr2k(u, c, 2, ctx=gpu), oracle.trssyr2k(2, u, c))


def test_kernels(gpu, oracle):
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(5)
    for p in (2, 7, 131, 8388593):
        for (m, n, k) in [(9, 11, 13), (70, 130, 65), (1, 1, 1), (200, 3, 300)]:
            c = rng.integers(0, p, (m, n), dtype=np.uint64)
            a = rng.integers(0, p, (m, k), dtype=np.uint64)
            b = rng.integers(0, p, (k, n), dtype=np.uint64)
            assert np.array_equal(ffb.gemm_sub(c, a, b, p, ctx=gpu), oracle.gemm_sub(p, c, a, b))
        for n in (5, 64, 100):
            t = rng.integers(0, p, (n, n), dtype=np.uint64)
            t[np.diag_indices(n)] = rng.integers(1, p, n).astype(np.uint64)
            bb = rng.integers(0, p, (n, 7), dtype=np.uint64)
            cc = rng.integers(0, p, (n, 7), dtype=np.uint64)
            for up, tr, un in itertools.product((0, 1), repeat=3):
                assert np.array_equal(ffb.trsm_inplace(t, up, tr, un, bb, p, ctx=gpu),
                                      oracle.trsm_inplace(p, t, up, tr, un, bb))
                assert np.array_equal(ffb.trmm_sub(cc, t, up, tr, un, bb, p, ctx=gpu),
                                      oracle.trmm_sub(p, cc, t, up, tr, un, bb))
        n = 20
        g = rng.integers(0, p, (n, 6), dtype=np.uint64)
        cs = rand_sym(rng, p, n)
        blocks = [ffb.ScalarBlock(int(rng.integers(1, p))), ffb.AntiDiagBlock(int(rng.integers(1, p))),
                  ffb.ScalarBlock(int(rng.integers(1, p)))]
        blocks.append(ffb.AntiTriBlock(1, 1) if p == 2 else ffb.AntiDiagBlock(int(rng.integers(1, p))))
        d = ffb.BlockDiag(blocks)
        kind, val, val2 = d.columns()
        assert np.array_equal(ffb.syrdk_sub(cs, g, d, p, ctx=gpu), oracle.syrdk_sub(p, cs, g, kind, val, val2))
        a2 = rng.integers(0, p, (4, n), dtype=np.uint64)
        b2 = rng.integers(0, p, (4, n), dtype=np.uint64)
        assert np.array_equal(ffb.syr2k_sub(cs, a2, b2, p, ctx=gpu), oracle.syr2k_sub(p, cs, a2, b2))


def test_errors(gpu):
    import paper_1802_10453_b200 as ffb
    with pytest.raises(ffb.DimensionMismatch):
        ffb.ldlt(np.zeros((2, 3), np.uint64), 7, ctx=gpu)
    a = np.zeros((2, 2), np.uint64)
    a[0, 1] = 1
    with pytest.raises(ffb.NotSymmetric):
        ffb.ldlt(a, 7, ctx=gpu)
    with pytest.raises(ffb.NotPrime):
        ffb.ldlt(np.zeros((2, 2), np.uint64), 8, ctx=gpu)
    with pytest.raises(ffb.DimensionMismatch):
        ffb.ldlt_zero_leading(np.zeros((2, 3), np.uint64), rand_sym(np.random.default_rng(0), 7, 4), 7, ctx=gpu)
    zasym = np.zeros((3, 3), np.uint64)
    zasym[0, 2] = 1
    with pytest.raises(ffb.NotSymmetric):
        ffb.ldlt_zero_leading(np.zeros((2, 3), np.uint64), zasym, 7, ctx=gpu)
    with pytest.raises(ffb.Unsupported):
        ffb.ldlt(np.zeros((2, 2), np.uint64), 2147483659, ctx=gpu)
    u = np.eye(3, dtype=np.uint64)
    u[1, 1] = 2
    with pytest.raises(ffb.NonUnitTriangular):
        ffb.trssyr2k(u, np.zeros((3, 3), np.uint64), 7, ctx=gpu)


def test_device_generator_matches_host(gpu):
    from paper_1802_10453_b200 import configs
    for c in (1, 2, 3, 4, 5):
        w = configs.CONFIGS[c].scaled(300)
        d = configs.generate_device(w, gpu).cpu().numpy().view(np.uint32).astype(np.uint64)
        assert np.array_equal(d, configs.generate(w)), c


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_config_families_bit_exact(gpu, oracle, c):
    """Each benchmark family at sizes the oracle finishes in seconds."""
    from paper_1802_10453_b200 import configs
    for n in (256, 1024):
        w = configs.CONFIGS[c].scaled(n)
        a = configs.generate(w)
        g = check(gpu, oracle, w.p, a)
        if c == 5:
            assert g.rank == w.r


def test_golden_reference_outputs(gpu):
    """GPU against the UNMODIFIED reference's pinned outputs (tests/golden/ref_outputs.npz)."""
    import paper_1802_10453_b200 as ffb
    from golden_cases import golden_cases
    z = np.load(os.path.join(GOLDEN, "ref_outputs.npz"))
    for name, p, a, v, t in golden_cases():
        g = ffb.ldlt(a, p, cfg(v, t), ctx=gpu)
        kind, val, val2 = g.diag.columns()
        assert g.rank == int(z[f"{name}/rank"][0]), name
        assert np.array_equal(g.perm.image_array(), z[f"{name}/perm"]), name
        assert np.array_equal(g.lower, z[f"{name}/lower"].astype(np.uint64)), name
        assert np.array_equal(kind, z[f"{name}/dkind"].astype(np.int32)), name
        assert np.array_equal(val, z[f"{name}/dval"].astype(np.uint64)), name
        assert np.array_equal(val2, z[f"{name}/dval2"].astype(np.uint64)), name


def _run_in_subprocess(env_extra, code):
    import subprocess
    import sys
    env = dict(os.environ, **env_extra)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


PLDUQ_PATH_CHECK = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
import paper_1802_10453_b200 as ffb
from oracle.bind import Checker
from helpers import rand_rook_rpm, rand_sym, fact_equal
o = Checker("oracle")
for p in (2, 3, 131, 8388593):
    rng = np.random.default_rng(p)
    for (m, n) in [(1, 1), (5, 9), (64, 40), (130, 90), (300, 257), (129, 700)]:
        for b in (rng.integers(0, p, (m, n), dtype=np.uint64),
                  (rng.integers(0, p, (m, 3)).astype(object).dot(rng.integers(0, p, (3, n))) % p).astype(np.uint64),
                  np.zeros((m, n), np.uint64)):
            g = ffb.plduq(b, p); r = o.plduq(p, b)
            assert g.rank == r["rank"], (p, m, n)
            assert np.array_equal(g.row_perm.image_array(), r["row_image"])
            assert np.array_equal(g.col_perm.image_array(), r["col_image"])
            assert np.array_equal(g.lower, r["lower"]) and np.array_equal(g.upper, r["upper"])
            assert np.array_equal(g.diag, r["diag"])
    for n in (64, 130, 400):
        a = rand_rook_rpm(rng, p, n, n // 2)
        assert fact_equal(ffb.ldlt(a, p), o.ldlt(p, a)), (p, n)
print("ok")
'''


@pytest.mark.parametrize("env", [{"FFB_PLDUQ_SEQ_ROWS": "0"},
                                 {"FFB_PLDUQ_SEQ_ROWS": "0", "FFB_PLDUQ_FORCE_FALLBACK": "1"},
                                 {"FFB_PLDUQ_SEQ_ROWS": "0", "FFB_PLDUQ_SKETCH_COLS": "3"},
                                 {"FFB_PLDUQ_SEQ_ROWS": "100000"}],
                         ids=["parallel", "exact-forced", "sketch-misses-certificate", "sequential"])
def test_plduq_paths(gpu, env):
    """Every PLDUQ path (sketch-based parallel, its exact fallback, the sequential kernel)."""
    _run_in_subprocess(env, PLDUQ_PATH_CHECK)


@pytest.mark.parametrize("n,cols", [(64, 64), (256, 65), (300, 130), (700, 64), (1000, 200), (129, 1)])
@pytest.mark.parametrize("p", [2, 3, 131, 251, 257])
def test_trsm_panel_paths(gpu, oracle, n, cols, p):
    """Unit lower solves through the 256-row panel kernels (int8 mma.sync for p <= 255,
    SIMT above), with 64-row blocks, ragged blocks, recursive splits and ragged column tiles."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(n * 31 + cols + p)
    t = rng.integers(0, p, (n, n), dtype=np.uint64)
    bb = rng.integers(0, p, (n, cols), dtype=np.uint64)
    for up, tr in ((0, 0), (1, 0)):
        assert np.array_equal(ffb.trsm_inplace(t, up, tr, 1, bb, p, ctx=gpu),
                              oracle.trsm_inplace(p, t, up, tr, 1, bb))


@pytest.mark.parametrize("p", [131, 8388593])
def test_repeated_calls_same_context(gpu, oracle, p):
    """Back-to-back factorizations on one context reuse the same workspace addresses, and
    kernels are chained with programmatic dependent launch: a kernel that read producer
    data through the non-coherent path could see a stale line from the previous call
    (caught once as a rank-1 2x2 factored as rank 2).  Repeat small and medium cases."""
    rng = np.random.default_rng(p)
    cases = [np.array([[3531144, 3586508], [3586508, 3074401]], dtype=np.uint64) % p,
             rand_low_rank(rng, p, 5, 2), rand_sym(rng, p, 70), rand_low_rank(rng, p, 130, 60)]
    for rep in range(6):
        for a in cases:
            for v, t in (("recursive", 64), ("cascade", 4)):
                check(gpu, oracle, p, a, v, t)


@pytest.mark.parametrize("v", ["cascade", "crout"])
def test_banded_upload_matches_device_path(gpu, v):
    """n >= 4096 host calls stream the input in row bands while the recursion runs
    (ffb_ldlt_compact); the result must equal the device-resident path bit for bit."""
    import torch
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200 import configs
    from paper_1802_10453_b200.device import ldlt_device
    n = 4096
    w = configs.CONFIGS[5].scaled(n)
    a = configs.generate(w)
    g = ffb.ldlt(a, w.p, cfg(v, 64), ctx=gpu)
    d = ldlt_device(torch.from_numpy(a.astype(np.int32)).cuda(), w.p, cfg(v, 64), gpu)
    kind, val, val2 = g.diag.columns()
    assert g.rank == d.rank == w.r
    assert np.array_equal(g.perm.image_array(), d.perm.cpu().numpy())
    assert np.array_equal(g.lower, d.lower[:, :d.rank].cpu().numpy().astype(np.uint64))
    r = g.rank
    assert np.array_equal(kind, d.dkind[:r].cpu().numpy())
    assert np.array_equal(val, d.dval[:r].cpu().numpy().astype(np.uint64))
    assert np.array_equal(val2, d.dval2[:r].cpu().numpy().astype(np.uint64))
    # one asymmetric entry in the last band: refused, and the context stays usable
    b = a.copy()
    b[n - 1, 3] = (b[n - 1, 3] + 1) % w.p
    with pytest.raises(ffb.NotSymmetric):
        ffb.ldlt(b, w.p, cfg(v, 64), ctx=gpu)
    g2 = ffb.ldlt(a, w.p, cfg(v, 64), ctx=gpu)
    assert g2.rank == g.rank and np.array_equal(g2.lower, g.lower)


@pytest.mark.parametrize("p", [3, 131, 8388593])
def test_plduq_adaptive_chunks(gpu, oracle, p):
    """The parallel PLDUQ sizes its row chunks from the previous chunk's density (128 up to
    640 rows, narrow 64-column row detection).  This Y is sparse on top (rank 4 over 768
    rows: the chunks grow) and dense below (a 640-row chunk is cut after its first 32 new
    rows -- p >= 4096: finds >= 48 rows and shrinks to 128 rows -- with its sketch rows
    recomputed, then dense 128-row chunks, then growth again once the rank is exhausted).
    Bit-exact against the oracle."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(p + 11)
    m, n, top = 1500, 300, 768
    basis = rng.integers(0, p, (4, n)).astype(object)
    coef = rng.integers(0, p, (top, 4)).astype(object)
    y = np.zeros((m, n), dtype=np.uint64)
    y[:top] = (coef.dot(basis) % p).astype(np.uint64)
    y[top:] = rng.integers(0, p, (m - top, n), dtype=np.uint64)
    g = ffb.plduq(y, p, ctx=gpu)
    o = oracle.plduq(p, y)
    assert g.rank == o["rank"]
    assert np.array_equal(g.row_perm.image_array(), o["row_image"])
    assert np.array_equal(g.col_perm.image_array(), o["col_image"])
    assert np.array_equal(g.lower, o["lower"]) and np.array_equal(g.upper, o["upper"])
    assert np.array_equal(g.diag, o["diag"])


@pytest.mark.parametrize("p", [2, 131, 251, 257])
def test_plduq_shared_memory_kernel(gpu, oracle, p):
    """k_plduq_smem (p <= 255, Y as bytes in shared memory): every short Y, and speculatively Y
    up to 512 rows with a cap of 12 pivots -- rank 3 and 12 finish there, rank 13 and 40 give
    up and take the chunked pipeline on the untouched input; a Y too large for shared memory
    (480 x 700) and p = 257 never enter it.  Leading zero rows and columns, bit-exact."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(7 * p + 2)
    for m, n, r in [(150, 1200, 9), (199, 260, 150), (260, 300, 3), (400, 450, 12), (400, 450, 13),
                    (512, 380, 40), (480, 700, 5), (300, 257, 0)]:
        y = (rng.integers(0, p, (m, max(r, 1))).astype(object).dot(rng.integers(0, p, (max(r, 1), n))) % p)
        y = y.astype(np.uint64) if r else np.zeros((m, n), np.uint64)
        y[:7] = 0
        y[:, :3] = 0
        g = ffb.plduq(y, p, ctx=gpu)
        o = oracle.plduq(p, y)
        assert g.rank == o["rank"], (m, n, r)
        assert np.array_equal(g.row_perm.image_array(), o["row_image"])
        assert np.array_equal(g.col_perm.image_array(), o["col_image"])
        assert np.array_equal(g.lower, o["lower"]) and np.array_equal(g.upper, o["upper"])
        assert np.array_equal(g.diag, o["diag"])


@pytest.mark.parametrize("p", [3, 131, 251])
def test_plduq_detection_cap(gpu, oracle, p):
    """Row detection stops after 32 new rows and cuts the chunk there (k_rrp2, p < 4096), so
    the register-resident CRP kernels (k <= 32) take every chunk.  Dense rows give a cut in
    almost every chunk: serially detected chunks (the sketch rows after the cut were
    overwritten in place and are recomputed) and pipelined ones (the stacked detection is
    capped too), after a sparse top block and until the rank is exhausted; the rows after
    that are dependent.  Bit-exact against the oracle."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(3 * p + 1)
    m, n, top = 1100, 400, 140
    basis = rng.integers(0, p, (10, n)).astype(object)
    y = np.zeros((m, n), dtype=np.uint64)
    y[:top] = (rng.integers(0, p, (top, 10)).astype(object).dot(basis) % p).astype(np.uint64)
    y[top:] = rng.integers(0, p, (m - top, n), dtype=np.uint64)
    g = ffb.plduq(y, p, ctx=gpu)
    o = oracle.plduq(p, y)
    assert g.rank == o["rank"] == n
    assert np.array_equal(g.row_perm.image_array(), o["row_image"])
    assert np.array_equal(g.col_perm.image_array(), o["col_image"])
    assert np.array_equal(g.lower, o["lower"]) and np.array_equal(g.upper, o["upper"])
    assert np.array_equal(g.diag, o["diag"])


@pytest.mark.parametrize("p", [2, 3, 131])
def test_fused_small_nodes(gpu, oracle, p):
    """k_node128 (recursive_step of a node whose children are leaves, in one launch): nodes
    of 65..128 rows with rook-placement rank profiles take both of its exits -- leaf(Z) on
    the device (Y = 0, or m - r1 = 0) and the hand-back to the host's zero_leading_pairs
    (Y != 0) -- plus full-rank, hollow and low-rank inputs; thresholds 64 and 32."""
    rng = np.random.default_rng(1000 + p)
    for n in (65, 77, 96, 127, 128):
        for a in (rand_rook_rpm(rng, p, n, n // 2), rand_rook_rpm(rng, p, n, n // 4),
                  rand_sym(rng, p, n), hollow(rng, p, n), rand_low_rank(rng, p, n, 9)):
            check(gpu, oracle, p, a, "cascade", 64)
    for n in (33, 50, 64):
        check(gpu, oracle, p, rand_rook_rpm(rng, p, n, n // 2), "cascade", 32)


@pytest.mark.parametrize("p", [2, 131, 8388593])
def test_plduq_pipelined_detection(gpu, oracle, p):
    """Dense 128-row chunks that each add ~20 new directions: chunk c+1's sketch and row
    detection run beside chunk c's CRP on a second stream, on the stack [S_I(c); S(c+1)]
    (plduq_parallel, PIPE_KMAX).  A block with 40 new directions exceeds PIPE_KMAX (serial
    detection again), and a zero block gives k = 0.  Bit-exact against the oracle."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(p + 5)
    nb, n = 22, 500
    basis = rng.integers(0, p, (n, n)).astype(object)
    blocks, d = [], 0
    for j in range(nb):
        d = min(n, d + (40 if j == 7 else 0 if j == 12 else 20))
        coef = rng.integers(0, p, (128, d)).astype(object)
        blk = (coef.dot(basis[:d]) % p) if j != 12 else np.zeros((128, n), dtype=object)
        blocks.append(blk)
    y = np.vstack(blocks).astype(np.uint64)
    g = ffb.plduq(y, p, ctx=gpu)
    o = oracle.plduq(p, y)
    assert g.rank == o["rank"]
    assert np.array_equal(g.row_perm.image_array(), o["row_image"])
    assert np.array_equal(g.col_perm.image_array(), o["col_image"])
    assert np.array_equal(g.lower, o["lower"]) and np.array_equal(g.upper, o["upper"])
    assert np.array_equal(g.diag, o["diag"])


@pytest.mark.parametrize("pos", [(1, 0), (31, 0), (32, 31), (999, 3), (500, 470), (999, 998), (640, 0)])
def test_asymmetry_anywhere(gpu, pos):
    """The device symmetry check (k_any_asym: row bands walk their tiles left of the
    diagonal with a stride) finds a single asymmetric pair wherever it lies."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(sum(pos))
    a = rand_sym(rng, 131, 1000)
    i, j = pos
    a[i, j] = (a[j, i] + 1) % 131
    with pytest.raises(ffb.NotSymmetric):
        ffb.ldlt(a, 131, ctx=gpu)
    a[i, j] = a[j, i]
    ffb.ldlt(a, 131, ctx=gpu)


def test_banded_symmetry_check_race_free(gpu):
    """with the banded upload the symmetry check runs on the copy stream
    while the recursion already updates W in place.  The check reads the raw staging
    buffer (never written by the engine), so a symmetric U64 input at n = 8192 is never
    refused, over repeated calls; an unreduced pair (x, x + p) counts as symmetric (as on
    the small-n path, which compares reduced residues), and a real asymmetry in each
    element type is refused."""
    import ctypes as C
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200 import configs
    from paper_1802_10453_b200._lib import lib
    w = configs.CONFIGS[5].scaled(8192)
    a = configs.generate(w)
    for _ in range(20):
        g = ffb.ldlt(a, w.p, ctx=gpu)
        assert g.rank == w.r
    b = a.copy()
    b[17, 4000] += w.p  # same residue as b[4000, 17]
    assert ffb.ldlt(b, w.p, ctx=gpu).rank == w.r
    n = 4096
    a4 = configs.generate(configs.CONFIGS[1].scaled(n))
    for dt, eb in ((np.uint8, 1), (np.uint16, 2), (np.uint32, 4), (np.uint64, 8)):
        for i, j in ((n - 1, 0), (2048, 2047), (5, 4090)):
            h = np.ascontiguousarray(a4.astype(dt))
            h[i, j] = (int(h[j, i]) + 1) % 131
            out = [np.zeros(n, np.int64), np.zeros(n * n * 8, np.uint8), np.zeros(n, np.int32),
                   np.zeros(n, np.uint64), np.zeros(n, np.uint64)]
            rank = C.c_size_t(0)
            ptr = lambda x: x.ctypes.data_as(C.c_void_p)
            code = lib().ffb_ldlt_compact(gpu.handle, 131, n, ptr(h), eb, 2, 64, ptr(out[0]),
                                          ptr(out[1]), 8, ptr(out[2]), ptr(out[3]), ptr(out[4]),
                                          C.byref(rank))
            assert code == 2, (eb, i, j, code)  # FFB_NOT_SYMMETRIC


def test_two_devices_one_thread():
    """streams, scratch and kernel attributes are per device, so one
    thread can drive contexts on two GPUs alternately."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200 import configs
    w = configs.CONFIGS[5].scaled(2048)
    a = configs.generate(w)
    want = None
    for dev in (0, 1, 0, 1):
        g = ffb.ldlt(a, w.p, ctx=ffb.default_context(dev))
        if want is None:
            want = g
        assert g.rank == want.rank and np.array_equal(g.lower, want.lower)


def test_secondary_kernels_on_device(gpu, oracle):
    """trsm_inplace / trmm_sub / syrdk_sub build their triangular or block-diagonal operand on
    the device (ffb_api.cu); larger solves take the recursive panel path; a zero pivot raises
    SingularTriangular (kernels.cpp:64-71); the span overload of syrdk_sub
    (kernels.cpp:108-119) matches the oracle."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(17)
    for p in (2, 131, 8388593):
        for n in (1, 300, 513):
            t = rng.integers(0, p, (n, n), dtype=np.uint64)
            t[np.diag_indices(n)] = rng.integers(1, p, n).astype(np.uint64)
            bb = rng.integers(0, p, (n, 37), dtype=np.uint64)
            for up, tr, un in itertools.product((0, 1), repeat=3):
                assert np.array_equal(ffb.trsm_inplace(t, up, tr, un, bb, p, ctx=gpu),
                                      oracle.trsm_inplace(p, t, up, tr, un, bb)), (p, n, up, tr, un)
        t[3 % n, 3 % n] = 0
        with pytest.raises(ffb.SingularTriangular):
            ffb.trsm_inplace(t, 0, 0, 0, bb, p, ctx=gpu)
        ffb.trsm_inplace(t, 0, 0, 1, bb, p, ctx=gpu)  # unit: the diagonal is not read
        for n, k in ((1, 1), (20, 6), (300, 129)):
            c = rand_sym(rng, p, n)
            g = rng.integers(0, p, (n, k), dtype=np.uint64)
            d = rng.integers(0, p, k, dtype=np.uint64)
            assert np.array_equal(ffb.syrdk_sub(c, g, list(d), p, ctx=gpu),
                                  oracle.syrdk_sub_diag(p, c, g, d))


def test_strictify_matches_oracle(gpu, oracle):
    """strictify (rpmtools.cpp:74-132) on the device: host API on ldlt outputs and the
    device API on ldlt_device outputs, against the oracle (itself pinned to the unmodified
    reference in test_oracle.py), stats included; WrongCharacteristic over odd p."""
    import torch
    import ctypes as C
    import paper_1802_10453_b200 as ffb
    from oracle.bind import Fact
    from paper_1802_10453_b200._lib import lib
    from paper_1802_10453_b200.device import ldlt_device
    rng = np.random.default_rng(23)
    seen = 0
    for n in (2, 17, 64, 130, 301):
        for a in (hollow(rng, 2, n), rand_rook_rpm(rng, 2, n, n // 2), rand_sym(rng, 2, n)):
            g = ffb.ldlt(a, 2, ctx=gpu)
            o = oracle.ldlt(2, a)
            want, (nb, nt) = oracle.strictify(2, o)
            seen += nb
            st = ffb.StrictifyStats()
            ffb.strictify(g, st, ctx=gpu)
            kind, val, val2 = g.diag.columns()
            assert (st.blocks_converted, st.entries_touched) == (nb, nt)
            assert np.array_equal(g.perm.image_array(), want.perm) and np.array_equal(g.lower, want.lower)
            assert np.array_equal(kind, want.dkind) and np.array_equal(val, want.dval)
            assert np.array_equal(val2, want.dval2)
    assert seen > 5
    n = 2048
    a = rand_sym(rng, 2, n)  # random diagonal: 2x2 pivots with y != 0 (AntiTri) occur
    f = ldlt_device(torch.from_numpy(a.astype(np.int32)).cuda(), 2, ctx=gpu)
    o = oracle.ldlt(2, a)
    want, (nb, nt) = oracle.strictify(2, o)
    bc, et = C.c_uint64(0), C.c_uint64(0)
    assert lib().ffb_strictify_device(gpu.handle, 2, n, f.rank, f.perm.data_ptr(), f.lower.data_ptr(),
                                      f.lower.stride(0), f.dkind.data_ptr(), f.dval.data_ptr(),
                                      f.dval2.data_ptr(), C.byref(bc), C.byref(et)) == 0
    r = f.rank
    assert (bc.value, et.value) == (nb, nt) and nb > 0
    assert np.array_equal(f.perm.cpu().numpy(), want.perm)
    assert np.array_equal(f.lower[:, :r].cpu().numpy().astype(np.uint64), want.lower)
    assert np.array_equal(f.dkind[:r].cpu().numpy(), want.dkind)
    assert np.array_equal(f.dval[:r].cpu().numpy().astype(np.uint64), want.dval)
    g = ffb.ldlt(hollow(rng, 2, 40), 2, ctx=gpu)
    if g.diag.has_antitriangular():
        g.p = 3
        with pytest.raises(ffb.WrongCharacteristic):
            ffb.strictify(g, ctx=gpu)


@pytest.mark.parametrize("t", [64, 128, 256])
def test_band_schur_updates(gpu, oracle, t):
    """The symmetric Schur updates compute only the upper band of their output on the
    tcgen05 path (BandScope; tiles below j >= i - max(T, 128) are skipped) and
    zero_leading_pairs mirrors the lower part back before its symmetric gather: at n = 4096
    (rank-half rook profiles, so pairs nodes at several levels) the result is bit-exact
    against the oracle for T = 64, 128, 256, and equals the full-update run."""
    import subprocess
    import sys
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200 import configs
    w = configs.CONFIGS[5].scaled(4096)
    a = configs.generate(w)
    g = check(gpu, oracle, w.p, a, "cascade", t)
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_1802_10453_b200 as ffb; "
            "from paper_1802_10453_b200 import configs; w = configs.CONFIGS[5].scaled(4096); "
            "g = ffb.ldlt(configs.generate(w), w.p, ffb.SytrfConfig(ffb.Variant.Cascade, %d)); "
            "np.save(sys.argv[1], g.lower)" % (ROOT, t))
    import os
    import tempfile
    out = os.path.join(tempfile.mkdtemp(), "full.npy")
    env = dict(os.environ, FFB_NO_BAND="1")
    subprocess.run([sys.executable, "-c", code, out], check=True, env=env)
    assert np.array_equal(np.load(out), g.lower)


@pytest.mark.parametrize("p", [2, 131, 4093])
def test_plduq_staircase_wide(gpu, oracle, p):
    """Chunk residuals R_I whose pivot columns spread over many column blocks (a staircase
    basis over n = 9000 columns, chunk ranks 25 and one 40-row chunk), as in config 5's
    large PLDUQs.  Bit-exact against the oracle."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(p + 21)
    m, n, r = 896, 9000, 150
    # staircase basis: row t is zero left of its start column, dense after it
    starts = np.sort(rng.choice(n - 50, r, replace=False))
    basis = rng.integers(0, p, (r, n)).astype(object)
    for t in range(r):
        basis[t, :starts[t]] = 0
    perm = rng.permutation(r)
    blocks, d = [], 0
    for j in range(m // 128):
        d = min(r, d + (40 if j == 3 else 25))
        coef = rng.integers(0, p, (128, d)).astype(object)
        blocks.append(coef.dot(basis[perm[:d]]) % p)
    y = np.vstack(blocks).astype(np.uint64)
    g = ffb.plduq(y, p, ctx=gpu)
    o = oracle.plduq(p, y)
    assert g.rank == o["rank"]
    assert np.array_equal(g.row_perm.image_array(), o["row_image"])
    assert np.array_equal(g.col_perm.image_array(), o["col_image"])
    assert np.array_equal(g.lower, o["lower"]) and np.array_equal(g.upper, o["upper"])
    assert np.array_equal(g.diag, o["diag"])
