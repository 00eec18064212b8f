"""The tcgen05 int8 GEMM path (p <= 255, large shapes) against the oracle, for every
operand orientation the engine uses (NN via gemm_sub/trmm_sub, TN via syr2k_sub, NT via
syrdk_sub), ragged sizes (partial M/N tiles, K not a multiple of the 128-byte stage), and
the int32 accumulator headroom (K up to 20000 with |x| = 65)."""
import numpy as np
import pytest

from helpers import rand_sym

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k", [(128, 128, 128), (256, 512, 256), (300, 500, 700),
                                   (129, 257, 65), (1000, 64, 200), (64, 1000, 3000),
                                   (513, 300, 20000),
                                   # small M (rows beyond M are TMA zero-fill) and short K
                                   # (the 2-stage, two-CTAs-per-SM variant)
                                   (8, 4096, 1024), (17, 3000, 500), (100, 2048, 64),
                                   (1000, 3000, 16), (700, 2500, 250), (128, 128, 4096),
                                   (513, 1000, 1), (300, 777, 37), (2000, 300, 128)])
@pytest.mark.parametrize("p", [131, 251, 2, 3])
@pytest.mark.parametrize("path", ["tc", "mma", "rankk"])
def test_tc_gemm_nn(gpu, oracle, m, n, k, p, path, monkeypatch):
    """Both int8 paths: tcgen05 (packed, TMA) and warp mma.sync (raw residues)."""
    import paper_1802_10453_b200 as ffb
    monkeypatch.setenv("FFB_GEMM_PATH", path)
    rng = np.random.default_rng(m * 7 + n * 3 + k + p)
    if p == 131 and k == 20000:
        a = np.full((m, k), 65, np.uint64)  # worst case |centered| for p=131
        b = np.full((k, n), 66, np.uint64)  # = -65
    else:
        a = rng.integers(0, p, (m, k), dtype=np.uint64)
        b = rng.integers(0, p, (k, n), dtype=np.uint64)
    c = rng.integers(0, p, (m, n), dtype=np.uint64)
    assert np.array_equal(ffb.gemm_sub(c, a, b, p, ctx=gpu), oracle.gemm_sub(p, c, a, b))


@pytest.mark.parametrize("n,k", [(300, 200), (520, 130), (256, 2048)])
@pytest.mark.parametrize("path", ["tc", "mma", "simt", "rankk"])
def test_tc_gemm_transposed_operands(gpu, oracle, n, k, path, monkeypatch):
    import paper_1802_10453_b200 as ffb
    monkeypatch.setenv("FFB_GEMM_PATH", path)
    p = 131
    rng = np.random.default_rng(n + k)
    c = rand_sym(rng, p, n)
    a = rng.integers(0, p, (k, n), dtype=np.uint64)
    b = rng.integers(0, p, (k, n), dtype=np.uint64)
    assert np.array_equal(ffb.syr2k_sub(c, a, b, p, ctx=gpu), oracle.syr2k_sub(p, c, a, b))
    g = rng.integers(0, p, (n, k - k % 2), dtype=np.uint64)
    kk = g.shape[1]
    blocks = []
    t = 0
    while t < kk:
        if t + 1 < kk and rng.integers(0, 3) == 0:
            blocks.append(ffb.AntiDiagBlock(int(rng.integers(1, p))))
            t += 2
        else:
            blocks.append(ffb.ScalarBlock(int(rng.integers(1, p))))
            t += 1
    d = ffb.BlockDiag(blocks)
    kind, val, val2 = d.columns()
    assert np.array_equal(ffb.syrdk_sub(c, g, d, p, ctx=gpu), oracle.syrdk_sub(p, c, g, kind, val, val2))


@pytest.mark.parametrize("m,n,k", [(128, 64, 128), (300, 500, 700), (129, 257, 65), (513, 300, 8000),
                                   (9, 4000, 600)])
@pytest.mark.parametrize("p", [8388593, 65521, 1000003, 257])
def test_tc_limb_gemm(gpu, oracle, m, n, k, p):
    """int8-limb tcgen05 path (255 < p < 2^23): 9 limb products into 5 shift classes."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(m + n + k + p)
    if k == 8000:  # extreme centered residues: |x| = (p-1)/2
        a = np.full((m, k), (p - 1) // 2, np.uint64)
        b = np.full((k, n), (p + 1) // 2, np.uint64)
    else:
        a = rng.integers(0, p, (m, k), dtype=np.uint64)
        b = rng.integers(0, p, (k, n), dtype=np.uint64)
    c = rng.integers(0, p, (m, n), dtype=np.uint64)
    assert np.array_equal(ffb.gemm_sub(c, a, b, p, ctx=gpu), oracle.gemm_sub(p, c, a, b))
    c2 = rand_sym(rng, p, n)
    a2 = rng.integers(0, p, (k, n), dtype=np.uint64)
    b2 = rng.integers(0, p, (k, n), dtype=np.uint64)
    assert np.array_equal(ffb.syr2k_sub(c2, a2, b2, p, ctx=gpu), oracle.syr2k_sub(p, c2, a2, b2))


@pytest.mark.parametrize("m,n,k", [(2048, 2560, 512), (3000, 2000, 300), (1100, 4400, 1000)])
@pytest.mark.parametrize("p", [131, 2])
def test_tc_gemm_persistent(gpu, oracle, m, n, k, p, monkeypatch):
    """The persistent tcgen05 kernel (128x256 tiles, double-buffered TMEM accumulators):
    large outputs with partial M/N tiles and K not a multiple of the 128-byte stage."""
    import paper_1802_10453_b200 as ffb
    monkeypatch.setenv("FFB_GEMM_PATH", "tc")
    rng = np.random.default_rng(m + n + k + p)
    a = rng.integers(0, p, (m, k), dtype=np.uint64)
    b = rng.integers(0, p, (k, n), dtype=np.uint64)
    c = rng.integers(0, p, (m, n), dtype=np.uint64)
    assert np.array_equal(ffb.gemm_sub(c, a, b, p, ctx=gpu), oracle.gemm_sub(p, c, a, b))


@pytest.mark.parametrize("n,k", [(1024, 131), (1536, 200), (2304, 64)])
@pytest.mark.parametrize("p", [2, 131])
def test_syr2k_single_accumulator(gpu, oracle, n, k, p):
    """SYR2K C -= A^T B + B^T A as ONE tcgen05 GEMM over the K-concatenated terms
    (tc_gemm2: each 16-padded K segment packed side by side, one TMEM accumulator,
    kernels.cpp:121-135), including odd K (zero padding between the segments)."""
    import paper_1802_10453_b200 as ffb
    rng = np.random.default_rng(n + k + p)
    c = rand_sym(rng, p, n)
    a = rng.integers(0, p, (k, n), dtype=np.uint64)
    b = rng.integers(0, p, (k, n), dtype=np.uint64)
    assert np.array_equal(ffb.syr2k_sub(c, a, b, p, ctx=gpu), oracle.syr2k_sub(p, c, a, b))
