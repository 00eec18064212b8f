"""Full-size parity (BASELINE.json sizes) and the device-side verification API.

Bit-exact: test_full_size_bit_exact hashes ffb_ldlt_device's P, L, D and rank at the stated
size of every configuration and compares them with tests/golden/fullsize.json -- the CPU
oracle's outputs on the same seeded inputs (tests/golden/make_fullsize.py; config 2 also
cross-checked against the unmodified reference).  Since (P, L, D) depend on the recursion
tree for non-generic rank profiles, this is the check that pins the triple.

On top of that, size-independent properties, all computed on the device through the C-ABI
(ffb_verify_device, ffb_pivoting_partners_device):
  * reconstruction: P L D L^T P^T == A entry for entry (blockdiag.hpp:161-182), 0 mismatches;
  * structure (test_sytrf.cpp:19-52): L unit lower trapezoidal in position order, perm a
    permutation with the pivotless rows ascending, D blocks well formed and invertible;
  * rank (configs 2 and 5 have it by construction) and, for config 5, the rank profile
    matrix Pi = P support(D) P^T equal to the generator's R (rpmtools.cpp:61-68).
The verification API itself is pinned against the oracle at small sizes.
"""
import numpy as np
import pytest

from helpers import rand_rook_rpm, rand_sym

pytestmark = pytest.mark.gpu


def _factor(gpu, a0, p, v="cascade", t=64):
    import paper_1802_10453_b200 as ffb
    from paper_1802_10453_b200.device import ldlt_device
    cfg = ffb.SytrfConfig({"cascade": ffb.Variant.Cascade, "crout": ffb.Variant.Crout}[v], t)
    return ldlt_device(a0.clone(), p, cfg, gpu)


def _structure(f, n):
    import torch
    r = f.rank
    perm = f.perm.cpu().numpy()
    assert np.array_equal(np.sort(perm), np.arange(n))
    assert np.all(np.diff(perm[r:]) > 0), "pivotless rows must stay ascending"
    if r == 0:
        return
    top = f.lower[:r, :r]
    assert bool(torch.all(torch.diagonal(top) == 1)), "L must be unit on the pivot block"
    assert bool(torch.all(torch.triu(top, 1) == 0)), "L must be lower trapezoidal"
    kind = f.dkind[:r].cpu().numpy()
    val = f.dval[:r].cpu().numpy()
    assert np.all(val != 0)
    t = 0
    while t < r:
        if kind[t] == 0:
            t += 1
        else:
            assert kind[t] in (1, 3) and t + 1 < r and kind[t + 1] == kind[t] + 1
            t += 2


class _DeviceRows:
    """Row blocks of a device int32 matrix, fetched on demand as uint32 numpy arrays."""

    def __init__(self, t):
        self.t = t

    def __getitem__(self, idx):
        return self.t[idx].cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_full_size_bit_exact(gpu, c):
    """P, L, D, rank at the configuration's stated size == the oracle's, digest for digest."""
    import json
    import os
    import sys
    from paper_1802_10453_b200 import configs
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from make_fullsize import digest
    with open(os.path.join(here, "fullsize.json")) as fh:
        gold = json.load(fh)[str(c)]
    w = configs.CONFIGS[c]
    assert (gold["n"], gold["p"], gold["seed"], gold["rank_param"]) == (w.n, w.p, w.seed, w.r)
    a0 = configs.generate_device(w, gpu)
    f = _factor(gpu, a0, w.p)
    del a0
    r = f.rank
    d = digest(f.perm.cpu().numpy().astype(np.int64), _DeviceRows(f.lower),
               f.dkind[:r].cpu().numpy(), f.dval[:r].cpu().numpy().view(np.uint32),
               f.dval2[:r].cpu().numpy().view(np.uint32), r)
    assert d["rank"] == gold["rank"]
    assert d["perm"] == gold["perm"], "P differs"
    assert d["dkind"] == gold["dkind"] and d["dval"] == gold["dval"] and d["dval2"] == gold["dval2"], "D differs"
    bad = [i for i, (x, y) in enumerate(zip(d["lower_blocks"], gold["lower_blocks"])) if x != y]
    assert not bad and len(d["lower_blocks"]) == len(gold["lower_blocks"]), f"L differs in row blocks {bad}"


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_full_size_properties(gpu, c):
    from paper_1802_10453_b200 import configs
    from paper_1802_10453_b200.device import pivoting_partners, reconstruction_mismatches
    w = configs.CONFIGS[c]
    a0 = configs.generate_device(w, gpu)
    f = _factor(gpu, a0, w.p)
    _structure(f, w.n)
    if c in (2, 5):
        assert f.rank == w.r
    assert reconstruction_mismatches(a0, f, w.p, gpu) == 0
    if c == 5:
        part = pivoting_partners(f, gpu).cpu().numpy()
        assert np.array_equal(part, configs.config5_partners(w).astype(np.int32))


def test_verification_detects_corruption(gpu):
    """The checker is not vacuous: one changed entry of L or D is caught."""
    from paper_1802_10453_b200 import configs
    from paper_1802_10453_b200.device import reconstruction_mismatches
    w = configs.CONFIGS[5].scaled(2048)
    a0 = configs.generate_device(w, gpu)
    f = _factor(gpu, a0, w.p)
    assert reconstruction_mismatches(a0, f, w.p, gpu) == 0
    f.lower[w.n - 1, 5] = (f.lower[w.n - 1, 5] + 1) % w.p
    assert reconstruction_mismatches(a0, f, w.p, gpu) > 0
    f.lower[w.n - 1, 5] = (f.lower[w.n - 1, 5] + w.p - 1) % w.p
    f.dval[0] = (f.dval[0] % (w.p - 1)) + 1 if int(f.dval[0]) != 1 else 2
    assert reconstruction_mismatches(a0, f, w.p, gpu) > 0


@pytest.mark.parametrize("p", [2, 3, 131, 8388593])
def test_verification_api_matches_oracle(gpu, oracle, p):
    """Partners equal the oracle's pivoting_matrix; reconstruction is exact, including
    AntiDiag and (p = 2) AntiTri blocks."""
    import torch
    from oracle.bind import pivoting_matrix
    from paper_1802_10453_b200.device import pivoting_partners, reconstruction_mismatches
    rng = np.random.default_rng(11 + p)
    for n in (1, 7, 64, 130, 300):
        for a in (rand_sym(rng, p, n), rand_rook_rpm(rng, p, n, n // 2)):
            a0 = torch.from_numpy(a.astype(np.int64)).to(torch.int32).cuda()
            f = _factor(gpu, a0, p)
            o = oracle.ldlt(p, a, "cascade", 64)
            assert f.rank == o.rank
            assert reconstruction_mismatches(a0, f, p, gpu) == 0, (p, n)
            pi = pivoting_matrix(o)
            want = np.where(pi.any(axis=1), pi.argmax(axis=1), -1)
            assert np.array_equal(pivoting_partners(f, gpu).cpu().numpy(), want), (p, n)
