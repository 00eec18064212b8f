"""The seeded cases whose reference outputs are pinned in tests/golden/ref_outputs.npz."""
import numpy as np

from helpers import hollow, rand_low_rank, rand_rook_rpm, rand_sym


def golden_cases():
    """Yield (name, p, a, variant, threshold) deterministically."""
    from paper_1802_10453_b200 import configs
    cases = []
    for p in (2, 3, 7, 131, 8388593):
        rng = np.random.default_rng(1000 + p)
        for n in (5, 17, 40, 64, 65, 96, 130):
            cases.append((f"sym/p{p}/n{n}", p, rand_sym(rng, p, n), "cascade", 64))
            cases.append((f"low/p{p}/n{n}", p, rand_low_rank(rng, p, n, n // 2), "cascade", 64))
            cases.append((f"rook/p{p}/n{n}", p, rand_rook_rpm(rng, p, n, n // 2), "cascade", 64))
            cases.append((f"hollow/p{p}/n{n}", p, hollow(rng, p, n), "cascade", 64))
        for v, T in (("recursive", 64), ("cascade", 8), ("cascade", 3)):
            cases.append((f"var/{v}{T}/p{p}", p, rand_rook_rpm(rng, p, 48, 24), v, T))
    for c in (1, 2, 3, 4, 5):
        for n in (128, 256):
            w = configs.CONFIGS[c].scaled(n)
            cases.append((f"config{c}/n{n}", w.p, configs.generate(w), "cascade", 64))
    return cases
