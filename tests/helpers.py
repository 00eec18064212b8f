"""Shared test helpers: seeded inputs and comparisons of GPU vs oracle outputs."""
import numpy as np


def rand_sym(rng, p, n):
    a = rng.integers(0, p, (n, n), dtype=np.uint64)
    a = np.triu(a)
    return a + np.triu(a, 1).T


def rand_low_rank(rng, p, n, k):
    """X^T S X with X k x n and S symmetric k x k (test oracle.hpp:101-144 family)."""
    if k == 0 or n == 0:
        return np.zeros((n, n), np.uint64)
    x = rng.integers(0, p, (k, n)).astype(object)
    s = rand_sym(rng, p, k).astype(object)
    return (x.T.dot(s).dot(x) % p).astype(np.uint64)


def rand_rook_rpm(rng, p, n, r):
    """L R L^T with a random symmetric rook placement R of rank r (genbench.hpp:19-30 family)."""
    perm = rng.permutation(n)
    R = np.zeros((n, n), dtype=object)
    npairs = r // 4
    nfixed = r - 2 * npairs
    for i in perm[:nfixed]:
        R[i, i] = int(rng.integers(1, p))
    for t in range(npairs):
        a, b = perm[nfixed + 2 * t], perm[nfixed + 2 * t + 1]
        v = int(rng.integers(1, p))
        R[a, b] = R[b, a] = v
    L = np.tril(rng.integers(0, p, (n, n)), -1).astype(object) + np.eye(n, dtype=object)
    return ((L.dot(R).dot(L.T)) % p).astype(np.uint64)


def hollow(rng, p, n):
    a = rand_sym(rng, p, n)
    np.fill_diagonal(a, 0)
    return a


def fact_equal(gpu_fact, orc_fact) -> bool:
    """Bit-exact comparison of ffldl.Factorization (GPU) with oracle.bind.Fact."""
    kind, val, val2 = gpu_fact.diag.columns()
    return (gpu_fact.rank == orc_fact.rank
            and np.array_equal(gpu_fact.perm.image_array(), orc_fact.perm)
            and np.array_equal(gpu_fact.lower, orc_fact.lower)
            and np.array_equal(kind, orc_fact.dkind)
            and np.array_equal(val, orc_fact.dval)
            and np.array_equal(val2, orc_fact.dval2))


def describe_diff(g, o) -> str:
    kind, val, val2 = g.diag.columns()
    parts = [f"rank {g.rank} vs {o.rank}"]
    if g.rank == o.rank:
        parts.append(f"perm eq {np.array_equal(g.perm.image_array(), o.perm)}")
        parts.append(f"lower eq {np.array_equal(g.lower, o.lower)}")
        parts.append(f"dkind eq {np.array_equal(kind, o.dkind)} dval eq {np.array_equal(val, o.dval)}")
        if not np.array_equal(g.lower, o.lower):
            bad = np.argwhere(g.lower != o.lower)
            parts.append(f"first lower diffs {bad[:5].tolist()}")
    return "; ".join(parts)
