/* gen_oracle.c -- TEST INFRASTRUCTURE ONLY: the benchmark input generators on the CPU.
 *
 * A plain-C restatement of the seeded counter-based generators of the five
 * BASELINE.json configurations (the product's csrc/ffb_gen.cu), so the
 * CPU legs of bench.py (--impl reference, cpu_baseline) and the golden scripts can
 * build their inputs without loading the product library.  Each entry is a pure
 * function of (seed, stream, i, j); tests/test_oracle.py checks this file against
 * ffb_generate_host element for element.
 *
 *   1/3  dense symmetric, upper entries uniform in [0, p), mirrored
 *   2    A = M' diag(d) M'^T with M' = Q M (rows permuted), M uniform, d in [1, p)
 *   4    hollow: zero diagonal, off-diagonal uniform
 *   5    A = L R L^T, L unit lower (strict part uniform), R a symmetric partial
 *        permutation with r - 2*(r/4) fixed points and r/4 transposition pairs.
 */
#include <stdint.h>
#include <stdlib.h>

#include "oracle_api.h"

typedef unsigned __int128 u128;

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t hash4(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j) {
    uint64_t z = mix64(seed + 0x9E3779B97F4A7C15ull * (stream + 1));
    z = mix64(z ^ (i + 0x632BE59BD9B4E019ull));
    z = mix64(z ^ (j * 0x9E3779B97F4A7C15ull + 0x8CB92BA72F3D8DD7ull));
    return z;
}

/* uniform in [0, range): high word of hash * range */
static uint64_t uni(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j, uint64_t range) {
    return (uint64_t)(((u128)hash4(seed, stream, i, j) * range) >> 64);
}

typedef struct {
    uint64_t key;
    int64_t idx;
} KeyIdx;

static int cmp_key(const void* a, const void* b) {
    const KeyIdx* x = (const KeyIdx*)a;
    const KeyIdx* y = (const KeyIdx*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* seeded permutation of [0, n): indices sorted by hashed key, ties by index */
static void permutation(int64_t n, uint64_t seed, uint64_t stream, int64_t* out) {
    KeyIdx* k = (KeyIdx*)malloc((size_t)(n ? n : 1) * sizeof(KeyIdx));
    for (int64_t i = 0; i < n; ++i) {
        k[i].key = hash4(seed, stream, (uint64_t)i, 0);
        k[i].idx = i;
    }
    qsort(k, (size_t)n, sizeof(KeyIdx), cmp_key);
    for (int64_t i = 0; i < n; ++i) out[i] = k[i].idx;
    free(k);
}

static uint64_t dense_entry(uint64_t seed, uint64_t p, int64_t i, int64_t j, int hollow) {
    if (hollow && i == j) return 0;
    const int64_t a = i < j ? i : j, b = i < j ? j : i;
    return uni(seed, 0, (uint64_t)a, (uint64_t)b, p);
}

static uint64_t l5_entry(uint64_t seed, uint64_t p, int64_t i, int64_t a) {
    if (a > i) return 0;
    if (a == i) return 1 % p;
    return uni(seed, 1, (uint64_t)i, (uint64_t)a, p);
}

/* partner[a] of configuration 5's R (-1: row a of R is zero) */
int orc_config5_partners(size_t n_, size_t r_, uint64_t seed, int64_t* partner) {
    const int64_t n = (int64_t)n_, r = (int64_t)r_;
    if (r > n) return ORC_DIMENSION_MISMATCH;
    int64_t* pi = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
    permutation(n, seed, 4, pi);
    for (int64_t i = 0; i < n; ++i) partner[i] = -1;
    const int64_t npairs = r / 4, nfixed = r - 2 * npairs;
    for (int64_t k = 0; k < nfixed; ++k) partner[pi[k]] = pi[k];
    for (int64_t t = 0; t < npairs; ++t) {
        const int64_t a = pi[nfixed + 2 * t], b = pi[nfixed + 2 * t + 1];
        partner[a] = b;
        partner[b] = a;
    }
    free(pi);
    return ORC_OK;
}

/* out: n x n uint64 residues of configuration `config` (1..5), rank parameter r */
int orc_generate(int config, size_t n_, size_t r_, uint64_t p, uint64_t seed, uint64_t* out) {
    if (config < 1 || config > 5) return ORC_OTHER;
    if (p < 2 || p >= (1ull << 31)) return ORC_OTHER;
    const int64_t n = (int64_t)n_, r = (int64_t)r_;
    if ((config == 2 || config == 5) && r > n) return ORC_DIMENSION_MISMATCH;
    if (config == 1 || config == 3 || config == 4) {
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) out[i * n + j] = dense_entry(seed, p, i, j, config == 4);
        return ORC_OK;
    }
    /* A = U V^T with U, V n x r */
    uint64_t* U = (uint64_t*)malloc((size_t)(n > 0 && r > 0 ? n * r : 1) * sizeof(uint64_t));
    uint64_t* V = (uint64_t*)malloc((size_t)(n > 0 && r > 0 ? n * r : 1) * sizeof(uint64_t));
    if (config == 2) {
        int64_t* q = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
        permutation(n, seed, 3, q);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t k = 0; k < r; ++k) {
                const uint64_t m = uni(seed, 1, (uint64_t)q[i], (uint64_t)k, p);
                const uint64_t d = 1 + uni(seed, 2, (uint64_t)k, 0, p - 1);
                V[i * r + k] = m;
                U[i * r + k] = (m * d) % p;
            }
        free(q);
    } else {
        int64_t* partner = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
        orc_config5_partners(n_, r_, seed, partner);
        int64_t* ua = (int64_t*)malloc((size_t)(r ? r : 1) * sizeof(int64_t));
        int64_t* ub = (int64_t*)malloc((size_t)(r ? r : 1) * sizeof(int64_t));
        int64_t t = 0;
        for (int64_t a = 0; a < n; ++a)
            if (partner[a] >= 0) {
                ua[t] = a;
                ub[t] = partner[a];
                ++t;
            }
        for (int64_t i = 0; i < n; ++i)
            for (int64_t k = 0; k < r; ++k) {
                U[i * r + k] = l5_entry(seed, p, i, ua[k]);
                V[i * r + k] = l5_entry(seed, p, i, ub[k]);
            }
        free(partner);
        free(ua);
        free(ub);
    }
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            const uint64_t* u = U + i * r;
            const uint64_t* v = V + j * r;
            if (p < 65536) { /* products < 2^32: 2^32 of them fit one uint64 */
                uint64_t acc = 0;
                for (int64_t k = 0; k < r; ++k) acc += u[k] * v[k];
                out[i * n + j] = acc % p;
            } else {
                u128 acc = 0;
                for (int64_t k = 0; k < r; ++k) acc += (u128)(u[k] * v[k]); /* p < 2^31 */
                out[i * n + j] = (uint64_t)(acc % p);
            }
        }
    free(U);
    free(V);
    return ORC_OK;
}
