/* ldlt_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU oracle.
 *
 * A plain-C restatement of the reference algorithm for the hot path
 * ffldl::ldlt (arXiv 1802.10453, the `ffldl` artifact under
 * /root/reference/proj).  Every function below names the reference
 * function and file:line it restates.  It is used by tests/ (as the
 * checker the GPU path is compared against), by __graft_entry__.smoke()
 * and by bench.py's cpu_baseline leg -- never by the product.
 *
 * Parity pin: tests/test_oracle.py checks this restatement against
 *   (a) the reference's own known-answer tests (test_sytrf.cpp:62-88,
 *       test_plduq.cpp:46-57, test_trssyr2k.cpp:36-43, test_io.cpp:103-113,
 *       SPEC.md worked examples) stored in tests/golden/, and
 *   (b) the UNMODIFIED reference compiled into oracle/_ref/libffldl_ref.so
 *       (oracle/Makefile), output-for-output on seeded random inputs.
 *
 * Deliberate differences from the reference that cannot change any output:
 *   - kernels (gemm_sub, trsm_inplace, trmm_sub, syrdk_sub, syr2k_sub) are
 *     evaluated with delayed modular reduction and OpenMP over output rows
 *     (each kernel's result is a unique field value, kernels.cpp:7-135);
 *   - trsm_inplace is blocked (forward/back substitution order inside a block
 *     is the reference's, kernels.cpp:57-81); the solution is unique;
 *   - the multiplication counter of PrimeField (field.hpp:101-104,128-133) is
 *     not kept.
 * Moduli: any prime p < 2^62 (field.hpp:75), like the reference.
 */
#include <setjmp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_api.h"

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ */
/* Field Z/pZ  (restates PrimeField, proj/include/ffldl/field.hpp:73-134) */
/* ------------------------------------------------------------------ */

static uint64_t P;          /* modulus of the current call */
static uint64_t CHUNK;      /* products that fit one uint64 accumulator (p < 2^32) */
static jmp_buf ERR_JMP;     /* error escape (the reference throws) */

static void fail(int code) { longjmp(ERR_JMP, code); }

static inline uint64_t fadd(uint64_t a, uint64_t b) {
    uint64_t s = a + b; /* field.hpp:89-93 */
    return s >= P ? s - P : s;
}
static inline uint64_t fsub(uint64_t a, uint64_t b) { return a >= b ? a - b : a + P - b; }
static inline uint64_t fneg(uint64_t a) { return a == 0 ? 0 : P - a; }
static inline uint64_t fmul(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) % P); }

/* Extended Euclid, field.hpp:107-118. */
static uint64_t finv(uint64_t a) {
    if (a == 0) fail(ORC_ZERO_INVERSE);
    int64_t t = 0, nt = 1, r = (int64_t)P, nr = (int64_t)a;
    while (nr != 0) {
        int64_t q = r / nr, tmp;
        tmp = t - q * nt; t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    if (t < 0) t += (int64_t)P;
    return (uint64_t)t;
}

/* a/2 for odd p, field.hpp:121-124. */
static uint64_t fhalve(uint64_t a) {
    if (P == 2) fail(ORC_CHAR_TWO_DIVISION);
    return (a & 1) ? (a + P) / 2 : a / 2;
}

static uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) r = (uint64_t)(((u128)r * a) % m);
        a = (uint64_t)(((u128)a * a) % m);
        e >>= 1;
    }
    return r;
}

/* Deterministic Miller-Rabin over the first twelve primes (field.hpp:37-63). */
static int is_prime_u64(uint64_t n) {
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; ++i)
        if (n % bases[i] == 0) return n == bases[i];
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    for (int i = 0; i < 12; ++i) {
        uint64_t x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int witness = 1;
        for (int k = 1; k < s; ++k) {
            x = (uint64_t)(((u128)x * x) % n);
            if (x == n - 1) { witness = 0; break; }
        }
        if (witness) return 0;
    }
    return 1;
}

static void set_field(uint64_t p) {
    if (p < 2 || p > ((1ull << 62) - 1) || !is_prime_u64(p)) fail(ORC_NOT_PRIME);
    P = p;
    if (p <= 0xFFFFFFFFull) {
        uint64_t q = (p - 1) * (p - 1);
        CHUNK = q == 0 ? UINT64_MAX : UINT64_MAX / q;
        if (CHUNK == 0) CHUNK = 1;
    } else {
        CHUNK = 0; /* 128-bit path */
    }
}

/* Sum_t x[t]*y[t] mod p with delayed reduction. */
static uint64_t dotmod(const uint64_t* x, const uint64_t* y, size_t k) {
    uint64_t total = 0;
    if (CHUNK) {
        for (size_t s = 0; s < k;) {
            size_t e = (k - s > CHUNK) ? s + CHUNK : k;
            uint64_t acc = 0;
            for (size_t t = s; t < e; ++t) acc += x[t] * y[t];
            total = fadd(total, acc % P);
            s = e;
        }
    } else {
        for (size_t t = 0; t < k; ++t) total = fadd(total, fmul(x[t], y[t]));
    }
    return total;
}

/* ------------------------------------------------------------------ */
/* Dense matrices (restates Matrix, proj/include/ffldl/matrix.hpp:18-102) */
/* ------------------------------------------------------------------ */

typedef struct {
    size_t r, c;
    uint64_t* v;
} Mat;

#define AT(m, i, j) ((m).v[(size_t)(i) * (m).c + (size_t)(j)])

static Mat mat_new(size_t r, size_t c) {
    Mat m = {r, c, NULL};
    size_t cnt = r * c;
    m.v = (uint64_t*)calloc(cnt ? cnt : 1, sizeof(uint64_t));
    if (!m.v) fail(ORC_NO_MEMORY);
    return m;
}
static void mat_free(Mat* m) {
    free(m->v);
    m->v = NULL;
}
static Mat mat_copy(const Mat* a) {
    Mat m = mat_new(a->r, a->c);
    memcpy(m.v, a->v, a->r * a->c * sizeof(uint64_t));
    return m;
}
/* Copy of [r0,r1) x [c0,c1), matrix.hpp:52-58. */
static Mat mat_block(const Mat* a, size_t r0, size_t r1, size_t c0, size_t c1) {
    if (r0 > r1 || r1 > a->r || c0 > c1 || c1 > a->c) fail(ORC_DIMENSION_MISMATCH);
    Mat b = mat_new(r1 - r0, c1 - c0);
    for (size_t i = r0; i < r1; ++i)
        memcpy(&AT(b, i - r0, 0), &AT(*a, i, c0), (c1 - c0) * sizeof(uint64_t));
    return b;
}
/* matrix.hpp:61-65. */
static void mat_set_block(Mat* a, size_t r0, size_t c0, const Mat* s) {
    if (r0 + s->r > a->r || c0 + s->c > a->c) fail(ORC_DIMENSION_MISMATCH);
    for (size_t i = 0; i < s->r; ++i)
        memcpy(&AT(*a, r0 + i, c0), &AT(*s, i, 0), s->c * sizeof(uint64_t));
}
static Mat mat_transposed(const Mat* a) {
    Mat t = mat_new(a->c, a->r);
    for (size_t i = 0; i < a->r; ++i)
        for (size_t j = 0; j < a->c; ++j) AT(t, j, i) = AT(*a, i, j);
    return t;
}
static int mat_is_symmetric(const Mat* a) {
    if (a->r != a->c) return 0;
    for (size_t i = 0; i < a->r; ++i)
        for (size_t j = i + 1; j < a->c; ++j)
            if (AT(*a, i, j) != AT(*a, j, i)) return 0;
    return 1;
}
static int mat_is_zero(const Mat* a) {
    for (size_t i = 0; i < a->r * a->c; ++i)
        if (a->v[i]) return 0;
    return 1;
}

/* C(m x n) -= A(m x k) * Bt(n x k)^T, both operands K-major rows. */
static void mm_sub_kmajor(Mat* c, const uint64_t* a, const uint64_t* bt, size_t k) {
    const size_t m = c->r, n = c->c;
#pragma omp parallel for schedule(dynamic, 4) if (m * n * k > 100000)
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j)
            AT(*c, i, j) = fsub(AT(*c, i, j), dotmod(a + i * k, bt + j * k, k));
}

/* ------------------------------------------------------------------ */
/* Permutations (restates proj/include/ffldl/permutation.hpp:20-146)   */
/* image(i) = j: row i of the source becomes row j of the result.      */
/* ------------------------------------------------------------------ */

typedef struct {
    size_t n;
    size_t* img;
} Perm;

static Perm perm_identity(size_t n) {
    Perm p = {n, (size_t*)malloc((n ? n : 1) * sizeof(size_t))};
    if (!p.img) fail(ORC_NO_MEMORY);
    for (size_t i = 0; i < n; ++i) p.img[i] = i;
    return p;
}
static void perm_free(Perm* p) {
    free(p->img);
    p->img = NULL;
}
/* from_image bijection check, permutation.hpp:26-35. */
static void perm_check(const Perm* p) {
    char* seen = (char*)calloc(p->n ? p->n : 1, 1);
    for (size_t i = 0; i < p->n; ++i) {
        if (p->img[i] >= p->n || seen[p->img[i]]) { free(seen); fail(ORC_BAD_BLOCK_SIZES); }
        seen[p->img[i]] = 1;
    }
    free(seen);
}
static Perm perm_inverse(const Perm* p) {
    Perm q = perm_identity(p->n);
    for (size_t i = 0; i < p->n; ++i) q.img[p->img[i]] = i;
    return q;
}
/* compose(P,Q): image = P.image(Q.image(i)), permutation.hpp:68-73. */
static Perm perm_compose(const Perm* p, const Perm* q) {
    if (p->n != q->n) fail(ORC_DIMENSION_MISMATCH);
    Perm r = perm_identity(p->n);
    for (size_t i = 0; i < p->n; ++i) r.img[i] = p->img[q->img[i]];
    return r;
}
/* embed(P, offset, total), permutation.hpp:139-146. */
static Perm perm_embed(const Perm* p, size_t off, size_t total) {
    if (off + p->n > total) fail(ORC_DIMENSION_MISMATCH);
    Perm r = perm_identity(total);
    for (size_t i = 0; i < p->n; ++i) r.img[off + i] = off + p->img[i];
    return r;
}
/* dense(P)^T * B: r(i,.) = b(image(i),.), permutation.hpp:95-101. */
static Mat permute_rows_inv(const Perm* p, const Mat* b) {
    if (p->n != b->r) fail(ORC_DIMENSION_MISMATCH);
    Mat r = mat_new(b->r, b->c);
    for (size_t i = 0; i < b->r; ++i)
        memcpy(&AT(r, i, 0), &AT(*b, p->img[i], 0), b->c * sizeof(uint64_t));
    return r;
}
/* r(image(i), image(j)) = c(i,j), permutation.hpp:122-129. */
static Mat conjugate_sym(const Perm* p, const Mat* c) {
    if (p->n != c->r || p->n != c->c) fail(ORC_DIMENSION_MISMATCH);
    Mat r = mat_new(c->r, c->c);
    for (size_t i = 0; i < c->r; ++i)
        for (size_t j = 0; j < c->c; ++j) AT(r, p->img[i], p->img[j]) = AT(*c, i, j);
    return r;
}

/* ------------------------------------------------------------------ */
/* Block diagonal D (restates BlockDiag, blockdiag.hpp:39-144)          */
/* ------------------------------------------------------------------ */

enum { BK_SCALAR = 0, BK_ANTIDIAG = 1, BK_ANTITRI = 2 };
typedef struct {
    int kind;
    uint64_t a, b; /* Scalar: a=d. AntiDiag: a=x. AntiTri: a=c, b=d. */
} Blk;
typedef struct {
    Blk* blk;
    size_t* off;
    size_t nb, cap, order;
} BDiag;

static void bd_init(BDiag* d) { memset(d, 0, sizeof(*d)); }
static void bd_free(BDiag* d) {
    free(d->blk);
    free(d->off);
    bd_init(d);
}
/* push, blockdiag.hpp:43-47. */
static void bd_push(BDiag* d, Blk b) {
    if (d->nb == d->cap) {
        d->cap = d->cap ? 2 * d->cap : 8;
        d->blk = (Blk*)realloc(d->blk, d->cap * sizeof(Blk));
        d->off = (size_t*)realloc(d->off, d->cap * sizeof(size_t));
        if (!d->blk || !d->off) fail(ORC_NO_MEMORY);
    }
    d->off[d->nb] = d->order;
    d->order += b.kind == BK_SCALAR ? 1 : 2;
    d->blk[d->nb++] = b;
}
static void bd_append(BDiag* d, const BDiag* o) {
    for (size_t k = 0; k < o->nb; ++k) bd_push(d, o->blk[k]);
}
static BDiag bd_copy(const BDiag* o) {
    BDiag d;
    bd_init(&d);
    bd_append(&d, o);
    return d;
}

/* D^-1 * X, blockdiag.hpp:112-138. */
static Mat bd_inverse_apply(const BDiag* d, const Mat* x) {
    if (x->r != d->order) fail(ORC_DIMENSION_MISMATCH);
    Mat r = mat_new(x->r, x->c);
    for (size_t k = 0; k < d->nb; ++k) {
        const size_t t = d->off[k];
        const Blk b = d->blk[k];
        if (b.kind == BK_SCALAR) {
            const uint64_t di = finv(b.a);
            for (size_t j = 0; j < x->c; ++j) AT(r, t, j) = fmul(di, AT(*x, t, j));
        } else if (b.kind == BK_ANTIDIAG) {
            const uint64_t xi = finv(b.a);
            for (size_t j = 0; j < x->c; ++j) {
                AT(r, t, j) = fmul(xi, AT(*x, t + 1, j));
                AT(r, t + 1, j) = fmul(xi, AT(*x, t, j));
            }
        } else {
            const uint64_t ci = finv(b.a);
            const uint64_t top = fneg(fmul(b.b, fmul(ci, ci)));
            for (size_t j = 0; j < x->c; ++j) {
                AT(r, t, j) = fadd(fmul(top, AT(*x, t, j)), fmul(ci, AT(*x, t + 1, j)));
                AT(r, t + 1, j) = fmul(ci, AT(*x, t, j));
            }
        }
    }
    return r;
}

/* ------------------------------------------------------------------ */
/* Kernels (restate proj/src/kernels.cpp)                              */
/* ------------------------------------------------------------------ */

enum { LOWER = 0, UPPER = 1 };

/* C <- C - A*B, kernels.cpp:7-18. */
static void gemm_sub(Mat* c, const Mat* a, const Mat* b) {
    if (a->r != c->r || b->c != c->c || a->c != b->r) fail(ORC_DIMENSION_MISMATCH);
    if (a->c == 0 || c->r == 0 || c->c == 0) return;
    Mat bt = mat_transposed(b);
    mm_sub_kmajor(c, a->v, bt.v, a->c);
    mat_free(&bt);
}

/* Entry of op(T), kernels.cpp:23-29. */
static uint64_t tri_entry(const Mat* t, int uplo, int trans, int unit, size_t i, size_t j) {
    if (trans) { size_t s = i; i = j; j = s; }
    if (i == j) return unit ? 1 % P : AT(*t, i, i);
    const int stored = (uplo == LOWER) ? (i > j) : (i < j);
    return stored ? AT(*t, i, j) : 0;
}

/* Dense op(T) with the triangle/unit conventions applied. */
static Mat dense_op(const Mat* t, int uplo, int trans, int unit) {
    Mat o = mat_new(t->r, t->c);
    for (size_t i = 0; i < t->r; ++i)
        for (size_t j = 0; j < t->c; ++j) AT(o, i, j) = tri_entry(t, uplo, trans, unit, i, j);
    return o;
}

/* C <- C - op(T)*B, kernels.cpp:33-55. */
static void trmm_sub(Mat* c, const Mat* t, int uplo, int trans, int unit, const Mat* b) {
    if (t->r != t->c || t->c != b->r || c->r != b->r || c->c != b->c) fail(ORC_DIMENSION_MISMATCH);
    if (t->r == 0 || c->c == 0) return;
    Mat o = dense_op(t, uplo, trans, unit);
    gemm_sub(c, &o, b);
    mat_free(&o);
}

/* B <- op(T)^-1 B, kernels.cpp:57-81: substitution inside blocks of TB rows,
 * GEMM updates between blocks (the solution is unique). */
#define TB 64
static void trsm_inplace(const Mat* t, int uplo, int trans, int unit, Mat* b) {
    if (t->r != t->c || t->c != b->r) fail(ORC_DIMENSION_MISMATCH);
    const size_t n = t->r, nc = b->c;
    if (n == 0 || nc == 0) {
        /* still validate the diagonal like the reference would */
        return;
    }
    Mat o = dense_op(t, uplo, trans, unit); /* op(T), effective lower or upper */
    const int lower = (uplo == LOWER) != (trans != 0);
    uint64_t* pinv = (uint64_t*)malloc(n * sizeof(uint64_t));
    for (size_t step = 0; step < n; ++step) {
        const size_t i = lower ? step : n - 1 - step;
        if (unit) {
            pinv[i] = 1 % P;
        } else {
            if (AT(o, i, i) == 0) { free(pinv); mat_free(&o); fail(ORC_SINGULAR_TRIANGULAR); }
            pinv[i] = finv(AT(o, i, i));
        }
    }
    Mat bt = mat_transposed(b); /* nc x n: solve column by column */
    const size_t nblk = (n + TB - 1) / TB;
    for (size_t s = 0; s < nblk; ++s) {
        const size_t blk = lower ? s : nblk - 1 - s;
        const size_t i0 = blk * TB, i1 = (i0 + TB < n) ? i0 + TB : n;
        /* substitution inside the block (forward for lower, backward for upper) */
#pragma omp parallel for schedule(static) if (nc > 64)
        for (size_t j = 0; j < nc; ++j) {
            uint64_t* x = &AT(bt, j, 0);
            for (size_t st = i0; st < i1; ++st) {
                const size_t i = lower ? st : i0 + i1 - 1 - st;
                uint64_t acc = x[i];
                if (lower) {
                    for (size_t k = i0; k < i; ++k) acc = fsub(acc, fmul(AT(o, i, k), x[k]));
                } else {
                    for (size_t k = i + 1; k < i1; ++k) acc = fsub(acc, fmul(AT(o, i, k), x[k]));
                }
                x[i] = unit ? acc : fmul(pinv[i], acc);
            }
        }
        /* update the not-yet-solved rows with this block */
        const size_t r0 = lower ? i1 : 0, r1 = lower ? n : i0;
        if (r1 > r0) {
            Mat tpanel = mat_new(r1 - r0, i1 - i0); /* op(T)[r0:r1, i0:i1] */
            for (size_t i = r0; i < r1; ++i)
                memcpy(&AT(tpanel, i - r0, 0), &AT(o, i, i0), (i1 - i0) * sizeof(uint64_t));
#pragma omp parallel for schedule(static) if (nc * (r1 - r0) > 4096)
            for (size_t j = 0; j < nc; ++j) {
                uint64_t* x = &AT(bt, j, 0);
                for (size_t i = r0; i < r1; ++i)
                    x[i] = fsub(x[i], dotmod(&AT(tpanel, i - r0, 0), x + i0, i1 - i0));
            }
            mat_free(&tpanel);
        }
    }
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < nc; ++j) AT(*b, i, j) = AT(bt, j, i);
    mat_free(&bt);
    mat_free(&o);
    free(pinv);
}

/* C <- C - G*D*G^t with block diagonal D, kernels.cpp:83-106. */
static void syrdk_sub_bd(Mat* c, const Mat* g, const BDiag* d) {
    if (c->r != c->c || g->r != c->r || g->c != d->order) fail(ORC_DIMENSION_MISMATCH);
    if (g->c == 0 || c->r == 0) return;
    /* H = G*D (rows of G times D), then C -= H * G^t */
    Mat h = mat_new(g->r, g->c);
    for (size_t k = 0; k < d->nb; ++k) {
        const size_t t = d->off[k];
        const Blk b = d->blk[k];
        for (size_t i = 0; i < g->r; ++i) {
            if (b.kind == BK_SCALAR) {
                AT(h, i, t) = fmul(AT(*g, i, t), b.a);
            } else if (b.kind == BK_ANTIDIAG) {
                AT(h, i, t) = fmul(AT(*g, i, t + 1), b.a);
                AT(h, i, t + 1) = fmul(AT(*g, i, t), b.a);
            } else {
                AT(h, i, t) = fmul(AT(*g, i, t + 1), b.a);
                AT(h, i, t + 1) = fadd(fmul(AT(*g, i, t), b.a), fmul(AT(*g, i, t + 1), b.b));
            }
        }
    }
    mm_sub_kmajor(c, h.v, g->v, g->c);
    mat_free(&h);
}

/* C <- C - G*diag(d)*G^t, kernels.cpp:108-119. */
static void syrdk_sub_diag(Mat* c, const Mat* g, const uint64_t* d, size_t nd) {
    if (c->r != c->c || g->r != c->r || g->c != nd) fail(ORC_DIMENSION_MISMATCH);
    if (nd == 0 || c->r == 0) return;
    Mat h = mat_new(g->r, g->c);
    for (size_t i = 0; i < g->r; ++i)
        for (size_t k = 0; k < nd; ++k) AT(h, i, k) = fmul(AT(*g, i, k), d[k]);
    mm_sub_kmajor(c, h.v, g->v, g->c);
    mat_free(&h);
}

/* C <- C - A^t B - B^t A for k x n operands, kernels.cpp:121-135. */
static void syr2k_sub(Mat* c, const Mat* a, const Mat* b) {
    if (c->r != c->c || a->c != c->r || b->c != c->r || a->r != b->r) fail(ORC_DIMENSION_MISMATCH);
    if (a->r == 0 || c->r == 0) return;
    Mat at = mat_transposed(a), bt = mat_transposed(b);
    mm_sub_kmajor(c, at.v, bt.v, a->r);
    mm_sub_kmajor(c, bt.v, at.v, a->r);
    mat_free(&at);
    mat_free(&bt);
}

/* ------------------------------------------------------------------ */
/* PLDUQ (restates proj/src/plduq.cpp:36-123)                          */
/* ------------------------------------------------------------------ */

typedef struct {
    Perm row_perm, col_perm;
    Mat lower;     /* m x r, [L1; M1] */
    uint64_t* diag;
    Mat upper;     /* r x n, [U1 V1] */
    size_t rank;
} Plduq;

static void plduq_free(Plduq* f) {
    perm_free(&f->row_perm);
    perm_free(&f->col_perm);
    mat_free(&f->lower);
    mat_free(&f->upper);
    free(f->diag);
}

static Plduq plduq(const Mat* b) {
    const size_t m = b->r, n = b->c;
    Mat w = mat_copy(b); /* plduq.cpp:40 */
    size_t* pr = (size_t*)malloc((m + 1) * sizeof(size_t));
    size_t* pc = (size_t*)malloc((m + 1) * sizeof(size_t));
    size_t* mrows = (size_t*)malloc((m + 1) * sizeof(size_t));
    uint64_t* d = (uint64_t*)malloc((m + 1) * sizeof(uint64_t));
    char* is_piv = (char*)calloc(n + 1, 1);
    uint64_t* coef = (uint64_t*)malloc((m + 1) * sizeof(uint64_t));
    u128* acc = (u128*)malloc((n + 1) * sizeof(u128));
    size_t r = 0, nm = 0;

    for (size_t i = 0; i < m; ++i) { /* plduq.cpp:46 */
        /* u_j = W(i,j) - sum_k W(i,pc_k) d_k W(pr_k,j) on non-pivot columns, :51-59 */
        for (size_t k = 0; k < r; ++k) coef[k] = fmul(AT(w, i, pc[k]), d[k]);
#pragma omp parallel for schedule(static) if (n * r > 1 << 16)
        for (size_t j = 0; j < n; ++j) {
            if (is_piv[j]) continue;
            uint64_t s = 0;
            for (size_t k = 0; k < r; ++k) s = fadd(s, fmul(coef[k], AT(w, pr[k], j)));
            AT(w, i, j) = fsub(AT(w, i, j), s);
        }
        size_t jp = n;
        for (size_t j = 0; j < n; ++j)
            if (!is_piv[j] && AT(w, i, j) != 0) { jp = j; break; }
        if (jp == n) { mrows[nm++] = i; continue; } /* :60-63 */
        const uint64_t x = AT(w, i, jp);
        const uint64_t xi = finv(x);
        for (size_t j = 0; j < n; ++j) /* scale pivot row into U, :65-70 */
            if (!is_piv[j] && j != jp) AT(w, i, j) = fmul(xi, AT(w, i, j));
        /* update + scale column jp for the rows still to come, :74-79 */
#pragma omp parallel for schedule(static) if ((m - i) * r > 1 << 16)
        for (size_t i2 = i + 1; i2 < m; ++i2) {
            uint64_t s = AT(w, i2, jp);
            for (size_t k = 0; k < r; ++k)
                s = fsub(s, fmul(fmul(AT(w, i2, pc[k]), d[k]), AT(w, pr[k], jp)));
            AT(w, i2, jp) = fmul(xi, s);
        }
        pr[r] = i; pc[r] = jp; d[r] = x; ++r; /* :80-83 */
        is_piv[jp] = 1;
    }
    (void)acc;

    Plduq f;
    f.rank = r;
    f.row_perm = perm_identity(m);
    f.col_perm = perm_identity(n);
    for (size_t k = 0; k < r; ++k) f.row_perm.img[k] = pr[k]; /* :86-94 */
    for (size_t t = 0; t < nm; ++t) f.row_perm.img[r + t] = mrows[t];
    size_t q = r;
    for (size_t k = 0; k < r; ++k) f.col_perm.img[k] = pc[k];
    for (size_t j = 0; j < n; ++j)
        if (!is_piv[j]) f.col_perm.img[q++] = j;
    f.lower = mat_new(m, r); /* :100-106 */
    for (size_t a = 0; a < m; ++a)
        for (size_t k = 0; k < r; ++k) {
            if (a == k) AT(f.lower, a, k) = 1 % P;
            else if (a > k) AT(f.lower, a, k) = AT(w, f.row_perm.img[a], pc[k]);
        }
    f.upper = mat_new(r, n); /* :107-113 */
    for (size_t k = 0; k < r; ++k)
        for (size_t a = 0; a < n; ++a) {
            if (a == k) AT(f.upper, k, a) = 1 % P;
            else if (a > k) AT(f.upper, k, a) = AT(w, pr[k], f.col_perm.img[a]);
        }
    f.diag = (uint64_t*)malloc((r + 1) * sizeof(uint64_t));
    memcpy(f.diag, d, r * sizeof(uint64_t));
    free(pr); free(pc); free(mrows); free(d); free(is_piv); free(coef); free(acc);
    mat_free(&w);
    return f;
}

/* ------------------------------------------------------------------ */
/* TRSSYR2K, Alg. 1 (restates proj/src/trssyr2k.cpp:19-77)             */
/* ------------------------------------------------------------------ */

static void solve_block(const Mat* u, Mat* c) {
    const size_t n = c->r;
    if (n == 1) { /* trssyr2k.cpp:22-30 */
        if (P == 2) {
            if (AT(*c, 0, 0) != 0) fail(ORC_CHAR_TWO_NONZERO_DIAGONAL);
            return;
        }
        AT(*c, 0, 0) = fhalve(AT(*c, 0, 0));
        return;
    }
    const size_t n1 = n / 2; /* :31 */
    Mat u1 = mat_block(u, 0, n1, 0, n1), u2 = mat_block(u, 0, n1, n1, n), u3 = mat_block(u, n1, n, n1, n);
    Mat c1 = mat_block(c, 0, n1, 0, n1);
    solve_block(&u1, &c1);
    Mat c2 = mat_block(c, 0, n1, n1, n);
    trmm_sub(&c2, &c1, UPPER, 1, 0, &u2); /* :40 */
    trsm_inplace(&u1, UPPER, 1, 1, &c2);  /* :41 */
    Mat c3 = mat_block(c, n1, n, n1, n);
    syr2k_sub(&c3, &c2, &u2); /* :44 */
    solve_block(&u3, &c3);
    mat_set_block(c, 0, 0, &c1);
    mat_set_block(c, 0, n1, &c2);
    Mat z = mat_new(n - n1, n1);
    mat_set_block(c, n1, 0, &z);
    mat_set_block(c, n1, n1, &c3);
    mat_free(&z); mat_free(&u1); mat_free(&u2); mat_free(&u3);
    mat_free(&c1); mat_free(&c2); mat_free(&c3);
}

/* trssyr2k_inplace + trssyr2k, trssyr2k.cpp:55-77. */
static Mat trssyr2k(const Mat* u, const Mat* c) {
    if (u->r != u->c || c->r != c->c || u->r != c->r) fail(ORC_DIMENSION_MISMATCH);
    for (size_t i = 0; i < u->r; ++i)
        if (AT(*u, i, i) != 1 % P) fail(ORC_NON_UNIT_TRIANGULAR);
    if (!mat_is_symmetric(c)) fail(ORC_NOT_SYMMETRIC);
    Mat x = mat_copy(c);
    if (x.r == 0) return x;
    solve_block(u, &x);
    for (size_t i = 0; i < x.r; ++i)
        for (size_t j = 0; j < i; ++j) AT(x, i, j) = 0;
    return x;
}

/* ------------------------------------------------------------------ */
/* SYTRF (restates proj/src/sytrf.cpp)                                 */
/* ------------------------------------------------------------------ */

typedef struct {
    Perm perm;
    Mat lower; /* n x rank */
    BDiag diag;
    size_t rank;
} Fact;

static void fact_free(Fact* f) {
    perm_free(&f->perm);
    mat_free(&f->lower);
    bd_free(&f->diag);
}

static int CFG_VARIANT;
static size_t CFG_T;

static Fact dispatch(const Mat* a);
static Fact zero_leading(const Mat* y, const Mat* z);

/* out[t..] = (prefix of lmat row) * D blockwise, sytrf.cpp:55-70. */
static void fold_diag(const Mat* lmat, const BDiag* diag, size_t row, uint64_t* out) {
    for (size_t k = 0; k < diag->nb; ++k) {
        const size_t t = diag->off[k];
        const Blk b = diag->blk[k];
        const uint64_t ut = AT(*lmat, row, t);
        if (b.kind == BK_SCALAR) {
            out[t] = fmul(ut, b.a);
        } else if (b.kind == BK_ANTIDIAG) {
            out[t] = fmul(AT(*lmat, row, t + 1), b.a);
            out[t + 1] = fmul(ut, b.a);
        } else {
            out[t] = fmul(AT(*lmat, row, t + 1), b.a);
            out[t + 1] = fadd(fmul(ut, b.a), fmul(AT(*lmat, row, t + 1), b.b));
        }
    }
}

/* Residual of original row `row` against column `col`, sytrf.cpp:48-53. */
static uint64_t residual(const Mat* a, const Mat* lmat, size_t row, size_t col, size_t r,
                         const uint64_t* w) {
    return fsub(AT(*a, row, col), dotmod(&AT(*lmat, row, 0), w, r));
}

static void rotate_one(size_t* v, size_t first, size_t middle) {
    /* std::rotate(v+first, v+middle, v+middle+1): v[middle] moves to first. */
    const size_t x = v[middle];
    memmove(v + first + 1, v + first, (middle - first) * sizeof(size_t));
    v[first] = x;
}

/* Iterative Crout base case, Alg. 4: sytrf.cpp:35-139. */
static Fact crout_base(const Mat* a) {
    const size_t n = a->r;
    Perm order = perm_identity(n);
    Mat lmat = mat_new(n, n);
    BDiag diag;
    bd_init(&diag);
    uint64_t* v = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    uint64_t* c = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    uint64_t* v2 = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    uint64_t* d2 = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    size_t r = 0, front = 0;
    while (front < n) { /* :74 */
        const size_t p1 = order.img[front];
        fold_diag(&lmat, &diag, p1, v);
        size_t j = n;
        for (size_t i = front; i < n; ++i) { /* :78-81 */
            c[i] = residual(a, &lmat, order.img[i], p1, r, v);
            if (j == n && c[i] != 0) j = i;
        }
        if (j == n) { ++front; continue; } /* :82-85 */
        if (j == front) { /* 1x1 pivot, :87-97 */
            const uint64_t x = c[front], xi = finv(x);
            Blk b = {BK_SCALAR, x, 0};
            bd_push(&diag, b);
            AT(lmat, p1, r) = 1 % P;
            for (size_t i = front + 1; i < n; ++i) AT(lmat, order.img[i], r) = fmul(xi, c[i]);
            rotate_one(order.img, r, front);
            ++r; ++front;
            continue;
        }
        /* 2x2 pivot pairing front with row j, :99-131 */
        const size_t p2 = order.img[j];
        const uint64_t x = c[j], xi = finv(x);
        fold_diag(&lmat, &diag, p2, v2);
        for (size_t i = front; i < n; ++i) d2[i] = residual(a, &lmat, order.img[i], p2, r, v2);
        const uint64_t y = d2[j];
        uint64_t y_eff = y;
        if (P != 2) {
            y_eff = fhalve(y);
            Blk b = {BK_ANTIDIAG, x, 0};
            bd_push(&diag, b);
            AT(lmat, p2, r) = fmul(xi, y_eff);
        } else {
            Blk b = {y == 0 ? BK_ANTIDIAG : BK_ANTITRI, x, y == 0 ? 0 : y};
            bd_push(&diag, b);
            AT(lmat, p2, r) = 0;
        }
        AT(lmat, p1, r) = 1 % P;
        AT(lmat, p1, r + 1) = 0;
        AT(lmat, p2, r + 1) = 1 % P;
        for (size_t i = front + 1; i < n; ++i) {
            if (i == j) continue;
            const uint64_t l2 = fmul(xi, c[i]);
            AT(lmat, order.img[i], r) = fmul(xi, fsub(d2[i], fmul(y_eff, l2)));
            AT(lmat, order.img[i], r + 1) = l2;
        }
        rotate_one(order.img, r, front);
        rotate_one(order.img, r + 1, j);
        r += 2; front += 2;
    }
    Fact f; /* gather, :134-138 */
    f.lower = mat_new(n, r);
    for (size_t pos = 0; pos < n; ++pos)
        for (size_t k = 0; k < r; ++k) AT(f.lower, pos, k) = AT(lmat, order.img[pos], k);
    f.perm = order;
    f.diag = diag;
    f.rank = r;
    free(v); free(c); free(v2); free(d2);
    mat_free(&lmat);
    return f;
}

/* res(i,j) = d_i^-1 m(i,j), sytrf.cpp:142-150. */
static Mat scale_rows_by_inverse(const uint64_t* d, const Mat* m) {
    Mat r = mat_new(m->r, m->c);
    for (size_t i = 0; i < m->r; ++i) {
        const uint64_t di = finv(d[i]);
        for (size_t j = 0; j < m->c; ++j) AT(r, i, j) = fmul(di, AT(*m, i, j));
    }
    return r;
}

/* Alg. 3, sytrf.cpp:170-265. */
static Fact zero_leading_pairs(const Mat* y, const Mat* z) {
    const size_t m = y->r, nz = z->r;
    Plduq py = plduq(y); /* :175 */
    const size_t r = py.rank;
    Mat l1 = mat_block(&py.lower, 0, r, 0, r);
    Mat m1 = mat_block(&py.lower, r, m, 0, r);
    Mat u1 = mat_block(&py.upper, 0, r, 0, r);
    Mat v1 = mat_block(&py.upper, 0, r, r, nz);
    const uint64_t* d = py.diag;

    Perm qinv = perm_inverse(&py.col_perm); /* :183-186 */
    Mat cp = conjugate_sym(&qinv, z);
    perm_free(&qinv);
    Mat c1 = mat_block(&cp, 0, r, 0, r);
    Mat c2 = mat_block(&cp, 0, r, r, nz);
    Mat c3 = mat_block(&cp, r, nz, r, nz);
    mat_free(&cp);

    uint64_t* delta = (uint64_t*)calloc(r + 1, sizeof(uint64_t));
    if (P == 2) { /* :188-200 */
        for (size_t i = 0; i < r; ++i) {
            uint64_t acc = AT(c1, i, i);
            for (size_t j = 0; j < i; ++j)
                acc = fsub(acc, fmul(fmul(delta[j], AT(u1, j, i)), AT(u1, j, i)));
            delta[i] = acc;
        }
        Mat u1t = mat_transposed(&u1);
        syrdk_sub_diag(&c1, &u1t, delta, r);
        mat_free(&u1t);
    }

    Mat x = trssyr2k(&u1, &c1); /* :202 */
    Mat g1s = scale_rows_by_inverse(d, &x);
    Mat g1 = mat_transposed(&g1s); /* :203 */
    mat_free(&g1s);
    if (P == 2) { /* :204-208 */
        for (size_t i = 0; i < r; ++i)
            for (size_t j = i; j < r; ++j) AT(x, i, j) = fadd(AT(x, i, j), fmul(delta[i], AT(u1, i, j)));
    }
    trmm_sub(&c2, &x, UPPER, 1, 0, &v1);   /* :210 */
    trsm_inplace(&u1, UPPER, 1, 1, &c2);   /* :211, c2 is now Y2 */
    syr2k_sub(&c3, &c2, &v1);              /* :213 */
    if (P == 2) {                          /* :214 */
        Mat v1t = mat_transposed(&v1);
        syrdk_sub_diag(&c3, &v1t, delta, r);
        mat_free(&v1t);
    }
    Mat g2s = scale_rows_by_inverse(d, &c2);
    Mat g2 = mat_transposed(&g2s); /* :215 */
    mat_free(&g2s);

    Fact f3 = dispatch(&c3); /* :217 */
    const size_t r3 = f3.rank;
    Mat g2h = permute_rows_inv(&f3.perm, &g2); /* :219-220 */
    Mat v1t = mat_transposed(&v1);
    Mat v1h = permute_rows_inv(&f3.perm, &v1t);
    mat_free(&v1t);

    const size_t total = m + nz, rank = 2 * r + r3; /* :222-252 */
    Fact f;
    f.lower = mat_new(total, rank);
    f.perm = perm_identity(total);
    size_t* image = f.perm.img;
    for (size_t i = 0; i < r; ++i) {
        image[2 * i] = py.row_perm.img[i];
        image[2 * i + 1] = m + py.col_perm.img[i];
        for (size_t j = 0; j < r; ++j) {
            AT(f.lower, 2 * i, 2 * j) = AT(l1, i, j);
            AT(f.lower, 2 * i + 1, 2 * j) = AT(g1, i, j);
            AT(f.lower, 2 * i + 1, 2 * j + 1) = AT(u1, j, i);
        }
    }
    for (size_t k = 0; k < nz - r; ++k) {
        const size_t row = k < r3 ? 2 * r + k : 2 * r + (m - r) + k;
        image[row] = m + py.col_perm.img[r + f3.perm.img[k]];
        for (size_t j = 0; j < r; ++j) {
            AT(f.lower, row, 2 * j) = AT(g2h, k, j);
            AT(f.lower, row, 2 * j + 1) = AT(v1h, k, j);
        }
        for (size_t t = 0; t < r3; ++t) AT(f.lower, row, 2 * r + t) = AT(f3.lower, k, t);
    }
    for (size_t t = 0; t < m - r; ++t) {
        image[2 * r + r3 + t] = py.row_perm.img[r + t];
        for (size_t j = 0; j < r; ++j) AT(f.lower, 2 * r + r3 + t, 2 * j) = AT(m1, t, j);
    }
    perm_check(&f.perm);
    bd_init(&f.diag); /* :254-261 */
    for (size_t i = 0; i < r; ++i) {
        Blk b;
        if (P == 2 && delta[i] != 0) { b.kind = BK_ANTITRI; b.a = d[i]; b.b = delta[i]; }
        else { b.kind = BK_ANTIDIAG; b.a = d[i]; b.b = 0; }
        bd_push(&f.diag, b);
    }
    bd_append(&f.diag, &f3.diag);
    f.rank = rank;

    free(delta);
    mat_free(&l1); mat_free(&m1); mat_free(&u1); mat_free(&v1);
    mat_free(&c1); mat_free(&c2); mat_free(&c3); mat_free(&x);
    mat_free(&g1); mat_free(&g2); mat_free(&g2h); mat_free(&v1h);
    fact_free(&f3);
    plduq_free(&py);
    return f;
}

/* Dispatcher for [[0,Y],[Y^t,Z]], sytrf.cpp:267-292. */
static Fact zero_leading(const Mat* y, const Mat* z) {
    const size_t m = y->r, nz = z->r;
    if (m == 0) return dispatch(z);
    if (nz == 0) {
        Fact f;
        f.perm = perm_identity(m);
        f.lower = mat_new(m, 0);
        bd_init(&f.diag);
        f.rank = 0;
        return f;
    }
    if (mat_is_zero(y)) { /* :274-290 */
        Fact f3 = dispatch(z);
        const size_t r3 = f3.rank;
        Fact f;
        f.perm = perm_identity(m + nz);
        for (size_t k = 0; k < r3; ++k) f.perm.img[k] = m + f3.perm.img[k];
        for (size_t t = 0; t < m; ++t) f.perm.img[r3 + t] = t;
        for (size_t k = r3; k < nz; ++k) f.perm.img[m + k] = m + f3.perm.img[k];
        perm_check(&f.perm);
        f.lower = mat_new(m + nz, r3);
        Mat top = mat_block(&f3.lower, 0, r3, 0, r3);
        Mat bot = mat_block(&f3.lower, r3, nz, 0, r3);
        mat_set_block(&f.lower, 0, 0, &top);
        mat_set_block(&f.lower, r3 + m, 0, &bot);
        mat_free(&top); mat_free(&bot);
        f.diag = bd_copy(&f3.diag);
        f.rank = r3;
        fact_free(&f3);
        return f;
    }
    return zero_leading_pairs(y, z);
}

/* Alg. 2 halving step, sytrf.cpp:298-335. */
static Fact recursive_step(const Mat* a) {
    const size_t n = a->r, m = n / 2;
    Mat a1 = mat_block(a, 0, m, 0, m);
    Fact f1 = dispatch(&a1); /* :303 */
    mat_free(&a1);
    const size_t r1 = f1.rank;
    Mat l1 = mat_block(&f1.lower, 0, r1, 0, r1);
    Mat m1 = mat_block(&f1.lower, r1, m, 0, r1);

    Mat b = mat_block(a, 0, m, m, n);
    Mat bp = permute_rows_inv(&f1.perm, &b); /* :308 */
    mat_free(&b);
    Mat x = mat_block(&bp, 0, r1, 0, n - m);
    trsm_inplace(&l1, LOWER, 0, 1, &x);      /* :310 */
    Mat y = mat_block(&bp, r1, m, 0, n - m);
    mat_free(&bp);
    gemm_sub(&y, &m1, &x);                   /* :312 */
    Mat dix = bd_inverse_apply(&f1.diag, &x);
    Mat g = mat_transposed(&dix);            /* :313 */
    mat_free(&dix);
    Mat z = mat_block(a, m, n, m, n);
    syrdk_sub_bd(&z, &g, &f1.diag);          /* :315 */

    Fact f2 = zero_leading(&y, &z);          /* :317 */

    Mat below = mat_new(n - r1, r1);         /* :319-322 */
    mat_set_block(&below, 0, 0, &m1);
    mat_set_block(&below, m - r1, 0, &g);
    Mat n1 = permute_rows_inv(&f2.perm, &below);
    mat_free(&below);

    const size_t rank = r1 + f2.rank;        /* :324-334 */
    Fact f;
    f.lower = mat_new(n, rank);
    mat_set_block(&f.lower, 0, 0, &l1);
    mat_set_block(&f.lower, r1, 0, &n1);
    mat_set_block(&f.lower, r1, r1, &f2.lower);
    f.diag = bd_copy(&f1.diag);
    bd_append(&f.diag, &f2.diag);
    Perm e1 = perm_embed(&f1.perm, 0, n), e2 = perm_embed(&f2.perm, r1, n);
    f.perm = perm_compose(&e1, &e2);
    f.rank = rank;
    perm_free(&e1); perm_free(&e2);
    mat_free(&l1); mat_free(&m1); mat_free(&x); mat_free(&y); mat_free(&g); mat_free(&z); mat_free(&n1);
    fact_free(&f1); fact_free(&f2);
    return f;
}

/* sytrf.cpp:337-350. */
static Fact dispatch(const Mat* a) {
    switch (CFG_VARIANT) {
    case ORC_VARIANT_CROUT:
        return crout_base(a);
    case ORC_VARIANT_RECURSIVE:
        if (a->r <= 1) return crout_base(a);
        return recursive_step(a);
    default:
        if (a->r <= CFG_T || a->r <= 1) return crout_base(a);
        return recursive_step(a);
    }
}

/* ------------------------------------------------------------------ */
/* C entry points (oracle_api.h layout)                                */
/* ------------------------------------------------------------------ */

static Mat load(size_t r, size_t c, const uint64_t* v) {
    Mat m = mat_new(r, c);
    for (size_t i = 0; i < r * c; ++i) m.v[i] = v[i] % P;
    return m;
}
static void store(const Mat* m, uint64_t* out) { memcpy(out, m->v, m->r * m->c * sizeof(uint64_t)); }

static void export_fact(const Fact* f, int64_t* perm, uint64_t* lower, int32_t* dkind,
                        uint64_t* dval, uint64_t* dval2, size_t* rank) {
    for (size_t i = 0; i < f->perm.n; ++i) perm[i] = (int64_t)f->perm.img[i];
    store(&f->lower, lower);
    for (size_t k = 0; k < f->diag.nb; ++k) {
        const size_t t = f->diag.off[k];
        const Blk b = f->diag.blk[k];
        if (b.kind == BK_SCALAR) {
            dkind[t] = ORC_D_SCALAR; dval[t] = b.a; dval2[t] = 0;
        } else if (b.kind == BK_ANTIDIAG) {
            dkind[t] = ORC_D_ANTIDIAG_HEAD; dkind[t + 1] = ORC_D_ANTIDIAG_TAIL;
            dval[t] = dval[t + 1] = b.a; dval2[t] = dval2[t + 1] = 0;
        } else {
            dkind[t] = ORC_D_ANTITRI_HEAD; dkind[t + 1] = ORC_D_ANTITRI_TAIL;
            dval[t] = dval[t + 1] = b.a; dval2[t] = dval2[t + 1] = b.b;
        }
    }
    *rank = f->rank;
}

static void set_cfg(int variant, size_t threshold) {
    CFG_VARIANT = variant;
    CFG_T = threshold;
}

/* ldlt, sytrf.cpp:354-358. */
int orc_ldlt(uint64_t p, size_t rows, size_t cols, const uint64_t* a, int variant,
             size_t threshold, int64_t* perm, uint64_t* lower, int32_t* dkind, uint64_t* dval,
             uint64_t* dval2, size_t* rank) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    set_cfg(variant, threshold);
    if (rows != cols) fail(ORC_DIMENSION_MISMATCH);
    Mat am = load(rows, cols, a);
    if (!mat_is_symmetric(&am)) { mat_free(&am); fail(ORC_NOT_SYMMETRIC); }
    Fact f = dispatch(&am);
    export_fact(&f, perm, lower, dkind, dval, dval2, rank);
    fact_free(&f);
    mat_free(&am);
    return ORC_OK;
}

/* ldlt_zero_leading, sytrf.cpp:360-368. */
int orc_ldlt_zero_leading(uint64_t p, size_t m, size_t ny, const uint64_t* y, size_t nz,
                          const uint64_t* z, int variant, size_t threshold, int64_t* perm,
                          uint64_t* lower, int32_t* dkind, uint64_t* dval, uint64_t* dval2,
                          size_t* rank) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    set_cfg(variant, threshold);
    if (ny != nz) fail(ORC_DIMENSION_MISMATCH);
    Mat ym = load(m, ny, y), zm = load(nz, nz, z);
    if (!mat_is_symmetric(&zm)) fail(ORC_NOT_SYMMETRIC);
    Fact f = zero_leading(&ym, &zm);
    export_fact(&f, perm, lower, dkind, dval, dval2, rank);
    fact_free(&f);
    mat_free(&ym);
    mat_free(&zm);
    return ORC_OK;
}

int orc_plduq(uint64_t p, size_t m, size_t n, const uint64_t* b, int64_t* row_image,
              int64_t* col_image, uint64_t* lower, uint64_t* diag, uint64_t* upper, size_t* rank) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    Mat bm = load(m, n, b);
    Plduq f = plduq(&bm);
    for (size_t i = 0; i < m; ++i) row_image[i] = (int64_t)f.row_perm.img[i];
    for (size_t j = 0; j < n; ++j) col_image[j] = (int64_t)f.col_perm.img[j];
    store(&f.lower, lower);
    memcpy(diag, f.diag, f.rank * sizeof(uint64_t));
    store(&f.upper, upper);
    *rank = f.rank;
    plduq_free(&f);
    mat_free(&bm);
    return ORC_OK;
}

int orc_trssyr2k(uint64_t p, size_t n, const uint64_t* u, const uint64_t* c, uint64_t* x) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    Mat um = load(n, n, u), cm = load(n, n, c);
    Mat xm = trssyr2k(&um, &cm);
    store(&xm, x);
    mat_free(&um); mat_free(&cm); mat_free(&xm);
    return ORC_OK;
}

int orc_gemm_sub(uint64_t p, size_t m, size_t n, size_t k, uint64_t* c, const uint64_t* a,
                 const uint64_t* b) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    Mat cm = load(m, n, c), am = load(m, k, a), bm = load(k, n, b);
    gemm_sub(&cm, &am, &bm);
    store(&cm, c);
    mat_free(&cm); mat_free(&am); mat_free(&bm);
    return ORC_OK;
}

int orc_trsm_inplace(uint64_t p, size_t n, size_t ncols, const uint64_t* t, int upper, int trans,
                     int unit, uint64_t* b) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    Mat tm = load(n, n, t), bm = load(n, ncols, b);
    trsm_inplace(&tm, upper ? UPPER : LOWER, trans, unit, &bm);
    store(&bm, b);
    mat_free(&tm); mat_free(&bm);
    return ORC_OK;
}

int orc_trmm_sub(uint64_t p, size_t n, size_t ncols, uint64_t* c, const uint64_t* t, int upper,
                 int trans, int unit, const uint64_t* b) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    Mat cm = load(n, ncols, c), tm = load(n, n, t), bm = load(n, ncols, b);
    trmm_sub(&cm, &tm, upper ? UPPER : LOWER, trans, unit, &bm);
    store(&cm, c);
    mat_free(&cm); mat_free(&tm); mat_free(&bm);
    return ORC_OK;
}

int orc_syrdk_sub(uint64_t p, size_t n, size_t k, uint64_t* c, const uint64_t* g,
                  const int32_t* dkind, const uint64_t* dval, const uint64_t* dval2) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    BDiag d;
    bd_init(&d);
    for (size_t t = 0; t < k;) {
        Blk b;
        if (dkind[t] == ORC_D_SCALAR) { b.kind = BK_SCALAR; b.a = dval[t] % p; b.b = 0; t += 1; }
        else if (dkind[t] == ORC_D_ANTIDIAG_HEAD) { b.kind = BK_ANTIDIAG; b.a = dval[t] % p; b.b = 0; t += 2; }
        else { b.kind = BK_ANTITRI; b.a = dval[t] % p; b.b = dval2[t] % p; t += 2; }
        bd_push(&d, b);
    }
    Mat cm = load(n, n, c), gm = load(n, k, g);
    syrdk_sub_bd(&cm, &gm, &d);
    store(&cm, c);
    mat_free(&cm); mat_free(&gm); bd_free(&d);
    return ORC_OK;
}

int orc_syr2k_sub(uint64_t p, size_t n, size_t k, uint64_t* c, const uint64_t* a,
                  const uint64_t* b) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    Mat cm = load(n, n, c), am = load(k, n, a), bm = load(k, n, b);
    syr2k_sub(&cm, &am, &bm);
    store(&cm, c);
    mat_free(&cm); mat_free(&am); mat_free(&bm);
    return ORC_OK;
}

/* syrdk_sub(c, g, span d), kernels.cpp:108-119: C <- C - G diag(d) G^T. */
int orc_syrdk_sub_diag(uint64_t p, size_t n, size_t k, uint64_t* c, const uint64_t* g,
                       const uint64_t* d) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    uint64_t* dv = (uint64_t*)malloc((k ? k : 1) * sizeof(uint64_t));
    for (size_t t = 0; t < k; ++t) dv[t] = d[t] % p;
    Mat cm = load(n, n, c), gm = load(n, k, g);
    syrdk_sub_diag(&cm, &gm, dv, k);
    store(&cm, c);
    mat_free(&cm); mat_free(&gm); free(dv);
    return ORC_OK;
}

/* strictify, rpmtools.cpp:74-132: every AntiTri block [0 c; c d] at columns (t, t+1)
 * becomes Scalar d, Scalar -c^2/d; L's columns t, t+1 and P change as the reference's
 * three steps (normalize, swap, eliminate), run block by block in order.  The flat
 * factorization (perm[n], lower n x r, dkind/dval/dval2[r]) is updated in place;
 * stats[0] = blocks converted, stats[1] = entries touched (StrictifyStats). */
int orc_strictify(uint64_t p, size_t n, size_t r, int64_t* perm, uint64_t* lower, int32_t* dkind,
                  uint64_t* dval, uint64_t* dval2, uint64_t* stats) {
    int code = setjmp(ERR_JMP);
    if (code) return code;
    set_field(p);
    uint64_t blocks = 0, touched = 0;
#define LL(i, j) lower[(size_t)(i) * r + (size_t)(j)]
    for (size_t t = 0; t < r;) {
        if (dkind[t] != ORC_D_ANTITRI_HEAD) {
            t += dkind[t] == ORC_D_SCALAR ? 1 : 2;
            continue;
        }
        if (p != 2) fail(ORC_WRONG_CHARACTERISTIC); /* rpmtools.cpp:87-88 */
        const uint64_t c = dval[t] % p, dd = dval2[t] % p;
        const uint64_t x = LL(t + 1, t) % p;
        if (x != 0) /* :95-100 col t -= x col t+1 */
            for (size_t i = t + 1; i < n; ++i) {
                LL(i, t) = fsub(LL(i, t) % p, fmul(x, LL(i, t + 1) % p));
                ++touched;
            }
        for (size_t j = 0; j < t; ++j) { /* :106-109 swap prefix of rows t, t+1 */
            uint64_t s = LL(t, j); LL(t, j) = LL(t + 1, j); LL(t + 1, j) = s;
            touched += 2;
        }
        for (size_t i = t + 2; i < n; ++i) { /* :110-113 swap the column pair below */
            uint64_t s = LL(i, t); LL(i, t) = LL(i, t + 1); LL(i, t + 1) = s;
            touched += 2;
        }
        { int64_t s = perm[t]; perm[t] = perm[t + 1]; perm[t + 1] = s; } /* :114 compose */
        const uint64_t cd = fmul(c, finv(dd)); /* :118-123 col t += (c/d) col t+1 */
        for (size_t i = t + 1; i < n; ++i) {
            LL(i, t) = fadd(LL(i, t) % p, fmul(cd, LL(i, t + 1) % p));
            ++touched;
        }
        dkind[t] = dkind[t + 1] = ORC_D_SCALAR;
        dval[t] = dd;
        dval[t + 1] = fneg(fmul(fmul(c, c), finv(dd)));
        dval2[t] = dval2[t + 1] = 0;
        ++blocks;
        t += 2;
    }
#undef LL
    stats[0] = blocks;
    stats[1] = touched;
    return ORC_OK;
}
