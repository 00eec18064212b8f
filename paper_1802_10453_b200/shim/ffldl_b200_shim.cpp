// ffldl_b200_shim.cpp -- C++ drop-in for the reference's hot path.
//
// Compile this file INSTEAD OF proj/src/{sytrf,plduq,trssyr2k,kernels}.cpp,
// against the reference's own headers (proj/include/ffldl/*.hpp), and link
// libffldl_b200.so.  Every definition keeps the reference's signature and
// error behaviour; the arithmetic runs on the B200 through the C-ABI of
// include/ffldl_b200.h.  Documented deviation: the GPU path does not update
// PrimeField::mul_count (field.hpp:101-104).
//
// Replaced definitions (declaration -> reference implementation):
//   ldlt                 sytrf.hpp:30      -> sytrf.cpp:354-358
//   ldlt_zero_leading    sytrf.hpp:41      -> sytrf.cpp:360-368
//   plduq                plduq.hpp:42      -> plduq.cpp:36-123 (+ reconstruct/rank_profile)
//   trssyr2k[_inplace]   trssyr2k.hpp:17,20 -> trssyr2k.cpp:55-77
//   gemm_sub, trmm_sub, trsm_inplace, syrdk_sub x2, syr2k_sub  kernels.hpp:13-32
//   strictify            rpmtools.hpp:39   -> rpmtools.cpp:74-132 (with the rest of
//                        rpmtools.cpp: pivoting_matrix, rank_profile_bruteforce,
//                        verify_revealing -- compile this file instead of rpmtools.cpp too)
#include <cstdlib>
#include <mutex>
#include <variant>
#include <vector>

#include "ffb_dropin_includes.hpp"
#include "ffldl_b200.h"

namespace ffldl {

namespace {

ffb_context* ctx() {
    static ffb_context* c = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* d = std::getenv("FFLDL_B200_DEVICE");
        if (ffb_create(&c, d ? std::atoi(d) : 0) != FFB_OK)
            throw Error(std::string("ffldl_b200: cannot create a CUDA context: ") + ffb_last_error());
    });
    return c;
}

[[noreturn]] void raise(int s) {
    const std::string msg = ffb_last_error();
    switch (s) {
    case FFB_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case FFB_NOT_SYMMETRIC: throw NotSymmetric(msg);
    case FFB_NOT_PRIME: throw NotPrime(msg);
    case FFB_ZERO_INVERSE: throw ZeroInverse(msg);
    case FFB_CHAR_TWO_DIVISION: throw CharTwoDivision(msg);
    case FFB_NON_UNIT_TRIANGULAR: throw NonUnitTriangular(msg);
    case FFB_SINGULAR_TRIANGULAR: throw SingularTriangular(msg);
    case FFB_CHAR_TWO_NONZERO_DIAGONAL: throw CharTwoNonzeroDiagonal(msg);
    case FFB_BAD_BLOCK_SIZES: throw BadBlockSizes(msg);
    case FFB_WRONG_CHARACTERISTIC: throw WrongCharacteristic(msg);
    case FFB_PARSE_ERROR: throw ParseError(msg);
    default: throw Error("ffldl_b200: " + msg);
    }
}
void check(int s) {
    if (s != FFB_OK) raise(s);
}

std::vector<uint64_t> flat(const Matrix& m) {
    std::vector<uint64_t> v(m.rows() * m.cols());
    for (std::size_t i = 0; i < m.rows(); ++i)
        for (std::size_t j = 0; j < m.cols(); ++j) v[i * m.cols() + j] = m(i, j).value;
    return v;
}
Matrix unflat(const PrimeField& f, std::size_t rows, std::size_t cols, const uint64_t* v) {
    Matrix m(f, rows, cols);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < cols; ++j) m(i, j) = f.element(v[i * cols + j]);
    return m;
}
int variant_code(Variant v) {
    return v == Variant::Recursive ? FFB_VARIANT_RECURSIVE
           : v == Variant::Crout   ? FFB_VARIANT_CROUT
                                   : FFB_VARIANT_CASCADE;
}

Factorization make_fact(const PrimeField& f, std::size_t n, const std::vector<int64_t>& perm,
                        const std::vector<uint64_t>& lower, const std::vector<int32_t>& dk,
                        const std::vector<uint64_t>& dv, const std::vector<uint64_t>& dv2,
                        std::size_t r) {
    std::vector<std::size_t> image(perm.begin(), perm.begin() + n);
    BlockDiag d;
    for (std::size_t t = 0; t < r;) {
        if (dk[t] == FFB_D_SCALAR) {
            d.push(ScalarBlock{f.element(dv[t])});
            t += 1;
        } else if (dk[t] == FFB_D_ANTIDIAG_HEAD) {
            d.push(AntiDiagBlock{f.element(dv[t])});
            t += 2;
        } else {
            d.push(AntiTriBlock{f.element(dv[t]), f.element(dv2[t])});
            t += 2;
        }
    }
    return Factorization{Permutation::from_image(std::move(image)), unflat(f, n, r, lower.data()),
                         std::move(d), r};
}

}  // namespace

Factorization ldlt(const Matrix& a, const SytrfConfig& config) {
    const PrimeField& f = a.field();
    const std::size_t n = a.rows();
    if (a.rows() != a.cols()) throw DimensionMismatch("ldlt: matrix must be square");
    std::vector<uint64_t> av = flat(a), lower(std::max<std::size_t>(n * n, 1)), dv(n + 1), dv2(n + 1);
    std::vector<int64_t> perm(n + 1);
    std::vector<int32_t> dk(n + 1);
    std::size_t r = 0;
    check(ffb_ldlt(ctx(), f.modulus(), a.rows(), a.cols(), av.data(), variant_code(config.variant),
                   config.base_case_threshold, perm.data(), lower.data(), dk.data(), dv.data(),
                   dv2.data(), &r));
    return make_fact(f, n, perm, lower, dk, dv, dv2, r);
}

Factorization ldlt_zero_leading(const Matrix& y, const Matrix& z, const SytrfConfig& config) {
    if (z.rows() != z.cols()) throw DimensionMismatch("ldlt_zero_leading: Z must be square");
    if (y.cols() != z.rows())
        throw DimensionMismatch("ldlt_zero_leading: Y and Z have mismatched widths");
    if (y.field().modulus() != z.field().modulus())
        throw DimensionMismatch("ldlt_zero_leading: operands over different fields");
    const PrimeField& f = z.field();
    const std::size_t n = y.rows() + z.rows();
    std::vector<uint64_t> yv = flat(y), zv = flat(z), lower(std::max<std::size_t>(n * n, 1)),
                          dv(n + 1), dv2(n + 1);
    std::vector<int64_t> perm(n + 1);
    std::vector<int32_t> dk(n + 1);
    std::size_t r = 0;
    check(ffb_ldlt_zero_leading(ctx(), f.modulus(), y.rows(), y.cols(), yv.data(), z.rows(),
                                zv.data(), variant_code(config.variant), config.base_case_threshold,
                                perm.data(), lower.data(), dk.data(), dv.data(), dv2.data(), &r));
    return make_fact(f, n, perm, lower, dk, dv, dv2, r);
}

Matrix PlduqFactorization::reconstruct() const {  // plduq.cpp:7-18 semantics
    const PrimeField& f = lower.field();
    const std::size_t m = lower.rows(), n = upper.cols();
    Matrix k(f, m, n);
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j) {
            FieldElement acc = f.zero();
            for (std::size_t t = 0; t < rank; ++t)
                acc = f.add(acc, f.mul(f.mul(lower(i, t), diag[t]), upper(t, j)));
            k(i, j) = acc;
        }
    return permute_rows(row_perm, permute_cols(col_perm, k));
}

Matrix PlduqFactorization::rank_profile() const {
    const PrimeField& f = lower.field();
    Matrix r(f, lower.rows(), upper.cols());
    for (std::size_t k = 0; k < rank; ++k) r(row_perm.image(k), col_perm.image(k)) = f.one();
    return r;
}

PlduqFactorization plduq(const Matrix& b) {
    const PrimeField& f = b.field();
    const std::size_t m = b.rows(), n = b.cols(), mn = std::min(m, n);
    std::vector<uint64_t> bv = flat(b), lo(std::max<std::size_t>(m * mn, 1)), dg(mn + 1),
                          up(std::max<std::size_t>(mn * n, 1));
    std::vector<int64_t> ri(m + 1), ci(n + 1);
    std::size_t r = 0;
    check(ffb_plduq(ctx(), f.modulus(), m, n, bv.data(), ri.data(), ci.data(), lo.data(), dg.data(),
                    up.data(), &r));
    std::vector<FieldElement> d(r);
    for (std::size_t k = 0; k < r; ++k) d[k] = f.element(dg[k]);
    return PlduqFactorization{Permutation::from_image(std::vector<std::size_t>(ri.begin(), ri.begin() + m)),
                              Permutation::from_image(std::vector<std::size_t>(ci.begin(), ci.begin() + n)),
                              unflat(f, m, r, lo.data()), std::move(d), unflat(f, r, n, up.data()), r};
}

void trssyr2k_inplace(const Matrix& u, Matrix& c) {
    if (u.rows() != u.cols() || c.rows() != c.cols() || u.rows() != c.rows())
        throw DimensionMismatch("trssyr2k: operands must be square of equal order");
    if (u.field().modulus() != c.field().modulus())
        throw DimensionMismatch("trssyr2k: operands over different fields");
    const std::size_t n = u.rows();
    std::vector<uint64_t> uv = flat(u), cv = flat(c), xv(std::max<std::size_t>(n * n, 1));
    check(ffb_trssyr2k(ctx(), c.field().modulus(), n, uv.data(), cv.data(), xv.data()));
    c = unflat(c.field(), n, n, xv.data());
}

Matrix trssyr2k(const Matrix& u, const Matrix& c) {
    Matrix x = c;
    trssyr2k_inplace(u, x);
    return x;
}

void gemm_sub(Matrix& c, const Matrix& a, const Matrix& b) {
    if (a.rows() != c.rows() || b.cols() != c.cols() || a.cols() != b.rows())
        throw DimensionMismatch("gemm_sub: incompatible shapes");
    std::vector<uint64_t> cv = flat(c), av = flat(a), bv = flat(b);
    check(ffb_gemm_sub(ctx(), c.field().modulus(), c.rows(), c.cols(), a.cols(), cv.data(), av.data(),
                       bv.data()));
    c = unflat(c.field(), c.rows(), c.cols(), cv.data());
}

void trmm_sub(Matrix& c, const Matrix& t, Uplo uplo, bool trans, bool unit, const Matrix& b) {
    if (t.rows() != t.cols() || t.cols() != b.rows() || c.rows() != b.rows() || c.cols() != b.cols())
        throw DimensionMismatch("trmm_sub: incompatible shapes");
    std::vector<uint64_t> cv = flat(c), tv = flat(t), bv = flat(b);
    check(ffb_trmm_sub(ctx(), c.field().modulus(), t.rows(), c.cols(), cv.data(), tv.data(),
                       uplo == Uplo::Upper, trans, unit, bv.data()));
    c = unflat(c.field(), c.rows(), c.cols(), cv.data());
}

void trsm_inplace(const Matrix& t, Uplo uplo, bool trans, bool unit, Matrix& b) {
    if (t.rows() != t.cols() || t.cols() != b.rows())
        throw DimensionMismatch("trsm_inplace: incompatible shapes");
    std::vector<uint64_t> tv = flat(t), bv = flat(b);
    check(ffb_trsm_inplace(ctx(), b.field().modulus(), t.rows(), b.cols(), tv.data(),
                           uplo == Uplo::Upper, trans, unit, bv.data()));
    b = unflat(b.field(), b.rows(), b.cols(), bv.data());
}

void syrdk_sub(Matrix& c, const Matrix& g, const BlockDiag& d) {
    if (c.rows() != c.cols() || g.rows() != c.rows() || g.cols() != d.order())
        throw DimensionMismatch("syrdk_sub: incompatible shapes");
    const std::size_t k = d.order();
    std::vector<int32_t> kind(k + 1);
    std::vector<uint64_t> val(k + 1), val2(k + 1);
    for (std::size_t b = 0; b < d.block_count(); ++b) {
        const std::size_t t = d.offset(b);
        if (const auto* s = std::get_if<ScalarBlock>(&d.block(b))) {
            kind[t] = FFB_D_SCALAR;
            val[t] = s->d.value;
        } else if (const auto* a = std::get_if<AntiDiagBlock>(&d.block(b))) {
            kind[t] = FFB_D_ANTIDIAG_HEAD;
            kind[t + 1] = FFB_D_ANTIDIAG_TAIL;
            val[t] = val[t + 1] = a->x.value;
        } else {
            const auto& at = std::get<AntiTriBlock>(d.block(b));
            kind[t] = FFB_D_ANTITRI_HEAD;
            kind[t + 1] = FFB_D_ANTITRI_TAIL;
            val[t] = val[t + 1] = at.c.value;
            val2[t] = val2[t + 1] = at.d.value;
        }
    }
    std::vector<uint64_t> cv = flat(c), gv = flat(g);
    check(ffb_syrdk_sub(ctx(), c.field().modulus(), c.rows(), k, cv.data(), gv.data(), kind.data(),
                        val.data(), val2.data()));
    c = unflat(c.field(), c.rows(), c.cols(), cv.data());
}

void syrdk_sub(Matrix& c, const Matrix& g, std::span<const FieldElement> d) {
    if (c.rows() != c.cols() || g.rows() != c.rows() || g.cols() != d.size())
        throw DimensionMismatch("syrdk_sub: incompatible shapes");
    std::vector<uint64_t> cv = flat(c), gv = flat(g), dv(d.size() + 1);
    for (std::size_t k = 0; k < d.size(); ++k) dv[k] = d[k].value;
    check(ffb_syrdk_sub_diag(ctx(), c.field().modulus(), c.rows(), d.size(), cv.data(), gv.data(), dv.data()));
    c = unflat(c.field(), c.rows(), c.cols(), cv.data());
}

void syr2k_sub(Matrix& c, const Matrix& a, const Matrix& b) {
    if (c.rows() != c.cols() || a.cols() != c.rows() || b.cols() != c.rows() || a.rows() != b.rows())
        throw DimensionMismatch("syr2k_sub: incompatible shapes");
    std::vector<uint64_t> cv = flat(c), av = flat(a), bv = flat(b);
    check(ffb_syr2k_sub(ctx(), c.field().modulus(), c.rows(), a.rows(), cv.data(), av.data(), bv.data()));
    c = unflat(c.field(), c.rows(), c.cols(), cv.data());
}

// ---- rpmtools.hpp (replaces rpmtools.cpp) ------------------------------------------

// strictify, rpmtools.cpp:74-132: on the device (ffb_strictify), the factorization is
// rewritten in place like the reference's.
void strictify(Factorization& f, StrictifyStats* stats) {
    const PrimeField& field = f.lower.field();
    const std::size_t n = f.dimension(), r = f.rank;
    std::vector<int64_t> perm(n + 1);
    for (std::size_t i = 0; i < n; ++i) perm[i] = (int64_t)f.perm.image(i);
    std::vector<uint64_t> lower = flat(f.lower);
    lower.resize(n * r + 1);
    std::vector<int32_t> kind(r + 1);
    std::vector<uint64_t> val(r + 1), val2(r + 1);
    for (std::size_t b = 0; b < f.diag.block_count(); ++b) {
        const std::size_t t = f.diag.offset(b);
        if (const auto* s = std::get_if<ScalarBlock>(&f.diag.block(b))) {
            kind[t] = FFB_D_SCALAR;
            val[t] = s->d.value;
        } else if (const auto* a = std::get_if<AntiDiagBlock>(&f.diag.block(b))) {
            kind[t] = FFB_D_ANTIDIAG_HEAD;
            kind[t + 1] = FFB_D_ANTIDIAG_TAIL;
            val[t] = val[t + 1] = a->x.value;
        } else {
            const auto& at = std::get<AntiTriBlock>(f.diag.block(b));
            kind[t] = FFB_D_ANTITRI_HEAD;
            kind[t + 1] = FFB_D_ANTITRI_TAIL;
            val[t] = val[t + 1] = at.c.value;
            val2[t] = val2[t + 1] = at.d.value;
        }
    }
    uint64_t blocks = 0, touched = 0;
    check(ffb_strictify(ctx(), field.modulus(), n, r, perm.data(), lower.data(), kind.data(), val.data(),
                        val2.data(), &blocks, &touched));
    f = make_fact(field, n, perm, lower, kind, val, val2, r);
    if (stats != nullptr) {
        stats->blocks_converted = blocks;
        stats->entries_touched = touched;
    }
}

Matrix pivoting_matrix(const Factorization& f) {  // rpmtools.cpp:61-68
    const PrimeField& field = f.lower.field();
    const std::size_t n = f.dimension();
    Matrix pi(field, n, n);
    for (const auto& [a, b] : f.diag.support()) pi(f.perm.image(a), f.perm.image(b)) = field.one();
    return pi;
}

// The brute-force checker of rpmtools.cpp:43-59 (verification only, host): the column rank
// profile of the first i rows grows by the leading column of row i reduced against the
// reduced basis of the earlier rows, and R(i, that column) = 1 -- the same matrix as the
// reference's inclusion-exclusion over leading ranks.
Matrix rank_profile_bruteforce(const Matrix& a) {
    const PrimeField& f = a.field();
    const std::size_t m = a.rows(), n = a.cols();
    Matrix r(f, m, n);
    std::vector<std::vector<FieldElement>> basis;
    std::vector<std::size_t> piv;
    for (std::size_t i = 0; i < m; ++i) {
        std::vector<FieldElement> row(n);
        for (std::size_t j = 0; j < n; ++j) row[j] = a(i, j);
        for (std::size_t b = 0; b < basis.size(); ++b) {
            const FieldElement c = row[piv[b]];
            if (f.is_zero(c)) continue;
            for (std::size_t j = 0; j < n; ++j) row[j] = f.sub(row[j], f.mul(c, basis[b][j]));
        }
        std::size_t c = 0;
        while (c < n && f.is_zero(row[c])) ++c;
        if (c == n) continue;
        const FieldElement s = f.inv(row[c]);
        for (auto& x : row) x = f.mul(x, s);
        for (std::size_t b = 0; b < basis.size(); ++b) {
            const FieldElement t = basis[b][c];
            if (f.is_zero(t)) continue;
            for (std::size_t j = 0; j < n; ++j) basis[b][j] = f.sub(basis[b][j], f.mul(t, row[j]));
        }
        basis.push_back(row);
        piv.push_back(c);
        r(i, c) = f.one();
    }
    return r;
}

bool verify_revealing(const Factorization& f, const Matrix& a) {  // rpmtools.cpp:70-72
    return f.reconstruct() == a && pivoting_matrix(f) == rank_profile_bruteforce(a);
}

}  // namespace ffldl
