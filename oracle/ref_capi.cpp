// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/oracle_api.h).
//
// A thin extern "C" driver around the UNMODIFIED reference library.  It is
// compiled together with /root/reference/proj/src/{sytrf,kernels,plduq,
// trssyr2k,rpmtools}.cpp by oracle/Makefile into oracle/_ref/libffldl_ref.so
// so that Python tests can call the reference's own ldlt / plduq / trssyr2k /
// kernels on the same inputs as the GPU path.  Nothing here re-implements the
// algorithm; it only converts flat arrays to ffldl::Matrix and back, and maps
// the reference's exceptions (proj/include/ffldl/errors.hpp) to status codes.

#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <span>
#include <variant>
#include <vector>

#include "ffldl/errors.hpp"
#include "ffldl/io.hpp"
#include "ffldl/kernels.hpp"
#include "ffldl/plduq.hpp"
#include "ffldl/rpmtools.hpp"
#include "ffldl/sytrf.hpp"
#include "ffldl/trssyr2k.hpp"

extern "C" {
#include "oracle_api.h"
}

using namespace ffldl;

namespace {

Matrix to_matrix(const PrimeField& f, size_t rows, size_t cols, const uint64_t* v) {
    Matrix m(f, rows, cols);
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) m(i, j) = f.element(v[i * cols + j]);
    return m;
}

void from_matrix(const Matrix& m, uint64_t* out) {
    for (size_t i = 0; i < m.rows(); ++i)
        for (size_t j = 0; j < m.cols(); ++j) out[i * m.cols() + j] = m(i, j).value;
}

SytrfConfig make_cfg(int variant, size_t threshold) {
    SytrfConfig c;
    c.variant = variant == ORC_VARIANT_RECURSIVE ? Variant::Recursive
                : variant == ORC_VARIANT_CROUT   ? Variant::Crout
                                                 : Variant::Cascade;
    c.base_case_threshold = threshold;
    return c;
}

void export_fact(const Factorization& f, int64_t* perm, uint64_t* lower, int32_t* dkind,
                 uint64_t* dval, uint64_t* dval2, size_t* rank) {
    const size_t n = f.dimension();
    for (size_t i = 0; i < n; ++i) perm[i] = static_cast<int64_t>(f.perm.image(i));
    from_matrix(f.lower, lower);
    for (size_t k = 0; k < f.diag.block_count(); ++k) {
        const size_t t = f.diag.offset(k);
        const DiagBlock& b = f.diag.block(k);
        if (const auto* s = std::get_if<ScalarBlock>(&b)) {
            dkind[t] = ORC_D_SCALAR;
            dval[t] = s->d.value;
            dval2[t] = 0;
        } else if (const auto* a = std::get_if<AntiDiagBlock>(&b)) {
            dkind[t] = ORC_D_ANTIDIAG_HEAD;
            dkind[t + 1] = ORC_D_ANTIDIAG_TAIL;
            dval[t] = dval[t + 1] = a->x.value;
            dval2[t] = dval2[t + 1] = 0;
        } else {
            const auto& at = std::get<AntiTriBlock>(b);
            dkind[t] = ORC_D_ANTITRI_HEAD;
            dkind[t + 1] = ORC_D_ANTITRI_TAIL;
            dval[t] = dval[t + 1] = at.c.value;
            dval2[t] = dval2[t + 1] = at.d.value;
        }
    }
    *rank = f.rank;
}

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return ORC_OK;
    } catch (const DimensionMismatch&) {
        return ORC_DIMENSION_MISMATCH;
    } catch (const NotSymmetric&) {
        return ORC_NOT_SYMMETRIC;
    } catch (const NotPrime&) {
        return ORC_NOT_PRIME;
    } catch (const ZeroInverse&) {
        return ORC_ZERO_INVERSE;
    } catch (const CharTwoDivision&) {
        return ORC_CHAR_TWO_DIVISION;
    } catch (const NonUnitTriangular&) {
        return ORC_NON_UNIT_TRIANGULAR;
    } catch (const SingularTriangular&) {
        return ORC_SINGULAR_TRIANGULAR;
    } catch (const CharTwoNonzeroDiagonal&) {
        return ORC_CHAR_TWO_NONZERO_DIAGONAL;
    } catch (const BadBlockSizes&) {
        return ORC_BAD_BLOCK_SIZES;
    } catch (const WrongCharacteristic&) {
        return ORC_WRONG_CHARACTERISTIC;
    } catch (const ParseError&) {
        return ORC_PARSE_ERROR;
    } catch (const std::bad_alloc&) {
        return ORC_NO_MEMORY;
    } catch (...) {
        return ORC_OTHER;
    }
}

BlockDiag to_blockdiag(const PrimeField& f, size_t k, const int32_t* dkind, const uint64_t* dval,
                       const uint64_t* dval2) {
    BlockDiag d;
    for (size_t t = 0; t < k;) {
        if (dkind[t] == ORC_D_SCALAR) {
            d.push(ScalarBlock{f.element(dval[t])});
            t += 1;
        } else if (dkind[t] == ORC_D_ANTIDIAG_HEAD) {
            d.push(AntiDiagBlock{f.element(dval[t])});
            t += 2;
        } else {
            d.push(AntiTriBlock{f.element(dval[t]), f.element(dval2[t])});
            t += 2;
        }
    }
    return d;
}

} // namespace

extern "C" {

int ref_ldlt(uint64_t p, size_t rows, size_t cols, const uint64_t* a, int variant,
             size_t threshold, int64_t* perm, uint64_t* lower, int32_t* dkind, uint64_t* dval,
             uint64_t* dval2, size_t* rank) {
    return guarded([&] {
        const PrimeField f(p);
        const Factorization fac = ldlt(to_matrix(f, rows, cols, a), make_cfg(variant, threshold));
        export_fact(fac, perm, lower, dkind, dval, dval2, rank);
    });
}

int ref_ldlt_zero_leading(uint64_t p, size_t m, size_t ny, const uint64_t* y, size_t nz,
                          const uint64_t* z, int variant, size_t threshold, int64_t* perm,
                          uint64_t* lower, int32_t* dkind, uint64_t* dval, uint64_t* dval2,
                          size_t* rank) {
    return guarded([&] {
        const PrimeField f(p);
        const Factorization fac = ldlt_zero_leading(to_matrix(f, m, ny, y), to_matrix(f, nz, nz, z),
                                                    make_cfg(variant, threshold));
        export_fact(fac, perm, lower, dkind, dval, dval2, rank);
    });
}

int ref_plduq(uint64_t p, size_t m, size_t n, const uint64_t* b, int64_t* row_image,
              int64_t* col_image, uint64_t* lower, uint64_t* diag, uint64_t* upper,
              size_t* rank) {
    return guarded([&] {
        const PrimeField f(p);
        const PlduqFactorization pf = plduq(to_matrix(f, m, n, b));
        for (size_t i = 0; i < m; ++i) row_image[i] = static_cast<int64_t>(pf.row_perm.image(i));
        for (size_t j = 0; j < n; ++j) col_image[j] = static_cast<int64_t>(pf.col_perm.image(j));
        from_matrix(pf.lower, lower);
        for (size_t k = 0; k < pf.rank; ++k) diag[k] = pf.diag[k].value;
        from_matrix(pf.upper, upper);
        *rank = pf.rank;
    });
}

int ref_trssyr2k(uint64_t p, size_t n, const uint64_t* u, const uint64_t* c, uint64_t* x) {
    return guarded([&] {
        const PrimeField f(p);
        from_matrix(trssyr2k(to_matrix(f, n, n, u), to_matrix(f, n, n, c)), x);
    });
}

int ref_gemm_sub(uint64_t p, size_t m, size_t n, size_t k, uint64_t* c, const uint64_t* a,
                 const uint64_t* b) {
    return guarded([&] {
        const PrimeField f(p);
        Matrix cm = to_matrix(f, m, n, c);
        gemm_sub(cm, to_matrix(f, m, k, a), to_matrix(f, k, n, b));
        from_matrix(cm, c);
    });
}

int ref_trsm_inplace(uint64_t p, size_t n, size_t ncols, const uint64_t* t, int upper, int trans,
                     int unit, uint64_t* b) {
    return guarded([&] {
        const PrimeField f(p);
        Matrix bm = to_matrix(f, n, ncols, b);
        trsm_inplace(to_matrix(f, n, n, t), upper ? Uplo::Upper : Uplo::Lower, trans != 0,
                     unit != 0, bm);
        from_matrix(bm, b);
    });
}

int ref_trmm_sub(uint64_t p, size_t n, size_t ncols, uint64_t* c, const uint64_t* t, int upper,
                 int trans, int unit, const uint64_t* b) {
    return guarded([&] {
        const PrimeField f(p);
        Matrix cm = to_matrix(f, n, ncols, c);
        trmm_sub(cm, to_matrix(f, n, n, t), upper ? Uplo::Upper : Uplo::Lower, trans != 0,
                 unit != 0, to_matrix(f, n, ncols, b));
        from_matrix(cm, c);
    });
}

// D given in the per-column encoding of oracle_api.h.
int ref_syrdk_sub_diag(uint64_t p, size_t n, size_t k, uint64_t* c, const uint64_t* g,
                       const uint64_t* d) {
    return guarded([&] {
        const PrimeField f(p);
        std::vector<FieldElement> dv;
        for (size_t t = 0; t < k; ++t) dv.push_back(f.element(d[t]));
        Matrix cm = to_matrix(f, n, n, c);
        syrdk_sub(cm, to_matrix(f, n, k, g), std::span<const FieldElement>(dv));
        from_matrix(cm, c);
    });
}

// strictify (rpmtools.cpp:74-132) of a factorization given in the flat layout; the
// result overwrites the same arrays.
int ref_strictify(uint64_t p, size_t n, size_t r, int64_t* perm, uint64_t* lower, int32_t* dkind,
                  uint64_t* dval, uint64_t* dval2, uint64_t* stats) {
    return guarded([&] {
        const PrimeField f(p);
        std::vector<std::size_t> img(n);
        for (size_t i = 0; i < n; ++i) img[i] = static_cast<std::size_t>(perm[i]);
        Factorization fac{Permutation::from_image(std::move(img)), to_matrix(f, n, r, lower),
                          to_blockdiag(f, r, dkind, dval, dval2), r};
        StrictifyStats st;
        strictify(fac, &st);
        size_t rank = 0;
        export_fact(fac, perm, lower, dkind, dval, dval2, &rank);
        stats[0] = st.blocks_converted;
        stats[1] = st.entries_touched;
    });
}

int ref_syrdk_sub(uint64_t p, size_t n, size_t k, uint64_t* c, const uint64_t* g,
                  const int32_t* dkind, const uint64_t* dval, const uint64_t* dval2) {
    return guarded([&] {
        const PrimeField f(p);
        const BlockDiag d = to_blockdiag(f, k, dkind, dval, dval2);
        Matrix cm = to_matrix(f, n, n, c);
        syrdk_sub(cm, to_matrix(f, n, k, g), d);
        from_matrix(cm, c);
    });
}

int ref_syr2k_sub(uint64_t p, size_t n, size_t k, uint64_t* c, const uint64_t* a,
                  const uint64_t* b) {
    return guarded([&] {
        const PrimeField f(p);
        Matrix cm = to_matrix(f, n, n, c);
        syr2k_sub(cm, to_matrix(f, k, n, a), to_matrix(f, k, n, b));
        from_matrix(cm, c);
    });
}

int ref_rank_profile(uint64_t p, size_t m, size_t n, const uint64_t* a, uint64_t* out) {
    return guarded([&] {
        const PrimeField f(p);
        from_matrix(rank_profile_bruteforce(to_matrix(f, m, n, a)), out);
    });
}

// Files (io.cpp): the reference parses `in` (MatrixFile or FactorizationFile, by `kind`
// 0/1) and emits it again to `out` -- so a file written by the B200 library can be checked
// byte for byte against the reference's own emit, and read by the reference's parser.
int ref_file_reemit(int kind, const char* in, const char* out) {
    return guarded([&] {
        std::ifstream is(in, std::ios::binary);
        if (!is) throw ParseError("cannot open input");
        std::ostringstream os;
        if (kind == 0) MatrixFile::parse(is).emit(os);
        else FactorizationFile::parse(is).emit(os);
        std::ofstream o(out, std::ios::binary);
        o << os.str();
    });
}

// FactorizationFile::from(f).emit of a flat factorization (the reference's writer).
int ref_factorization_emit(uint64_t p, size_t n, size_t r, const int64_t* perm, const uint64_t* lower,
                           const int32_t* dkind, const uint64_t* dval, const uint64_t* dval2,
                           const char* out) {
    return guarded([&] {
        const PrimeField f(p);
        std::vector<std::size_t> img(n);
        for (size_t i = 0; i < n; ++i) img[i] = static_cast<std::size_t>(perm[i]);
        const Factorization fac{Permutation::from_image(std::move(img)), to_matrix(f, n, r, lower),
                                to_blockdiag(f, r, dkind, dval, dval2), r};
        std::ofstream o(out, std::ios::binary);
        FactorizationFile::from(fac).emit(o);
    });
}

} // extern "C"
