/* ffldl_b200.h -- C-ABI of the B200-native PLDL^TP^T engine (libffldl_b200.so).
 *
 * Drop-in boundary for the reference's hot path.  The reference (`ffldl`,
 * /root/reference/proj) has no FFI: its public surface is the C++ API in
 * proj/include/ffldl/.  Each entry point below replaces one function of that
 * API with plain pointers and sizes (no C++ or torch types); the C++ shim in
 * paper_1802_10453_b200/shim/ and the Python mirror in
 * paper_1802_10453_b200/ffldl.py bind to it.  See INTEGRATION.md.
 *
 * Conventions (identical to the reference):
 *   - matrices are row-major arrays of canonical residues in [0, p)
 *     (FieldElement, proj/include/ffldl/field.hpp:12-16); host entry points
 *     accept uint64 elements (the reference's element type);
 *   - a factorization of an n x n matrix of rank r is returned as
 *       perm[n]     perm.image(pos) = original row at position pos
 *                   (proj/include/ffldl/permutation.hpp:11-19),
 *       lower[n*r]  row-major n x r, unit lower on its top r rows,
 *       dkind[r], dval[r], dval2[r]  D per pivot column: FFB_D_* kind,
 *                   Scalar d / AntiDiag x / AntiTri c, and AntiTri d
 *                   (proj/include/ffldl/blockdiag.hpp:20-33,153);
 *     callers size perm/dkind/dval/dval2 with n entries and lower with n*n;
 *   - variant/threshold follow SytrfConfig (proj/include/ffldl/sytrf.hpp:8-17);
 *   - every entry point returns FFB_OK or an FFB_* status that maps 1:1 to the
 *     reference's exception classes (proj/include/ffldl/errors.hpp:9-55);
 *     FFB_CUDA_ERROR / FFB_UNSUPPORTED are new (device failure, p >= 2^31).
 *   - all work runs on ONE CUDA stream owned by the context.
 */
#ifndef FFLDL_B200_H
#define FFLDL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFB_OK 0
#define FFB_DIMENSION_MISMATCH 1     /* ffldl::DimensionMismatch */
#define FFB_NOT_SYMMETRIC 2          /* ffldl::NotSymmetric */
#define FFB_NOT_PRIME 3              /* ffldl::NotPrime */
#define FFB_ZERO_INVERSE 4           /* ffldl::ZeroInverse */
#define FFB_CHAR_TWO_DIVISION 5      /* ffldl::CharTwoDivision */
#define FFB_NON_UNIT_TRIANGULAR 6    /* ffldl::NonUnitTriangular */
#define FFB_SINGULAR_TRIANGULAR 7    /* ffldl::SingularTriangular */
#define FFB_CHAR_TWO_NONZERO_DIAGONAL 8 /* ffldl::CharTwoNonzeroDiagonal */
#define FFB_BAD_BLOCK_SIZES 9        /* ffldl::BadBlockSizes */
#define FFB_ERROR 10                 /* ffldl::Error (other) */
#define FFB_NO_MEMORY 11             /* device workspace exhausted */
#define FFB_CUDA_ERROR 12            /* CUDA runtime failure (new) */
#define FFB_UNSUPPORTED 13           /* modulus outside the device range (new) */
#define FFB_WRONG_CHARACTERISTIC 14  /* ffldl::WrongCharacteristic (strictify) */
#define FFB_PARSE_ERROR 15           /* ffldl::ParseError (matrix / factorization files) */

#define FFB_VARIANT_RECURSIVE 0
#define FFB_VARIANT_CROUT 1
#define FFB_VARIANT_CASCADE 2

#define FFB_D_SCALAR 0
#define FFB_D_ANTIDIAG_HEAD 1
#define FFB_D_ANTIDIAG_TAIL 2
#define FFB_D_ANTITRI_HEAD 3
#define FFB_D_ANTITRI_TAIL 4

/* Element types of host buffers for the compact entry points. */
#define FFB_U8 1
#define FFB_U16 2
#define FFB_U32 4
#define FFB_U64 8

typedef struct ffb_context ffb_context;

/* Library identity and status text. */
int ffb_version(void);
const char* ffb_status_string(int status);
/* Last error message of the calling thread (detail for the previous non-OK status). */
const char* ffb_last_error(void);

/* One context = one device, one stream, one cached workspace. */
int ffb_create(ffb_context** ctx, int device);
int ffb_destroy(ffb_context* ctx);
/* The context's CUDA stream (cudaStream_t), for callers that time on it. */
void* ffb_stream(ffb_context* ctx);
/* Kernel launches issued by the most recent call (instrumentation). */
uint64_t ffb_launch_count(ffb_context* ctx);
/* Host<->device synchronization points (rank/permutation read-backs) of the most recent call. */
uint64_t ffb_sync_count(ffb_context* ctx);
/* Per-kernel-class timing of subsequent calls (CUDA events around every launch, on the
 * launching stream; adds overhead, off by default).  enable resets the totals.
 * Classes: 0 GEMM, 1 Crout leaf, 2 PLDUQ row detection / sequential kernel, 3 TRSM base,
 * 4 data movement, 5 other, 6 PLDUQ sketch, 7 PLDUQ column rank profile, 8 PLDUQ pairing,
 * 9 LDU base, 10 tensor-core operand packing, 11 PLDUQ row elimination on candidates. */
int ffb_profile_enable(ffb_context* ctx, int enable);
int ffb_profile_read(ffb_context* ctx, int klass, uint64_t* launches, double* ms, double* ops,
                     double* bytes);

/* ffldl::ldlt(const Matrix&, const SytrfConfig&)  -- proj/include/ffldl/sytrf.hpp:30,
 * proj/src/sytrf.cpp:354-358.  Host buffers. */
int ffb_ldlt(ffb_context* ctx, uint64_t p, size_t rows, size_t cols, const uint64_t* a,
             int variant, size_t threshold, int64_t* perm, uint64_t* lower, int32_t* dkind,
             uint64_t* dval, uint64_t* dval2, size_t* rank);

/* Same contract with compact host element types (a_type, lower_type in FFB_U8..FFB_U64);
 * used by the end-to-end benchmark to move fewer bytes over PCIe. */
int ffb_ldlt_compact(ffb_context* ctx, uint64_t p, size_t n, const void* a, int a_type,
                     int variant, size_t threshold, int64_t* perm, void* lower, int lower_type,
                     int32_t* dkind, uint64_t* dval, uint64_t* dval2, size_t* rank);

/* ffldl::ldlt_zero_leading(y, z, cfg) -- sytrf.hpp:41, sytrf.cpp:360-368.
 * y is m x ny, z is nz x nz; outputs have dimension m + nz. */
int ffb_ldlt_zero_leading(ffb_context* ctx, uint64_t p, size_t m, size_t ny, const uint64_t* y,
                          size_t nz, const uint64_t* z, int variant, size_t threshold,
                          int64_t* perm, uint64_t* lower, int32_t* dkind, uint64_t* dval,
                          uint64_t* dval2, size_t* rank);

/* Device-resident factorization (the benchmark's timed region).
 * d_a: n x n uint32 residues, row stride lda, OVERWRITTEN (used as workspace).
 * d_perm[n] (int32), d_lower (n x n uint32, row stride ldl; first r columns valid),
 * d_dkind/d_dval/d_dval2[n] receive the factorization; *rank on the host.
 * Runs on the context stream; returns after the factorization is complete. */
int ffb_ldlt_device(ffb_context* ctx, uint64_t p, size_t n, uint32_t* d_a, size_t lda,
                    int variant, size_t threshold, int32_t* d_perm, uint32_t* d_lower,
                    size_t ldl, int32_t* d_dkind, uint32_t* d_dval, uint32_t* d_dval2,
                    size_t* rank);

/* Device-side verification, on the outputs of ffb_ldlt_device.
 * ffb_verify_device: *mismatches = the number of entries (i, j) where P L D L^T P^T differs
 * from A (Factorization::reconstruct, proj/include/ffldl/blockdiag.hpp:161-182; computed as
 * one modular GEMM and an entry-wise comparison, so 0 is an exact proof of the identity).
 * d_a is the ORIGINAL input (n x n uint32 residues, row stride lda), not overwritten. */
int ffb_verify_device(ffb_context* ctx, uint64_t p, size_t n, const uint32_t* d_a, size_t lda,
                      const int32_t* d_perm, const uint32_t* d_lower, size_t ldl,
                      const int32_t* d_dkind, const uint32_t* d_dval, const uint32_t* d_dval2,
                      size_t rank, uint64_t* mismatches);

/* pivoting_matrix(f) -- proj/src/rpmtools.cpp:61-68.  Pi = P support(D) P^T has at most one
 * nonzero per row; d_partner[i] = j where Pi(i, j) = 1, else -1 (n int32, device). */
int ffb_pivoting_partners_device(ffb_context* ctx, size_t n, const int32_t* d_perm,
                                 const int32_t* d_dkind, size_t rank, int32_t* d_partner);

/* ffldl::plduq(b) -- proj/include/ffldl/plduq.hpp:42, proj/src/plduq.cpp:36-123.
 * Caller sizes: row_image[m], col_image[n], lower[m*min(m,n)], diag[min(m,n)],
 * upper[min(m,n)*n]; lower is m x r and upper r x n on return. */
int ffb_plduq(ffb_context* ctx, uint64_t p, size_t m, size_t n, const uint64_t* b,
              int64_t* row_image, int64_t* col_image, uint64_t* lower, uint64_t* diag,
              uint64_t* upper, size_t* rank);

/* ffldl::trssyr2k(u, c) -- proj/include/ffldl/trssyr2k.hpp:17, proj/src/trssyr2k.cpp:55-77. */
int ffb_trssyr2k(ffb_context* ctx, uint64_t p, size_t n, const uint64_t* u, const uint64_t* c,
                 uint64_t* x);

/* BLAS3 kernels -- proj/include/ffldl/kernels.hpp:13-32 (Uplo: 0 Lower, 1 Upper). */
int ffb_gemm_sub(ffb_context* ctx, uint64_t p, size_t m, size_t n, size_t k, uint64_t* c,
                 const uint64_t* a, const uint64_t* b);
int ffb_trmm_sub(ffb_context* ctx, uint64_t p, size_t n, size_t ncols, uint64_t* c,
                 const uint64_t* t, int upper, int trans, int unit, const uint64_t* b);
int ffb_trsm_inplace(ffb_context* ctx, uint64_t p, size_t n, size_t ncols, const uint64_t* t,
                     int upper, int trans, int unit, uint64_t* b);
int ffb_syrdk_sub(ffb_context* ctx, uint64_t p, size_t n, size_t k, uint64_t* c,
                  const uint64_t* g, const int32_t* dkind, const uint64_t* dval,
                  const uint64_t* dval2);
int ffb_syr2k_sub(ffb_context* ctx, uint64_t p, size_t n, size_t k, uint64_t* c,
                  const uint64_t* a, const uint64_t* b);
/* syrdk_sub(Matrix& c, const Matrix& g, std::span<const FieldElement> d) -- the diagonal
 * overload, kernels.hpp:29, kernels.cpp:108-119: C -= G diag(d) G^T (g is n x k, d[k]). */
int ffb_syrdk_sub_diag(ffb_context* ctx, uint64_t p, size_t n, size_t k, uint64_t* c,
                       const uint64_t* g, const uint64_t* d);

/* strictify(Factorization&, StrictifyStats*) -- proj/include/ffldl/rpmtools.hpp:39,
 * proj/src/rpmtools.cpp:74-132.  Rewrites every characteristic-2 AntiTri block [0 c; c d]
 * into Scalar d, Scalar -c^2/d, adjusting two columns of L and composing a transposition
 * into P per block (all on the device).  Host buffers in the ffb_ldlt layout (perm[n],
 * lower n x rank, dkind/dval/dval2[rank]), updated in place; the two counters receive
 * StrictifyStats (may be NULL).  FFB_WRONG_CHARACTERISTIC for an AntiTri block over odd p. */
int ffb_strictify(ffb_context* ctx, uint64_t p, size_t n, size_t rank, int64_t* perm,
                  uint64_t* lower, int32_t* dkind, uint64_t* dval, uint64_t* dval2,
                  uint64_t* blocks_converted, uint64_t* entries_touched);
/* Same on a device factorization (the ffb_ldlt_device output layout, row stride ldl). */
int ffb_strictify_device(ffb_context* ctx, uint64_t p, size_t n, size_t rank, int32_t* d_perm,
                         uint32_t* d_lower, size_t ldl, int32_t* d_dkind, uint32_t* d_dval,
                         uint32_t* d_dval2, uint64_t* blocks_converted, uint64_t* entries_touched);

/* Device-buffer modular GEMM (the engine's contraction kernel, kernels.hpp:13 semantics):
 * C (m x n) = C - op(A) op(B) (mode 0), C + op(A) op(B) (mode 1), op(A) op(B) (mode 2);
 * op(A) = A (m x k) or A^T when ta (A stored k x m); op(B) = B (k x n) or B^T when tb.
 * uint32 residues, row strides ldc/lda/ldb, on the context stream (asynchronous). */
int ffb_gemm_device(ffb_context* ctx, uint64_t p, int mode, size_t m, size_t n, size_t k,
                    uint32_t* d_c, size_t ldc, const uint32_t* d_a, size_t lda, int ta,
                    const uint32_t* d_b, size_t ldb, int tb);

/* Matrix and factorization files: MatrixFile / FactorizationFile,
 * proj/include/ffldl/io.hpp:22-62, proj/src/io.cpp:39-222.  Readers accept the reference's
 * text format (byte-compatible) and a checksummed binary format (binary != 0 on write; see
 * csrc/ffb_io.cu).  Read with NULL arrays first to get the dimensions, then again with
 * caller-sized buffers (values rows*cols; perm n, lower n*rank, dkind/dval/dval2 rank) in
 * the element type given.  Parse failures return FFB_PARSE_ERROR (ffldl::ParseError). */
int ffb_matrix_read(const char* path, uint64_t* rows, uint64_t* cols, uint64_t* modulus, int* symmetric,
                    void* values, int elem_type);
int ffb_matrix_write(const char* path, int binary, uint64_t rows, uint64_t cols, uint64_t modulus,
                     int symmetric, const void* values, int elem_type);
int ffb_factorization_read(const char* path, uint64_t* n, uint64_t* modulus, uint64_t* rank, int64_t* perm,
                           void* lower, int lower_type, int32_t* dkind, uint64_t* dval, uint64_t* dval2);
int ffb_factorization_write(const char* path, int binary, uint64_t n, uint64_t modulus, uint64_t rank,
                            const int64_t* perm, const void* lower, int lower_type, const int32_t* dkind,
                            const uint64_t* dval, const uint64_t* dval2);

/* Seeded counter-based generators of the benchmark configurations
 * (BASELINE.json configs 1..5).  Host version
 * writes uint64 residues; device version writes uint32 residues (row stride n).
 * Both are bit-identical.  config: 1 dense, 2 M diag(d) M^T permuted (rank r),
 * 3 dense (any p), 4 hollow, 5 L R L^T (rank r). */
int ffb_generate_host(int config, size_t n, size_t r, uint64_t p, uint64_t seed, uint64_t* out);
int ffb_generate_device(ffb_context* ctx, int config, size_t n, size_t r, uint64_t p,
                        uint64_t seed, uint32_t* d_out);
/* The rank profile matrix R of configuration 5 as a partner array:
 * partner[i] = j if R(i,j) = 1, -1 if row i of R is zero. */
int ffb_config5_partners(size_t n, size_t r, uint64_t seed, int64_t* partner);

#ifdef __cplusplus
}
#endif

#endif /* FFLDL_B200_H */
