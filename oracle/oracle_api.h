/* oracle_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Common C interface of the two CPU checkers that live under oracle/:
 *   - liboracle.so   : the plain-C restatement of the reference algorithm
 *                      (oracle/ldlt_oracle.c, prefix orc_), and
 *   - libffldl_ref.so: the UNMODIFIED reference sources compiled from
 *                      /root/reference/proj/src by oracle/Makefile, behind a
 *                      thin C driver (oracle/ref_capi.cpp, prefix ref_).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these.  The product (paper_1802_10453_b200)
 * never links or calls anything here.
 *
 * Output layout of a factorization of an n x n matrix of rank r (matches the
 * reference's Factorization, proj/include/ffldl/blockdiag.hpp:153):
 *   perm[n]        perm.image(pos): original row placed at position pos
 *                  (proj/include/ffldl/permutation.hpp:11-19)
 *   lower[n*r]     row-major n x r, unit lower on its top r rows
 *   dkind[r]       per pivot column: 0 Scalar, 1/2 AntiDiag head/tail,
 *                  3/4 AntiTri head/tail (blockdiag.hpp:20-33)
 *   dval[r]        Scalar d / AntiDiag x / AntiTri c (same on head and tail)
 *   dval2[r]       AntiTri d (0 otherwise)
 * Caller allocates perm/dkind/dval/dval2 with n entries and lower with n*n.
 *
 * Status codes mirror the reference exception tree (proj/include/ffldl/errors.hpp:9-55).
 */
#ifndef FFLDL_ORACLE_API_H
#define FFLDL_ORACLE_API_H

#include <stddef.h>
#include <stdint.h>

#define ORC_OK 0
#define ORC_DIMENSION_MISMATCH 1
#define ORC_NOT_SYMMETRIC 2
#define ORC_NOT_PRIME 3
#define ORC_ZERO_INVERSE 4
#define ORC_CHAR_TWO_DIVISION 5
#define ORC_NON_UNIT_TRIANGULAR 6
#define ORC_SINGULAR_TRIANGULAR 7
#define ORC_CHAR_TWO_NONZERO_DIAGONAL 8
#define ORC_BAD_BLOCK_SIZES 9
#define ORC_OTHER 10
#define ORC_NO_MEMORY 11
#define ORC_WRONG_CHARACTERISTIC 12
#define ORC_PARSE_ERROR 13

#define ORC_VARIANT_RECURSIVE 0
#define ORC_VARIANT_CROUT 1
#define ORC_VARIANT_CASCADE 2

#define ORC_D_SCALAR 0
#define ORC_D_ANTIDIAG_HEAD 1
#define ORC_D_ANTIDIAG_TAIL 2
#define ORC_D_ANTITRI_HEAD 3
#define ORC_D_ANTITRI_TAIL 4

#endif
