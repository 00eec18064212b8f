// Device-side verification of a factorization.
//
//  * reconstruct (blockdiag.hpp:161-182): P L D L^T P^T, computed as H = L D (one
//    pass over L) and C = H L^T (one modular GEMM on the engine's GEMM path), then
//    compared entry by entry with the input A (C(i, j) against A(perm(i), perm(j)),
//    conjugate_sym of permutation.hpp:122).  The mismatch count is exact.
//  * pivoting_matrix (rpmtools.cpp:61-68): Pi = P support(D) P^T has at most one 1 per
//    row (the support of D is a symmetric partial permutation), so it is returned as
//    a partner array: partner[perm(a)] = perm(b) for every (a, b) in support(D)
//    (blockdiag.hpp support()), -1 for rows without a pivot.
#include <algorithm>

#include "ffb_kernels.cuh"

#define FFB_ROWCHUNK 65535

namespace ffb {

// H (n x r) = L (n x r) * D, D in the per-column encoding of the C-ABI:
// kind 0 Scalar(d); 1/2 first/second column of AntiDiag(x) = [0 x; x 0];
// 3/4 first/second column of AntiTri(c, d) = [0 c; c d] (blockdiag.hpp:15-33).
__global__ void k_apply_d(Fp f, uint32_t* H, int64_t ldh, const uint32_t* L, int64_t ldl, int64_t n,
                          int64_t r, const int32_t* kind, const uint32_t* val, const uint32_t* val2) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    if (i >= n) return;
    const uint32_t* l = L + i * ldl;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < r; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t k = __ldcg(kind + t);
        uint32_t h;
        if (k == 0) {
            h = fmul(f, __ldcg(l + t), __ldcg(val + t));
        } else if (k == 1 || k == 3) {  // column t of [0 x; x 0] / [0 c; c d]: x * L(:, t+1)
            h = fmul(f, __ldcg(l + t + 1), __ldcg(val + t));
        } else if (k == 2) {             // column t+1 of [0 x; x 0]: x * L(:, t)
            h = fmul(f, __ldcg(l + t - 1), __ldcg(val + t));
        } else {                          // column t+1 of [0 c; c d]: c L(:, t) + d L(:, t+1)
            h = fadd(f, fmul(f, __ldcg(l + t - 1), __ldcg(val + t)), fmul(f, __ldcg(l + t), __ldcg(val2 + t)));
        }
        H[i * ldh + t] = h;
    }
}

// Count (i, j) with C(i, j) != A(perm(i), perm(j)); one warp-aggregated atomic per warp.
__global__ void k_compare_conj(const uint32_t* C, int64_t ldc, const uint32_t* A, int64_t lda,
                               const int32_t* perm, int64_t row0, int64_t n, unsigned long long* count) {
    FFB_PDL_ENTRY();
    const int64_t i = row0 + blockIdx.y;
    const uint32_t* arow = A + (int64_t)__ldcg(perm + i) * lda;
    const uint32_t* crow = C + i * ldc;
    unsigned bad = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        bad += __ldcg(crow + j) != __ldcg(arow + __ldcg(perm + j));
    for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, (unsigned long long)bad);
}

__global__ void k_partners(const int32_t* perm, const int32_t* kind, int64_t n, int64_t r, int32_t* partner) {
    FFB_PDL_ENTRY();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    int32_t q = -1;
    if (t < r) {
        const int32_t k = kind[t];
        q = k == 0 ? perm[t] : (k == 1 || k == 3) ? perm[t + 1] : perm[t - 1];
    }
    partner[perm[t]] = q;
}

void reconstruct_mismatches(const Fp& f, cudaStream_t st, DMat A, const int32_t* perm, DMat L, DDiag D,
                            int64_t r, DMat H, DMat C, unsigned long long* dcount) {
    const int64_t n = A.rows;
    if (n <= 0) return;
    for (int64_t r0 = 0; r > 0 && r0 < n; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, n - r0);
        launch_k(k_apply_d, dim3((unsigned)std::min<int64_t>(cdiv(r, 256), 64), (unsigned)nr), 256, 0, st, f,
                 H.ptr + r0 * H.ld, H.ld, L.ptr + r0 * L.ld, L.ld, nr, r, D.kind, D.val, D.val2);
        ++g_launches;
    }
    gemm(f, st, GEMM_SET, C, H, false, L, true, n, n, r);  // C = (L D) L^T
    for (int64_t r0 = 0; r0 < n; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, n - r0);
        launch_k(k_compare_conj, dim3((unsigned)std::min<int64_t>(cdiv(n, 1024), 32), (unsigned)nr), 256, 0, st,
                 C.ptr, C.ld, A.ptr, A.ld, perm, r0, n, dcount);
        ++g_launches;
    }
    FFB_CHECK_LAUNCH();
}

void pivoting_partners(cudaStream_t st, const int32_t* perm, const int32_t* kind, int64_t n, int64_t r,
                       int32_t* partner) {
    if (n <= 0) return;
    launch_k(k_partners, (unsigned)cdiv(n, 256), 256, 0, st, perm, kind, n, r, partner);
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

}  // namespace ffb
