// ffb_api.cu -- device kernels behind the secondary C-ABI entry points: the triangular
// operands of trmm_sub / trsm_inplace (kernels.cpp:23-81), the block-diagonal factor of
// syrdk_sub (kernels.cpp:83-119) and strictify (rpmtools.cpp:74-132).  All modular
// arithmetic of these entry points runs here; the host only moves buffers.
#include "ffb_kernels.cuh"

namespace ffb {
namespace {

// op(T)(i, k) under the triangle / unit-diagonal conventions of tri_entry
// (kernels.cpp:23-29): the stored triangle of T, transposed when trans, unit diagonal.
__device__ __forceinline__ uint32_t tri_entry(const uint32_t* T, int64_t ld, bool upper, bool trans,
                                              bool unit, uint32_t one, int64_t i, int64_t k) {
    if (trans) {
        const int64_t s = i;
        i = k;
        k = s;
    }
    if (i == k) return unit ? one : __ldcg(T + i * ld + i);
    const bool stored = upper ? (i < k) : (i > k);
    return stored ? __ldcg(T + i * ld + k) : 0u;
}

// out(i, k) = op(T)(a_i, a_k), a_i = n-1-i when rev (the index reversal that turns an
// effective-upper op(T) into a lower one).  With dinv: the unit-lower normalisation
// dinv(a_i) * op(T)(a_i, a_k) below the diagonal, 1 on it, 0 above.
__global__ void k_tri_dense(Fp f, const uint32_t* T, int64_t ldt, int64_t n, int upper, int trans,
                            int unit, int rev, const uint32_t* dinv, uint32_t* out, int64_t ldo, int64_t i0) {
    FFB_PDL_ENTRY();
    const int64_t i = i0 + blockIdx.y;
    const int64_t ai = rev ? n - 1 - i : i;
    const uint32_t one = 1u % f.p;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t ak = rev ? n - 1 - k : k;
        uint32_t v;
        if (dinv) v = k < i ? fmul(f, tri_entry(T, ldt, upper, trans, unit, one, ai, ak), __ldcg(dinv + ai))
                            : (k == i ? one : 0u);
        else v = tri_entry(T, ldt, upper, trans, unit, one, ai, ak);
        out[i * ldo + k] = v;
    }
}

// diag[i] = T(i, i); *flag |= 1 if one is zero (SingularTriangular, kernels.cpp:64-71)
__global__ void k_tri_diag(const uint32_t* T, int64_t ld, int64_t n, uint32_t* diag, int32_t* flag) {
    FFB_PDL_ENTRY();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t d = __ldcg(T + i * ld + i);
    diag[i] = d;
    if (d == 0) atomicOr(flag, 1);
}

// dst(i, j) = src(a_i, j) * (dinv ? dinv(a_i) : 1)
__global__ void k_rows_rev_scaled(Fp f, uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds, int64_t n,
                                  int64_t ncols, int rev, const uint32_t* dinv, int64_t i0) {
    FFB_PDL_ENTRY();
    const int64_t i = i0 + blockIdx.y;
    const int64_t ai = rev ? n - 1 - i : i;
    const uint32_t s = dinv ? __ldcg(dinv + ai) : 0u;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < ncols; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = __ldcg(src + ai * lds + j);
        dst[i * ldd + j] = dinv ? fmul(f, v, s) : v;
    }
}

// H = G * D for the per-column encoding of a BlockDiag (blockdiag.hpp:20-33): Scalar d,
// AntiDiag [0 x; x 0], AntiTri [0 c; c d] (head column t, tail t+1), so that
// C - H G^T = C - G D G^T (syrdk_sub, kernels.cpp:83-106; a plain diagonal for the span
// overload, kernels.cpp:108-119).
__global__ void k_apply_d(Fp f, uint32_t* H, int64_t ldh, const uint32_t* G, int64_t ldg, int64_t n, int64_t k,
                          const int32_t* kind, const uint32_t* val, const uint32_t* val2) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    const uint32_t* g = G + i * ldg;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < k; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t kd = __ldcg(kind + t);
        const uint32_t v = __ldcg(val + t);
        uint32_t h;
        if (kd == FFB_D_SCALAR) h = fmul(f, __ldcg(g + t), v);
        else if (kd == FFB_D_ANTIDIAG_HEAD || kd == FFB_D_ANTITRI_HEAD) h = fmul(f, __ldcg(g + t + 1), v);
        else if (kd == FFB_D_ANTIDIAG_TAIL) h = fmul(f, __ldcg(g + t - 1), v);
        else h = fadd(f, fmul(f, __ldcg(g + t - 1), v), fmul(f, __ldcg(g + t), __ldcg(val2 + t)));
        H[i * ldh + t] = h;
    }
}

// ---- strictify (rpmtools.cpp:74-132) -------------------------------------------------
// For an AntiTri block [0 c; c d] at pivot columns (t, t+1) of L (n x r):
//   x = L(t+1, t), cd = c / d;
//   rows t, t+1 swap their prefix columns [0, t); P absorbs the transposition (t t+1);
//   the block rows become [1 0; cd 1]; every later row i >= t+2 maps its column pair
//   (a, b) = (L(i,t), L(i,t+1)) to (b + cd (a - x b), a - x b);
//   D gets Scalar d, Scalar -c^2/d.
// The per-block column maps act identically on both rows of every other block's swap
// (those rows lie strictly below), so all blocks are applied in parallel.
__global__ void k_strict_prep(Fp f, const uint32_t* L, int64_t ld, const int32_t* heads, int64_t nb,
                              const uint32_t* val, const uint32_t* val2, uint32_t* x, uint32_t* cd,
                              uint32_t* dnew, int64_t n, unsigned long long* touched) {
    FFB_PDL_ENTRY();
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    const int64_t t = heads[b];
    const uint32_t c = __ldcg(val + t), d = __ldcg(val2 + t);
    const uint32_t xv = __ldcg(L + (t + 1) * ld + t);
    const uint32_t q = fmul(f, c, finv(f, d));
    x[b] = xv;
    cd[b] = q;
    dnew[2 * b] = d;
    dnew[2 * b + 1] = fneg(f, fmul(f, fmul(f, c, c), finv(f, d)));
    // entries_touched of rpmtools.cpp:95-123
    const unsigned long long m1 = (unsigned long long)(n - t - 1);
    atomicAdd(touched, (xv ? m1 : 0ull) + 2ull * (unsigned long long)t +
                           2ull * (unsigned long long)(n > t + 2 ? n - t - 2 : 0) + m1);
}

// one CTA row per matrix row: apply every block's column map to that row
__global__ void k_strict_cols(Fp f, uint32_t* L, int64_t ld, int64_t n, const int32_t* heads, int64_t nb,
                              const uint32_t* x, const uint32_t* cd) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.x;
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
        const int64_t t = heads[b];
        if (i < t) continue;
        uint32_t* row = L + i * ld;
        if (i == t) continue;  // row t of the block stays (1, 0)
        if (i == t + 1) {      // [x 1] -> [cd 1]
            row[t] = cd[b];
            continue;
        }
        const uint32_t a = row[t], bb = row[t + 1];
        const uint32_t e = fsub(f, a, fmul(f, x[b], bb));
        row[t] = fadd(f, bb, fmul(f, cd[b], e));
        row[t + 1] = e;
    }
}

// rows t, t+1 swap their prefix columns [0, t); the permutation images swap; D rewritten
__global__ void k_strict_rows(uint32_t* L, int64_t ld, const int32_t* heads, int64_t nb, int32_t* perm,
                              int32_t* kind, uint32_t* val, uint32_t* val2, uint32_t* inv, const uint32_t* dnew,
                              Fp f) {
    FFB_PDL_ENTRY();
    const int64_t b = blockIdx.y;
    if (b >= nb) return;
    const int64_t t = heads[b];
    uint32_t* r0 = L + t * ld;
    uint32_t* r1 = L + (t + 1) * ld;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < t; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t u = r0[j];
        r0[j] = r1[j];
        r1[j] = u;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int32_t pi = perm[t];
        perm[t] = perm[t + 1];
        perm[t + 1] = pi;
        kind[t] = kind[t + 1] = FFB_D_SCALAR;
        val[t] = dnew[2 * b];
        val[t + 1] = dnew[2 * b + 1];
        val2[t] = val2[t + 1] = 0;
        if (inv) {
            inv[t] = finv(f, dnew[2 * b]);
            inv[t + 1] = finv(f, dnew[2 * b + 1]);
        }
    }
}

unsigned gx_for(int64_t cols) { return (unsigned)std::min<int64_t>(64, std::max<int64_t>(1, cdiv(cols, 256))); }

}  // namespace

void tri_dense(const Fp& f, cudaStream_t st, DMat out, DMat T, bool upper, bool trans, bool unit, bool rev,
               const uint32_t* dinv) {
    const int64_t n = T.rows;
    if (n <= 0) return;
    for (int64_t i0 = 0; i0 < n; i0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, n - i0);
        launch_k(k_tri_dense, dim3(gx_for(n), (unsigned)nr), 256, 0, st, f, T.ptr, T.ld, n, (int)upper,
                 (int)trans, (int)unit, (int)rev, dinv, out.ptr, out.ld, i0);
        ++g_launches;
    }
    FFB_CHECK_LAUNCH();
}

void tri_diag(cudaStream_t st, DMat T, uint32_t* diag, int32_t* flag) {
    if (T.rows <= 0) return;
    launch_k(k_tri_diag, (unsigned)cdiv(T.rows, 256), 256, 0, st, T.ptr, T.ld, T.rows, diag, flag);
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

void rows_rev_scaled(const Fp& f, cudaStream_t st, DMat dst, DMat src, bool rev, const uint32_t* dinv) {
    if (dst.rows <= 0 || dst.cols <= 0) return;
    for (int64_t i0 = 0; i0 < dst.rows; i0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, dst.rows - i0);
        launch_k(k_rows_rev_scaled, dim3(gx_for(dst.cols), (unsigned)nr), 256, 0, st, f, dst.ptr, dst.ld,
                 src.ptr, src.ld, dst.rows, dst.cols, (int)rev, dinv, i0);
        ++g_launches;
    }
    FFB_CHECK_LAUNCH();
}

void apply_d(const Fp& f, cudaStream_t st, DMat H, DMat G, const int32_t* kind, const uint32_t* val,
             const uint32_t* val2) {
    if (G.rows <= 0 || G.cols <= 0) return;
    for (int64_t i0 = 0; i0 < G.rows; i0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, G.rows - i0);
        launch_k(k_apply_d, dim3(gx_for(G.cols), (unsigned)nr), 256, 0, st, f, H.ptr + i0 * H.ld, H.ld,
                 G.ptr + i0 * G.ld, G.ld, nr, G.cols, kind, val, val2);
        ++g_launches;
    }
    FFB_CHECK_LAUNCH();
}

void strictify_device(const Fp& f, cudaStream_t st, DMat L, int64_t n, const int32_t* heads, int64_t nb,
                      int32_t* perm, DDiag D, uint32_t* scratch, unsigned long long* touched) {
    if (nb <= 0) return;
    uint32_t* x = scratch;
    uint32_t* cd = scratch + nb;
    uint32_t* dnew = scratch + 2 * nb;
    launch_k(k_strict_prep, (unsigned)cdiv(nb, 128), 128, 0, st, f, L.ptr, L.ld, heads, nb, D.val, D.val2, x, cd,
             dnew, n, touched);
    launch_k(k_strict_cols, (unsigned)n, 128, 0, st, f, L.ptr, L.ld, n, heads, nb, x, cd);
    for (int64_t b0 = 0; b0 < nb; b0 += 65535) {
        const int64_t m = std::min<int64_t>(65535, nb - b0);
        launch_k(k_strict_rows, dim3(gx_for(n), (unsigned)m), 256, 0, st, L.ptr, L.ld, heads + b0, m, perm,
                 D.kind, D.val, D.val2, D.inv, dnew + 2 * b0, f);
    }
    g_launches += 3;
    FFB_CHECK_LAUNCH();
}

}  // namespace ffb
