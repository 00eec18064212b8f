// ffb_plduq.cu -- parallel rank-profile-revealing PLDUQ (plduq.cpp:36-123).
//
// The reference's PLDUQ is a row-sequential Crout: row i's pivot is the
// leftmost nonzero of its residual against all earlier pivots.  Its output
// is unique: the pivots are the rank profile matrix (RPM) of Y, row_perm =
// pivot rows ascending then the rest ascending, col_perm = pivot columns in
// pivot order then the rest ascending, and [L1;M1], d, [U1 V1] are then
// determined (plduq.hpp:24-40).  This file computes the same thing in two
// phases:
//
//  1. Pivot search (the RPM), in row chunks of B rows:
//       R   = Y_c - Y_c[:, pc] * Uhat         residual against earlier pivots (GEMM)
//       S   = R * Omega                        random sketch, Omega n x (B+16)
//       I   = rows of S independent of the earlier rows of S   (1 CTA, tiny)
//       J   = column rank profile of R[I, :]   (parallel local scan + merge)
//       pairing = RPM of the k x k block R[I, J]  (1 CTA, tiny)
//     Rows of S independent => rows of R independent; the converse holds
//     unless Omega is degenerate on the row space of R, which the exact check
//     R - R[:, J] * (R[I,J]^-1 R[I,:]) == 0 rules out; on failure the chunk
//     is redone by the sequential kernel, so the result is always exact.
//     Uhat (rows fully reduced at their pivot columns) absorbs each chunk's
//     new rows by one GEMM.
//  2. Factors from the pivots: K = Y[pr, pc] = L1 D U1 (LDU without pivoting,
//     leading minors are the Crout pivots), U = D^-1 L1^-1 Y[pr, Q] and
//     M1 = Y[np, pc] U1^-1 D^-1 (TRSM + scaling).
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ffb_kernels.cuh"
#include "ffb_plduq.cuh"

namespace ffb {

namespace {

inline void count_launch() { ++g_launches; }

// dst[a][b] = src[ridx ? ridx[a] : a][cidx[b]]
__global__ void k_gather2d(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                           const int32_t* ridx, const int32_t* cidx, int64_t cols) {
    const int64_t a = blockIdx.y;
    const int64_t sr = ridx ? ridx[a] : a;
    const uint32_t* s = src + sr * lds;
    uint32_t* d = dst + a * ldd;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < cols;
         b += (int64_t)gridDim.x * blockDim.x)
        d[b] = s[cidx[b]];
}

__global__ void k_copy_rows(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                            int64_t cols) {
    const int64_t a = blockIdx.y;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < cols;
         b += (int64_t)gridDim.x * blockDim.x)
        dst[a * ldd + b] = src[a * lds + b];
}

__global__ void k_random(uint32_t* out, int64_t n, uint64_t seed, uint32_t p) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    out[i] = (uint32_t)umulhi64(z, p);
}

inline dim3 rgrid(int64_t rows, int64_t cols) {
    int64_t gx = cdiv(cols, 256);
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    return dim3((unsigned)gx, (unsigned)rows);
}

// ---------------------------------------------------------------------------
// Row detection on the sketch S (b x s, b <= 128, s <= 160), one CTA.
// Fully reduced basis: E_t with pivot column rho_t (E_t[rho_t] = 1, other
// basis rows 0 there).  Row i is independent iff its reduction is nonzero.
// out: out[0] = k, out[1..k] = independent rows (ascending).
// ---------------------------------------------------------------------------
constexpr int RD_MAX_B = 128;

__global__ void __launch_bounds__(256) k_row_detect(Fp f, const uint32_t* S, int64_t lds, int b,
                                                    int s, int32_t* out) {
    extern __shared__ uint32_t sm[];
    uint32_t* E = sm;                            // RD_MAX_B x s basis rows
    uint32_t* v = E + (size_t)RD_MAX_B * s;      // current row (s)
    __shared__ int rho[RD_MAX_B];
    __shared__ uint32_t coef[RD_MAX_B];
    __shared__ int kcount, firstnz;
    __shared__ uint32_t inv_lead;
    const int tid = threadIdx.x;
    if (tid == 0) kcount = 0;
    __syncthreads();
    for (int i = 0; i < b; ++i) {
        const int k = kcount;
        // v = S_i - sum_t S_i[rho_t] E_t
        for (int j = tid; j < s; j += blockDim.x) {
            uint64_t acc = 0;
            const uint32_t* si = S + (int64_t)i * lds;
            for (int t = 0; t < k; ++t) {
                acc += (uint64_t)si[rho[t]] * E[(size_t)t * s + j];
                if ((t & 15) == 15 && f.p >= (1u << 26)) acc = red64(f, acc);
            }
            v[j] = fsub(f, si[j], red64(f, acc));
        }
        if (tid == 0) firstnz = s;
        __syncthreads();
        for (int j = tid; j < s; j += blockDim.x)
            if (v[j] != 0) atomicMin(&firstnz, j);
        __syncthreads();
        const int rh = firstnz;
        __syncthreads();  // everyone has read firstnz before it is reset
        if (rh == s) continue;  // dependent row (uniform)
        if (tid == 0) inv_lead = finv(f, v[rh]);
        __syncthreads();
        const uint32_t il = inv_lead;
        for (int j = tid; j < s; j += blockDim.x) v[j] = fmul(f, v[j], il);
        __syncthreads();
        // eliminate column rh from the existing basis rows (coefficients are
        // snapshotted first: the update itself zeroes column rh), append v
        for (int t = tid; t < k; t += blockDim.x) coef[t] = E[(size_t)t * s + rh];
        __syncthreads();
        for (int e = tid; e < k * s; e += blockDim.x) {
            const int t = e / s, j = e % s;
            const uint32_t c = coef[t];
            if (c) E[(size_t)t * s + j] = fsub(f, E[(size_t)t * s + j], fmul(f, c, v[j]));
        }
        __syncthreads();
        for (int j = tid; j < s; j += blockDim.x) E[(size_t)k * s + j] = v[j];
        if (tid == 0) {
            rho[k] = rh;
            out[1 + k] = i;
            kcount = k + 1;
        }
        __syncthreads();
    }
    if (tid == 0) out[0] = kcount;
}

// ---------------------------------------------------------------------------
// Column rank profile (CRP) of RI (k x n) by a reduction tree.  Each CTA scans
// an ordered set of columns and keeps those independent of the earlier
// columns of the set (a local CRP).  A column dropped at any level depends on
// earlier columns, so it is dependent globally too, and the CRP of a union of
// surviving sets equals the CRP of the union of the underlying column ranges.
// Level 0 (range mode): CTA g scans columns [g*CRP_W, (g+1)*CRP_W).
// Level > 0 (list mode): CTA g scans the concatenation of input lists
// g*fan .. g*fan+fan-1 (each <= k columns, ascending).  Output: out[g*k + t],
// ocount[g].  The last level (one CTA) yields the CRP J.
// ---------------------------------------------------------------------------
constexpr int CRP_W = 256, CRP_G = 32, CRP_KMAX = 128, CRP_FAN = 8;

__global__ void __launch_bounds__(256) k_crp_list(Fp f, const uint32_t* RI, int64_t ldr, int k,
                                                  int64_t n, const int32_t* in, const int32_t* icount,
                                                  int nin, int32_t* out, int32_t* ocount) {
    extern __shared__ uint32_t sm[];
    uint32_t* E = sm;                           // basis: up to k vectors of length k
    uint32_t* V = E + (size_t)CRP_KMAX * k;     // CRP_G columns, each length k: V[c*k + i]
    __shared__ int rho[CRP_KMAX];
    __shared__ int colid[CRP_G];
    __shared__ int nb;
    __shared__ int nzmask[CRP_G];
    __shared__ int total, lead;
    __shared__ uint32_t vr[CRP_KMAX];
    __shared__ uint32_t coefs[CRP_KMAX];
    __shared__ uint32_t il;
    const int tid = threadIdx.x;
    const int g = blockIdx.x;
    // the ordered column set of this CTA
    auto column_at = [&](int idx) -> int {
        if (!in) return g * CRP_W + idx;
        int q = idx;
        for (int l = g * CRP_FAN; l < g * CRP_FAN + CRP_FAN && l < nin; ++l) {
            const int c = icount[l];
            if (q < c) return in[(int64_t)l * k + q];
            q -= c;
        }
        return -1;
    };
    if (tid == 0) {
        nb = 0;
        if (!in) {
            const int64_t c0 = (int64_t)g * CRP_W;
            total = (int)((c0 + CRP_W < n ? c0 + CRP_W : n) - c0);
        } else {
            int t = 0;
            for (int l = g * CRP_FAN; l < g * CRP_FAN + CRP_FAN && l < nin; ++l) t += icount[l];
            total = t;
        }
    }
    __syncthreads();
    for (int s0 = 0; s0 < total && nb < k; s0 += CRP_G) {
        const int gw = (s0 + CRP_G <= total) ? CRP_G : total - s0;
        if (tid < gw) colid[tid] = column_at(s0 + tid);
        if (tid < CRP_G) nzmask[tid] = 0;
        __syncthreads();
        for (int e = tid; e < gw * k; e += blockDim.x) {
            const int c = e % gw, i = e / gw;
            V[(size_t)c * k + i] = RI[(int64_t)i * ldr + colid[c]];
        }
        __syncthreads();
        // reduce every column of the group against the current basis; flag the
        // columns that stay nonzero (candidates for a new basis vector)
        const int kb = nb;
        for (int e = tid; e < gw * k; e += blockDim.x) {
            const int c = e / k, i = e % k;
            uint64_t acc = 0;
            for (int t = 0; t < kb; ++t) {
                acc += (uint64_t)V[(size_t)c * k + rho[t]] * E[(size_t)t * k + i];
                if ((t & 15) == 15 && f.p >= (1u << 26)) acc = red64(f, acc);
            }
            if (fsub(f, V[(size_t)c * k + i], red64(f, acc)) != 0) atomicOr(&nzmask[c], 1);
        }
        __syncthreads();
        // flagged columns in order: exact reduction against the current basis
        for (int c = 0; c < gw; ++c) {
            if (!nzmask[c]) continue;  // uniform (shared)
            const int kb2 = nb;
            for (int i = tid; i < k; i += blockDim.x) {
                uint64_t acc = 0;
                for (int t = 0; t < kb2; ++t) {
                    acc += (uint64_t)V[(size_t)c * k + rho[t]] * E[(size_t)t * k + i];
                    if ((t & 15) == 15 && f.p >= (1u << 26)) acc = red64(f, acc);
                }
                vr[i] = fsub(f, V[(size_t)c * k + i], red64(f, acc));
            }
            if (tid == 0) lead = k;
            __syncthreads();
            for (int i = tid; i < k; i += blockDim.x)
                if (vr[i]) atomicMin(&lead, i);
            __syncthreads();
            const int ld = lead;
            if (ld < k) {
                if (tid == 0) il = finv(f, vr[ld]);
                __syncthreads();
                for (int i = tid; i < k; i += blockDim.x) vr[i] = fmul(f, vr[i], il);
                __syncthreads();
                for (int t = tid; t < kb2; t += blockDim.x) coefs[t] = E[(size_t)t * k + ld];
                __syncthreads();
                for (int e = tid; e < kb2 * k; e += blockDim.x) {
                    const int t = e / k, i = e % k;
                    const uint32_t cc = coefs[t];
                    if (cc) E[(size_t)t * k + i] = fsub(f, E[(size_t)t * k + i], fmul(f, cc, vr[i]));
                }
                __syncthreads();
                for (int i = tid; i < k; i += blockDim.x) E[(size_t)kb2 * k + i] = vr[i];
                if (tid == 0) {
                    rho[kb2] = ld;
                    out[(int64_t)g * k + kb2] = colid[c];
                    nb = kb2 + 1;
                }
            }
            __syncthreads();
            if (nb >= k) break;
        }
        __syncthreads();
    }
    if (tid == 0) ocount[g] = nb;
}

// Append a chunk's pivots to the device bookkeeping: Uhat row order J,
// pivot rows c0 + I[t] with columns J[sigma[t]].
__global__ void k_append_pivots(int32_t* uhat_col, int32_t* prow, int32_t* pcol, int64_t r,
                                int64_t c0, const int32_t* I, const int32_t* J,
                                const int32_t* sigma, int k) {
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        uhat_col[r + t] = J[t];
        prow[r + t] = (int32_t)(c0 + I[t]);
        pcol[r + t] = J[sigma[t]];
    }
}

// ---------------------------------------------------------------------------
// Pairing + inverse (1 CTA): Kc = RI[:, J] (k x k, nonsingular).  Row-order
// leftmost elimination gives sigma (row t -> column sigma[t] of Kc); Gauss-
// Jordan gives Kinv.  out: sigma[k]; Kinv (k x k).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_pair(Fp f, const uint32_t* Kc, int64_t ldk, int k,
                                              int32_t* sigma, uint32_t* Kinv, int64_t ldi,
                                              int32_t* fail) {
    extern __shared__ uint32_t sm[];
    uint32_t* A = sm;                       // k x k working copy (row-order elimination)
    uint32_t* G = A + (size_t)k * k;        // k x 2k Gauss-Jordan
    __shared__ int colused[CRP_KMAX];
    __shared__ int lead;
    __shared__ uint32_t il;
    const int tid = threadIdx.x;
    for (int e = tid; e < k * k; e += blockDim.x) {
        const int i = e / k, j = e % k;
        const uint32_t v = Kc[(int64_t)i * ldk + j];
        A[e] = v;
        G[(size_t)i * 2 * k + j] = v;
        G[(size_t)i * 2 * k + k + j] = (i == j) ? 1 % f.p : 0;
    }
    for (int j = tid; j < k; j += blockDim.x) colused[j] = 0;
    __syncthreads();
    // row-order leftmost (the reference's Crout rule restricted to Kc)
    for (int t = 0; t < k; ++t) {
        if (tid == 0) lead = k;
        __syncthreads();
        for (int j = tid; j < k; j += blockDim.x)
            if (!colused[j] && A[(size_t)t * k + j] != 0) atomicMin(&lead, j);
        __syncthreads();
        const int jp = lead;
        if (jp == k) {  // cannot happen for a nonsingular Kc
            if (tid == 0) *fail = 1;
            return;
        }
        if (tid == 0) {
            sigma[t] = jp;
            colused[jp] = 1;
            il = finv(f, A[(size_t)t * k + jp]);
        }
        __syncthreads();
        // eliminate column jp from the rows below t
        for (int e = tid; e < (k - t - 1) * k; e += blockDim.x) {
            const int i = t + 1 + e / k, j = e % k;
            if (colused[j] && j != jp) continue;
            const uint32_t m = fmul(f, A[(size_t)i * k + jp], il);
            if (j == jp) continue;
            A[(size_t)i * k + j] = fsub(f, A[(size_t)i * k + j], fmul(f, m, A[(size_t)t * k + j]));
        }
        __syncthreads();
        for (int i = t + 1 + tid; i < k; i += blockDim.x) A[(size_t)i * k + jp] = 0;
        __syncthreads();
    }
    // Gauss-Jordan inverse (any nonzero pivot; result unique)
    const int w = 2 * k;
    for (int c = 0; c < k; ++c) {
        if (tid == 0) lead = k;
        __syncthreads();
        for (int i = c + tid; i < k; i += blockDim.x)
            if (G[(size_t)i * w + c] != 0) atomicMin(&lead, i);
        __syncthreads();
        const int pr = lead;
        if (pr == k) {
            if (tid == 0) *fail = 1;
            return;
        }
        if (pr != c)
            for (int j = tid; j < w; j += blockDim.x) {
                const uint32_t tmp = G[(size_t)c * w + j];
                G[(size_t)c * w + j] = G[(size_t)pr * w + j];
                G[(size_t)pr * w + j] = tmp;
            }
        __syncthreads();
        if (tid == 0) il = finv(f, G[(size_t)c * w + c]);
        __syncthreads();
        for (int j = tid; j < w; j += blockDim.x) G[(size_t)c * w + j] = fmul(f, G[(size_t)c * w + j], il);
        __syncthreads();
        for (int e = tid; e < k * w; e += blockDim.x) {
            const int i = e / w, j = e % w;
            if (i == c) continue;
            const uint32_t m = G[(size_t)i * w + c];
            if (m && j != c) G[(size_t)i * w + j] = fsub(f, G[(size_t)i * w + j], fmul(f, m, G[(size_t)c * w + j]));
        }
        __syncthreads();
        for (int i = tid; i < k; i += blockDim.x)
            if (i != c) G[(size_t)i * w + c] = 0;
        __syncthreads();
    }
    for (int e = tid; e < k * k; e += blockDim.x) {
        const int i = e / k, j = e % k;
        Kinv[(int64_t)i * ldi + j] = G[(size_t)i * w + k + j];
    }
}

// ---------------------------------------------------------------------------
// LDU without pivoting of a <= 64 x 64 block in place (1 CTA):
// strict lower <- L, diagonal <- d, strict upper <- U.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ldu_base(Fp f, uint32_t* K, int64_t ldk, int n,
                                                  int32_t* fail) {
    __shared__ uint32_t A[64][65];
    __shared__ uint32_t il;
    const int tid = threadIdx.x;
    for (int e = tid; e < n * n; e += blockDim.x) A[e / n][e % n] = K[(int64_t)(e / n) * ldk + e % n];
    __syncthreads();
    for (int t = 0; t < n; ++t) {
        if (tid == 0) {
            if (A[t][t] == 0) *fail = 1;
            il = A[t][t] ? finv(f, A[t][t]) : 0;
        }
        __syncthreads();
        const int w = n - t - 1;
        for (int e = tid; e < w * w; e += blockDim.x) {
            const int i = t + 1 + e / w, j = t + 1 + e % w;
            A[i][j] = fsub(f, A[i][j], fmul(f, fmul(f, A[i][t], il), A[t][j]));
        }
        __syncthreads();
        for (int i = t + 1 + tid; i < n; i += blockDim.x) {
            A[i][t] = fmul(f, A[i][t], il);  // L
            A[t][i] = fmul(f, A[t][i], il);  // U
        }
        __syncthreads();
    }
    for (int e = tid; e < n * n; e += blockDim.x) K[(int64_t)(e / n) * ldk + e % n] = A[e / n][e % n];
}

// L (unit lower with zeros above) from the packed LDU block; d from the diagonal.
__global__ void k_unpack_l(uint32_t* L, int64_t ldl, const uint32_t* K, int64_t ldk, int64_t n,
                           uint32_t* d, uint32_t one) {
    const int64_t i = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = K[i * ldk + j];
        L[i * ldl + j] = j < i ? v : (j == i ? one : 0);
        if (j == i) d[i] = v;
    }
}

}  // namespace

// ===========================================================================
// Host side
// ===========================================================================

void gather2d(cudaStream_t st, DMat dst, DMat src, const int32_t* ridx, const int32_t* cidx) {
    if (dst.rows <= 0 || dst.cols <= 0) return;
    ProfScope ps(K_MOVE, st, 0.0, 8.0 * dst.rows * dst.cols);
    for (int64_t r0 = 0; r0 < dst.rows; r0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, dst.rows - r0);
        k_gather2d<<<rgrid(nr, dst.cols), 256, 0, st>>>(dst.ptr + r0 * dst.ld, dst.ld, src.ptr, src.ld,
                                                        ridx ? ridx + r0 : nullptr, cidx, dst.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void copy_mat(cudaStream_t st, DMat dst, DMat src) {
    if (src.rows <= 0 || src.cols <= 0) return;
    ProfScope ps(K_MOVE, st, 0.0, 8.0 * src.rows * src.cols);
    if (dst.ld == src.ld && dst.ld == src.cols) {
        FFB_CUDA(cudaMemcpyAsync(dst.ptr, src.ptr, (size_t)src.rows * src.cols * 4,
                                 cudaMemcpyDeviceToDevice, st));
        return;
    }
    FFB_CUDA(cudaMemcpy2DAsync(dst.ptr, dst.ld * 4, src.ptr, src.ld * 4, src.cols * 4, src.rows,
                               cudaMemcpyDeviceToDevice, st));
}

// LDU without pivoting of K (n x n, in place), recursive.
void ldu_inplace(const Fp& f, cudaStream_t st, DMat K, Workspace& ws, int32_t* fail) {
    const int64_t n = K.rows;
    if (n <= 0) return;
    if (n <= 64) {
        ProfScope ps(K_PLDUQ, st, 2.0 * n * n * n / 3.0, 8.0 * n * n);
        k_ldu_base<<<1, 256, 0, st>>>(f, K.ptr, K.ld, (int)n, fail);
        count_launch();
        FFB_CHECK_LAUNCH();
        return;
    }
    int64_t n1 = (n / 2) / 64 * 64;
    if (n1 < 64) n1 = 64;
    const int64_t n2 = n - n1;
    DMat K11 = K.sub(0, 0, n1, n1), K12 = K.sub(0, n1, n1, n2), K21 = K.sub(n1, 0, n2, n1),
         K22 = K.sub(n1, n1, n2, n2);
    ldu_inplace(f, st, K11, ws, fail);
    const size_t mk = ws.mark();
    uint32_t* dinv = ws.vec<uint32_t>(n1);
    uint32_t* d = ws.vec<uint32_t>(n1);
    DMat L11 = ws.mat(n1, n1);
    k_unpack_l<<<rgrid(n1, n1), 256, 0, st>>>(L11.ptr, L11.ld, K11.ptr, K11.ld, n1, d, 1 % f.p);
    count_launch();
    invert_vec(f, st, dinv, d, n1);
    // U12 = D1^-1 L11^-1 K12 (in place)
    trsm_lower_unit(f, st, L11, K12);
    scale_rows(f, st, K12, K12, dinv);
    // Z = K21 U11^-1:  U11^T Z^T = K21^T
    DMat Zt = ws.mat(n1, n2);
    transpose(st, Zt, K21);
    DMat U11t = ws.mat(n1, n1);
    transpose(st, U11t, K11);  // strict lower of U11t = U11^T (strict upper of K11)
    trsm_lower_unit(f, st, U11t, Zt);
    // Schur complement: K22 - L21 D1 U12 = K22 - Z U12
    gemm(f, st, GEMM_SUB, K22, Zt, true, K12, false, n2, n2, n1);
    // L21 = Z D1^-1
    scale_T(f, st, K21, Zt, dinv);
    ws.release(mk);
    ldu_inplace(f, st, K22, ws, fail);
}

PlduqOut plduq_parallel(const Fp& f, cudaStream_t st, DMat Y, Workspace& ws, const PlduqIO& io) {
    const int64_t m = Y.rows, n = Y.cols, mn = std::min(m, n);
    const int B = 128, SK = B + 16;
    PlduqOut out;
    DMat Uhat = ws.mat(std::max<int64_t>(mn, 1), n);
    DMat Om = ws.mat(n, SK);
    {
        k_random<<<(unsigned)cdiv(n * SK, 256), 256, 0, st>>>(Om.ptr, n * SK, 0x5EEDull + n, f.p);
        count_launch();
    }
    DMat R = ws.mat(B, n), S = ws.mat(B, SK), RI = ws.mat(B, n), Unew = ws.mat(B, n);
    DMat Kc = ws.mat(B, B), Kinv = ws.mat(B, B), G = ws.mat(B, std::max<int64_t>(mn, 1));
    DMat Gc = ws.mat(B, B), Upd = ws.mat(std::max<int64_t>(mn, 1), B);
    const int nblk0 = (int)cdiv(n, CRP_W);
    int32_t* dinfo = ws.vec<int32_t>(2 * B + 16);     // row detect: k, I[0..k)
    int32_t* lists[2] = {ws.vec<int32_t>((int64_t)nblk0 * B), ws.vec<int32_t>((int64_t)nblk0 * B)};
    int32_t* counts[2] = {ws.vec<int32_t>(nblk0), ws.vec<int32_t>(nblk0)};
    int32_t* dsig = ws.vec<int32_t>(B);
    int32_t* dflag = ws.vec<int32_t>(4);              // sticky: any chunk failed its exact check
    int32_t* d_uhat_col = ws.vec<int32_t>(std::max<int64_t>(mn, 1));
    int32_t* d_prow = ws.vec<int32_t>(std::max<int64_t>(mn, 1));
    int32_t* d_pcol = ws.vec<int32_t>(std::max<int64_t>(mn, 1));

    const size_t rd_smem = ((size_t)RD_MAX_B * SK + SK) * 4;
    const size_t crp_smem = ((size_t)CRP_KMAX * CRP_KMAX + (size_t)CRP_G * CRP_KMAX) * 4;
    static bool attrs = false;
    if (!attrs) {
        FFB_CUDA(cudaFuncSetAttribute(k_row_detect, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rd_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_crp_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)crp_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * CRP_KMAX * CRP_KMAX * 4)));
        attrs = true;
    }
    static const bool force_exact = getenv("FFB_PLDUQ_FORCE_FALLBACK") != nullptr;  // test hook

    // Residual of chunk rows [c0, c0+bc) against the r pivots found so far.
    auto residual = [&](DMat Rc, DMat Yc, int64_t bc, int64_t r) {
        {
            ProfScope ps(K_MOVE, st, 0.0, 8.0 * bc * n);
            k_copy_rows<<<rgrid(bc, n), 256, 0, st>>>(Rc.ptr, Rc.ld, Yc.ptr, Yc.ld, n);
            count_launch();
        }
        if (r > 0) {
            DMat Gv = G.sub(0, 0, bc, r);
            gather2d(st, Gv, Yc, nullptr, d_uhat_col);
            gemm(f, st, GEMM_SUB, Rc, Gv, false, Uhat.sub(0, 0, r, n), false, bc, n, r);
        }
    };
    // Given the chunk's pivot rows (device dI, k of them) and pivot column set
    // (device dJ, ascending) with the pairing dsig: Uhat absorbs the chunk.
    auto absorb = [&](DMat Rc, int64_t bc, int64_t r, int k, const int32_t* dI, const int32_t* dJ,
                      bool verify, int64_t c0) {
        DMat RIk = RI.sub(0, 0, k, n), Un = Unew.sub(0, 0, k, n);
        DMat Kck = Kc.sub(0, 0, k, k), Kik = Kinv.sub(0, 0, k, k);
        gather2d(st, Kck, RIk, nullptr, dJ);
        {
            ProfScope ps(K_PLDUQ, st, 0.0, 0.0);
            k_pair<<<1, 256, (size_t)3 * k * k * 4, st>>>(f, Kck.ptr, Kck.ld, k, dsig, Kik.ptr,
                                                          Kik.ld, dflag);
            count_launch();
            FFB_CHECK_LAUNCH();
        }
        gemm(f, st, GEMM_SET, Un, Kik, false, RIk, false, k, n, k);  // Unew = Kc^-1 R_I
        if (verify) {  // exact check: R - R[:, J] Unew == 0 (sticky flag)
            DMat Gck = Gc.sub(0, 0, bc, k);
            gather2d(st, Gck, Rc, nullptr, dJ);
            gemm(f, st, GEMM_SUB, Rc, Gck, false, Un, false, bc, n, k);
            any_nonzero(st, Rc, dflag);
        }
        if (r > 0) {  // Uhat_old -= Uhat_old[:, J] Unew
            DMat Up = Upd.sub(0, 0, r, k);
            gather2d(st, Up, Uhat.sub(0, 0, r, n), nullptr, dJ);
            gemm(f, st, GEMM_SUB, Uhat.sub(0, 0, r, n), Up, false, Un, false, r, n, k);
        }
        copy_mat(st, Uhat.sub(r, 0, k, n), Un);
        k_append_pivots<<<1, 128, 0, st>>>(d_uhat_col, d_prow, d_pcol, r, c0, dI, dJ, dsig, k);
        count_launch();
    };

    int64_t r = 0;
    bool exact = force_exact;
    for (int attempt = 0; attempt < 2; ++attempt) {
        r = 0;
        FFB_CUDA(cudaMemsetAsync(dflag, 0, 4, st));
        for (int64_t c0 = 0; c0 < m; c0 += B) {
            const int64_t bc = std::min<int64_t>(B, m - c0);
            DMat Yc = Y.sub(c0, 0, bc, n), Rc = R.sub(0, 0, bc, n);
            residual(Rc, Yc, bc, r);
            if (!exact) {
                // pivot rows from the sketch
                DMat Sc = S.sub(0, 0, bc, SK);
                gemm(f, st, GEMM_SET, Sc, Rc, false, Om, false, bc, SK, n);
                {
                    ProfScope ps(K_PLDUQ, st, 0.0, 0.0);
                    k_row_detect<<<1, 256, rd_smem, st>>>(f, Sc.ptr, Sc.ld, (int)bc, SK, dinfo);
                    count_launch();
                    FFB_CHECK_LAUNCH();
                }
                const int k = *(const int32_t*)io.readback(dinfo, 4);
                if (k == 0) {
                    any_nonzero(st, Rc, dflag);  // the chunk must be entirely dependent
                    continue;
                }
                const int32_t* dI = dinfo + 1;
                gather_rows(st, RI.sub(0, 0, k, n), Rc, dI);
                // pivot column set: CRP reduction tree
                {
                    ProfScope ps(K_PLDUQ, st, 0.0, 0.0);
                    k_crp_list<<<nblk0, 256, crp_smem, st>>>(f, RI.ptr, RI.ld, k, n, nullptr, nullptr,
                                                             0, lists[0], counts[0]);
                    count_launch();
                    int groups = nblk0, cur = 0;
                    while (groups > 1) {
                        const int ng = (groups + CRP_FAN - 1) / CRP_FAN;
                        k_crp_list<<<ng, 256, crp_smem, st>>>(f, RI.ptr, RI.ld, k, n, lists[cur],
                                                              counts[cur], groups, lists[cur ^ 1],
                                                              counts[cur ^ 1]);
                        count_launch();
                        groups = ng;
                        cur ^= 1;
                    }
                    FFB_CHECK_LAUNCH();
                    absorb(Rc, bc, r, k, dI, lists[cur], true, c0);
                }
                r += k;
            } else {
                // Exact row-order kernel on a copy of the residual.
                const size_t mk = ws.mark();
                DMat Rw = ws.mat(bc, n);
                copy_mat(st, Rw, Rc);
                int32_t* info = ws.vec<int32_t>(1 + bc + n + bc);
                int32_t* colflag = ws.vec<int32_t>(n);
                uint32_t* lvec = ws.vec<uint32_t>(bc);
                DMat Lo = ws.mat(bc, std::min<int64_t>(bc, n)), Uo = ws.mat(std::min<int64_t>(bc, n), n);
                uint32_t* dd = ws.vec<uint32_t>(bc);
                plduq(f, st, Rw, info, colflag, lvec, Lo, dd, Uo);
                const int32_t* hi = (const int32_t*)io.readback(info, (size_t)(1 + bc + n + bc) * 4);
                const int k = hi[0];
                std::vector<int32_t> I(hi + 1, hi + 1 + k);
                std::vector<int32_t> J(hi + 1 + bc + n, hi + 1 + bc + n + k);
                std::sort(J.begin(), J.end());
                ws.release(mk);
                if (k == 0) continue;
                const int32_t* dI = io.upload(I);
                gather_rows(st, RI.sub(0, 0, k, n), Rc, dI);
                absorb(Rc, bc, r, k, dI, io.upload(J), false, c0);
                r += k;
            }
        }
        if (exact) break;
        if (*(const int32_t*)io.readback(dflag, 4) == 0) break;
        ++out.fallbacks;  // the sketch missed rank somewhere: redo exactly
        exact = true;
    }
    std::vector<int32_t> pr, pcol_rows;
    if (r > 0) {
        const int32_t* hp = (const int32_t*)io.readback(d_prow, (size_t)r * 4);
        pr.assign(hp, hp + r);
        const int32_t* hc = (const int32_t*)io.readback(d_pcol, (size_t)r * 4);
        pcol_rows.assign(hc, hc + r);
    }

    // ---- phase 2: factors from the pivots ----
    out.r = r;
    std::vector<char> isp(n, 0), isr(m, 0);
    for (int64_t t = 0; t < r; ++t) {
        isp[pcol_rows[t]] = 1;
        isr[pr[t]] = 1;
    }
    out.rimg = pr;
    for (int64_t i = 0; i < m; ++i)
        if (!isr[i]) out.rimg.push_back((int32_t)i);
    out.cimg = pcol_rows;
    for (int64_t j = 0; j < n; ++j)
        if (!isp[j]) out.cimg.push_back((int32_t)j);
    if (r == 0) return out;
    FFB_CUDA(cudaMemsetAsync(dflag, 0, 4, st));
    DMat Kf = ws.mat(r, r);
    const int32_t* dpr = io.upload(pr);
    const int32_t* dpc = io.upload(pcol_rows);
    gather2d(st, Kf, Y, dpr, dpc);
    ldu_inplace(f, st, Kf, ws, dflag);
    // L1 into Lo rows [0, r), d
    k_unpack_l<<<rgrid(r, r), 256, 0, st>>>(io.Lo.ptr, io.Lo.ld, Kf.ptr, Kf.ld, r, io.d, 1 % f.p);
    count_launch();
    invert_vec(f, st, io.dinv, io.d, r);
    // U = D^-1 L1^-1 Y[pr, Q]
    DMat Uo = io.Uo.sub(0, 0, r, n);
    gather2d(st, Uo, Y, dpr, io.upload(out.cimg));
    trsm_lower_unit(f, st, io.Lo.sub(0, 0, r, r), Uo);
    scale_rows(f, st, Uo, Uo, io.dinv);
    // M1 = Y[np, pc] U1^-1 D^-1
    if (m > r) {
        std::vector<int32_t> np(out.rimg.begin() + r, out.rimg.end());
        DMat T = ws.mat(m - r, r), Tt = ws.mat(r, m - r), U1t = ws.mat(r, r);
        gather2d(st, T, Y, io.upload(np), dpc);
        transpose(st, Tt, T);
        transpose(st, U1t, Uo.sub(0, 0, r, r));
        trsm_lower_unit(f, st, U1t, Tt);
        scale_T(f, st, io.Lo.sub(r, 0, m - r, r), Tt, io.dinv);
    }
    if (*(const int32_t*)io.readback(dflag, 4)) throw Status(FFB_ERROR, "plduq: singular pivot block");
    return out;
}

}  // namespace ffb
