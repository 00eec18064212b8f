// ffb_plduq.cu -- parallel rank-profile-revealing PLDUQ (plduq.cpp:36-123).
//
// The reference's PLDUQ is a row-sequential Crout: row i's pivot is the
// leftmost nonzero of its residual against all earlier pivots.  Its output
// is unique: the pivots are the rank profile matrix (RPM) of Y, row_perm =
// pivot rows ascending then the rest ascending, col_perm = pivot columns in
// pivot order then the rest ascending, and [L1;M1], d, [U1 V1] are then
// determined (plduq.hpp:24-40).  Two phases:
//
//  1. Pivot search (the RPM) in row chunks of B rows, against a basis Uhat of
//     the pivot rows found so far (each row 1 at its own pivot column, 0 at
//     the others):
//       S   = (Y Omega)_c - Y_c[:, pc] (Uhat Omega)   sketch of the chunk residual
//       I   = rows of S independent of the earlier rows of S      (1 CTA)
//       R_I = Y_I - Y_I[:, pc] Uhat                   exact residual of those rows
//       J   = column rank profile of R_I              (reduction tree of local CRPs)
//       pairing = RPM of R_I[:, J]; Unew = R_I[:,J]^-1 R_I joins Uhat (GEMMs)
//     Y Omega is computed once; Uhat Omega is maintained alongside Uhat.
//  2. Factors from the pivots: K = Y[pr, pc] = L1 D U1 (LDU without pivoting),
//     U = D^-1 L1^-1 Y[pr, Q], M1 = Y[np, pc] U1^-1 D^-1.
//
// Exactness (Las Vegas): a sketch can only MISS rank (rows of S independent
// => rows of R independent).  A miss makes the result either fail to
// reproduce Y or contain a pivotless row that depends on a LATER pivot row,
// so the certificate  P [L1;M1] D [U1 V1] Q^T == Y  and  M1(t,k) == 0 for
// pr_k > t  (plus nonzero LDU pivots) accepts exactly the reference's output.
// On rejection (probability ~ p^-16 per chunk) the search is redone with the
// exact row-sequential kernel.
#include <climits>
#include <type_traits>
#include <stdlib.h>

#include <algorithm>
#include <functional>
#include <vector>

#include "ffb_kernels.cuh"
#include "ffb_plduq.cuh"

namespace ffb {

namespace {

inline void count_launch() { ++g_launches; }

// dst[a][b] = src[roff + (ridx ? ridx[a] : a)][cidx[b]]
__global__ void k_gather2d(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                           const int32_t* ridx, int64_t roff, const int32_t* cidx, int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t a = blockIdx.y;
    const int64_t sr = roff + (ridx ? ridx[a] : a);
    const uint32_t* s = src + sr * lds;
    uint32_t* d = dst + a * ldd;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < cols;
         b += (int64_t)gridDim.x * blockDim.x)
        d[b] = s[cidx[b]];
}

// rows [0, rows) of src into dst (grid.y = row, grid-stride columns)
__global__ void k_copy_rows(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds, int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t a = blockIdx.y;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < cols; b += (int64_t)gridDim.x * blockDim.x)
        dst[a * ldd + b] = __ldcg(src + a * lds + b);
}

__global__ void k_random(uint32_t* out, int64_t n, uint64_t seed, uint32_t p) {
    FFB_PDL_ENTRY();
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
// Row detection on the sketch S (b x s, b <= 128, s <= 160), one CTA, S in
// shared memory.  Fully reduced basis E_t with pivot position rho_t.  A
// dependent row costs one barrier (__syncthreads_or); an independent row is
// normalised and eliminated from the basis.  The pivot position of a basis
// vector is arbitrary (any nonzero entry), only independence matters.
// out: out[0] = k, out[1..k] = independent rows (ascending).
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Batch reduction against a fully reduced basis (row detection and CRP):
//   X[r][j] = X0[r][j] - sum_{t<kb} CF[r][t] E[t][j]   (r < nr <= 32, j < len <= 32 NQ)
// and bit r of *mask is set when row r stays nonzero.  Warp w owns the row
// pairs (2w, 2w+1), (2w+2nw, ...); lane l the components l + 32q, so every
// thread keeps 2 NQ independent accumulators and each E load feeds two MACs.
// MODE 0: 32-bit lazy sums (kb p^2 < 2^31), 1: 64-bit lazy (p < 2^26), 2: reduce per term.
// X may alias X0 (each element is read and written by the same thread).
// ---------------------------------------------------------------------------
template <int NQ, int MODE>
__device__ __forceinline__ void reduce_rows(const Fp& f, uint32_t* X, int ldx, const uint32_t* X0,
                                            int ldx0, const uint32_t* CF, int ldcf,
                                            const uint32_t* E, int lde, int nr, int len, int kb,
                                            unsigned* mask) {
    using Acc = typename std::conditional<MODE == 0, uint32_t, uint64_t>::type;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int ra = 2 * wp; ra < nr; ra += 2 * nw) {
        const int rb = ra + 1;
        const bool hb = rb < nr;
        Acc a0[NQ], a1[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) a0[q] = a1[q] = 0;
        const uint32_t* cfa = CF + (size_t)ra * ldcf;
        const uint32_t* cfb = CF + (size_t)(hb ? rb : ra) * ldcf;
        for (int t = 0; t < kb; ++t) {
            const uint32_t ca = cfa[t], cb = cfb[t];
            const uint32_t* et = E + (size_t)t * lde;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int j = lane + 32 * q;
                const uint32_t e = j < len ? et[j] : 0u;
                if (MODE == 2) {
                    a0[q] = red64(f, (uint64_t)a0[q] + (uint64_t)ca * e);
                    a1[q] = red64(f, (uint64_t)a1[q] + (uint64_t)cb * e);
                } else {
                    a0[q] += (Acc)ca * e;
                    a1[q] += (Acc)cb * e;
                }
            }
        }
        int nza = 0, nzb = 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int j = lane + 32 * q;
            if (j < len) {
                const uint32_t xa = fsub(f, X0[(size_t)ra * ldx0 + j],
                                         MODE == 0 ? red32(f, (uint32_t)a0[q]) : red64(f, (uint64_t)a0[q]));
                X[(size_t)ra * ldx + j] = xa;
                nza |= xa != 0;
                if (hb) {
                    const uint32_t xb = fsub(f, X0[(size_t)rb * ldx0 + j],
                                             MODE == 0 ? red32(f, (uint32_t)a1[q]) : red64(f, (uint64_t)a1[q]));
                    X[(size_t)rb * ldx + j] = xb;
                    nzb |= xb != 0;
                }
            }
        }
        nza = __any_sync(0xffffffffu, nza);
        nzb = __any_sync(0xffffffffu, nzb);
        if (lane == 0 && (nza || nzb)) atomicOr(mask, (nza ? 1u << ra : 0u) | (nzb ? 1u << rb : 0u));
    }
}
template <int NQ>
__device__ __forceinline__ void reduce_rows_any(const Fp& f, uint32_t* X, int ldx, const uint32_t* X0,
                                                int ldx0, const uint32_t* CF, int ldcf,
                                                const uint32_t* E, int lde, int nr, int len, int kb,
                                                unsigned* mask) {
    if (f.p < 4096u && kb <= 128)
        reduce_rows<NQ, 0>(f, X, ldx, X0, ldx0, CF, ldcf, E, lde, nr, len, kb, mask);
    else if (f.p < (1u << 26))
        reduce_rows<NQ, 1>(f, X, ldx, X0, ldx0, CF, ldcf, E, lde, nr, len, kb, mask);
    else
        reduce_rows<NQ, 2>(f, X, ldx, X0, ldx0, CF, ldcf, E, lde, nr, len, kb, mask);
}

constexpr int RD_MAX_B = 128, RD_S = 144;
constexpr int RD_NARROW = 64;  // sketch columns of the first row-detection pass
constexpr int RD_MAX_ROWS = 640;  // chunk rows of a narrow row detection (adaptive chunks)
static const bool rd_narrow_on = getenv("FFB_RD_WIDE") == nullptr;  // A/B hook

constexpr int RD_BATCH = 16;
// pipelined detection: chunks of B rows whose predecessor found <= PIPE_KMAX rows; the
// stacked detection is trusted up to PIPE_TRUST rows (a margin of RD_S - PIPE_TRUST sketch
// columns), above that the chunk is detected again serially
constexpr int PIPE_KMAX = 32, PIPE_TRUST = 64, RD_PIPE = 96;
__host__ __device__ inline size_t rd_smem_bytes(int b, int s) {
    return ((size_t)b * s + (size_t)std::min(b, s) * s + (size_t)RD_BATCH * s) * 4;
}
__host__ __device__ inline size_t rd_smem_bytes_pre(int b, int s) {  // with a pre-basis: s basis rows
    return ((size_t)b * s + (size_t)s * s + (size_t)RD_BATCH * s) * 4;
}

// Blocked insertion of the flagged vectors of a reduced batch into a fully
// reduced basis.  V holds nr <= 32 vectors (stride ldv, length len), each
// already reduced against E (kb rows of stride len, pivots rho); bits of
// `pend` mark the nonzero ones.  Pass 1 walks the flagged vectors in order:
// a vector still nonzero gets its leading entry as pivot, which is eliminated
// from the other live vectors of the batch only (one barrier per vector).
// Pass 2 applies all new pivots to the basis at once,
//   E <- E - E[:, piv] N   (N = normalised new vectors, coefficients by shuffle),
// and appends N.  Returns the count; ins[a] = batch index of the a-th new vector.
// At most kmax - kb vectors are inserted.  Uniform control flow; 256 threads.
// ---------------------------------------------------------------------------
struct BatchScratch {
    int ins[32];
    int piv[32];
    uint32_t il[32];
};
template <int NQ>
__device__ int batch_insert(const Fp& f, const SmemInv& inv, uint32_t* V, int ldv, unsigned pend,
                            int len, uint32_t* E, int kb, int kmax, int* rho, BatchScratch& bs) {
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    int cnt = 0;
    unsigned done = 0;
    while (pend && kb + cnt < kmax) {
        const int r = __ffs(pend) - 1;
        pend &= pend - 1;
        const uint32_t* v = V + (size_t)r * ldv;
        // leading entry, found by every warp with ballots (v is stable: the last
        // write to it was before the previous insertion's barrier)
        int rh = len;
#pragma unroll
        for (int qq = 0; qq < NQ; ++qq) {
            const int j = lane + 32 * qq;
            const unsigned bal = __ballot_sync(0xffffffffu, j < len && v[j] != 0);
            if (bal && rh == len) rh = 32 * qq + __ffs(bal) - 1;
        }
        if (rh >= len) continue;  // dependent on the vectors inserted before it (uniform)
        const uint32_t il = inv(f, v[rh]);
        {  // live batch vectors (inserted and pending): the rk-th one goes to warp rk mod 8
            const unsigned live = done | pend;
            const bool has = (live >> lane) & 1;
            const int rank = __popc(live & ((1u << lane) - 1));
            const int nlive = __popc(live);
            for (int rk = wp; rk < nlive; rk += 8) {
                const int q = __ffs(__ballot_sync(0xffffffffu, has && rank == rk)) - 1;
                uint32_t* dst = V + (size_t)q * ldv;
                const uint32_t c = dst[rh];
                __syncwarp();
                if (c) {
                    const uint32_t cn = fmul(f, c, il);
#pragma unroll
                    for (int qq = 0; qq < NQ; ++qq) {
                        const int j = lane + 32 * qq;
                        if (j < len) dst[j] = fmsub(f, dst[j], cn, v[j]);
                    }
                }
            }
        }
        if (tid == 0) {
            bs.ins[cnt] = r;
            bs.piv[cnt] = rh;
            bs.il[cnt] = il;
        }
        done |= 1u << r;
        ++cnt;
        __syncthreads();
    }
    if (cnt == 0) return 0;
    // pass 2: E <- E - E[:, piv] N, row t by warp t mod 8, lane a holds coefficient a
    const bool small = f.p < 4096u;
    for (int t = wp; t < kb; t += 8) {
        uint32_t* et = E + (size_t)t * len;
        const uint32_t ct = lane < cnt ? fmul(f, et[bs.piv[lane]], bs.il[lane]) : 0u;
        __syncwarp();
        uint64_t acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0;
        for (int a = 0; a < cnt; ++a) {
            const uint32_t ca = __shfl_sync(0xffffffffu, ct, a);
            if (!ca) continue;  // warp-uniform
            const uint32_t* na = V + (size_t)bs.ins[a] * ldv;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const int j = lane + 32 * q;
                const uint64_t prod = (uint64_t)ca * (j < len ? na[j] : 0u);
                acc[q] = small ? acc[q] + prod : (uint64_t)red64(f, acc[q] + prod);
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int j = lane + 32 * q;
            if (j < len) et[j] = fsub(f, et[j], red64(f, acc[q]));
        }
    }
    // append the normalised new vectors
    for (int a = wp; a < cnt; a += 8) {
        const uint32_t* na = V + (size_t)bs.ins[a] * ldv;
        const uint32_t il = bs.il[a];
        uint32_t* dst = E + (size_t)(kb + a) * len;
        for (int j = lane; j < len; j += 32) dst[j] = fmul(f, na[j], il);
    }
    if (tid < cnt) rho[kb + tid] = bs.piv[tid];
    __syncthreads();
    return cnt;
}

// Row rank profile of a b x s chunk sketch (b <= 128, s <= 160), 1 CTA.
// Batches of 16 rows are reduced against the basis in parallel; a row that
// reduces to zero lies in the span of earlier rows and is dependent for good,
// so only the flagged rows go through the sequential insertion.
// out[0] = k, out[1..k] = independent rows (ascending).
// Optional pre-basis (pipelined detection): kpre = *kpre_ptr fully reduced rows Epre
// (stride s) with pivots rho_pre are loaded first; rows are then detected modulo their
// span (k counts the new rows only).  Eout / rho_out (optional): the final basis.
template <int NQ>  // ceil(s / 32)
__global__ void __launch_bounds__(256) k_row_detect(Fp f, const uint32_t* S, int64_t lds, int b,
                                                    int s, int32_t* out, MboxPost mp, const uint32_t* Epre,
                                                    const int32_t* rho_pre, const int32_t* kpre_ptr, uint32_t* Eout,
                                                    int32_t* rho_out) {
    FFB_PDL_ENTRY();
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* Ss = sm;                          // b x s (b <= RD_MAX_ROWS)
    uint32_t* E = Ss + (size_t)b * s;           // basis rows (fully reduced), <= min(b, s)
    uint32_t* V = E + (size_t)(kpre_ptr ? s : std::min(b, s)) * s;  // RD_BATCH reduced rows of the current batch
    __shared__ int rho[RD_MAX_B];
    __shared__ uint32_t cfb[RD_BATCH][RD_MAX_B];  // batch coefficients S_i[rho_t]
    __shared__ unsigned fmask[2];
    __shared__ BatchScratch bs;
    __shared__ uint32_t sinv[SINV_MAX];
    __shared__ uint64_t bar;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    if (lds == s && bulk_ok(S, (size_t)b * s * 4))
        bulk_stage(Ss, S, (uint32_t)((size_t)b * s * 4), &bar);
    else
        load_tile<16>(Ss, s, S, lds, b, s);
    const SmemInv inv = stage_inverses(f, sinv);
    int k = 0, bi = 0;
    if (kpre_ptr) {
        k = min(__ldcg(kpre_ptr), min(s, RD_MAX_B));
        for (int e = tid; e < k * s; e += 256) E[e] = __ldcg(Epre + e);
        for (int t = tid; t < k; t += 256) rho[t] = __ldcg(rho_pre + t);
    }
    const int kp = k;
    __syncthreads();
    for (int i0 = 0; i0 < b; i0 += RD_BATCH, ++bi) {
        const int nr = min(RD_BATCH, b - i0);
        for (int r = wp; r < nr; r += 8)
            for (int t = lane; t < k; t += 32) cfb[r][t] = Ss[(size_t)(i0 + r) * s + rho[t]];
        if (tid == 0) fmask[bi & 1] = 0;
        __syncthreads();
        reduce_rows_any<NQ>(f, V, s, Ss + (size_t)i0 * s, s, &cfb[0][0], RD_MAX_B, E, s, nr, s, k,
                           &fmask[bi & 1]);
        __syncthreads();
        const unsigned pending = fmask[bi & 1];  // rows outside the span of the batch-start basis
        if (!pending) continue;
        const int cnt = batch_insert<NQ>(f, inv, V, s, pending, s, E, k, min(s, RD_MAX_B), rho, bs);
        if (tid < cnt) out[1 + k - kp + tid] = i0 + bs.ins[tid];  // inserted in row order
        k += cnt;
    }
    if (Eout) {
        for (int e = tid; e < k * s; e += 256) Eout[e] = E[e];
        for (int t = tid; t < k; t += 256) rho_out[t] = rho[t];
    }
    if (tid == 0) {
        const int kn = k - kp;
        out[0] = kn;
        if (mp.dst) mbox_publish(mp, &kn, 1);  // the host's read-back of k, without a k_post
    }
}

// ---------------------------------------------------------------------------
// Row rank profile, register-resident (p < 4096; same contract as k_row_detect).
// The stack [Epre; S] (kpre + b rows x s columns) lives in registers: warp w holds
// rows w + NW u (u < RU), lane l the columns l + 32 q (q < NQ), as lazy sums (< p +
// 128 p^2 < 2^32).  Rows are visited in rounds of NW (rows NW u .. NW u + NW - 1):
// every warp reduces its row of the round, one barrier publishes the nonzero flags,
// and the first nonzero row is the next pivot -- the pending rows before it are
// dependent for good (the span only grows).  A pivot step is right-looking: the
// owner normalizes its row at its first nonzero column and publishes it, one barrier,
// then every warp subtracts it from its later rows (and, when the basis is written
// out, from the earlier pivot rows: Gauss-Jordan, so Eout is fully reduced).  A
// round costs one barrier, a pivot two; no per-row insertion chain.
// ---------------------------------------------------------------------------
template <int NQ, int RU, int NW>
__global__ void __launch_bounds__(32 * NW) k_rrp(Fp f, const uint32_t* S, int64_t lds, int b, int s, int32_t* out,
                                                 MboxPost mp, const uint32_t* Epre, const int32_t* kpre_ptr,
                                                 uint32_t* Eout, int32_t* rho_out) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ uint32_t sinv[SINV_MAX];
    __shared__ __align__(16) uint32_t prow[2][32 * NQ];
    __shared__ int tflag[2][NW];
    __shared__ int pcol_s[2];
    __shared__ int16_t rho_s[RD_MAX_B], tof[RU * NW];
    const SmemInv inv = stage_inverses(f, sinv);  // independent of the predecessor
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int kpre = kpre_ptr ? min(__ldcg(kpre_ptr), min(s, RD_MAX_B)) : 0;
    const int nrows = min(kpre + b, RU * NW);
    uint32_t v[RU][NQ];
#pragma unroll
    for (int u = 0; u < RU; ++u) {
        const int i = NW * u + wp;
        const uint32_t* src = i < kpre ? Epre + (int64_t)i * s : S + (int64_t)(i - kpre) * lds;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int c = lane + 32 * q;
            v[u][q] = (i < nrows && c < s) ? __ldcg(src + c) : 0u;
        }
    }
    const bool gj = Eout != nullptr;  // Gauss-Jordan: earlier pivot rows take the updates too
    uint32_t ispiv = 0;               // bit u: this warp's row of round u is a pivot (warp-uniform)
    int k = 0, kn = 0, tb = 0, pb = 0;
    for (int u = 0; u < RU; ++u) {
        const int base = NW * u;
        if (base >= nrows) break;
        unsigned pend = nrows - base >= NW ? (NW == 32 ? 0xffffffffu : (1u << NW) - 1u) : (1u << (nrows - base)) - 1u;
        // the round's row lives in cur[] while the round runs (rows v[u] is stale until written back)
        uint32_t cur[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            uint32_t x = v[0][q];
#pragma unroll
            for (int uu = 1; uu < RU; ++uu) x = uu == u ? v[uu][q] : x;
            cur[q] = x;
        }
        while (pend) {
            bool nz = false;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                cur[q] = red32(f, cur[q]);
                nz |= cur[q] != 0;
            }
            nz = __any_sync(0xffffffffu, nz);
            if (lane == 0) tflag[tb][wp] = nz;
            __syncthreads();
            const unsigned nzm =
                __ballot_sync(0xffffffffu, lane < NW && ((pend >> lane) & 1) && tflag[tb][lane & (NW - 1)]);
            tb ^= 1;
            if (!nzm) break;  // every pending row of the round is dependent
            const int ws = __ffs(nzm) - 1;
            pend &= ~((2u << ws) - 1u);
            if (wp == ws) {  // normalize the pivot row at its first nonzero column, publish it
                int cq = NQ;
                unsigned bl = 0;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const unsigned bq = __ballot_sync(0xffffffffu, cur[q] != 0);
                    if (cq == NQ && bq) {
                        cq = q;
                        bl = bq;
                    }
                }
                const int cl = __ffs(bl) - 1;
                uint32_t xp = cur[0];
#pragma unroll
                for (int q = 1; q < NQ; ++q) xp = q == cq ? cur[q] : xp;
                const uint32_t il = inv(f, __shfl_sync(0xffffffffu, xp, cl));
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    cur[q] = red32(f, cur[q] * il);
                    prow[pb][lane + 32 * q] = cur[q];
                }
                if (lane == 0) {
                    pcol_s[pb] = 32 * cq + cl;
                    rho_s[k] = (int16_t)(32 * cq + cl);
                    tof[base + ws] = (int16_t)k;
                }
                ispiv |= 1u << u;
            }
            __syncthreads();
            const int col = pcol_s[pb], cq = col >> 5, cl = col & 31;
            uint32_t pr[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) pr[q] = prow[pb][lane + 32 * q];
            pb ^= 1;
            // rows of later rounds, and (Gauss-Jordan) earlier pivot rows: branch-free, a masked
            // row adds 0; an unmasked row with a zero multiplier adds p * pr (= 0 mod p)
            const uint32_t later = u + 1 < RU ? ~0u << (u + 1) : 0u;
            const uint32_t upd = later | (gj ? ispiv & ~(1u << u) : 0u);
#pragma unroll
            for (int uu = 0; uu < RU; ++uu) {
                uint32_t mv = v[uu][0];
#pragma unroll
                for (int q = 1; q < NQ; ++q) mv = q == cq ? v[uu][q] : mv;
                const uint32_t mn = ((upd >> uu) & 1) ? f.p - red32(f, __shfl_sync(0xffffffffu, mv, cl)) : 0u;
#pragma unroll
                for (int q = 0; q < NQ; ++q) v[uu][q] += mn * pr[q];
            }
            {  // this round's rows after the pivot (and, Gauss-Jordan, a pivot row of this round)
                uint32_t mv = cur[0];
#pragma unroll
                for (int q = 1; q < NQ; ++q) mv = q == cq ? cur[q] : mv;
                const bool on = wp > ws || (gj && ((ispiv >> u) & 1) && wp != ws);
                const uint32_t mn = on ? f.p - red32(f, __shfl_sync(0xffffffffu, mv, cl)) : 0u;
#pragma unroll
                for (int q = 0; q < NQ; ++q) cur[q] += mn * pr[q];
            }
            if (base + ws >= kpre) {
                if (tid == 0) out[1 + kn] = base + ws - kpre;
                ++kn;
            }
            ++k;
        }
#pragma unroll
        for (int uu = 0; uu < RU; ++uu)
            if (uu == u)
#pragma unroll
                for (int q = 0; q < NQ; ++q) v[uu][q] = cur[q];
    }
    if (Eout) {  // the pivot rows, fully reduced, in pivot order
#pragma unroll
        for (int uu = 0; uu < RU; ++uu)
            if ((ispiv >> uu) & 1) {
                const int t = tof[NW * uu + wp];
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int c = lane + 32 * q;
                    if (c < s) Eout[(int64_t)t * s + c] = red32(f, v[uu][q]);
                }
            }
        for (int t = tid; t < k; t += blockDim.x) rho_out[t] = rho_s[t];
    }
    if (tid == 0) {
        out[0] = kn;
        if (mp.dst) mbox_publish(mp, &kn, 1);
    }
}

// ---------------------------------------------------------------------------
// Row rank profile, left-looking rounds (p < 4096; same contract as k_row_detect with
// rho_pre as the pre-basis pivots).  The basis E lives in shared memory, normalized and
// fully reduced (Gauss-Jordan): the coefficients of a row against it are the row's own
// entries at the pivot columns, so a row is reduced against all k basis rows without a
// dependency chain -- lane t takes coefficient t from the warp's copy of the row, the
// loop over t is shuffles and multiply-adds.  Rows are visited in rounds of NW (one row
// per warp, the next round's row prefetched): reduce, one barrier for the nonzero flags;
// the first nonzero pending row is a pivot (the pending rows before it are dependent for
// good).  A pivot step touches only the round's later pending rows and the basis (row t
// of E by warp t mod NW), two barriers.  A pre-basis costs no pivot steps at all.
// kcap > 0: stop after kcap new rows; out[0] then carries the rows consumed in bits 16..
// (the chunk is cut there: the fast CRP kernels take at most 32 rows).
// ---------------------------------------------------------------------------
template <int NQ>
__device__ __forceinline__ uint32_t reg_col(const uint32_t (&v)[NQ], int col, int lane) {
    uint32_t mv = v[0];
#pragma unroll
    for (int q = 1; q < NQ; ++q) mv = q == (col >> 5) ? v[q] : mv;
    return __shfl_sync(0xffffffffu, mv, col & 31);
}
template <int NQ, int NW>
__global__ void __launch_bounds__(32 * NW) k_rrp2(Fp f, const uint32_t* S, int64_t lds, int b, int s, int32_t* out,
                                                  MboxPost mp, const uint32_t* Epre, const int32_t* rho_pre,
                                                  const int32_t* kpre_ptr, uint32_t* Eout, int32_t* rho_out, int kcap) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    constexpr int W = 32 * NQ, KMAX = W < 128 ? W : 128, KS = KMAX / 32, SINV = 1024;
    __shared__ uint16_t E[KMAX][W];
    __shared__ uint16_t rowbuf[NW][W];
    __shared__ int16_t rho[KMAX];
    __shared__ int flag[2][NW];
    __shared__ int pcol_s[2];
    __shared__ uint32_t sinv[SINV];
    const SmemInv inv = f.p <= (uint32_t)SINV ? stage_inverses(f, sinv) : SmemInv{nullptr};
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int kpre = kpre_ptr ? min(__ldcg(kpre_ptr), min(s, KMAX)) : 0;
    for (int e = tid; e < kpre * W; e += 32 * NW) {
        const int t = e / W, c = e - t * W;
        E[t][c] = c < s ? (uint16_t)__ldcg(Epre + (int64_t)t * s + c) : (uint16_t)0;
    }
    for (int t = tid; t < kpre; t += 32 * NW) rho[t] = (int16_t)__ldcg(rho_pre + t);
    uint32_t nxt[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) nxt[q] = (wp < b && lane + 32 * q < s) ? __ldcg(S + (int64_t)wp * lds + lane + 32 * q) : 0u;
    __syncthreads();
    if (kcap <= 0) kcap = KMAX;
    int k = kpre, kn = 0, tb = 0, pb = 0, done = 0;
    for (int base = 0; base < b && k < KMAX && kn < kcap; base += NW) {
        const int i = base + wp;
        uint32_t cur[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            cur[q] = nxt[q];
            nxt[q] = (i + NW < b && lane + 32 * q < s) ? __ldcg(S + (int64_t)(i + NW) * lds + lane + 32 * q) : 0u;
        }
        if (k > 0) {  // cur -= sum_t cur[rho_t] E_t
#pragma unroll
            for (int q = 0; q < NQ; ++q) rowbuf[wp][lane + 32 * q] = (uint16_t)cur[q];
            __syncwarp();
            uint32_t cs[KS];
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int t = lane + 32 * j;
                const uint32_t c = t < k ? rowbuf[wp][rho[t]] : 0u;
                cs[j] = c ? f.p - c : 0u;
            }
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                const int kt = min(32, k - 32 * j);  // uniform
#pragma unroll 4
                for (int tt = 0; tt < kt; ++tt) {
                    const uint32_t c = __shfl_sync(0xffffffffu, cs[j], tt);
                    const uint16_t* er = E[32 * j + tt];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) cur[q] += c * er[lane + 32 * q];
                }
            }
            __syncwarp();
        }
        bool nz = false;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            cur[q] = red32(f, cur[q]);
            nz |= cur[q] != 0;
        }
        nz = __any_sync(0xffffffffu, nz);
        if (lane == 0) flag[tb][wp] = nz;
        __syncthreads();
        unsigned pend = b - base >= NW ? (NW == 32 ? 0xffffffffu : (1u << NW) - 1u) : (1u << (b - base)) - 1u;
        while (k < KMAX && kn < kcap) {
            const unsigned nzm = __ballot_sync(0xffffffffu, lane < NW && ((pend >> lane) & 1) && flag[tb][lane & (NW - 1)]);
            tb ^= 1;
            if (!nzm) break;  // every pending row of the round is dependent
            const int ws = __ffs(nzm) - 1, i_piv = base + ws;
            pend &= ~((2u << ws) - 1u);
            if (wp == ws) {  // normalize at the first nonzero column, append to the basis
                int cq = NQ;
                unsigned bl = 0;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const unsigned bq = __ballot_sync(0xffffffffu, cur[q] != 0);
                    if (cq == NQ && bq) {
                        cq = q;
                        bl = bq;
                    }
                }
                const int cl = __ffs(bl) - 1;
                uint32_t xp = cur[0];
#pragma unroll
                for (int q = 1; q < NQ; ++q) xp = q == cq ? cur[q] : xp;
                const uint32_t il = inv(f, __shfl_sync(0xffffffffu, xp, cl));
#pragma unroll
                for (int q = 0; q < NQ; ++q) E[k][lane + 32 * q] = (uint16_t)red32(f, cur[q] * il);
                if (lane == 0) {
                    pcol_s[pb] = 32 * cq + cl;
                    rho[k] = (int16_t)(32 * cq + cl);
                    out[1 + kn] = i;
                }
            }
            __syncthreads();
            const int col = pcol_s[pb];
            pb ^= 1;
            uint32_t en[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) en[q] = E[k][lane + 32 * q];
            if (wp > ws && ((pend >> wp) & 1)) {  // the round's later rows (warp-uniform)
                const uint32_t m = reg_col<NQ>(cur, col, lane);
                const uint32_t mn = m ? f.p - m : 0u;
                bool z = false;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    cur[q] = red32(f, cur[q] + mn * en[q]);
                    z |= cur[q] != 0;
                }
                z = __any_sync(0xffffffffu, z);
                if (lane == 0) flag[tb][wp] = z;
            }
            for (int t = wp; t < k; t += NW) {  // basis rows: E_t -= E_t[col] E_k
                const uint32_t m = E[t][col];
                __syncwarp();
                if (m) {
                    const uint32_t mn = f.p - m;
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        E[t][lane + 32 * q] = (uint16_t)red32(f, E[t][lane + 32 * q] + mn * en[q]);
                }
            }
            ++k;
            ++kn;
            if (kn == kcap) done = i_piv + 1;  // rows after the capped pivot stay for the next chunk
            __syncthreads();
        }
    }
    if (Eout) {  // the basis, fully reduced, in pivot order
        for (int e = tid; e < k * s; e += 32 * NW) {
            const int t = e / s, c = e - t * s;
            Eout[e] = E[t][c];
        }
        for (int t = tid; t < k; t += 32 * NW) rho_out[t] = rho[t];
    }
    if (tid == 0) {  // new rows found; bits 16..: rows consumed when the cap cut the chunk short, else 0
        const int word = kn | ((done > 0 && done < b) ? done << 16 : 0);
        out[0] = word;
        if (mp.dst) mbox_publish(mp, &word, 1);
    }
}

// ---------------------------------------------------------------------------
// Candidate columns for the column rank profile of RI (k x n): CTA g scans
// columns [g*CRP_W, (g+1)*CRP_W) in groups of CRP_G and keeps those
// independent of the earlier columns of its range (a local CRP).  A dropped
// column depends on earlier columns, so it is dependent globally too: the
// union of the kept lists contains the CRP J.  Output out[g*k + t], ocount[g].
// ---------------------------------------------------------------------------
constexpr int CRP_W = 256, CRP_G = 32, CRP_KMAX = 128;

// Column scan shared by the level-0 CTAs and the chunk finish: the columns
// colfn(0 .. total) of RI (in this order) are processed in groups of CRP_G
// (prefetched into registers one group ahead), each reduced against the basis
// E in parallel; the flagged ones go through the blocked insertion.  The ids
// of the independent columns are written to out[0 .. nb) in scan order.
// Stops once k columns are found.  E, V, VC: shared (see k_crp_list).
// NQ = ceil(k / 32): vector slots per lane (k <= 32 NQ), so short vectors do not pay
// for the 128-entry maximum (the instantiation is picked at run time).
template <int NQ, class ColFn>
__device__ int crp_scan(const Fp& f, const SmemInv& inv, const uint32_t* RI, int64_t ldr,
                        int k, int total, ColFn colfn, uint32_t* E, uint32_t* V, uint32_t* VC, int* rho,
                        unsigned* fmask, BatchScratch& bs, int32_t* out) {
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    constexpr int RU = 4 * NQ;  // rows per lane: wp + 8u, u < RU covers k <= 32 NQ
    uint32_t vv[RU];  // thread (wp, lane) holds rows wp + 8u of column lane of a group
    auto fetch = [&](int s0) {
        const bool ok = s0 + lane < total;
        const uint32_t* src = RI + (ok ? colfn(s0 + lane) : 0);
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int i = wp + 8 * u;
            vv[u] = (ok && i < k) ? __ldcg(src + (int64_t)i * ldr) : 0u;
        }
    };
    fetch(0);
    int nb = 0, gi = 0;
    for (int s0 = 0; s0 < total && nb < k; s0 += CRP_G, ++gi) {
        const int gw = min(CRP_G, total - s0);
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int i = wp + 8 * u;
            if (i < k) V[(size_t)lane * k + i] = vv[u];
        }
        if (s0 + CRP_G < total) fetch(s0 + CRP_G);  // overlaps this group's work
        if (tid == 0) fmask[gi & 1] = 0;
        __syncthreads();
        for (int c = wp; c < gw; c += 8)  // coefficients V[c][rho_t]
            for (int t = lane; t < nb; t += 32) VC[(size_t)c * CRP_KMAX + t] = V[(size_t)c * k + rho[t]];
        __syncthreads();
        // reduce the group against the basis; flagged columns are outside its span
        reduce_rows_any<NQ>(f, V, k, V, k, VC, CRP_KMAX, E, k, gw, k, nb, &fmask[gi & 1]);
        __syncthreads();
        const unsigned pending = fmask[gi & 1];
        if (!pending) continue;
        const int cnt = batch_insert<NQ>(f, inv, V, k, pending, k, E, nb, k, rho, bs);
        if (tid < cnt) out[nb + tid] = colfn(s0 + bs.ins[tid]);
        nb += cnt;
    }
    return nb;
}

#define FFB_CRP_SCAN(...)                                                 \
    (k <= 32 ? crp_scan<1>(__VA_ARGS__) : k <= 64 ? crp_scan<2>(__VA_ARGS__) \
             : k <= 96 ? crp_scan<3>(__VA_ARGS__) : crp_scan<4>(__VA_ARGS__))
__global__ void __launch_bounds__(256) k_crp_list(Fp f, const uint32_t* RI, int64_t ldr,
                                                  int k, int64_t n, int32_t* out, int32_t* ocount) {
    FFB_PDL_ENTRY();
    extern __shared__ uint32_t sm[];
    uint32_t* E = sm;                           // basis: up to k vectors of length k
    uint32_t* V = E + (size_t)CRP_KMAX * k;     // CRP_G columns, each length k: V[c*k + i]
    uint32_t* VC = V + (size_t)CRP_G * k;       // CRP_G x CRP_KMAX gathered coefficients
    __shared__ int rho[CRP_KMAX];
    __shared__ unsigned fmask[2];
    __shared__ BatchScratch bs;
    __shared__ uint32_t sinv[SINV_MAX];
    __shared__ int32_t nzc[CRP_W];  // the block's nonzero columns, ascending
    __shared__ int wcnt[CRP_W / 32];
    const int g = blockIdx.x;
    const int64_t c0 = (int64_t)g * CRP_W;
    const int total = (int)std::min<int64_t>(CRP_W, n - c0);
    const SmemInv inv = stage_inverses(f, sinv);
    // all-zero columns never enter the CRP: compact the nonzero ones (thread = column,
    // all k loads in flight), so the scan below visits only those
    {
        const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
        int nz = 0;
        if (t < total) {
            const uint32_t* col = RI + c0 + t;
            for (int i0 = 0; i0 < k; i0 += 16) {
                uint32_t v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = i0 + u < k ? __ldcg(col + (int64_t)(i0 + u) * ldr) : 0u;
#pragma unroll
                for (int u = 0; u < 16; ++u) nz |= v[u] != 0;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, nz);
        if (lane == 0) wcnt[wp] = __popc(bal);
        __syncthreads();
        int base = 0;
        for (int w = 0; w < wp; ++w) base += wcnt[w];
        if (nz) nzc[base + __popc(bal & ((1u << lane) - 1))] = (int32_t)(c0 + t);
        __syncthreads();
    }
    int cnt = 0;
    for (int w = 0; w < CRP_W / 32; ++w) cnt += wcnt[w];
    auto colfn = [&](int idx) { return nzc[idx]; };
    const int nb = FFB_CRP_SCAN(f, inv, RI, ldr, k, cnt, colfn, E, V, VC, rho, fmask, bs, out + (int64_t)g * k);
    if (threadIdx.x == 0) ocount[g] = nb;
}

// ---------------------------------------------------------------------------
// Local CRP of a 256-column block, register-resident (k <= K <= 32, p < 4096;
// same contract as k_crp_list).  Thread t owns column c0 + t, its k entries in
// registers.  Gaussian elimination by pivot steps, not by columns: with the
// pivots so far applied (right-looking), a column is independent of the earlier
// ones iff its residual is nonzero on a row that is not yet a pivot row, so the
// next CRP column is the first such column right of the last one (one block
// min-reduction), and the columns skipped on the way are dependent for good
// (later pivot rows are zero there).  Its owner takes the first live row with a
// nonzero as the pivot row and publishes its column; every later column c
// subtracts v_jp * (v_c[pr] / x).  Two barriers per pivot, none per dependent
// column.  Entries are never reduced: each pivot adds < p^2, so they stay below
// p + 32 p^2 < 2^32, and a zero test is one multiplication by p^-1 mod 2^32 (odd
// p: p | v iff v p^-1 mod 2^32 <= (2^32 - 1) / p; p = 2: the low bit).
// ---------------------------------------------------------------------------
struct ZeroTest {
    // odd p: p^-1 mod 2^32 and (2^32 - 1) / p; p = 2: 2^31 and 0 (v 2^31 mod 2^32 != 0 iff v odd)
    uint32_t pinv, thr;
    __device__ explicit ZeroTest(uint32_t p) {
        uint32_t x = p;  // Newton: x = p^-1 mod 2^(2^i) (odd p)
#pragma unroll
        for (int i = 0; i < 5; ++i) x *= 2u - p * x;
        pinv = (p & 1) ? x : 0x80000000u;
        thr = (p & 1) ? 0xffffffffu / p : 0u;
    }
    __device__ __forceinline__ bool nonzero(uint32_t v) const { return v * pinv > thr; }
};
// v[idx] with a log-depth select tree (idx < K, K a power of two)
template <int K>
__device__ __forceinline__ uint32_t sel_tree(const uint32_t (&v)[K], int idx) {
    uint32_t t[K / 2];
#pragma unroll
    for (int i = 0; i < K / 2; ++i) t[i] = (idx & 1) ? v[2 * i + 1] : v[2 * i];
#pragma unroll
    for (int w = K / 4, b = 2; w >= 1; w /= 2, b *= 2)
#pragma unroll
        for (int i = 0; i < w; ++i) t[i] = (idx & b) ? t[2 * i + 1] : t[2 * i];
    return t[0];
}
// bit i set iff v[i] != 0 mod p, OR-tree
template <int K>
__device__ __forceinline__ uint32_t nz_mask(const ZeroTest& zt, const uint32_t (&v)[K]) {
    uint32_t t[K];
#pragma unroll
    for (int i = 0; i < K; ++i) t[i] = (uint32_t)zt.nonzero(v[i]) << i;
#pragma unroll
    for (int w = K / 2; w >= 1; w /= 2)
#pragma unroll
        for (int i = 0; i < w; ++i) t[i] |= t[i + w];
    return t[0];
}
template <int K>
__global__ void __launch_bounds__(256) k_crp_list_reg(Fp f, const uint32_t* RI, int64_t ldr, int k, int64_t n,
                                                      int32_t* out, int32_t* ocount) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ uint32_t sinv[SINV_MAX];
    __shared__ __align__(16) uint32_t raw[2][32];  // the pivot column (owner's registers)
    __shared__ __align__(16) uint32_t qcol[2][32];  // p - v_jp[i] (reduced) on live rows != pr, else 0
    __shared__ int wmin[2][8];
    __shared__ int prow_s[2];
    __shared__ uint32_t xinv_s[2];
    const SmemInv inv = stage_inverses(f, sinv);  // independent of the predecessor
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * CRP_W;
    const bool have = c0 + tid < n;
    const ZeroTest zt(f.p);
    uint32_t v[K];
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] = (have && i < k) ? __ldcg(RI + (int64_t)i * ldr + c0 + tid) : 0u;
    uint32_t live = k >= 32 ? 0xffffffffu : (1u << k) - 1u;  // rows not yet pivot rows (uniform)
    int last = -1, nb = 0, par = 0;
    int32_t* o = out + (int64_t)blockIdx.x * k;
    for (;;) {
        const uint32_t nzm = nz_mask<K>(zt, v) & live;
        const int cand = __reduce_min_sync(0xffffffffu, (nzm && tid > last) ? tid : CRP_W);
        if (lane == 0) wmin[par][wp] = cand;
        __syncthreads();
        int jp = wmin[par][0];
#pragma unroll
        for (int w = 1; w < 8; ++w) jp = min(jp, wmin[par][w]);
        if (jp >= CRP_W) break;
        if (wp == (jp >> 5)) {  // the owner's warp publishes the pivot column
            if (tid == jp) {
                const int pr = __ffs(nzm) - 1;
                const uint32_t x = sel_tree<K>(v, pr);
#pragma unroll
                for (int i = 0; i < K; i += 4)
                    *reinterpret_cast<uint4*>(&raw[par][i]) = make_uint4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                prow_s[par] = pr;
                xinv_s[par] = inv(f, red32(f, x));
                o[nb] = (int32_t)(c0 + jp);
            }
            __syncwarp();
            const int pr = prow_s[par];
            qcol[par][lane] = (lane < K && ((live >> lane) & 1) && lane != pr) ? f.p - red32(f, raw[par][lane]) : 0u;
        }
        __syncthreads();
        const int pr = prow_s[par];
        const uint32_t xi = xinv_s[par];
        live &= ~(1u << pr);
        last = jp;
        ++nb;
        if (!live) break;
        const uint32_t b = tid > jp ? red32(f, red32(f, sel_tree<K>(v, pr)) * xi) : 0u;  // v_c[pr] / x
#pragma unroll
        for (int i = 0; i < K; i += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(&qcol[par][i]);
            v[i] += q.x * b;
            v[i + 1] += q.y * b;
            v[i + 2] += q.z * b;
            v[i + 3] += q.w * b;
        }
        par ^= 1;
    }
    if (tid == 0) ocount[blockIdx.x] = nb;
}

// ---------------------------------------------------------------------------
// RPM of the chunk's pivot rows from the level-0 candidates (1 CTA).  Every
// column dropped by a level-0 scan depends on earlier columns, so the RPM of
// R_I equals the RPM of R_I restricted to the candidate columns C (ascending).
// Row-order leftmost elimination on R_I[:, C] (the reference's Crout rule,
// plduq.cpp:46-84, on the compressed problem) yields each pivot row's column:
//   J = sorted pivot columns, sigma[t] = index in J of row t's pivot column.
// Rc lives in shared memory when k*|C| fits, else in the global scratch.
// ---------------------------------------------------------------------------
constexpr int RE_SMEM_WORDS = 40 * 1024;
__global__ void __launch_bounds__(256) k_crp_rowelim(Fp f, const uint32_t* RI, int64_t ldr, int k,
                                                     const int32_t* lists, const int32_t* counts,
                                                     int nblk, uint32_t* gscratch, int32_t* Jout,
                                                     int32_t* sigma_out, int32_t* fail) {
    FFB_PDL_ENTRY();
    extern __shared__ uint32_t sm[];
    __shared__ int32_t off[1025];
    __shared__ int32_t pcol[CRP_KMAX];
    __shared__ uint32_t mcol[CRP_KMAX];
    __shared__ uint32_t sinv[SINV_MAX];
    __shared__ int lead, total;
    const int tid = threadIdx.x;
    const SmemInv inv = stage_inverses(f, sinv);
    if (tid == 0) {
        int t = 0;
        for (int b = 0; b < nblk; ++b) {
            off[b] = t;
            t += counts[b];
        }
        off[nblk] = t;
        total = t;
    }
    __syncthreads();
    const int C = total;
    uint32_t* Rc = ((size_t)k * C <= RE_SMEM_WORDS) ? sm : gscratch;
    int32_t* cand = (int32_t*)(gscratch + (size_t)CRP_KMAX * nblk * CRP_KMAX);  // column ids
    for (int b = 0; b < nblk; ++b)
        for (int q = tid; q < counts[b]; q += blockDim.x) cand[off[b] + q] = lists[(int64_t)b * k + q];
    __syncthreads();
    {
        const int lane = tid & 31, wp = tid >> 5;
        for (int i = wp; i < k; i += 8)
            for (int j0 = lane; j0 < C; j0 += 128) {
                uint32_t vv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + 32 * u;
                    vv[u] = j < C ? __ldcg(RI + (int64_t)i * ldr + cand[j]) : 0u;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + 32 * u;
                    if (j < C) Rc[(size_t)i * C + j] = vv[u];
                }
            }
    }
    __syncthreads();
    for (int t = 0; t < k; ++t) {
        if (tid == 0) lead = C;
        __syncthreads();
        const uint32_t* rt = Rc + (size_t)t * C;
        for (int j = tid; j < C; j += blockDim.x)
            if (rt[j]) atomicMin(&lead, j);  // used columns are already zero in row t
        __syncthreads();
        const int jp = lead;
        if (jp >= C) {
            if (tid == 0) *fail = 1;
            return;
        }
        const uint32_t xi = inv(f, rt[jp]);
        for (int i = t + 1 + tid; i < k; i += blockDim.x) mcol[i] = fmul(f, Rc[(size_t)i * C + jp], xi);
        if (tid == 0) pcol[t] = cand[jp];
        __syncthreads();
        {
            const int lane = tid & 31, wp = tid >> 5;
            for (int i = t + 1 + wp; i < k; i += 8) {
                const uint32_t m = mcol[i];
                if (!m) continue;
                uint32_t* ri = Rc + (size_t)i * C;
                for (int j = jp + lane; j < C; j += 32) ri[j] = fsub(f, ri[j], fmul(f, m, rt[j]));
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        // J = sorted pivot columns; sigma[t] = position of pcol[t] in J
        int32_t js[CRP_KMAX];
        for (int t = 0; t < k; ++t) js[t] = pcol[t];
        for (int a = 1; a < k; ++a) {
            const int32_t v = js[a];
            int b = a - 1;
            while (b >= 0 && js[b] > v) { js[b + 1] = js[b]; --b; }
            js[b + 1] = v;
        }
        for (int t = 0; t < k; ++t) Jout[t] = js[t];
        for (int t = 0; t < k; ++t) {
            int lo = 0, hi = k - 1;
            while (lo < hi) {
                const int mid = (lo + hi) / 2;
                if (js[mid] < pcol[t]) lo = mid + 1; else hi = mid;
            }
            sigma_out[t] = lo;
        }
    }
}

// ---------------------------------------------------------------------------
// Chunk finish (1 CTA): RPM of R_I on the level-0 candidate columns, the
// inverse of Kc = R_I[:, J] and the chunk bookkeeping, in one launch.
//   1. candidate list C (ascending) from the level-0 lists (warp scan);
//   2. row-order leftmost elimination on R_I[:, C] (plduq.cpp:46-84 on the
//      compressed problem): row t's pivot is its leading nonzero; the same row
//      operations on the identity give L^-1, the reduced rows give U' (row t,
//      pivot column of row t') upper triangular;
//   3. X = U'^-1 L^-1 by back substitution (one barrier per row);
//   4. J = sorted pivot columns, sigma[t] = position of row t's column in J,
//      Kinv = (R_I[:, J])^-1 = row sigma[t] <- X[t];  UO[r + i] = (Kinv S_I)[i];
//      uhat_col[r+i] = J[i], prow[r+t] = c0 + I[t], pcol[r+t] = J[sigma t].
// Pivot searches are ballots in every warp (no atomics); each elimination row
// belongs to one warp, so a step needs one block barrier.
// ---------------------------------------------------------------------------
// dynamic smem: G (k^2) + max(rc_cap = min(k nblk k, CF_RC_WORDS), scan buffers)
constexpr int CF_RC_WORDS = 32 * 1024;
constexpr int CF_SMEM_WORDS = CRP_KMAX * CRP_KMAX + CF_RC_WORDS;
// si_off: word offset of a dedicated S_I region (early copy) when everything fits
// in 190 KB of dynamic smem, else -1 (S_I staged late into the free M buffer)
__host__ __device__ inline size_t cf_smem_bytes(int k, int nblk, int* rc_cap, int* si_off) {
    *rc_cap = (int)std::min<int64_t>((int64_t)k * nblk * k, CF_RC_WORDS);
    const size_t scan = (size_t)(CRP_KMAX + CRP_G) * k + CRP_G * CRP_KMAX;
    const size_t sketch = (size_t)k * RD_S;  // staged S_I rows
    const size_t base = (size_t)k * k + std::max<size_t>(std::max<size_t>((size_t)*rc_cap, scan), sketch);
    const size_t base4 = (base + 3) & ~(size_t)3;  // 16-byte aligned S_I region
    if ((base4 + sketch) * 4 <= (size_t)190 * 1024) {
        *si_off = (int)base4;
        return (base4 + sketch) * 4;
    }
    *si_off = -1;
    return base * 4;
}
// phase timestamps of the last k_crp_finish (globaltimer, thread 0; read by dbg_pq_bench)
__device__ unsigned long long g_cf_stamp[8];
#define CF_STAMP(i)                                                                           \
    do {                                                                                      \
        __syncthreads();                                                                      \
        if (threadIdx.x == 0) {                                                               \
            unsigned long long t_;                                                            \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                            \
            g_cf_stamp[i] = t_;                                                               \
        }                                                                                     \
    } while (0)
__global__ void __launch_bounds__(256) k_crp_finish(
    Fp f, const uint32_t* RI, int64_t ldr, int k, const int32_t* lists,
    const int32_t* counts, int nblk, int32_t* cand_g, int rc_cap, const int32_t* I, int64_t c0,
    const uint32_t* S, int64_t lds, int s, uint32_t* Kinv, int32_t* Jout, uint32_t* UO, int64_t lduo,
    int32_t* uhat_col, int32_t* prow, int32_t* pcol, int64_t r, int32_t* fail, int si_off, int s_compact,
    uint32_t* Ld, uint32_t* dval) {
    FFB_PDL_ENTRY();
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ int32_t off[1025];
    __shared__ int32_t cand_s[2048];  // candidate list in smem when it fits
    __shared__ int32_t Js[CRP_KMAX], rho[CRP_KMAX], pci[CRP_KMAX], pcv[CRP_KMAX], sig[CRP_KMAX], Is[CRP_KMAX];
    __shared__ int lead8[2][8];
    __shared__ uint32_t dinv[CRP_KMAX];
    __shared__ unsigned fmask[2];
    __shared__ BatchScratch bs;
    __shared__ uint32_t sinv[SINV_MAX];
    __shared__ int total;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    CF_STAMP(0);
    const SmemInv inv = stage_inverses(f, sinv);
    if (wp == 0) {  // exclusive offsets of the level-0 lists
        int run = 0;
        for (int b0 = 0; b0 < nblk; b0 += 32) {
            const int c = b0 + lane < nblk ? counts[b0 + lane] : 0;
            int x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (b0 + lane < nblk) off[b0 + lane] = run + x - c;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) total = run;
    }
    for (int t = tid; t < k; t += 256) Is[t] = I ? I[t] : 0;
    __syncthreads();
    // the k sketch rows S_I depend only on the inputs: start their copy now
    // (16-byte cp.async.cg into a dedicated region), consumed by the UO phase
    const bool si_early = S && si_off >= 0 && ((lds & 3) == 0) && ((s & 3) == 0) &&
                          ((((uintptr_t)S) & 15) == 0);
    if (si_early) {
        const int s4 = s >> 2;
        for (int u = wp; u < k; u += 8)
            for (int q = lane; q < s4; q += 32) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(sm + si_off + (size_t)u * s + 4 * q)),
                         "l"(S + (int64_t)(s_compact ? u : Is[u]) * lds + 4 * q));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const int C = total;
    int32_t* cand = C <= 2048 ? cand_s : cand_g;
    for (int b = wp; b < nblk; b += 8) {
        const int cb = counts[b], ob = off[b];
        for (int q = lane; q < cb; q += 32) cand[ob + q] = lists[(int64_t)b * k + q];
    }
    __syncthreads();
    // 1. the k x Cx elimination matrix M: R_I on all candidates when it fits
    //    (Cx = C, ids = cand), else R_I on J = its column rank profile over the
    //    candidates, found by the batched scan (Cx = k, ids = Js): the RPM of R_I
    //    is the RPM of M either way, every other column depending on earlier ones
    uint32_t* G = sm;                   // k x k: L^-1, then U'^-1 L^-1
    uint32_t* M = sm + (size_t)k * k;
    const bool direct = k * C <= rc_cap;
    const int Cx = direct ? C : k;
    const int32_t* ids = direct ? cand : Js;
    if (!direct) {
        uint32_t* E = M;
        uint32_t* V = E + (size_t)CRP_KMAX * k;
        uint32_t* VC = V + (size_t)CRP_G * k;
        auto colfn = [cand](int idx) { return cand[idx]; };
        const int nb = FFB_CRP_SCAN(f, inv, RI, ldr, k, C, colfn, E, V, VC, rho, fmask, bs, Js);
        if (nb < k) {  // R_I rank deficient: cannot happen for detected rows
            if (tid == 0) *fail = 1;
            return;
        }
        __syncthreads();
    }
    for (int i = wp; i < k; i += 8)
        for (int j = lane; j < k; j += 32) G[(size_t)i * k + j] = (i == j) ? 1 % f.p : 0u;
    for (int i = wp; i < k; i += 8)  // scattered gather, every copy in flight
        for (int j = lane; j < Cx; j += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(M + (size_t)i * Cx + j)),
                         "l"(RI + (int64_t)i * ldr + ids[j]));
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    CF_STAMP(1);
    // 2. row-order leftmost elimination on M, tracking L^-1 in G.  The leading
    //    entry of row t: each thread scans a strided slice, warps reduce, one
    //    barrier combines (lead8 rotates over 2 slots, so no reset barrier).
    // lazy: rows below the pivot accumulate unreduced sums x + (p - m) v (< p + k p^2),
    // reduced only when a row becomes the pivot row (its leading search) or when a
    // coefficient is read; exact per-term reduction otherwise
    const bool lazy = (uint64_t)k * (f.p - 1) * (f.p - 1) + f.p < (1ull << 32);
    for (int t = 0; t < k; ++t) {
        uint32_t* rt = M + (size_t)t * Cx;
        int mine = Cx;
        if (lazy) {  // reduce the whole row (it feeds the elimination), first nonzero
            for (int j = tid; j < Cx; j += 256) {
                const uint32_t v = red32(f, rt[j]);
                rt[j] = v;
                if (v != 0 && mine == Cx) mine = j;
            }
        } else {
            for (int j = tid; j < Cx; j += 256)
                if (rt[j] != 0) {
                    mine = j;
                    break;
                }
        }
        mine = __reduce_min_sync(0xffffffffu, mine);
        if (lane == 0) lead8[t & 1][wp] = mine;
        __syncthreads();
        int jp = lead8[t & 1][0];
#pragma unroll
        for (int w = 1; w < 8; ++w) jp = min(jp, lead8[t & 1][w]);
        if (jp >= Cx) {
            if (tid == 0) *fail = 1;
            return;
        }
        const uint32_t il = inv(f, rt[jp]);
        if (tid == 0) {
            pci[t] = jp;
            pcv[t] = ids[jp];
            dinv[t] = il;
        }
        const uint32_t* gt = G + (size_t)t * k;
        for (int i = t + 1 + wp; i < k; i += 8) {
            uint32_t* ri = M + (size_t)i * Cx;
            const uint32_t c = lazy ? red32(f, ri[jp]) : ri[jp];
            __syncwarp();
            if (!c) continue;
            const uint32_t m = fmul(f, c, il);
            int j = jp + lane;
            if (lazy) {  // 4 independent load pairs in flight per lane
                const uint32_t mn = f.p - m;
                for (; j + 96 < Cx; j += 128) {
                    const uint32_t a0 = ri[j], a1 = ri[j + 32], a2 = ri[j + 64], a3 = ri[j + 96];
                    const uint32_t b0 = rt[j], b1 = rt[j + 32], b2 = rt[j + 64], b3 = rt[j + 96];
                    ri[j] = a0 + mn * b0;
                    ri[j + 32] = a1 + mn * b1;
                    ri[j + 64] = a2 + mn * b2;
                    ri[j + 96] = a3 + mn * b3;
                }
                for (; j < Cx; j += 32) ri[j] += mn * rt[j];
            } else {
                for (; j + 96 < Cx; j += 128) {
                    const uint32_t a0 = ri[j], a1 = ri[j + 32], a2 = ri[j + 64], a3 = ri[j + 96];
                    const uint32_t b0 = rt[j], b1 = rt[j + 32], b2 = rt[j + 64], b3 = rt[j + 96];
                    ri[j] = fmsub(f, a0, m, b0);
                    ri[j + 32] = fmsub(f, a1, m, b1);
                    ri[j + 64] = fmsub(f, a2, m, b2);
                    ri[j + 96] = fmsub(f, a3, m, b3);
                }
                for (; j < Cx; j += 32) ri[j] = fmsub(f, ri[j], m, rt[j]);
            }
            uint32_t* gi = G + (size_t)i * k;
            for (int j = lane; j <= t; j += 32) gi[j] = fmsub(f, gi[j], m, gt[j]);
        }
        __syncthreads();
    }
    CF_STAMP(2);
    // 2b. the chunk's block of the PLDUQ's D and of D^-1 L^-1 (row order = pivot order):
    //     R_I = L D U'' with U'' the chunk's rows of the echelon U, so U'' = (D^-1 L^-1) R_I
    if (Ld) {
        for (int t = wp; t < k; t += 8)
            for (int j = lane; j < k; j += 32) Ld[(int64_t)t * k + j] = j <= t ? fmul(f, G[(size_t)t * k + j], dinv[t]) : 0u;
        for (int t = tid; t < k; t += 256) dval[t] = M[(size_t)t * Cx + pci[t]];
    }
    // 3. back substitution X = U'^-1 L^-1, U'[t][t'] = M[t][pci[t']]
    for (int tp = k - 1; tp > 0; --tp) {
        const uint32_t* gp = G + (size_t)tp * k;
        const int jc = pci[tp];
        const uint32_t dp = dinv[tp];
        for (int t = wp; t < tp; t += 8) {
            const uint32_t c = M[(size_t)t * Cx + jc];
            if (!c) continue;  // warp-uniform
            const uint32_t m = fmul(f, c, dp);
            uint32_t* gr = G + (size_t)t * k;
            for (int j = lane; j < k; j += 32) gr[j] = fmsub(f, gr[j], m, gp[j]);
        }
        __syncthreads();
    }
    CF_STAMP(3);
    // 4. outputs: J = sorted pivot columns, sigma[t] = rank of row t's column,
    //    Kinv row sigma[t] = X[t]
    for (int t = tid; t < k; t += 256) {
        int rank = 0;
        const int v = pcv[t];
        for (int u = 0; u < k; ++u) rank += pcv[u] < v;
        sig[t] = rank;
        Jout[rank] = v;
    }
    __syncthreads();
    for (int t = wp; t < k; t += 8) {  // row t of X, scaled: row sig[t] of Kinv
        const uint32_t dt = dinv[t];
        for (int j = lane; j < k; j += 32) {
            const uint32_t v = fmul(f, G[(size_t)t * k + j], dt);
            G[(size_t)t * k + j] = v;
            Kinv[(int64_t)sig[t] * k + j] = v;
        }
    }
    CF_STAMP(4);
    if (S) {  // UO rows from the k sketch rows S_I (copied early, or staged now in the free M buffer)
        uint32_t* SI = si_early ? sm + si_off : M;
        if (!si_early)
            for (int u = wp; u < k; u += 8)
                for (int col = lane; col < s; col += 32)
                    SI[(size_t)u * s + col] = __ldcg(S + (int64_t)(s_compact ? u : Is[u]) * lds + col);
        __syncthreads();
        const bool lz = (uint64_t)k * (f.p - 1) * (f.p - 1) < (1ull << 32) && f.mu32;  // 32-bit sums
        for (int t = wp; t < k; t += 8) {
            const uint32_t* xt = G + (size_t)t * k;
            uint32_t* uo = UO + (r + sig[t]) * lduo;
            for (int col = lane; col < s; col += 32) {
                if (lz) {
                    uint32_t acc = 0;
                    for (int u = 0; u < k; ++u) acc += xt[u] * SI[(size_t)u * s + col];
                    uo[col] = red32(f, acc);
                } else {
                    uint64_t acc = 0;
                    for (int u = 0; u < k; ++u) {
                        acc += (uint64_t)xt[u] * SI[(size_t)u * s + col];
                        if (f.p >= (1u << 23)) acc = red64(f, acc);
                    }
                    uo[col] = red64(f, acc);
                }
            }
        }
    }
    for (int t = tid; t < k; t += 256) {
        uhat_col[r + sig[t]] = pcv[t];
        prow[r + t] = (int32_t)(c0 + Is[t]);
        pcol[r + t] = pcv[t];
    }
    CF_STAMP(5);
}

// ---------------------------------------------------------------------------
// Register-resident chunk finish for k <= 32, p <= 255 (the same outputs as k_crp_finish;
// every one of them is unique given R_I and the candidates, so the two kernels agree
// bit for bit).  1024 threads; thread c owns candidate columns c and c + 1024 as packed
// bytes (8 registers per column, raw R_I values, never modified).  The elimination is
// left-looking on the candidates and right-looking on G = L^-1 only:
//   * thread (warp i, lane j) owns G[i][j];
//   * step t: every thread forms the residual of row t on its columns, G[t] . M[:, c] (8
//     dp4a against the published packed row G[t]); warps reduce the leftmost nonzero and
//     publish that column (barrier 1); all warps read the winner jp; warp i > t forms
//     c_i = G[i] . M[:, jp] (one warp add-reduction), G[i] -= c_i d^-1 G[t]; warp t+1
//     publishes its finished row (barrier 2);
//   * U'[t][t'] = G[t] . M[:, jp(t')] afterwards (dp4a), the back substitution
//     X = U'^-1 L^-1 one thread per column without barriers, then Kinv, UO rows, bookkeeping.
// No candidate matrix in shared memory, two barriers per pivot.
// ---------------------------------------------------------------------------
constexpr int CFR_CPT = 2;                     // candidate columns per thread
constexpr int CFR_MAXC = 1024 * CFR_CPT;       // host: nblk * k <= CFR_MAXC
constexpr int CFR_MAXBLK = 128;                // host: nblk <= CFR_MAXBLK
__global__ void __launch_bounds__(1024) k_crp_finish_reg(
    Fp f, const uint32_t* RI, int64_t ldr, int k, const int32_t* lists, const int32_t* counts, int nblk,
    const int32_t* I, int64_t c0, const uint32_t* S, int64_t lds, int s, uint32_t* Kinv, int32_t* Jout,
    uint32_t* UO, int64_t lduo, int32_t* uhat_col, int32_t* prow, int32_t* pcol, int64_t r, int32_t* fail,
    int s_compact, uint32_t* Ld, uint32_t* dval) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ uint32_t sinv[256];
    __shared__ int32_t off[CFR_MAXBLK + 1];
    __shared__ uint32_t SI[32 * RD_S];
    __shared__ __align__(16) uint32_t gp[8];          // the published row G[t], packed bytes
    __shared__ uint32_t Gs[32][33];                   // finished rows of L^-1
    __shared__ __align__(16) uint32_t GsP[32][8];     // the same, packed
    __shared__ int32_t slot_idx[32], slot_id[32];
    __shared__ uint32_t slot_val[32];
    __shared__ __align__(16) uint32_t slot_col[32][8];
    __shared__ __align__(16) uint32_t PC[32][8];      // pivot columns (raw, packed), pivot order
    __shared__ int32_t pcv[32], sig[32], Is[32];
    __shared__ uint32_t dv[32], dinvs[32];
    __shared__ uint32_t Us[32][33], Xs[32][33];
    __shared__ int total;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    if (tid < 256) sinv[tid] = ((uint32_t)tid < f.p && tid > 0) ? (f.inv ? __ldcg(f.inv + tid) : finv_euclid(f.p, tid)) : 0u;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (wp == 0) {  // exclusive offsets of the level-0 lists
        int run = 0;
        for (int b0 = 0; b0 < nblk; b0 += 32) {
            const int c = b0 + lane < nblk ? __ldcg(counts + b0 + lane) : 0;
            int x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (b0 + lane < nblk) off[b0 + lane] = run + x - c;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) {
            total = run;
            off[nblk] = run;
        }
    }
    if (tid >= 32 && tid < 64) Is[lane] = (I && lane < k) ? __ldcg(I + lane) : 0;
    if (tid >= 64 && tid < 72) gp[tid - 64] = tid == 64 ? 1u : 0u;  // G[0] = e_0
    if (tid >= 96 && tid < 128) Gs[0][lane] = lane == 0 ? 1u : 0u;
    if (tid >= 128 && tid < 136) GsP[0][tid - 128] = tid == 128 ? 1u : 0u;
    __syncthreads();
    if (S) {  // the k sketch rows S_I: copies in flight until the UO phase
        for (int e = tid; e < k * s; e += 1024) {
            const int u = e / s, col = e - u * s;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(SI + u * RD_S + col)),
                         "l"(S + (int64_t)(s_compact ? u : Is[u]) * lds + col));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const int C = total;
    // my candidate columns: raw R_I entries as packed bytes (row i = byte i & 3 of word i >> 2)
    uint32_t Mr[CFR_CPT][8];
    int32_t colid[CFR_CPT];
#pragma unroll
    for (int q = 0; q < CFR_CPT; ++q) {
        const int c = tid + 1024 * q;
        colid[q] = -1;
#pragma unroll
        for (int w = 0; w < 8; ++w) Mr[q][w] = 0u;
        if (c < C) {
            int lo = 0, hi = nblk - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (off[mid] <= c) lo = mid;
                else hi = mid - 1;
            }
            const int32_t id = __ldcg(lists + (int64_t)lo * k + (c - off[lo]));
            colid[q] = id;
            uint32_t v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = i < k ? __ldcg(RI + (int64_t)i * ldr + id) : 0u;
#pragma unroll
            for (int w = 0; w < 8; ++w)
                Mr[q][w] = v[4 * w] | (v[4 * w + 1] << 8) | (v[4 * w + 2] << 16) | (v[4 * w + 3] << 24);
        }
    }
    uint32_t g = wp == lane ? 1u : 0u;  // G[wp][lane]
    const int sh = 8 * (lane & 3);
    for (int t = 0; t < k; ++t) {
        {  // residual of row t on my columns, leftmost nonzero of the warp
            const uint4 ga = *reinterpret_cast<const uint4*>(gp), gb = *reinterpret_cast<const uint4*>(gp + 4);
            int mine = INT_MAX, mq = 0;
            uint32_t mval = 0;
#pragma unroll
            for (int q = CFR_CPT - 1; q >= 0; --q) {
                if (1024 * q >= C) continue;  // uniform
                uint32_t a = __dp4a(Mr[q][0], ga.x, 0u);
                a = __dp4a(Mr[q][1], ga.y, a);
                a = __dp4a(Mr[q][2], ga.z, a);
                a = __dp4a(Mr[q][3], ga.w, a);
                a = __dp4a(Mr[q][4], gb.x, a);
                a = __dp4a(Mr[q][5], gb.y, a);
                a = __dp4a(Mr[q][6], gb.z, a);
                a = __dp4a(Mr[q][7], gb.w, a);
                a = red32(f, a);
                if (a != 0 && colid[q] >= 0) {
                    mine = tid + 1024 * q;
                    mq = q;
                    mval = a;
                }
            }
            const int wmin = __reduce_min_sync(0xffffffffu, mine);
            if (wmin == INT_MAX) {
                if (lane == 0) slot_idx[wp] = INT_MAX;
            } else if (mine == wmin) {
                slot_idx[wp] = wmin;
                slot_val[wp] = mval;
                slot_id[wp] = mq ? colid[CFR_CPT - 1] : colid[0];
#pragma unroll
                for (int w = 0; w < 8; ++w) slot_col[wp][w] = mq ? Mr[CFR_CPT - 1][w] : Mr[0][w];
            }
        }
        __syncthreads();
        const int my = slot_idx[lane];
        const int jp = __reduce_min_sync(0xffffffffu, my);
        if (jp == INT_MAX) {  // R_I rank deficient: cannot happen for detected rows
            if (tid == 0) *fail = 1;
            return;
        }
        const int win = __ffs(__ballot_sync(0xffffffffu, my == jp)) - 1;
        const uint32_t d = slot_val[win], di = sinv[d];
        const uint32_t mc = (slot_col[win][lane >> 2] >> sh) & 0xffu;  // M[lane][jp]
        if (wp == 0) {
            if (lane < 8) PC[t][lane] = slot_col[win][lane];
            if (lane == 8) {
                pcv[t] = slot_id[win];
                dv[t] = d;
                dinvs[t] = di;
            }
        }
        if (wp > t && wp < k) {  // G[wp] -= (G[wp] . M[:, jp]) d^-1 G[t]
            const uint32_t ci = red32(f, __reduce_add_sync(0xffffffffu, g * mc));
            const uint32_t m = red32(f, ci * di);
            g = red32(f, g + (f.p - m) * Gs[t][lane]);
            if (wp == t + 1) {  // row t + 1 is final: publish it
                Gs[t + 1][lane] = g;
                uint32_t x = g << sh;
                x |= __shfl_xor_sync(0xffffffffu, x, 1);
                x |= __shfl_xor_sync(0xffffffffu, x, 2);
                if ((lane & 3) == 0) {
                    gp[lane >> 2] = x;
                    GsP[t + 1][lane >> 2] = x;
                }
            }
        }
        __syncthreads();
    }
    // sigma, J, bookkeeping
    if (tid < k) {
        int rank = 0;
        const int v = pcv[tid];
        for (int u = 0; u < k; ++u) rank += pcv[u] < v;
        sig[tid] = rank;
        Jout[rank] = v;
        uhat_col[r + rank] = v;
        prow[r + tid] = (int32_t)(c0 + Is[tid]);
        pcol[r + tid] = v;
    }
    if (wp < k && lane < k) {  // U'[t][t'] = G[t] . M[:, jp(t')]; the chunk's D^-1 L^-1 and D
        const int t = wp, tp = lane;
        uint32_t a = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) a = __dp4a(GsP[t][w], PC[tp][w], a);
        Us[t][tp] = red32(f, a);
        if (Ld) {
            Ld[(int64_t)t * k + tp] = tp <= t ? red32(f, Gs[t][tp] * dinvs[t]) : 0u;
            if (tp == 0) dval[t] = dv[t];
        }
    }
    __syncthreads();
    if (tid < k) {  // column tid of X = U'^-1 L^-1: x_t = d_t^-1 (G[t][j] - sum_{t' > t} U'[t][t'] x_t')
        uint32_t x[32];
#pragma unroll
        for (int t = 31; t >= 0; --t) {
            x[t] = 0u;
            if (t < k) {
                uint32_t acc = 0;
#pragma unroll
                for (int tp = t + 1; tp < 32; ++tp) acc += Us[t][tp] * x[tp];
                const uint32_t v = red32(f, Gs[t][tid] + f.p - red32(f, acc));
                x[t] = red32(f, v * dinvs[t]);
                Xs[t][tid] = x[t];
                Kinv[(int64_t)sig[t] * k + tid] = x[t];
            }
        }
    }
    if (S) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        for (int e = tid; e < k * s; e += 1024) {  // UO[r + sigma(t)] = X[t] S_I
            const int t = e / s, col = e - t * s;
            uint32_t acc = 0;
            for (int u = 0; u < k; ++u) acc += Xs[t][u] * SI[u * RD_S + col];
            UO[(r + sig[t]) * lduo + col] = red32(f, acc);
        }
    }
}

// ---------------------------------------------------------------------------
// Pairing + inverse + bookkeeping (1 CTA).  Kc = RI[:, J] (k x k, nonsingular).
// Row-order leftmost elimination on Kc gives the RPM pairing sigma (the
// reference's Crout rule restricted to Kc); Gauss-Jordan gives Kinv.  Then:
//   Kinv -> global (for Unew = Kinv RI), UO[r+i] = (Kinv S[I,:])[i] when
//   sketching, uhat_col[r+t] = J[t], prow[r+t] = c0+I[t], pcol[r+t] = J[sigma t].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_pair2(Fp f, const uint32_t* RI, int64_t ldr, int k,
                                               const int32_t* J, const int32_t* I, int64_t c0,
                                               const uint32_t* S, int64_t lds, int s,
                                               uint32_t* Kinv, uint32_t* UO, int64_t lduo,
                                               int32_t* uhat_col, int32_t* prow, int32_t* pcol,
                                               int64_t r, int32_t* fail, const int32_t* sigma_in) {
    FFB_PDL_ENTRY();
    extern __shared__ uint32_t sm[];
    uint32_t* A = sm;                       // k x k working copy (row-order elimination)
    uint32_t* G = A + (size_t)k * k;        // k x 2k Gauss-Jordan
    __shared__ int colused[CRP_KMAX];
    __shared__ int sig[CRP_KMAX];
    __shared__ int lead;
    __shared__ uint32_t il;
    __shared__ uint32_t sinv[SINV_MAX];
    const int tid = threadIdx.x;
    const SmemInv inv = stage_inverses(f, sinv);
    for (int e = tid; e < k * k; e += blockDim.x) {
        const int i = e / k, j = e % k;
        const uint32_t v = __ldcg(RI + (int64_t)i * ldr + J[j]);
        A[e] = v;
        G[(size_t)i * 2 * k + j] = v;
        G[(size_t)i * 2 * k + k + j] = (i == j) ? 1 % f.p : 0;
    }
    for (int j = tid; j < k; j += blockDim.x) colused[j] = 0;
    if (sigma_in)
        for (int t = tid; t < k; t += blockDim.x) sig[t] = sigma_in[t];
    __syncthreads();
    for (int t = 0; t < (sigma_in ? 0 : k); ++t) {
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
            sig[t] = jp;
            colused[jp] = 1;
            il = inv(f, A[(size_t)t * k + jp]);
        }
        __syncthreads();
        for (int e = tid; e < (k - t - 1) * k; e += blockDim.x) {
            const int i = t + 1 + e / k, j = e % k;
            if (colused[j]) continue;  // jp included: its column is zeroed below
            const uint32_t m = fmul(f, A[(size_t)i * k + jp], il);
            A[(size_t)i * k + j] = fsub(f, A[(size_t)i * k + j], fmul(f, m, A[(size_t)t * k + j]));
        }
        __syncthreads();
        for (int i = t + 1 + tid; i < k; i += blockDim.x) A[(size_t)i * k + jp] = 0;
        __syncthreads();
    }
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
        if (tid == 0) il = inv(f, G[(size_t)c * w + c]);
        __syncthreads();
        for (int j = tid; j < w; j += blockDim.x) G[(size_t)c * w + j] = fmul(f, G[(size_t)c * w + j], il);
        __syncthreads();
        {
            const int lane = tid & 31, wp = tid >> 5;
            for (int i = wp; i < k; i += 8) {
                if (i == c) continue;
                const uint32_t m = G[(size_t)i * w + c];
                if (!m) continue;
                for (int j = lane; j < w; j += 32)
                    if (j != c) G[(size_t)i * w + j] = fsub(f, G[(size_t)i * w + j], fmul(f, m, G[(size_t)c * w + j]));
            }
        }
        __syncthreads();
        for (int i = tid; i < k; i += blockDim.x)
            if (i != c) G[(size_t)i * w + c] = 0;
        __syncthreads();
    }
    for (int e = tid; e < k * k; e += blockDim.x) {
        const int i = e / k, j = e % k;
        Kinv[(int64_t)i * k + j] = G[(size_t)i * w + k + j];
    }
    if (S) {
        for (int e = tid; e < k * s; e += blockDim.x) {
            const int i = e / s, col = e % s;
            uint64_t acc = 0;
            for (int t = 0; t < k; ++t) {
                acc += (uint64_t)G[(size_t)i * w + k + t] * S[(int64_t)I[t] * lds + col];
                if (f.p >= (1u << 23)) acc = red64(f, acc);
            }
            UO[(r + i) * lduo + col] = red64(f, acc);
        }
    }
    for (int t = tid; t < k; t += blockDim.x) {
        uhat_col[r + t] = J[t];
        prow[r + t] = (int32_t)(c0 + I[t]);
        pcol[r + t] = J[sig[t]];
    }
}

// H[i][t] = L[i][t] * d[t]
// H[ridx ? ridx[i] : i][t] = L[i][t] d[t]
__global__ void k_scale_cols(Fp f, uint32_t* H, int64_t ldh, const uint32_t* L, int64_t ldl,
                             const uint32_t* d, int64_t cols, const int32_t* ridx) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    uint32_t* h = H + (ridx ? (int64_t)ridx[i] : i) * ldh;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < cols;
         t += (int64_t)gridDim.x * blockDim.x)
        h[t] = fmul(f, L[i * ldl + t], d[t]);
}

// dst[a][cidx[b]] = src[a][b]: columns back to their original positions
__global__ void k_scatter_cols(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds, const int32_t* cidx,
                               int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t a = blockIdx.y;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < cols; b += (int64_t)gridDim.x * blockDim.x)
        dst[a * ldd + cidx[b]] = src[a * lds + b];
}

// Certificate part: pivotless row t (= np[a]) may only depend on pivots found before it.
__global__ void k_m1_pattern(const uint32_t* M1, int64_t ldm, const int32_t* np,
                             const int32_t* prow, int64_t r, int32_t* flag) {
    FFB_PDL_ENTRY();
    const int64_t a = blockIdx.y;
    const int32_t t = np[a];
    int bad = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < r;
         k += (int64_t)gridDim.x * blockDim.x)
        bad |= prow[k] > t && M1[a * ldm + k] != 0;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// ---------------------------------------------------------------------------
// LDU without pivoting of a <= 64 x 64 block in place (1 CTA):
// strict lower <- L, diagonal <- d, strict upper <- U.
// ---------------------------------------------------------------------------
template <bool kSmall>
__global__ void __launch_bounds__(256) k_ldu_base(Fp f, uint32_t* K, int64_t ldk, int n,
                                                  int32_t* fail) {
    FFB_PDL_ENTRY();
    // Register ownership as in the leaf: thread (ty, tx) holds K[ty + 4q][tx].
    // Step t broadcasts column t and row t (double-buffered) with one barrier.
    // kSmall: 32-bit Barrett arithmetic (p < 2^16), no 64-bit path in the loop.
    __shared__ uint32_t colb[2][64], rowb[2][64];
    __shared__ uint32_t sinv[SINV_MAX];
    const Ar<kSmall> ar(f);
    const int tid = threadIdx.x, tx = tid & 63, ty = tid >> 6;
    uint32_t A[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int i = ty + 4 * q;
        A[q] = (i < n && tx < n) ? K[(int64_t)i * ldk + tx] : 0;
    }
    const SmemInv inv = stage_inverses(f, sinv);
    for (int t = 0; t < n; ++t) {
        uint32_t* cb = colb[t & 1];
        uint32_t* rb = rowb[t & 1];
        if (tx == t) {
#pragma unroll
            for (int q = 0; q < 16; ++q) cb[ty + 4 * q] = A[q];
        }
        if (ty == (t & 3)) rb[tx] = A[t >> 2];
        __syncthreads();
        const uint32_t d = cb[t];
        if (d == 0) {
            if (tid == 0) *fail = 1;
            return;  // uniform
        }
        const uint32_t di = inv(f, d);
        const uint32_t uj = ar.mul(rb[tx], di);  // U[t][tx] for tx > t
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int i = ty + 4 * q;
            const uint32_t ci = cb[i];
            const uint32_t upd = ar.sub(A[q], ar.mul(ci, uj));
            const uint32_t lij = ar.mul(ci, di);
            // i > t: trailing update (tx > t) or L[i][t] (tx == t); i == t: U[t][tx] (tx > t)
            A[q] = i > t ? (tx > t ? upd : (tx == t ? lij : A[q])) : ((i == t && tx > t) ? uj : A[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int i = ty + 4 * q;
        if (i < n && tx < n) K[(int64_t)i * ldk + tx] = A[q];
    }
}

// ---------------------------------------------------------------------------
// LDU without pivoting of an n <= 128 block in place, 2 <= p < 4096 (1 CTA of 512).
// Right-looking elimination over the whole block (no recursion, no off-diagonal
// solves): thread (rg, cg) keeps the 4 x 8 tile K[4rg .. +3][8cg .. +7] in
// registers, lazily reduced -- entries only grow, by (p - l) u < p^2 per step, so
// after <= 128 steps they stay below 2^32 (p < 4096) and are reduced by 32-bit
// Barrett when they become a pivot row or column.  Step t: the owners of column t
// and of row t publish them reduced (static register indices: the step loop is
// unrolled by 8), one barrier, then every live tile takes its update.  Result:
// strict lower <- L, diagonal <- d, strict upper <- U (unit upper, row t / d_t).
// ---------------------------------------------------------------------------
template <int TR>  // rows per register tile: 4 (512 threads) or 8 (256 threads)
__global__ void __launch_bounds__(128 * 16 / TR) k_ldu128(Fp f, uint32_t* K, int64_t ldk, int n, int32_t* fail) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ uint32_t colv[2][128], rowv[2][128];
    __shared__ uint32_t sinv[SINV_MAX];
    const int tid = threadIdx.x, rg = tid >> 4, cg = tid & 15;
    const SmemInv inv = stage_inverses(f, sinv);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int r0 = TR * rg, c0 = 8 * cg;
    uint32_t T[TR][8];
#pragma unroll
    for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b)
            T[a][b] = (r0 + a < n && c0 + b < n) ? __ldcg(K + (int64_t)(r0 + a) * ldk + c0 + b) : 0u;
    const uint32_t p = f.p;
    for (int tb = 0; tb < (n + 7) / 8; ++tb) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int t = 8 * tb + jj;
            if (t >= n) break;  // uniform
            const int buf = t & 1;
            if (cg == tb) {  // column t (reduced), rows of this tile
#pragma unroll
                for (int a = 0; a < TR; ++a) colv[buf][r0 + a] = red32(f, T[a][jj]);
            }
            if (rg == t / TR) {  // row t (reduced), columns of this tile
#pragma unroll
                for (int b = 0; b < 8; ++b) rowv[buf][c0 + b] = red32(f, T[jj % TR][b]);
            }
            __syncthreads();
            const uint32_t d = rowv[buf][t];
            if (d == 0) {  // a singular leading minor: LDU without pivoting does not exist
                if (tid == 0) *fail = 1;
                return;  // uniform
            }
            const bool rows_live = r0 + TR - 1 > t, cols_live = c0 + 7 > t;
            const bool col_owner = cg == tb, row_owner = rg == t / TR;
            // only tiles with live rows AND live columns take the update; the owners of
            // column t / row t also write their L / U outputs (U needs d^-1)
            if ((rows_live && cols_live) || col_owner || row_owner) {
                const uint32_t di = inv(f, d);
                uint32_t l[TR], u[8];
#pragma unroll
                for (int a = 0; a < TR; ++a) l[a] = red32(f, colv[buf][r0 + a] * di);
#pragma unroll
                for (int b = 0; b < 8; ++b) u[b] = rowv[buf][c0 + b];
                if (rows_live && cols_live) {
#pragma unroll
                    for (int a = 0; a < TR; ++a)
#pragma unroll
                        for (int b = 0; b < 8; ++b)
                            if (r0 + a > t && c0 + b > t) T[a][b] += (p - l[a]) * u[b];
                }
                // outputs of step t: L column t, d, U row t
                if (col_owner) {
#pragma unroll
                    for (int a = 0; a < TR; ++a)
                        if (r0 + a > t) T[a][jj] = l[a];
                }
                if (row_owner) {
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        if (c0 + b > t) T[jj % TR][b] = red32(f, u[b] * di);
                        else if (c0 + b == t) T[jj % TR][b] = d;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (r0 + a < n && c0 + b < n) K[(int64_t)(r0 + a) * ldk + c0 + b] = T[a][b];
}

// U (unit upper with zeros below) from the packed LDU block.
__global__ void k_unpack_u(uint32_t* U, int64_t ldu, const uint32_t* K, int64_t ldk, int64_t n, uint32_t one) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        U[i * ldu + j] = j > i ? K[i * ldk + j] : (j == i ? one : 0);
}

// L (unit lower with zeros above) from the packed LDU block; d from the diagonal.
__global__ void k_unpack_l(uint32_t* L, int64_t ldl, const uint32_t* K, int64_t ldk, int64_t n,
                           uint32_t* d, uint32_t one) {
    FFB_PDL_ENTRY();
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

void gather2d(cudaStream_t st, DMat dst, DMat src, const int32_t* ridx, const int32_t* cidx,
              int64_t roff) {
    if (dst.rows <= 0 || dst.cols <= 0) return;
    ProfScope ps(K_MOVE, st, 0.0, 8.0 * dst.rows * dst.cols);
    for (int64_t r0 = 0; r0 < dst.rows; r0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, dst.rows - r0);
        launch_k(k_gather2d, rgrid(nr, dst.cols), 256, 0, st, dst.ptr + r0 * dst.ld, dst.ld, src.ptr, src.ld,
                                                        ridx ? ridx + r0 : nullptr,
                                                        ridx ? roff : roff + r0, cidx, dst.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void copy_mat(cudaStream_t st, DMat dst, DMat src) {
    if (src.rows <= 0 || src.cols <= 0) return;
    ProfScope ps(K_MOVE, st, 0.0, 8.0 * src.rows * src.cols);
    if (dst.ld == src.ld && dst.ld == src.cols) {
        FFB_CUDA(cudaMemcpyAsync(dst.ptr, src.ptr, (size_t)src.rows * src.cols * 4,
                                 cudaMemcpyDeviceToDevice, st)); pdl_fence(st);
        return;
    }
    FFB_CUDA(cudaMemcpy2DAsync(dst.ptr, dst.ld * 4, src.ptr, src.ld * 4, src.cols * 4, src.rows,
                               cudaMemcpyDeviceToDevice, st));
}

// LDU without pivoting of K (n x n, in place), recursive.
void ldu_inplace(const Fp& f, cudaStream_t st, DMat K, Workspace& ws, int32_t* fail) {
    const int64_t n = K.rows;
    if (n <= 0) return;
    static const bool l128 = getenv("FFB_NO_LDU128") == nullptr;  // A/B hook
    if (l128 && f.p < 4096u && f.mu32 && n <= 128) {
        ProfScope ps(K_LDU, st, 2.0 * n * n * n / 3.0, 8.0 * n * n);
        // 4-row tiles, 512 threads (8-row tiles on 256 threads measured 49 vs 46 us per call)
        static const bool big_tiles = getenv("FFB_LDU_TILE8") != nullptr;  // A/B hook
        if (big_tiles) launch_k(k_ldu128<8>, 1, 256, 0, st, f, K.ptr, K.ld, (int)n, fail);
        else launch_k(k_ldu128<4>, 1, 512, 0, st, f, K.ptr, K.ld, (int)n, fail);
        count_launch();
        FFB_CHECK_LAUNCH();
        return;
    }
    if (n <= 64) {
        ProfScope ps(K_LDU, st, 2.0 * n * n * n / 3.0, 8.0 * n * n);
        if (f.p < 65536u)
            launch_k(k_ldu_base<true>, 1, 256, 0, st, f, K.ptr, K.ld, (int)n, fail);
        else
            launch_k(k_ldu_base<false>, 1, 256, 0, st, f, K.ptr, K.ld, (int)n, fail);
        count_launch();
        FFB_CHECK_LAUNCH();
        return;
    }
    const int64_t base = (l128 && f.p < 4096u && f.mu32) ? 128 : 64;
    int64_t n1 = (n / 2) / base * base;
    if (n1 < base) n1 = base;
    const int64_t n2 = n - n1;
    DMat K11 = K.sub(0, 0, n1, n1), K12 = K.sub(0, n1, n1, n2), K21 = K.sub(n1, 0, n2, n1),
         K22 = K.sub(n1, n1, n2, n2);
    ldu_inplace(f, st, K11, ws, fail);
    const size_t mk = ws.mark();
    uint32_t* dinv = ws.vec<uint32_t>(n1);
    uint32_t* d = ws.vec<uint32_t>(n1);
    DMat L11 = ws.mat(n1, n1);
    launch_k(k_unpack_l, rgrid(n1, n1), 256, 0, st, L11.ptr, L11.ld, K11.ptr, K11.ld, n1, d, 1 % f.p);
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
    // test hook: a narrow sketch makes misses likely, exercising the certificate
    static const int sk_env = getenv("FFB_PLDUQ_SKETCH_COLS") ? atoi(getenv("FFB_PLDUQ_SKETCH_COLS")) : 0;
    // register-resident row detection (k_rrp) for p < 4096; FFB_RD_BATCHED: the batched kernel (A/B hook)
    static const bool rrp_env = getenv("FFB_RD_BATCHED") == nullptr;
    const bool rrp = rrp_env && f.p < 4096u && f.mu32;
    // left-looking rounds over a shared Gauss-Jordan basis (k_rrp2); FFB_RRP_V1: the right-looking kernel (A/B hook)
    static const bool rrp2_env = getenv("FFB_RRP_V1") == nullptr;
    const bool rrp2 = rrp && rrp2_env;
    // detection stops after kcap rows and cuts the chunk there, so every chunk takes the
    // register-resident CRP kernels (k <= 32) and stays in the pipeline; FFB_PLDUQ_KCAP=0: no cap (A/B hook)
    static const int kcap_env = getenv("FFB_PLDUQ_KCAP") ? atoi(getenv("FFB_PLDUQ_KCAP")) : 32;
    const int kcap = rrp2 ? kcap_env : 0;
    // chunk rows (taller chunks with the cap, 160 / 192 / 256 rows: 86.8 / 86.2 / 86.1 ms against 86.6 ms
    // on config 5 -- not worth a second size for the exact path's buffers)
    const int B = 128;
    const int SK = (sk_env > 0 && sk_env <= RD_S) ? sk_env : RD_S;
    PlduqOut out;
    const size_t mark0 = ws.mark();
    DMat Uhat = ws.mat(std::max<int64_t>(mn, 1), n);
    DMat UO = ws.mat(std::max<int64_t>(mn, 1), SK);   // Uhat * Omega
    // adaptive chunks: sparse residuals take up to RD_MAX_ROWS rows per chunk (narrow detection)
    const bool adaptive = SK > RD_NARROW && rd_narrow_on && !getenv("FFB_PLDUQ_FIXED_CHUNKS");
    const int Bmax = adaptive ? RD_MAX_ROWS : B;
    DMat RIb[2] = {ws.mat(B, n), ws.mat(B, n)};
    DMat RI = RIb[0], Gs = ws.mat(Bmax, std::max<int64_t>(mn, 1));
    DMat Kinv = ws.mat(B, B), Gi = ws.mat(B, std::max<int64_t>(mn, 1)), Gi2 = ws.mat(B, std::max<int64_t>(mn, 1));
    // the echelon U of the PLDUQ, chunk by chunk: rows (D^-1 L^-1)_c R_I in pivot order, natural
    // columns (k_crp_finish's Ld block times R_I), with D written into io.d as the chunks go;
    // the factor phase then needs no LDU of K (FFB_PLDUQ_LDU: the LDU-based phase, A/B hook)
    static const bool ufull_env = getenv("FFB_PLDUQ_LDU") == nullptr;
    DMat Ldb = ws.mat(B, B), Ufull = ufull_env ? ws.mat(std::max<int64_t>(mn, 1), n) : DMat{};
    DMat Gi3 = ws.mat(B, std::max<int64_t>(mn, 1)), Cg = ws.mat(B, B);
    DMat Upd = ws.mat(std::max<int64_t>(mn, 1), B);
    const int nblk0 = (int)cdiv(n, CRP_W);
    int32_t* dinfo = ws.vec<int32_t>(2 * Bmax + 16);  // row detect: k, I[0..k)
    int32_t* lists[2] = {ws.vec<int32_t>((int64_t)nblk0 * B), ws.vec<int32_t>((int64_t)nblk0 * B)};
    int32_t* counts[2] = {ws.vec<int32_t>(nblk0), ws.vec<int32_t>(nblk0)};
    int32_t* dflag = ws.vec<int32_t>(4);
    int32_t* dsig = ws.vec<int32_t>(B);
    uint32_t* re_scratch = ws.vec<uint32_t>((int64_t)nblk0 * CRP_KMAX + 64);  // candidate list
    // pivot rows, pivot columns (pivot order) and the pivot column of each Uhat row,
    // adjacent: one read-back after the row loop
    const int64_t pstride = (std::max<int64_t>(mn, 1) + 63) / 64 * 64;
    int32_t* d_prow = ws.vec<int32_t>(3 * pstride);
    int32_t* d_pcol = d_prow + pstride;
    int32_t* d_uhat_col = d_prow + 2 * pstride;

    const size_t rd_smem = std::max({rd_smem_bytes(RD_MAX_B, SK), rd_smem_bytes(RD_MAX_ROWS, RD_NARROW),
                                      rd_smem_bytes(PIPE_KMAX + 128, SK)});
    const size_t crp_smem = ((size_t)CRP_KMAX * CRP_KMAX + 2 * (size_t)CRP_G * CRP_KMAX) * 4;
    static DeviceOnce attrs;
    if (!attrs.done()) {
        FFB_CUDA(cudaFuncSetAttribute(k_row_detect<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rd_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_row_detect<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rd_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_row_detect<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rd_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_crp_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)crp_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_pair2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * CRP_KMAX * CRP_KMAX * 4)));
        FFB_CUDA(cudaFuncSetAttribute(k_crp_rowelim, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        FFB_CUDA(cudaFuncSetAttribute(k_crp_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)((size_t)CF_SMEM_WORDS * 4)));
        attrs.mark();
    }
    static const bool force_exact = getenv("FFB_PLDUQ_FORCE_FALLBACK") != nullptr;  // test hook
    // register-resident local CRPs (k_crp_list_reg) for k <= 32, p < 2^16; FFB_CRP_SCAN: the scan kernel (A/B hook)
    static const bool crp_reg_env = getenv("FFB_CRP_SCAN") == nullptr;
    const bool crp_reg = crp_reg_env && f.p < 4096u && f.mu32;

    // side stream for the Uhat updates (see absorb)
    // (per device: a thread may drive contexts on several GPUs)
    struct SideStreams {
        cudaStream_t side = nullptr, side2 = nullptr, side3 = nullptr, side4 = nullptr;
        cudaEvent_t ev_main = nullptr, ev_side = nullptr, ev_gk = nullptr, ev_si = nullptr, ev_sk = nullptr,
                    ev_det = nullptr, ev_t1 = nullptr, ev_un = nullptr, ev_uf = nullptr;
    };
    static thread_local SideStreams side_dev[FFB_MAX_DEVICES];
    SideStreams& ss = side_dev[current_device()];
    static const bool overlap_ok = !getenv("FFB_PLDUQ_NO_OVERLAP");  // test hook
    if (!ss.side) {
        int least = 0, greatest = 0;  // lowest priority: the main stream's chunk kernels go first
        FFB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        ss.side = make_side_stream(least);  // the Uhat absorb: in the bulk-update SM partition
        // side2: pipelined sketch + row detection of the next chunk (highest priority: its
        // 1-CTA detection is latency-bound and must not queue behind the Uhat updates)
        FFB_CUDA(cudaStreamCreateWithPriority(&ss.side2, cudaStreamNonBlocking, greatest));
        FFB_CUDA(cudaStreamCreateWithPriority(&ss.side3, cudaStreamNonBlocking, greatest));
        FFB_CUDA(cudaStreamCreateWithPriority(&ss.side4, cudaStreamNonBlocking, greatest));  // T1 of the next chunk
        for (cudaEvent_t* e : {&ss.ev_main, &ss.ev_side, &ss.ev_gk, &ss.ev_si, &ss.ev_sk, &ss.ev_det, &ss.ev_t1,
                               &ss.ev_un, &ss.ev_uf})
            FFB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    cudaStream_t side = ss.side, side2 = ss.side2, side3 = ss.side3, side4 = ss.side4;
    cudaEvent_t ev_main = ss.ev_main, ev_side = ss.ev_side, ev_gk = ss.ev_gk, ev_si = ss.ev_si, ev_sk = ss.ev_sk,
                ev_det = ss.ev_det, ev_t1 = ss.ev_t1, ev_un = ss.ev_un, ev_uf = ss.ev_uf;
    static const bool pipe_on = overlap_ok && !getenv("FFB_PLDUQ_NO_PIPE");  // A/B hook
    DMat T2[2] = {ws.mat(PIPE_KMAX + B, SK), ws.mat(PIPE_KMAX + B, SK)};
    int32_t* pinfo[2] = {ws.vec<int32_t>(2 * (PIPE_KMAX + B) + 16), ws.vec<int32_t>(2 * (PIPE_KMAX + B) + 16)};
    // pre-basis of the pipelined detection: reduced rows of S_I(c) (k_row_detect on S_I alone)
    uint32_t* Epre = ws.vec<uint32_t>((int64_t)PIPE_KMAX * RD_PIPE);
    int32_t* rho_pre = ws.vec<int32_t>(PIPE_KMAX);
    int32_t* pre_out = ws.vec<int32_t>(2 * PIPE_KMAX + 16);
    const size_t mark1b = ws.mark();
    bool side_pending = false;
    auto join_side = [&]() {
        if (side_pending) {
            FFB_CUDA(cudaStreamWaitEvent(st, ev_side, 0)); pdl_fence(st);
            side_pending = false;
        }
    };

    // Given the chunk's pivot rows (device dI: chunk-local rows, k of them, with
    // R_I in RI) and pivot column set dJ (ascending): pairing, Unew into Uhat
    // rows [r, r+k), old rows reduced at J, Uhat*Omega maintained when sketching.
    auto absorb = [&](int64_t r, int k, const int32_t* dI, const int32_t* dJ, int64_t c0,
                      bool sketching, const int32_t* sigma_in, DMat Sk, bool paired,
                      const std::function<bool()>& mid = {}) {
        DMat RIk = RI.sub(0, 0, k, n), Kik = Kinv.sub(0, 0, k, k);
        Kik.ld = k;
        if (!paired) {
            ProfScope ps(K_PQ_PAIR, st, 0.0, 0.0);
            launch_k(k_pair2, 1, 256, (size_t)3 * k * k * 4, st, f, RIk.ptr, RIk.ld, k, dJ, dI, c0, sketching ? Sk.ptr : nullptr, Sk.ld, SK, Kik.ptr,
                UO.ptr, UO.ld, d_uhat_col, d_prow, d_pcol, r, dflag, sigma_in);
            ++g_launches;
            FFB_CHECK_LAUNCH();
        }
        DMat Un = Uhat.sub(r, 0, k, n);
        // Unew = Kc^-1 R_I and Uhat_old -= Up Unew are needed only by the next
        // chunk's residual: when sketching they run on the side stream, overlapped
        // with the next chunk's sketch, row detection and read-back (join_side).
        // Unew goes first (the next chunk's residual correction waits for it, ev_un),
        // the echelon U rows after it (ev_uf), then the main-stream part (Up, Uhat Omega).
        cudaStream_t us = st;
        if (sketching && overlap_ok) {
            FFB_CUDA(cudaEventRecord(ev_main, st));
            FFB_CUDA(cudaStreamWaitEvent(side, ev_main, 0)); pdl_fence(side);
            us = side;
        }
        {
            GreenScope green(us != st);
            SlotGuard slot(us == st ? g_slot : 1);
            gemm(f, us, GEMM_SET, Un, Kik, false, RIk, false, k, n, k);  // Unew = Kc^-1 R_I
            FFB_CUDA(cudaEventRecord(ev_un, us));
            if (ufull_env && paired) {  // the chunk's rows of the echelon U (before RI is reused)
                DMat Ldk = Ldb.sub(0, 0, k, k);
                Ldk.ld = k;
                gemm(f, us, GEMM_SET, Ufull.sub(r, 0, k, n), Ldk, false, RIk, false, k, n, k);
            }
            FFB_CUDA(cudaEventRecord(ev_uf, us));
        }
        DMat Up;
        if (r > 0) {  // Up = Uhat_old[:, J] before Uhat_old changes
            Up = Upd.sub(0, 0, r, k);
            gather2d(st, Up, Uhat.sub(0, 0, r, n), nullptr, dJ, 0);
            if (sketching)
                gemm(f, st, GEMM_SUB, UO.sub(0, 0, r, SK), Up, false, UO.sub(r, 0, k, SK), false, r,
                     SK, k);
        }
        // mid: issued between the main-stream part and the Uhat update (the pipelined next
        // chunk's T1, which must read Uhat_old before the update below); true: wait for it
        const bool t1_wait = mid ? mid() : false;
        if (us != st) {
            FFB_CUDA(cudaEventRecord(ev_main, st));
            FFB_CUDA(cudaStreamWaitEvent(side, ev_main, 0)); pdl_fence(side);
        }
        {
            GreenScope green(us != st);
            SlotGuard slot(us == st ? g_slot : 1);
            if (t1_wait) {  // the next chunk's T1 reads Uhat_old first
                FFB_CUDA(cudaStreamWaitEvent(us, ev_t1, 0)); pdl_fence(us);
            }
            if (r > 0) gemm(f, us, GEMM_SUB, Uhat.sub(0, 0, r, n), Up, false, Un, false, r, n, k);
            if (us != st) {
                FFB_CUDA(cudaEventRecord(ev_side, side));
                side_pending = true;
            }
        }
    };

    int64_t r = 0;
    bool exact = force_exact;
    for (int attempt = 0; attempt < 2; ++attempt) {
        ws.release(mark1b);
        r = 0;
        fill_words(st, (uint32_t*)dflag, 1, 0u);
        DMat YO, Om;
        phase_mark("pq: begin", m + n, st);
        if (!exact) {  // Y * Omega, once
            Om = ws.mat(n, SK);
            launch_k(k_random, (unsigned)cdiv(n * SK, 256), 256, 0, st, Om.ptr, n * SK, 0x5EEDull + n + 977 * attempt, f.p);
            ++g_launches;
            YO = ws.mat(m, SK);
            gemm(f, st, GEMM_SET, YO, Y, false, Om, false, m, SK, n);
        }
        // diagnostics: FFB_PLDUQ_CHUNK_TRACE=<file> records event marks per chunk (m >= 4096)
        static FILE* ctr = getenv("FFB_PLDUQ_CHUNK_TRACE") ? fopen(getenv("FFB_PLDUQ_CHUNK_TRACE"), "a") : nullptr;
        const bool ctrace = ctr && m >= 4096;
        std::vector<cudaEvent_t> cev;
        auto mark = [&]() {
            if (!ctrace) return;
            cudaEvent_t e;
            cudaEventCreate(&e);
            cudaEventRecord(e, st);
            cev.push_back(e);
        };
        // chunk rows: 128, or a multiple of 128 up to RD_MAX_ROWS where the previous chunk was
        // sparse, aiming at ~24 detected rows per chunk (a chunk costs ~55 us + ~9 us per
        // detected row; measured sweep of the target: 16 / 24 / 32 / 40 -> 128.3 / 126.7 /
        // 126.8 / 128.3 ms on config 5)
        // the first chunk is optimistic (the largest narrow chunk): residuals that reach
        // the parallel path are mostly sparse, and a dense first chunk only costs a shrink
        static const bool first_big = getenv("FFB_PLDUQ_FIRST_128") == nullptr;  // A/B hook
        int64_t bc = 0, Bcur = (adaptive && first_big) ? RD_MAX_ROWS : B;
        // pipelined detection (dense chunks): chunk c+1's sketch and row detection run on
        // side2 beside chunk c's residual / CRP / finish.  The sketch of c+1 is taken
        // against the basis before chunk c (UO[0:r], r at chunk c), so the detection is
        // run on the stack [S_I(c); S(c+1)]: S_I(c) = sketches of chunk c's detected rows
        // against the same basis, inserted first.  A row of c+1 independent of them and
        // of its earlier rows (modulo span(Uhat_old)) is independent of span(Uhat_new).
        phase_mark("pq: Y Omega", m + n, st);
        bool pre = false, pre_done = false, t1 = false;
        int pre_k = 0, pb = 0, pre_kt = 0, rb = 0, prev_k = 0;
        RI = RIb[0];
        int64_t pre_bc = 0;
        MboxPost pre_mp;
        for (int64_t c0 = 0; c0 < m; c0 += bc) {
            bc = std::min<int64_t>(exact ? B : Bcur, m - c0);
            if (pre) bc = pre_bc;
            DMat Yc = Y.sub(c0, 0, bc, n);
            mark();
            if (!exact) {
                DMat Sc = YO.sub(c0, 0, bc, SK);
                int k = 0, cut = 0;
                const int32_t* dI = dinfo + 1;
                int64_t base = c0;  // row c0' + dI[t] of Y is detected row t
                bool det_pipe = false;
                bool use_t1 = false;
                if (pre) {
                    pre = false;
                    const int32_t word =
                        pre_done ? pre_kt : *(const int32_t*)(pre_mp.dst ? io.wait(pre_mp) : io.readback(pinfo[pb], 4));
                    const int kt = word & 0xffff;
                    pre_done = false;
                    use_t1 = t1;
                    t1 = false;
                    FFB_CUDA(cudaStreamWaitEvent(st, ev_det, 0)); pdl_fence(st);
                    if (pre_k + kt <= PIPE_TRUST) {
                        k = kt;
                        dI = pinfo[pb] + 1;
                        det_pipe = true;
                        if ((word >> 16) > 0 && (word >> 16) < bc) {  // capped: the chunk ends at the cut
                            bc = word >> 16;
                            Yc = Y.sub(c0, 0, bc, n);
                            Sc = YO.sub(c0, 0, bc, SK);
                        }
                    }  // else: near the sketch capacity -- detect again below, serially
                }
                if (!det_pipe) {
                    // sketch of the chunk residual, in place in its (otherwise unused)
                    // rows of Y*Omega: S = (Y Omega)_c - Y_c[:, pc] (Uhat Omega), a GEMM
                    if (r > 0) {
                        DMat Gc = Gs.sub(0, 0, bc, r);
                        {
                            ProfScope ps(K_PQ_SKETCH, st, 0.0, 0.0);
                            gather2d(st, Gc, Yc, nullptr, d_uhat_col, 0);
                        }
                        gemm(f, st, GEMM_SUB, Sc, Gc, false, UO.sub(0, 0, r, SK), false, bc, SK, r);
                    }
                    mark();
                    // row detection on the first RD_NARROW sketch columns (2 ballot groups instead
                    // of 5): rows independent there are independent in R; a chunk that finds
                    // k >= RD_NARROW - 16 may have more than the narrow sketch can show, and is
                    // re-detected on all SK columns (the certificate guards both)
                    for (int wide = (SK <= RD_NARROW || !rd_narrow_on) ? 1 : 0; wide < 2; ++wide) {
                        if (wide && bc > B) {
                            // a dense chunk after all: keep its first B rows; the sketch rows
                            // after them were overwritten in place and are recomputed, Y Omega
                            gemm(f, st, GEMM_SET, YO.sub(c0 + B, 0, bc - B, SK), Y.sub(c0 + B, 0, bc - B, n), false, Om,
                                 false, bc - B, SK, n);
                            bc = B;
                            Yc = Y.sub(c0, 0, bc, n);
                            Sc = YO.sub(c0, 0, bc, SK);
                        }
                        const MboxPost mp = io.post ? io.post() : MboxPost();
                        {
                            ProfScope ps(K_PLDUQ, st, 0.0, 0.0);
                            if (rrp2 && wide)
                                launch_k(k_rrp2<5, 8>, 1, 256, 0, st, f, Sc.ptr, Sc.ld, (int)bc, SK, dinfo, mp, nullptr,
                                         nullptr, nullptr, nullptr, nullptr, kcap);
                            else if (rrp2)
                                launch_k(k_rrp2<2, 32>, 1, 1024, 0, st, f, Sc.ptr, Sc.ld, (int)bc, RD_NARROW, dinfo, mp,
                                         nullptr, nullptr, nullptr, nullptr, nullptr, kcap);
                            else if (rrp && wide)
                                launch_k(k_rrp<5, 16, 8>, 1, 256, 0, st, f, Sc.ptr, Sc.ld, (int)bc, SK, dinfo, mp, nullptr,
                                         nullptr, nullptr, nullptr);
                            else if (rrp)
                                launch_k(k_rrp<2, 20, 32>, 1, 1024, 0, st, f, Sc.ptr, Sc.ld, (int)bc, RD_NARROW, dinfo, mp,
                                         nullptr, nullptr, nullptr, nullptr);
                            else if (wide)
                                launch_k(k_row_detect<5>, 1, 256, rd_smem_bytes((int)bc, SK), st, f, Sc.ptr, Sc.ld, (int)bc,
                                         SK, dinfo, mp, nullptr, nullptr, nullptr, nullptr, nullptr);
                            else
                                launch_k(k_row_detect<2>, 1, 256, rd_smem_bytes((int)bc, RD_NARROW), st, f, Sc.ptr, Sc.ld,
                                         (int)bc, RD_NARROW, dinfo, mp, nullptr, nullptr, nullptr, nullptr, nullptr);
                            ++g_launches;
                            FFB_CHECK_LAUNCH();
                        }
                        const int32_t word = *(const int32_t*)(mp.dst ? io.wait(mp) : io.readback(dinfo, 4));
                        k = word & 0xffff;
                        cut = word >> 16;
                        if (k < RD_NARROW - 16) break;
                    }
                    if (cut > 0 && cut < bc) {  // capped: the rows after the cut go to the next chunk;
                        // their sketch rows were overwritten in place and are recomputed, Y Omega
                        if (r > 0)
                            gemm(f, st, GEMM_SET, YO.sub(c0 + cut, 0, bc - cut, SK), Y.sub(c0 + cut, 0, bc - cut, n),
                                 false, Om, false, bc - cut, SK, n);
                        bc = cut;
                        Yc = Y.sub(c0, 0, bc, n);
                        Sc = YO.sub(c0, 0, bc, SK);
                    }
                } else {
                    mark();
                }
                if (adaptive) {  // next chunk size from this chunk's density
                    static const double tk = getenv("FFB_PLDUQ_TARGET_K") ? atof(getenv("FFB_PLDUQ_TARGET_K")) : 24.0;
                    static const int64_t rmax = getenv("FFB_PLDUQ_MAX_ROWS") ? atoll(getenv("FFB_PLDUQ_MAX_ROWS")) : RD_MAX_ROWS;
                    const int64_t cap = std::min<int64_t>(rmax, RD_MAX_ROWS);
                    const double target = k > 0 ? std::min(tk * (double)bc / k, (double)cap) : (double)cap;
                    Bcur = std::min<int64_t>(std::max<int64_t>((int64_t)(target / B) * B, B), cap);
                }
                mark();
                if (k == 0) {
                    mark(); mark(); mark();
                    continue;
                }
                // On side2, beside this chunk's residual / CRP / finish: S_I against the
                // current basis in T rows [0, k) (a detected chunk's own sketch rows when it
                // was detected serially; recomputed from Y Omega after a pipelined
                // detection), then chunk c+1's sketch and its stacked detection on the
                // first RD_PIPE sketch columns
                const int64_t c0n = c0 + bc;
                const bool pipe = pipe_on && SK == RD_S && c0n < m && Bcur == B && k <= PIPE_KMAX;
                const bool compact = pipe || det_pipe;
                DMat Sfin = Sc;
                if (compact) {
                    pb ^= 1;
                    DMat T = T2[pb];
                    FFB_CUDA(cudaEventRecord(ev_gk, st));
                    FFB_CUDA(cudaStreamWaitEvent(side2, ev_gk, 0)); pdl_fence(side2);
                    SlotGuard slot(3);
                    Sfin = T.sub(0, 0, k, SK);
                    if (det_pipe) {
                        gather_rows(side2, Sfin, YO.sub(base, 0, m - base, SK), dI);
                        if (r > 0) {
                            DMat Gk2 = Gi2.sub(0, 0, k, r);
                            gather2d(side2, Gk2, Y, dI, d_uhat_col, base);
                            gemm(f, side2, GEMM_SUB, Sfin, Gk2, false, UO.sub(0, 0, r, SK), false, k, SK, r);
                        }
                    } else {
                        gather_rows(side2, Sfin, Sc, dI);
                    }
                    FFB_CUDA(cudaEventRecord(ev_si, side2));
                    if (pipe) {
                        const int64_t bcn = std::min<int64_t>(B, m - c0n);
                        // the reduced basis of S_I (side2) beside chunk c+1's sketch (side3),
                        // then the detection of c+1 modulo that basis (side2)
                        if (rrp2)
                            launch_k(k_rrp2<3, 8>, 1, 256, 0, side2, f, Sfin.ptr, Sfin.ld, k, RD_PIPE, pre_out,
                                     MboxPost(), nullptr, nullptr, nullptr, Epre, rho_pre, 0);
                        else if (rrp)
                            launch_k(k_rrp<3, 20, 8>, 1, 256, 0, side2, f, Sfin.ptr, Sfin.ld, k, RD_PIPE, pre_out,
                                     MboxPost(), nullptr, nullptr, Epre, rho_pre);
                        else
                            launch_k(k_row_detect<3>, 1, 256, rd_smem_bytes(k, RD_PIPE), side2, f, Sfin.ptr, Sfin.ld,
                                     k, RD_PIPE, pre_out, MboxPost(), nullptr, nullptr, nullptr, Epre, rho_pre);
                        ++g_launches;
                        FFB_CUDA(cudaStreamWaitEvent(side3, ev_gk, 0)); pdl_fence(side3);
                        SlotGuard slot3(4);
                        DMat Sn = T.sub(PIPE_KMAX, 0, bcn, SK);
                        launch_k(k_copy_rows, dim3(1, (unsigned)bcn), 160, 0, side3, Sn.ptr, Sn.ld,
                                 YO.ptr + c0n * YO.ld, YO.ld, (int64_t)SK);
                        ++g_launches;
                        if (r > 0) {
                            DMat Gc = Gs.sub(0, 0, bcn, r);
                            gather2d(side3, Gc, Y.sub(c0n, 0, bcn, n), nullptr, d_uhat_col, 0);
                            gemm(f, side3, GEMM_SUB, Sn, Gc, false, UO.sub(0, 0, r, SK), false, bcn, SK, r);
                        }
                        FFB_CUDA(cudaEventRecord(ev_sk, side3));
                        FFB_CUDA(cudaStreamWaitEvent(side2, ev_sk, 0)); pdl_fence(side2);
                        pre_mp = io.post ? io.post() : MboxPost();
                        {
                            ProfScope ps(K_PLDUQ, side2, 0.0, 0.0);
                            if (rrp2)
                                launch_k(k_rrp2<3, 8>, 1, 256, 0, side2, f, Sn.ptr, Sn.ld, (int)bcn, RD_PIPE,
                                         pinfo[pb], pre_mp, Epre, rho_pre, pre_out, nullptr, nullptr, kcap);
                            else if (rrp)
                                launch_k(k_rrp<3, 20, 8>, 1, 256, 0, side2, f, Sn.ptr, Sn.ld, (int)bcn, RD_PIPE,
                                         pinfo[pb], pre_mp, Epre, pre_out, nullptr, nullptr);
                            else
                                launch_k(k_row_detect<3>, 1, 256, rd_smem_bytes_pre((int)bcn, RD_PIPE), side2, f,
                                         Sn.ptr, Sn.ld, (int)bcn, RD_PIPE, pinfo[pb], pre_mp, Epre, rho_pre, pre_out,
                                         nullptr, nullptr);
                            ++g_launches;
                            FFB_CHECK_LAUNCH();
                        }
                        FFB_CUDA(cudaEventRecord(ev_det, side2));
                        if (!pre_mp.dst) {  // read-back without a mailbox: plain copy after the event
                            FFB_CUDA(cudaStreamWaitEvent(st, ev_det, 0)); pdl_fence(st);
                        }
                        pre = true;
                        pre_k = k;
                        pre_bc = bcn;
                    }
                }
                DMat RIk;
                if (use_t1) {
                    // T1 = Y_I - Y_I[:, pc_old] Uhat_old was computed on side2 beside the previous
                    // chunk's CRP (other RI buffer); with that chunk's rows Unew (pivot columns J):
                    //   R_I = Y_I - Y_I[:, pc_new] Uhat_new = T1 - T1[:, J] Unew
                    // so the Uhat_old update stays off this chain
                    rb ^= 1;
                    RI = RIb[rb];
                    RIk = RI.sub(0, 0, k, n);
                    FFB_CUDA(cudaStreamWaitEvent(st, ev_t1, 0));
                    FFB_CUDA(cudaStreamWaitEvent(st, ev_un, 0)); pdl_fence(st);
                    DMat Ck = Cg.sub(0, 0, k, prev_k);
                    gather2d(st, Ck, RIk, nullptr, lists[1], 0);
                    gemm(f, st, GEMM_SUB, RIk, Ck, false, Uhat.sub(r - prev_k, 0, prev_k, n), false, k, n, prev_k);
                } else {
                    join_side();  // the previous chunk's Uhat update, before RI / Kinv / Upd are reused
                    // exact residual of the k detected rows: R_I = Y_I - Y_I[:, pc] Uhat
                    RIk = RI.sub(0, 0, k, n);
                    const DMat Yb = Y.sub(base, 0, m - base, n);
                    gather_rows(st, RIk, Yb, dI);
                    DMat Gk = Gi.sub(0, 0, k, r);
                    if (r > 0) {
                        gather2d(st, Gk, Y, dI, d_uhat_col, base);
                        gemm(f, st, GEMM_SUB, RIk, Gk, false, Uhat.sub(0, 0, r, n), false, k, n, r);
                    }
                }
                mark();
                {
                    ProfScope ps(K_PQ_CRP, st, 0.0, 0.0);
                    // level 0: local CRPs of 256-column blocks (parallel)
                    if (crp_reg && k <= 16)
                        launch_k(k_crp_list_reg<16>, nblk0, 256, 0, st, f, RI.ptr, RI.ld, k, n, lists[0], counts[0]);
                    else if (crp_reg && k <= 32)
                        launch_k(k_crp_list_reg<32>, nblk0, 256, 0, st, f, RI.ptr, RI.ld, k, n, lists[0], counts[0]);
                    else
                        launch_k(k_crp_list, nblk0, 256, crp_smem, st, f, RI.ptr, RI.ld, k, n, lists[0], counts[0]);
                    ++g_launches;
                }
                if (compact) {
                    FFB_CUDA(cudaStreamWaitEvent(st, ev_si, 0)); pdl_fence(st);
                }
                if (use_t1) {  // the finish rewrites Ldb: the previous chunk's echelon-U GEMM reads it
                    FFB_CUDA(cudaStreamWaitEvent(st, ev_uf, 0)); pdl_fence(st);
                }
                {
                    ProfScope ps(K_PQ_ROWELIM, st, 0.0, 0.0);
                    // RPM of R_I on the candidates, Kinv and bookkeeping (1 CTA)
                    int rc_cap, si_off;
                    const size_t cfmem = cf_smem_bytes(k, nblk0, &rc_cap, &si_off);
                    static const int rc_lim = getenv("FFB_CF_DIRECT_MAX") ? atoi(getenv("FFB_CF_DIRECT_MAX")) : -1;
                    if (rc_lim >= 0) rc_cap = std::min(rc_cap, rc_lim);  // A/B hook: direct vs scan path
                    DMat Kik = Kinv.sub(0, 0, k, k);
                    // register-resident finish (k <= 32, p <= 255); FFB_CF_SMEM: the smem kernel (A/B hook)
                    static const bool cf_reg_env = getenv("FFB_CF_SMEM") == nullptr;
                    if (cf_reg_env && f.p <= 255u && k <= 32 && nblk0 <= CFR_MAXBLK && nblk0 * k <= CFR_MAXC && SK <= RD_S)
                        launch_k(k_crp_finish_reg, 1, 1024, 0, st, f, RI.ptr, RI.ld, k, lists[0], counts[0], nblk0, dI,
                                 base, Sfin.ptr, Sfin.ld, SK, Kik.ptr, lists[1], UO.ptr, UO.ld, d_uhat_col, d_prow,
                                 d_pcol, r, dflag, compact ? 1 : 0, Ldb.ptr, io.d + r);
                    else
                    launch_k(k_crp_finish, 1, 256, cfmem, st, f, RI.ptr, RI.ld, k, lists[0], counts[0], nblk0,
                                                        (int32_t*)re_scratch, rc_cap, dI, base, Sfin.ptr, Sfin.ld, SK,
                                                        Kik.ptr, lists[1], UO.ptr, UO.ld, d_uhat_col,
                                                        d_prow, d_pcol, r, dflag, si_off, compact ? 1 : 0,
                                                        Ldb.ptr, io.d + r);
                    ++g_launches;
                    FFB_CHECK_LAUNCH();
                }
                if (pipe) {  // side2 read UO[0:r] and d_uhat_col[0:r]: before absorb changes UO
                    FFB_CUDA(cudaStreamWaitEvent(st, ev_sk, 0)); pdl_fence(st);
                }
                static const char* dump = getenv("FFB_PLDUQ_DUMP");  // diagnostics: one top-level R_I
                static int dumped = 0;
                if (dump && !dumped && n >= 16384 && c0 >= 20 * B) {
                    dumped = 1;
                    std::vector<uint32_t> h((size_t)k * n);
                    FFB_CUDA(cudaStreamSynchronize(st));
                    FFB_CUDA(cudaMemcpy2D(h.data(), n * 4, RI.ptr, RI.ld * 4, n * 4, k, cudaMemcpyDeviceToHost));
                    if (FILE* fd = fopen(dump, "wb")) {
                        const int64_t hdr[2] = {k, n};
                        fwrite(hdr, sizeof(hdr), 1, fd);
                        fwrite(h.data(), 4, h.size(), fd);
                        fclose(fd);
                    }
                }
                static FILE* jtr = getenv("FFB_PLDUQ_JTRACE") ? fopen(getenv("FFB_PLDUQ_JTRACE"), "a") : nullptr;
                if (jtr && !pre) {  // diagnostics: k, n, candidate count, pivot column positions
                    const int32_t* hc = (const int32_t*)io.readback(counts[0], (size_t)nblk0 * 4);
                    int64_t C = 0;
                    for (int b = 0; b < nblk0; ++b) C += hc[b];
                    const int32_t* hj = (const int32_t*)io.readback(lists[1], (size_t)k * 4);
                    fprintf(jtr, "%d %lld %lld %lld %d %d %d\n", k, (long long)n, (long long)C, (long long)r,
                            hj[0], hj[k / 2], hj[k - 1]);
                }
                bool t1_launch = false;
                // chunk c+1's detection (side2) ends before this finish: after the absorb's
                // main-stream part is queued, take its rows and start T1 = Y_I' - Y_I'[:, pc]
                // Uhat (current basis) on side2, before the Uhat update of this chunk
                auto launch_t1 = [&]() -> bool {
                    if (!pipe) return false;
                    pre_kt = *(const int32_t*)(pre_mp.dst ? io.wait(pre_mp) : io.readback(pinfo[pb], 4));
                    pre_done = true;
                    const int kn = pre_kt & 0xffff;
                    if (!(k + kn <= PIPE_TRUST && kn > 0)) return false;
                    SlotGuard slot(5);
                    DMat RIn = RIb[rb ^ 1].sub(0, 0, kn, n);
                    const int32_t* dIn = pinfo[pb] + 1;
                    const int64_t basen = c0n;
                    // on side4 (beside S_I and the stacked detection of the chunk after, side2):
                    // after the detection that wrote dIn; the chunk before this one read that RI
                    // buffer in its Unew / echelon GEMMs and Uhat must hold its update (ev_side)
                    FFB_CUDA(cudaStreamWaitEvent(side4, ev_det, 0));
                    FFB_CUDA(cudaStreamWaitEvent(side4, ev_side, 0));
                    pdl_fence(side4);
                    gather_rows(side4, RIn, Y.sub(basen, 0, m - basen, n), dIn);
                    if (r > 0) {
                        DMat G3 = Gi3.sub(0, 0, kn, r);
                        gather2d(side4, G3, Y, dIn, d_uhat_col, basen);
                        gemm(f, side4, GEMM_SUB, RIn, G3, false, Uhat.sub(0, 0, r, n), false, kn, n, r);
                    }
                    FFB_CUDA(cudaEventRecord(ev_t1, side4));
                    t1_launch = true;
                    return true;
                };
                join_side();  // Up below reads Uhat: the previous chunk's update first
                mark();
                absorb(r, k, dI, lists[1], base, true, dsig, Sc, true, launch_t1);
                t1 = t1_launch;
                prev_k = k;
                r += k;
            } else {
                // exact: residual of the whole chunk, then the row-sequential kernel
                join_side();
                const size_t mk = ws.mark();
                DMat Rc = ws.mat(bc, n);
                copy_mat(st, Rc, Yc);
                if (r > 0) {
                    DMat Gk = Gi.sub(0, 0, bc, r);
                    gather2d(st, Gk, Yc, nullptr, d_uhat_col, 0);
                    gemm(f, st, GEMM_SUB, Rc, Gk, false, Uhat.sub(0, 0, r, n), false, bc, n, r);
                }
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
                if (k > 0) {
                    const int32_t* dI = io.upload(I);
                    gather_rows(st, RI.sub(0, 0, k, n), Rc, dI);
                    absorb(r, k, dI, io.upload(J), c0, false, nullptr, DMat{}, false);
                    r += k;
                }
                ws.release(mk);
            }
        }
        join_side();
        phase_mark("pq: chunk loop", m + n, st);
        if (ctrace && !cev.empty()) {  // 5 marks per chunk: start, detect, readback, crp, finish
            mark();
            cudaEventSynchronize(cev.back());
            double acc[5] = {0, 0, 0, 0, 0};
            const size_t nc = (cev.size() - 1) / 5;
            for (size_t c = 0; c < nc; ++c)
                for (int j = 0; j < 5; ++j) {
                    float t = 0;
                    cudaEventElapsedTime(&t, cev[5 * c + j], cev[5 * c + j + 1]);
                    acc[j] += t;
                }
            fprintf(ctr, "m=%lld n=%lld chunks=%zu sketch=%.2f detect+post=%.2f gathers+residual=%.2f crp+finish=%.2f absorb+next=%.2f ms\n",
                    (long long)m, (long long)n, nc, acc[0], acc[1], acc[2], acc[3], acc[4]);
            fflush(ctr);
            for (auto e : cev) cudaEventDestroy(e);
        }
        out.r = r;
        std::vector<int32_t> pr, pcol_rows, uhat_cols;
        if (r > 0) {  // d_prow, d_pcol and d_uhat_col are adjacent: one read-back
            const int32_t* hp = (const int32_t*)io.readback(d_prow, (size_t)(3 * pstride) * 4);
            pr.assign(hp, hp + r);
            pcol_rows.assign(hp + pstride, hp + pstride + r);
            uhat_cols.assign(hp + 2 * pstride, hp + 2 * pstride + r);
        }

        // ---- phase 2: factors from the pivots ----
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
        if (io.pivots_ready && r > 0) io.pivots_ready(out.cimg);
        if (r == 0) {
            if (exact) break;
            // certificate: Y must be zero
            any_nonzero(st, Y, dflag);
            if (*(const int32_t*)io.readback(dflag, 4) == 0) break;
            ++out.fallbacks;
            exact = true;
            continue;
        }
        // every index array of phase 2 and the certificate in one upload (one fetch launch)
        const int64_t rA = (r + 3) & ~3, nA = (n + 3) & ~3, mA = (m + 3) & ~3;
        std::vector<int32_t> idx((size_t)(3 * rA + nA + 2 * mA), 0);
        {  // upos[t]: the Uhat row whose pivot column is pc[t]
            std::vector<int32_t> at(n, -1);
            for (int64_t i = 0; i < r; ++i) at[uhat_cols[i]] = (int32_t)i;
            for (int64_t t = 0; t < r; ++t) idx[2 * rA + nA + 2 * mA + t] = at[pcol_rows[t]];
        }
        std::copy(pr.begin(), pr.end(), idx.begin());
        std::copy(pcol_rows.begin(), pcol_rows.end(), idx.begin() + rA);
        std::copy(out.cimg.begin(), out.cimg.end(), idx.begin() + 2 * rA);
        std::copy(out.rimg.begin() + r, out.rimg.end(), idx.begin() + 2 * rA + nA);
        std::copy(out.rimg.begin(), out.rimg.end(), idx.begin() + 2 * rA + nA + mA);
        const int32_t* didx = io.upload(idx);
        const int32_t* dpr = didx;
        const int32_t* dpc = didx + rA;
        DMat Uo = io.Uo.sub(0, 0, r, n);
        const int32_t* dcimg = didx + 2 * rA;
        const int32_t* dnp = nullptr;
        if (!exact && ufull_env) {
            // U = the echelon rows gathered by Q; D from the chunks; [L1; M1] = Y[P, pc] U1^-1 D^-1
            // for all m rows at once (K = L1 D U1 gives L1 exactly: unit lower, no LDU of K)
            gather2d(st, Uo, Ufull.sub(0, 0, r, n), nullptr, dcimg, 0);
            invert_vec(f, st, io.dinv, io.d, r);
            DMat T = ws.mat(m, r), Tt = ws.mat(r, m), U1t = ws.mat(r, r);
            gather2d(st, T, Y, didx + 2 * rA + nA + mA, dpc, 0);
            transpose(st, Tt, T);
            transpose(st, U1t, Uo.sub(0, 0, r, r));
            trsm_lower_unit(f, st, U1t, Tt);
            scale_T(f, st, io.Lo.sub(0, 0, m, r), Tt, io.dinv);
            if (m > r) dnp = didx + 2 * rA + nA;
        } else {
        DMat Kf = ws.mat(r, r);
        gather2d(st, Kf, Y, dpr, dpc, 0);
        ldu_inplace(f, st, Kf, ws, dflag);
        launch_k(k_unpack_l, rgrid(r, r), 256, 0, st, io.Lo.ptr, io.Lo.ld, Kf.ptr, Kf.ld, r, io.d, 1 % f.p);
        ++g_launches;
        invert_vec(f, st, io.dinv, io.d, r);
        {
            // U = D^-1 L1^-1 Y[pr, Q].  The row loop left Uhat = Y[pr, pcu]^-1 Y[pr, :]
            // (fully reduced: identity on its pivot columns pcu), and Y[pr, pcu] = K Pi with
            // K = L1 D U1, so U = U1 (Pi Uhat)[:, Q]: one r x r x n GEMM instead of the
            // r x r triangular solve on r x n right-hand sides
            DMat Ug = ws.mat(r, n), U1 = ws.mat(r, r);
            gather2d(st, Ug, Uhat.sub(0, 0, r, n), didx + 2 * rA + nA + 2 * mA, dcimg, 0);
            launch_k(k_unpack_u, rgrid(r, r), 256, 0, st, U1.ptr, U1.ld, Kf.ptr, Kf.ld, r, 1 % f.p);
            ++g_launches;
            gemm(f, st, GEMM_SET, Uo, U1, false, Ug, false, r, n, r);
        }
        if (m > r) {
            dnp = didx + 2 * rA + nA;
            DMat T = ws.mat(m - r, r), Tt = ws.mat(r, m - r), U1t = ws.mat(r, r);
            gather2d(st, T, Y, dnp, dpc, 0);
            transpose(st, Tt, T);
            transpose(st, U1t, Uo.sub(0, 0, r, r));
            trsm_lower_unit(f, st, U1t, Tt);
            scale_T(f, st, io.Lo.sub(r, 0, m - r, r), Tt, io.dinv);
        }
        }
        phase_mark("pq: factors", m + n, st);
        if (exact) {
            if (*(const int32_t*)io.readback(dflag, 4)) throw Status(FFB_ERROR, "plduq: singular pivot block");
            break;
        }
        // ---- certificate (sketch path only): Y - P L D U Q == 0, checked in place on Y in
        // its own order (no m x n gather): H = P (L D), Up = U Q; Y is not needed after the
        // PLDUQ, and a failed certificate adds the product back before the exact retry ----
        DMat H = ws.mat(m, r), Up = ws.mat(r, n);
        {
            launch_k(k_scale_cols, rgrid(m, r), 256, 0, st, f, H.ptr, H.ld, io.Lo.ptr, io.Lo.ld, io.d, r,
                     didx + 2 * rA + nA + mA);
            launch_k(k_scatter_cols, rgrid(r, n), 256, 0, st, Up.ptr, Up.ld, Uo.ptr, Uo.ld, dcimg, n);
            g_launches += 2;
            gemm(f, st, GEMM_SUB, Y, H, false, Up, false, m, n, r);
            any_nonzero(st, Y, dflag);
            if (m > r) {
                launch_k(k_m1_pattern, rgrid(m - r, r), 256, 0, st, io.Lo.ptr + r * io.Lo.ld, io.Lo.ld, dnp,
                                                              d_prow, r, dflag);
                ++g_launches;
            }
        }
        phase_mark("pq: certificate", m + n, st);
        if (*(const int32_t*)io.readback(dflag, 4) == 0) break;
        gemm(f, st, GEMM_ADD, Y, H, false, Up, false, m, n, r);  // Y restored for the exact retry
        ++out.fallbacks;  // a sketch missed rank: redo the search exactly
        exact = true;
    }
    ws.release(mark0);
    return out;
}

// ---------------------------------------------------------------------------
// Kernel micro-benchmark (tools/pq_kernel_bench.py; not part of the C-ABI):
//   which 0: row detection of S (rows x cols)         ms[0]
//   which 1: CRP list, row elimination, pairing of R  ms[0..2]
// on a device matrix, averaged over reps launches (CUDA events).
// ---------------------------------------------------------------------------
void dbg_pq_bench(const Fp& f, cudaStream_t st, int which, int rows, int cols, const uint32_t* d_in,
                  int reps, double* ms, int32_t* out_k) {
    cudaEvent_t e[4];
    for (auto& x : e) FFB_CUDA(cudaEventCreate(&x));
    float t = 0;
    if (which == 0) {
        const size_t rd_smem = ((size_t)2 * RD_MAX_B * cols + (size_t)RD_BATCH * cols) * 4;
        FFB_CUDA(cudaFuncSetAttribute(k_row_detect<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rd_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_row_detect<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rd_smem));
        int32_t* info;
        FFB_CUDA(cudaMalloc(&info, (2 * RD_MAX_B + 16) * 4));
        launch_k(k_row_detect<5>, 1, 256, rd_smem, st, f, d_in, cols, rows, cols, info, MboxPost(), nullptr, nullptr, nullptr, nullptr,
                 nullptr);
        FFB_CUDA(cudaEventRecord(e[0], st));
        for (int i = 0; i < reps; ++i) launch_k(k_row_detect<5>, 1, 256, rd_smem, st, f, d_in, cols, rows, cols, info, MboxPost(), nullptr, nullptr, nullptr, nullptr,
                 nullptr);
        FFB_CUDA(cudaEventRecord(e[1], st));
        FFB_CUDA(cudaEventSynchronize(e[1]));
        FFB_CUDA(cudaEventElapsedTime(&t, e[0], e[1]));
        ms[0] = t / reps;
        FFB_CUDA(cudaMemcpy(out_k, info, (size_t)(1 + std::min(rows, cols)) * 4, cudaMemcpyDeviceToHost));
        if (rows <= 128 && cols <= 160 && f.p < 4096u) {  // the register-resident kernel on the same sketch
            int32_t* info2;
            FFB_CUDA(cudaMalloc(&info2, (2 * RD_MAX_B + 16) * 4));
            auto rrp_k = k_rrp2<5, 8>;
            launch_k(rrp_k, 1, 256, 0, st, f, d_in, cols, rows, cols, info2, MboxPost(), nullptr, nullptr, nullptr,
                     nullptr, nullptr, 0);
            FFB_CUDA(cudaEventRecord(e[2], st));
            for (int i = 0; i < reps; ++i)
                launch_k(rrp_k, 1, 256, 0, st, f, d_in, cols, rows, cols, info2, MboxPost(), nullptr, nullptr,
                         nullptr, nullptr, nullptr, 0);
            FFB_CUDA(cudaEventRecord(e[3], st));
            FFB_CUDA(cudaEventSynchronize(e[3]));
            FFB_CUDA(cudaEventElapsedTime(&t, e[2], e[3]));
            ms[1] = t / reps;
            std::vector<int32_t> h2(1 + std::min(rows, cols));
            FFB_CUDA(cudaMemcpy(h2.data(), info2, h2.size() * 4, cudaMemcpyDeviceToHost));
            ms[2] = 1.0;  // identical row sets
            for (int j = 0; j <= h2[0] && j < (int)h2.size(); ++j)
                if (h2[j] != out_k[j]) ms[2] = 0.0;
            FFB_CUDA(cudaFree(info2));
        }
        FFB_CUDA(cudaFree(info));
    } else {
        const int k = rows;
        const int64_t n = cols;
        const int nblk0 = (int)cdiv(n, CRP_W);
        const size_t crp_smem = ((size_t)CRP_KMAX * CRP_KMAX + 2 * (size_t)CRP_G * CRP_KMAX) * 4;
        FFB_CUDA(cudaFuncSetAttribute(k_crp_list, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)crp_smem));
        FFB_CUDA(cudaFuncSetAttribute(k_crp_rowelim, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        FFB_CUDA(cudaFuncSetAttribute(k_crp_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)((size_t)CF_SMEM_WORDS * 4)));
        FFB_CUDA(cudaFuncSetAttribute(k_pair2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(3 * CRP_KMAX * CRP_KMAX * 4)));
        int32_t *lists0, *counts0, *lists1, *dsig, *flag, *ucol, *prow, *pcol, *dI;
        uint32_t *re_scratch, *Kinv;
        FFB_CUDA(cudaMalloc(&lists0, (size_t)nblk0 * k * 4));
        int32_t *lists_r, *counts_r;
        FFB_CUDA(cudaMalloc(&lists_r, (size_t)nblk0 * k * 4));
        FFB_CUDA(cudaMalloc(&counts_r, (size_t)nblk0 * 4));
        FFB_CUDA(cudaMalloc(&counts0, (size_t)nblk0 * 4));
        FFB_CUDA(cudaMalloc(&lists1, (size_t)k * 4 + 64));
        FFB_CUDA(cudaMalloc(&dsig, (size_t)k * 4 + 64));
        FFB_CUDA(cudaMalloc(&flag, 64));
        FFB_CUDA(cudaMalloc(&ucol, (size_t)k * 4 + 64));
        FFB_CUDA(cudaMalloc(&prow, (size_t)k * 4 + 64));
        FFB_CUDA(cudaMalloc(&pcol, (size_t)k * 4 + 64));
        FFB_CUDA(cudaMalloc(&dI, (size_t)k * 4 + 64));
        FFB_CUDA(cudaMalloc(&Kinv, (size_t)k * k * 4 + 64));
        FFB_CUDA(cudaMalloc(&re_scratch, ((size_t)CRP_KMAX * nblk0 * CRP_KMAX + (size_t)nblk0 * CRP_KMAX + 64) * 4));
        FFB_CUDA(cudaMemset(flag, 0, 64));
        FFB_CUDA(cudaMemset(dI, 0, (size_t)k * 4));
        const int64_t maxc = (int64_t)nblk0 * k;
        const size_t resmem = std::min<int64_t>((int64_t)k * maxc, RE_SMEM_WORDS) * 4;
        double acc[3] = {0, 0, 0};
        for (int i = 0; i <= reps; ++i) {
            FFB_CUDA(cudaEventRecord(e[0], st));
            launch_k(k_crp_list, nblk0, 256, crp_smem, st, f, d_in, n, k, n, lists0, counts0);
            FFB_CUDA(cudaEventRecord(e[1], st));
            {
                int rc_cap, si_off;
                const size_t cfmem = cf_smem_bytes(k, nblk0, &rc_cap, &si_off);
                launch_k(k_crp_finish, 1, 256, cfmem, st, f, d_in, n, k, lists0, counts0, nblk0, (int32_t*)re_scratch,
                                                    rc_cap, dI, 0, nullptr, 0, 0, Kinv, lists1, nullptr, 0, ucol,
                                                    prow, pcol, 0, flag, si_off, 0, nullptr, nullptr);
            }
            FFB_CUDA(cudaEventRecord(e[2], st));
            if (k <= 16 && f.p < 4096u)
                launch_k(k_crp_list_reg<16>, nblk0, 256, 0, st, f, d_in, n, k, n, lists_r, counts_r);
            else if (k <= 32 && f.p < 4096u)
                launch_k(k_crp_list_reg<32>, nblk0, 256, 0, st, f, d_in, n, k, n, lists_r, counts_r);
            FFB_CUDA(cudaEventRecord(e[3], st));
            FFB_CUDA(cudaEventSynchronize(e[3]));
            if (i == 0) continue;  // warm-up
            for (int j = 0; j < 3; ++j) {
                FFB_CUDA(cudaEventElapsedTime(&t, e[j], e[j + 1]));
                acc[j] += t;
            }
        }
        for (int j = 0; j < 3; ++j) ms[j] = acc[j] / reps;
        {  // the register-resident list kernel must give the same lists
            std::vector<int32_t> ha((size_t)nblk0 * (k + 1)), hb((size_t)nblk0 * (k + 1));
            FFB_CUDA(cudaMemcpy(ha.data(), counts0, (size_t)nblk0 * 4, cudaMemcpyDeviceToHost));
            FFB_CUDA(cudaMemcpy(hb.data(), counts_r, (size_t)nblk0 * 4, cudaMemcpyDeviceToHost));
            std::vector<int32_t> la((size_t)nblk0 * k), lb((size_t)nblk0 * k);
            FFB_CUDA(cudaMemcpy(la.data(), lists0, la.size() * 4, cudaMemcpyDeviceToHost));
            FFB_CUDA(cudaMemcpy(lb.data(), lists_r, lb.size() * 4, cudaMemcpyDeviceToHost));
            int same = 1;
            for (int b = 0; b < nblk0 && same; ++b) {
                if (ha[b] != hb[b]) same = 0;
                for (int t = 0; t < ha[b] && same; ++t) same = la[(size_t)b * k + t] == lb[(size_t)b * k + t];
            }
            out_k[1 + 2 * k] = (k <= 32 && f.p < 4096u) ? same : -1;
            unsigned long long st8[8];
            FFB_CUDA(cudaMemcpyFromSymbol(st8, g_cf_stamp, sizeof(st8)));
            for (int q = 0; q < 5; ++q) out_k[2 + 2 * k + q] = (int32_t)(st8[q + 1] - st8[q]);  // ns per phase
        }
        out_k[7 + 2 * k] = -1;
        out_k[8 + 2 * k] = 0;
        if (f.p <= 255u && k <= 32 && nblk0 <= CFR_MAXBLK && nblk0 * k <= CFR_MAXC) {
            // the register-resident finish against the smem finish: every output, with sketch rows
            const int sk = RD_S;
            const int64_t r0 = 3;  // rows already in the basis (offsets of the bookkeeping outputs)
            uint32_t *Ssk, *buf[2];
            int32_t* ib[2];
            const size_t nw = (size_t)k * k * 2 + k + (size_t)(r0 + k) * sk, ni = 4 * (size_t)(r0 + k);
            FFB_CUDA(cudaMalloc(&Ssk, (size_t)k * sk * 4));
            launch_k(k_random, (unsigned)cdiv((int64_t)k * sk, 256), 256, 0, st, Ssk, (int64_t)k * sk, 0x1234ull, f.p);
            for (int v = 0; v < 2; ++v) {
                FFB_CUDA(cudaMalloc(&buf[v], nw * 4));
                FFB_CUDA(cudaMalloc(&ib[v], ni * 4));
                FFB_CUDA(cudaMemsetAsync(buf[v], 0, nw * 4, st));
                FFB_CUDA(cudaMemsetAsync(ib[v], 0, ni * 4, st));
            }
            auto run = [&](int v) {
                uint32_t *kinv = buf[v], *ld = kinv + (size_t)k * k, *dvl = ld + (size_t)k * k, *uo = dvl + k;
                int32_t *jo = ib[v], *uc = jo + (r0 + k), *pr = uc + (r0 + k), *pc = pr + (r0 + k);
                if (v == 0) {
                    int rc_cap, si_off;
                    const size_t cfmem = cf_smem_bytes(k, nblk0, &rc_cap, &si_off);
                    launch_k(k_crp_finish, 1, 256, cfmem, st, f, d_in, n, k, lists0, counts0, nblk0,
                             (int32_t*)re_scratch, rc_cap, dI, 5, Ssk, sk, sk, kinv, jo, uo, sk, uc, pr, pc, r0, flag,
                             si_off, 1, ld, dvl);
                } else {
                    launch_k(k_crp_finish_reg, 1, 1024, 0, st, f, d_in, n, k, lists0, counts0, nblk0, dI, 5, Ssk, sk,
                             sk, kinv, jo, uo, sk, uc, pr, pc, r0, flag, 1, ld, dvl);
                }
            };
            run(0);
            run(1);
            FFB_CUDA(cudaEventRecord(e[0], st));
            for (int i = 0; i < reps; ++i) run(1);
            FFB_CUDA(cudaEventRecord(e[1], st));
            FFB_CUDA(cudaEventSynchronize(e[1]));
            FFB_CUDA(cudaEventElapsedTime(&t, e[0], e[1]));
            out_k[8 + 2 * k] = (int32_t)(t / reps * 1e6);  // ns
            std::vector<uint32_t> h0(nw), h1(nw);
            std::vector<int32_t> i0(ni), i1(ni);
            FFB_CUDA(cudaMemcpy(h0.data(), buf[0], nw * 4, cudaMemcpyDeviceToHost));
            FFB_CUDA(cudaMemcpy(h1.data(), buf[1], nw * 4, cudaMemcpyDeviceToHost));
            FFB_CUDA(cudaMemcpy(i0.data(), ib[0], ni * 4, cudaMemcpyDeviceToHost));
            FFB_CUDA(cudaMemcpy(i1.data(), ib[1], ni * 4, cudaMemcpyDeviceToHost));
            out_k[7 + 2 * k] = (h0 == h1 && i0 == i1) ? 1 : 0;
            FFB_CUDA(cudaFree(Ssk));
            for (int v = 0; v < 2; ++v) {
                FFB_CUDA(cudaFree(buf[v]));
                FFB_CUDA(cudaFree(ib[v]));
            }
        }
        int32_t hf = 0;
        FFB_CUDA(cudaMemcpy(&hf, flag, 4, cudaMemcpyDeviceToHost));
        out_k[0] = hf;
        FFB_CUDA(cudaMemcpy(out_k + 1, lists1, (size_t)k * 4, cudaMemcpyDeviceToHost));
        FFB_CUDA(cudaMemcpy(out_k + 1 + k, dsig, (size_t)k * 4, cudaMemcpyDeviceToHost));
        for (void* q : {(void*)lists0, (void*)counts0, (void*)lists1, (void*)dsig, (void*)flag, (void*)ucol,
                        (void*)prow, (void*)pcol, (void*)dI, (void*)Kinv, (void*)re_scratch, (void*)lists_r,
                        (void*)counts_r})
            FFB_CUDA(cudaFree(q));
    }
    FFB_CHECK_LAUNCH();
    for (auto& x : e) FFB_CUDA(cudaEventDestroy(x));
}

}  // namespace ffb

