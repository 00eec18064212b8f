// ffb_fast.cu -- latency-critical small kernels: the 64x64 Crout leaf and the
// inverse-based triangular-solve base.
//
// Leaf (Alg. 4, sytrf.cpp:35-139), right-looking, one CTA of 256 threads:
// thread (ty, tx) owns S[ty + 4q][tx], q < 16, in registers, so the Schur
// update has no index arithmetic and no shared-memory traffic for S.  The
// pivot search of a step is a 64-bit ballot over the residual column masked
// by the active rows; L is staged in shared memory and written to HBM once.
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ffb_kernels.cuh"
#include "ffb_mma.cuh"

namespace ffb {

namespace {

// Leaf outputs (after a barrier): L columns [coff, coff + r) of the leaf rows
// (warp w writes rows w, w+8, ...: coalesced row segments), and
// out = [r, pivot order, pivotless rows ascending] -- to HBM and, when requested,
// to the host mailbox by all threads in parallel (fence, barrier, sequence word).
__device__ __forceinline__ void leaf_epilogue(int s, int r, const int32_t* srows, const uint32_t (*Ls)[65],
                                              const int32_t* order, const int32_t* pless, uint32_t* Lg,
                                              int64_t ldL, int64_t coff, int32_t* out, const MboxPost& mp) {
    const int tid = threadIdx.x, wp = tid >> 5, lane = tid & 31;
    for (int i = wp; i < s; i += 8) {
        uint32_t* dst = Lg + (int64_t)srows[i] * ldL + coff;
        for (int c = lane; c < r; c += 32) dst[c] = Ls[i][c];
    }
    for (int e = tid; e <= s; e += blockDim.x) {
        const int32_t v = e == 0 ? r : (e <= r ? order[e - 1] : pless[e - 1 - r]);
        out[e] = v;
        if (mp.dst) mp.dst[e] = (uint32_t)v;
    }
    if (mp.dst) {
        __threadfence_system();
        __syncthreads();
        if (tid == 0) *(volatile uint32_t*)mp.seq_ptr = mp.seq;
    }
}

template <bool kSmall>
__global__ void __launch_bounds__(256) k_leaf64(Fp f, const uint32_t* A, int64_t lda,
                                                int s, const int32_t* rows,
                                                uint32_t* Lg, int64_t ldL, int64_t coff, DDiag D,
                                                int32_t* out, MboxPost mp) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t Ls[64][65];
    __shared__ uint32_t colb[2][64];  // residual column of the front row, double-buffered
    __shared__ uint32_t col2[64];     // residual column of the 2x2 partner
    __shared__ int32_t order[64];
    __shared__ int32_t pless[64];   // pivotless rows in discovery (= ascending) order
    __shared__ int32_t srows[64];
    __shared__ uint32_t sinv[SINV_MAX];
    const Ar<kSmall> ar(f);
    const int tid = threadIdx.x, tx = tid & 63, ty = tid >> 6, lane = tid & 31;
    const uint32_t one = 1 % f.p;
    if (tid < s) srows[tid] = __ldcg(rows + tid);
    uint32_t S[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const int i = ty + 4 * q;
        S[q] = (i < s && tx < s) ? __ldcg(A + (int64_t)i * lda + tx) : 0;
    }
    for (int e = tid; e < 64 * 65; e += 256) (&Ls[0][0])[e] = 0;
    const SmemInv inv = stage_inverses(f, sinv);
    uint64_t active = (s == 64) ? ~0ull : ((1ull << s) - 1);
    int r = 0, npl = 0, buf = 0;
    __syncthreads();
    for (int p1 = 0; p1 < s; ++p1) {
        if (!((active >> p1) & 1)) continue;  // consumed as a 2x2 partner (uniform)
        uint32_t* col1 = colb[buf];
        buf ^= 1;
        if (tx == p1) {
#pragma unroll
            for (int q = 0; q < 16; ++q) col1[ty + 4 * q] = S[q];
        }
        __syncthreads();
        // every warp finds the first active row with a nonzero residual (sytrf.cpp:78-81)
        const uint32_t b0 = __ballot_sync(0xffffffffu, col1[lane] != 0);
        const uint32_t b1 = __ballot_sync(0xffffffffu, col1[lane + 32] != 0);
        const uint64_t msk = (((uint64_t)b1 << 32) | b0) & active;
        const int j = msk ? __ffsll((long long)msk) - 1 : s;
        if (j >= s) {  // pivotless (sytrf.cpp:82-85)
            if (tid == 0) pless[npl] = p1;
            ++npl;
            active &= ~(1ull << p1);
            continue;
        }
        if (j == p1) {  // 1x1 pivot (sytrf.cpp:87-97)
            const uint32_t x = col1[p1];
            const uint32_t xi = inv(f, x);
            active &= ~(1ull << p1);
            const uint32_t lk = ar.mul(col1[tx], xi);  // multiplier of this thread's column
#pragma unroll
            for (int q = 0; q < 16; ++q) S[q] = ar.sub(S[q], ar.mul(col1[ty + 4 * q], lk));
            if (ty == 0) {
                if (tx == p1) Ls[p1][r] = one;
                else if ((active >> tx) & 1) Ls[tx][r] = lk;
            }
            if (tid == 0) {
                D.kind[coff + r] = D_SCALAR;
                D.val[coff + r] = x;
                D.val2[coff + r] = 0;
                D.inv[coff + r] = xi;
                order[r] = p1;
            }
            r += 1;
            continue;
        }
        // 2x2 antidiagonal pivot pairing p1 with p2 = j (sytrf.cpp:99-131)
        const int p2 = j;
        if (tx == p2) {
#pragma unroll
            for (int q = 0; q < 16; ++q) col2[ty + 4 * q] = S[q];
        }
        __syncthreads();
        const uint32_t x = col1[p2];
        const uint32_t xi = inv(f, x);
        const uint32_t y = col2[p2];
        const uint32_t y_eff = f.char2 ? y : fhalve(f, y);
        const uint32_t yd = f.char2 ? y : 0;
        active &= ~((1ull << p1) | (1ull << p2));
        // multipliers of this thread's column k = tx
        const uint32_t l2k = ar.mul(xi, col1[tx]);
        const uint32_t l1k = ar.mul(xi, ar.sub(col2[tx], ar.mul(y_eff, l2k)));
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int i = ty + 4 * q;
            const uint32_t l2i = ar.mul(xi, col1[i]);
            const uint32_t l1i = ar.mul(xi, ar.sub(col2[i], ar.mul(y_eff, l2i)));
            uint32_t v = ar.add(ar.mul(ar.mul(x, l1i), l2k), ar.mul(ar.mul(x, l2i), l1k));
            if (yd) v = ar.add(v, ar.mul(ar.mul(yd, l2i), l2k));
            S[q] = ar.sub(S[q], v);
        }
        if (ty == 0) {
            if (tx == p1) {
                Ls[p1][r] = one;
            } else if (tx == p2) {
                Ls[p2][r + 1] = one;
                Ls[p2][r] = f.char2 ? 0 : ar.mul(xi, y_eff);
            } else if ((active >> tx) & 1) {
                Ls[tx][r] = l1k;
                Ls[tx][r + 1] = l2k;
            }
        }
        if (tid == 0) {
            const int32_t hk = yd ? D_ANTITRI_HEAD : D_ANTIDIAG_HEAD;
            D.kind[coff + r] = hk;
            D.kind[coff + r + 1] = hk + 1;
            D.val[coff + r] = D.val[coff + r + 1] = x;
            D.val2[coff + r] = D.val2[coff + r + 1] = yd;
            D.inv[coff + r] = D.inv[coff + r + 1] = xi;
            order[r] = p1;
            order[r + 1] = p2;
        }
        r += 2;
    }
    __syncthreads();
    leaf_epilogue(s, r, srows, Ls, order, pless, Lg, ldL, coff, out, mp);
}

// Lazily reduced leaf for 2 <= p < 4096 (same algorithm and outputs as k_leaf64).
// 4 warps: warp w owns columns 16w .. 16w+15, lane l rows l and l+32 (32 int32
// registers per thread, static indices).  A step:
//   * the owner lane of row p1 (= column p1, mod p: S stays symmetric) in every
//     warp stores the warp's 16 raw words of that row (4 x 16-byte stores); barrier;
//   * every lane reduces the residual of its own two rows, c_i; ballot -> first
//     active nonzero (sytrf.cpp:78-81);
//   * row multipliers l_i = c_i x^-1 are computed redundantly by every warp and the
//     16 column multipliers a warp needs are shuffled in: the update
//     S[i][k] -= c_i l_k is 32 IMADs per thread, no reduction and no second barrier.
// Entries only decrease, by < p^2 per pivot (< 1.5 p^2 per pivot for an AntiTri 2x2,
// char 2), so after <= 64 pivots S lies in (-96 p^2, p): int32-safe, and
// S + 96 p^2 < 2^32 is reduced by 32-bit Barrett.
// Accumulator traits of the lazy leaf.  Narrow (p < 4096): int32 entries, products
// < 2^24 reduced by 32-bit Barrett.  Wide (4096 <= p < 2^26, config 3's large prime):
// int64 entries, the same bounds with 64-bit products (96 p^2 < 2^59), 64-bit Barrett.
struct LzNarrow {
    using T = int32_t;
    __device__ __forceinline__ static uint32_t off(const Fp& f) { return 96u * f.p * f.p; }
    __device__ __forceinline__ static uint32_t red(const Fp& f, T v, uint32_t o) {
        return red32(f, (uint32_t)v + o);
    }
    __device__ __forceinline__ static uint32_t mul(const Fp& f, uint32_t a, uint32_t b) { return red32(f, a * b); }
    // d - y l (all reduced)
    __device__ __forceinline__ static uint32_t msub(const Fp& f, uint32_t d, uint32_t y, uint32_t l) {
        return red32(f, d + f.p * f.p - y * l);
    }
};
struct LzWide {
    using T = int64_t;
    __device__ __forceinline__ static uint64_t off(const Fp& f) { return 96ull * f.p * f.p; }
    __device__ __forceinline__ static uint32_t red(const Fp& f, T v, uint64_t o) {
        return red64(f, (uint64_t)v + o);
    }
    __device__ __forceinline__ static uint32_t mul(const Fp& f, uint32_t a, uint32_t b) {
        return red64(f, (uint64_t)a * b);
    }
    __device__ __forceinline__ static uint32_t msub(const Fp& f, uint32_t d, uint32_t y, uint32_t l) {
        return fsub(f, d, red64(f, (uint64_t)y * l));
    }
};
// Shared memory of the lazy leaf core (one 128-thread CTA).
template <class Acc>
struct LeafSmemT {
    uint32_t Ls[64][65];                          // input tile first, then L (row i, pivot column c)
    __align__(16) typename Acc::T rowb[2][64];    // raw residual row of the front
    __align__(16) typename Acc::T row2[64];       // raw residual row of the 2x2 partner
    int32_t order[64];                            // pivot rows in pivot order
    int32_t pless[64];                            // pivotless rows, ascending
    int32_t dkind[64];                            // D of the leaf's pivot columns (written to D after the loop)
    uint32_t dval[64], dval2[64], dinv[64];
};
using LeafSmem = LeafSmemT<LzNarrow>;
// the warp's 16 raw entries of one row -> dst (16-byte stores)
__device__ __forceinline__ void lz_store16(int32_t* dst, const int32_t (&v)[16]) {
    int4* d = reinterpret_cast<int4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}
__device__ __forceinline__ void lz_store16(int64_t* dst, const int64_t (&v)[16]) {
    longlong2* d = reinterpret_cast<longlong2*>(dst);
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = make_longlong2(v[2 * q], v[2 * q + 1]);
}

// The leaf elimination (Alg. 4) of the s x s block at src (row stride lds; global
// memory when kGlobal, else shared), s <= 64, by 128 threads.  Fills sm (L, order,
// pless, D of columns coff ..) and writes D; returns the rank.  Ends with a barrier.
template <bool kGlobal, class Acc = LzNarrow>
__device__ int leaf_core(const Fp& f, const SmemInv& inv, const uint32_t* src, int64_t lds, int s,
                         LeafSmemT<Acc>& sm, DDiag D, int64_t coff) {
    using T = typename Acc::T;
    constexpr bool kWide = sizeof(T) == 8;
    const int tid = threadIdx.x, wp = tid >> 5, lane = tid & 31;
    const uint32_t one = 1 % f.p;
    const auto off = Acc::off(f);
    {  // coalesced tile load, all loads of a thread in flight at once
        uint32_t v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const int e = tid + 128 * u, i = e >> 6, k = e & 63;
            v[u] = (i < s && k < s) ? (kGlobal ? __ldcg(src + (int64_t)i * lds + k) : src[(int64_t)i * lds + k])
                                    : 0u;
        }
        bool nzt = false;
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const int e = tid + 128 * u;
            sm.Ls[e >> 6][e & 63] = v[u];
            nzt |= v[u] != 0;
        }
        // an all-zero block (rank-0 leaves of exactly zero Schur complements, config 2):
        // every row is pivotless, in order (sytrf.cpp:82-85 at each front)
        if (!__syncthreads_or(nzt)) {
            for (int e = tid; e < 64 * 65; e += 128) (&sm.Ls[0][0])[e] = 0;
            for (int i = tid; i < s; i += 128) sm.pless[i] = i;
            __syncthreads();
            return 0;
        }
    }
    T S0[16], S1[16];  // S[lane][16wp + t], S[lane + 32][16wp + t]
#pragma unroll
    for (int t = 0; t < 16; ++t) {
        S0[t] = (T)sm.Ls[lane][16 * wp + t];
        S1[t] = (T)sm.Ls[lane + 32][16 * wp + t];
    }
    __syncthreads();
    for (int e = tid; e < 64 * 65; e += 128) (&sm.Ls[0][0])[e] = 0;
    // active rows as two 32-bit halves (uniform)
    uint32_t alo = s >= 32 ? 0xffffffffu : ((1u << s) - 1), ahi = s >= 64 ? 0xffffffffu : (s > 32 ? ((1u << (s - 32)) - 1) : 0u);
    auto clear_bit = [&](int b) {
        if (b < 32) alo &= ~(1u << b);
        else ahi &= ~(1u << (b - 32));
    };
    int r = 0, npl = 0, buf = 0;
    const bool lo = wp < 2;  // this warp's columns are rows < 32
    for (int p1 = 0; p1 < s; ++p1) {
        if (!(((p1 < 32 ? alo : ahi) >> (p1 & 31)) & 1)) continue;  // consumed as a 2x2 partner (uniform)
        T* rb = sm.rowb[buf];
        buf ^= 1;
        if (lane == (p1 & 31)) {
            if (p1 < 32) lz_store16(rb + 16 * wp, S0);
            else lz_store16(rb + 16 * wp, S1);
        }
        __syncthreads();
        const uint32_t c0 = Acc::red(f, rb[lane], off), c1 = Acc::red(f, rb[lane + 32], off);
        const uint32_t b0 = __ballot_sync(0xffffffffu, c0 != 0) & alo;
        const uint32_t b1 = __ballot_sync(0xffffffffu, c1 != 0) & ahi;
        if (!(b0 | b1)) {  // pivotless (sytrf.cpp:82-85)
            if (tid == 0) sm.pless[npl] = p1;
            ++npl;
            clear_bit(p1);
            continue;
        }
        const int j = b0 ? __ffs(b0) - 1 : 31 + __ffs(b1);
        // the inverse of this lane's residuals and the residuals of this warp's 16 columns
        // (wide: one broadcast load of the pivot's inverse from the global table once the
        // pivot is known -- per-lane prefetches of every candidate measured slower)
        const uint32_t* itab = kWide ? nullptr : inv.t;
        const uint32_t i0v = itab ? itab[c0] : 0u, i1v = itab ? itab[c1] : 0u;
        const uint32_t csrc = lo ? c0 : c1;
        T ck[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) ck[t] = (T)__shfl_sync(0xffffffffu, csrc, (16 * wp + t) & 31);
        if (j == p1) {  // 1x1 pivot (sytrf.cpp:87-97)
            const int src_l = p1 & 31;
            const uint32_t x = __shfl_sync(0xffffffffu, p1 < 32 ? c0 : c1, src_l);
            const uint32_t xi = itab ? __shfl_sync(0xffffffffu, p1 < 32 ? i0v : i1v, src_l) : inv(f, x);
            clear_bit(p1);
            const uint32_t l0 = Acc::mul(f, c0, xi), l1 = Acc::mul(f, c1, xi);  // row multipliers
            // S[i][k] -= c_i l_k = l_i c_k (mod p): row multiplier times column residual
            // negated multipliers: two negations instead of one per column residual
            const T nl0 = (T)0 - (T)l0, nl1 = (T)0 - (T)l1;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                S0[t] += nl0 * ck[t];
                S1[t] += nl1 * ck[t];
            }
            if (wp == 0) {
                if ((alo >> lane) & 1) sm.Ls[lane][r] = l0;
                if ((ahi >> lane) & 1) sm.Ls[lane + 32][r] = l1;
                if (lane == 0) {
                    sm.Ls[p1][r] = one;
                    sm.dkind[r] = D_SCALAR;
                    sm.dval[r] = x;
                    sm.dval2[r] = 0;
                    sm.dinv[r] = xi;
                    sm.order[r] = p1;
                }
            }
            r += 1;
            continue;
        }
        // 2x2 antidiagonal pivot pairing p1 with p2 = j (sytrf.cpp:99-131)
        const int p2 = j;
        if (lane == (p2 & 31)) {
            if (p2 < 32) lz_store16(sm.row2 + 16 * wp, S0);
            else lz_store16(sm.row2 + 16 * wp, S1);
        }
        __syncthreads();
        const uint32_t d0 = Acc::red(f, sm.row2[lane], off), d1 = Acc::red(f, sm.row2[lane + 32], off);
        const uint32_t x = __shfl_sync(0xffffffffu, p2 < 32 ? c0 : c1, p2 & 31);
        const uint32_t y = __shfl_sync(0xffffffffu, p2 < 32 ? d0 : d1, p2 & 31);
        const uint32_t xi = itab ? __shfl_sync(0xffffffffu, p2 < 32 ? i0v : i1v, p2 & 31) : inv(f, x);
        const uint32_t y_eff = f.char2 ? y : fhalve(f, y);
        const uint32_t yd = f.char2 ? y : 0;
        clear_bit(p1);
        clear_bit(p2);
        // row multipliers of this lane's rows: l2 = x^-1 c, l1 = x^-1 (d - y_eff l2)
        const uint32_t l2a = Acc::mul(f, xi, c0), l2b = Acc::mul(f, xi, c1);
        const uint32_t l1a = Acc::mul(f, xi, Acc::msub(f, d0, y_eff, l2a));
        const uint32_t l1b = Acc::mul(f, xi, Acc::msub(f, d1, y_eff, l2b));
        // S -= x l1_i l2_k + x l2_i l1_k (+ yd l2_i l2_k)
        const T ga = (T)0 - (T)(Acc::mul(f, x, l1a) + Acc::mul(f, yd, l2a));  // negated, as above
        const T gb = (T)0 - (T)(Acc::mul(f, x, l1b) + Acc::mul(f, yd, l2b));
        const T ba = (T)0 - (T)Acc::mul(f, x, l2a), bb = (T)0 - (T)Acc::mul(f, x, l2b);
        const uint32_t s2 = lo ? l2a : l2b, s1 = lo ? l1a : l1b;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const int src_l = (16 * wp + t) & 31;
            const T l2k = (T)__shfl_sync(0xffffffffu, s2, src_l);
            const T l1k = (T)__shfl_sync(0xffffffffu, s1, src_l);
            S0[t] += ga * l2k + ba * l1k;
            S1[t] += gb * l2k + bb * l1k;
        }
        if (wp == 0) {
            if ((alo >> lane) & 1) {
                sm.Ls[lane][r] = l1a;
                sm.Ls[lane][r + 1] = l2a;
            }
            if ((ahi >> lane) & 1) {
                sm.Ls[lane + 32][r] = l1b;
                sm.Ls[lane + 32][r + 1] = l2b;
            }
            if (lane == 0) {
                sm.Ls[p1][r] = one;
                sm.Ls[p2][r + 1] = one;
                sm.Ls[p2][r] = f.char2 ? 0 : Acc::mul(f, xi, y_eff);
                const int32_t hk = yd ? D_ANTITRI_HEAD : D_ANTIDIAG_HEAD;
                sm.dval[r] = sm.dval[r + 1] = x;
                sm.dkind[r] = hk;
                sm.dkind[r + 1] = hk + 1;
                sm.dval2[r] = sm.dval2[r + 1] = yd;
                sm.dinv[r] = sm.dinv[r + 1] = xi;
                sm.order[r] = p1;
                sm.order[r + 1] = p2;
            }
        }
        r += 2;
    }
    __syncthreads();
    // D of the leaf's pivot columns, in one coalesced pass (the per-pivot global stores sat on
    // warp 0's path to the next barrier)
    for (int t = tid; t < r; t += 128) {
        D.kind[coff + t] = sm.dkind[t];
        D.val[coff + t] = sm.dval[t];
        D.val2[coff + t] = sm.dval2[t];
        D.inv[coff + t] = sm.dinv[t];
    }
    return r;
}

template <class Acc>
__global__ void __launch_bounds__(128) k_leaf64_lazy(Fp f, const uint32_t* A, int64_t lda,
                                                     int s, const int32_t* rows,
                                                     uint32_t* Lg, int64_t ldL, int64_t coff, DDiag D,
                                                     int32_t* out, MboxPost mp) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ LeafSmemT<Acc> sm;
    __shared__ int32_t srows[64];
    __shared__ uint32_t sinv[SINV_MAX];
    const int tid = threadIdx.x;
    const SmemInv inv = stage_inverses(f, sinv);  // independent of the predecessor
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid < 64) srows[tid] = tid < s ? __ldcg(rows + tid) : 0;
    const int r = leaf_core<true, Acc>(f, inv, A, lda, s, sm, D, coff);
    // L columns [coff, coff + r) of the leaf rows: thread t < s writes row t
    if (tid < s) {
        uint32_t* d = Lg + (int64_t)srows[tid] * ldL + coff;
#pragma unroll 8
        for (int c = 0; c < r; ++c) d[c] = sm.Ls[tid][c];
    }
    for (int e = tid; e <= s; e += 128) {
        const int32_t v = e == 0 ? r : (e <= r ? sm.order[e - 1] : sm.pless[e - 1 - r]);
        out[e] = v;
        if (mp.dst) mp.dst[e] = (uint32_t)v;
    }
    if (mp.dst) {
        __threadfence_system();
        __syncthreads();
        if (tid == 0) *(volatile uint32_t*)mp.seq_ptr = mp.seq;
    }
}

// ---------------------------------------------------------------------------
// Fused small node (p < 4096, children are leaves: s <= 2T, T <= 64): one CTA runs
// recursive_step (sytrf.cpp:298-335) on an s x s node, s <= 128, held in shared
// memory -- leaf(A1), B' = P1^T B, X = L1^-1 B'1, G = (D1^-1 X)^T (also written
// to the L rows of N1), Y = B'2 - M1 X, Z = C - G X, then zero_leading
// (sytrf.cpp:267-292): m - r1 = 0 or Y = 0 -> leaf(Z) and the permutation
// composition on the device; Y != 0 (zero_leading_pairs) -> bail out: Y goes to
// yout (ld ns), Z to A[m:, m:], and the host continues from leaf(A1)'s result.
// out / mailbox: [0, rank, perm(s)] when done, [1, r1, perm1(m)] on bail-out.
// ---------------------------------------------------------------------------
constexpr int NODE_LD = 129;  // row stride of the node matrix in shared memory
constexpr int NODE_W = 65;    // row stride of the 64-wide work matrices
constexpr int NODE_B8 = 68;   // row stride (bytes) of the K-contiguous byte copies (17 words: conflict-free)
constexpr size_t node_smem_bytes() {
    return (size_t)(128 * NODE_LD + 3 * 64 * NODE_W) * 4 + 3 * 64 * NODE_B8;
}
// SM-clock stamps of the last k_node128 (thread 0; diagnostics read by ffb_dbg_node_stamps):
// wait done, node loaded, leaf(A1), B'/[L1; M1] gathered, X, G, [Y; Z] updated, leaf(Z), exit
__device__ long long g_node_stamp[9];
#define NODE_STAMP(i)                                  \
    do {                                               \
        if (threadIdx.x == 0) g_node_stamp[i] = clock64(); \
    } while (0)
__global__ void __launch_bounds__(128) k_node128(Fp f, uint32_t* A, int64_t lda, int s, const int32_t* rows,
                                                 uint32_t* Lg, int64_t ldL, int64_t coff, DDiag D,
                                                 uint32_t* yout, int32_t* out, MboxPost mp) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ __align__(16) uint32_t nsm[];
    uint32_t* Am = nsm;                       // s x s node (C becomes Z in place)
    uint32_t* BP = Am + 128 * NODE_LD;        // m x ns: X in rows [0, r1), Y in [r1, m)
    uint32_t* LM = BP + 64 * NODE_W;          // m x r1: [L1; M1]
    uint32_t* Gs = LM + 64 * NODE_W;          // ns x r1: G
    // p <= 255: byte copies with K contiguous for the dp4a update -- M1 rows, G rows, X^T rows
    uint8_t* M8 = reinterpret_cast<uint8_t*>(Gs + 64 * NODE_W);
    uint8_t* G8 = M8 + 64 * NODE_B8;
    uint8_t* XT8 = G8 + 64 * NODE_B8;
    const bool bytes = f.p <= 255u;
    __shared__ LeafSmem sm;
    __shared__ int32_t srows[128];
    __shared__ int32_t perm1[64], perm2[128];
    __shared__ uint32_t sinv[SINV_MAX];
    __shared__ int ynz;
    const int tid = threadIdx.x, wp = tid >> 5, lane = tid & 31;
    const SmemInv inv = stage_inverses(f, sinv);  // independent of the predecessor
    asm volatile("griddepcontrol.wait;" ::: "memory");
    NODE_STAMP(0);
    const int m = s / 2, ns = s - m;
    for (int i0 = 0; i0 < s; i0 += 32) {  // node matrix: 32 rows per round, loads in flight
        uint32_t v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const int i = i0 + u, k = tid;
            v[u] = (i < s && k < s) ? __ldcg(A + (int64_t)i * lda + k) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) Am[(i0 + u) * NODE_LD + tid] = v[u];
    }
    srows[tid] = tid < s ? __ldcg(rows + tid) : 0;
    if (tid == 0) ynz = 0;
    __syncthreads();
    NODE_STAMP(1);
    // ---- leaf(A1) (:303) ----
    const int r1 = leaf_core<false>(f, inv, Am, NODE_LD, m, sm, D, coff);
    NODE_STAMP(2);
    const int mp1 = m - r1;
    if (tid < m) {
        uint32_t* d = Lg + (int64_t)srows[tid] * ldL + coff;
        for (int c = 0; c < r1; ++c) d[c] = sm.Ls[tid][c];
        perm1[tid] = tid < r1 ? sm.order[tid] : sm.pless[tid - r1];
    }
    __syncthreads();
    // ---- B' = P1^T B (:308), [L1; M1] in position order ----
    {  // thread = column j, rows ih + 2u; 8 rows of loads in flight
        const int j = tid & 63, ih = tid >> 6;
#pragma unroll 1
        for (int ub = 0; ub < 32; ub += 8) {
            if (ih + 2 * ub >= m) break;  // uniform per warp
            int src[8];
            uint32_t vb[8], vl[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = ih + 2 * (ub + u);
                src[u] = i < m ? perm1[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                vb[u] = Am[src[u] * NODE_LD + m + j];
                vl[u] = sm.Ls[src[u]][j];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = ih + 2 * (ub + u);
                if (i < m) {
                    if (j < ns) BP[i * NODE_W + j] = vb[u];
                    if (j < r1) LM[i * NODE_W + j] = vl[u];
                    if (bytes && i >= r1) M8[(i - r1) * NODE_B8 + j] = (uint8_t)(j < r1 ? vl[u] : 0u);
                }
            }
        }
    }
    __syncthreads();
    NODE_STAMP(3);
    if (r1 > 0) {
        // ---- X = L1^-1 B'1 (:310): warp w owns columns 16w + c, lanes 2c, 2c+1 split k ----
        {
            const int c = 16 * wp + (lane >> 1), q = lane & 1;
            for (int i0 = 0; i0 < r1; i0 += 4) {
                uint32_t acc[4] = {0, 0, 0, 0};
                for (int k = q; k < i0; k += 2) {
                    const uint32_t xk = BP[k * NODE_W + c];
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) acc[rr] += LM[(i0 + rr) * NODE_W + k] * xk;
                }
                uint32_t sum[4];
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) sum[rr] = red32(f, acc[rr] + __shfl_xor_sync(0xffffffffu, acc[rr], 1));
                if (q == 0 && c < ns) {
                    uint32_t x[4];
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) {
                        if (i0 + rr >= r1) break;
                        uint32_t v = fsub(f, BP[(i0 + rr) * NODE_W + c], sum[rr]);
#pragma unroll
                        for (int t = 0; t < rr; ++t) v = fsub(f, v, fmul(f, LM[(i0 + rr) * NODE_W + i0 + t], x[t]));
                        x[rr] = v;
                        BP[(i0 + rr) * NODE_W + c] = v;
                        if (bytes) XT8[c * NODE_B8 + i0 + rr] = (uint8_t)v;
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();
        NODE_STAMP(4);
        // ---- G = (D1^-1 X)^T (:313, blockdiag.hpp:112-138), also the L rows of N1 ----
        {  // thread = pivot column k, rows jh + 2u: v = ca X[k1][j] + cb X[k2][j]
            const int k = tid & 63, jh = tid >> 6;
            int k1 = 0, k2 = 0;
            uint32_t ca = 0, cb = 0;
            if (k < r1) {
                const int32_t kind = sm.dkind[k];
                const uint32_t iv = sm.dinv[k];
                k1 = k2 = k;
                ca = iv;
                if (kind == D_ANTIDIAG_HEAD) {
                    k1 = k + 1;
                } else if (kind == D_ANTIDIAG_TAIL || kind == D_ANTITRI_TAIL) {
                    k1 = k - 1;
                } else if (kind != D_SCALAR) {  // AntiTri head: -d c^-2 x_t + c^-1 x_{t+1}
                    ca = fneg(f, fmul(f, sm.dval2[k], fmul(f, iv, iv)));
                    k2 = k + 1;
                    cb = iv;
                }
            }
#pragma unroll 1
            for (int ub = 0; ub < 32; ub += 8) {
                if (jh + 2 * ub >= ns) break;  // uniform per warp
                uint32_t x1[8], x2[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = min(jh + 2 * (ub + u), ns - 1);
                    x1[u] = BP[k1 * NODE_W + j];
                    x2[u] = BP[k2 * NODE_W + j];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int j = jh + 2 * (ub + u);
                    if (j >= ns) continue;
                    const uint32_t v = red32(f, ca * x1[u] + cb * x2[u]);
                    if (k < r1) {
                        Gs[j * NODE_W + k] = v;
                        Lg[(int64_t)srows[m + j] * ldL + coff + k] = v;
                    }
                    if (bytes) G8[j * NODE_B8 + k] = (uint8_t)(k < r1 ? v : 0u);
                }
            }
        }
        __syncthreads();
    }
    NODE_STAMP(5);
    // ---- [Y; Z] -= [M1; G] X (:312, :315): thread = 8 rows x 8 columns ----
    {
        const int rg = tid >> 3, cg = tid & 7;
        const int R = mp1 + ns;
        uint32_t acc[8][8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = 0;
        const uint32_t* lrow[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int rho = 8 * rg + a;
            lrow[a] = rho < mp1 ? LM + (r1 + rho) * NODE_W : Gs + (rho < R ? rho - mp1 : 0) * NODE_W;
        }
        if (bytes) {  // four k per dp4a: the byte rows of [M1; G] against the byte rows of X^T
            const uint32_t* lw8[8];
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int rho = 8 * rg + a;
                lw8[a] = reinterpret_cast<const uint32_t*>(
                    rho < mp1 ? M8 + rho * NODE_B8 : G8 + (rho < R ? rho - mp1 : 0) * NODE_B8);
            }
            const uint32_t* xw8 = reinterpret_cast<const uint32_t*>(XT8 + 8 * cg * NODE_B8);
            const int k4n = (r1 + 3) >> 2;
#pragma unroll 2
            for (int k4 = 0; k4 < k4n; ++k4) {
                uint32_t xv[8], lv[8];
#pragma unroll
                for (int b = 0; b < 8; ++b) xv[b] = xw8[b * (NODE_B8 / 4) + k4];
#pragma unroll
                for (int a = 0; a < 8; ++a) lv[a] = lw8[a][k4];
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a][b] = __dp4a(lv[a], xv[b], acc[a][b]);
            }
        } else {
            for (int k = 0; k < r1; ++k) {
                uint32_t xv[8], lv[8];
#pragma unroll
                for (int b = 0; b < 8; ++b) xv[b] = BP[k * NODE_W + 8 * cg + b];
#pragma unroll
                for (int a = 0; a < 8; ++a) lv[a] = lrow[a][k];
#pragma unroll
                for (int a = 0; a < 8; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) acc[a][b] += lv[a] * xv[b];
            }
        }
        int nz = 0;
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const int rho = 8 * rg + a;
            if (rho >= R) break;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int j = 8 * cg + b;
                if (j >= ns) break;
                uint32_t* cp = rho < mp1 ? BP + (r1 + rho) * NODE_W + j : Am + (m + rho - mp1) * NODE_LD + m + j;
                const uint32_t v = fsub(f, *cp, red32(f, acc[a][b]));
                *cp = v;
                if (rho < mp1) nz |= v != 0;
            }
        }
        if (nz) ynz = 1;
    }
    __syncthreads();
    NODE_STAMP(6);
    if (mp1 > 0 && ynz) {
        // ---- zero_leading_pairs: hand Y and Z to the host ----
        for (int e = tid; e < mp1 * 64; e += 128) {
            const int i = e >> 6, j = e & 63;
            if (j < ns) yout[(int64_t)i * ns + j] = BP[(r1 + i) * NODE_W + j];
        }
        for (int e = tid; e < ns * 128; e += 128) {
            const int i = e >> 7, j = e & 127;
            if (j < ns) A[(int64_t)(m + i) * lda + m + j] = Am[(m + i) * NODE_LD + m + j];
        }
        for (int e = tid; e < m + 2; e += 128) {
            const int32_t v = e == 0 ? 1 : (e == 1 ? r1 : perm1[e - 2]);
            out[e] = v;
            if (mp.dst) mp.dst[e] = (uint32_t)v;
        }
    } else {
        // ---- leaf(Z) (:317 via zero_leading :273 / :276) ----
        const int r3 = leaf_core<false>(f, inv, Am + m * NODE_LD + m, NODE_LD, ns, sm, D, coff + r1);
        NODE_STAMP(7);
        if (tid < ns) {
            uint32_t* d = Lg + (int64_t)srows[m + tid] * ldL + coff + r1;
            for (int c = 0; c < r3; ++c) d[c] = sm.Ls[tid][c];
        }
        // f2 = zero_leading's permutation of [Y rows (mp1), Z rows (ns)] (:284-289)
        for (int pos = tid; pos < mp1 + ns; pos += 128) {
            int v;
            if (mp1 == 0) {
                v = pos < r3 ? sm.order[pos] : sm.pless[pos - r3];
            } else if (pos < r3) {
                v = mp1 + sm.order[pos];
            } else if (pos < r3 + mp1) {
                v = pos - r3;
            } else {
                v = mp1 + sm.pless[pos - mp1 - r3];
            }
            perm2[pos] = v;
        }
        __syncthreads();
        // P = compose(embed(P1, 0, n), embed(P2, r1, n)) (:332-334)
        for (int e = tid; e < s + 2; e += 128) {
            int32_t v;
            if (e == 0) v = 0;
            else if (e == 1) v = r1 + r3;
            else {
                const int pos = e - 2;
                if (pos < r1) v = perm1[pos];
                else {
                    const int cix = perm2[pos - r1];
                    v = cix < mp1 ? perm1[r1 + cix] : m + (cix - mp1);
                }
            }
            out[e] = v;
            if (mp.dst) mp.dst[e] = (uint32_t)v;
        }
    }
    if (mp.dst) {
        __threadfence_system();
        __syncthreads();
        if (tid == 0) *(volatile uint32_t*)mp.seq_ptr = mp.seq;
    }
    NODE_STAMP(8);
}

// Inverse of the unit lower triangular 64x64 diagonal blocks of T, one CTA per
// block, by recursive doubling: each warp inverts one 8x8 diagonal block by
// forward substitution (warp-local), then three levels h = 8, 16, 32 fill the
// off-diagonal blocks of every 2h x 2h diagonal block,
//   inv([[A, 0], [C, B]]) = [[A^-1, 0], [-B^-1 (C A^-1), B^-1]],
// as parallel products (two barriers per level instead of two per row).
// Rows >= nb of a ragged last block are completed with the identity.
// kMode 0: 32-bit sums (p < 4096), 1: 64-bit lazy (p < 2^23), 2: reduce per product.
template <int kMode>
__device__ __forceinline__ uint32_t dot_lt(const Fp& f, const uint32_t* a, int sa, const uint32_t* b, int sb,
                                           int k0, int k1) {
    if (kMode == 0) {
        uint32_t acc = 0;
        for (int k = k0; k < k1; ++k) acc += a[k * sa] * b[k * sb];
        return red32(f, acc);
    }
    uint64_t acc = 0;
    for (int k = k0; k < k1; ++k) {
        const uint64_t prod = (uint64_t)a[k * sa] * b[k * sb];
        acc = kMode == 1 ? acc + prod : (uint64_t)red64(f, acc + prod);
    }
    return red64(f, acc);
}
// X = inverse of the unit lower nb x nb block at Tb (nb <= 64, identity beyond),
// in shared memory; Ts is scratch (W = C A^-1 of a level lives transposed in its
// upper triangle).  All 256 threads; ends with a barrier.
template <int kMode>
__device__ __forceinline__ void trinv64_block(const Fp& f, const uint32_t* Tb, int64_t ldt, int nb,
                                              uint32_t (*Ts)[65], uint32_t (*X)[65]) {
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    load_tile<16>(&Ts[0][0], 65, Tb, ldt, nb, nb);
    __syncthreads();
    for (int e = tid; e < 64 * 64; e += 256) {
        const int i = e >> 6, k = e & 63;
        if (i >= nb || k >= i) Ts[i][k] = 0;  // strict lower part only (unit diagonal implied)
        X[i][k] = 0;
    }
    __syncthreads();
    {  // 8x8 diagonal blocks: warp wp, lane l < 8 computes column 8wp + l
        const int o = 8 * wp;
        if (lane < 8) {
            uint32_t x[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                uint64_t acc = 0;
#pragma unroll
                for (int k = 0; k < i; ++k) {
                    const uint64_t prod = (uint64_t)Ts[o + i][o + k] * x[k];
                    acc = kMode == 2 ? (uint64_t)red64(f, acc + prod) : acc + prod;
                }
                x[i] = fsub(f, i == lane ? 1 % f.p : 0u, red64(f, acc));
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) X[o + i][o + lane] = x[i];
        }
    }
    __syncthreads();
    for (int lg = 3; lg <= 5; ++lg) {  // h = 8, 16, 32
        const int h = 1 << lg, npair = 32 >> lg, per = h * h;
        // W = C A^-1 : W[r][c] = sum_{k >= c} C[r][k] A^-1[k][c]
        for (int e = tid; e < npair * per; e += 256) {
            const int j = e >> (2 * lg), r = (e >> lg) & (h - 1), c = e & (h - 1);
            const int a0 = 2 * j * h, b0 = a0 + h;
            Ts[a0 + c][b0 + r] = dot_lt<kMode>(f, &Ts[b0 + r][a0], 1, &X[a0][a0 + c], 65, c, h);
        }
        __syncthreads();
        // X_BA = -B^-1 W : X[r][c] = -sum_{k <= r} B^-1[r][k] W[k][c]
        for (int e = tid; e < npair * per; e += 256) {
            const int j = e >> (2 * lg), r = (e >> lg) & (h - 1), c = e & (h - 1);
            const int a0 = 2 * j * h, b0 = a0 + h;
            X[b0 + r][a0 + c] = fneg(f, dot_lt<kMode>(f, &X[b0 + r][b0], 1, &Ts[a0 + c][b0], 1, 0, r + 1));
        }
        __syncthreads();
    }
}

template <int kMode>
__global__ void __launch_bounds__(256) k_trinv64(Fp f, const uint32_t* T, int64_t ldt,
                                                 int64_t n, uint32_t* Tinv) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t Ts[64][65];
    __shared__ uint32_t X[64][65];
    const int b = blockIdx.x;
    const int64_t i0 = (int64_t)b * 64;
    const int nb = (int)std::min<int64_t>(64, n - i0);
    const int tid = threadIdx.x;
    trinv64_block<kMode>(f, T + i0 * ldt + i0, ldt, nb, Ts, X);
    uint32_t* o = Tinv + (int64_t)b * 64 * 64;
    for (int e = tid; e < 64 * 64; e += 256) o[e] = X[e >> 6][e & 63];
}

// Unit lower solve for n <= 64 in one launch: every CTA inverts the block in
// shared memory (as k_trinv64) and applies it to its 64-column tile of B,
// X = T^-1 B, with register-blocked dot products (thread: one column, 16 rows).
template <int kMode>
__global__ void __launch_bounds__(256) k_trsm_small(Fp f, const uint32_t* T, int64_t ldt, int n, uint32_t* B,
                                                    int64_t ldb, int64_t ncols) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t Ts[64][65];
    __shared__ uint32_t X[64][65];
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * 64;
    const int bc = (int)std::min<int64_t>(64, ncols - c0);
    // the B tile does not depend on the inverse: its loads are issued first
    uint32_t bv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int r = wp + 8 * (u >> 1), c = lane + 32 * (u & 1);
        bv[u] = (r < n && c < bc) ? __ldcg(B + (int64_t)r * ldb + c0 + c) : 0u;
    }
    trinv64_block<kMode>(f, T, ldt, n, Ts, X);
#pragma unroll
    for (int u = 0; u < 16; ++u) Ts[wp + 8 * (u >> 1)][lane + 32 * (u & 1)] = bv[u];  // Ts is free now
    __syncthreads();
    const int j = tid & 63, i0 = tid >> 6;  // a warp shares its rows: X[i][k] is a broadcast
    if (kMode == 0) {  // p < 4096: 64 products < 2^24 sum in 32 bits
        uint32_t acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = 0;
        for (int k = 0; k < n; ++k) {
            const uint32_t bk = Ts[k][j];
#pragma unroll
            for (int q = 0; q < 16; ++q) acc[q] += X[i0 + 4 * q][k] * bk;
        }
        if (j < bc) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int i = i0 + 4 * q;
                if (i < n) B[(int64_t)i * ldb + c0 + j] = red32(f, acc[q]);
            }
        }
        return;
    }
    uint64_t acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0;
    for (int k = 0; k < n; ++k) {
        const uint32_t bk = Ts[k][j];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const uint64_t prod = (uint64_t)X[i0 + 4 * q][k] * bk;  // X is lower: zero for k > i
            acc[q] = kMode == 2 ? (uint64_t)red64(f, acc[q] + prod) : acc[q] + prod;
        }
    }
    if (j < bc) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int i = i0 + 4 * q;
            if (i < n) B[(int64_t)i * ldb + c0 + j] = red64(f, acc[q]);
        }
    }
}

// Unit lower solve for n <= 64 by blocked forward substitution, X = T^-1 B, in
// place.  CTA: 64 columns of B; warp w owns columns 8w .. 8w+7 and solves them
// alone (no block barrier after staging): lane = 4 c + q handles column c's dot
// products over k = q (mod 4) for a block of 4 rows, the partial sums meet by
// xor-shuffles and lane q = 0 solves the block's 4 x 4 diagonal part.  Xs row stride 72 words: the 32 lanes of a warp hit 32 banks.
// kMode 0 (p < 4096): 32-bit sums (63 products < 2^24); 1 (p < 2^23): 64-bit
// sums; 2: reduce per product.  Only the strict lower part of T is read.
template <int kMode>
__global__ void __launch_bounds__(256) k_trsm_fwd(Fp f, const uint32_t* T, int64_t ldt, int n, uint32_t* B,
                                                  int64_t ldb, int64_t ncols) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t Ts[64][65];
    __shared__ uint32_t Xs[64][72];
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * 64;
    const int bc = (int)std::min<int64_t>(64, ncols - c0);
    {  // stage T (strict lower) and the B tile, all loads of a thread in flight
        uint32_t tv[16], bv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = tid + 256 * u, i = e >> 6, k = e & 63;
            tv[u] = (i < n && k < i) ? __ldcg(T + (int64_t)i * ldt + k) : 0u;
            bv[u] = (i < n && k < bc) ? __ldcg(B + (int64_t)i * ldb + c0 + k) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = tid + 256 * u, i = e >> 6, k = e & 63;
            Ts[i][k] = tv[u];
            Xs[i][k] = bv[u];
        }
    }
    __syncthreads();
    const int c = 8 * wp + (lane >> 2), q = lane & 3;
    // blocks of 4 rows: partial sums over the solved rows k < i0 (4-way split over the
    // lanes), then lane q = 0 finishes the 4 x 4 unit-lower diagonal block serially
    for (int i0 = 0; i0 < n; i0 += 4) {
        uint32_t sum[4];
        if (kMode == 0) {
            uint32_t acc[4] = {0, 0, 0, 0};
            for (int k = q; k < i0; k += 4) {
                const uint32_t xk = Xs[k][c];
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[r] += Ts[i0 + r][k] * xk;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 1);
                acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 2);
                sum[r] = red32(f, acc[r]);
            }
        } else {
            uint64_t acc[4] = {0, 0, 0, 0};
            for (int k = q; k < i0; k += 4) {
                const uint32_t xk = Xs[k][c];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const uint64_t prod = (uint64_t)Ts[i0 + r][k] * xk;
                    acc[r] = kMode == 2 ? (uint64_t)red64(f, acc[r] + prod) : acc[r] + prod;
                }
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (kMode == 2) acc[r] = red64(f, acc[r]);
                acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 1);
                acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], 2);
                sum[r] = red64(f, acc[r]);
            }
        }
        if (q == 0) {
            uint32_t x[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                uint32_t v = fsub(f, Xs[i0 + r][c], sum[r]);
#pragma unroll
                for (int t = 0; t < r; ++t) v = fsub(f, v, fmul(f, Ts[i0 + r][i0 + t], x[t]));
                x[r] = v;
                Xs[i0 + r][c] = v;
            }
        }
        __syncwarp();
    }
    if (c < bc) {  // lanes q write rows q, q+4, ... of column c (each row segment of 8 columns
                   // of the warp is one 32-byte sector)
        for (int i = q; i < n; i += 4) B[(int64_t)i * ldb + c0 + c] = Xs[i][c];
    }
}

// Panel solve: rows [r0, r0 + nb) (nb <= 256, 64-aligned r0), column tile of
// 32: x_b = Tinv_b (b_b - sum_{c<b} T_{bc} x_c) block by block, in place.
// The four diagonal inverses and the strictly lower 64x64 couplings are read
// from L2 per tile (they are shared by all column tiles).
constexpr int PNL_COLS = 32;
// NC columns per CTA (32, or 8 for narrow right-hand sides: 4x the CTAs, a quarter of the
// per-stage work); 256 / NC row groups, thread rows rg + G u (u < 64 / G) of each block.
template <bool kSmall, int NC = PNL_COLS>
__global__ void __launch_bounds__(256) k_trsm_panel(Fp f, const uint32_t* T, int64_t ldt,
                                                    const uint32_t* Tinv, uint32_t* B,
                                                    int64_t ldb, int nb, int64_t ncols) {
    FFB_PDL_ENTRY();
    constexpr int G = 256 / NC, RU = 64 / G;
    extern __shared__ uint32_t sm[];
    uint32_t* Xs = sm;                  // 256 x (NC+1)
    uint32_t* Ms = Xs + 256 * (NC + 1);  // one 64 x 65 matrix block
    const int tid = threadIdx.x;
    const int64_t c0 = (int64_t)blockIdx.x * NC;
    const int bc = (int)std::min<int64_t>(NC, ncols - c0);
    load_tile<8>(Xs, NC + 1, B + c0, ldb, nb, bc);
    const int nblk = (nb + 63) / 64;
    const int col = tid % NC, rg = tid / NC;
    for (int bi = 0; bi < nblk; ++bi) {
        const int rb = bi * 64, rows = std::min(64, nb - rb);
        // b_bi -= T_{bi,bj} x_bj for bj < bi: the thread's RU rows are independent
        // accumulator chains sharing each x load (stale Ms rows >= `rows` are discarded)
        for (int bj = 0; bj < bi; ++bj) {
            __syncthreads();
            load_tile<16>(Ms, 65, T + (int64_t)rb * ldt + bj * 64, ldt, rows, 64);
            __syncthreads();
            uint64_t acc[RU];
#pragma unroll
            for (int u = 0; u < RU; ++u) acc[u] = 0;
            for (int k = 0; k < 64; ++k) {
                const uint64_t xv = Xs[(bj * 64 + k) * (NC + 1) + col];
#pragma unroll
                for (int u = 0; u < RU; ++u) {
                    const uint64_t prod = (uint64_t)Ms[(rg + G * u) * 65 + k] * xv;
                    acc[u] = kSmall ? acc[u] + prod : (uint64_t)red64(f, acc[u] + prod);
                }
            }
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const int r = rg + G * u;
                if (r < rows) {
                    uint32_t* x = &Xs[(rb + r) * (NC + 1) + col];
                    *x = fsub(f, *x, red64(f, acc[u]));
                }
            }
        }
        // x_bi = Tinv_bi b_bi (Tinv lower triangular: the k > r terms are masked)
        __syncthreads();
        load_tile<16>(Ms, 65, Tinv + (int64_t)(rb / 64) * 64 * 64, 64, 64, 64);
        __syncthreads();
        uint64_t acc[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) acc[u] = 0;
        for (int k = 0; k < 64; ++k) {
            const uint64_t xv = Xs[(rb + k) * (NC + 1) + col];
#pragma unroll
            for (int u = 0; u < RU; ++u) {
                const int r = rg + G * u;
                const uint64_t prod = k <= r ? (uint64_t)Ms[r * 65 + k] * xv : 0ull;
                acc[u] = kSmall ? acc[u] + prod : (uint64_t)red64(f, acc[u] + prod);
            }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int r = rg + G * u;
            if (r < rows) Xs[(rb + r) * (NC + 1) + col] = red64(f, acc[u]);
        }
    }
    __syncthreads();
    for (int e = tid; e < nb * bc; e += 256) {
        const int r = e / bc, cc = e % bc;
        B[(int64_t)r * ldb + c0 + cc] = Xs[r * (NC + 1) + cc];
    }
}

// ---------------------------------------------------------------------------
// Panel solve on the int8 tensor cores (p <= 255): mma.sync m16n8k32 s8 x s8
// -> s32 with residues centered to [-(p-1)/2, (p-1)/2].  Rows [0, nb) of the
// panel (nb <= 256) x PM_COLS columns per CTA:
//   for each 64-row block bi:  Y = X_bi - sum_{bj<bi} T_{bi,bj} X_bj,
//                              X_bi = Tinv_bi Y        (both as warp MMAs)
// X lives in shared memory as exact residues (u32) and as a transposed int8
// copy (the B operand).  Warp w owns the 16-row m-tile (w & 3) and four 8-col
// n-tiles of the 64 x PM_COLS block result; |acc| <= 192 * 127^2 < 2^31.
// ---------------------------------------------------------------------------
constexpr int PM_COLS = 64, PM_XU = PM_COLS + 8, PM_XB = 256 + 16, PM_AB = 64 + 16;
constexpr size_t PM_SMEM = (size_t)256 * PM_XU * 4 + (size_t)PM_COLS * PM_XB + (size_t)64 * PM_AB;

// 64 x 64 block of u32 residues (rows < rv, cols < cv; zero elsewhere) -> centered int8 in Ab
__device__ __forceinline__ void pm_load_a(int8_t* Ab, const uint32_t* src, int64_t ld, int rv,
                                          int cv, uint32_t p, uint32_t half) {
    uint32_t v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int e = threadIdx.x + 256 * u, r = e >> 6, c = e & 63;
        v[u] = (r < rv && c < cv) ? __ldcg(src + (int64_t)r * ld + c) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
        const int e = threadIdx.x + 256 * u, r = e >> 6, c = e & 63;
        Ab[r * PM_AB + c] = center8(v[u], p, half);
    }
}
// acc[t] += A(64x64 block in Ab, rows of m-tile mt) x X^T[k0 .. k0+64)[n-tiles nt0..nt0+3]
__device__ __forceinline__ void pm_mma(int (&acc)[4][4], const int8_t* Ab, const int8_t* XbT, int k0, int mt,
                                       int nt0, int gid, int tig) {
#pragma unroll
    for (int ks = 0; ks < 64; ks += 32) {
        const int8_t* ar0 = Ab + (16 * mt + gid) * PM_AB + ks + tig * 4;
        const int8_t* ar1 = ar0 + 8 * PM_AB;
        const uint32_t a0 = *(const uint32_t*)ar0, a1 = *(const uint32_t*)ar1;
        const uint32_t a2 = *(const uint32_t*)(ar0 + 16), a3 = *(const uint32_t*)(ar1 + 16);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int8_t* bp = XbT + (8 * (nt0 + t) + gid) * PM_XB + k0 + ks + tig * 4;
            mma_s8_16832(acc[t], a0, a1, a2, a3, *(const uint32_t*)bp, *(const uint32_t*)(bp + 16));
        }
    }
}
__global__ void __launch_bounds__(256, 2) k_trsm_panel_mma(Fp f, const uint32_t* T, int64_t ldt,
                                                           const uint32_t* Tinv, uint32_t* B,
                                                           int64_t ldb, int nb, int64_t ncols) {
    FFB_PDL_ENTRY();
    extern __shared__ __align__(16) uint8_t pm_smem[];
    uint32_t* Xu = (uint32_t*)pm_smem;                     // 256 x PM_XU
    int8_t* XbT = (int8_t*)(Xu + 256 * PM_XU);             // PM_COLS x PM_XB (column-major int8 X)
    int8_t* Ab = XbT + PM_COLS * PM_XB;                    // 64 x PM_AB
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, gid = lane >> 2, tig = lane & 3;
    const int mt = wp & 3, nt0 = (wp >> 2) * 4;
    const int64_t c0 = (int64_t)blockIdx.x * PM_COLS;
    const int bc = (int)std::min<int64_t>(PM_COLS, ncols - c0);
    const uint32_t p = f.p, half = (p - 1) / 2, bias = (uint32_t)(0x80000000ull % p);
    // panel -> Xu (zero outside rows < nb, cols < bc) and its int8 transpose
    for (int r0 = wp; r0 < 256; r0 += 64) {
        uint32_t v[8][2];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int r = r0 + 8 * u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = lane + 32 * h;
                v[u][h] = (r < nb && c < bc) ? B[(int64_t)r * ldb + c0 + c] : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int r = r0 + 8 * u;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = lane + 32 * h;
                Xu[r * PM_XU + c] = v[u][h];
                XbT[c * PM_XB + r] = center8(v[u][h], p, half);
            }
        }
    }
    const int nblk = (nb + 63) >> 6;
    auto reduce_acc = [&](int a) -> uint32_t {  // s32 accumulator -> residue
        return fsub(f, red32(f, (uint32_t)a ^ 0x80000000u), bias);
    };
    // A-operand blocks in processing order: T(bi, 0..bi-1), then Tinv(bi).  The next
    // block's loads are in flight (registers) while the current one is multiplied.
    uint32_t pv[16];
    auto fetch = [&](int bi, int bj) {  // bj < 0: Tinv(bi)
        const int rb = bi * 64, rv = min(64, nb - rb);
        const uint32_t* src = bj < 0 ? Tinv + (int64_t)bi * 64 * 64 : T + (int64_t)rb * ldt + bj * 64;
        const int64_t ld = bj < 0 ? 64 : ldt;
        const int rmax = bj < 0 ? 64 : rv;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = threadIdx.x + 256 * u, r = e >> 6, c = e & 63;
            pv[u] = r < rmax ? __ldcg(src + (int64_t)r * ld + c) : 0u;
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = threadIdx.x + 256 * u, r = e >> 6, c = e & 63;
            Ab[r * PM_AB + c] = center8(pv[u], p, half);
        }
    };
    fetch(0, -1);
    for (int bi = 0; bi < nblk; ++bi) {
        const int rb = bi * 64;
        int acc[4][4];
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0;
        for (int bj = 0; bj < bi; ++bj) {
            __syncthreads();  // Ab free, X_bj complete
            store();
            __syncthreads();
            fetch(bi, bj + 1 < bi ? bj + 1 : -1);
            pm_mma(acc, Ab, XbT, bj * 64, mt, nt0, gid, tig);
        }
        __syncthreads();  // Ab free; XbT rows of block bi not read any more by the updates
        store();  // Tinv(bi)
        if (bi + 1 < nblk) fetch(bi + 1, 0);
        // Y = X_bi - acc (own fragment elements), exact and int8
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int row = rb + 16 * mt + gid + 8 * (e >> 1), col = 8 * (nt0 + t) + 2 * tig + (e & 1);
                const uint32_t y = fsub(f, Xu[row * PM_XU + col], reduce_acc(acc[t][e]));
                Xu[row * PM_XU + col] = y;
                XbT[col * PM_XB + row] = center8(y, p, half);
            }
        __syncthreads();
        int acc2[4][4];
#pragma unroll
        for (int t = 0; t < 4; ++t) acc2[t][0] = acc2[t][1] = acc2[t][2] = acc2[t][3] = 0;
        pm_mma(acc2, Ab, XbT, rb, mt, nt0, gid, tig);
        __syncthreads();  // every warp has read Y before X_bi overwrites it
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int row = rb + 16 * mt + gid + 8 * (e >> 1), col = 8 * (nt0 + t) + 2 * tig + (e & 1);
                const uint32_t x = row < nb ? reduce_acc(acc2[t][e]) : 0u;
                Xu[row * PM_XU + col] = x;
                XbT[col * PM_XB + row] = center8(x, p, half);
            }
    }
    __syncthreads();
    for (int r0 = wp; r0 < nb; r0 += 8)
        for (int c = lane; c < bc; c += 32) B[(int64_t)r0 * ldb + c0 + c] = Xu[r0 * PM_XU + c];
}

struct TrsmScratch {
    uint32_t* ptr = nullptr;
    size_t cap = 0;
};
thread_local TrsmScratch g_tscratch_dev[FFB_MAX_DEVICES];

uint32_t* trsm_scratch(size_t words) {
    TrsmScratch& g_tscratch = g_tscratch_dev[current_device()];
    if (g_tscratch.cap < words) {
        if (g_tscratch.ptr) {
            FFB_CUDA(cudaDeviceSynchronize());
            FFB_CUDA(cudaFree(g_tscratch.ptr));
        }
        const size_t cap = std::max(words * 2, (size_t)1 << 20);
        FFB_CUDA(cudaMalloc(&g_tscratch.ptr, cap * sizeof(uint32_t)));
        g_tscratch.cap = cap;
    }
    return g_tscratch.ptr;
}

void solve_rec(const Fp& f, cudaStream_t st, DMat T, DMat B, const uint32_t* Tinv, int64_t i0) {
    const int64_t n = T.rows;
    if (n <= 256) {
        ProfScope ps(K_TRSM, st, 2.0 * n * n * B.cols / 2, 8.0 * n * B.cols, n, B.cols, 1);
        const uint32_t* ti = Tinv + (i0 / 64) * 64 * 64;
        static const bool no_mma = getenv("FFB_TRSM_SIMT") != nullptr;  // test hook
        if (f.p <= 255 && !no_mma) {
            static DeviceOnce attr_mma;
            if (!attr_mma.done()) {
                FFB_CUDA(cudaFuncSetAttribute(k_trsm_panel_mma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)PM_SMEM));
                attr_mma.mark();
            }
            launch_k(k_trsm_panel_mma, (unsigned)cdiv(B.cols, PM_COLS), 256, PM_SMEM, st, f, T.ptr, T.ld, ti, B.ptr,
                                                                                 B.ld, (int)n, B.cols);
            ++g_launches;
            FFB_CHECK_LAUNCH();
            return;
        }
        const size_t smem = (size_t)(256 * (PNL_COLS + 1) + 64 * 65) * 4;
        static DeviceOnce attr;
        if (!attr.done()) {
            FFB_CUDA(cudaFuncSetAttribute(k_trsm_panel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            FFB_CUDA(cudaFuncSetAttribute(k_trsm_panel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr.mark();
        }
        // narrow right-hand sides (< 4 CTAs per SM at 32 columns): 8 columns per CTA
        const bool narrow = B.cols < (int64_t)PNL_COLS * 148;
        const size_t smem8 = (size_t)(256 * (8 + 1) + 64 * 65) * 4;
        if (narrow && f.p < (1u << 23))
            launch_k(k_trsm_panel<true, 8>, dim3((unsigned)cdiv(B.cols, 8)), 256, smem8, st, f, T.ptr, T.ld, ti,
                     B.ptr, B.ld, (int)n, B.cols);
        else if (narrow)
            launch_k(k_trsm_panel<false, 8>, dim3((unsigned)cdiv(B.cols, 8)), 256, smem8, st, f, T.ptr, T.ld, ti,
                     B.ptr, B.ld, (int)n, B.cols);
        else if (f.p < (1u << 23))
            launch_k(k_trsm_panel<true>, dim3((unsigned)cdiv(B.cols, PNL_COLS)), 256, smem, st, f, T.ptr, T.ld, ti,
                     B.ptr, B.ld, (int)n, B.cols);
        else
            launch_k(k_trsm_panel<false>, dim3((unsigned)cdiv(B.cols, PNL_COLS)), 256, smem, st, f, T.ptr, T.ld, ti,
                     B.ptr, B.ld, (int)n, B.cols);
        ++g_launches;
        FFB_CHECK_LAUNCH();
        return;
    }
    int64_t n1 = (n / 2) / 256 * 256;
    if (n1 < 256) n1 = 256;
    const int64_t n2 = n - n1;
    DMat B1 = B.sub(0, 0, n1, B.cols), B2 = B.sub(n1, 0, n2, B.cols);
    solve_rec(f, st, T.sub(0, 0, n1, n1), B1, Tinv, i0);
    gemm(f, st, GEMM_SUB, B2, T.sub(n1, 0, n2, n1), false, B1, false, n2, B.cols, n1);
    solve_rec(f, st, T.sub(n1, n1, n2, n2), B2, Tinv, i0 + n1);
}

}  // namespace

// Leaf micro-benchmark (tools/leaf_bench.py; not part of the C-ABI): reps launches of
// the leaf kernel on an s x s device matrix, average ms (CUDA events), rank in out[0].
void dbg_leaf_bench(const Fp& f, cudaStream_t st, int s, const uint32_t* d_a, int reps, double* ms,
                    int32_t* out_rank) {
    uint32_t* Lg;
    int32_t *rows, *out;
    DDiag D;
    FFB_CUDA(cudaMalloc(&Lg, (size_t)s * s * 4));
    FFB_CUDA(cudaMalloc(&rows, (size_t)s * 4 + 64));
    FFB_CUDA(cudaMalloc(&out, (size_t)(s + 2) * 4 + 64));
    FFB_CUDA(cudaMalloc(&D.kind, (size_t)s * 4 + 64));
    FFB_CUDA(cudaMalloc(&D.val, (size_t)s * 4 + 64));
    FFB_CUDA(cudaMalloc(&D.val2, (size_t)s * 4 + 64));
    FFB_CUDA(cudaMalloc(&D.inv, (size_t)s * 4 + 64));
    std::vector<int32_t> h(s);
    for (int i = 0; i < s; ++i) h[i] = i;
    FFB_CUDA(cudaMemcpy(rows, h.data(), (size_t)s * 4, cudaMemcpyHostToDevice));
    DMat A{const_cast<uint32_t*>(d_a), s, s, s}, L{Lg, s, s, s};
    cudaEvent_t e0, e1;
    FFB_CUDA(cudaEventCreate(&e0));
    FFB_CUDA(cudaEventCreate(&e1));
    leaf64(f, st, A, rows, L, 0, D, out, MboxPost());
    FFB_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; ++i) leaf64(f, st, A, rows, L, 0, D, out, MboxPost());
    FFB_CUDA(cudaEventRecord(e1, st));
    FFB_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    FFB_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / reps;
    FFB_CUDA(cudaMemcpy(out_rank, out, 4, cudaMemcpyDeviceToHost));
    for (void* q : {(void*)Lg, (void*)rows, (void*)out, (void*)D.kind, (void*)D.val, (void*)D.val2, (void*)D.inv})
        FFB_CUDA(cudaFree(q));
    FFB_CUDA(cudaEventDestroy(e0));
    FFB_CUDA(cudaEventDestroy(e1));
}

bool leaf64_supported(int64_t s) { return s <= 64; }

bool node128_supported(const Fp& f, int64_t s, int64_t T) {
    static const bool off = getenv("FFB_NO_NODE128") != nullptr;  // A/B hook
    return !off && f.p < 4096u && T <= 64 && s > T && s <= 2 * T && s <= 128;
}

void node128(const Fp& f, cudaStream_t st, DMat A, const int32_t* rows, DMat Lg, int64_t coff, DDiag D,
             uint32_t* yout, int32_t* out, const MboxPost& mp) {
    const int s = (int)A.rows;
    ProfScope ps(K_LEAF, st, 2.0 * s * s * s / 3.0, 4.0 * s * s);
    static DeviceOnce attr;
    if (!attr.done()) {
        FFB_CUDA(cudaFuncSetAttribute(k_node128, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)node_smem_bytes()));
        attr.mark();
    }
    launch_k(k_node128, 1, 128, node_smem_bytes(), st, f, A.ptr, A.ld, s, rows, Lg.ptr, Lg.ld, coff, D, yout, out,
             mp);
    ++g_launches;
    FFB_CHECK_LAUNCH();
}


void leaf64(const Fp& f, cudaStream_t st, DMat A, const int32_t* rows, DMat Lg, int64_t coff,
            DDiag D, int32_t* out, const MboxPost& mp) {
    const int s = (int)A.rows;
    ProfScope ps(K_LEAF, st, 2.0 * s * s * s / 3.0, 4.0 * s * s);
    static const bool eager = getenv("FFB_LEAF_EAGER") != nullptr;  // A/B hook
    if (f.p < 4096u && !eager)
        launch_k(k_leaf64_lazy<LzNarrow>, 1, 128, 0, st, f, A.ptr, A.ld, s, rows, Lg.ptr, Lg.ld, coff, D, out, mp);
    else if (f.p < (1u << 26) && !eager)  // large primes (config 3): int64 lazy entries
        launch_k(k_leaf64_lazy<LzWide>, 1, 128, 0, st, f, A.ptr, A.ld, s, rows, Lg.ptr, Lg.ld, coff, D, out, mp);
    else if (f.p < (1u << 16))
        launch_k(k_leaf64<true>, 1, 256, 0, st, f, A.ptr, A.ld, s, rows, Lg.ptr, Lg.ld, coff, D, out, mp);
    else
        launch_k(k_leaf64<false>, 1, 256, 0, st, f, A.ptr, A.ld, s, rows, Lg.ptr, Lg.ld, coff, D, out, mp);
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

void trsm_lower_unit(const Fp& f, cudaStream_t st, DMat T, DMat B) {
    const int64_t n = T.rows;
    if (n <= 0 || B.cols <= 0) return;
    if (n <= 64) {  // one launch: inverse and apply per 64-column tile
        ProfScope ps(K_TRSM, st, (double)n * n * B.cols, 8.0 * n * B.cols, n, B.cols, 2);
        const unsigned g = (unsigned)cdiv(B.cols, 64);
        static const bool inv_path = getenv("FFB_TRSM_INV") != nullptr;  // A/B hook
        if (inv_path) {
            if (f.p < 4096u) launch_k(k_trsm_small<0>, g, 256, 0, st, f, T.ptr, T.ld, (int)n, B.ptr, B.ld, B.cols);
            else if (f.p < (1u << 23))
                launch_k(k_trsm_small<1>, g, 256, 0, st, f, T.ptr, T.ld, (int)n, B.ptr, B.ld, B.cols);
            else launch_k(k_trsm_small<2>, g, 256, 0, st, f, T.ptr, T.ld, (int)n, B.ptr, B.ld, B.cols);
        } else {
            if (f.p < 4096u) launch_k(k_trsm_fwd<0>, g, 256, 0, st, f, T.ptr, T.ld, (int)n, B.ptr, B.ld, B.cols);
            else if (f.p < (1u << 23))
                launch_k(k_trsm_fwd<1>, g, 256, 0, st, f, T.ptr, T.ld, (int)n, B.ptr, B.ld, B.cols);
            else launch_k(k_trsm_fwd<2>, g, 256, 0, st, f, T.ptr, T.ld, (int)n, B.ptr, B.ld, B.cols);
        }
        ++g_launches;
        FFB_CHECK_LAUNCH();
        return;
    }
    const int64_t nblk = cdiv(n, 64);
    uint32_t* Tinv = trsm_scratch((size_t)nblk * 64 * 64);
    {
        ProfScope ps(K_TRSM, st, (double)n * 64 * 64 / 3, 8.0 * n * 64, n, B.cols, 0);
        if (f.p < 4096u)
            launch_k(k_trinv64<0>, (unsigned)nblk, 256, 0, st, f, T.ptr, T.ld, n, Tinv);
        else if (f.p < (1u << 23))
            launch_k(k_trinv64<1>, (unsigned)nblk, 256, 0, st, f, T.ptr, T.ld, n, Tinv);
        else
            launch_k(k_trinv64<2>, (unsigned)nblk, 256, 0, st, f, T.ptr, T.ld, n, Tinv);
        ++g_launches;
        FFB_CHECK_LAUNCH();
    }
    solve_rec(f, st, T, B, Tinv, 0);
}

}  // namespace ffb

// diagnostics: SM-clock stamps of the last fused small node (tools/node_stamps.py)
extern "C" int ffb_dbg_node_stamps(long long* out9) {
    return cudaMemcpyFromSymbol(out9, ffb::g_node_stamp, 9 * sizeof(long long)) == cudaSuccess ? 0 : 1;
}
