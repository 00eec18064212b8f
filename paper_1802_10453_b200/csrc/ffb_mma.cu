// ffb_mma.cu -- modular GEMM on the warp-level int8 tensor cores (mma.sync
// m16n8k32) for p <= 255 and small / mid shapes:
//   C (M x N) = C -/+ op(A) op(B)   or   op(A) op(B)    (mod p)
// The u32 operands are read directly (no packing pass): each 64-deep K chunk
// of the 64 x 64 output tile is fetched into registers (the next chunk's
// loads overlap this chunk's MMAs), centered to int8 and staged in shared
// memory k-contiguous for the fragments.  Products accumulate exactly in s32
// (|acc| <= K 127^2 < 2^31); the epilogue reduces once per output.
// Large GEMMs use the tcgen05/TMA kernel (ffb_tc_gemm.cu) instead.
#include <algorithm>

#include "ffb_kernels.cuh"
#include "ffb_mma.cuh"

namespace ffb {

namespace {

constexpr int MM_T = 64, MM_S = 64 + 16;  // tile edge, smem row stride in bytes (conflict-free frags)

// Split K: CTA z covers k in [z kc, (z+1) kc) and, when gridDim.z > 1, writes
// its reduced partial tile to W[z] (M x N, ld N) for k_splitk_fold.
// Second problem of a paired launch (blockIdx.z = 1), same mode and orientation.
struct MmaProb {
    uint32_t* C;
    int64_t ldc;
    const uint32_t* A;
    int64_t lda;
    const uint32_t* B;
    int64_t ldb;
    int64_t M, N, K;
};
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_gemm_mma(Fp f, int mode, uint32_t* C, int64_t ldc,
                                                  const uint32_t* A, int64_t lda,
                                                  const uint32_t* B, int64_t ldb, int64_t M,
                                                  int64_t N, int64_t K, int64_t kc, uint32_t* W,
                                                  int pair, MmaProb p2, int32_t* nzflag, int32_t nztag) {
    FFB_PDL_ENTRY();
    // pair: blockIdx.z selects the problem (no split-K); problem 0 may publish nztag
    // to *nzflag when any output is nonzero (the zero test of the next recursion step)
    if (pair && blockIdx.z == 1) {
        C = p2.C, ldc = p2.ldc, A = p2.A, lda = p2.lda, B = p2.B, ldb = p2.ldb, M = p2.M, N = p2.N, K = p2.K;
        nzflag = nullptr;
    }
    if ((int64_t)blockIdx.y * MM_T >= M || (int64_t)blockIdx.x * MM_T >= N) return;  // uniform
    const bool splitk = !pair && gridDim.z > 1;
    __shared__ __align__(16) int8_t As[MM_T * MM_S];  // op(A) tile [m][k]
    __shared__ __align__(16) int8_t Bs[MM_T * MM_S];  // op(B) tile transposed [n][k]
    __shared__ uint32_t Cs[MM_T][MM_T + 1];           // reduced tile, for a coalesced epilogue
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, gid = lane >> 2, tig = lane & 3;
    const int mt = wp & 3, nt0 = (wp >> 2) * 4;
    const int64_t m0 = (int64_t)blockIdx.y * MM_T, n0 = (int64_t)blockIdx.x * MM_T;
    const uint32_t p = f.p, half = (p - 1) / 2, bias = (uint32_t)(0x80000000ull % p);
    uint32_t ra[16], rb[16];
    // element u of this thread: e = tid + 256 u, (hi, lo) = (e / 64, e % 64), lo along the
    // contiguous dimension of the stored operand (coalesced loads)
    auto fetch = [&](int64_t k0) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = tid + 256 * u, hi = e >> 6, lo = e & 63;
            {
                const int64_t m = m0 + (TA ? lo : hi), k = k0 + (TA ? hi : lo);
                ra[u] = (m < M && k < K) ? __ldcg(TA ? A + k * lda + m : A + m * lda + k) : 0u;
            }
            {
                const int64_t n = n0 + (TB ? hi : lo), k = k0 + (TB ? lo : hi);
                rb[u] = (n < N && k < K) ? __ldcg(TB ? B + n * ldb + k : B + k * ldb + n) : 0u;
            }
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = tid + 256 * u, hi = e >> 6, lo = e & 63;
            As[(TA ? lo : hi) * MM_S + (TA ? hi : lo)] = center8(ra[u], p, half);
            Bs[(TB ? hi : lo) * MM_S + (TB ? lo : hi)] = center8(rb[u], p, half);
        }
    };
    const int64_t kb = splitk ? (int64_t)blockIdx.z * kc : 0;
    K = splitk ? std::min<int64_t>(K, kb + kc) : K;  // this CTA's K range is [kb, K)
    int acc[4][4];
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0;
    // the C values of this thread's epilogue slots (rows wp + 8i, columns lane, lane + 32)
    // do not depend on the product: load them now, overlapped with the K loop
    uint32_t cpre[16];
    const bool direct = !splitk && mode != GEMM_SET;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t row = m0 + wp + 8 * i, col = n0 + lane + 32 * h;
            cpre[2 * i + h] = (direct && row < M && col < N) ? __ldcg(C + row * ldc + col) : 0u;
        }
    fetch(kb);
    for (int64_t k0 = kb; k0 < K; k0 += MM_T) {
        __syncthreads();  // the previous chunk's fragments have been read
        stash();
        __syncthreads();
        if (k0 + MM_T < K) fetch(k0 + MM_T);  // in flight during the MMAs
#pragma unroll
        for (int ks = 0; ks < MM_T; ks += 32) {
            const int8_t* ar0 = As + (16 * mt + gid) * MM_S + ks + tig * 4;
            const int8_t* ar1 = ar0 + 8 * MM_S;
            const uint32_t a0 = *(const uint32_t*)ar0, a1 = *(const uint32_t*)ar1;
            const uint32_t a2 = *(const uint32_t*)(ar0 + 16), a3 = *(const uint32_t*)(ar1 + 16);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int8_t* bp = Bs + (8 * (nt0 + t) + gid) * MM_S + ks + tig * 4;
                mma_s8_16832(acc[t], a0, a1, a2, a3, *(const uint32_t*)bp, *(const uint32_t*)(bp + 16));
            }
        }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int e = 0; e < 4; ++e)
            Cs[16 * mt + gid + 8 * (e >> 1)][8 * (nt0 + t) + 2 * tig + (e & 1)] = mma_reduce(f, acc[t][e], bias);
    __syncthreads();
    // coalesced epilogue: warp per row, lanes along the columns
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = wp + 8 * i;
        const int64_t row = m0 + r;
        if (row >= M) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t col = n0 + lane + 32 * h;
            if (col >= N) continue;
            const uint32_t v = Cs[r][lane + 32 * h];
            if (splitk) {
                W[((int64_t)blockIdx.z * M + row) * N + col] = v;
                continue;
            }
            const uint32_t c0 = cpre[2 * i + h];
            uint32_t* c = C + row * ldc + col;
            uint32_t o;
            if (mode == GEMM_SUB) o = fsub(f, c0, v);
            else if (mode == GEMM_ADD) o = fadd(f, c0, v);
            else o = v;
            *c = o;
            if (nzflag && o) *nzflag = nztag;
        }
    }
}

// C = C -/+ sum_z W[z]  or  sum_z W[z]   (mod p)
__global__ void k_splitk_fold(Fp f, int mode, uint32_t* C, int64_t ldc, const uint32_t* W, int64_t M,
                              int64_t N, int S) {
    FFB_PDL_ENTRY();
    const int64_t row = blockIdx.y;
    for (int64_t col = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; col < N;
         col += (int64_t)gridDim.x * blockDim.x) {
        uint64_t acc = 0;
        for (int z = 0; z < S; ++z) acc += W[((int64_t)z * M + row) * N + col];
        const uint32_t v = red64(f, acc);
        uint32_t* c = C + row * ldc + col;
        if (mode == GEMM_SUB) *c = fsub(f, *c, v);
        else if (mode == GEMM_ADD) *c = fadd(f, *c, v);
        else *c = v;
    }
}

struct MmaScratch {
    uint32_t* ptr = nullptr;
    size_t cap = 0;
};
thread_local MmaScratch g_mscratch_slots[FFB_MAX_DEVICES][6];
uint32_t* mma_scratch(size_t words) {
    MmaScratch& g_mscratch = g_mscratch_slots[current_device()][g_slot];
    if (g_mscratch.cap < words) {
        if (g_mscratch.ptr) {
            FFB_CUDA(cudaDeviceSynchronize());
            FFB_CUDA(cudaFree(g_mscratch.ptr));
        }
        const size_t cap = std::max(words * 2, (size_t)1 << 22);
        FFB_CUDA(cudaMalloc(&g_mscratch.ptr, cap * sizeof(uint32_t)));
        g_mscratch.cap = cap;
    }
    return g_mscratch.ptr;
}

}  // namespace

bool mma_gemm_supported(const Fp& f, int64_t M, int64_t N, int64_t K) {
    static const bool disabled = getenv("FFB_DISABLE_MMA") != nullptr;  // test hook
    return !disabled && f.p <= 255 && K <= 120000 && M < (1ll << 31) / MM_T * MM_T &&
           cdiv(M, MM_T) <= 65535;
}

void mma_gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
              int64_t M, int64_t N, int64_t K) {
    ProfScope ps(K_GEMM, st, 2.0 * M * N * K, 4.0 * (M * K + K * N + 2 * M * N), M, -N, K);  // -N marks mma
    // split K when the output has too few tiles to fill the GPU and K is long
    const int64_t tiles = cdiv(N, MM_T) * cdiv(M, MM_T);
    int S = 1;
    static const int64_t split_ctas = getenv("FFB_MMA_SPLIT_CTAS") ? atoll(getenv("FFB_MMA_SPLIT_CTAS")) : 148;
    if (tiles < split_ctas && K >= 512 && M * N <= ((int64_t)1 << 24))
        S = (int)std::min<int64_t>(cdiv(K, 256), std::max<int64_t>(1, 2 * split_ctas / tiles));
    const int64_t kc = cdiv(cdiv(K, S), MM_T) * MM_T;
    S = (int)cdiv(K, kc);
    uint32_t* W = S > 1 ? mma_scratch((size_t)S * M * N) : nullptr;
    const dim3 grid((unsigned)cdiv(N, MM_T), (unsigned)cdiv(M, MM_T), (unsigned)S);
#define FFB_MMA_LAUNCH(TA, TB)                                                                       \
    launch_k(k_gemm_mma<TA, TB>, grid, 256, 0, st, f, (int)mode, C.ptr, C.ld, A.ptr, A.ld, B.ptr, B.ld, M, N, K, \
                                             kc, W, 0, MmaProb{}, (int32_t*)nullptr, 0)
    if (!ta && !tb) FFB_MMA_LAUNCH(false, false);
    else if (ta && !tb) FFB_MMA_LAUNCH(true, false);
    else if (!ta && tb) FFB_MMA_LAUNCH(false, true);
    else FFB_MMA_LAUNCH(true, true);
#undef FFB_MMA_LAUNCH
    if (S > 1) {
        ++g_launches;
        launch_k(k_splitk_fold, dim3((unsigned)cdiv(N, 256), (unsigned)M), 256, 0, st, f, (int)mode, C.ptr, C.ld, W, M,
                                                                                  N, S);
    }
    ++g_launches;
    FFB_CHECK_LAUNCH();
}


// ===========================================================================
// Short-K update (p <= 255, K <= 128): C -/+= op(A) op(B) or C = op(A) op(B)
// is a stream over C with K multiply-adds per element, so it is written as a
// bandwidth kernel: a CTA owns 256 columns and a strip of TR rows; op(B) for
// its columns and op(A) for its rows are staged once in shared memory as
// centered int8 x 4 packs along k, and each thread streams 16-byte C vectors
// (4 columns), RK rows in flight, with one dp4a per k-quad and column.
// ===========================================================================
namespace {

constexpr int RK_COLS = 256, RK_RU = 4;  // columns per CTA, row unroll (loads in flight)

__device__ __forceinline__ uint32_t pack4c(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t p,
                                           uint32_t half) {
    return (uint32_t)(uint8_t)center8(a, p, half) | ((uint32_t)(uint8_t)center8(b, p, half) << 8) |
           ((uint32_t)(uint8_t)center8(c, p, half) << 16) | ((uint32_t)(uint8_t)center8(d, p, half) << 24);
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_rankk_dp4a(Fp f, int mode, uint32_t* C, int64_t ldc,
                                                    const uint32_t* A, int64_t lda,
                                                    const uint32_t* B, int64_t ldb, int64_t M,
                                                    int64_t N, int K, int TR) {
    FFB_PDL_ENTRY();
    extern __shared__ __align__(16) uint32_t rk_sm[];
    const int K4 = (K + 3) >> 2;
    uint32_t* Bp = rk_sm;                       // [K4][RK_COLS]  packs of op(B)[4q..4q+3][j]
    uint32_t* Ap = Bp + (size_t)K4 * RK_COLS;   // [TR][K4]       packs of op(A)[i][4q..4q+3]
    const int tid = threadIdx.x;
    const int64_t n0 = (int64_t)blockIdx.x * RK_COLS, m0 = (int64_t)blockIdx.y * TR;
    const int rows = (int)std::min<int64_t>(TR, M - m0);
    const uint32_t p = f.p, half = (p - 1) / 2, bias = (uint32_t)(0x80000000ull % p);
    auto opB = [&](int k, int64_t n) -> uint32_t {
        return (k < K && n < N) ? __ldcg(TB ? B + n * ldb + k : B + (int64_t)k * ldb + n) : 0u;
    };
    auto opA = [&](int64_t m, int k) -> uint32_t {
        return (k < K && m < M) ? __ldcg(TA ? A + (int64_t)k * lda + m : A + m * lda + k) : 0u;
    };
    for (int e = tid; e < K4 * RK_COLS; e += 256) {
        const int q = e / RK_COLS, j = e - q * RK_COLS;
        const int64_t n = n0 + j;
        Bp[e] = pack4c(opB(4 * q, n), opB(4 * q + 1, n), opB(4 * q + 2, n), opB(4 * q + 3, n), p, half);
    }
    for (int e = tid; e < rows * K4; e += 256) {
        const int i = e / K4, q = e - i * K4;
        const int64_t m = m0 + i;
        Ap[e] = pack4c(opA(m, 4 * q), opA(m, 4 * q + 1), opA(m, 4 * q + 2), opA(m, 4 * q + 3), p, half);
    }
    __syncthreads();
    const int cg = tid & 63, rp = tid >> 6;  // 4 columns per thread, 4 row phases
    const int64_t col = n0 + 4 * cg;
    const bool vec = col + 3 < N && ((ldc & 3) == 0) && ((((uintptr_t)C) & 15) == 0);
    for (int i0 = rp; i0 < rows; i0 += 4 * RK_RU) {
        uint4 cv[RK_RU];
#pragma unroll
        for (int u = 0; u < RK_RU; ++u) {  // C loads in flight
            const int i = i0 + 4 * u;
            cv[u] = make_uint4(0, 0, 0, 0);
            if (i < rows && mode != GEMM_SET) {
                const uint32_t* cp = C + (m0 + i) * ldc + col;
                if (vec) cv[u] = __ldcg(reinterpret_cast<const uint4*>(cp));
                else {
                    cv[u].x = col < N ? cp[0] : 0u;
                    cv[u].y = col + 1 < N ? cp[1] : 0u;
                    cv[u].z = col + 2 < N ? cp[2] : 0u;
                    cv[u].w = col + 3 < N ? cp[3] : 0u;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < RK_RU; ++u) {
            const int i = i0 + 4 * u;
            if (i >= rows) break;
            const uint32_t* ai = Ap + (size_t)i * K4;
            int a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            for (int q = 0; q < K4; ++q) {
                const int av = (int)ai[q];
                const uint4 bv = *reinterpret_cast<const uint4*>(Bp + (size_t)q * RK_COLS + 4 * cg);
                a0 = __dp4a(av, (int)bv.x, a0);
                a1 = __dp4a(av, (int)bv.y, a1);
                a2 = __dp4a(av, (int)bv.z, a2);
                a3 = __dp4a(av, (int)bv.w, a3);
            }
            uint32_t v[4] = {mma_reduce(f, a0, bias), mma_reduce(f, a1, bias), mma_reduce(f, a2, bias),
                             mma_reduce(f, a3, bias)};
            uint32_t c[4] = {cv[u].x, cv[u].y, cv[u].z, cv[u].w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if (mode == GEMM_SUB) c[h] = fsub(f, c[h], v[h]);
                else if (mode == GEMM_ADD) c[h] = fadd(f, c[h], v[h]);
                else c[h] = v[h];
            }
            uint32_t* cp = C + (m0 + i) * ldc + col;
            if (vec) *reinterpret_cast<uint4*>(cp) = make_uint4(c[0], c[1], c[2], c[3]);
            else
                for (int h = 0; h < 4; ++h)
                    if (col + h < N) cp[h] = c[h];
        }
    }
}

}  // namespace

bool mma_gemm_pair(const Fp& f, cudaStream_t st, DMat C1, DMat A1, DMat B1, int64_t M1, int64_t N1, int64_t K1,
                   DMat C2, DMat A2, DMat B2, int64_t M2, int64_t N2, int64_t K2, int32_t* nzflag, int32_t tag) {
    // both on the mma path without split-K (small products), non-transposed, GEMM_SUB
    auto small = [&](int64_t M, int64_t N, int64_t K) {
        const int64_t tiles = cdiv(N, MM_T) * cdiv(M, MM_T);
        const bool split = tiles < 148 && K >= 512 && M * N <= ((int64_t)1 << 24);
        return M > 0 && N > 0 && K > 0 && !split && mma_gemm_supported(f, M, N, K) &&
               !(M >= 128 && N >= 128 && (double)M * N * K >= 2.7e8) && !(K <= 32 && rankk_supported(f, M, N, K));
    };
    if (getenv("FFB_GEMM_PATH") || !small(M1, N1, K1) || !small(M2, N2, K2)) return false;
    ProfScope ps(K_GEMM, st, 2.0 * (M1 * N1 * K1 + M2 * N2 * K2), 0.0, M1, -N1, K1);
    const dim3 grid((unsigned)std::max(cdiv(N1, MM_T), cdiv(N2, MM_T)),
                    (unsigned)std::max(cdiv(M1, MM_T), cdiv(M2, MM_T)), 2);
    const MmaProb p2{C2.ptr, C2.ld, A2.ptr, A2.ld, B2.ptr, B2.ld, M2, N2, K2};
    launch_k(k_gemm_mma<false, false>, grid, 256, 0, st, f, (int)GEMM_SUB, C1.ptr, C1.ld, A1.ptr, A1.ld, B1.ptr,
             B1.ld, M1, N1, K1, K1, (uint32_t*)nullptr, 1, p2, nzflag, tag);
    ++g_launches;
    FFB_CHECK_LAUNCH();
    return true;
}

bool rankk_supported(const Fp& f, int64_t M, int64_t N, int64_t K) {
    static const bool disabled = getenv("FFB_DISABLE_RANKK") != nullptr;  // test hook
    return !disabled && f.p <= 255 && K >= 1 && K <= 128 && N >= 64 && M * N >= ((int64_t)1 << 18);
}

void rankk_gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
                int64_t M, int64_t N, int64_t K) {
    ProfScope ps(K_GEMM, st, 2.0 * M * N * K, 8.0 * M * N, -M, -N, K);  // -M,-N marks the rank-k kernel
    // rows per CTA: B re-reads (M / TR) K N 4 bytes stay <= 1/4 of the C traffic 8 M N
    int TR = (int)std::max<int64_t>(64, 2 * K);
    const int64_t ncb = cdiv(N, RK_COLS);
    while (TR > 16 && ncb * cdiv(M, TR) < 4 * 148) TR /= 2;  // enough CTAs to fill the GPU
    const int K4 = (int)((K + 3) / 4);
    const size_t smem = ((size_t)K4 * RK_COLS + (size_t)TR * K4) * 4;
    static DeviceOnce attr;
    if (!attr.done()) {
        for (auto fn : {k_rankk_dp4a<false, false>, k_rankk_dp4a<true, false>, k_rankk_dp4a<false, true>,
                        k_rankk_dp4a<true, true>})
            FFB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        attr.mark();
    }
    const dim3 grid((unsigned)ncb, (unsigned)cdiv(M, TR));
#define FFB_RK_LAUNCH(TA, TB) \
    launch_k(k_rankk_dp4a<TA, TB>, grid, 256, smem, st, f, (int)mode, C.ptr, C.ld, A.ptr, A.ld, B.ptr, B.ld, M, N, (int)K, TR)
    if (!ta && !tb) FFB_RK_LAUNCH(false, false);
    else if (ta && !tb) FFB_RK_LAUNCH(true, false);
    else if (!ta && tb) FFB_RK_LAUNCH(false, true);
    else FFB_RK_LAUNCH(true, true);
#undef FFB_RK_LAUNCH
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

}  // namespace ffb
