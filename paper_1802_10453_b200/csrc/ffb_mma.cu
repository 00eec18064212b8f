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
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_gemm_mma(Fp f, int mode, uint32_t* __restrict__ C, int64_t ldc,
                                                  const uint32_t* __restrict__ A, int64_t lda,
                                                  const uint32_t* __restrict__ B, int64_t ldb, int64_t M,
                                                  int64_t N, int64_t K, int64_t kc, uint32_t* __restrict__ W) {
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
                ra[u] = (m < M && k < K) ? __ldg(TA ? A + k * lda + m : A + m * lda + k) : 0u;
            }
            {
                const int64_t n = n0 + (TB ? hi : lo), k = k0 + (TB ? lo : hi);
                rb[u] = (n < N && k < K) ? __ldg(TB ? B + n * ldb + k : B + k * ldb + n) : 0u;
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
    const int64_t kb = (int64_t)blockIdx.z * kc;
    K = std::min<int64_t>(K, kb + kc);  // this CTA's K range is [kb, K)
    int acc[4][4];
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0;
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
    for (int r = wp; r < MM_T; r += 8) {
        const int64_t row = m0 + r;
        if (row >= M) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int64_t col = n0 + lane + 32 * h;
            if (col >= N) continue;
            const uint32_t v = Cs[r][lane + 32 * h];
            if (gridDim.z > 1) {
                W[((int64_t)blockIdx.z * M + row) * N + col] = v;
                continue;
            }
            uint32_t* c = C + row * ldc + col;
            if (mode == GEMM_SUB) *c = fsub(f, *c, v);
            else if (mode == GEMM_ADD) *c = fadd(f, *c, v);
            else *c = v;
        }
    }
}

// C = C -/+ sum_z W[z]  or  sum_z W[z]   (mod p)
__global__ void k_splitk_fold(Fp f, int mode, uint32_t* C, int64_t ldc, const uint32_t* W, int64_t M,
                              int64_t N, int S) {
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
thread_local MmaScratch g_mscratch;
uint32_t* mma_scratch(size_t words) {
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
    if (tiles < 148 && K >= 512 && M * N <= ((int64_t)1 << 24))
        S = (int)std::min<int64_t>(cdiv(K, 256), std::max<int64_t>(1, 296 / tiles));
    const int64_t kc = cdiv(cdiv(K, S), MM_T) * MM_T;
    S = (int)cdiv(K, kc);
    uint32_t* W = S > 1 ? mma_scratch((size_t)S * M * N) : nullptr;
    const dim3 grid((unsigned)cdiv(N, MM_T), (unsigned)cdiv(M, MM_T), (unsigned)S);
#define FFB_MMA_LAUNCH(TA, TB)                                                                       \
    k_gemm_mma<TA, TB><<<grid, 256, 0, st>>>(f, (int)mode, C.ptr, C.ld, A.ptr, A.ld, B.ptr, B.ld, M, N, K, \
                                             kc, W)
    if (!ta && !tb) FFB_MMA_LAUNCH(false, false);
    else if (ta && !tb) FFB_MMA_LAUNCH(true, false);
    else if (!ta && tb) FFB_MMA_LAUNCH(false, true);
    else FFB_MMA_LAUNCH(true, true);
#undef FFB_MMA_LAUNCH
    if (S > 1) {
        ++g_launches;
        k_splitk_fold<<<dim3((unsigned)cdiv(N, 256), (unsigned)M), 256, 0, st>>>(f, (int)mode, C.ptr, C.ld, W, M,
                                                                                  N, S);
    }
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

}  // namespace ffb
