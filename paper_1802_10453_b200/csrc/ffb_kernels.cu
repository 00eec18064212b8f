// ffb_kernels.cu -- SIMT kernels of the PLDL^TP^T engine.
//
// Bandwidth-bound helpers (gathers, transposes, scaling), the Crout leaf
// (Alg. 4), PLDUQ (row-order Crout with leftmost pivots), the small
// triangular solves, and the generic modular GEMM used for every
// contraction that the tcgen05 path (ffb_tc_gemm.cu) does not take.
#include <string.h>
#include <cstdio>
#include <stdlib.h>

#include <algorithm>

#include "ffb_kernels.cuh"

namespace ffb {

thread_local uint64_t g_launches = 0;
thread_local int64_t g_node = 0;
thread_local int g_slot = 0;
thread_local bool g_tc_shared_sms = false;
thread_local int g_band_halo = -1;
thread_local Profiler* g_prof = nullptr;

static inline void count_launch() { ++g_launches; }

cudaEvent_t Profiler::get() {
    if (!pool.empty()) {
        cudaEvent_t e = pool.back();
        pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    FFB_CUDA(cudaEventCreate(&e));
    return e;
}
void Profiler::flush() {
    // FFB_PROF_TRACE=<file>: one line per profiled launch (class, shape, ms), appended
    static FILE* trace = getenv("FFB_PROF_TRACE") ? fopen(getenv("FFB_PROF_TRACE"), "a") : nullptr;
    for (Rec& r : recs) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) ms[r.cls] += t;
        if (trace)
            fprintf(trace, "%d %lld %lld %lld %.4f %lld %.6g\n", r.cls, (long long)r.m, (long long)r.n,
                    (long long)r.k, t, (long long)r.node, r.ops);
        ops[r.cls] += r.ops;
        bytes[r.cls] += r.bytes;
        cnt[r.cls] += 1;
        pool.push_back(r.a);
        pool.push_back(r.b);
    }
    recs.clear();
    if (trace) fflush(trace);
}
void Profiler::reset() {
    for (int i = 0; i < K_NCLASS; ++i) ms[i] = ops[i] = bytes[i] = 0, cnt[i] = 0;
}
ProfScope::ProfScope(int cls, cudaStream_t s, double ops, double bytes, int64_t m, int64_t n,
                     int64_t k)
    : st(s) {
    live = g_prof && g_prof->on;
    if (!live) return;
    rec.cls = cls;
    rec.m = m;
    rec.n = n;
    rec.k = k;
    rec.node = g_node;
    rec.ops = ops;
    rec.bytes = bytes;
    rec.a = g_prof->get();
    rec.b = g_prof->get();
    cudaEventRecord(rec.a, st);
}
ProfScope::~ProfScope() {
    if (!live) return;
    cudaEventRecord(rec.b, st);
    g_prof->recs.push_back(rec);
}

namespace {
struct PhaseRec { const char* label; int64_t size; cudaEvent_t e; };
thread_local std::vector<PhaseRec> g_phase;
const char* phase_path() {
    static const char* p = getenv("FFB_PHASE_TRACE");
    return p;
}
}  // namespace
void phase_mark(const char* label, int64_t size, cudaStream_t st) {
    static const int64_t min_size = getenv("FFB_PHASE_MIN") ? atoll(getenv("FFB_PHASE_MIN")) : 8192;
    if (!phase_path() || size < min_size) return;
    cudaEvent_t e;
    FFB_CUDA(cudaEventCreate(&e));
    FFB_CUDA(cudaEventRecord(e, st));
    g_phase.push_back({label, size, e});
}
void phase_dump(cudaStream_t st) {
    if (!phase_path() || g_phase.empty()) return;
    FFB_CUDA(cudaStreamSynchronize(st));
    if (FILE* fd = fopen(phase_path(), "a")) {
        float prev = 0.f;
        for (const PhaseRec& r : g_phase) {
            float t = 0.f;
            cudaEventElapsedTime(&t, g_phase[0].e, r.e);
            fprintf(fd, "%9.3f %8.3f %6lld %s\n", t, t - prev, (long long)r.size, r.label);
            prev = t;
        }
        fprintf(fd, "--\n");
        fclose(fd);
    }
    for (const PhaseRec& r : g_phase) cudaEventDestroy(r.e);
    g_phase.clear();
}

// ===========================================================================
// Generic modular GEMM (SIMT).  64x64 tile, 256 threads, 4x4 per thread,
// uint64 accumulation with delayed reduction (p < 2^23: one reduction per
// output; larger p: products reduced before accumulation).
// ===========================================================================
namespace {

constexpr int GB_M = 64, GB_N = 64, GB_K = 16;

template <bool TA, bool TB, bool kLargeP>
__global__ void __launch_bounds__(256) k_gemm_simt(Fp f, int mode, uint32_t* C,
                                                   int64_t ldc, const uint32_t* A,
                                                   int64_t lda, const uint32_t* B,
                                                   int64_t ldb, int64_t M, int64_t N, int64_t K) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t As[GB_K][GB_M + 4];
    __shared__ uint32_t Bs[GB_K][GB_N + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = (int64_t)blockIdx.y * GB_M, n0 = (int64_t)blockIdx.x * GB_N;
    uint64_t acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0;

    // Each thread moves 4 A and 4 B elements per K tile; the next tile is
    // prefetched into registers while the current one is consumed.
    uint32_t ra[4], rb[4];
    auto fetch = [&](int64_t k0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = threadIdx.x + 256 * u;
            int i, kk;
            if (TA) { i = e % GB_M; kk = e / GB_M; } else { kk = e % GB_K; i = e / GB_K; }
            const int64_t gi = m0 + i, gk = k0 + kk;
            ra[u] = (gi < M && gk < K) ? __ldcg(TA ? A + gk * lda + gi : A + gi * lda + gk) : 0u;
            int j, kb;
            if (TB) { kb = e % GB_K; j = e / GB_K; } else { j = e % GB_N; kb = e / GB_N; }
            const int64_t gj = n0 + j, gkb = k0 + kb;
            rb[u] = (gj < N && gkb < K) ? __ldcg(TB ? B + gj * ldb + gkb : B + gkb * ldb + gj) : 0u;
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = threadIdx.x + 256 * u;
            int i, kk;
            if (TA) { i = e % GB_M; kk = e / GB_M; } else { kk = e % GB_K; i = e / GB_K; }
            As[kk][i] = ra[u];
            int j, kb;
            if (TB) { kb = e % GB_K; j = e / GB_K; } else { j = e % GB_N; kb = e / GB_N; }
            Bs[kb][j] = rb[u];
        }
    };
    fetch(0);
    for (int64_t k0 = 0; k0 < K; k0 += GB_K) {
        stash();
        __syncthreads();
        if (k0 + GB_K < K) fetch(k0 + GB_K);
#pragma unroll
        for (int kk = 0; kk < GB_K; ++kk) {
            uint32_t a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint64_t prod = (uint64_t)a[i] * b[j];
                    acc[i][j] += kLargeP ? (uint64_t)red64(f, prod) : prod;
                }
        }
        __syncthreads();
        if (!kLargeP && ((k0 / GB_K) & 0x1FFF) == 0x1FFF) {  // 2^17 products: fold
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = red64(f, acc[i][j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gi = m0 + ty + 16 * i;
        if (gi >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gj = n0 + tx + 16 * j;
            if (gj >= N) continue;
            const uint32_t v = red64(f, acc[i][j]);
            uint32_t* c = C + gi * ldc + gj;
            if (mode == GEMM_SUB) *c = fsub(f, *c, v);
            else if (mode == GEMM_ADD) *c = fadd(f, *c, v);
            else *c = v;
        }
    }
}

template <bool TA, bool TB>
void launch_gemm_simt(const Fp& f, cudaStream_t st, int mode, DMat C, DMat A, DMat B, int64_t M,
                      int64_t N, int64_t K) {
    dim3 grid((unsigned)cdiv(N, GB_N), (unsigned)cdiv(M, GB_M));
    ProfScope ps(K_GEMM, st, 2.0 * M * N * K, 4.0 * (M * K + K * N + 2 * M * N), -M, N, K);  // -M marks SIMT
    if (f.p < (1u << 23))
        launch_k(k_gemm_simt<TA, TB, false>, grid, 256, 0, st, f, mode, C.ptr, C.ld, A.ptr, A.ld, B.ptr,
                                                          B.ld, M, N, K);
    else
        launch_k(k_gemm_simt<TA, TB, true>, grid, 256, 0, st, f, mode, C.ptr, C.ld, A.ptr, A.ld, B.ptr,
                                                         B.ld, M, N, K);
    count_launch();
    FFB_CHECK_LAUNCH();
}

}  // namespace

void gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
          int64_t M, int64_t N, int64_t K) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0) {
        if (mode == GEMM_SET) zero_mat(st, C.sub(0, 0, M, N));
        return;
    }
    // p <= 255: the tcgen05 pipeline (packed operands, TMA) from ~2^28 MACs with
    // both output dims >= 128; warp-level mma.sync on the raw residues below that
    // (measured crossover, tools/gemm_bench.py)
    bool big = M >= 128 && N >= 128 && (double)M * N * K >= 2.7e8;
    // test hook, read per call: FFB_GEMM_PATH=tc|mma|simt forces a path where it applies
    const char* force = getenv("FFB_GEMM_PATH");
    bool rk = K <= 32 && rankk_supported(f, M, N, K);  // short K: C streaming dominates
    if (force) {
        rk = !strcmp(force, "rankk") && rankk_supported(f, M, N, K);
        if (!strcmp(force, "tc")) big = true;
        else if (!strcmp(force, "simt")) goto simt;
        else if (!strcmp(force, "mma")) big = false;
    }
    if (rk) {
        rankk_gemm(f, st, mode, C, A, ta, B, tb, M, N, K);
        return;
    }
    if ((f.p > 255 || big) && tc_gemm_supported(f, M, N, K)) {
        tc_gemm(f, st, mode, C, A, ta, B, tb, M, N, K);
        return;
    }
    if (mma_gemm_supported(f, M, N, K)) {
        mma_gemm(f, st, mode, C, A, ta, B, tb, M, N, K);
        return;
    }
simt:
    if (!ta && !tb) launch_gemm_simt<false, false>(f, st, mode, C, A, B, M, N, K);
    else if (ta && !tb) launch_gemm_simt<true, false>(f, st, mode, C, A, B, M, N, K);
    else if (!ta && tb) launch_gemm_simt<false, true>(f, st, mode, C, A, B, M, N, K);
    else launch_gemm_simt<true, true>(f, st, mode, C, A, B, M, N, K);
}

// C op= op(A1) op(B1) + op(A2) op(B2) (e.g. SYR2K, kernels.cpp:121-135): one tcgen05
// accumulator over the K-concatenated terms when the tensor-core path applies (C is read
// and written once), else two GEMMs.
void gemm2(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A1, bool ta1, DMat B1, bool tb1, DMat A2,
           bool ta2, DMat B2, bool tb2, int64_t M, int64_t N, int64_t K1, int64_t K2) {
    if (M <= 0 || N <= 0) return;
    const bool big = M >= 128 && N >= 128 && (double)M * N * (K1 + K2) >= 2.7e8;
    if (big && K1 > 0 && K2 > 0 && !getenv("FFB_GEMM_PATH") &&
        tc_gemm2(f, st, mode, C, A1, ta1, B1, tb1, A2, ta2, B2, tb2, M, N, K1, K2))
        return;
    gemm(f, st, mode, C, A1, ta1, B1, tb1, M, N, K1);
    gemm(f, st, mode == GEMM_SET ? GEMM_ADD : mode, C, A2, ta2, B2, tb2, M, N, K2);
}

// ===========================================================================
// Bandwidth-bound data movement.
// ===========================================================================
namespace {

// Row copy d[0..cols) = s[0..cols) by the threads of a grid-x stride loop:
// 16-byte vectors (two in flight) when both rows are 16-byte aligned.
__device__ __forceinline__ void copy_row(uint32_t* d, const uint32_t* s, int64_t cols) {
    const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * blockDim.x;
    if ((((uintptr_t)d | (uintptr_t)s) & 15) == 0) {
        const int64_t c4 = cols >> 2;
        const uint4* s4 = reinterpret_cast<const uint4*>(s);
        uint4* d4 = reinterpret_cast<uint4*>(d);
        int64_t j = start;
        for (; j + step < c4; j += 2 * step) {
            const uint4 a = __ldcg(s4 + j), b = __ldcg(s4 + j + step);
            d4[j] = a;
            d4[j + step] = b;
        }
        for (; j < c4; j += step) d4[j] = __ldcg(s4 + j);
        for (int64_t t = 4 * c4 + start; t < cols; t += step) d[t] = s[t];
        return;
    }
    for (int64_t j = start; j < cols; j += step) d[j] = s[j];
}

// Row kernels loop over rows (grid.y strides them): a few thousand CTAs move the whole
// block instead of one tiny CTA per (row, column slice) -- at 16384 rows the per-CTA
// launch cost, not HBM, bounded the one-row-per-CTA form.
// dst[i][j] = src[idx[i]][c0 + j]: R rows per iteration, so each thread keeps R 16-byte
// loads in flight behind one round of index loads
template <int R>
__device__ __forceinline__ void copy_rows_r(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                                            const int32_t* idx, int64_t c0, int64_t rows, int64_t cols) {
    const int64_t start = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t step = (int64_t)gridDim.x * blockDim.x, gy = gridDim.y;
    const bool vec = ((((uintptr_t)dst | (uintptr_t)(src + c0)) & 15) == 0) && (ldd & 3) == 0 && (lds & 3) == 0;
    for (int64_t i0 = blockIdx.y; i0 < rows; i0 += R * gy) {
        const uint32_t* s[R];
        uint32_t* d[R];
        bool ok[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int64_t i = i0 + u * gy;
            ok[u] = i < rows;
            s[u] = src + (ok[u] ? (int64_t)__ldcg(idx + i) : 0) * lds + c0;
            d[u] = dst + (ok[u] ? i : 0) * ldd;
        }
        if (vec) {
            const int64_t c4 = cols >> 2;
            for (int64_t j = start; j < c4; j += step) {
                uint4 v[R];
#pragma unroll
                for (int u = 0; u < R; ++u)
                    if (ok[u]) v[u] = __ldcg(reinterpret_cast<const uint4*>(s[u]) + j);
#pragma unroll
                for (int u = 0; u < R; ++u)
                    if (ok[u]) reinterpret_cast<uint4*>(d[u])[j] = v[u];
            }
            for (int64_t t = 4 * c4 + start; t < cols; t += step)
#pragma unroll
                for (int u = 0; u < R; ++u)
                    if (ok[u]) d[u][t] = __ldcg(s[u] + t);
        } else {
            for (int64_t j = start; j < cols; j += step)
#pragma unroll
                for (int u = 0; u < R; ++u)
                    if (ok[u]) d[u][j] = __ldcg(s[u] + j);
        }
    }
}

__global__ void k_gather_rows(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                              const int32_t* idx, int64_t rows, int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    copy_row(dst + i * ldd, src + (int64_t)idx[i] * lds, cols);
}
__global__ void __launch_bounds__(256, 4) k_gather_rows_loop(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                                   const int32_t* idx, int64_t rows, int64_t cols) {
    FFB_PDL_ENTRY();
    copy_rows_r<2>(dst, ldd, src, lds, idx, 0, rows, cols);
}

// Two independent row gathers in one launch (blockIdx.z): dst[i][j] = src[idx[i]][c0 + j].
struct RowGather {
    uint32_t* dst;
    int64_t ldd;
    const uint32_t* src;
    int64_t lds;
    const int32_t* idx;
    int64_t c0, rows, cols;
};
__global__ void k_gather_rows2(RowGather g0, RowGather g1) {
    FFB_PDL_ENTRY();
    const RowGather& g = blockIdx.z == 0 ? g0 : g1;
    const int64_t i = blockIdx.y;
    if (i >= g.rows) return;
    copy_row(g.dst + i * g.ldd, g.src + (int64_t)g.idx[i] * g.lds + g.c0, g.cols);
}
__global__ void __launch_bounds__(256, 4) k_gather_rows2_loop(RowGather g0, RowGather g1) {
    FFB_PDL_ENTRY();
    if (blockIdx.z == 0) copy_rows_r<2>(g0.dst, g0.ldd, g0.src, g0.lds, g0.idx, g0.c0, g0.rows, g0.cols);
    else copy_rows_r<2>(g1.dst, g1.ldd, g1.src, g1.lds, g1.idx, g1.c0, g1.rows, g1.cols);
}

// dst[a][b] = src[ridx[a]][idx[b]] with the source row staged in shared memory
// (n words): coalesced 16-byte row reads, coalesced writes, the column permutation
// served from smem.  One CTA per row at a time, rows strided by gridDim.x.
__global__ void __launch_bounds__(512) k_gather_sym_smem(uint32_t* dst, int64_t ldd, const uint32_t* src,
                                                        int64_t lds, const int32_t* ridx, const int32_t* idx,
                                                        int64_t rows, int64_t n) {
    FFB_PDL_ENTRY();
    extern __shared__ __align__(16) uint32_t gs_row[];
    const int64_t n4 = n >> 2;
    for (int64_t a = blockIdx.x; a < rows; a += gridDim.x) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src + (int64_t)__ldcg(ridx + a) * lds);
        for (int64_t j = threadIdx.x; j < n4; j += blockDim.x)
            reinterpret_cast<uint4*>(gs_row)[j] = __ldcg(s4 + j);
        for (int64_t j = 4 * n4 + threadIdx.x; j < n; j += blockDim.x)
            gs_row[j] = __ldcg(src + (int64_t)__ldcg(ridx + a) * lds + j);
        __syncthreads();
        uint32_t* d = dst + a * ldd;
        for (int64_t b = threadIdx.x; b < n; b += blockDim.x) d[b] = gs_row[__ldcg(idx + b)];
        __syncthreads();
    }
}

__global__ void k_gather_sym(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                             const int32_t* ridx, const int32_t* idx, int64_t n) {
    FFB_PDL_ENTRY();
    const int64_t a = blockIdx.y;
    const uint32_t* s = src + (int64_t)ridx[a] * lds;
    uint32_t* d = dst + a * ldd;
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x)
        d[b] = s[idx[b]];
}

__global__ void k_transpose(uint32_t* dst, int64_t ldd, const uint32_t* src, int64_t lds,
                            int64_t rows, int64_t cols) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + k, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[k][threadIdx.x] = src[r * lds + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t c = c0 + k, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][k];
    }
}

// Z[i][j] = Z[j][i] for j < i - halo: restores the strict lower part a band-only
// symmetric update (g_band_halo) left stale.  CTA (x, y): the 32x32 tile (y, x) of the
// lower triangle, read through the transposed tile (x, y) of the upper triangle.
__global__ void k_mirror_lower(uint32_t* Z, int64_t ld, int64_t n, int64_t halo) {
    FFB_PDL_ENTRY();
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    if (c0 >= r0 + 31 - halo) return;  // no entry with j < i - halo in this tile
    __shared__ uint32_t tile[32][33];
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {  // upper tile (c0.., r0..)
        const int64_t r = c0 + k, c = r0 + threadIdx.x;
        if (r < n && c < n) tile[k][threadIdx.x] = __ldcg(Z + r * ld + c);
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t i = r0 + k, j = c0 + threadIdx.x;
        if (i < n && j < n && j < i - halo) Z[i * ld + j] = tile[threadIdx.x][k];
    }
}

__global__ void k_scatter_lg(uint32_t* Lg, int64_t ldl, const int32_t* ids, int64_t col0,
                             int cstride, const uint32_t* src, int64_t lds, int64_t rows,
                             int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    uint32_t* d = Lg + (int64_t)ids[i] * ldl + col0;
    const uint32_t* s = src + i * lds;
    if (cstride == 1) {
        copy_row(d, s, cols);
        return;
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += (int64_t)gridDim.x * blockDim.x)
        d[j * cstride] = s[j];
}

// Interleaved pair scatter: Lg[ids[i]][col0 + 2j] = e[i][j], [col0 + 2j + 1] = o[i][j]
// (the even/odd L columns of the 2x2 pivot pairs, one coalesced 8-byte store each).
__global__ void k_scatter_lg_pair(uint32_t* Lg, int64_t ldl, const int32_t* ids, int64_t col0,
                                  const uint32_t* e, int64_t lde, const uint32_t* o, int64_t ldo,
                                  int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    uint32_t* d = Lg + (int64_t)ids[i] * ldl + col0;
    const uint32_t* se = e + i * lde;
    const uint32_t* so = o + i * ldo;
    const bool vec = ((((uintptr_t)d) & 7) == 0);
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t a = __ldcg(se + j), b = __ldcg(so + j);
        if (vec) reinterpret_cast<uint2*>(d)[j] = make_uint2(a, b);
        else {
            d[2 * j] = a;
            d[2 * j + 1] = b;
        }
    }
}

__global__ void __launch_bounds__(256, 4) k_gather_lg(uint32_t* dst, int64_t ldd, const uint32_t* Lg, int64_t ldl,
                            const int32_t* ids, int64_t col0, int64_t cols, int64_t rows) {
    FFB_PDL_ENTRY();
    copy_rows_r<2>(dst, ldd, Lg, ldl, ids, col0, rows, cols);
}

// G[j][k] = (D^-1 X)[k][j], X is r x ncols.  Tile: 32 k x 32 j, with one
// extra row on each side for the 2x2 partners.
__global__ void k_inverse_apply_T(Fp f, uint32_t* G, int64_t ldg, const uint32_t* X,
                                  int64_t ldx, int64_t r, int64_t ncols, DDiag D, int64_t coff,
                                  uint32_t* Lg, int64_t ldl, const int32_t* ids) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t tile[34][33];
    const int64_t k0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
    for (int kk = threadIdx.y; kk < 34; kk += blockDim.y) {
        const int64_t k = k0 - 1 + kk, j = j0 + threadIdx.x;
        tile[kk][threadIdx.x] = (k >= 0 && k < r && j < ncols) ? X[k * ldx + j] : 0;
    }
    __syncthreads();
    for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
        const int64_t j = j0 + jj, k = k0 + threadIdx.x;
        if (j >= ncols || k >= r) continue;
        const int kk = threadIdx.x + 1;
        const int32_t kind = D.kind[coff + k];
        const uint32_t inv = D.inv[coff + k];
        uint32_t v;
        if (kind == D_SCALAR) {
            v = fmul(f, inv, tile[kk][jj]);
        } else if (kind == D_ANTIDIAG_HEAD) {
            v = fmul(f, inv, tile[kk + 1][jj]);
        } else if (kind == D_ANTIDIAG_TAIL || kind == D_ANTITRI_TAIL) {
            v = fmul(f, inv, tile[kk - 1][jj]);
        } else {  // AntiTri head: -d c^-2 x_t + c^-1 x_{t+1}   (blockdiag.hpp:127-134)
            const uint32_t top = fneg(f, fmul(f, D.val2[coff + k], fmul(f, inv, inv)));
            v = fadd(f, fmul(f, top, tile[kk][jj]), fmul(f, inv, tile[kk + 1][jj]));
        }
        G[j * ldg + k] = v;
        if (Lg) Lg[(int64_t)ids[j] * ldl + coff + k] = v;  // rows of N1 (sytrf.cpp:319-322)
    }
}

__global__ void k_scale_T(Fp f, uint32_t* G, int64_t ldg, const uint32_t* X, int64_t ldx,
                          int64_t r, int64_t ncols, const uint32_t* dinv) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t tile[32][33];
    const int64_t k0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
    for (int kk = threadIdx.y; kk < 32; kk += blockDim.y) {
        const int64_t k = k0 + kk, j = j0 + threadIdx.x;
        tile[kk][threadIdx.x] = (k < r && j < ncols) ? fmul(f, dinv[k], X[k * ldx + j]) : 0;
    }
    __syncthreads();
    for (int jj = threadIdx.y; jj < 32; jj += blockDim.y) {
        const int64_t j = j0 + jj, k = k0 + threadIdx.x;
        if (j < ncols && k < r) G[j * ldg + k] = tile[threadIdx.x][jj];
    }
}

__global__ void k_invert_vec(Fp f, uint32_t* out, const uint32_t* v, int64_t n) {
    FFB_PDL_ENTRY();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = finv(f, v[i]);
}

// *flag = value if any entry of m is nonzero.  Grid-stride over rows, a warp per
// row (16-byte loads, 4 in flight per lane when aligned); a warp that finds a
// nonzero publishes and exits, and every warp polls the flag (read at the start of
// a row, tested after its loads) so a nonzero matrix is abandoned early.
__global__ void __launch_bounds__(256) k_any_nonzero(const uint32_t* m, int64_t ld, int64_t rows, int64_t cols,
                                                     int32_t* flag, int32_t value) {
    FFB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const bool vec = ((((uintptr_t)m) & 15) == 0) && ((ld & 3) == 0) && ((cols & 3) == 0);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < rows; i += nwarps) {
        const int32_t seen = *(volatile const int32_t*)flag;
        const uint32_t* row = m + i * ld;
        bool nz = false;
        if (vec) {
            const uint4* r4 = reinterpret_cast<const uint4*>(row);
            const int64_t c4 = cols >> 2;
            int64_t j = lane;
            for (; j + 96 < c4; j += 128) {
                const uint4 a = __ldcg(r4 + j), b = __ldcg(r4 + j + 32), c = __ldcg(r4 + j + 64), d = __ldcg(r4 + j + 96);
                nz |= (a.x | a.y | a.z | a.w | b.x | b.y | b.z | b.w | c.x | c.y | c.z | c.w | d.x | d.y | d.z | d.w) != 0;
            }
            for (; j < c4; j += 32) {
                const uint4 a = __ldcg(r4 + j);
                nz |= (a.x | a.y | a.z | a.w) != 0;
            }
        } else {
            for (int64_t j = lane; j < cols; j += 32) nz |= __ldcg(row + j) != 0;
        }
        if (__any_sync(0xffffffffu, nz)) {
            if (lane == 0) *flag = value;
            return;
        }
        if (__shfl_sync(0xffffffffu, seen, 0) == value) return;  // another warp found one
    }
}

// Symmetry check: CTA (x, y) walks the 32x32 tiles of row band y left of the diagonal
// with stride gridDim.x (no CTAs for the upper triangle), the next tile's loads issued
// before the current tile's comparisons.  T is the element type: uint32 residues of a
// device matrix (p = 0: already reduced), or the caller's raw host element type staged
// in HBM (u8/u16/u32/u64, compared as residues mod p; the reduction only runs for a pair
// whose raw values differ).
template <typename T>
__global__ void k_any_asym(const T* a, int64_t ld, int64_t n, uint64_t p, int32_t* flag) {
    FFB_PDL_ENTRY();
    __shared__ T tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32;
    int bad = 0;
    auto valid = [&](int64_t t) { return t * 32 <= r0 + 31 && t * 32 < n; };
    T up[4], lo[4];
    auto load = [&](int64_t t) {
        const int64_t c0 = t * 32;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = threadIdx.y + 8 * u;
            const int64_t r = c0 + k, c = r0 + threadIdx.x;  // transposed tile
            up[u] = (r < n && c < n) ? __ldcg(a + r * ld + c) : T(0);
            const int64_t rr = r0 + k, cc = c0 + threadIdx.x;
            lo[u] = (rr < n && cc < n) ? __ldcg(a + rr * ld + cc) : T(0);
        }
    };
    int64_t t = blockIdx.x;
    if (valid(t)) load(t);
    while (valid(t)) {  // uniform
        const int64_t c0 = t * 32;
        __syncthreads();  // previous tile's comparisons done
#pragma unroll
        for (int u = 0; u < 4; ++u) tile[threadIdx.y + 8 * u][threadIdx.x] = up[u];
        __syncthreads();
        T cur[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) cur[u] = lo[u];
        const int64_t tn = t + gridDim.x;
        if (valid(tn)) load(tn);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = threadIdx.y + 8 * u;
            const int64_t r = r0 + k, c = c0 + threadIdx.x;
            const T x = cur[u], y = tile[threadIdx.x][k];
            if (r < n && c < n && x != y)
                bad |= p == 0 || (uint64_t)x % p != (uint64_t)y % p;
        }
        t = tn;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0 && threadIdx.y == 0) atomicOr(flag, 1);
}

__global__ void k_trssyr2k_mid(Fp f, uint32_t* C, int64_t ld, int64_t n, int32_t* flag) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t* c = C + i * ld + j;
        if (j < i) {
            *c = 0;
        } else if (j == i) {
            if (f.char2) {
                if (*c) atomicOr(flag, 1);
                *c = 0;
            } else {
                *c = fhalve(f, *c);
            }
        }
    }
}

__global__ void k_write_pair_diag(DDiag D, int64_t coff, const uint32_t* d, const uint32_t* dinv,
                                  const uint32_t* delta, int64_t r) {
    FFB_PDL_ENTRY();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r) return;
    const uint32_t dl = delta ? delta[i] : 0;
    const int64_t t = coff + 2 * i;
    D.kind[t] = dl ? D_ANTITRI_HEAD : D_ANTIDIAG_HEAD;
    D.kind[t + 1] = dl ? D_ANTITRI_TAIL : D_ANTIDIAG_TAIL;
    D.val[t] = D.val[t + 1] = d[i];
    D.val2[t] = D.val2[t + 1] = dl;
    D.inv[t] = D.inv[t + 1] = dinv[i];
}

__global__ void k_char2_delta(Fp f, const uint32_t* C1, int64_t ldc, const uint32_t* U1,
                              int64_t ldu, int64_t r, uint32_t* delta) {
    FFB_PDL_ENTRY();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int64_t i = 0; i < r; ++i) {
        uint32_t acc = C1[i * ldc + i];
        for (int64_t j = 0; j < i; ++j) {
            const uint32_t u = U1[j * ldu + i];
            acc = fsub(f, acc, fmul(f, fmul(f, delta[j], u), u));
        }
        delta[i] = acc;
    }
}

__global__ void k_scale_rows(Fp f, uint32_t* H, int64_t ldh, const uint32_t* S, int64_t lds,
                             int64_t cols, const uint32_t* v) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    const uint32_t s = v[i];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += (int64_t)gridDim.x * blockDim.x)
        H[i * ldh + j] = fmul(f, s, S[i * lds + j]);
}

__global__ void k_add_scaled_rows_upper(Fp f, uint32_t* X, int64_t ldx, const uint32_t* U,
                                        int64_t ldu, int64_t cols, const uint32_t* v) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    const uint32_t s = v[i];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += (int64_t)gridDim.x * blockDim.x)
        if (j >= i) X[i * ldx + j] = fadd(f, X[i * ldx + j], fmul(f, s, U[i * ldu + j]));
}

__global__ void k_zero(uint32_t* m, int64_t ld, int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += (int64_t)gridDim.x * blockDim.x)
        m[i * ld + j] = 0;
}

template <typename T>
__global__ void k_convert_in(Fp f, uint32_t* dst, int64_t ldd, const T* src, int64_t rows,
                             int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = (uint64_t)src[i * cols + j];
        dst[i * ldd + j] = red64(f, v);
    }
}

template <typename T>
__global__ void k_convert_out(T* dst, const uint32_t* src, int64_t lds, int64_t rows,
                              int64_t cols) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < cols;
         j += (int64_t)gridDim.x * blockDim.x)
        dst[i * cols + j] = (T)src[i * lds + j];
}

// for the row-looping kernels: about 16 CTAs per SM in total
inline dim3 rowgrid_loop(int64_t rows, int64_t cols, int threads = 256, int per_thread = 1) {
    int64_t gx = cdiv(cdiv(cols, per_thread), threads);
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    const int64_t gy = std::min<int64_t>(std::max<int64_t>(rows, 1), std::max<int64_t>(1, 16 * 148 / gx));
    return dim3((unsigned)gx, (unsigned)gy);
}
inline dim3 rowgrid(int64_t rows, int64_t cols, int threads = 256, int per_thread = 1) {
    int64_t gx = cdiv(cdiv(cols, per_thread), threads);
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    return dim3((unsigned)gx, (unsigned)rows);
}

}  // namespace

// Row-indexed launches put rows on grid.y (max 65535); split bigger jobs.
#define FFB_ROWCHUNK 65535

void gather_rows(cudaStream_t st, DMat dst, DMat src, const int32_t* idx) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (dst.rows <= 0 || dst.cols <= 0) return;
    for (int64_t r0 = 0; r0 < dst.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, dst.rows - r0);
        // big gathers: row-looping CTAs (fewer, fatter); small ones: a CTA per row slice
        const bool big = nr * dst.cols >= ((int64_t)1 << 22);
        launch_k(big ? k_gather_rows_loop : k_gather_rows, big ? rowgrid_loop(nr, dst.cols, 256, 4)
                                                                : rowgrid(nr, dst.cols, 256, 4), 256, 0, st, dst.ptr + r0 * dst.ld, dst.ld, src.ptr,
                                                             src.ld, idx + r0, nr, dst.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void gather_sym(cudaStream_t st, DMat dst, DMat src, const int32_t* idx) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (dst.rows <= 0) return;
    const size_t row_bytes = (size_t)dst.cols * 4;
    if (dst.cols >= 1024 && row_bytes <= 200 * 1024 && (src.ld & 3) == 0 && (((uintptr_t)src.ptr) & 15) == 0) {
        static DeviceOnce attr;
        if (!attr.done()) {
            FFB_CUDA(cudaFuncSetAttribute(k_gather_sym_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            attr.mark();
        }
        const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(4, (int64_t)(227 * 1024) / (int64_t)(row_bytes + 1024)));
        const int64_t grid = std::min<int64_t>(dst.rows, 148 * per_sm);
        launch_k(k_gather_sym_smem, (unsigned)grid, 512, row_bytes, st, dst.ptr, dst.ld, src.ptr, src.ld, idx, idx,
                 dst.rows, dst.cols);
        count_launch();
        FFB_CHECK_LAUNCH();
        return;
    }
    for (int64_t r0 = 0; r0 < dst.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, dst.rows - r0);
        launch_k(k_gather_sym, rowgrid(nr, dst.cols), 256, 0, st, dst.ptr + r0 * dst.ld, dst.ld, src.ptr,
                                                            src.ld, idx + r0, idx, dst.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void transpose(cudaStream_t st, DMat dst, DMat src) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (src.rows <= 0 || src.cols <= 0) return;
    dim3 grid((unsigned)cdiv(src.cols, 32), (unsigned)cdiv(src.rows, 32));
    launch_k(k_transpose, grid, dim3(32, 8), 0, st, dst.ptr, dst.ld, src.ptr, src.ld, src.rows, src.cols);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void mirror_lower(cudaStream_t st, DMat Z, int halo) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (Z.rows <= halo + 1) return;
    const int64_t nt = cdiv(Z.rows, 32);  // <= 65535 tile rows for n < 2^21
    launch_k(k_mirror_lower, dim3((unsigned)nt, (unsigned)nt), dim3(32, 8), 0, st, Z.ptr, Z.ld, Z.rows,
             (int64_t)halo);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void scatter_lg(cudaStream_t st, DMat Lg, const int32_t* ids, int64_t col0, int cstride, DMat src) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (src.rows <= 0 || src.cols <= 0) return;
    for (int64_t r0 = 0; r0 < src.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, src.rows - r0);
        launch_k(k_scatter_lg, rowgrid(nr, src.cols), 256, 0, st, Lg.ptr, Lg.ld, ids + r0, col0, cstride,
                                                            src.ptr + r0 * src.ld, src.ld, nr,
                                                            src.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

// The three writes that end zero_leading_pairs in one launch (rows of [L1; M1] into the even
// columns, rows of [G1; G2] / [U1^T; V1^T] into the column pairs, the 2x2 blocks of D): block
// row y < my scatters a Y row, y < my + nz a Z row, the last block row writes D.
__global__ void k_zlp_scatter(uint32_t* Lg, int64_t ldl, int64_t col0, const int32_t* idy, int64_t my,
                              const uint32_t* L, int64_t ldL, const int32_t* idz, int64_t nz, const uint32_t* e,
                              int64_t lde, const uint32_t* o, int64_t ldo, int64_t r, DDiag D, const uint32_t* dv,
                              const uint32_t* dinv, const uint32_t* delta) {
    FFB_PDL_ENTRY();
    const int64_t y = blockIdx.y, t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                  step = (int64_t)gridDim.x * blockDim.x;
    if (y < my) {
        uint32_t* d = Lg + (int64_t)__ldcg(idy + y) * ldl + col0;
        const uint32_t* s = L + y * ldL;
        for (int64_t j = t0; j < r; j += step) d[2 * j] = __ldcg(s + j);
    } else if (y < my + nz) {
        const int64_t i = y - my;
        uint32_t* d = Lg + (int64_t)__ldcg(idz + i) * ldl + col0;
        const uint32_t* se = e + i * lde;
        const uint32_t* so = o + i * ldo;
        const bool vec = ((((uintptr_t)d) & 7) == 0);
        for (int64_t j = t0; j < r; j += step) {
            const uint32_t a = __ldcg(se + j), b = __ldcg(so + j);
            if (vec) reinterpret_cast<uint2*>(d)[j] = make_uint2(a, b);
            else {
                d[2 * j] = a;
                d[2 * j + 1] = b;
            }
        }
    } else {
        for (int64_t i = t0; i < r; i += step) {
            const uint32_t dl = delta ? __ldcg(delta + i) : 0;
            const int64_t t = col0 + 2 * i;
            D.kind[t] = dl ? D_ANTITRI_HEAD : D_ANTIDIAG_HEAD;
            D.kind[t + 1] = dl ? D_ANTITRI_TAIL : D_ANTIDIAG_TAIL;
            D.val[t] = D.val[t + 1] = __ldcg(dv + i);
            D.val2[t] = D.val2[t + 1] = dl;
            D.inv[t] = D.inv[t + 1] = __ldcg(dinv + i);
        }
    }
}
bool zlp_scatter(cudaStream_t st, DMat Lg, int64_t col0, const int32_t* idy, DMat L, const int32_t* idz, DMat even,
                 DMat odd, DDiag D, const uint32_t* d, const uint32_t* dinv, const uint32_t* delta, int64_t r) {
    if (r <= 0 || L.rows + even.rows + 1 > 65535) return false;
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    launch_k(k_zlp_scatter, rowgrid(L.rows + even.rows + 1, r), 256, 0, st, Lg.ptr, Lg.ld, col0, idy, L.rows, L.ptr,
             L.ld, idz, even.rows, even.ptr, even.ld, odd.ptr, odd.ld, r, D, d, dinv, delta);
    count_launch();
    FFB_CHECK_LAUNCH();
    return true;
}
void scatter_lg_pair(cudaStream_t st, DMat Lg, const int32_t* ids, int64_t col0, DMat even, DMat odd) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (even.rows <= 0 || even.cols <= 0) return;
    for (int64_t r0 = 0; r0 < even.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, even.rows - r0);
        launch_k(k_scatter_lg_pair, rowgrid(nr, even.cols), 256, 0, st, Lg.ptr, Lg.ld, ids + r0, col0,
                 even.ptr + r0 * even.ld, even.ld, odd.ptr + r0 * odd.ld, odd.ld, even.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void gather_rows2(cudaStream_t st, DMat d0, DMat s0, const int32_t* i0, int64_t c0, DMat d1, DMat s1,
                  const int32_t* i1, int64_t c1) {
    const int64_t rows = std::max(d0.rows, d1.rows), cols = std::max(d0.cols, d1.cols);
    if (rows <= 0 || cols <= 0) return;
    if (rows > FFB_ROWCHUNK) {  // rare: fall back to two launches
        gather_rows(st, d0, s0.sub(0, c0, s0.rows, d0.cols), i0);
        gather_rows(st, d1, s1.sub(0, c1, s1.rows, d1.cols), i1);
        return;
    }
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    RowGather g0{d0.ptr, d0.ld, s0.ptr, s0.ld, i0, c0, d0.cols > 0 ? d0.rows : 0, d0.cols};
    RowGather g1{d1.ptr, d1.ld, s1.ptr, s1.ld, i1, c1, d1.cols > 0 ? d1.rows : 0, d1.cols};
    const bool big = rows * cols >= ((int64_t)1 << 22);
    dim3 g = big ? rowgrid_loop(rows, cols, 256, 4) : rowgrid(rows, cols, 256, 4);
    g.z = 2;
    launch_k(big ? k_gather_rows2_loop : k_gather_rows2, g, 256, 0, st, g0, g1);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void gather_lg(cudaStream_t st, DMat dst, DMat Lg, const int32_t* ids, int64_t col0) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (dst.rows <= 0 || dst.cols <= 0) return;
    for (int64_t r0 = 0; r0 < dst.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, dst.rows - r0);
        // 16 words (four 16-byte vectors) per thread: a few CTAs per row, loads in flight
        launch_k(k_gather_lg, rowgrid_loop(nr, dst.cols, 256, 4), 256, 0, st, dst.ptr + r0 * dst.ld, dst.ld,
                 Lg.ptr, Lg.ld, ids + r0, col0, dst.cols, nr);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void inverse_apply_T(const Fp& f, cudaStream_t st, DMat G, DMat X, DDiag D, int64_t coff,
                     DMat Lg, const int32_t* ids) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (X.rows <= 0 || X.cols <= 0) return;
    dim3 grid((unsigned)cdiv(X.cols, 32), (unsigned)cdiv(X.rows, 32));
    launch_k(k_inverse_apply_T, grid, dim3(32, 8), 0, st, f, G.ptr, G.ld, X.ptr, X.ld, X.rows, X.cols, D,
                                                    coff, ids ? Lg.ptr : nullptr, Lg.ld, ids);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void scale_T(const Fp& f, cudaStream_t st, DMat G, DMat X, const uint32_t* dinv) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (X.rows <= 0 || X.cols <= 0) return;
    dim3 grid((unsigned)cdiv(X.cols, 32), (unsigned)cdiv(X.rows, 32));
    launch_k(k_scale_T, grid, dim3(32, 8), 0, st, f, G.ptr, G.ld, X.ptr, X.ld, X.rows, X.cols, dinv);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void invert_vec(const Fp& f, cudaStream_t st, uint32_t* out, const uint32_t* v, int64_t n) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (n <= 0) return;
    launch_k(k_invert_vec, (unsigned)cdiv(n, 256), 256, 0, st, f, out, v, n);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void any_nonzero(cudaStream_t st, DMat m, int32_t* flag, int32_t value) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (m.rows <= 0 || m.cols <= 0) return;
    // a warp per row, at most 8 CTAs of 8 warps per SM
    const unsigned g = (unsigned)std::min<int64_t>(cdiv(m.rows, 8), 148 * 8);
    launch_k(k_any_nonzero, g, 256, 0, st, m.ptr, m.ld, m.rows, m.cols, flag, value);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void any_asymmetric(cudaStream_t st, DMat a, int32_t* flag) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (a.rows <= 1) return;
    dim3 grid((unsigned)std::min<int64_t>(8, cdiv(a.rows, 32)), (unsigned)cdiv(a.rows, 32));
    launch_k(k_any_asym<uint32_t>, grid, dim3(32, 8), 0, st, (const uint32_t*)a.ptr, a.ld, a.rows,
             (uint64_t)0, flag);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void any_asymmetric_raw(cudaStream_t st, const void* a, int64_t n, int eb, uint64_t p, int32_t* flag) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (n <= 1) return;
    dim3 grid((unsigned)std::min<int64_t>(8, cdiv(n, 32)), (unsigned)cdiv(n, 32));
    if (eb == 8) launch_k(k_any_asym<uint64_t>, grid, dim3(32, 8), 0, st, (const uint64_t*)a, n, n, p, flag);
    else if (eb == 4) launch_k(k_any_asym<uint32_t>, grid, dim3(32, 8), 0, st, (const uint32_t*)a, n, n, p, flag);
    else if (eb == 2) launch_k(k_any_asym<uint16_t>, grid, dim3(32, 8), 0, st, (const uint16_t*)a, n, n, p, flag);
    else launch_k(k_any_asym<uint8_t>, grid, dim3(32, 8), 0, st, (const uint8_t*)a, n, n, p, flag);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void trssyr2k_mid(const Fp& f, cudaStream_t st, DMat Ct, int32_t* flag) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (Ct.rows <= 0) return;
    launch_k(k_trssyr2k_mid, rowgrid(Ct.rows, Ct.cols), 256, 0, st, f, Ct.ptr, Ct.ld, Ct.rows, flag);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void write_pair_diag(const Fp& f, cudaStream_t st, DDiag D, int64_t coff, const uint32_t* d,
                     const uint32_t* dinv, const uint32_t* delta, int64_t r) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    (void)f;
    if (r <= 0) return;
    launch_k(k_write_pair_diag, (unsigned)cdiv(r, 256), 256, 0, st, D, coff, d, dinv, delta, r);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void char2_delta(const Fp& f, cudaStream_t st, DMat C1, DMat U1, uint32_t* delta) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (C1.rows <= 0) return;
    launch_k(k_char2_delta, 1, 32, 0, st, f, C1.ptr, C1.ld, U1.ptr, U1.ld, C1.rows, delta);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void scale_rows(const Fp& f, cudaStream_t st, DMat H, DMat S, const uint32_t* v) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (S.rows <= 0 || S.cols <= 0) return;
    launch_k(k_scale_rows, rowgrid(S.rows, S.cols), 256, 0, st, f, H.ptr, H.ld, S.ptr, S.ld, S.cols, v);
    count_launch();
    FFB_CHECK_LAUNCH();
}

void add_scaled_rows_upper(const Fp& f, cudaStream_t st, DMat X, DMat U, const uint32_t* v) {
    ProfScope ps_(K_OTHER, st, 0.0, 0.0);
    if (X.rows <= 0) return;
    launch_k(k_add_scaled_rows_upper, rowgrid(X.rows, X.cols), 256, 0, st, f, X.ptr, X.ld, U.ptr, U.ld,
                                                                     X.cols, v);
    count_launch();
    FFB_CHECK_LAUNCH();
}

// Word fill as a kernel (not a copy-engine memset): stays in the programmatic-launch
// chain and is not queued behind bulk host transfers on other streams.
__global__ void k_fill(uint32_t* p, int64_t n, uint32_t v) {
    FFB_PDL_ENTRY();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t mis = (int64_t)((16 - ((uintptr_t)p & 15)) & 15) / 4;
    const int64_t head = mis < n ? mis : n;
    if (i0 < head) p[i0] = v;
    const int64_t n4 = (n - head) >> 2;
    uint4* q = reinterpret_cast<uint4*>(p + head);
    for (int64_t i = i0; i < n4; i += stride) q[i] = make_uint4(v, v, v, v);
    for (int64_t i = head + 4 * n4 + i0; i < n; i += stride) p[i] = v;
}

void fill_words(cudaStream_t st, uint32_t* p, int64_t n, uint32_t v) {
    if (n <= 0) return;
    const int64_t blocks = std::min<int64_t>(148 * 8, std::max<int64_t>(1, cdiv(n, 4 * 256)));
    launch_k(k_fill, (unsigned)blocks, 256, 0, st, p, n, v);
    count_launch();
}

void zero_mat(cudaStream_t st, DMat m) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    if (m.rows <= 0 || m.cols <= 0) return;
    if (m.ld == m.cols) {
        fill_words(st, m.ptr, m.rows * m.cols, 0u);
        return;
    }
    for (int64_t r0 = 0; r0 < m.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, m.rows - r0);
        launch_k(k_zero, rowgrid(nr, m.cols), 256, 0, st, m.ptr + r0 * m.ld, m.ld, m.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void convert_in(const Fp& f, cudaStream_t st, DMat dst, const void* src, int eb) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    for (int64_t r0 = 0; r0 < dst.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, dst.rows - r0);
        dim3 g = rowgrid(nr, dst.cols);
        uint32_t* d = dst.ptr + r0 * dst.ld;
        const size_t off = (size_t)r0 * dst.cols;
        if (eb == 8) launch_k(k_convert_in<uint64_t>, g, 256, 0, st, f, d, dst.ld, (const uint64_t*)src + off, nr, dst.cols);
        else if (eb == 4) launch_k(k_convert_in<uint32_t>, g, 256, 0, st, f, d, dst.ld, (const uint32_t*)src + off, nr, dst.cols);
        else if (eb == 2) launch_k(k_convert_in<uint16_t>, g, 256, 0, st, f, d, dst.ld, (const uint16_t*)src + off, nr, dst.cols);
        else launch_k(k_convert_in<uint8_t>, g, 256, 0, st, f, d, dst.ld, (const uint8_t*)src + off, nr, dst.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void convert_out(cudaStream_t st, void* dst, int eb, DMat src) {
    ProfScope ps_(K_MOVE, st, 0.0, 0.0);
    for (int64_t r0 = 0; r0 < src.rows; r0 += FFB_ROWCHUNK) {
        const int64_t nr = std::min<int64_t>(FFB_ROWCHUNK, src.rows - r0);
        dim3 g = rowgrid(nr, src.cols);
        const uint32_t* s = src.ptr + r0 * src.ld;
        const size_t off = (size_t)r0 * src.cols;
        if (eb == 8) launch_k(k_convert_out<uint64_t>, g, 256, 0, st, (uint64_t*)dst + off, s, src.ld, nr, src.cols);
        else if (eb == 4) launch_k(k_convert_out<uint32_t>, g, 256, 0, st, (uint32_t*)dst + off, s, src.ld, nr, src.cols);
        else if (eb == 2) launch_k(k_convert_out<uint16_t>, g, 256, 0, st, (uint16_t*)dst + off, s, src.ld, nr, src.cols);
        else launch_k(k_convert_out<uint8_t>, g, 256, 0, st, (uint8_t*)dst + off, s, src.ld, nr, src.cols);
        count_launch();
    }
    FFB_CHECK_LAUNCH();
}

void gather_lower_out(cudaStream_t st, DMat out, DMat Lg, const int32_t* perm) {
    gather_lg(st, out, Lg, perm, 0);
}

// ===========================================================================
// Crout leaf, Alg. 4 (sytrf.cpp:35-139), executed right-looking.
//
// The reference recomputes each residual column from the stored multipliers
// (Crout); here the Schur complement S of the active rows is kept updated
// instead, which yields the same field values.  Rows are visited in index
// order (the rotations of `order` never reorder the unprocessed rows,
// sytrf.cpp:93,128-129); the first nonzero of the residual column among the
// active rows selects a 1x1 (j == front) or 2x2 antidiagonal pivot.
// ===========================================================================
namespace {

constexpr int LEAF_THREADS = 256;
constexpr int LEAF_SMEM_MAX_S = 200;

struct LeafState {  // laid out after S in (shared or global) scratch
    int32_t* status;  // 0 active, 1 pivot, 2 pivotless
    uint32_t* l1;
    uint32_t* l2;
    uint32_t* u1;
    uint32_t* u2;
};

__global__ void __launch_bounds__(LEAF_THREADS)
    k_leaf_crout(Fp f, const uint32_t* A, int64_t lda, int s, uint32_t* gscratch,
                 int use_smem, const int32_t* rows, uint32_t* Lg, int64_t ldL,
                 int64_t coff, DDiag D, int32_t* out) {
    FFB_PDL_ENTRY();
    extern __shared__ uint32_t smem[];
    uint32_t* base = use_smem ? smem : gscratch;
    uint32_t* S = base;
    LeafState st;
    st.status = (int32_t*)(base + (size_t)s * s);
    st.l1 = (uint32_t*)(st.status + s);
    st.l2 = st.l1 + s;
    st.u1 = st.l2 + s;
    st.u2 = st.u1 + s;
    __shared__ int jmin;
    __shared__ uint32_t sx, sxi, syeff, syd;
    const int tid = threadIdx.x;

    for (int e = tid; e < s * s; e += LEAF_THREADS) S[e] = A[(int64_t)(e / s) * lda + (e % s)];
    for (int i = tid; i < s; i += LEAF_THREADS) st.status[i] = 0;
    __syncthreads();

    int r = 0;
    int npl = 0;  // pivotless rows found so far (their order is ascending)
    for (int p1 = 0; p1 < s; ++p1) {
        if (st.status[p1] != 0) continue;  // consumed as a 2x2 partner (uniform)
        if (tid == 0) jmin = s;
        __syncthreads();
        for (int i = p1 + tid; i < s; i += LEAF_THREADS)
            if (st.status[i] == 0 && S[(size_t)i * s + p1] != 0) atomicMin(&jmin, i);
        __syncthreads();
        const int j = jmin;
        if (j == s) {  // zero residual column: pivotless (sytrf.cpp:82-85)
            if (tid == 0) {
                st.status[p1] = 2;
                out[1 + (s - 1 - npl)] = p1;  // temporarily stored from the back
            }
            ++npl;
            __syncthreads();
            continue;
        }
        if (j == p1) {  // 1x1 pivot (sytrf.cpp:87-97)
            if (tid == 0) {
                const uint32_t x = S[(size_t)p1 * s + p1];
                const uint32_t xi = finv(f, x);
                sx = x;
                sxi = xi;
                D.kind[coff + r] = D_SCALAR;
                D.val[coff + r] = x;
                D.val2[coff + r] = 0;
                D.inv[coff + r] = xi;
                Lg[(int64_t)rows[p1] * ldL + coff + r] = 1 % f.p;
                st.status[p1] = 1;
                out[1 + r] = p1;
            }
            __syncthreads();
            const uint32_t xi = sxi;
            for (int i = p1 + 1 + tid; i < s; i += LEAF_THREADS) {
                if (st.status[i] != 0) continue;
                const uint32_t l = fmul(f, S[(size_t)i * s + p1], xi);
                st.l1[i] = l;
                Lg[(int64_t)rows[i] * ldL + coff + r] = l;
            }
            __syncthreads();
            const int w = s - p1 - 1;
            for (int e = tid; e < w * w; e += LEAF_THREADS) {
                const int i = p1 + 1 + e / w, k = p1 + 1 + e % w;
                if (st.status[i] != 0 || st.status[k] != 0) continue;
                uint32_t* sik = &S[(size_t)i * s + k];
                *sik = fsub(f, *sik, fmul(f, S[(size_t)i * s + p1], st.l1[k]));
            }
            r += 1;
            __syncthreads();
            continue;
        }
        // 2x2 antidiagonal pivot pairing p1 with p2 = j (sytrf.cpp:99-131)
        const int p2 = j;
        if (tid == 0) {
            const uint32_t x = S[(size_t)p2 * s + p1];
            const uint32_t xi = finv(f, x);
            const uint32_t y = S[(size_t)p2 * s + p2];
            const uint32_t y_eff = f.char2 ? y : fhalve(f, y);
            const uint32_t yd = f.char2 ? y : 0;  // AntiTri d (char 2 only)
            sx = x;
            sxi = xi;
            syeff = y_eff;
            syd = yd;
            const int32_t hk = yd ? D_ANTITRI_HEAD : D_ANTIDIAG_HEAD;
            D.kind[coff + r] = hk;
            D.kind[coff + r + 1] = hk + 1;
            D.val[coff + r] = D.val[coff + r + 1] = x;
            D.val2[coff + r] = D.val2[coff + r + 1] = yd;
            D.inv[coff + r] = D.inv[coff + r + 1] = xi;
            Lg[(int64_t)rows[p1] * ldL + coff + r] = 1 % f.p;
            Lg[(int64_t)rows[p2] * ldL + coff + r + 1] = 1 % f.p;
            Lg[(int64_t)rows[p2] * ldL + coff + r] = f.char2 ? 0 : fmul(f, xi, y_eff);
            st.status[p1] = 1;
            st.status[p2] = 1;
            out[1 + r] = p1;
            out[2 + r] = p2;
        }
        __syncthreads();
        {
            const uint32_t x = sx, xi = sxi, y_eff = syeff;
            for (int i = p1 + 1 + tid; i < s; i += LEAF_THREADS) {
                if (st.status[i] != 0) continue;
                const uint32_t l2 = fmul(f, xi, S[(size_t)i * s + p1]);
                const uint32_t l1 = fmul(f, xi, fsub(f, S[(size_t)i * s + p2], fmul(f, y_eff, l2)));
                st.l1[i] = l1;
                st.l2[i] = l2;
                st.u1[i] = fmul(f, x, l1);
                st.u2[i] = fmul(f, x, l2);
                Lg[(int64_t)rows[i] * ldL + coff + r] = l1;
                Lg[(int64_t)rows[i] * ldL + coff + r + 1] = l2;
            }
        }
        __syncthreads();
        {
            const uint32_t yd = syd;
            const int w = s - p1 - 1;
            for (int e = tid; e < w * w; e += LEAF_THREADS) {
                const int i = p1 + 1 + e / w, k = p1 + 1 + e % w;
                if (st.status[i] != 0 || st.status[k] != 0) continue;
                uint64_t t = (uint64_t)st.u1[i] * st.l2[k] + (uint64_t)st.u2[i] * st.l1[k];
                uint32_t v = red64(f, t);
                if (yd) v = fadd(f, v, fmul(f, fmul(f, yd, st.l2[i]), st.l2[k]));
                uint32_t* sik = &S[(size_t)i * s + k];
                *sik = fsub(f, *sik, v);
            }
        }
        r += 2;
        __syncthreads();
    }
    // Pivotless rows were stored from the back in ascending order of discovery;
    // reverse them into positions [r, s).
    __syncthreads();
    if (tid == 0) {
        out[0] = r;
        for (int a = 0, b = npl - 1; a < b; ++a, --b) {
            const int32_t t = out[1 + r + a];
            out[1 + r + a] = out[1 + r + b];
            out[1 + r + b] = t;
        }
    }
}

}  // namespace

size_t leaf_scratch_words(int64_t s) { return (size_t)s * s + 5 * (size_t)s + 8; }

bool leaf_crout(const Fp& f, cudaStream_t st, DMat A, const int32_t* rows, DMat Lg, int64_t coff,
                DDiag D, int32_t* out, uint32_t* scratch, const MboxPost& mp) {
    const int s = (int)A.rows;
    static const bool generic_only = getenv("FFB_GENERIC_LEAF") != nullptr;  // test hook
    if (!generic_only && leaf64_supported(s)) {
        leaf64(f, st, A, rows, Lg, coff, D, out, mp);
        return mp.dst != nullptr;
    }
    const bool smem = s <= LEAF_SMEM_MAX_S;
    size_t bytes = smem ? leaf_scratch_words(s) * sizeof(uint32_t) : 0;
    if (smem && bytes > 48 * 1024) {
        FFB_CUDA(cudaFuncSetAttribute(k_leaf_crout, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)bytes));
    }
    ProfScope ps(K_LEAF, st, 2.0 * s * s * s / 3.0, 4.0 * s * s);
    launch_k(k_leaf_crout, 1, LEAF_THREADS, bytes, st, f, A.ptr, A.ld, s, scratch, smem ? 1 : 0, rows,
                                                 Lg.ptr, Lg.ld, coff, D, out);
    count_launch();
    FFB_CHECK_LAUNCH();
    return false;
}

// ===========================================================================
// PLDUQ (plduq.cpp:36-123), right-looking row-order Crout in one CTA.
// Rows are processed in order; the pivot of a row is the leftmost nonzero of
// its residual over non-pivot columns.  W keeps the reference's packed
// storage: U coefficients in pivot rows, L multipliers in pivot columns,
// explicit zeros for rows that went pivotless before a pivot column appeared.
// ===========================================================================
namespace {

constexpr int PLDUQ_THREADS = 1024;

__global__ void __launch_bounds__(PLDUQ_THREADS)
    k_plduq_v1(Fp f, uint32_t* W, int64_t ldw, int m, int n, int32_t* info, int32_t* colflag,
               uint32_t* lvec, uint32_t* Lo, int64_t ldlo, uint32_t* d, uint32_t* Uo, int64_t lduo) {
    FFB_PDL_ENTRY();
    __shared__ int jmin, nrow;
    __shared__ uint32_t sxi;
    const int tid = threadIdx.x;
    int32_t* row_image = info + 1;
    int32_t* col_image = info + 1 + m;
    int32_t* pc = info + 1 + m + n;
    for (int j = tid; j < n; j += PLDUQ_THREADS) colflag[j] = 0;
    if (tid == 0) nrow = m;
    __syncthreads();
    {  // the first row with a nonzero entry
        int mine = m;
        const int64_t total = (int64_t)m * n;
        for (int64_t e = tid; e < total; e += PLDUQ_THREADS) {
            const int i2 = (int)(e / n);
            if (i2 < mine && W[(int64_t)i2 * ldw + (int)(e % n)] != 0) mine = i2;
        }
        if (mine < m) atomicMin(&nrow, mine);
    }
    int r = 0, nm = 0, i = 0;
    // The trailing update of a pivot step also finds the next row whose residual is nonzero:
    // the rows before it are pivotless (plduq.cpp:60-63) and are skipped in one step, so the
    // loop runs once per pivot, not once per row.
    while (true) {
        __syncthreads();
        const int nx = nrow;
        for (int t = tid; t < nx - i; t += PLDUQ_THREADS) row_image[m - 1 - (nm + t)] = i + t;  // from the back for now
        nm += nx - i;
        if (nx >= m) break;
        i = nx;
        __syncthreads();
        if (tid == 0) {
            jmin = n;
            nrow = m;
        }
        __syncthreads();
        uint32_t* wi = W + (int64_t)i * ldw;
        for (int j = tid; j < n; j += PLDUQ_THREADS)
            if (!colflag[j] && wi[j] != 0) atomicMin(&jmin, j);
        __syncthreads();
        const int jp = jmin;
        if (tid == 0) {
            const uint32_t x = wi[jp];
            sxi = finv(f, x);
            d[r] = x;
            row_image[r] = i;
            pc[r] = jp;
        }
        __syncthreads();
        const uint32_t xi = sxi;
        for (int j = tid; j < n; j += PLDUQ_THREADS)  // U coefficients (plduq.cpp:65-70)
            if (!colflag[j] && j != jp) wi[j] = fmul(f, xi, wi[j]);
        for (int i2 = i + 1 + tid; i2 < m; i2 += PLDUQ_THREADS) lvec[i2] = W[(int64_t)i2 * ldw + jp];
        __syncthreads();
        // trailing rows: residual update on non-pivot columns, L multiplier in column jp
        const int rows_left = m - i - 1;
        const int64_t total = (int64_t)rows_left * n;
        int mine = m;
        for (int64_t e = tid; e < total; e += PLDUQ_THREADS) {
            const int i2 = i + 1 + (int)(e / n), j = (int)(e % n);
            if (colflag[j]) continue;
            uint32_t* w = W + (int64_t)i2 * ldw + j;
            if (j == jp) {
                *w = fmul(f, lvec[i2], xi);
            } else {
                const uint32_t v = fsub(f, *w, fmul(f, lvec[i2], wi[j]));
                *w = v;
                if (v != 0 && i2 < mine) mine = i2;
            }
        }
        if (mine < m) atomicMin(&nrow, mine);
        __syncthreads();
        if (tid == 0) colflag[jp] = 1;
        ++r;
        ++i;
    }
    __syncthreads();
    // Pivotless rows ascending after the pivot rows (plduq.cpp:86-90).
    if (tid == 0) {
        info[0] = r;
        for (int a = 0, b = nm - 1; a < b; ++a, --b) {
            const int32_t t = row_image[r + a];
            row_image[r + a] = row_image[r + b];
            row_image[r + b] = t;
        }
        for (int k = 0; k < r; ++k) col_image[k] = pc[k];
        int q = r;
        for (int j = 0; j < n; ++j)
            if (!colflag[j]) col_image[q++] = j;
    }
    __syncthreads();
    // Dense factors (plduq.cpp:96-115).
    for (int64_t e = tid; e < (int64_t)m * r; e += PLDUQ_THREADS) {
        const int a = (int)(e / r), k = (int)(e % r);
        uint32_t v = 0;
        if (a == k) v = 1 % f.p;
        else if (a > k) v = W[(int64_t)row_image[a] * ldw + pc[k]];
        Lo[(int64_t)a * ldlo + k] = v;
    }
    for (int64_t e = tid; e < (int64_t)r * n; e += PLDUQ_THREADS) {
        const int k = (int)(e / n), a = (int)(e % n);
        uint32_t v = 0;
        if (a == k) v = 1 % f.p;
        else if (a > k) v = W[(int64_t)row_image[k] * ldw + col_image[a]];
        Uo[(int64_t)k * lduo + a] = v;
    }
}


// The same elimination for p <= 255 with W held in shared memory as bytes (m * n up to
// ~220 KB): the passes of a pivot step (U coefficients, trailing update with the search for
// the next nonzero row, one warp per row) run at shared-memory speed and cost ~ the rank, so
// short-and-wide or low-rank Y need not take the chunked pipeline.  W in global memory is only
// read: with rcap < min(m, n) the kernel gives up after rcap pivots (info[0] = -1, nothing
// else written that matters) and the caller runs the parallel PLDUQ on the untouched input.
__global__ void __launch_bounds__(PLDUQ_THREADS)
    k_plduq_smem(Fp f, const uint32_t* W, int64_t ldw, int m, int n, int32_t* info, uint32_t* Lo, int64_t ldlo,
                 uint32_t* d, uint32_t* dinv, uint32_t* Uo, int64_t lduo, int rcap) {
    FFB_PDL_ENTRY();
    extern __shared__ __align__(16) uint8_t ps_raw[];
    const int ns = (n + 3) & ~3, ms4 = (m + 3) & ~3;
    uint8_t* W8 = ps_raw;                                   // m x ns
    uint8_t* cf = W8 + (size_t)m * ns;                      // ns column flags
    uint8_t* lv = cf + ns;                                  // m multipliers of the pivot column
    int32_t* rimg = reinterpret_cast<int32_t*>(lv + ms4);   // m
    int32_t* pcs = rimg + m;                                // min(m, n) pivot columns
    int32_t* cimg = pcs + min(m, n);                        // n
    __shared__ int jmin, nrow;
    __shared__ uint32_t sxi;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    {  // stage W (a warp per row) and find the first row with a nonzero entry
        int mine = m;
        for (int i = wp; i < m; i += 32) {
            bool nz = false;
            const uint32_t* src = W + (int64_t)i * ldw;
            for (int j0 = lane; j0 < ns; j0 += 32 * 8) {  // 8 loads in flight per lane
                uint32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = j0 + 32 * u < n ? __ldcg(src + j0 + 32 * u) : 0u;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (j0 + 32 * u < ns) {
                        W8[(size_t)i * ns + j0 + 32 * u] = (uint8_t)v[u];
                        nz |= v[u] != 0;
                    }
            }
            if (__any_sync(0xffffffffu, nz) && i < mine) mine = i;
        }
        for (int j = tid; j < ns; j += PLDUQ_THREADS) cf[j] = 0;
        if (tid == 0) nrow = m;
        __syncthreads();
        if (lane == 0 && mine < m) atomicMin(&nrow, mine);
    }
    int r = 0, nm = 0, i = 0;
    bool bail = false;
    while (true) {
        __syncthreads();
        const int nx = nrow;
        for (int t = tid; t < nx - i; t += PLDUQ_THREADS) rimg[m - 1 - (nm + t)] = i + t;  // from the back for now
        nm += nx - i;
        if (nx >= m) break;
        if (r >= rcap) {  // uniform
            bail = true;
            break;
        }
        i = nx;
        __syncthreads();
        if (tid == 0) {
            jmin = n;
            nrow = m;
        }
        __syncthreads();
        uint8_t* wi = W8 + (size_t)i * ns;
        for (int j = tid; j < n; j += PLDUQ_THREADS)
            if (!cf[j] && wi[j] != 0) atomicMin(&jmin, j);
        __syncthreads();
        const int jp = jmin;
        if (tid == 0) {
            const uint32_t x = wi[jp];
            sxi = finv(f, x);
            d[r] = x;
            dinv[r] = sxi;
            rimg[r] = i;
            pcs[r] = jp;
        }
        __syncthreads();
        const uint32_t xi = sxi;
        for (int j = tid; j < n; j += PLDUQ_THREADS)  // U coefficients (plduq.cpp:65-70)
            if (!cf[j] && j != jp) wi[j] = (uint8_t)red32(f, xi * wi[j]);
        for (int i2 = i + 1 + tid; i2 < m; i2 += PLDUQ_THREADS) lv[i2] = W8[(size_t)i2 * ns + jp];
        if (tid == 0) cf[jp] = 1;  // from here on column jp is a pivot column (skipped below)
        __syncthreads();
        int mine = m;
        const uint32_t* cfw = reinterpret_cast<const uint32_t*>(cf);
        const uint32_t* uw = reinterpret_cast<const uint32_t*>(wi);
        for (int i2 = i + 1 + wp; i2 < m; i2 += 32) {  // trailing rows, a warp per row, 4 columns per lane
            const uint32_t l = lv[i2];
            uint32_t* w = reinterpret_cast<uint32_t*>(W8 + (size_t)i2 * ns);
            bool nz = false;
            if (l) {  // residual update on non-pivot columns, L multiplier in column jp
                const uint32_t nl = f.p - l;
                for (int jw = lane; jw < (ns >> 2); jw += 32) {
                    const uint32_t fm = cfw[jw] * 0xffu, u4 = uw[jw], w4 = w[jw];
                    uint32_t o = w4 & fm;  // pivot columns keep their L multipliers
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const uint32_t v = red32(f, ((w4 >> (8 * b)) & 0xffu) + nl * ((u4 >> (8 * b)) & 0xffu));
                        o |= (v << (8 * b)) & ~fm;
                    }
                    w[jw] = o;
                    nz |= (o & ~fm) != 0;
                }
                __syncwarp();
                if (lane == 0) W8[(size_t)i2 * ns + jp] = (uint8_t)red32(f, l * xi);
            } else {  // multiplier 0: the row is unchanged (its entry in column jp is 0)
                for (int jw = lane; jw < (ns >> 2); jw += 32) nz |= (w[jw] & ~(cfw[jw] * 0xffu)) != 0;
            }
            if (__any_sync(0xffffffffu, nz) && i2 < mine) mine = i2;
        }
        if (lane == 0 && mine < m) atomicMin(&nrow, mine);
        ++r;
        ++i;
    }
    __syncthreads();
    if (bail) {
        if (tid == 0) info[0] = -1;
        return;
    }
    // pivotless rows ascending after the pivot rows (plduq.cpp:86-90); column image: the pivot
    // columns in pivot order, then the others ascending
    for (int t = tid; t < nm / 2; t += PLDUQ_THREADS) {
        const int32_t a = rimg[r + t];
        rimg[r + t] = rimg[r + nm - 1 - t];
        rimg[r + nm - 1 - t] = a;
    }
    for (int k = tid; k < r; k += PLDUQ_THREADS) cimg[k] = pcs[k];
    if (wp == 0) {
        int q = r;
        for (int j0 = 0; j0 < n; j0 += 32) {
            const int j = j0 + lane;
            const bool fr = j < n && !cf[j];
            const unsigned bal = __ballot_sync(0xffffffffu, fr);
            if (fr) cimg[q + __popc(bal & ((1u << lane) - 1u))] = j;
            q += __popc(bal);
        }
    }
    __syncthreads();
    int32_t* row_image = info + 1;
    int32_t* col_image = info + 1 + m;
    int32_t* pc = info + 1 + m + n;
    if (tid == 0) info[0] = r;
    for (int t = tid; t < m; t += PLDUQ_THREADS) row_image[t] = rimg[t];
    for (int t = tid; t < n; t += PLDUQ_THREADS) col_image[t] = cimg[t];
    for (int t = tid; t < r; t += PLDUQ_THREADS) pc[t] = pcs[t];
    // dense factors (plduq.cpp:96-115)
    for (int64_t e = tid; e < (int64_t)m * r; e += PLDUQ_THREADS) {
        const int a = (int)(e / r), k = (int)(e % r);
        uint32_t v = 0;
        if (a == k) v = 1 % f.p;
        else if (a > k) v = W8[(size_t)rimg[a] * ns + pcs[k]];
        Lo[(int64_t)a * ldlo + k] = v;
    }
    for (int k = wp; k < r; k += 32) {  // a warp per U row
        const uint8_t* wr = W8 + (size_t)rimg[k] * ns;
        for (int a = lane; a < n; a += 32) {
            uint32_t v = 0;
            if (a == k) v = 1 % f.p;
            else if (a > k) v = wr[cimg[a]];
            Uo[(int64_t)k * lduo + a] = v;
        }
    }
}

}  // namespace

void plduq(const Fp& f, cudaStream_t st, DMat W, int32_t* info, int32_t* colflag, uint32_t* lvec,
           DMat Lo, uint32_t* d, DMat Uo) {
    ProfScope ps(K_PLDUQ, st, 0.0, 4.0 * W.rows * W.cols);
    launch_k(k_plduq_v1, 1, PLDUQ_THREADS, 0, st, f, W.ptr, W.ld, (int)W.rows, (int)W.cols, info, colflag,
                                            lvec, Lo.ptr, Lo.ld, d, Uo.ptr, Uo.ld);
    count_launch();
    FFB_CHECK_LAUNCH();
}

size_t plduq_smem_bytes(int64_t m, int64_t n) {
    const int64_t ns = (n + 3) & ~3, ms4 = (m + 3) & ~3;
    return (size_t)(m * ns + ns + ms4 + 4 * (m + std::min(m, n) + n));
}

bool plduq_smem(const Fp& f, cudaStream_t st, DMat W, int32_t* info, DMat Lo, uint32_t* d, uint32_t* dinv, DMat Uo,
                int rcap) {
    const size_t bytes = plduq_smem_bytes(W.rows, W.cols);
    constexpr size_t cap = (size_t)226 * 1024;  // 227 KB per CTA less the static words
    if (f.p > 255u || !f.mu32 || bytes > cap || W.rows <= 0 || W.cols <= 0) return false;
    static DeviceOnce attr;
    if (!attr.done()) {
        FFB_CUDA(cudaFuncSetAttribute(k_plduq_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap));
        attr.mark();
    }
    ProfScope ps(K_PLDUQ, st, 0.0, 4.0 * W.rows * W.cols);
    launch_k(k_plduq_smem, 1, PLDUQ_THREADS, bytes, st, f, (const uint32_t*)W.ptr, W.ld, (int)W.rows, (int)W.cols, info,
             Lo.ptr, Lo.ld, d, dinv, Uo.ptr, Uo.ld, rcap);
    count_launch();
    FFB_CHECK_LAUNCH();
    return true;
}

}  // namespace ffb
