// ffb_tc_gemm.cu -- tcgen05 / TMEM / TMA modular GEMM for small primes (p <= 255).
//
//   C (M x N, uint32 residues) = C -/+ op(A) op(B)  or  op(A) op(B)   (mod p)
//
// Operands are first packed (bandwidth-bound kernel) into centered int8
// K-major buffers: x in [0,p) -> x or x-p in [-127, 127].  The products are
// exact in int32 (|acc| <= K * 127^2 < 2^31 for K < 133k), so the modular
// reduction is delayed to the epilogue: one Barrett reduction per output.
//
// Kernel (one 128 x BN output tile per CTA, 6 warps):
//   warp 0      TMA producer: 128x128 B A-tile + BNx128 B B-tile per stage,
//               SWIZZLE_128B, mbarrier expect_tx
//   warp 1      TMEM allocation + single-thread tcgen05.mma.kind::i8 issue
//               (M=128, N=BN, K=32 per instruction, 4 per stage), commit
//               frees the stage / signals the accumulator
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> mod p -> smem transpose ->
//               coalesced read-modify-write of C
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "ffb_kernels.cuh"

namespace ffb {

namespace {

constexpr int TC_BM = 128;
constexpr int TC_BK = 128;  // bytes = int8 elements per stage (one 128B swizzle atom)
constexpr int TC_THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
    d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;        // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                  // descriptor version (sm100)
    d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN, int ST = 0>
struct TcCfg {
    static constexpr int STAGES = ST ? ST : (BN == 256 ? 4 : 6);
    static constexpr int A_BYTES = TC_BM * TC_BK;
    static constexpr int B_BYTES = BN * TC_BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BYTES = 4 * 32 * 33 * 4;
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + 256;
    static constexpr uint32_t IDESC = (2u << 4)           // D format: s32
                                      | (1u << 7)         // A: signed int8
                                      | (1u << 10)        // B: signed int8
                                      | ((uint32_t)(BN >> 3) << 17)  // N
                                      | ((uint32_t)(TC_BM >> 4) << 24);  // M
};

template <int BN, int ST>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_gemm_i8_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 uint32_t* C, int64_t ldc, int M, int N, int nk, Fp f, int mode, int halo) {
    FFB_PDL_ENTRY();
    using Cfg = TcCfg<BN, ST>;
    // upper band (halo >= 0): tiles entirely below the band j >= i - halo are not computed
    if (halo >= 0 && (int64_t)(blockIdx.x + 1) * BN + halo <= (int64_t)blockIdx.y * TC_BM) return;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;
    uint8_t* sB = smem + Cfg::STAGES * Cfg::A_BYTES;
    uint32_t* sEpi = (uint32_t*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t* full = (uint64_t*)(sEpi + 4 * 32 * 33);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* accfull = empty + Cfg::STAGES;
    uint32_t* tmem_slot = (uint32_t*)(accfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * TC_BM, n0 = blockIdx.x * BN;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
        for (int s = 0; s < Cfg::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"((uint32_t)BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer ----
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % Cfg::STAGES;
                const uint32_t ph = (kb / Cfg::STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
                tma_load_2d(sA + s * Cfg::A_BYTES, &tmA, &full[s], kb * TC_BK, m0);
                tma_load_2d(sB + s * Cfg::B_BYTES, &tmB, &full[s], kb * TC_BK, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer (single thread) ----
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % Cfg::STAGES;
                const uint32_t ph = (kb / Cfg::STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a0 = smem_u32(sA + s * Cfg::A_BYTES);
                const uint32_t b0 = smem_u32(sB + s * Cfg::B_BYTES);
#pragma unroll
                for (int kk = 0; kk < TC_BK / 32; ++kk)
                    mma_i8(tmem, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), Cfg::IDESC,
                           (kb | kk) != 0);
                mma_commit(&empty[s]);  // stage free once these MMAs have read it
            }
            mma_commit(accfull);
        }
    } else {
        // ---- epilogue: warps 2..5 own TMEM lanes 32*(warp%4) .. +31 ----
        const int q = warp & 3;
        uint32_t* tile = sEpi + (warp - 2) * 32 * 33;
        // acc in (-2^31, 2^31): (acc + 2^31) mod p by 32-bit Barrett, minus 2^31 mod p
        const Fp16 h(f.p);
        const uint32_t bias = (uint32_t)((0x80000000ull) % f.p);
        const int rbase = m0 + 32 * q;
        // the C slab is read before the accumulator is waited on (and, for the
        // next slab, while this one is reduced): C traffic overlaps the MMAs
        uint32_t cv[32];
        auto load_c = [&](int c) {
            const int col = n0 + c + lane;
            const bool colok = col < N;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) {
                const int row = rbase + rr;
                cv[rr] = (mode != GEMM_SET && colok && row < M) ? __ldcg(C + (int64_t)row * ldc + col) : 0u;
            }
        };
        load_c(0);
        mbar_wait(accfull, 0);
        tc_fence_after();
        for (int c = 0; c < BN; c += 32) {
            if (n0 + c >= N) break;
            uint32_t r[32];
            tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c, r);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t x = r[j] ^ 0x80000000u;  // = acc + 2^31 as unsigned
                tile[lane * 33 + j] = h.sub(h.red(x), bias);
            }
            __syncwarp();
            const int col = n0 + c + lane;
            const bool colok = col < N;
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) {
                const int row = rbase + rr;
                if (colok && row < M) {
                    const uint32_t v = tile[rr * 33 + lane];
                    uint32_t o;
                    if (mode == GEMM_SUB) o = h.sub(cv[rr], v);
                    else if (mode == GEMM_ADD) o = fadd(f, cv[rr], v);
                    else o = v;
                    C[(int64_t)row * ldc + col] = o;
                }
            }
            if (c + 32 < BN && n0 + c + 32 < N) load_c(c + 32);
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"((uint32_t)BN));
    }
}

// ---------------------------------------------------------------------------
// Persistent variant for large products (p <= 255): one CTA per SM walks the
// 128 x 256 output tiles (M fastest, so the CTAs in flight share B tiles);
// the accumulator is double-buffered in TMEM (2 x 256 columns), so the
// epilogue of tile t (8 warps: TMEM lane quadrant warp % 4, column half) runs
// while the MMA warp accumulates tile t+1.  Pipelines: smem full/empty
// (TMA <-> MMA) and TMEM full/empty (MMA <-> epilogue).
// ---------------------------------------------------------------------------
constexpr int TP_BN = 256, TP_STAGES = 3, TP_EPI_WARPS = 8, TP_THREADS = (2 + TP_EPI_WARPS) * 32;
struct TpCfg {
    static constexpr int A_BYTES = TC_BM * TC_BK;
    static constexpr int B_BYTES = TP_BN * TC_BK;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BYTES = TP_EPI_WARPS * 32 * 33 * 4;
    static constexpr int SMEM = 1024 + TP_STAGES * STAGE_BYTES + EPI_BYTES + 256;
};
// Grouped raster: groups of TP_GM M-tiles, N walking inside a group, so the
// ~148 tiles in flight touch TP_GM A tiles and ~148/TP_GM B tiles (an L2-resident
// working set) instead of every A tile per wave.
constexpr int TP_GM = 16;
__device__ __forceinline__ void tp_tile(int t, int num_m, int num_n, int& m_blk, int& n_blk) {
    const int per = TP_GM * num_n, g = t / per, r = t - g * per;
    const int gm = min(TP_GM, num_m - g * TP_GM);
    m_blk = g * TP_GM + r % gm;
    n_blk = r / gm;
}
// Upper band (halo >= 0): tile (mb, nb) is live iff it holds an entry with j >= i - halo.
__device__ __forceinline__ bool tp_live(int t, int num_m, int num_n, int halo) {
    if (halo < 0) return true;
    int mb, nb;
    tp_tile(t, num_m, num_n, mb, nb);
    return (int64_t)(nb + 1) * TP_BN + halo > (int64_t)mb * TC_BM;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(TP_THREADS, 1)
    k_gemm_i8_tcp(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  uint32_t* C, int64_t ldc, int M, int N, int nk, Fp f, int mode, int num_m, int num_tiles,
                  int halo) {
    const int num_n = num_tiles / num_m;
    FFB_PDL_ENTRY();
    extern __shared__ __align__(1024) uint8_t tp_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)tp_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;
    uint8_t* sB = smem + TP_STAGES * TpCfg::A_BYTES;
    uint32_t* sEpi = (uint32_t*)(smem + TP_STAGES * TpCfg::STAGE_BYTES);
    uint64_t* full = (uint64_t*)(sEpi + TP_EPI_WARPS * 32 * 33);
    uint64_t* empty = full + TP_STAGES;
    uint64_t* tfull = empty + TP_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
        for (int s = 0; s < TP_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], TP_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(2u * TP_BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    constexpr uint32_t IDESC = TcCfg<TP_BN>::IDESC;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer ----
            int s = 0;
            uint32_t ph = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                if (!tp_live(t, num_m, num_n, halo)) continue;
                int mb, nbk;
                tp_tile(t, num_m, num_n, mb, nbk);
                const int m0 = mb * TC_BM, n0 = nbk * TP_BN;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], TpCfg::STAGE_BYTES);
                    tma_load_2d(sA + s * TpCfg::A_BYTES, &tmA, &full[s], kb * TC_BK, m0);
                    tma_load_2d(sB + s * TpCfg::B_BYTES, &tmB, &full[s], kb * TC_BK, n0);
                    if (++s == TP_STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer ----
            int s = 0, acc = 0;
            uint32_t ph = 0, aph = 0;
            for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
                if (!tp_live(t, num_m, num_n, halo)) continue;
                mbar_wait(&tempty[acc], aph ^ 1);  // the epilogue has drained this accumulator
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * TP_BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + s * TpCfg::A_BYTES);
                    const uint32_t b0 = smem_u32(sB + s * TpCfg::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < TC_BK / 32; ++kk)
                        mma_i8(d, sw128_desc(a0 + kk * 32), sw128_desc(b0 + kk * 32), IDESC, (kb | kk) != 0);
                    mma_commit(&empty[s]);
                    if (++s == TP_STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    aph ^= 1;
                }
            }
        }
    } else {
        // ---- epilogue: TMEM lanes 32*(warp % 4), columns [128 h, 128 h + 128) ----
        const int q = warp & 3, h = (warp - 2) >> 2;
        uint32_t* tile = sEpi + (warp - 2) * 32 * 33;
        const Fp16 hf(f.p);
        const uint32_t bias = (uint32_t)((0x80000000ull) % f.p);
        int acc = 0;
        uint32_t aph = 0;
        uint32_t cv[32];
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            if (!tp_live(t, num_m, num_n, halo)) continue;
            int mb, nbk;
            tp_tile(t, num_m, num_n, mb, nbk);
            const int m0 = mb * TC_BM, n0 = nbk * TP_BN + 128 * h;
            const int rbase = m0 + 32 * q;
            auto load_c = [&](int c) {
                const int col = n0 + c + lane;
                const bool colok = col < N;
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) {
                    const int row = rbase + rr;
                    cv[rr] = (mode != GEMM_SET && colok && row < M) ? __ldcg(C + (int64_t)row * ldc + col) : 0u;
                }
            };
            load_c(0);  // C does not depend on the accumulator
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
            for (int c = 0; c < 128; c += 32) {
                if (n0 + c >= N) break;
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * TP_BN + 128 * h + c), r);
#pragma unroll
                for (int j = 0; j < 32; ++j) tile[lane * 33 + j] = hf.sub(hf.red(r[j] ^ 0x80000000u), bias);
                __syncwarp();
                const int col = n0 + c + lane;
                const bool colok = col < N;
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) {
                    const int row = rbase + rr;
                    if (colok && row < M) {
                        const uint32_t v = tile[rr * 33 + lane];
                        uint32_t o;
                        if (mode == GEMM_SUB) o = hf.sub(cv[rr], v);
                        else if (mode == GEMM_ADD) o = fadd(f, cv[rr], v);
                        else o = v;
                        C[(int64_t)row * ldc + col] = o;
                    }
                }
                if (c + 32 < 128 && n0 + c + 32 < N) load_c(c + 32);
                __syncwarp();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);  // accumulator free for tile t + 2
            if (++acc == 2) {
                acc = 0;
                aph ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2u * TP_BN));
    }
}

// ---------------------------------------------------------------------------
// Limb variant for 255 < p < 2^23 (configuration 3).  A centered residue x,
// |x| < 2^22, is split into signed int8 limbs x = a0 + 2^8 a1 + 2^16 a2
// (|a2| <= 64).  Per 32-deep K step the single MMA thread issues the 9 limb
// products A_i B_j^T into 5 TMEM accumulators, one per shift class s = i + j
// (5 x 64 columns); each class sum is exact in int32 for K < 65536.  The
// epilogue folds  sum_s (acc_s mod p) * (2^{8s} mod p)  mod p.
// Operands: 3 limb planes stacked by rows ([plane][rows][Kp]); one 2-D tensor
// map covers all planes (rows a plane over-reads land only in masked output
// rows/columns; the last plane is zero-filled by TMA).
// ---------------------------------------------------------------------------
constexpr int LB_BN = 64, LB_STAGES = 2;
constexpr int LB_A_BYTES = 3 * TC_BM * TC_BK, LB_B_BYTES = 3 * LB_BN * TC_BK;
constexpr int LB_STAGE_BYTES = LB_A_BYTES + LB_B_BYTES;
constexpr int LB_EPI_BYTES = 4 * 32 * 33 * 4;
constexpr int LB_SMEM = 1024 + LB_STAGES * LB_STAGE_BYTES + LB_EPI_BYTES + 256;
constexpr uint32_t LB_IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(LB_BN >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);

__global__ void __launch_bounds__(TC_THREADS, 1)
    k_gemm_limb_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   uint32_t* C, int64_t ldc, int M, int N, int nk, int Mrows, int Nrows,
                   Fp f, int mode) {
    FFB_PDL_ENTRY();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;
    uint8_t* sB = smem + LB_STAGES * LB_A_BYTES;
    uint32_t* sEpi = (uint32_t*)(smem + LB_STAGES * LB_STAGE_BYTES);
    uint64_t* full = (uint64_t*)(sEpi + 4 * 32 * 33);
    uint64_t* empty = full + LB_STAGES;
    uint64_t* accfull = empty + LB_STAGES;
    uint32_t* tmem_slot = (uint32_t*)(accfull + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * TC_BM, n0 = blockIdx.x * LB_BN;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmB) : "memory");
        for (int s = 0; s < LB_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(accfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % LB_STAGES;
                const uint32_t ph = (kb / LB_STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], LB_STAGE_BYTES);
                for (int l = 0; l < 3; ++l) {
                    tma_load_2d(sA + s * LB_A_BYTES + l * TC_BM * TC_BK, &tmA, &full[s], kb * TC_BK,
                                l * Mrows + m0);
                    tma_load_2d(sB + s * LB_B_BYTES + l * LB_BN * TC_BK, &tmB, &full[s], kb * TC_BK,
                                l * Nrows + n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % LB_STAGES;
                const uint32_t ph = (kb / LB_STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a0 = smem_u32(sA + s * LB_A_BYTES);
                const uint32_t b0 = smem_u32(sB + s * LB_B_BYTES);
#pragma unroll
                for (int kk = 0; kk < TC_BK / 32; ++kk)
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int j = 0; j < 3; ++j) {
                            // first product of each shift class in this (i, j) order
                            const bool first = (i == 0) || (i == 1 && j == 2) || (i == 2 && j == 2);
                            mma_i8(tmem + (uint32_t)((i + j) * LB_BN),
                                   sw128_desc(a0 + i * TC_BM * TC_BK + kk * 32),
                                   sw128_desc(b0 + j * LB_BN * TC_BK + kk * 32), LB_IDESC,
                                   ((kb | kk) != 0 || !first) ? 1u : 0u);
                        }
                mma_commit(&empty[s]);
            }
            mma_commit(accfull);
        }
    } else {
        const int q = warp & 3;
        uint32_t* tile = sEpi + (warp - 2) * 32 * 33;
        const uint32_t mu32 = (uint32_t)(0x100000000ull / f.p);
        const uint32_t bias = (uint32_t)((0x80000000ull) % f.p);
        mbar_wait(accfull, 0);
        tc_fence_after();
        const int rbase = m0 + 32 * q;
        for (int c = 0; c < LB_BN; c += 32) {
            if (n0 + c >= N) break;
            // sum_s 2^(8s) class_s mod p: 64-bit sums of reduced terms (< 5 p^2 < 2^49), one
            // 64-bit reduction per element; the class loop is not unrolled (code size: a short
            // launch is otherwise bound by instruction fetch)
            uint64_t v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0;
            uint32_t w = 1 % f.p;  // 2^(8s) mod p
#pragma unroll 1
            for (int s = 0; s < 5; ++s) {
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(s * LB_BN + c), r);
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const uint32_t x = r[j] ^ 0x80000000u;  // acc + 2^31
                    uint32_t qq = __umulhi(x, mu32);
                    uint32_t rr = x - qq * f.p;
                    if (rr >= f.p) rr -= f.p;
                    rr = fsub(f, rr, bias);                  // acc mod p
                    v[j] += (uint64_t)rr * w;
                }
                w = (uint32_t)(((uint64_t)w << 8) % f.p);
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) tile[lane * 33 + j] = red64(f, v[j]);
            __syncwarp();
            const int col = n0 + c + lane;
            const bool colok = col < N;
            uint32_t cv[32];
            if (mode != GEMM_SET) {
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) {
                    const int row = rbase + rr;
                    cv[rr] = (colok && row < M) ? __ldcg(C + (int64_t)row * ldc + col) : 0u;
                }
            }
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) {
                const int row = rbase + rr;
                if (colok && row < M) {
                    const uint32_t val = tile[rr * 33 + lane];
                    uint32_t o;
                    if (mode == GEMM_SUB) o = fsub(f, cv[rr], val);
                    else if (mode == GEMM_ADD) o = fadd(f, cv[rr], val);
                    else o = val;
                    C[(int64_t)row * ldc + col] = o;
                }
            }
            __syncwarp();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

// 3 limb planes of centered op(src): dst[l][i][k]  (plane stride rows*ldd)
__device__ __forceinline__ void limbs(uint32_t x, uint32_t p, int8_t& a0, int8_t& a1, int8_t& a2) {
    int32_t c = x > (p >> 1) ? (int32_t)x - (int32_t)p : (int32_t)x;
    const int32_t l0 = ((c + 128) & 255) - 128;
    c = (c - l0) >> 8;
    const int32_t l1 = ((c + 128) & 255) - 128;
    c = (c - l1) >> 8;
    a0 = (int8_t)l0;
    a1 = (int8_t)l1;
    a2 = (int8_t)c;
}

__global__ void k_pack_limb_n(int8_t* dst, int64_t ldd, int64_t plane, const uint32_t* src,
                              int64_t lds, int64_t rows, int64_t K, uint32_t p) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < ldd;
         k += (int64_t)gridDim.x * blockDim.x) {
        int8_t a0 = 0, a1 = 0, a2 = 0;
        if (i < rows && k < K) limbs(src[i * lds + k], p, a0, a1, a2);
        dst[i * ldd + k] = a0;
        dst[plane + i * ldd + k] = a1;
        dst[2 * plane + i * ldd + k] = a2;
    }
}

__global__ void k_pack_limb_t(int8_t* dst, int64_t ldd, int64_t plane, const uint32_t* src,
                              int64_t lds, int64_t rows, int64_t K, uint32_t p) {
    FFB_PDL_ENTRY();
    __shared__ uint32_t tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 32;
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int64_t k = k0 + yy, i = i0 + threadIdx.x;
        tile[yy][threadIdx.x] = (k < K && i < rows) ? src[k * lds + i] : 0u;
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int64_t i = i0 + yy, k = k0 + threadIdx.x;
        if (i < rows && k < ldd) {
            int8_t a0, a1, a2;
            limbs(tile[threadIdx.x][yy], p, a0, a1, a2);
            dst[i * ldd + k] = a0;
            dst[plane + i * ldd + k] = a1;
            dst[2 * plane + i * ldd + k] = a2;
        }
    }
}

// ---------------------------------------------------------------------------
// Packing: dst (rows x ldd int8, K-major) <- centered op(src), zero padding.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int8_t center(uint32_t x, uint32_t p) {
    return (int8_t)(x > (p >> 1) ? (int32_t)x - (int32_t)p : (int32_t)x);
}

// Both operands in one launch: blockIdx.z selects the job.
struct PackJob {
    int8_t* dst;
    int64_t ldd;  // row stride of the packed operand
    const uint32_t* src;
    int64_t lds;
    int64_t rows, K;
    int trans;
    int64_t kw;  // packed k written: [0, kw) (= ldd, or one K segment of a concatenation)
};
// Both operands of a GEMM in one launch (blockIdx.z = job), 64 x 64 tiles of
// the packed (rows x ldd) int8 output per CTA, 16-byte vector stores.  Not
// transposed: thread = 16 consecutive k of one row (4 x 16-byte loads).
// Transposed (src is K x rows): the tile goes through shared memory, loads
// 16-byte along rows of src, stores 16 bytes along k.  Unaligned operands
// take scalar loads (same tiles).
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t p) {
    return (uint32_t)(uint8_t)center(a, p) | ((uint32_t)(uint8_t)center(b, p) << 8) |
           ((uint32_t)(uint8_t)center(c, p) << 16) | ((uint32_t)(uint8_t)center(d, p) << 24);
}
__global__ void __launch_bounds__(256) k_pack2(PackJob j0, PackJob j1, uint32_t p) {
    FFB_PDL_ENTRY();
    const PackJob& j = blockIdx.z == 0 ? j0 : j1;
    __shared__ __align__(16) uint8_t tile[64][64 + 16];
    const int64_t i0 = (int64_t)blockIdx.y * 64, k0 = (int64_t)blockIdx.x * 64;
    if (i0 >= j.rows || k0 >= j.kw) return;  // uniform per block
    const int t = threadIdx.x;
    const bool vec = ((j.lds & 3) == 0) && ((((uintptr_t)j.src) & 15) == 0);
    if (!j.trans) {
        const int64_t i = i0 + (t >> 2), k = k0 + 16 * (t & 3);
        if (i >= j.rows || k >= j.kw) return;
        uint32_t v[16];
        const uint32_t* sp = j.src + i * j.lds + k;
        if (vec && k + 16 <= j.K) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 w = __ldcg(reinterpret_cast<const uint4*>(sp) + q);
                v[4 * q] = w.x, v[4 * q + 1] = w.y, v[4 * q + 2] = w.z, v[4 * q + 3] = w.w;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = (k + e < j.K) ? sp[e] : 0u;
        }
        uint4 o;
        o.x = pack4(v[0], v[1], v[2], v[3], p);
        o.y = pack4(v[4], v[5], v[6], v[7], p);
        o.z = pack4(v[8], v[9], v[10], v[11], p);
        o.w = pack4(v[12], v[13], v[14], v[15], p);
        *reinterpret_cast<uint4*>(j.dst + i * j.ldd + k) = o;  // ldd, k multiples of 16
        return;
    }
    // transposed: tile[kk][ii] = center(src[k0 + kk][i0 + ii])
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int kk = (t >> 4) + 16 * u, ii = 4 * (t & 15);
        const int64_t k = k0 + kk, i = i0 + ii;
        uint32_t w[4];
        const uint32_t* sp = j.src + k * j.lds + i;
        if (vec && k < j.K && i + 4 <= j.rows) {
            const uint4 x = __ldcg(reinterpret_cast<const uint4*>(sp));
            w[0] = x.x, w[1] = x.y, w[2] = x.z, w[3] = x.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) w[e] = (k < j.K && i + e < j.rows) ? sp[e] : 0u;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) tile[kk][ii + e] = (uint8_t)center(w[e], p);
    }
    __syncthreads();
    const int ii = t >> 2, ks = 16 * (t & 3);
    const int64_t i = i0 + ii, k = k0 + ks;
    if (i >= j.rows || k >= j.kw) return;
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        o[q] = (uint32_t)tile[ks + 4 * q][ii] | ((uint32_t)tile[ks + 4 * q + 1][ii] << 8) |
               ((uint32_t)tile[ks + 4 * q + 2][ii] << 16) | ((uint32_t)tile[ks + 4 * q + 3][ii] << 24);
    *reinterpret_cast<uint4*>(j.dst + i * j.ldd + k) = make_uint4(o[0], o[1], o[2], o[3]);
}

// not transposed: op(src)[i][k] = src[i][k]
__global__ void k_pack_n(int8_t* dst, int64_t ldd, const uint32_t* src, int64_t lds, int64_t rows,
                         int64_t K, uint32_t p) {
    FFB_PDL_ENTRY();
    const int64_t i = blockIdx.y;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < ldd;
         k += (int64_t)gridDim.x * blockDim.x)
        dst[i * ldd + k] = (i < rows && k < K) ? center(src[i * lds + k], p) : (int8_t)0;
}

// transposed: op(src)[i][k] = src[k][i]  (src is K x rows)
__global__ void k_pack_t(int8_t* dst, int64_t ldd, const uint32_t* src, int64_t lds, int64_t rows,
                         int64_t K, uint32_t p) {
    FFB_PDL_ENTRY();
    __shared__ int8_t tile[32][33];
    const int64_t i0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 32;
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int64_t k = k0 + yy, i = i0 + threadIdx.x;
        tile[yy][threadIdx.x] = (k < K && i < rows) ? center(src[k * lds + i], p) : (int8_t)0;
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int64_t i = i0 + yy, k = k0 + threadIdx.x;
        if (i < rows && k < ldd) dst[i * ldd + k] = tile[threadIdx.x][yy];
    }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

void load_encode() {
    static std::once_flag once;
    std::call_once(once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    });
    if (!g_encode) throw Status(FFB_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
}

CUtensorMap make_map(const int8_t* base, int64_t rows, int64_t ld, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)base, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Status(FFB_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

struct Scratch {
    int8_t* ptr = nullptr;
    size_t cap = 0;
};
thread_local Scratch g_scratch_slots[FFB_MAX_DEVICES][6];

int8_t* scratch(size_t bytes) {
    Scratch& g_scratch = g_scratch_slots[current_device()][g_slot];
    if (g_scratch.cap < bytes) {
        if (g_scratch.ptr) {
            FFB_CUDA(cudaDeviceSynchronize());
            FFB_CUDA(cudaFree(g_scratch.ptr));
        }
        const size_t cap = std::max(bytes + bytes / 4, (size_t)64 << 20);
        FFB_CUDA(cudaMalloc(&g_scratch.ptr, cap));
        g_scratch.cap = cap;
    }
    return g_scratch.ptr;
}

void pack(cudaStream_t st, int8_t* dst, int64_t ldd, DMat src, bool trans, int64_t rows, int64_t K,
          uint32_t p) {
    if (!trans) {
        for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
            const int64_t nr = std::min<int64_t>(65535, rows - r0);
            int64_t gx = std::min<int64_t>(64, cdiv(ldd, 256));
            launch_k(k_pack_n, dim3((unsigned)gx, (unsigned)nr), 256, 0, st, dst + r0 * ldd, ldd, src.ptr + r0 * src.ld, src.ld, nr, K, p);
        }
    } else {
        dim3 grid((unsigned)cdiv(ldd, 32), (unsigned)cdiv(rows, 32));
        launch_k(k_pack_t, grid, dim3(32, 8), 0, st, dst, ldd, src.ptr, src.ld, rows, K, p);
    }
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

template <int BN, int ST = 0>
void launch_tc(cudaStream_t st, const CUtensorMap& ma, const CUtensorMap& mb, DMat C, int64_t M,
               int64_t N, int64_t nk, const Fp& f, int mode, int halo) {
    using Cfg = TcCfg<BN, ST>;
    static DeviceOnce attr;
    if (!attr.done()) {
        FFB_CUDA(cudaFuncSetAttribute(k_gemm_i8_tc<BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg::SMEM));
        attr.mark();
    }
    dim3 grid((unsigned)cdiv(N, BN), (unsigned)cdiv(M, TC_BM));
    launch_k(k_gemm_i8_tc<BN, ST>, grid, TC_THREADS, Cfg::SMEM, st, ma, mb, C.ptr, C.ld, (int)M, (int)N,
                                                          (int)nk, f, mode, halo);
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

}  // namespace

bool tc_gemm_supported(const Fp& f, int64_t M, int64_t N, int64_t K) {
    static const bool disabled = getenv("FFB_DISABLE_TC") != nullptr;
    if (disabled) return false;
    // small M is fine: TMA zero-fills the rows of the A box beyond M
    const bool shape = M >= 8 && N >= 64 && K >= 16 && (double)M * N * K >= 1.0e6 &&
                       M < (1ll << 30) && N < (1ll << 30);
    if (f.p <= 255) return shape && K <= 120000;
    return f.p < (1u << 23) && shape && K <= 40000;  // int8 limbs: 3 * 2^14 * K < 2^31
}

void tc_gemm_limb(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B,
                  bool tb, int64_t M, int64_t N, int64_t K) {
    const int64_t Kp = (K + 15) / 16 * 16;
    const int64_t Mr = cdiv(M, TC_BM) * TC_BM, Nr = cdiv(N, LB_BN) * LB_BN;
    const size_t aplane = (size_t)Mr * Kp, bplane = (size_t)Nr * Kp;
    const size_t abytes = (3 * aplane + 1023) / 1024 * 1024, bbytes = (3 * bplane + 1023) / 1024 * 1024;
    int8_t* buf = scratch(abytes + bbytes);
    int8_t* Ap = buf;
    int8_t* Bp = buf + abytes;
    {
        ProfScope ps(K_PACK, st, 0.0, 7.0 * (M * K + N * K));
        FFB_CUDA(cudaMemsetAsync(buf, 0, abytes + bbytes, st)); pdl_fence(st);
        auto pk = [&](int8_t* dst, size_t plane, DMat src, bool trans, int64_t rows) {
            if (!trans) {
                for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
                    const int64_t nr = std::min<int64_t>(65535, rows - r0);
                    launch_k(k_pack_limb_n, dim3((unsigned)std::min<int64_t>(64, cdiv(Kp, 256)), (unsigned)nr), 256, 0, st, dst + r0 * Kp, Kp, (int64_t)plane, src.ptr + r0 * src.ld, src.ld, nr, K, f.p);
                }
            } else {
                launch_k(k_pack_limb_t, dim3((unsigned)cdiv(Kp, 32), (unsigned)cdiv(rows, 32)), dim3(32, 8), 0, st, dst, Kp, (int64_t)plane, src.ptr, src.ld, rows, K, f.p);
            }
            ++g_launches;
            FFB_CHECK_LAUNCH();
        };
        pk(Ap, aplane, A, ta, M);
        pk(Bp, bplane, B, !tb, N);
    }
    static DeviceOnce attr;
    if (!attr.done()) {
        FFB_CUDA(cudaFuncSetAttribute(k_gemm_limb_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, LB_SMEM));
        attr.mark();
    }
    ProfScope ps(K_GEMM, st, 2.0 * M * N * K, 3.0 * (M * K + N * K) + 8.0 * M * N, M, N, -K);
    CUtensorMap ma = make_map(Ap, 3 * Mr, Kp, TC_BM), mb = make_map(Bp, 3 * Nr, Kp, LB_BN);
    dim3 grid((unsigned)cdiv(N, LB_BN), (unsigned)cdiv(M, TC_BM));
    launch_k(k_gemm_limb_tc, grid, TC_THREADS, LB_SMEM, st, ma, mb, C.ptr, C.ld, (int)M, (int)N,
                                                     (int)cdiv(Kp, TC_BK), (int)Mr, (int)Nr, f, mode);
    ++g_launches;
    FFB_CHECK_LAUNCH();
}

// Fraction of the M x N output in tiles (bm x bn) that touch the band j >= i - halo.
double band_fraction(int64_t M, int64_t N, int bm, int bn, int halo) {
    if (halo < 0 || M <= 0 || N <= 0) return 1.0;
    const int64_t nm = cdiv(M, bm), nn = cdiv(N, bn);
    int64_t live = 0;
    for (int64_t mb = 0; mb < nm; ++mb)
        for (int64_t nb = 0; nb < nn; ++nb) live += (nb + 1) * bn + halo > mb * bm;
    return (double)live / (double)(nm * nn);
}

// One GEMM term op(A) op(B) with inner dimension K; several terms share one accumulator
// when their operands are packed as one K-concatenated problem (tc_gemm2).
struct TcSeg {
    DMat A;
    bool ta;
    DMat B;
    bool tb;
    int64_t K;
};

// Pack the terms side by side along k (each segment padded to 16) and run one tcgen05 GEMM:
// C op= sum_s op(A_s) op(B_s).  p <= 255.
static void tc_run(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, int64_t M, int64_t N, const TcSeg* sg,
                   int nseg) {
    int64_t Kp = 0, K = 0;
    for (int i = 0; i < nseg; ++i) {
        Kp += (sg[i].K + 15) / 16 * 16;
        K += sg[i].K;
    }
    const size_t abytes = ((size_t)M * Kp + 1023) / 1024 * 1024;
    const size_t bbytes = ((size_t)N * Kp + 1023) / 1024 * 1024;
    int8_t* buf = scratch(abytes + bbytes);
    int8_t* Ap = buf;
    int8_t* Bp = buf + abytes;
    {
        ProfScope ps(K_PACK, st, 0.0, 5.0 * (M * K + N * K));
        int64_t off = 0;
        for (int i = 0; i < nseg; ++i) {
            const TcSeg& q = sg[i];
            const int64_t kw = (q.K + 15) / 16 * 16;
            // B^T (N x K) is needed: transposed pack unless tb
            PackJob ja{Ap + off, Kp, q.A.ptr, q.A.ld, M, q.K, q.ta ? 1 : 0, kw},
                jb{Bp + off, Kp, q.B.ptr, q.B.ld, N, q.K, q.tb ? 0 : 1, kw};
            const int64_t rmax = std::max(M, N);
            if (rmax <= (int64_t)65535 * 64) {
                dim3 grid((unsigned)cdiv(kw, 64), (unsigned)cdiv(rmax, 64), 2);
                launch_k(k_pack2, grid, 256, 0, st, ja, jb, f.p);
                ++g_launches;
                FFB_CHECK_LAUNCH();
            } else {  // (a single term only: see tc_gemm2)
                pack(st, Ap, Kp, q.A, q.ta, M, q.K, f.p);
                pack(st, Bp, Kp, q.B, !q.tb, N, q.K, f.p);
            }
            off += kw;
        }
    }
    const int64_t nk = cdiv(Kp, TC_BK);
    const bool wide = N >= 256 && M * N >= (int64_t)148 * 128 * 256;
    const int halo = g_band_halo;  // >= 0: only the upper band of a symmetric update
    const int bn = nk <= 2 || !wide ? 128 : 256;
    const double live = band_fraction(M, N, TC_BM, bn, halo);
    ProfScope ps(K_GEMM, st, 2.0 * M * N * K * live, (double)M * K + N * K + 8.0 * M * N * live, M, N, K);
    if (nk <= 2) {  // short K: epilogue-bound, 2 CTAs per SM (2-stage pipeline)
        CUtensorMap ma = make_map(Ap, M, Kp, TC_BM), mb = make_map(Bp, N, Kp, 128);
        launch_tc<128, 2>(st, ma, mb, C, M, N, nk, f, mode, halo);
    } else if (wide && !getenv("FFB_TC_NONPERSISTENT")) {
        CUtensorMap ma = make_map(Ap, M, Kp, TC_BM), mb = make_map(Bp, N, Kp, TP_BN);
        static DeviceOnce attr;
        static int nsm_dev[FFB_MAX_DEVICES];
        if (!attr.done()) {
            FFB_CUDA(cudaFuncSetAttribute(k_gemm_i8_tcp, cudaFuncAttributeMaxDynamicSharedMemorySize, TpCfg::SMEM));
            int dev = 0;
            FFB_CUDA(cudaGetDevice(&dev));
            FFB_CUDA(cudaDeviceGetAttribute(&nsm_dev[current_device()], cudaDevAttrMultiProcessorCount, dev));
            attr.mark();
        }
        const int nsm = nsm_dev[current_device()];
        const int num_m = (int)cdiv(M, TC_BM), num_tiles = num_m * (int)cdiv(N, TP_BN);
        // beside the critical path: a persistent grid on part of the SMs only, the rest
        // stay free for the engine stream's latency kernels
        // (inside the green SM partition the whole partition is available to it)
        static const int shared_env = getenv("FFB_Z_OVERLAP_SMS") ? atoi(getenv("FFB_Z_OVERLAP_SMS")) : 0;
        const GreenSide& gs = green_side();
        const int shared_sms = shared_env ? shared_env : (gs.ok ? gs.sms : 100);
        const int ctas = std::min(num_tiles, g_tc_shared_sms ? std::min(shared_sms, nsm) : nsm);
        launch_k(k_gemm_i8_tcp, ctas, TP_THREADS, TpCfg::SMEM, st, ma, mb, C.ptr, C.ld,
                 (int)M, (int)N, (int)nk, f, (int)mode, num_m, num_tiles, halo);
        ++g_launches;
        FFB_CHECK_LAUNCH();
    } else if (wide) {
        CUtensorMap ma = make_map(Ap, M, Kp, TC_BM), mb = make_map(Bp, N, Kp, 256);
        launch_tc<256>(st, ma, mb, C, M, N, nk, f, mode, halo);
    } else {
        CUtensorMap ma = make_map(Ap, M, Kp, TC_BM), mb = make_map(Bp, N, Kp, 128);
        launch_tc<128>(st, ma, mb, C, M, N, nk, f, mode, halo);
    }
}


void tc_gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
             int64_t M, int64_t N, int64_t K) {
    load_encode();
    if (f.p > 255) {
        tc_gemm_limb(f, st, mode, C, A, ta, B, tb, M, N, K);
        return;
    }
    const TcSeg sg{A, ta, B, tb, K};
    tc_run(f, st, mode, C, M, N, &sg, 1);
}

bool tc_gemm2(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A1, bool ta1, DMat B1, bool tb1, DMat A2,
              bool ta2, DMat B2, bool tb2, int64_t M, int64_t N, int64_t K1, int64_t K2) {
    if (f.p > 255 || std::max(M, N) > (int64_t)65535 * 64 || !tc_gemm_supported(f, M, N, K1 + K2)) return false;
    load_encode();
    const TcSeg sg[2] = {{A1, ta1, B1, tb1, K1}, {A2, ta2, B2, tb2, K2}};
    tc_run(f, st, mode, C, M, N, sg, 2);
    return true;
}

}  // namespace ffb
