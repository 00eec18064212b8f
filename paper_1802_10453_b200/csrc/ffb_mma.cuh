// ffb_mma.cuh -- warp-level int8 tensor-core helpers (mma.sync m16n8k32,
// s8 x s8 -> s32) for the latency-sized kernels of small primes (p <= 255):
// residues are centered to [-(p-1)/2, (p-1)/2] so products are exact in s32.
//
// Fragment layout (m16n8k32, gid = lane / 4, tig = lane % 4):
//   A (16 x 32, row-major, k contiguous): a0 = A[gid][4 tig .. +3], a1 = A[gid + 8][same],
//                                         a2 = A[gid][16 + 4 tig ..], a3 = A[gid + 8][16 + ...]
//   B (32 x 8, k contiguous per column):  b0 = B[4 tig .. +3][gid], b1 = B[16 + 4 tig ..][gid]
//   D (16 x 8):  d0, d1 = D[gid][2 tig, +1], d2, d3 = D[gid + 8][2 tig, +1]
#pragma once

#include "ffb_common.cuh"

namespace ffb {

__device__ __forceinline__ void mma_s8_16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ int8_t center8(uint32_t x, uint32_t p, uint32_t half) {
    return (int8_t)(x > half ? (int)x - (int)p : (int)x);
}
// s32 accumulator of centered products -> residue: (acc + 2^31) mod p - 2^31 mod p
__device__ __forceinline__ uint32_t mma_reduce(const Fp& f, int acc, uint32_t bias) {
    return fsub(f, red32(f, (uint32_t)acc ^ 0x80000000u), bias);
}

}  // namespace ffb
