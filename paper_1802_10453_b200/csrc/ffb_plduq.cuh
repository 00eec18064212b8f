// ffb_plduq.cuh -- parallel PLDUQ + LDU helpers (ffb_plduq.cu).
#pragma once

#include <functional>
#include <string>
#include <vector>

#include "ffb_kernels.cuh"

namespace ffb {

// Stack-allocator view over the context workspace (stream-ordered reuse).
struct Workspace {
    char* base = nullptr;
    size_t cap = 0;
    size_t* top = nullptr;
    size_t mark() const { return *top; }
    void release(size_t m) { *top = m; }
    void* alloc(size_t bytes) {
        const size_t a = (*top + 255) & ~(size_t)255;
        if (a + bytes > cap)
            throw Status(FFB_NO_MEMORY, "device workspace exhausted (" + std::to_string(a + bytes) +
                                            " > " + std::to_string(cap) + " bytes)");
        *top = a + bytes;
        return base + a;
    }
    DMat mat(int64_t rows, int64_t cols) {
        DMat m;
        m.rows = rows;
        m.cols = cols;
        m.ld = cols > 0 ? cols : 1;
        m.ptr = (uint32_t*)alloc((size_t)(rows > 0 ? rows : 1) * m.ld * sizeof(uint32_t));
        return m;
    }
    template <class T>
    T* vec(int64_t n) {
        return (T*)alloc((size_t)(n > 0 ? n : 1) * sizeof(T));
    }
};

struct PlduqIO {
    std::function<const int32_t*(const std::vector<int32_t>&)> upload;
    std::function<const void*(const void*, size_t)> readback;
    // optional: reserve a kernel-published read-back, and wait for it
    std::function<MboxPost()> post;
    std::function<const void*(const MboxPost&)> wait;
    // optional: called with the column image as soon as the pivots are known (before the
    // factors are formed; again if a failed certificate forces the exact retry)
    std::function<void(const std::vector<int32_t>&)> pivots_ready;
    DMat Lo, Uo;        // m x min(m,n) and min(m,n) x n outputs
    uint32_t* d = nullptr;
    uint32_t* dinv = nullptr;
};

struct PlduqOut {
    int64_t r = 0;
    std::vector<int32_t> rimg, cimg;
    int fallbacks = 0;
};

// PLDUQ of Y (m x n, preserved) into io.Lo/io.Uo/io.d/io.dinv.
PlduqOut plduq_parallel(const Fp& f, cudaStream_t st, DMat Y, Workspace& ws, const PlduqIO& io);

void gather2d(cudaStream_t st, DMat dst, DMat src, const int32_t* ridx, const int32_t* cidx,
              int64_t roff = 0);
void copy_mat(cudaStream_t st, DMat dst, DMat src);
// In-place LDU without pivoting (strict lower L, diagonal d, strict upper U).
void ldu_inplace(const Fp& f, cudaStream_t st, DMat K, Workspace& ws, int32_t* fail);

// Kernel micro-benchmark hook (see ffb_plduq.cu).
void dbg_pq_bench(const Fp& f, cudaStream_t st, int which, int rows, int cols, const uint32_t* d_in,
                  int reps, double* ms, int32_t* out_k);

}  // namespace ffb
