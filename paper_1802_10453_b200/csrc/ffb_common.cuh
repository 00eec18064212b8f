// ffb_common.cuh -- shared device/host definitions of the B200 PLDL^TP^T engine.
//
// Residues of GF(p) live in HBM as uint32 in [0, p) (p < 2^31).  Field
// arithmetic follows the reference's PrimeField semantics
// (proj/include/ffldl/field.hpp:73-134): add/sub/neg canonical, multiply with
// Barrett reduction instead of a 128-bit '%', inverse by extended Euclid
// (or a table for p < 2^16), halve for odd p.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <atomic>
#include <stdexcept>
#include <string>

#include "../../include/ffldl_b200.h"

namespace ffb {

// Per-device CUDA state.  A context may live on any device and one thread may use
// several (ffldl.default_context(device)), so streams, events, scratch buffers and
// cudaFuncSetAttribute guards are kept per device, never per process or thread only.
constexpr int FFB_MAX_DEVICES = 32;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & (FFB_MAX_DEVICES - 1);
}
// "done once on this device" flag (e.g. the >48 KB dynamic shared memory attribute):
// if (!g.done()) { cudaFuncSetAttribute(...); g.mark(); }  -- a repeated set is harmless.
// Driver-API entry points used by the engine, resolved at run time through the runtime
// (cudaGetDriverEntryPoint) so the library has no link-time dependency on libcuda and still
// loads on a host without a GPU driver (null entries: feature unavailable).
struct DriverApi {
    decltype(&cuCtxGetCurrent) ctxGetCurrent = nullptr;
    decltype(&cuCtxSetCurrent) ctxSetCurrent = nullptr;
    decltype(&cuDeviceGet) deviceGet = nullptr;
    decltype(&cuDeviceGetDevResource) deviceGetDevResource = nullptr;
    decltype(&cuDevSmResourceSplitByCount) smResourceSplitByCount = nullptr;
    decltype(&cuDevResourceGenerateDesc) resourceGenerateDesc = nullptr;
    decltype(&cuGreenCtxCreate) greenCtxCreate = nullptr;
    decltype(&cuCtxFromGreenCtx) ctxFromGreenCtx = nullptr;
    decltype(&cuGreenCtxStreamCreate) greenCtxStreamCreate = nullptr;
};
const DriverApi& drv();  // ffb_engine.cu
inline CUcontext current_ctx() {
    CUcontext c = nullptr;
    if (drv().ctxGetCurrent) drv().ctxGetCurrent(&c);
    return c;
}

// Kernel attributes belong to a CUDA context: keyed by the current one (the device's primary
// context, or the side-stream green context of GreenScope).
struct DeviceOnce {
    std::atomic<void*> ctx[16] = {};
    bool done() const {
        const CUcontext c = current_ctx();
        for (const auto& x : ctx)
            if (x.load(std::memory_order_acquire) == (void*)c) return true;
        return false;
    }
    void mark() {
        const CUcontext c = current_ctx();
        for (auto& x : ctx) {
            void* e = nullptr;
            if (x.compare_exchange_strong(e, (void*)c) || e == (void*)c) return;
        }
    }
};

// Optional SM partition (FFB_GREEN=1) for the streams that run bulk updates beside the
// critical path (the large Schur update on zst, PLDUQ's Uhat absorb): a green context
// holding all but a reserve of SMs (FFB_GREEN_RESERVE, default 16), so the 1-CTA latency
// kernels of the critical path never share an SM with those GEMMs.  Work enqueued on such a
// stream is issued with the green context current (GreenScope).  Measured neutral on
// config 5 (113.8 vs 113.1 ms), so off by default.
struct GreenSide {
    bool ok = false;
    CUgreenCtx g = nullptr;
    CUcontext gctx = nullptr;
    int sms = 0;
};
GreenSide& green_side();  // per device, created on first use (ffb_engine.cu)
struct GreenScope {
    CUcontext prev = nullptr;
    bool on = false;
    explicit GreenScope(bool enable) {
        if (!enable) return;
        GreenSide& g = green_side();
        if (!g.ok) return;
        drv().ctxGetCurrent(&prev);
        drv().ctxSetCurrent(g.gctx);
        on = true;
    }
    ~GreenScope() {
        if (on) drv().ctxSetCurrent(prev);
    }
};
// A stream of the device's green context (or an ordinary stream when it is disabled).
cudaStream_t make_side_stream(int priority);

// ---------------------------------------------------------------------------
// Errors: the C-ABI maps these 1:1 to FFB_* status codes.
// ---------------------------------------------------------------------------
struct Status : std::runtime_error {
    int code;
    Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FFB_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            throw ::ffb::Status(FFB_CUDA_ERROR, std::string(#call) + ": " +                  \
                                                    cudaGetErrorString(e_));                 \
    } while (0)

#define FFB_CHECK_LAUNCH() FFB_CUDA(cudaGetLastError())

// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Every kernel starts with FFB_PDL_ENTRY():
// it lets the next kernel in the stream be scheduled right away and then waits
// until this kernel's predecessor has completed (its writes visible) -- so a
// kernel never touches memory before its predecessor is done, while the
// launch latency and CTA ramp-up overlap the predecessor's tail.  Without a
// programmatic launch both instructions are no-ops.
//
// Consequence for loads: a kernel's lifetime now overlaps its predecessor's
// writes, which breaks the contract of the non-coherent read-only path
// (ld.global.nc: data read-only for the kernel's lifetime).  Kernels therefore
// use coherent loads only -- __ldcg (L2) instead of __ldg, and no __restrict__
// on pointers (nvcc turns const __restrict__ loads into ld.global.nc).  The
// SASS check is `cuobjdump -sass | grep LDG.*CONSTANT` (must be empty).
// ---------------------------------------------------------------------------
#define FFB_PDL_ENTRY()                                                    \
    do {                                                                   \
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");     \
        asm volatile("griddepcontrol.wait;" ::: "memory");                  \
    } while (0)

// kernel<<<grid, block, smem, st>>>(args...) with the programmatic-serialization
// attribute (FFB_NO_PDL=1 disables it); arguments are coerced to the kernel's
// parameter types like a <<<>>> launch.
//
// A programmatic launch may only follow a kernel: after a copy, memset or event
// wait on a stream, pdl_fence(stream) makes the next kernel there launch with
// full stream serialization (griddepcontrol.wait orders kernels, not copies).
struct PdlFences {
    cudaStream_t s[8];
    int n = 0;
};
inline PdlFences& pdl_fences() {
    static thread_local PdlFences f;
    return f;
}
inline void pdl_fence(cudaStream_t st) {
    PdlFences& f = pdl_fences();
    for (int i = 0; i < f.n; ++i)
        if (f.s[i] == st) return;
    if (f.n < 8) f.s[f.n++] = st;
}
inline bool pdl_take(cudaStream_t st) {
    PdlFences& f = pdl_fences();
    for (int i = 0; i < f.n; ++i)
        if (f.s[i] == st) {
            f.s[i] = f.s[--f.n];
            return true;
        }
    return false;
}

inline long long& pdl_launch_index() {
    static thread_local long long i = 0;
    return i;
}
inline bool& pdl_enabled() {
    static thread_local bool on = true;
    return on;
}
struct PdlScope {  // disables programmatic launches within a scope
    bool saved;
    explicit PdlScope(bool on) : saved(pdl_enabled()) { pdl_enabled() = on && saved; }
    ~PdlScope() { pdl_enabled() = saved; }
};

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
    static_assert(sizeof...(KArgs) == sizeof...(Args), "kernel argument count");
    static const bool pdl_on = getenv("FFB_NO_PDL") == nullptr;
    // bisection hook: FFB_PDL_RANGE=a:b (global launch indices)
    static long long ra = -1, rb = -1;
    static bool rinit = false;
    if (!rinit) {
        if (const char* r = getenv("FFB_PDL_RANGE")) sscanf(r, "%lld:%lld", &ra, &rb);
        rinit = true;
    }
    const long long me = pdl_launch_index()++;
    static const bool log = getenv("FFB_LAUNCH_LOG") != nullptr;
    if (log) {
        const char* nm = nullptr;
        cudaFuncGetName(&nm, (const void*)kern);
        fprintf(stderr, "[launch %lld] %s grid %u,%u,%u\n", me, nm ? nm : "?", grid.x, grid.y, grid.z);
    }
    const bool in_range = ra < 0 || (me >= ra && me < rb);
    const bool pdl = pdl_on && !pdl_take(st) && pdl_enabled() && in_range;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    if (e != cudaSuccess)
        throw Status(FFB_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Field constants (passed by value to every kernel).
// ---------------------------------------------------------------------------
struct Fp {
    uint32_t p;
    uint64_t mu;            // floor((2^64-1)/p), Barrett constant
    const uint32_t* inv;    // device inverse table (p < 2^16) or nullptr
    int char2;              // p == 2
    uint32_t mu32;          // floor(2^32/p) when p < 2^16 (32-bit Barrett), else 0
};

// Field constants for modulus p (host side).
inline Fp make_fp(uint64_t p, const uint32_t* inv_table) {
    Fp f;
    f.p = (uint32_t)p;
    f.mu = UINT64_MAX / p;
    f.inv = inv_table;
    f.char2 = p == 2;
    f.mu32 = p < 65536 ? (uint32_t)(0x100000000ull / p) : 0u;
    return f;
}

__host__ __device__ inline uint64_t umulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// x mod p for any 64-bit x.
__host__ __device__ inline uint32_t red64(const Fp& f, uint64_t x) {
    uint64_t q = umulhi64(x, f.mu);
    uint64_t r = x - q * f.p;
    while (r >= f.p) r -= f.p;
    return (uint32_t)r;
}
__host__ __device__ inline uint32_t fadd(const Fp& f, uint32_t a, uint32_t b) {
    uint32_t s = a + b;  // < 2^32 since p < 2^31
    return s >= f.p ? s - f.p : s;
}
__host__ __device__ inline uint32_t fsub(const Fp& f, uint32_t a, uint32_t b) {
    return a >= b ? a - b : a + f.p - b;
}
__host__ __device__ inline uint32_t fneg(const Fp& f, uint32_t a) { return a ? f.p - a : 0; }
__host__ __device__ inline uint32_t fmul(const Fp& f, uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    if (f.mu32) {  // p < 2^16: the product fits 32 bits (warp-uniform branch)
        const uint32_t x = a * b;
        const uint32_t q = __umulhi(x, f.mu32);
        const uint32_t r = x - q * f.p;
        return r >= f.p ? r - f.p : r;
    }
#endif
    return red64(f, (uint64_t)a * b);
}
// x mod p for x < 2^32 when p < 2^16 (f.mu32 set): 32-bit Barrett, one correction.
__device__ __forceinline__ uint32_t red32(const Fp& f, uint32_t x) {
    const uint32_t q = __umulhi(x, f.mu32);
    const uint32_t r = x - q * f.p;
    return r >= f.p ? r - f.p : r;
}
// d - c v mod p with one reduction when p < 2^16 (d + (p - c) v < p^2 < 2^32).
__host__ __device__ inline uint32_t fmsub(const Fp& f, uint32_t d, uint32_t c, uint32_t v) {
#ifdef __CUDA_ARCH__
    if (f.mu32) {
        const uint32_t x = d + (f.p - c) * v;
        const uint32_t q = __umulhi(x, f.mu32);
        const uint32_t r = x - q * f.p;
        return r >= f.p ? r - f.p : r;
    }
#endif
    return fsub(f, d, fmul(f, c, v));
}
// a/2 for odd p (field.hpp:121-124).
__host__ __device__ inline uint32_t fhalve(const Fp& f, uint32_t a) {
    return (a & 1) ? (uint32_t)(((uint64_t)a + f.p) >> 1) : (a >> 1);
}
// Extended Euclid (field.hpp:107-118); returns 0 for a == 0 (callers never pass 0).
__host__ __device__ inline uint32_t finv_euclid(uint32_t p, uint32_t a) {
    int64_t t = 0, nt = 1, r = p, nr = a;
    while (nr != 0) {
        int64_t q = r / nr, tmp;
        tmp = t - q * nt; t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    if (t < 0) t += p;
    return (uint32_t)t;
}
__device__ inline uint32_t finv(const Fp& f, uint32_t a) {
    if (f.inv) return f.inv[a];
    return finv_euclid(f.p, a);
}

// Inverse-table staging for latency-critical single-CTA kernels: for small p
// the table is copied to shared memory once (batched read-only loads), so an
// inverse on the critical path is a shared-memory lookup, not an L2 round trip.
constexpr int SINV_MAX = 4096;
struct SmemInv {
    const uint32_t* t;  // shared copy, or nullptr
    __device__ __forceinline__ uint32_t operator()(const Fp& f, uint32_t a) const {
        return t ? t[a] : finv(f, a);
    }
};
__device__ inline SmemInv stage_inverses(const Fp& f, uint32_t* buf /* SINV_MAX words */) {
    if (!f.inv || f.p > SINV_MAX) return SmemInv{nullptr};
    // 8 loads in flight per thread (one round trip for p <= 8 * blockDim)
    for (uint32_t a0 = threadIdx.x; a0 < f.p; a0 += 8 * blockDim.x) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t a = a0 + u * blockDim.x;
            v[u] = a < f.p ? __ldcg(f.inv + a) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t a = a0 + u * blockDim.x;
            if (a < f.p) buf[a] = v[u];
        }
    }
    __syncthreads();
    return SmemInv{buf};
}

// Batched read-only copy global -> shared of a rows x cols tile (row stride lds),
// with U independent loads in flight per thread.
template <int U>
__device__ __forceinline__ void load_tile(uint32_t* dst, int ldd, const uint32_t* src,
                                          int64_t lds, int rows, int cols) {
    // warp w copies rows w, w + nwarps, ...; lanes stride the columns; U rows
    // of loads are in flight before the stores (no integer division).
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r0 = w; r0 < rows; r0 += U * nw) {
        for (int c0 = lane; c0 < cols; c0 += 32) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = r0 + u * nw;
                v[u] = r < rows ? __ldcg(src + (int64_t)r * lds + c0) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = r0 + u * nw;
                if (r < rows) dst[r * ldd + c0] = v[u];
            }
        }
    }
}

// One-shot TMA bulk copy (cp.async.bulk) global -> shared of a contiguous
// range, completed on an mbarrier; used by the single-CTA latency kernels to
// stage their whole input with one instruction instead of rounds of loads.
// Requirements: dst, src and bytes multiples of 16.  Call with all threads.
__device__ __forceinline__ void bulk_stage(void* dst, const void* src, uint32_t bytes,
                                           uint64_t* bar) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                     : "memory");
        for (uint32_t off = 0; off < bytes; off += 32768u) {
            const uint32_t len = bytes - off < 32768u ? bytes - off : 32768u;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared((char*)dst + off)),
                "l"((const char*)src + off), "r"(len), "r"(b)
                : "memory");
        }
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "BULK_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@P1 bra BULK_DONE;\n"
        "bra BULK_WAIT;\n"
        "BULK_DONE:\n"
        "}\n" ::"r"(b)
        : "memory");
}
__host__ __device__ inline bool bulk_ok(const void* src, size_t bytes) {
    return ((uintptr_t)src & 15) == 0 && (bytes & 15) == 0;
}

// ---------------------------------------------------------------------------
// Strided row-major views of device matrices.
// ---------------------------------------------------------------------------
struct DMat {
    uint32_t* ptr = nullptr;
    int64_t ld = 0;
    int64_t rows = 0, cols = 0;
    __host__ __device__ uint32_t* at(int64_t i, int64_t j) const { return ptr + i * ld + j; }
    DMat sub(int64_t r0, int64_t c0, int64_t nr, int64_t nc) const {
        DMat m;
        m.ptr = ptr + r0 * ld + c0;
        m.ld = ld;
        m.rows = nr;
        m.cols = nc;
        return m;
    }
};

// Per-pivot-column encoding of D (mirrors BlockDiag, blockdiag.hpp:20-33).
enum DKind : int32_t {
    D_SCALAR = 0,
    D_ANTIDIAG_HEAD = 1,
    D_ANTIDIAG_TAIL = 2,
    D_ANTITRI_HEAD = 3,
    D_ANTITRI_TAIL = 4
};

// Global device-side D arrays, indexed by global pivot column.
// A read-back published directly by the producing kernel (no k_post launch): the
// kernel writes its words to dst (mapped pinned memory), fences at system scope
// and stores seq to *seq_ptr; the host spins on the sequence word.  dst == nullptr:
// not requested (the caller falls back to a posted read-back).
struct MboxPost {
    uint32_t* dst = nullptr;
    uint32_t* seq_ptr = nullptr;
    uint32_t seq = 0;
};
// one thread: words src[0 .. n) to the mailbox, then the sequence word
__device__ __forceinline__ void mbox_publish(const MboxPost& mp, const int32_t* src, int n) {
    for (int i = 0; i < n; ++i) mp.dst[i] = (uint32_t)src[i];
    __threadfence_system();
    *(volatile uint32_t*)mp.seq_ptr = mp.seq;
}

struct DDiag {
    int32_t* kind;
    uint32_t* val;   // Scalar d / AntiDiag x / AntiTri c
    uint32_t* val2;  // AntiTri d
    uint32_t* inv;   // inverse of val (d^-1, x^-1, c^-1)
};

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace ffb

namespace ffb {
// Fast arithmetic for p < 2^16 (products < 2^32): 32-bit Barrett.
struct Fp16 {
    uint32_t p;
    uint32_t mu;  // floor(2^32 / p)
    __host__ __device__ explicit Fp16(uint32_t pp) : p(pp), mu((uint32_t)(0x100000000ull / pp)) {}
    __device__ __forceinline__ uint32_t red(uint32_t x) const {
        uint32_t q = __umulhi(x, mu);
        uint32_t r = x - q * p;
        return r >= p ? r - p : r;
    }
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return red(a * b); }
    __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const {
        return a >= b ? a - b : a + p - b;
    }
};
// Field arithmetic selector: 32-bit Barrett for p < 2^16, 64-bit otherwise.
template <bool kSmall>
struct Ar;
template <>
struct Ar<true> {
    Fp16 h;
    Fp f;
    __device__ explicit Ar(const Fp& ff) : h(ff.p), f(ff) {}
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return h.mul(a, b); }
    __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const { return h.sub(a, b); }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const { return fadd(f, a, b); }
};
template <>
struct Ar<false> {
    Fp f;
    __device__ explicit Ar(const Fp& ff) : f(ff) {}
    __device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) const { return fmul(f, a, b); }
    __device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) const { return fsub(f, a, b); }
    __device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) const { return fadd(f, a, b); }
};

}  // namespace ffb

