// ffb_engine.cu -- host recursion of the B200 PLDL^TP^T engine + the C-ABI.
//
// The recursion tree is the reference's, node for node (proj/src/sytrf.cpp):
// dispatch (:337-350) -> crout leaf (:35-139) or recursive_step (:298-335),
// zero_leading (:267-292), zero_leading_pairs (:170-265).  The output triple
// (P, L, D) depends on that tree for non-generic rank profiles, so the host
// walks exactly the same nodes; each node's arithmetic runs on the device.
//
// Data layout in HBM:
//   W   n x n uint32 residues, the input; every node updates its own block
//       in place (Schur complements overwrite the trailing blocks).
//   Lg  n x n uint32: L indexed by (ORIGINAL row, global pivot column).  A
//       row's multipliers depend only on the row's identity, never on the
//       positions later permutations give it, so nodes write their columns
//       once and the final L is a single row gather by the output
//       permutation (no per-level row shuffles of L).
//   D   per-pivot-column kind / value / value2 / inverse arrays.
// Node-local permutations and ranks are read back to the host (they decide
// the shape of the next node); index arrays go down through a pinned ring.
#include <nvtx3/nvToolsExt.h>
#include <chrono>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <type_traits>
#include <mutex>
#include <atomic>
#include <array>
#include <vector>

#include "ffb_kernels.cuh"
#include "ffb_plduq.cuh"

using namespace ffb;

// ===========================================================================
// Context
// ===========================================================================
struct ffb_context {
    int device = 0;
    cudaStream_t stream = nullptr;
    char* ws_base = nullptr;
    size_t ws_cap = 0, ws_top = 0;
    char* up_host = nullptr;  // mapped pinned ring
    const char* up_dev = nullptr;  // its device alias
    size_t up_cap = 0, up_top = 0;
    char* down_host = nullptr;
    size_t down_cap = 0;
    uint32_t* inv_table = nullptr;
    uint32_t inv_p = 0;
    int32_t* flag = nullptr;  // device scratch flag
    int32_t* zero_flag = nullptr;  // is_zero tag (never reset; see is_zero)
    uint32_t zero_gen = 0;
    uint64_t launches = 0;
    uint64_t syncs = 0, syncs_last = 0;
    double sync_wait_ms = 0;  // host time blocked in read-backs (FFB_HOST_STATS)
    uint64_t uploads = 0;     // host -> device index uploads (FFB_HOST_STATS)
    // read-back mailbox (mapped pinned memory, see readback)
    uint32_t* mbox_host = nullptr;
    uint32_t* mbox_dev = nullptr;
    volatile uint32_t* mbox_seq_host = nullptr;
    uint32_t* mbox_seq_dev = nullptr;
    size_t mbox_cap = 0;
    uint32_t mbox_seq = 0;
    cudaStream_t copy_stream = nullptr;  // host <-> device transfers overlapped with the engine
    Profiler prof;
};

namespace ffb {
const DriverApi& drv() {
    static DriverApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, auto& fn) {
            void* p = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(p);
        };
        get("cuCtxGetCurrent", api.ctxGetCurrent);
        get("cuCtxSetCurrent", api.ctxSetCurrent);
        get("cuDeviceGet", api.deviceGet);
        get("cuDeviceGetDevResource", api.deviceGetDevResource);
        get("cuDevSmResourceSplitByCount", api.smResourceSplitByCount);
        get("cuDevResourceGenerateDesc", api.resourceGenerateDesc);
        get("cuGreenCtxCreate", api.greenCtxCreate);
        get("cuCtxFromGreenCtx", api.ctxFromGreenCtx);
        get("cuGreenCtxStreamCreate", api.greenCtxStreamCreate);
    });
    return api;
}

GreenSide& green_side() {
    static GreenSide gs[FFB_MAX_DEVICES];
    static std::once_flag once[FFB_MAX_DEVICES];
    const int d = current_device();
    std::call_once(once[d], [d] {
        GreenSide& g = gs[d];
        const DriverApi& a = drv();
        if (!getenv("FFB_GREEN") || !a.ctxGetCurrent || !a.ctxSetCurrent || !a.deviceGet ||
            !a.deviceGetDevResource || !a.smResourceSplitByCount || !a.resourceGenerateDesc || !a.greenCtxCreate ||
            !a.ctxFromGreenCtx || !a.greenCtxStreamCreate)
            return;
        const int reserve = getenv("FFB_GREEN_RESERVE") ? atoi(getenv("FFB_GREEN_RESERVE")) : 16;
        CUdevice dev;
        CUdevResource full, part, rem;
        unsigned nb = 1;
        if (a.deviceGet(&dev, d) != CUDA_SUCCESS) return;
        if (a.deviceGetDevResource(dev, &full, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return;
        const int want = (((int)full.sm.smCount - reserve) / 8) * 8;
        if (want < 8) return;
        if (a.smResourceSplitByCount(&part, &nb, &full, &rem, 0, (unsigned)want) != CUDA_SUCCESS || nb < 1)
            return;
        CUdevResourceDesc desc;
        if (a.resourceGenerateDesc(&desc, &part, 1) != CUDA_SUCCESS) return;
        if (a.greenCtxCreate(&g.g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return;
        if (a.ctxFromGreenCtx(&g.gctx, g.g) != CUDA_SUCCESS) return;
        g.sms = (int)part.sm.smCount;
        g.ok = true;
    });
    return gs[d];
}
cudaStream_t make_side_stream(int priority) {
    GreenSide& g = green_side();
    cudaStream_t s = nullptr;
    if (g.ok) {
        CUstream cs = nullptr;
        if (drv().greenCtxStreamCreate(&cs, g.g, CU_STREAM_NON_BLOCKING, priority) == CUDA_SUCCESS)
            return (cudaStream_t)cs;
    }
    FFB_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority));
    return s;
}
}  // namespace ffb

// Detail of the calling thread's last non-OK status (ffb_last_error); also set by ffb_io.cu.
thread_local std::string g_last_error;

namespace {

// ---------------------------------------------------------------------------
// Field setup (PrimeField checks, field.hpp:73-80).
// ---------------------------------------------------------------------------
uint64_t host_powmod(uint64_t a, uint64_t e, uint64_t m) {
    unsigned __int128 r = 1 % m, x = a % m;
    while (e) {
        if (e & 1) r = (r * x) % m;
        x = (x * x) % m;
        e >>= 1;
    }
    return (uint64_t)r;
}

bool host_is_prime(uint64_t n) {
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (uint64_t q : bases)
        if (n % q == 0) return n == q;
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; ++s; }
    for (uint64_t a : bases) {
        uint64_t x = host_powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int i = 1; i < s; ++i) {
            x = (uint64_t)(((unsigned __int128)x * x) % n);
            if (x == n - 1) { composite = false; break; }
        }
        if (composite) return false;
    }
    return true;
}

void check_modulus(uint64_t p) {
    if (p < 2 || p > ((1ull << 62) - 1) || !host_is_prime(p))
        throw Status(FFB_NOT_PRIME, "modulus " + std::to_string(p) + " is not a prime below 2^62");
    if (p >= (1ull << 31))
        throw Status(FFB_UNSUPPORTED, "device path supports primes below 2^31");
}

// ---------------------------------------------------------------------------
// Workspace: stack allocator over one device allocation (stream-ordered reuse
// is safe because every kernel runs on the context's single stream).
// ---------------------------------------------------------------------------
struct WsMark {
    size_t top;
};

void ensure_workspace(ffb_context* c, size_t bytes) {
    if (c->ws_cap >= bytes) return;
    if (c->ws_base) {
        FFB_CUDA(cudaStreamSynchronize(c->stream));
        FFB_CUDA(cudaFree(c->ws_base));
        c->ws_base = nullptr;
        c->ws_cap = 0;
    }
    size_t freeb = 0, totalb = 0;
    FFB_CUDA(cudaMemGetInfo(&freeb, &totalb));
    if (bytes > freeb) bytes = freeb > (1ull << 30) ? freeb - (1ull << 30) : freeb / 2;
    FFB_CUDA(cudaMalloc(&c->ws_base, bytes));
    c->ws_cap = bytes;
    c->ws_top = 0;
}

void* ws_alloc(ffb_context* c, size_t bytes) {
    const size_t a = (c->ws_top + 255) & ~(size_t)255;
    if (a + bytes > c->ws_cap)
        throw Status(FFB_NO_MEMORY, "device workspace exhausted (" + std::to_string(a + bytes) +
                                        " > " + std::to_string(c->ws_cap) + " bytes)");
    c->ws_top = a + bytes;
    return c->ws_base + a;
}

DMat ws_mat(ffb_context* c, int64_t rows, int64_t cols) {
    DMat m;
    m.rows = rows;
    m.cols = cols;
    m.ld = cols > 0 ? cols : 1;
    m.ptr = (uint32_t*)ws_alloc(c, (size_t)std::max<int64_t>(rows, 1) * m.ld * sizeof(uint32_t));
    return m;
}

template <class T>
T* ws_vec(ffb_context* c, int64_t n) {
    return (T*)ws_alloc(c, (size_t)std::max<int64_t>(n, 1) * sizeof(T));
}

// Upload ring fetch: the engine stream pulls the words from the mapped pinned
// ring with loads over the bus.  A kernel rather than a copy-engine operation:
// it stays in the programmatic-launch chain, and it is not queued behind bulk
// host-to-device copies on other streams (the banded input upload).
__global__ void __launch_bounds__(512) k_fetch(uint32_t* dst, const uint32_t* src, int64_t words) {
    FFB_PDL_ENTRY();
    const int64_t w4 = words >> 2, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < w4; i += stride)
        reinterpret_cast<uint4*>(dst)[i] = __ldcv(reinterpret_cast<const uint4*>(src) + i);
    for (int64_t i = 4 * w4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += stride)
        dst[i] = __ldcv(src + i);
}

// Pinned upload ring: index arrays going down to the device.
const int32_t* upload_into(ffb_context* c, int32_t* d, const int32_t* v, size_t n);
const int32_t* upload(ffb_context* c, const int32_t* v, size_t n) {
    return upload_into(c, ws_vec<int32_t>(c, (int64_t)n), v, n);
}
// ... into a given device buffer
const int32_t* upload_into(ffb_context* c, int32_t* d, const int32_t* v, size_t n) {
    if (n == 0) return d;
    const size_t bytes = n * sizeof(int32_t);
    if (bytes > c->up_cap) {  // rare: larger than the ring, copy synchronously
        FFB_CUDA(cudaStreamSynchronize(c->stream));
        FFB_CUDA(cudaMemcpy(d, v, bytes, cudaMemcpyHostToDevice));
        return d;
    }
    size_t off = (c->up_top + 15) & ~(size_t)15;
    if (off + bytes > c->up_cap) {
        FFB_CUDA(cudaStreamSynchronize(c->stream));
        off = 0;
    }
    memcpy(c->up_host + off, v, bytes);
    static const bool dma = getenv("FFB_UPLOAD_DMA") != nullptr;
    if (dma) {
        FFB_CUDA(cudaMemcpyAsync(d, c->up_host + off, bytes, cudaMemcpyHostToDevice, c->stream));
        pdl_fence(c->stream);
    } else {
        const int64_t words = (int64_t)n;
        const int blocks = (int)std::min<int64_t>(64, std::max<int64_t>(1, cdiv(words, 4 * 512)));
        launch_k(k_fetch, blocks, 512, 0, c->stream, (uint32_t*)d, (const uint32_t*)(c->up_dev + off), words);
    }
    ++c->uploads;
    c->up_top = off + bytes;
    return d;
}
const int32_t* upload(ffb_context* c, const std::vector<int32_t>& v) {
    return upload(c, v.data(), v.size());
}
// Several index arrays in one workspace block and one copy (each copy is a
// stream operation that also breaks the programmatic-launch chain).
template <size_t N>
std::array<const int32_t*, N> upload_batch(ffb_context* c, const std::array<const std::vector<int32_t>*, N>& vs) {
    std::array<size_t, N> off{};
    size_t total = 0;
    for (size_t i = 0; i < N; ++i) {
        off[i] = total;
        total += (vs[i]->size() + 3) & ~(size_t)3;  // 16-byte aligned sub-arrays
    }
    std::vector<int32_t> host(std::max<size_t>(total, 1), 0);
    for (size_t i = 0; i < N; ++i) std::copy(vs[i]->begin(), vs[i]->end(), host.begin() + off[i]);
    const int32_t* d = upload(c, host.data(), total);
    std::array<const int32_t*, N> out{};
    for (size_t i = 0; i < N; ++i) out[i] = d + off[i];
    return out;
}

// Device -> host read-back of a small array (a synchronization point).
// Read-back mailbox: a one-CTA kernel (chained behind the producer) copies the
// words into mapped pinned memory, fences at system scope and publishes a
// sequence number the host spins on.  No copy-engine operation and no blocking
// stream sync on the recursion's critical path.
__global__ void __launch_bounds__(1024) k_post(const uint32_t* src, uint32_t* dst, int64_t words,
                                               volatile uint32_t* seq_ptr, uint32_t seq) {
    FFB_PDL_ENTRY();
    // 16-byte stores over the bus where aligned, then one system-scope fence by
    // the publishing thread (cumulative over the block's writes via the barrier)
    const int64_t w4 = ((((uintptr_t)src) & 15) == 0) ? words >> 2 : 0;
    for (int64_t i = threadIdx.x; i < w4; i += blockDim.x)
        reinterpret_cast<uint4*>(dst)[i] = __ldcg(reinterpret_cast<const uint4*>(src) + i);
    for (int64_t i = 4 * w4 + threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldcg(src + i);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *seq_ptr = seq;
    }
}

static bool readback_dma() {
    static const bool dma = getenv("FFB_READBACK_DMA") != nullptr;  // test hook
    return dma;
}

// Reserve the next mailbox sequence number for a kernel that publishes its own
// read-back (MboxPost); empty under FFB_READBACK_DMA.
MboxPost mbox_reserve(ffb_context* c) {
    MboxPost mp;
    if (readback_dma()) return mp;
    mp.dst = c->mbox_dev;
    mp.seq_ptr = c->mbox_seq_dev;
    mp.seq = ++c->mbox_seq;
    return mp;
}

// Spin until the mailbox holds sequence mp.seq (published by k_post or by the
// producing kernel itself); returns the mailbox words.
const void* mbox_wait(ffb_context* c, const MboxPost& mp) {
    const auto t0 = std::chrono::steady_clock::now();
    volatile uint32_t* hs = c->mbox_seq_host;
    for (uint64_t spin = 1; *hs != mp.seq; ++spin)
        if ((spin & 0xFFFF) == 0) {  // surface device faults instead of spinning forever
            const cudaError_t q = cudaStreamQuery(c->stream);
            if (q != cudaSuccess && q != cudaErrorNotReady) FFB_CUDA(q);
        }
    std::atomic_thread_fence(std::memory_order_acquire);
    c->sync_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ++c->syncs;
    c->up_top = 0;  // the publishing kernel ran after every upload issued so far
    return c->mbox_host;
}

const void* readback(ffb_context* c, const void* dev, size_t bytes) {
    const auto t0 = std::chrono::steady_clock::now();
    if (!readback_dma() && bytes <= c->mbox_cap && (bytes & 3) == 0 && (((uintptr_t)dev) & 3) == 0) {
        const MboxPost mp = mbox_reserve(c);
        const int64_t words = (int64_t)(bytes / 4);
        const int threads = (int)std::min<int64_t>(1024, std::max<int64_t>(32, (cdiv(words, 4) + 31) / 32 * 32));
        launch_k(k_post, 1, threads, 0, c->stream, (const uint32_t*)dev, c->mbox_dev, words, c->mbox_seq_dev,
                 mp.seq);
        return mbox_wait(c, mp);
    }
    if (bytes > c->down_cap) {
        if (c->down_host) FFB_CUDA(cudaFreeHost(c->down_host));
        c->down_cap = std::max(bytes, (size_t)1 << 20);
        FFB_CUDA(cudaMallocHost(&c->down_host, c->down_cap));
    }
    FFB_CUDA(cudaMemcpyAsync(c->down_host, dev, bytes, cudaMemcpyDeviceToHost, c->stream)); pdl_fence(c->stream);
    FFB_CUDA(cudaStreamSynchronize(c->stream));
    c->sync_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ++c->syncs;
    c->up_top = 0;  // every upload issued so far has completed
    return c->down_host;
}

__global__ void k_inv_table(uint32_t* t, uint32_t p) {
    FFB_PDL_ENTRY();
    const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < p) t[a] = a ? finv_euclid(p, a) : 0u;
}

// Field constants; an inverse table for p < 2^24 (built once per modulus on
// the device) turns every pivot inverse into one load.
Fp make_field(ffb_context* c, uint64_t p) {
    Fp f = make_fp(p, nullptr);
    if (p < (1ull << 24)) {
        if (c->inv_p != p) {
            if (c->inv_table) FFB_CUDA(cudaFree(c->inv_table));
            c->inv_table = nullptr;
            c->inv_p = 0;
            FFB_CUDA(cudaMalloc(&c->inv_table, p * sizeof(uint32_t)));
            launch_k(k_inv_table, (unsigned)cdiv((int64_t)p, 256), 256, 0, c->stream, c->inv_table, (uint32_t)p);
            FFB_CHECK_LAUNCH();
            FFB_CUDA(cudaStreamSynchronize(c->stream));
            c->inv_p = (uint32_t)p;
        }
        f.inv = c->inv_table;
    }
    return f;
}

// ===========================================================================
// The recursion.
// ===========================================================================
// Y with at most this many rows goes to the one-launch sequential PLDUQ (200:
// measured crossover against the chunked pipeline on config 5).
static int64_t PLDUQ_SEQ_MAX_ROWS =
    getenv("FFB_PLDUQ_SEQ_ROWS") ? atoll(getenv("FFB_PLDUQ_SEQ_ROWS")) : 200;
// The shared-memory sequential kernel (p <= 255, Y as bytes <= 200 KB): rows and pivot cap of
// its speculative use above PLDUQ_SEQ_MAX_ROWS; FFB_PLDUQ_NO_SMEM: off (A/B hook).
static const bool PLDUQ_SMEM_ON = getenv("FFB_PLDUQ_NO_SMEM") == nullptr;
static int64_t PLDUQ_SMEM_MAX_ROWS =
    getenv("FFB_PLDUQ_SMEM_ROWS") ? atoll(getenv("FFB_PLDUQ_SMEM_ROWS")) : 512;
static int PLDUQ_SMEM_RCAP = getenv("FFB_PLDUQ_SMEM_RCAP") ? atoi(getenv("FFB_PLDUQ_SMEM_RCAP")) : 12;

struct HFact {
    std::vector<int32_t> perm;  // image: position -> local input row
    int64_t rank = 0;
};

// Input rows arriving in bands on the copy stream (ffb_ldlt_compact): row r of the
// input view is usable on the engine stream once the band holding it has landed.
struct UploadBands {
    const uint32_t* base = nullptr;
    int64_t ld = 0, rows = 0, ready = 0;      // rows [0, ready) known to be resident
    std::vector<std::pair<int64_t, cudaEvent_t>> ev;  // (band end row, landed)
};

// Schur updates at least this large overlap the zero test / PLDUQ of Y (side stream).
static const int64_t Z_OVERLAP_MIN =
    getenv("FFB_Z_OVERLAP_MIN") ? atoll(getenv("FFB_Z_OVERLAP_MIN")) : 2048;

struct Engine {
    ffb_context* c;
    cudaStream_t st;
    Fp f;
    int variant;
    int64_t T;
    DMat Lg;
    DDiag D;
    UploadBands* bands = nullptr;
    // side stream of the overlapped Schur update (lowest priority) and its events
    cudaStream_t zst = nullptr;
    cudaEvent_t zev_fork = nullptr, zev_done = nullptr;
    bool zpending = false;
    const uint32_t* z_mirrored = nullptr;  // the Z block whose lower part zst already restored
    void z_fork() {
        if (!zst) {
            int least = 0, greatest = 0;
            FFB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            static thread_local cudaStream_t s_zst[FFB_MAX_DEVICES] = {};
            static thread_local cudaEvent_t s_fork[FFB_MAX_DEVICES] = {}, s_done[FFB_MAX_DEVICES] = {};
            const int dev = current_device();
            if (!s_zst[dev]) {
                s_zst[dev] = make_side_stream(least);
                FFB_CUDA(cudaEventCreateWithFlags(&s_fork[dev], cudaEventDisableTiming));
                FFB_CUDA(cudaEventCreateWithFlags(&s_done[dev], cudaEventDisableTiming));
            }
            zst = s_zst[dev];
            zev_fork = s_fork[dev];
            zev_done = s_done[dev];
        }
        FFB_CUDA(cudaEventRecord(zev_fork, st));
        FFB_CUDA(cudaStreamWaitEvent(zst, zev_fork, 0));
        pdl_fence(zst);
    }
    void z_done() {
        FFB_CUDA(cudaEventRecord(zev_done, zst));
        zpending = true;
    }
    // the Schur update running beside the critical path must land before Z is read
    void join_z() {
        if (!zpending) return;
        FFB_CUDA(cudaStreamWaitEvent(st, zev_done, 0));
        pdl_fence(st);
        zpending = false;
    }

    // Before a node touches rows [m, s) of an input-resident A (the Z block): wait for them.
    void ensure_rows(DMat A, int64_t s) {
        if (!bands || bands->ready >= bands->rows) return;
        if (A.ptr < bands->base || A.ptr >= bands->base + bands->rows * bands->ld) return;
        const int64_t need = (A.ptr - bands->base) / bands->ld + s;
        for (auto& be : bands->ev)
            if (be.first > bands->ready && bands->ready < need) {
                FFB_CUDA(cudaStreamWaitEvent(st, be.second, 0));
                pdl_fence(st);
                bands->ready = be.first;
            }
    }

    // Symmetric Schur updates (Z = C - G X, C3 -= Y2^T V1 + V1^T Y2) only need the upper
    // band j >= i - halo of their output: recursive_step reads the upper blocks B and the
    // diagonal blocks, and the leaves / fused nodes read diagonal blocks of <= max(T, 128)
    // rows.  zero_leading_pairs mirrors the strict lower part back before its symmetric
    // gather (mirror_lower).  -1: full updates (FFB_NO_BAND, or very large leaves).
    int band_halo() const {
        static const bool off = getenv("FFB_NO_BAND") != nullptr;  // A/B hook
        if (off || variant == FFB_VARIANT_CROUT) return -1;
        const int64_t t = variant == FFB_VARIANT_RECURSIVE ? 1 : T;
        return t > 1024 ? -1 : (int)std::max<int64_t>(128, t);
    }

    bool is_leaf(int64_t s) const {
        if (variant == FFB_VARIANT_CROUT) return true;
        if (variant == FFB_VARIANT_RECURSIVE) return s <= 1;
        return s <= T || s <= 1;
    }

    // dispatch, sytrf.cpp:337-350
    // rows: original row ids of the node (host); drows: the same on the device
    // (a prefix/suffix of an array the parent uploaded) or nullptr
    HFact dispatch(DMat A, const std::vector<int32_t>& rows, const int32_t* drows, int64_t coff) {
        const int64_t saved = g_node;
        g_node = A.rows;  // trace tag: the innermost node a launch belongs to
        const int64_t teff = variant == FFB_VARIANT_RECURSIVE ? 1 : T;
        HFact h = is_leaf(A.rows)                                ? crout(A, rows, drows, coff)
                  : (variant != FFB_VARIANT_CROUT && node128_supported(f, A.rows, teff))
                      ? node_fused(A, rows, drows, coff)
                      : recursive_step(A, rows, drows, coff);
        g_node = saved;
        return h;
    }

    // crout_base, sytrf.cpp:35-139 (device kernel, one CTA)
    HFact crout(DMat A, const std::vector<int32_t>& rows, const int32_t* drows_in, int64_t coff) {
        const int64_t s = A.rows;
        HFact h;
        if (s == 0) return h;
        ensure_rows(A, s);  // (a leaf at the root of a Crout run reads every row)
        const WsMark mk{c->ws_top};
        const int32_t* drows = drows_in ? drows_in : upload(c, rows);
        int32_t* out = ws_vec<int32_t>(c, s + 1);
        uint32_t* scratch = nullptr;
        if (s > 200) scratch = ws_vec<uint32_t>(c, (int64_t)leaf_scratch_words(s));
        const MboxPost mp = s <= 64 ? mbox_reserve(c) : MboxPost();
        const int32_t* hb = (const int32_t*)(leaf_crout(f, st, A, drows, Lg, coff, D, out, scratch, mp)
                                                 ? mbox_wait(c, mp)
                                                 : readback(c, out, (size_t)(s + 1) * sizeof(int32_t)));
        h.rank = hb[0];
        h.perm.assign(hb + 1, hb + 1 + s);
        c->ws_top = mk.top;
        return h;
    }

    // recursive_step of a node whose children are leaves, fused into one launch
    // (k_node128); when Y != 0 the kernel hands over after the Schur updates and the
    // host continues with zero_leading_pairs exactly as recursive_step would.
    HFact node_fused(DMat A, const std::vector<int32_t>& rows, const int32_t* drows_in, int64_t coff) {
        const int64_t s = A.rows, m = s / 2, ns = s - m;
        ensure_rows(A, s);
        const WsMark mk{c->ws_top};
        const int32_t* drows = drows_in ? drows_in : upload(c, rows);
        int32_t* out = ws_vec<int32_t>(c, s + 2);
        uint32_t* yout = ws_vec<uint32_t>(c, m * ns);
        const MboxPost mp = mbox_reserve(c);
        node128(f, st, A, drows, Lg, coff, D, yout, out, mp);
        const int32_t* hb = (const int32_t*)(mp.dst ? mbox_wait(c, mp)
                                                     : readback(c, out, (size_t)(s + 2) * sizeof(int32_t)));
        HFact h;
        if (hb[0] == 0) {
            h.rank = hb[1];
            h.perm.assign(hb + 2, hb + 2 + s);
            c->ws_top = mk.top;
            return h;
        }
        const int64_t r1 = hb[1];
        std::vector<int32_t> perm1(hb + 2, hb + 2 + m);
        std::vector<int32_t> rowsz;  // rows of [[0 Y],[Y^t Z]] (sytrf.cpp:317)
        rowsz.reserve(s - r1);
        for (int64_t i = r1; i < m; ++i) rowsz.push_back(rows[perm1[i]]);
        for (int64_t i = m; i < s; ++i) rowsz.push_back(rows[i]);
        DMat Y;
        Y.ptr = yout;
        Y.ld = ns;
        Y.rows = m - r1;
        Y.cols = ns;
        HFact f2 = zero_leading_pairs(Y, A.sub(m, m, ns, ns), rowsz, coff + r1);
        h.rank = r1 + f2.rank;  // (:332-334)
        h.perm.resize(s);
        for (int64_t pos = 0; pos < r1; ++pos) h.perm[pos] = perm1[pos];
        for (int64_t pos = r1; pos < s; ++pos) {
            const int64_t cix = f2.perm[pos - r1];
            h.perm[pos] = cix < m - r1 ? perm1[r1 + cix] : (int32_t)(m + (cix - (m - r1)));
        }
        c->ws_top = mk.top;
        return h;
    }

    // Alg. 2, sytrf.cpp:298-335
    HFact recursive_step(DMat A, const std::vector<int32_t>& rows, const int32_t* drows, int64_t coff) {
        const int64_t s = A.rows, m = s / 2, ns = s - m;
        const WsMark mk{c->ws_top};
        std::vector<int32_t> rows1(rows.begin(), rows.begin() + m);
        phase_mark("rs: begin", s, st);
        HFact f1 = dispatch(A.sub(0, 0, m, m), rows1, drows, coff);  // :303
        const int64_t r1 = f1.rank;
        phase_mark("rs: A1 factored", s, st);

        // B' = P1^T B (:308) and [L1; M1] in f1's position order (from Lg), one launch
        DMat BP = ws_mat(c, m, ns);
        std::vector<int32_t> prow(m);
        for (int64_t i = 0; i < m; ++i) prow[i] = rows[f1.perm[i]];
        std::vector<int32_t> rows2(rows.begin() + m, rows.end());
        std::vector<int32_t> rowsz;  // rows of [[0 Y],[Y^t Z]]
        rowsz.reserve(s - r1);
        for (int64_t i = r1; i < m; ++i) rowsz.push_back(prow[i]);
        for (int64_t i = m; i < s; ++i) rowsz.push_back(rows[i]);
        // every index array of this node in one copy
        const auto up = upload_batch<4>(c, {&f1.perm, &prow, &rows2, &rowsz});
        DMat LM = ws_mat(c, m, r1);
        gather_rows2(st, BP, A, up[0], m, LM, Lg, up[1], coff);
        DMat X = BP.sub(0, 0, r1, ns);
        phase_mark("rs: B' gathered", s, st);
        trsm_lower_unit(f, st, LM.sub(0, 0, r1, r1), X);  // :310
        phase_mark("rs: X = L1^-1 B'", s, st);
        DMat Y = BP.sub(r1, 0, m - r1, ns);
        DMat G = ws_mat(c, ns, r1);
        DMat Z = A.sub(m, m, ns, ns);
        ensure_rows(A, s);  // Z and the recursion below read rows [m, s)
        // Large node with Y != empty: zero_leading's zero test and PLDUQ need Y only, so
        // G and the Schur update Z = C - G X run on a low-priority side stream beside
        // them; Z's consumers join first (join_z)
        static const bool z_overlap_on = getenv("FFB_NO_Z_OVERLAP") == nullptr;
        if (z_overlap_on && ns >= Z_OVERLAP_MIN && r1 > 0 && m - r1 > 0 && !zpending) {
            gemm(f, st, GEMM_SUB, Y, LM.sub(r1, 0, m - r1, r1), false, X, false, m - r1, ns, r1);  // :312
            {
                GreenScope green(true);  // zst lives in the SM partition of the bulk updates
                z_fork();
                SlotGuard slot(2);
                g_tc_shared_sms = true;
                inverse_apply_T(f, zst, G, X, D, coff, Lg, up[2]);  // :313 + rows m..s of N1
                BandScope band(band_halo());
                gemm(f, zst, GEMM_SUB, Z, G, false, X, false, ns, ns, r1);  // :315
                g_tc_shared_sms = false;
                // zero_leading_pairs' symmetric gather reads the lower part too: mirror it
                // back here, beside Y's zero test and PLDUQ
                if (band_halo() >= 0) {
                    mirror_lower(zst, Z, band_halo());
                    z_mirrored = Z.ptr;
                }
                z_done();
            }
            phase_mark("rs: Y updated, Z forked", s, st);
            HFact f2 = zero_leading(Y, Z, rowsz, up[3], coff + r1, 0);  // :317
            phase_mark("rs: zero_leading done", s, st);
            join_z();
            z_mirrored = nullptr;
            HFact h;  // (:332-334)
            h.rank = r1 + f2.rank;
            h.perm.resize(s);
            for (int64_t pos = 0; pos < r1; ++pos) h.perm[pos] = f1.perm[pos];
            for (int64_t pos = r1; pos < s; ++pos) {
                const int64_t cix = f2.perm[pos - r1];
                h.perm[pos] = cix < m - r1 ? f1.perm[r1 + cix] : (int32_t)(m + (cix - (m - r1)));
            }
            c->ws_top = mk.top;
            return h;
        }
        inverse_apply_T(f, st, G, X, D, coff, Lg, up[2]);  // :313 + rows m..s of N1
        // Y = B'' - M1 X (:312) and Z = C - G X (:315); small ones as one paired launch
        // whose Y epilogue also answers the zero test of zero_leading
        int32_t ytag = 0;
        if (r1 > 0 && m - r1 > 0) {
            const int32_t tag = (int32_t)(++c->zero_gen);
            if (mma_gemm_pair(f, st, Y, LM.sub(r1, 0, m - r1, r1), X, m - r1, ns, r1, Z, G, X, ns, ns, r1,
                              c->zero_flag, tag))
                ytag = tag;
        }
        if (!ytag) {
            gemm(f, st, GEMM_SUB, Y, LM.sub(r1, 0, m - r1, r1), false, X, false, m - r1, ns, r1);
            BandScope band(band_halo());
            gemm(f, st, GEMM_SUB, Z, G, false, X, false, ns, ns, r1);
        }

        HFact f2 = zero_leading(Y, Z, rowsz, up[3], coff + r1, ytag);  // :317

        HFact h;  // P = compose(embed(P1,0,n), embed(P2,r1,n)) (:332-334)
        h.rank = r1 + f2.rank;
        h.perm.resize(s);
        for (int64_t pos = 0; pos < r1; ++pos) h.perm[pos] = f1.perm[pos];
        for (int64_t pos = r1; pos < s; ++pos) {
            const int64_t cix = f2.perm[pos - r1];
            h.perm[pos] = cix < m - r1 ? f1.perm[r1 + cix] : (int32_t)(m + (cix - (m - r1)));
        }
        c->ws_top = mk.top;
        return h;
    }

    bool is_zero(DMat Y, int32_t pretag = 0) {
        // generation tag instead of a memset: the flag holds an older tag unless Y != 0
        // (pretag: the producing GEMM already tagged the flag)
        const int32_t tag = pretag ? pretag : (int32_t)(++c->zero_gen);
        if (!pretag) any_nonzero(st, Y, c->zero_flag, tag);
        const int32_t v = *(const int32_t*)readback(c, c->zero_flag, sizeof(int32_t));
        return v != tag;
    }

    // sytrf.cpp:267-292
    HFact zero_leading(DMat Y, DMat Z, const std::vector<int32_t>& rows, const int32_t* drows, int64_t coff,
                       int32_t ytag = 0) {
        const int64_t m = Y.rows, nz = Z.rows;
        if (m == 0) {
            join_z();
            return dispatch(Z, rows, drows, coff);
        }
        HFact h;
        if (nz == 0) {
            h.perm.resize(m);
            for (int64_t i = 0; i < m; ++i) h.perm[i] = (int32_t)i;
            return h;
        }
        if (is_zero(Y, ytag)) {  // :274-290
            join_z();
            z_mirrored = nullptr;
            std::vector<int32_t> rz(rows.begin() + m, rows.end());
            HFact f3 = dispatch(Z, rz, drows ? drows + m : nullptr, coff);
            const int64_t r3 = f3.rank;
            h.rank = r3;
            h.perm.resize(m + nz);
            for (int64_t k = 0; k < r3; ++k) h.perm[k] = (int32_t)(m + f3.perm[k]);
            for (int64_t t = 0; t < m; ++t) h.perm[r3 + t] = (int32_t)t;
            for (int64_t k = r3; k < nz; ++k) h.perm[m + k] = (int32_t)(m + f3.perm[k]);
            return h;
        }
        return zero_leading_pairs(Y, Z, rows, coff);  // (device rows rebuilt from the PLDUQ perms)
    }

    // PLDUQ of Y (destroyed); returns rank, fills row/col images and device factors.
    struct Pl {
        int64_t r;
        std::vector<int32_t> rimg, cimg;
        DMat L, U;
        uint32_t *d, *dinv;
    };
    double pq_t0 = 0;
    Pl run_plduq(DMat Y, const std::function<void(const std::vector<int32_t>&)>& pivots_ready = {}) {
        const int64_t m = Y.rows, n = Y.cols, mn = std::min(m, n);
        static const bool pq_pdl = getenv("FFB_PDL_NO_PLDUQ") == nullptr;  // bisection hook
        PdlScope pdl_scope(pq_pdl);
        Pl pl;
        if (getenv("FFB_PLDUQ_TRACE")) {
            FFB_CUDA(cudaStreamSynchronize(st));
            pq_t0 = std::chrono::duration<double, std::milli>(
                        std::chrono::steady_clock::now().time_since_epoch()).count();
        }
        // NVTX range around large PLDUQs (profiling filter; no-op without a tool)
        struct Range {
            bool on;
            explicit Range(bool b) : on(b) { if (on) nvtxRangePushA("plduq_big"); }
            ~Range() { if (on) nvtxRangePop(); }
        } range(m * n >= (int64_t)1 << 24);
        DMat Lo = ws_mat(c, m, mn), Uo = ws_mat(c, mn, n);
        pl.d = ws_vec<uint32_t>(c, mn);
        pl.dinv = ws_vec<uint32_t>(c, mn);
        auto take_seq = [&](const int32_t* hb, bool has_dinv) {
            pl.r = hb[0];
            pl.rimg.assign(hb + 1, hb + 1 + m);
            pl.cimg.assign(hb + 1 + m, hb + 1 + m + n);
            if (!has_dinv) invert_vec(f, st, pl.dinv, pl.d, pl.r);
        };
        // p <= 255 and Y fits shared memory as bytes: the sequential elimination there costs ~ its
        // rank, not its rows.  Short Y always; taller Y (up to PLDUQ_SMEM_MAX_ROWS) with a cap on the
        // pivots -- the kernel only reads Y, so past the cap the chunked pipeline starts from scratch.
        bool seq_done = false;
        if (m <= PLDUQ_SMEM_MAX_ROWS && PLDUQ_SMEM_ON) {
            const WsMark mk{c->ws_top};
            int32_t* info = ws_vec<int32_t>(c, 1 + m + n + mn);
            const int rcap = m <= PLDUQ_SEQ_MAX_ROWS ? (int)mn : PLDUQ_SMEM_RCAP;
            if (plduq_smem(f, st, Y, info, Lo, pl.d, pl.dinv, Uo, rcap)) {
                const int32_t* hb = (const int32_t*)readback(c, info, (size_t)(1 + m + n) * sizeof(int32_t));
                if (hb[0] >= 0) {
                    take_seq(hb, true);
                    seq_done = true;
                }
            }
            if (!seq_done) c->ws_top = mk.top;
        }
        if (seq_done) {
        } else if (m <= PLDUQ_SEQ_MAX_ROWS) {
            // short Y: one launch of the row-sequential kernel
            int32_t* info = ws_vec<int32_t>(c, 1 + m + n + mn);
            int32_t* colflag = ws_vec<int32_t>(c, n);
            uint32_t* lvec = ws_vec<uint32_t>(c, m);
            plduq(f, st, Y, info, colflag, lvec, Lo, pl.d, Uo);
            take_seq((const int32_t*)readback(c, info, (size_t)(1 + m + n) * sizeof(int32_t)), false);
        } else {
            Workspace ws{c->ws_base, c->ws_cap, &c->ws_top};
            PlduqIO io;
            io.upload = [this](const std::vector<int32_t>& v) { return upload(c, v); };
            io.readback = [this](const void* p, size_t b) { return readback(c, p, b); };
            io.post = [this]() { return mbox_reserve(c); };
            io.wait = [this](const MboxPost& mp) { return mbox_wait(c, mp); };
            io.pivots_ready = pivots_ready;
            io.Lo = Lo;
            io.Uo = Uo;
            io.d = pl.d;
            io.dinv = pl.dinv;
            const size_t mk = c->ws_top;
            PlduqOut o = plduq_parallel(f, st, Y, ws, io);
            c->ws_top = mk;
            pl.r = o.r;
            pl.rimg = std::move(o.rimg);
            pl.cimg = std::move(o.cimg);
        }
        pl.L = Lo.sub(0, 0, m, pl.r);
        pl.U = Uo.sub(0, 0, pl.r, n);
        static FILE* tr = getenv("FFB_PLDUQ_TRACE") ? fopen(getenv("FFB_PLDUQ_TRACE"), "a") : nullptr;
        if (tr) {  // shape + wall time of each PLDUQ (diagnostics; synchronizes)
            FFB_CUDA(cudaStreamSynchronize(st));
            const double t1 = std::chrono::duration<double, std::milli>(
                                  std::chrono::steady_clock::now().time_since_epoch()).count();
            fprintf(tr, "%lld %lld %lld %.3f\n", (long long)m, (long long)n, (long long)pl.r, t1 - pq_t0);
            fflush(tr);
        }
        return pl;
    }

    // Solve X^T U1 + U1^T X = C1 for upper X (Alg. 1, trssyr2k.cpp) in closed
    // form: Ct = U1^-T C1 U1^-1, Y = strict_upper(Ct) + diag(Ct)/2, X = Y U1.
    // The solution is unique for odd p (and unique with zero diagonal for
    // p = 2), so it equals the reference's halving recursion.  X -> Xout.
    void trssyr2k_dev(DMat U1, DMat U1T, DMat C1, DMat Xout, int32_t* flag) {
        const int64_t r = U1.rows;
        if (r == 0) return;
        const WsMark mk{c->ws_top};
        trsm_lower_unit(f, st, U1T, C1);  // W = U1^-T C1 (in place)
        DMat Wt = ws_mat(c, r, r);
        transpose(st, Wt, C1);
        trsm_lower_unit(f, st, U1T, Wt);  // Ct = U1^-T W^T
        trssyr2k_mid(f, st, Wt, flag);
        gemm(f, st, GEMM_SET, Xout, Wt, false, U1, false, r, r, r);
        c->ws_top = mk.top;
    }

    // Alg. 3, sytrf.cpp:170-265
    HFact zero_leading_pairs(DMat Y, DMat Z, const std::vector<int32_t>& rows, int64_t coff) {
        const int64_t m = Y.rows, nz = Z.rows;
        const WsMark mk{c->ws_top};
        DMat Cp = ws_mat(c, nz, nz);  // C' = Q^T Z Q (:183)
        int32_t* dq = ws_vec<int32_t>(c, nz);  // Q for the early gather (outside the PLDUQ's workspace)
        // C' needs only Q = the PLDUQ's column image: once the pivots are known it is
        // gathered on the Schur-update stream (after Z's update, mirrored back when
        // band-only), beside the PLDUQ's factor phase on the engine stream
        static const bool cp_overlap = getenv("FFB_NO_CP_OVERLAP") == nullptr;  // A/B hook
        bool cp_done = false;
        auto on_pivots = [&](const std::vector<int32_t>& qimg) {
            upload_into(c, dq, qimg.data(), qimg.size());
            z_fork();
            GreenScope green(true);
            if (band_halo() >= 0 && z_mirrored != Z.ptr) mirror_lower(zst, Z, band_halo());
            z_mirrored = Z.ptr;
            gather_sym(zst, Cp, Z, dq);
            z_done();
            cp_done = true;
        };
        phase_mark("zlp: begin", m + nz, st);
        Pl py = cp_overlap ? run_plduq(Y, on_pivots) : run_plduq(Y);  // :175
        phase_mark("zlp: plduq done", m + nz, st);
        const int64_t r = py.r;
        const std::vector<int32_t>& q = py.cimg;

        // L columns [coff, coff + 2r) (:222-252) are keyed by original row:
        //   Y rows (row_perm order), Z rows (col_perm order); all index arrays in one copy
        std::vector<int32_t> idy(m), idz(nz);
        for (int64_t a = 0; a < m; ++a) idy[a] = rows[py.rimg[a]];
        for (int64_t a = 0; a < nz; ++a) idz[a] = rows[m + q[a]];
        const auto up = upload_batch<3>(c, {&q, &idy, &idz});
        join_z();
        if (!cp_done) {
            if (band_halo() >= 0 && z_mirrored != Z.ptr) mirror_lower(st, Z, band_halo());  // band-only update
            gather_sym(st, Cp, Z, up[0]);
        }
        z_mirrored = nullptr;
        DMat C1 = Cp.sub(0, 0, r, r), C2 = Cp.sub(0, r, r, nz - r), C3 = Cp.sub(r, r, nz - r, nz - r);
        DMat U1 = py.U.sub(0, 0, r, r), V1 = py.U.sub(0, r, r, nz - r);
        DMat UpT = ws_mat(c, nz, r);  // [U1^T; V1^T]
        transpose(st, UpT, py.U);
        DMat U1T = UpT.sub(0, 0, r, r);

        uint32_t* delta = nullptr;
        if (f.char2) {  // :188-200
            delta = ws_vec<uint32_t>(c, r);
            char2_delta(f, st, C1, U1, delta);
            DMat H = ws_mat(c, r, r);
            scale_rows(f, st, H, U1, delta);
            gemm(f, st, GEMM_SUB, C1, H, true, U1, false, r, r, r);  // C1 -= U1^T diag(delta) U1
        }
        DMat X = ws_mat(c, r, r);
        if (f.char2) fill_words(st, (uint32_t*)c->flag, 1, 0u);  // (only characteristic 2 writes the flag)
        phase_mark("zlp: C' ready, U^T", m + nz, st);
        trssyr2k_dev(U1, U1T, C1, X, c->flag);  // :202
        phase_mark("zlp: trssyr2k", m + nz, st);
        DMat G12 = ws_mat(c, nz, r);  // [G1; G2]
        scale_T(f, st, G12.sub(0, 0, r, r), X, py.dinv);  // G1 = (diag(d)^-1 X)^T (:203)
        if (f.char2) add_scaled_rows_upper(f, st, X, U1, delta);  // X += Delta U1 (:204-208)
        gemm(f, st, GEMM_SUB, C2, X, true, V1, false, r, nz - r, r);  // C2 -= X^T V1 (:210)
        trsm_lower_unit(f, st, U1T, C2);  // Y2 = U1^-T C2 (:211)
        phase_mark("zlp: C2, Y2", m + nz, st);
        {
            BandScope band(band_halo());  // C3 is symmetric and read like Z
            // C3 -= Y2^T V1 + V1^T Y2 (:213), both terms into one accumulator
            gemm2(f, st, GEMM_SUB, C3, C2, true, V1, false, V1, true, C2, false, nz - r, nz - r, r, r);
            if (f.char2) {  // :214
                DMat H = ws_mat(c, r, nz - r);
                scale_rows(f, st, H, V1, delta);
                gemm(f, st, GEMM_SUB, C3, H, true, V1, false, nz - r, nz - r, r);
            }
        }
        scale_T(f, st, G12.sub(r, 0, nz - r, r), C2, py.dinv);  // G2 (:215)

        //   Y rows (row_perm order):  even columns <- [L1; M1]
        //   Z rows (col_perm order):  even <- [G1; G2], odd <- [U1^T; V1^T]
        const int32_t* didz = up[2];
        if (!zlp_scatter(st, Lg, coff, up[1], py.L, didz, G12, UpT, D, py.d, py.dinv, delta, r)) {
            scatter_lg(st, Lg, up[1], coff, 2, py.L);
            scatter_lg_pair(st, Lg, didz, coff, G12, UpT);  // even <- [G1; G2], odd <- [U1^T; V1^T]
            write_pair_diag(f, st, D, coff, py.d, py.dinv, delta, r);  // :254-260
        }

        std::vector<int32_t> rows3(idz.begin() + r, idz.end());
        phase_mark("zlp: C3 updated, L scattered", m + nz, st);
        HFact f3 = dispatch(C3, rows3, didz + r, coff + 2 * r);  // :217
        phase_mark("zlp: C3 factored", m + nz, st);
        const int64_t r3 = f3.rank;

        HFact h;  // P_i interleave + rotations (:226-251)
        h.rank = 2 * r + r3;
        h.perm.resize(m + nz);
        for (int64_t i = 0; i < r; ++i) {
            h.perm[2 * i] = py.rimg[i];
            h.perm[2 * i + 1] = (int32_t)(m + q[i]);
        }
        for (int64_t k = 0; k < nz - r; ++k) {
            const int64_t row = k < r3 ? 2 * r + k : 2 * r + (m - r) + k;
            h.perm[row] = (int32_t)(m + q[r + f3.perm[k]]);
        }
        for (int64_t t = 0; t < m - r; ++t) h.perm[2 * r + r3 + t] = py.rimg[r + t];
        c->ws_top = mk.top;
        return h;
    }
};

// Estimated workspace for an n x n factorization (W, Lg, D, recursion temps).
size_t workspace_bytes(int64_t n) {
    const size_t n2 = (size_t)n * n * sizeof(uint32_t);
    return 12 * n2 + 64 * (size_t)n * sizeof(uint32_t) + ((size_t)256 << 20);
}

int set_error(const std::exception& e) {
    g_last_error = e.what();
    if (const Status* s = dynamic_cast<const Status*>(&e)) return s->code;
    if (dynamic_cast<const std::bad_alloc*>(&e)) return FFB_NO_MEMORY;
    return FFB_ERROR;
}

template <class F>
int guarded(ffb_context* c, F&& fn) {
    try {
        if (!c) throw Status(FFB_ERROR, "null context");
        FFB_CUDA(cudaSetDevice(c->device));
        // every kernel goes through launch_k, which numbers them (pdl_launch_index)
        const uint64_t l0 = (uint64_t)pdl_launch_index(), s0 = c->syncs, u0 = c->uploads;
        const auto t0 = std::chrono::steady_clock::now();
        const double w0 = c->sync_wait_ms;
        g_prof = &c->prof;
        fn();
        static const bool host_stats = getenv("FFB_HOST_STATS") != nullptr;
        if (host_stats) {  // host-side balance: wall vs time blocked on the device
            FFB_CUDA(cudaStreamSynchronize(c->stream));
            const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            fprintf(stderr, "[ffb host] wall %.2f ms, blocked in %llu read-backs %.2f ms, launches %llu, uploads %llu\n",
                    wall, (unsigned long long)(c->syncs - s0), c->sync_wait_ms - w0,
                    (unsigned long long)((uint64_t)pdl_launch_index() - l0), (unsigned long long)(c->uploads - u0));
        }
        if (c->prof.on) {
            FFB_CUDA(cudaStreamSynchronize(c->stream));
            c->prof.flush();
        }
        g_prof = nullptr;
        c->launches = (uint64_t)pdl_launch_index() - l0;
        c->syncs_last = c->syncs - s0;
        g_last_error.clear();
        return FFB_OK;
    } catch (const std::exception& e) {
        g_prof = nullptr;
        if (c) {
            c->prof.recs.clear();
            cudaStreamSynchronize(c->stream);
            c->ws_top = 0;
            c->up_top = 0;
        }
        return set_error(e);
    }
}

struct DevFact {
    int64_t n = 0, rank = 0;
    std::vector<int32_t> perm;
    DMat Lg;
    DDiag D;
};

// Run the factorization of the n x n device matrix W (destroyed).
DevFact run_ldlt(ffb_context* c, const Fp& f, DMat W, int variant, int64_t threshold,
                 bool check_symmetric, UploadBands* bands = nullptr) {
    const int64_t n = W.rows;
    cudaStream_t st = c->stream;
    DevFact out;
    out.n = n;
    if (check_symmetric) {  // ldlt validation, sytrf.cpp:355-356
        fill_words(st, (uint32_t*)c->flag, 1, 0u);
        any_asymmetric(st, W, c->flag);
        if (*(const int32_t*)readback(c, c->flag, sizeof(int32_t)))
            throw Status(FFB_NOT_SYMMETRIC, "ldlt: matrix must be symmetric");
    }
    out.Lg = ws_mat(c, n, n);
    zero_mat(st, out.Lg);
    out.D.kind = ws_vec<int32_t>(c, n);
    out.D.val = ws_vec<uint32_t>(c, n);
    out.D.val2 = ws_vec<uint32_t>(c, n);
    out.D.inv = ws_vec<uint32_t>(c, n);
    Engine e{c, st, f, variant, (int64_t)threshold, out.Lg, out.D};
    e.bands = bands;
    std::vector<int32_t> rows(n);
    for (int64_t i = 0; i < n; ++i) rows[i] = (int32_t)i;
    if (n > 0) {
        HFact h = e.dispatch(W, rows, upload(c, rows), 0);
        phase_dump(st);
        out.rank = h.rank;
        out.perm = std::move(h.perm);
    }
    return out;
}

// Copy a device factorization to caller host buffers (uint64 element type).
void export_host(ffb_context* c, const DevFact& df, int64_t* perm, void* lower, int lower_eb,
                 int32_t* dkind, uint64_t* dval, uint64_t* dval2, size_t* rank) {
    cudaStream_t st = c->stream;
    const int64_t n = df.n, r = df.rank;
    for (int64_t i = 0; i < n; ++i) perm[i] = df.perm[i];
    *rank = (size_t)r;
    if (n == 0) return;
    if (r > 0) {
        DMat Lout = ws_mat(c, n, r);
        const int32_t* dperm = upload(c, df.perm);
        void* dl = ws_alloc(c, (size_t)n * r * lower_eb);
        // row bands: gather + convert on the engine stream, each band's copy to the
        // host on the copy stream while the next band is gathered
        const int64_t nb = n >= 4096 ? 8 : 1, step = cdiv(n, nb);
        std::vector<cudaEvent_t> evs;
        for (int64_t r0 = 0; r0 < n; r0 += step) {
            const int64_t nr = std::min<int64_t>(step, n - r0);
            gather_lower_out(st, Lout.sub(r0, 0, nr, r), df.Lg, dperm + r0);
            char* dband = (char*)dl + (size_t)r0 * r * lower_eb;
            convert_out(st, dband, lower_eb, Lout.sub(r0, 0, nr, r));
            if (nb == 1) {
                FFB_CUDA(cudaMemcpyAsync(lower, dl, (size_t)n * r * lower_eb, cudaMemcpyDeviceToHost, st));
                pdl_fence(st);
                break;
            }
            cudaEvent_t ev;
            FFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            FFB_CUDA(cudaEventRecord(ev, st));
            evs.push_back(ev);
            FFB_CUDA(cudaStreamWaitEvent(c->copy_stream, ev, 0));
            FFB_CUDA(cudaMemcpyAsync((char*)lower + (size_t)r0 * r * lower_eb, dband, (size_t)nr * r * lower_eb,
                                     cudaMemcpyDeviceToHost, c->copy_stream));
        }
        if (!evs.empty()) {
            FFB_CUDA(cudaStreamSynchronize(c->copy_stream));
            for (auto ev : evs) cudaEventDestroy(ev);
        }
        std::vector<int32_t> k(r);
        std::vector<uint32_t> v(r), v2(r);
        FFB_CUDA(cudaMemcpyAsync(k.data(), df.D.kind, r * sizeof(int32_t), cudaMemcpyDeviceToHost, st)); pdl_fence(st);
        FFB_CUDA(cudaMemcpyAsync(v.data(), df.D.val, r * sizeof(uint32_t), cudaMemcpyDeviceToHost, st)); pdl_fence(st);
        FFB_CUDA(cudaMemcpyAsync(v2.data(), df.D.val2, r * sizeof(uint32_t), cudaMemcpyDeviceToHost, st)); pdl_fence(st);
        FFB_CUDA(cudaStreamSynchronize(st));
        for (int64_t t = 0; t < r; ++t) {
            dkind[t] = k[t];
            dval[t] = v[t];
            dval2[t] = v2[t];
        }
    }
}

// Upload a host matrix (elem bytes eb, dense rows x cols) into a fresh device view.
DMat upload_matrix(ffb_context* c, const Fp& f, const void* h, int64_t rows, int64_t cols, int eb) {
    DMat m = ws_mat(c, rows, cols);
    if (rows * cols == 0) return m;
    const size_t bytes = (size_t)rows * cols * eb;
    void* tmp = ws_alloc(c, bytes);
    FFB_CUDA(cudaMemcpyAsync(tmp, h, bytes, cudaMemcpyHostToDevice, c->stream)); pdl_fence(c->stream);
    convert_in(f, c->stream, m, tmp, eb);
    return m;
}

void download_matrix(ffb_context* c, DMat m, uint64_t* h) {
    if (m.rows * m.cols == 0) return;
    void* tmp = ws_alloc(c, (size_t)m.rows * m.cols * 8);
    convert_out(c->stream, tmp, 8, m);
    FFB_CUDA(cudaMemcpyAsync(h, tmp, (size_t)m.rows * m.cols * 8, cudaMemcpyDeviceToHost, c->stream)); pdl_fence(c->stream);
    FFB_CUDA(cudaStreamSynchronize(c->stream));
}

int elem_bytes(int t) {
    if (t == FFB_U8 || t == FFB_U16 || t == FFB_U32 || t == FFB_U64) return t;
    throw Status(FFB_ERROR, "unknown element type");
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int ffb_version(void) { return 1; }

const char* ffb_status_string(int s) {
    switch (s) {
    case FFB_OK: return "OK";
    case FFB_DIMENSION_MISMATCH: return "DimensionMismatch";
    case FFB_NOT_SYMMETRIC: return "NotSymmetric";
    case FFB_NOT_PRIME: return "NotPrime";
    case FFB_ZERO_INVERSE: return "ZeroInverse";
    case FFB_CHAR_TWO_DIVISION: return "CharTwoDivision";
    case FFB_NON_UNIT_TRIANGULAR: return "NonUnitTriangular";
    case FFB_SINGULAR_TRIANGULAR: return "SingularTriangular";
    case FFB_CHAR_TWO_NONZERO_DIAGONAL: return "CharTwoNonzeroDiagonal";
    case FFB_BAD_BLOCK_SIZES: return "BadBlockSizes";
    case FFB_NO_MEMORY: return "NoMemory";
    case FFB_CUDA_ERROR: return "CudaError";
    case FFB_UNSUPPORTED: return "Unsupported";
    case FFB_WRONG_CHARACTERISTIC: return "WrongCharacteristic";
    case FFB_PARSE_ERROR: return "ParseError";
    default: return "Error";
    }
}

const char* ffb_last_error(void) { return g_last_error.c_str(); }

int ffb_create(ffb_context** out, int device) {
    try {
        ffb_context* c = new ffb_context();
        c->device = device;
        FFB_CUDA(cudaSetDevice(device));
        {  // the recursion's critical path: highest stream priority (side streams use the lowest)
            int least = 0, greatest = 0;
            FFB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            FFB_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, greatest));
        }
        c->up_cap = (size_t)64 << 20;
        {
            void* h = nullptr;
            FFB_CUDA(cudaHostAlloc(&h, c->up_cap, cudaHostAllocMapped));
            c->up_host = (char*)h;
            void* d = nullptr;
            FFB_CUDA(cudaHostGetDevicePointer(&d, h, 0));
            c->up_dev = (const char*)d;
        }
        c->down_cap = (size_t)16 << 20;
        FFB_CUDA(cudaMallocHost(&c->down_host, c->down_cap));
        {  // read-back mailbox: 256 KB of data + a sequence word, mapped pinned
            c->mbox_cap = (size_t)256 << 10;
            void* h = nullptr;
            FFB_CUDA(cudaHostAlloc(&h, c->mbox_cap + 256, cudaHostAllocMapped));
            c->mbox_host = (uint32_t*)h;
            c->mbox_seq_host = (volatile uint32_t*)((char*)h + c->mbox_cap);
            *c->mbox_seq_host = 0;
            void* d = nullptr;
            FFB_CUDA(cudaHostGetDevicePointer(&d, h, 0));
            c->mbox_dev = (uint32_t*)d;
            c->mbox_seq_dev = (uint32_t*)((char*)d + c->mbox_cap);
        }
        {
            int least = 0, greatest = 0;
            FFB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            FFB_CUDA(cudaStreamCreateWithPriority(&c->copy_stream, cudaStreamNonBlocking, least));
        }
        FFB_CUDA(cudaMalloc(&c->flag, 256));
        FFB_CUDA(cudaMemset(c->flag, 0, 256));
        c->zero_flag = c->flag + 32;
        *out = c;
        return FFB_OK;
    } catch (const std::exception& e) {
        *out = nullptr;
        return set_error(e);
    }
}

int ffb_destroy(ffb_context* c) {
    if (!c) return FFB_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->ws_base) cudaFree(c->ws_base);
    if (c->inv_table) cudaFree(c->inv_table);
    if (c->flag) cudaFree(c->flag);
    if (c->mbox_host) cudaFreeHost(c->mbox_host);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->up_host) cudaFreeHost(c->up_host);
    if (c->down_host) cudaFreeHost(c->down_host);
    cudaStreamDestroy(c->stream);
    delete c;
    return FFB_OK;
}

void* ffb_stream(ffb_context* c) { return c ? (void*)c->stream : nullptr; }
uint64_t ffb_sync_count(ffb_context* c) { return c ? c->syncs_last : 0; }

int ffb_profile_enable(ffb_context* c, int on) {
    if (!c) return FFB_ERROR;
    c->prof.on = on != 0;
    c->prof.reset();
    return FFB_OK;
}

int ffb_profile_read(ffb_context* c, int klass, uint64_t* launches, double* ms, double* ops,
                     double* bytes) {
    if (!c || klass < 0 || klass >= K_NCLASS) return FFB_ERROR;
    *launches = c->prof.cnt[klass];
    *ms = c->prof.ms[klass];
    *ops = c->prof.ops[klass];
    *bytes = c->prof.bytes[klass];
    return FFB_OK;
}
uint64_t ffb_launch_count(ffb_context* c) { return c ? c->launches : 0; }

int ffb_ldlt_compact(ffb_context* c, uint64_t p, size_t n, const void* a, int a_type, int variant,
                     size_t threshold, int64_t* perm, void* lower, int lower_type, int32_t* dkind,
                     uint64_t* dval, uint64_t* dval2, size_t* rank) {
    return guarded(c, [&] {
        check_modulus(p);
        const int aeb = elem_bytes(a_type), leb = elem_bytes(lower_type);
        ensure_workspace(c, workspace_bytes((int64_t)n) + (size_t)n * n * (aeb + leb));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        if (n < 4096 || getenv("FFB_NO_BANDS")) {
            DMat W = upload_matrix(c, f, a, (int64_t)n, (int64_t)n, aeb);
            DevFact df = run_ldlt(c, f, W, variant, (int64_t)threshold, true);
            export_host(c, df, perm, lower, leb, dkind, dval, dval2, rank);
            c->ws_top = 0;
            return;
        }
        // Large n: the input arrives in row bands (n/16, n/8, n/4, n/2, n) on the copy
        // stream, converted as it lands; the recursion starts on the first band and
        // waits for later rows only where a node first reads them (Engine::ensure_rows).
        // The engine reads only the upper blocks B and Z, so an asymmetric input factors
        // harmlessly as another symmetric matrix; the check runs on the copy stream
        // after the last band and the result is refused (NotSymmetric) before export.
        // It reads the raw staging buffer `tmp`, which the engine never writes (W is
        // updated in place by the recursion, concurrently with the check).
        const int64_t N = (int64_t)n;
        DMat W = ws_mat(c, N, N);
        char* tmp = (char*)ws_alloc(c, (size_t)N * N * aeb);
        UploadBands bands;
        bands.base = W.ptr;
        bands.ld = W.ld;
        bands.rows = N;
        for (int64_t e : {N / 16, N / 8, N / 4, N / 2, N}) {
            const int64_t r0 = bands.ev.empty() ? 0 : bands.ev.back().first;
            if (e <= r0) continue;
            FFB_CUDA(cudaMemcpyAsync(tmp + (size_t)r0 * N * aeb, (const char*)a + (size_t)r0 * N * aeb,
                                     (size_t)(e - r0) * N * aeb, cudaMemcpyHostToDevice, c->copy_stream));
            pdl_fence(c->copy_stream);
            convert_in(f, c->copy_stream, W.sub(r0, 0, e - r0, N), tmp + (size_t)r0 * N * aeb, aeb);
            cudaEvent_t ev;
            FFB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            FFB_CUDA(cudaEventRecord(ev, c->copy_stream));
            bands.ev.push_back({e, ev});
        }
        int32_t* aflag = c->flag + 16;  // asymmetry flag (copy stream)
        FFB_CUDA(cudaMemsetAsync(aflag, 0, sizeof(int32_t), c->copy_stream));
        pdl_fence(c->copy_stream);
        any_asymmetric_raw(c->copy_stream, tmp, N, aeb, p, aflag);
        cudaEvent_t checked;
        FFB_CUDA(cudaEventCreateWithFlags(&checked, cudaEventDisableTiming));
        FFB_CUDA(cudaEventRecord(checked, c->copy_stream));
        FFB_CUDA(cudaStreamWaitEvent(c->stream, bands.ev.front().second, 0));
        pdl_fence(c->stream);
        bands.ready = bands.ev.front().first;
        auto release = [&] {
            for (auto& be : bands.ev) cudaEventDestroy(be.second);
            cudaEventDestroy(checked);
        };
        auto asymmetric = [&] {
            FFB_CUDA(cudaStreamWaitEvent(c->stream, checked, 0));
            pdl_fence(c->stream);
            return *(const int32_t*)readback(c, aflag, sizeof(int32_t)) != 0;
        };
        DevFact df;
        try {
            df = run_ldlt(c, f, W, variant, (int64_t)threshold, false, &bands);
        } catch (const Status&) {
            cudaStreamSynchronize(c->copy_stream);
            const bool asym = asymmetric();
            release();
            if (asym) throw Status(FFB_NOT_SYMMETRIC, "ldlt: matrix must be symmetric");
            throw;
        }
        const bool asym = asymmetric();  // (also orders the last band before the export)
        release();
        if (asym) throw Status(FFB_NOT_SYMMETRIC, "ldlt: matrix must be symmetric");
        export_host(c, df, perm, lower, leb, dkind, dval, dval2, rank);
        c->ws_top = 0;
    });
}

int ffb_ldlt(ffb_context* c, uint64_t p, size_t rows, size_t cols, const uint64_t* a, int variant,
             size_t threshold, int64_t* perm, uint64_t* lower, int32_t* dkind, uint64_t* dval,
             uint64_t* dval2, size_t* rank) {
    if (rows != cols) {
        g_last_error = "ldlt: matrix must be square";
        return FFB_DIMENSION_MISMATCH;  // sytrf.cpp:355
    }
    return ffb_ldlt_compact(c, p, rows, a, FFB_U64, variant, threshold, perm, lower, FFB_U64,
                            dkind, dval, dval2, rank);
}

int ffb_ldlt_zero_leading(ffb_context* c, uint64_t p, size_t m, size_t ny, const uint64_t* y,
                          size_t nz, const uint64_t* z, int variant, size_t threshold,
                          int64_t* perm, uint64_t* lower, int32_t* dkind, uint64_t* dval,
                          uint64_t* dval2, size_t* rank) {
    return guarded(c, [&] {
        if (ny != nz) throw Status(FFB_DIMENSION_MISMATCH, "ldlt_zero_leading: Y and Z have mismatched widths");
        check_modulus(p);
        const int64_t N = (int64_t)(m + nz);
        ensure_workspace(c, workspace_bytes(N) + (size_t)N * N * 16);
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat Zd = upload_matrix(c, f, z, (int64_t)nz, (int64_t)nz, 8);
        {
            fill_words(c->stream, (uint32_t*)c->flag, 1, 0u);
            any_asymmetric(c->stream, Zd, c->flag);
            if (*(const int32_t*)readback(c, c->flag, sizeof(int32_t)))
                throw Status(FFB_NOT_SYMMETRIC, "ldlt_zero_leading: Z must be symmetric");
        }
        DMat Yd = upload_matrix(c, f, y, (int64_t)m, (int64_t)nz, 8);
        DevFact df;
        df.n = N;
        df.Lg = ws_mat(c, N, N);
        zero_mat(c->stream, df.Lg);
        df.D.kind = ws_vec<int32_t>(c, N);
        df.D.val = ws_vec<uint32_t>(c, N);
        df.D.val2 = ws_vec<uint32_t>(c, N);
        df.D.inv = ws_vec<uint32_t>(c, N);
        Engine e{c, c->stream, f, variant, (int64_t)threshold, df.Lg, df.D};
        std::vector<int32_t> rows(N);
        for (int64_t i = 0; i < N; ++i) rows[i] = (int32_t)i;
        HFact h = e.zero_leading(Yd, Zd, rows, upload(c, rows), 0);
        df.rank = h.rank;
        df.perm = h.perm;
        export_host(c, df, perm, lower, 8, dkind, dval, dval2, rank);
        c->ws_top = 0;
    });
}

int ffb_ldlt_device(ffb_context* c, uint64_t p, size_t n, uint32_t* d_a, size_t lda, int variant,
                    size_t threshold, int32_t* d_perm, uint32_t* d_lower, size_t ldl,
                    int32_t* d_dkind, uint32_t* d_dval, uint32_t* d_dval2, size_t* rank) {
    return guarded(c, [&] {
        check_modulus(p);
        ensure_workspace(c, workspace_bytes((int64_t)n));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat W;
        W.ptr = d_a;
        W.ld = (int64_t)lda;
        W.rows = W.cols = (int64_t)n;
        DevFact df = run_ldlt(c, f, W, variant, (int64_t)threshold, true);
        const int64_t r = df.rank;
        *rank = (size_t)r;
        if (n > 0) {
            const int32_t* dp = upload(c, df.perm);
            FFB_CUDA(cudaMemcpyAsync(d_perm, dp, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream)); pdl_fence(c->stream);
            DMat Lout;
            Lout.ptr = d_lower;
            Lout.ld = (int64_t)ldl;
            Lout.rows = (int64_t)n;
            Lout.cols = r;
            gather_lower_out(c->stream, Lout, df.Lg, dp);
            if (r > 0) {
                FFB_CUDA(cudaMemcpyAsync(d_dkind, df.D.kind, r * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream)); pdl_fence(c->stream);
                FFB_CUDA(cudaMemcpyAsync(d_dval, df.D.val, r * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->stream)); pdl_fence(c->stream);
                FFB_CUDA(cudaMemcpyAsync(d_dval2, df.D.val2, r * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->stream)); pdl_fence(c->stream);
            }
        }
        FFB_CUDA(cudaStreamSynchronize(c->stream));
        c->ws_top = 0;
    });
}

int ffb_verify_device(ffb_context* c, uint64_t p, size_t n, const uint32_t* d_a, size_t lda,
                      const int32_t* d_perm, const uint32_t* d_lower, size_t ldl, const int32_t* d_dkind,
                      const uint32_t* d_dval, const uint32_t* d_dval2, size_t rank, uint64_t* mismatches) {
    return guarded(c, [&] {
        check_modulus(p);
        if (rank > n) throw Status(FFB_DIMENSION_MISMATCH, "verify: rank exceeds n");
        const int64_t N = (int64_t)n, r = (int64_t)rank;
        ensure_workspace(c, (size_t)N * (r + N) * sizeof(uint32_t) + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat A, L;
        A.ptr = const_cast<uint32_t*>(d_a);
        A.ld = (int64_t)lda;
        A.rows = A.cols = N;
        L.ptr = const_cast<uint32_t*>(d_lower);
        L.ld = (int64_t)ldl;
        L.rows = N;
        L.cols = r;
        DDiag D{const_cast<int32_t*>(d_dkind), const_cast<uint32_t*>(d_dval), const_cast<uint32_t*>(d_dval2),
                nullptr};
        DMat H = ws_mat(c, N, std::max<int64_t>(r, 1)), C = ws_mat(c, N, N);
        auto* cnt = (unsigned long long*)(c->flag + 24);  // bytes 96..103 of the flag block
        fill_words(c->stream, (uint32_t*)cnt, 2, 0u);
        reconstruct_mismatches(f, c->stream, A, d_perm, L, D, r, H, C, cnt);
        *mismatches = *(const uint64_t*)readback(c, cnt, sizeof(uint64_t));
        c->ws_top = 0;
    });
}

int ffb_pivoting_partners_device(ffb_context* c, size_t n, const int32_t* d_perm, const int32_t* d_dkind,
                                 size_t rank, int32_t* d_partner) {
    return guarded(c, [&] {
        if (rank > n) throw Status(FFB_DIMENSION_MISMATCH, "pivoting_partners: rank exceeds n");
        pivoting_partners(c->stream, d_perm, d_dkind, (int64_t)n, (int64_t)rank, d_partner);
        FFB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ffb_plduq(ffb_context* c, uint64_t p, size_t m, size_t n, const uint64_t* b, int64_t* row_image,
              int64_t* col_image, uint64_t* lower, uint64_t* diag, uint64_t* upper, size_t* rank) {
    return guarded(c, [&] {
        check_modulus(p);
        // the chunked PLDUQ of a full-rank square input holds ~46 m x n word matrices at its peak
        // (factors, both bases, phase-2 products); measured at n = 2048
        ensure_workspace(c, (size_t)(m + 1) * (n + 1) * 256 + ((size_t)128 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat Y = upload_matrix(c, f, b, (int64_t)m, (int64_t)n, 8);
        Engine e{c, c->stream, f, FFB_VARIANT_CASCADE, 64, DMat(), DDiag()};
        Engine::Pl pl = e.run_plduq(Y);
        for (size_t i = 0; i < m; ++i) row_image[i] = pl.rimg[i];
        for (size_t j = 0; j < n; ++j) col_image[j] = pl.cimg[j];
        *rank = (size_t)pl.r;
        if (pl.r > 0) {
            download_matrix(c, pl.L, lower);
            download_matrix(c, pl.U, upper);
            std::vector<uint32_t> d(pl.r);
            FFB_CUDA(cudaMemcpy(d.data(), pl.d, pl.r * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            for (int64_t k = 0; k < pl.r; ++k) diag[k] = d[k];
        }
        c->ws_top = 0;
    });
}

int ffb_trssyr2k(ffb_context* c, uint64_t p, size_t n, const uint64_t* u, const uint64_t* cc,
                 uint64_t* x) {
    return guarded(c, [&] {
        check_modulus(p);  // validation order of trssyr2k.cpp:55-66
        for (size_t i = 0; i < n; ++i)
            if (u[i * n + i] % p != 1 % p)
                throw Status(FFB_NON_UNIT_TRIANGULAR, "trssyr2k: U must have unit diagonal");
        for (size_t i = 0; i < n; ++i)
            for (size_t j = i + 1; j < n; ++j)
                if (cc[i * n + j] % p != cc[j * n + i] % p)
                    throw Status(FFB_NOT_SYMMETRIC, "trssyr2k: C must be symmetric");
        if (n == 0) return;
        ensure_workspace(c, (size_t)n * n * 64 + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        const int64_t N = (int64_t)n;
        // Only the upper triangle of U is read (trssyr2k.hpp:8-10).
        std::vector<uint64_t> hu(n * n), hut(n * n);
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < n; ++j) {
                hu[i * n + j] = (j >= i) ? u[i * n + j] % p : 0;
                hut[j * n + i] = hu[i * n + j];
            }
        DMat U = upload_matrix(c, f, hu.data(), N, N, 8);
        DMat UT = upload_matrix(c, f, hut.data(), N, N, 8);
        DMat C = upload_matrix(c, f, cc, N, N, 8);
        DMat X = ws_mat(c, N, N);
        Engine e{c, c->stream, f, FFB_VARIANT_CASCADE, 64, DMat(), DDiag()};
        fill_words(c->stream, (uint32_t*)c->flag, 1, 0u);
        e.trssyr2k_dev(U, UT, C, X, c->flag);
        if (f.char2 && *(const int32_t*)readback(c, c->flag, sizeof(int32_t)))
            throw Status(FFB_CHAR_TWO_NONZERO_DIAGONAL, "trssyr2k: diagonal entry has no solution");
        download_matrix(c, X, x);
        c->ws_top = 0;
    });
}

int ffb_gemm_device(ffb_context* c, uint64_t p, int mode, size_t m, size_t n, size_t k,
                    uint32_t* d_c, size_t ldc, const uint32_t* d_a, size_t lda, int ta,
                    const uint32_t* d_b, size_t ldb, int tb) {
    return guarded(c, [&] {
        check_modulus(p);
        if (mode < 0 || mode > 2) throw Status(FFB_ERROR, "gemm: bad mode");
        Fp f = make_field(c, p);
        DMat C, A, B;
        C.ptr = d_c; C.ld = (int64_t)ldc; C.rows = (int64_t)m; C.cols = (int64_t)n;
        A.ptr = (uint32_t*)d_a; A.ld = (int64_t)lda; A.rows = ta ? (int64_t)k : (int64_t)m;
        A.cols = ta ? (int64_t)m : (int64_t)k;
        B.ptr = (uint32_t*)d_b; B.ld = (int64_t)ldb; B.rows = tb ? (int64_t)n : (int64_t)k;
        B.cols = tb ? (int64_t)k : (int64_t)n;
        gemm(f, c->stream, (GemmMode)mode, C, A, ta != 0, B, tb != 0, (int64_t)m, (int64_t)n,
             (int64_t)k);
    });
}

// ---- kernels.hpp:13-32 --------------------------------------------------------
int ffb_gemm_sub(ffb_context* c, uint64_t p, size_t m, size_t n, size_t k, uint64_t* cc,
                 const uint64_t* a, const uint64_t* b) {
    return guarded(c, [&] {
        check_modulus(p);
        ensure_workspace(c, ((size_t)m * n + m * k + k * n) * 16 + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat C = upload_matrix(c, f, cc, m, n, 8), A = upload_matrix(c, f, a, m, k, 8),
             B = upload_matrix(c, f, b, k, n, 8);
        gemm(f, c->stream, GEMM_SUB, C, A, false, B, false, m, n, k);
        download_matrix(c, C, cc);
        c->ws_top = 0;
    });
}

int ffb_trmm_sub(ffb_context* c, uint64_t p, size_t n, size_t ncols, uint64_t* cc, const uint64_t* t,
                 int upper, int trans, int unit, const uint64_t* b) {
    return guarded(c, [&] {
        check_modulus(p);
        ensure_workspace(c, ((size_t)n * ncols * 2 + n * n) * 16 + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat C = upload_matrix(c, f, cc, n, ncols, 8), T = upload_matrix(c, f, t, n, n, 8),
             B = upload_matrix(c, f, b, n, ncols, 8);
        DMat O = ws_mat(c, n, n);  // op(T) with its triangle / unit conventions (kernels.cpp:23-29)
        tri_dense(f, c->stream, O, T, upper != 0, trans != 0, unit != 0, false, nullptr);
        gemm(f, c->stream, GEMM_SUB, C, O, false, B, false, n, ncols, n);
        download_matrix(c, C, cc);
        c->ws_top = 0;
    });
}

int ffb_trsm_inplace(ffb_context* c, uint64_t p, size_t n, size_t ncols, const uint64_t* t, int upper,
                     int trans, int unit, uint64_t* b) {
    return guarded(c, [&] {
        check_modulus(p);
        ensure_workspace(c, ((size_t)n * ncols * 2 + n * n * 2) * 16 + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat T = upload_matrix(c, f, t, n, n, 8);
        // kernels.cpp:64-71: a zero pivot raises (before any row of B is written here)
        const uint32_t* dinv = nullptr;
        if (!unit && n > 0) {
            uint32_t* diag = ws_vec<uint32_t>(c, (int64_t)n);
            uint32_t* inv = ws_vec<uint32_t>(c, (int64_t)n);
            fill_words(c->stream, (uint32_t*)c->flag, 1, 0u);
            tri_diag(c->stream, T, diag, c->flag);
            if (*(const int32_t*)readback(c, c->flag, sizeof(int32_t)))
                throw Status(FFB_SINGULAR_TRIANGULAR, "trsm_inplace: zero diagonal");
            invert_vec(f, c->stream, inv, diag, (int64_t)n);
            dinv = inv;
        }
        if (n == 0 || ncols == 0) return;
        DMat B = upload_matrix(c, f, b, n, ncols, 8);
        // Normalise to a unit lower solve on the device: reverse the index order for an
        // effective-upper op(T), scale rows by the inverse diagonal when non-unit.
        const bool lower = (upper == 0) != (trans != 0);
        DMat L = ws_mat(c, n, n), X = ws_mat(c, n, ncols);
        tri_dense(f, c->stream, L, T, upper != 0, trans != 0, unit != 0, !lower, dinv);
        rows_rev_scaled(f, c->stream, X, B, !lower, dinv);
        trsm_lower_unit(f, c->stream, L, X);
        rows_rev_scaled(f, c->stream, B, X, !lower, nullptr);
        download_matrix(c, B, b);
        c->ws_top = 0;
    });
}

// C -= G D G^T with D given per column (kind/val/val2); shared by both syrdk_sub overloads.
static void syrdk_columns(ffb_context* c, uint64_t p, size_t n, size_t k, uint64_t* cc, const uint64_t* g,
                          const std::vector<int32_t>& kind, const uint64_t* dval, const uint64_t* dval2) {
    ensure_workspace(c, ((size_t)n * n + 2 * n * k + 2 * k) * 16 + ((size_t)64 << 20));
    c->ws_top = 0;
    Fp f = make_field(c, p);
    DMat C = upload_matrix(c, f, cc, n, n, 8), G = upload_matrix(c, f, g, n, k, 8);
    DMat V = upload_matrix(c, f, dval, 1, k, 8);
    DMat V2 = dval2 ? upload_matrix(c, f, dval2, 1, k, 8) : V;
    const int32_t* kd = upload(c, kind);
    DMat H = ws_mat(c, n, k);
    apply_d(f, c->stream, H, G, kd, V.ptr, V2.ptr);  // H = G D
    gemm(f, c->stream, GEMM_SUB, C, H, false, G, true, n, n, k);
    download_matrix(c, C, cc);
    c->ws_top = 0;
}

int ffb_syrdk_sub(ffb_context* c, uint64_t p, size_t n, size_t k, uint64_t* cc, const uint64_t* g,
                  const int32_t* dkind, const uint64_t* dval, const uint64_t* dval2) {
    return guarded(c, [&] {
        check_modulus(p);
        std::vector<int32_t> kind(dkind, dkind + k);
        for (size_t t = 0; t < k; ++t) {  // per-column encoding must describe whole blocks
            const int32_t kk = kind[t];
            const bool ok = kk == FFB_D_SCALAR ||
                            ((kk == FFB_D_ANTIDIAG_HEAD || kk == FFB_D_ANTITRI_HEAD) && t + 1 < k && kind[t + 1] == kk + 1) ||
                            ((kk == FFB_D_ANTIDIAG_TAIL || kk == FFB_D_ANTITRI_TAIL) && t > 0 && kind[t - 1] == kk - 1);
            if (!ok) throw Status(FFB_DIMENSION_MISMATCH, "syrdk_sub: malformed block diagonal");
        }
        syrdk_columns(c, p, n, k, cc, g, kind, dval, dval2);
    });
}

int ffb_syrdk_sub_diag(ffb_context* c, uint64_t p, size_t n, size_t k, uint64_t* cc, const uint64_t* g,
                       const uint64_t* d) {
    return guarded(c, [&] {
        check_modulus(p);
        syrdk_columns(c, p, n, k, cc, g, std::vector<int32_t>(k, FFB_D_SCALAR), d, nullptr);
    });
}

// strictify on a device factorization: heads of the AntiTri blocks from the kind array
static void strictify_dev(ffb_context* c, const Fp& f, int64_t n, int64_t r, int32_t* perm, DMat L, DDiag D,
                          uint64_t* blocks_converted, uint64_t* entries_touched) {
    std::vector<int32_t> kind(std::max<int64_t>(r, 1));
    if (r > 0) {
        FFB_CUDA(cudaMemcpyAsync(kind.data(), D.kind, r * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        pdl_fence(c->stream);
        FFB_CUDA(cudaStreamSynchronize(c->stream));
    }
    std::vector<int32_t> heads;
    for (int64_t t = 0; t < r; ++t)
        if (kind[t] == FFB_D_ANTITRI_HEAD) heads.push_back((int32_t)t);
    if (!heads.empty() && !f.char2)
        throw Status(FFB_WRONG_CHARACTERISTIC, "strictify: AntiTri block over odd characteristic");
    unsigned long long* touched = (unsigned long long*)ws_vec<uint64_t>(c, 1);
    FFB_CUDA(cudaMemsetAsync(touched, 0, sizeof(uint64_t), c->stream));
    pdl_fence(c->stream);
    const int64_t nb = (int64_t)heads.size();
    if (nb) {
        const int32_t* dh = upload(c, heads);
        uint32_t* scratch = ws_vec<uint32_t>(c, 4 * nb);
        strictify_device(f, c->stream, L, n, dh, nb, perm, D, scratch, touched);
    }
    const uint64_t tt = *(const uint64_t*)readback(c, touched, sizeof(uint64_t));
    if (blocks_converted) *blocks_converted = (uint64_t)nb;
    if (entries_touched) *entries_touched = tt;
}

int ffb_strictify_device(ffb_context* c, uint64_t p, size_t n, size_t rank, int32_t* d_perm, uint32_t* d_lower,
                         size_t ldl, int32_t* d_dkind, uint32_t* d_dval, uint32_t* d_dval2,
                         uint64_t* blocks_converted, uint64_t* entries_touched) {
    return guarded(c, [&] {
        check_modulus(p);
        if (rank > n) throw Status(FFB_DIMENSION_MISMATCH, "strictify: rank exceeds n");
        ensure_workspace(c, (size_t)n * 64 + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat L;
        L.ptr = d_lower;
        L.ld = (int64_t)ldl;
        L.rows = (int64_t)n;
        L.cols = (int64_t)rank;
        DDiag D{d_dkind, d_dval, d_dval2, nullptr};
        strictify_dev(c, f, (int64_t)n, (int64_t)rank, d_perm, L, D, blocks_converted, entries_touched);
        c->ws_top = 0;
    });
}

int ffb_strictify(ffb_context* c, uint64_t p, size_t n, size_t rank, int64_t* perm, uint64_t* lower,
                  int32_t* dkind, uint64_t* dval, uint64_t* dval2, uint64_t* blocks_converted,
                  uint64_t* entries_touched) {
    return guarded(c, [&] {
        check_modulus(p);
        if (rank > n) throw Status(FFB_DIMENSION_MISMATCH, "strictify: rank exceeds n");
        const int64_t N = (int64_t)n, R = (int64_t)rank;
        ensure_workspace(c, (size_t)N * std::max<int64_t>(R, 1) * 16 + (size_t)N * 64 + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat L = upload_matrix(c, f, lower, N, R, 8);
        std::vector<int32_t> pv(perm, perm + N), kd(dkind, dkind + R);
        int32_t* dperm = ws_vec<int32_t>(c, N);
        int32_t* dk = ws_vec<int32_t>(c, R);
        FFB_CUDA(cudaMemcpyAsync(dperm, upload(c, pv), N * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
        FFB_CUDA(cudaMemcpyAsync(dk, upload(c, kd), std::max<int64_t>(R, 1) * sizeof(int32_t),
                                 cudaMemcpyDeviceToDevice, c->stream));
        pdl_fence(c->stream);
        DMat V = upload_matrix(c, f, dval, 1, R, 8), V2 = upload_matrix(c, f, dval2, 1, R, 8);
        DDiag D{dk, V.ptr, V2.ptr, nullptr};
        strictify_dev(c, f, N, R, dperm, L, D, blocks_converted, entries_touched);
        download_matrix(c, L, lower);
        std::vector<int32_t> pout(std::max<int64_t>(N, 1)), kout(std::max<int64_t>(R, 1));
        std::vector<uint32_t> v(std::max<int64_t>(R, 1)), v2(std::max<int64_t>(R, 1));
        FFB_CUDA(cudaMemcpyAsync(pout.data(), dperm, N * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        if (R > 0) {
            FFB_CUDA(cudaMemcpyAsync(kout.data(), dk, R * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
            FFB_CUDA(cudaMemcpyAsync(v.data(), V.ptr, R * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
            FFB_CUDA(cudaMemcpyAsync(v2.data(), V2.ptr, R * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        }
        pdl_fence(c->stream);
        FFB_CUDA(cudaStreamSynchronize(c->stream));
        for (int64_t i = 0; i < N; ++i) perm[i] = pout[i];
        for (int64_t t = 0; t < R; ++t) {
            dkind[t] = kout[t];
            dval[t] = v[t];
            dval2[t] = v2[t];
        }
        c->ws_top = 0;
    });
}

int ffb_syr2k_sub(ffb_context* c, uint64_t p, size_t n, size_t k, uint64_t* cc, const uint64_t* a,
                  const uint64_t* b) {
    return guarded(c, [&] {
        check_modulus(p);
        ensure_workspace(c, ((size_t)n * n + 2 * n * k) * 16 + ((size_t)64 << 20));
        c->ws_top = 0;
        Fp f = make_field(c, p);
        DMat C = upload_matrix(c, f, cc, n, n, 8), A = upload_matrix(c, f, a, k, n, 8),
             B = upload_matrix(c, f, b, k, n, 8);
        gemm2(f, c->stream, GEMM_SUB, C, A, true, B, false, B, true, A, false, n, n, k, k);
        download_matrix(c, C, cc);
        c->ws_top = 0;
    });
}

}  // extern "C"

// Debug-only export (not declared in include/ffldl_b200.h): PLDUQ kernel
// micro-benchmark on a host matrix (tools/pq_kernel_bench.py).
extern "C" int ffb_dbg_pq_bench(ffb_context* c, uint64_t p, int which, int rows, int cols,
                                const uint32_t* host, int reps, double* ms, int32_t* out) {
    return guarded(c, [&] {
        Fp f = make_field(c, p);
        uint32_t* d;
        FFB_CUDA(cudaMalloc(&d, (size_t)rows * cols * 4));
        FFB_CUDA(cudaMemcpy(d, host, (size_t)rows * cols * 4, cudaMemcpyHostToDevice));
        if (which == 2) dbg_leaf_bench(f, c->stream, rows, d, reps, ms, out);
        else dbg_pq_bench(f, c->stream, which, rows, cols, d, reps, ms, out);
        FFB_CUDA(cudaFree(d));
    });
}
