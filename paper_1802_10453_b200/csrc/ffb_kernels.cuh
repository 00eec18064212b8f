// ffb_kernels.cuh -- host-side launchers of the device kernels (one stream).
#pragma once

#include <vector>

#include "ffb_common.cuh"

namespace ffb {

// Launch accounting (reported by ffb_launch_count and bench.py's gpu_launches).
extern thread_local uint64_t g_launches;

// Optional per-kernel-class instrumentation (ffb_profile_enable): CUDA events
// around each launch on the launching stream, summed per class.
enum KClass {
    K_GEMM = 0, K_LEAF = 1, K_PLDUQ = 2, K_TRSM = 3, K_MOVE = 4, K_OTHER = 5,
    K_PQ_SKETCH = 6, K_PQ_CRP = 7, K_PQ_PAIR = 8, K_LDU = 9, K_PACK = 10, K_PQ_ROWELIM = 11, K_NCLASS = 12
};
struct Profiler {
    struct Rec {
        int cls;
        cudaEvent_t a, b;
        double ops, bytes;
        int64_t m, n, k;  // GEMM shape (trace only)
        int64_t node;     // recursion node size (trace only)
    };
    bool on = false;
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    double ms[K_NCLASS] = {}, ops[K_NCLASS] = {}, bytes[K_NCLASS] = {};
    uint64_t cnt[K_NCLASS] = {};
    cudaEvent_t get();
    void flush();  // caller has synchronized the stream
    void reset();
};
extern thread_local Profiler* g_prof;
extern thread_local int64_t g_node;
// Scratch slot of the GEMM packing / split-K buffers: launches on a secondary
// stream use slot 1 so they never share a buffer with the main stream.
extern thread_local int g_slot;
// Set while a GEMM runs beside the critical path on a low-priority stream: the
// persistent tcgen05 GEMM then occupies only part of the SMs (FFB_Z_OVERLAP_SMS),
// leaving the rest to the engine stream's latency kernels.
extern thread_local bool g_tc_shared_sms;
// >= 0 while a symmetric Schur update is issued whose consumers read only its upper band
// (entries j >= i - halo, halo >= the largest diagonal block a leaf reads): the tcgen05
// kernels skip the output tiles below that band (SYRK-style work); paths without tile
// skipping compute everything, a superset.  See BandScope.
extern thread_local int g_band_halo;
struct BandScope {
    int saved;
    explicit BandScope(int halo) : saved(g_band_halo) { g_band_halo = halo; }
    ~BandScope() { g_band_halo = saved; }
};
struct SlotGuard {
    int saved;
    explicit SlotGuard(int s) : saved(g_slot) { g_slot = s; }
    ~SlotGuard() { g_slot = saved; }
};  // size of the recursion node being executed (trace tag)
struct ProfScope {
    Profiler::Rec rec;
    cudaStream_t st;
    bool live;
    ProfScope(int cls, cudaStream_t s, double ops, double bytes, int64_t m = 0, int64_t n = 0,
              int64_t k = 0);
    ~ProfScope();
};

// FFB_PHASE_TRACE=<file>: event marks at the phase boundaries of large nodes (no
// synchronisation; elapsed times are written by phase_dump() after the run).
void phase_mark(const char* label, int64_t size, cudaStream_t st);
void phase_dump(cudaStream_t st);

enum GemmMode { GEMM_SUB = 0, GEMM_ADD = 1, GEMM_SET = 2 };

// C (M x N) = C -/+ op(A) * op(B)  or  C = op(A) * op(B), all mod p.
// op(A) is M x K (A stored K x M when ta), op(B) is K x N (B stored N x K when tb).
void gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
          int64_t M, int64_t N, int64_t K);

// C op= op(A1) op(B1) + op(A2) op(B2): one accumulator on the tcgen05 path, else two gemm()
void gemm2(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A1, bool ta1, DMat B1, bool tb1, DMat A2,
           bool ta2, DMat B2, bool tb2, int64_t M, int64_t N, int64_t K1, int64_t K2);
bool tc_gemm2(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A1, bool ta1, DMat B1, bool tb1, DMat A2,
              bool ta2, DMat B2, bool tb2, int64_t M, int64_t N, int64_t K1, int64_t K2);

// int8 mma.sync path (ffb_mma.cu): p <= 255, small and mid shapes, no operand packing.
bool mma_gemm_supported(const Fp& f, int64_t M, int64_t N, int64_t K);
void mma_gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
              int64_t M, int64_t N, int64_t K);

// Two GEMM_SUB products in one mma.sync launch when both are small; problem 1 may set
// *nzflag = tag when any of its outputs is nonzero.  Returns false when not applicable.
bool mma_gemm_pair(const Fp& f, cudaStream_t st, DMat C1, DMat A1, DMat B1, int64_t M1, int64_t N1, int64_t K1,
                   DMat C2, DMat A2, DMat B2, int64_t M2, int64_t N2, int64_t K2, int32_t* nzflag, int32_t tag);

// short-K bandwidth kernel (ffb_mma.cu): p <= 255, K <= 128, dp4a on int8 packs.
bool rankk_supported(const Fp& f, int64_t M, int64_t N, int64_t K);
void rankk_gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
                int64_t M, int64_t N, int64_t K);

// tcgen05 int8 path (ffb_tc_gemm.cu), used by gemm() for p <= 255 and large shapes.
bool tc_gemm_supported(const Fp& f, int64_t M, int64_t N, int64_t K);
void tc_gemm(const Fp& f, cudaStream_t st, GemmMode mode, DMat C, DMat A, bool ta, DMat B, bool tb,
             int64_t M, int64_t N, int64_t K);

// B <- T^-1 B for unit lower triangular T (n x n, only the strict lower part is read).
void trsm_lower_unit(const Fp& f, cudaStream_t st, DMat T, DMat B);

// dst[i][j] = src[idx[i]][j]
void gather_rows(cudaStream_t st, DMat dst, DMat src, const int32_t* idx);
// dst[a][b] = src[idx[a]][idx[b]]
void gather_sym(cudaStream_t st, DMat dst, DMat src, const int32_t* idx);
// dst (cols x rows) = src^T
void transpose(cudaStream_t st, DMat dst, DMat src);
// Lg[ids[i]][col0 + j*cstride] = src[i][j]
// Lg[ids[i]][col0 + 2j] = even[i][j], Lg[ids[i]][col0 + 2j + 1] = odd[i][j]
void scatter_lg_pair(cudaStream_t st, DMat Lg, const int32_t* ids, int64_t col0, DMat even, DMat odd);
// scatter_lg (stride 2) + scatter_lg_pair + write_pair_diag of zero_leading_pairs in one launch;
// false (nothing launched) when r == 0 or the rows exceed one grid.
bool zlp_scatter(cudaStream_t st, DMat Lg, int64_t col0, const int32_t* idy, DMat L, const int32_t* idz, DMat even,
                 DMat odd, DDiag D, const uint32_t* d, const uint32_t* dinv, const uint32_t* delta, int64_t r);
void scatter_lg(cudaStream_t st, DMat Lg, const int32_t* ids, int64_t col0, int cstride, DMat src);
// dst[i][k] = Lg[ids[i]][col0 + k]
void gather_lg(cudaStream_t st, DMat dst, DMat Lg, const int32_t* ids, int64_t col0);
// G (ncols x r) = (D^-1 X)^T with D the global block diagonal at columns [coff, coff+r);
// when ids is given, also Lg[ids[j]][coff + k] = G[j][k] (fused scatter).
void inverse_apply_T(const Fp& f, cudaStream_t st, DMat G, DMat X, DDiag D, int64_t coff,
                     DMat Lg = DMat(), const int32_t* ids = nullptr);
// d0[i][j] = s0[i0[i]][c0 + j] and d1[i][j] = s1[i1[i]][c1 + j] in one launch
void gather_rows2(cudaStream_t st, DMat d0, DMat s0, const int32_t* i0, int64_t c0, DMat d1, DMat s1,
                  const int32_t* i1, int64_t c1);
// G (ncols x r) = (diag(dinv) X)^T
void scale_T(const Fp& f, cudaStream_t st, DMat G, DMat X, const uint32_t* dinv);
// out[i] = v[i]^-1
void invert_vec(const Fp& f, cudaStream_t st, uint32_t* out, const uint32_t* v, int64_t n);
// flag (device int) |= any nonzero in m
// *flag = value when m has a nonzero entry (untouched otherwise)
void any_nonzero(cudaStream_t st, DMat m, int32_t* flag, int32_t value = 1);
// flag |= any a[i][j] != a[j][i]
void any_asymmetric(cudaStream_t st, DMat a, int32_t* flag);
// flag |= any a[i][j] != a[j][i] (mod p) on a raw n x n row-major matrix of eb-byte
// unsigned elements (the staged host input; the engine never writes it)
void any_asymmetric_raw(cudaStream_t st, const void* a, int64_t n, int eb, uint64_t p, int32_t* flag);
// Y <- strict_upper(Ct) + diag(Ct)/2 (odd p) or 0 (p = 2); lower part zeroed; in place.
// flag |= nonzero diagonal when p = 2 (no solution: CharTwoNonzeroDiagonal).
void trssyr2k_mid(const Fp& f, cudaStream_t st, DMat Ct, int32_t* flag);
// Pair blocks of zero_leading_pairs: D[coff+2i], D[coff+2i+1] from d, dinv, delta.
void write_pair_diag(const Fp& f, cudaStream_t st, DDiag D, int64_t coff, const uint32_t* d,
                     const uint32_t* dinv, const uint32_t* delta, int64_t r);
// Characteristic-2 delta recurrence (sytrf.cpp:188-198): delta_i = C1_ii - sum_{j<i} delta_j U1_ji^2
void char2_delta(const Fp& f, cudaStream_t st, DMat C1, DMat U1, uint32_t* delta);
// H[i][j] = v[i] * S[i][j]  (row scaling)
void scale_rows(const Fp& f, cudaStream_t st, DMat H, DMat S, const uint32_t* v);
// X[i][j] += v[i] * U[i][j] for j >= i
void add_scaled_rows_upper(const Fp& f, cudaStream_t st, DMat X, DMat U, const uint32_t* v);
// Z[i][j] = Z[j][i] for j < i - halo (after a band-only symmetric update, see BandScope)
void mirror_lower(cudaStream_t st, DMat Z, int halo);
// Set a view to zero.
void zero_mat(cudaStream_t st, DMat m);
// Verification (ffb_verify.cu): *dcount += #{(i, j) : (L D L^T)(i, j) != A(perm i, perm j)}
// using H (n x r) and C (n x n) as scratch; partner[perm(a)] = perm(b) over support(D).
void reconstruct_mismatches(const Fp& f, cudaStream_t st, DMat A, const int32_t* perm, DMat L, DDiag D,
                            int64_t r, DMat H, DMat C, unsigned long long* dcount);
void pivoting_partners(cudaStream_t st, const int32_t* perm, const int32_t* kind, int64_t n, int64_t r,
                       int32_t* partner);
// n words at p := v (a kernel launch)
void fill_words(cudaStream_t st, uint32_t* p, int64_t n, uint32_t v);
// Residue conversion at the host boundary.
void convert_in(const Fp& f, cudaStream_t st, DMat dst, const void* src, int elem_bytes);
void convert_out(cudaStream_t st, void* dst, int elem_bytes, DMat src);
// Final L: out[pos][k] = Lg[perm[pos]][k]
void gather_lower_out(cudaStream_t st, DMat out, DMat Lg, const int32_t* perm);

// Crout leaf (Alg. 4, sytrf.cpp:35-139) on an s x s block; writes L columns
// [coff, coff+rank) of rows rows[0..s) into Lg, D entries, and out[0] = rank,
// out[1..s] = local permutation (image).  scratch: device buffer for large s.
// mp: when mp.dst is set and the 64-leaf kernel runs, it publishes out[0 .. s] itself;
// returns whether it did (else the caller reads out back)
bool leaf_crout(const Fp& f, cudaStream_t st, DMat A, const int32_t* rows, DMat Lg,
                int64_t coff, DDiag D, int32_t* out, uint32_t* scratch, const MboxPost& mp = MboxPost());
size_t leaf_scratch_words(int64_t s);
// Register-resident leaf for s <= 64 (ffb_fast.cu).
bool leaf64_supported(int64_t s);
void dbg_leaf_bench(const Fp& f, cudaStream_t st, int s, const uint32_t* d_a, int reps, double* ms,
                    int32_t* out_rank);
void leaf64(const Fp& f, cudaStream_t st, DMat A, const int32_t* rows, DMat Lg, int64_t coff,
            DDiag D, int32_t* out, const MboxPost& mp);
// Fused small node (ffb_fast.cu): recursive_step + zero_leading of an s x s node whose
// children are leaves, in one launch.  out[0..s+2) = [0, rank, perm] or, when Y != 0
// (zero_leading_pairs), [1, r1, perm1(m)] with Y in yout (m - r1 x ns, ld ns) and
// Z = C - G X written back to A[m:, m:].
bool node128_supported(const Fp& f, int64_t s, int64_t T);
void node128(const Fp& f, cudaStream_t st, DMat A, const int32_t* rows, DMat Lg, int64_t coff, DDiag D,
             uint32_t* yout, int32_t* out, const MboxPost& mp);

// Secondary C-ABI entry points (ffb_api.cu).
// out (n x n) = op(T)(a_i, a_k) with a_i = n-1-i when rev; with dinv the unit-lower
// normalisation dinv(a_i) op(T)(a_i, a_k) below the diagonal (kernels.cpp:23-29,57-81).
void tri_dense(const Fp& f, cudaStream_t st, DMat out, DMat T, bool upper, bool trans, bool unit, bool rev,
               const uint32_t* dinv);
// diag[i] = T(i, i); *flag |= 1 when one is zero
void tri_diag(cudaStream_t st, DMat T, uint32_t* diag, int32_t* flag);
// dst(i, :) = src(a_i, :) * dinv(a_i) (dinv may be null: no scaling)
void rows_rev_scaled(const Fp& f, cudaStream_t st, DMat dst, DMat src, bool rev, const uint32_t* dinv);
// H = G D for a per-column BlockDiag encoding (kind/val/val2)
void apply_d(const Fp& f, cudaStream_t st, DMat H, DMat G, const int32_t* kind, const uint32_t* val,
             const uint32_t* val2);
// strictify (rpmtools.cpp:74-132) of the AntiTri blocks with head columns heads[0..nb) on a
// device factorization (L n x r, perm, D); scratch >= 4 nb words; *touched += entries written
void strictify_device(const Fp& f, cudaStream_t st, DMat L, int64_t n, const int32_t* heads, int64_t nb,
                      int32_t* perm, DDiag D, uint32_t* scratch, unsigned long long* touched);

// PLDUQ (plduq.cpp:36-123) of W (m x n, destroyed).  Outputs: info[0] = r,
// info[1..m] row_image, info[1+m..1+m+n] col_image, pc[r] in info after that;
// Lo (m x min(m,n)) = [L1;M1], d (r), Uo (min(m,n) x n) = [U1 V1].
void plduq(const Fp& f, cudaStream_t st, DMat W, int32_t* info, int32_t* colflag,
           uint32_t* lvec, DMat Lo, uint32_t* d, DMat Uo);
// The same with W (only read) staged in shared memory as bytes: p <= 255 and
// plduq_smem_bytes(m, n) <= 226 KB, else returns false without a launch.  Stops after rcap
// pivots when more would follow: info[0] = -1 and the other outputs are unspecified.
bool plduq_smem(const Fp& f, cudaStream_t st, DMat W, int32_t* info, DMat Lo, uint32_t* d, uint32_t* dinv, DMat Uo,
                int rcap);  // (also writes the pivots' inverses)

}  // namespace ffb
