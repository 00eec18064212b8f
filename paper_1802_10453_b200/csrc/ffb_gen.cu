// ffb_gen.cu -- seeded, counter-based generators of the benchmark inputs.
//
// The five configurations of BASELINE.json.
// Every entry is a pure function of (seed, stream, i, j), so the host and the
// device versions are bit-identical and any n reproduces the same family:
//   1/3  dense symmetric, upper entries uniform in [0, p), mirrored
//   2    A = M' diag(d) M'^T, M' = Q M (rows permuted), M uniform, d in [1, p)
//   4    hollow: zero diagonal, off-diagonal uniform
//   5    A = L R L^T, L unit lower (strict part uniform), R a symmetric partial
//        permutation with r - 2*(r/4) fixed points and r/4 transposition pairs
//        at uniformly random positions; R is then A's rank profile matrix.
#include <algorithm>
#include <numeric>
#include <vector>

#include "ffb_kernels.cuh"

namespace ffb {
namespace gen {

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t hash4(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j) {
    uint64_t z = mix64(seed + 0x9E3779B97F4A7C15ull * (stream + 1));
    z = mix64(z ^ (i + 0x632BE59BD9B4E019ull));
    z = mix64(z ^ (j * 0x9E3779B97F4A7C15ull + 0x8CB92BA72F3D8DD7ull));
    return z;
}
// uniform in [0, range)
__host__ __device__ inline uint32_t uni(uint64_t seed, uint64_t stream, uint64_t i, uint64_t j,
                                        uint64_t range) {
    return (uint32_t)umulhi64(hash4(seed, stream, i, j), range);
}

// Seeded permutation of [0, n): sort by hashed keys (ties by index).
std::vector<int64_t> permutation(int64_t n, uint64_t seed, uint64_t stream) {
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::vector<uint64_t> key(n);
    for (int64_t i = 0; i < n; ++i) key[i] = hash4(seed, stream, (uint64_t)i, 0);
    std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
        return key[a] != key[b] ? key[a] < key[b] : a < b;
    });
    return idx;
}

// partner[a] of configuration 5's R (-1: row a of R is zero).
std::vector<int64_t> partners5(int64_t n, int64_t r, uint64_t seed) {
    std::vector<int64_t> pi = permutation(n, seed, 4), partner(n, -1);
    const int64_t npairs = r / 4, nfixed = r - 2 * npairs;
    for (int64_t k = 0; k < nfixed; ++k) partner[pi[k]] = pi[k];
    for (int64_t t = 0; t < npairs; ++t) {
        const int64_t a = pi[nfixed + 2 * t], b = pi[nfixed + 2 * t + 1];
        partner[a] = b;
        partner[b] = a;
    }
    return partner;
}

__host__ __device__ inline uint32_t dense_entry(uint64_t seed, uint64_t p, int64_t i, int64_t j,
                                                bool hollow) {
    if (hollow && i == j) return 0;
    const int64_t a = i < j ? i : j, b = i < j ? j : i;
    return uni(seed, 0, (uint64_t)a, (uint64_t)b, p);
}
__host__ __device__ inline uint32_t l5_entry(uint64_t seed, uint64_t p, int64_t i, int64_t a) {
    if (a > i) return 0;
    if (a == i) return 1 % (uint32_t)p;
    return uni(seed, 1, (uint64_t)i, (uint64_t)a, p);
}

__global__ void k_dense(uint32_t* out, int64_t i0, int64_t n, uint64_t p, uint64_t seed, int hollow) {
    const int64_t i = i0 + blockIdx.y;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x)
        out[(int64_t)blockIdx.y * n + j] = dense_entry(seed, p, i, j, hollow != 0);
}

// cfg2 factors: H = M' diag(d) (n x r) and M' (n x r)
__global__ void k_cfg2_factors(uint32_t* H, uint32_t* Mp, const int32_t* q, int64_t n, int64_t r,
                               uint64_t p, uint64_t seed, Fp f) {
    const int64_t i = blockIdx.y;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < r;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t m = uni(seed, 1, (uint64_t)q[i], (uint64_t)k, p);
        const uint32_t d = 1 + uni(seed, 2, (uint64_t)k, 0, p - 1);
        Mp[i * r + k] = m;
        H[i * r + k] = fmul(f, m, d);
    }
}

// cfg5 factors: Lu(i,t) = L(i, a_t), Lp(i,t) = L(i, partner(a_t))
__global__ void k_cfg5_factors(uint32_t* Lu, uint32_t* Lp, const int32_t* ua, const int32_t* ub,
                               int64_t i0, int64_t r, uint64_t p, uint64_t seed) {
    const int64_t il = blockIdx.y, i = i0 + il;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < r;
         t += (int64_t)gridDim.x * blockDim.x) {
        Lu[il * r + t] = l5_entry(seed, p, i, ua[t]);
        Lp[il * r + t] = l5_entry(seed, p, i, ub[t]);
    }
}

void used_columns(const std::vector<int64_t>& partner, std::vector<int32_t>& ua,
                  std::vector<int32_t>& ub) {
    for (int64_t a = 0; a < (int64_t)partner.size(); ++a)
        if (partner[a] >= 0) {
            ua.push_back((int32_t)a);
            ub.push_back((int32_t)partner[a]);
        }
}

}  // namespace gen
}  // namespace ffb

using namespace ffb;

namespace {

Fp host_field(uint64_t p) { return make_fp(p, nullptr); }

int check_gen_args(int config, size_t n, size_t r, uint64_t p) {
    if (config < 1 || config > 5) return FFB_ERROR;
    if (p < 2 || p >= (1ull << 31)) return FFB_UNSUPPORTED;
    if ((config == 2 || config == 5) && r > n) return FFB_DIMENSION_MISMATCH;
    return FFB_OK;
}

}  // namespace

extern "C" {

int ffb_config5_partners(size_t n, size_t r, uint64_t seed, int64_t* partner) {
    if (r > n) return FFB_DIMENSION_MISMATCH;
    std::vector<int64_t> pt = gen::partners5((int64_t)n, (int64_t)r, seed);
    std::copy(pt.begin(), pt.end(), partner);
    return FFB_OK;
}

int ffb_generate_host(int config, size_t n_, size_t r_, uint64_t p, uint64_t seed, uint64_t* out) {
    int s = check_gen_args(config, n_, r_, p);
    if (s != FFB_OK) return s;
    const int64_t n = (int64_t)n_, r = (int64_t)r_;
    const Fp f = host_field(p);
    if (config == 1 || config == 3 || config == 4) {
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) out[i * n + j] = gen::dense_entry(seed, p, i, j, config == 4);
        return FFB_OK;
    }
    std::vector<uint32_t> U(n * r), V(n * r);  // A = U V^T
    if (config == 2) {
        std::vector<int64_t> q = gen::permutation(n, seed, 3);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t k = 0; k < r; ++k) {
                const uint32_t m = gen::uni(seed, 1, (uint64_t)q[i], (uint64_t)k, p);
                const uint32_t d = 1 + gen::uni(seed, 2, (uint64_t)k, 0, p - 1);
                V[i * r + k] = m;
                U[i * r + k] = fmul(f, m, d);
            }
    } else {
        std::vector<int32_t> ua, ub;
        gen::used_columns(gen::partners5(n, r, seed), ua, ub);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t t = 0; t < r; ++t) {
                U[i * r + t] = gen::l5_entry(seed, p, i, ua[t]);
                V[i * r + t] = gen::l5_entry(seed, p, i, ub[t]);
            }
    }
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            uint64_t acc = 0;
            const uint32_t* u = &U[i * r];
            const uint32_t* v = &V[j * r];
            for (int64_t k = 0; k < r; ++k) {
                acc += (uint64_t)u[k] * v[k];
                if (f.p >= (1u << 23) || (k & 1023) == 1023) acc = red64(f, acc);
            }
            out[i * n + j] = red64(f, acc);
        }
    return FFB_OK;
}

int ffb_generate_device(ffb_context* ctx, int config, size_t n_, size_t r_, uint64_t p,
                        uint64_t seed, uint32_t* d_out) {
    int s = check_gen_args(config, n_, r_, p);
    if (s != FFB_OK) return s;
    try {
        cudaStream_t st = (cudaStream_t)ffb_stream(ctx);
        const int64_t n = (int64_t)n_, r = (int64_t)r_;
        const Fp f = host_field(p);
        if (config == 1 || config == 3 || config == 4) {
            for (int64_t i0 = 0; i0 < n; i0 += 65535) {
                const int64_t nr = std::min<int64_t>(65535, n - i0);
                dim3 g((unsigned)std::min<int64_t>(64, cdiv(n, 256)), (unsigned)nr);
                gen::k_dense<<<g, 256, 0, st>>>(d_out + i0 * n, i0, n, p, seed, config == 4);
            }
            FFB_CHECK_LAUNCH();
            FFB_CUDA(cudaStreamSynchronize(st));
            return FFB_OK;
        }
        uint32_t *U = nullptr, *V = nullptr;
        int32_t *ia = nullptr, *ib = nullptr;
        FFB_CUDA(cudaMalloc(&U, (size_t)n * r * 4));
        FFB_CUDA(cudaMalloc(&V, (size_t)n * r * 4));
        if (config == 2) {
            std::vector<int64_t> q64 = gen::permutation(n, seed, 3);
            std::vector<int32_t> q(q64.begin(), q64.end());
            FFB_CUDA(cudaMalloc(&ia, n * 4));
            FFB_CUDA(cudaMemcpy(ia, q.data(), n * 4, cudaMemcpyHostToDevice));
            for (int64_t i0 = 0; i0 < n; i0 += 65535) {
                const int64_t nr = std::min<int64_t>(65535, n - i0);
                dim3 g((unsigned)std::min<int64_t>(64, cdiv(r, 256)), (unsigned)nr);
                gen::k_cfg2_factors<<<g, 256, 0, st>>>(U + i0 * r, V + i0 * r, ia + i0, nr, r, p, seed, f);
            }
        } else {
            std::vector<int32_t> ua, ub;
            gen::used_columns(gen::partners5(n, r, seed), ua, ub);
            FFB_CUDA(cudaMalloc(&ia, r * 4 + 4));
            FFB_CUDA(cudaMalloc(&ib, r * 4 + 4));
            FFB_CUDA(cudaMemcpy(ia, ua.data(), r * 4, cudaMemcpyHostToDevice));
            FFB_CUDA(cudaMemcpy(ib, ub.data(), r * 4, cudaMemcpyHostToDevice));
            for (int64_t i0 = 0; i0 < n; i0 += 65535) {
                const int64_t nr = std::min<int64_t>(65535, n - i0);
                dim3 g((unsigned)std::min<int64_t>(64, cdiv(r, 256)), (unsigned)nr);
                gen::k_cfg5_factors<<<g, 256, 0, st>>>(U + i0 * r, V + i0 * r, ia, ib, i0, r, p, seed);
            }
        }
        FFB_CHECK_LAUNCH();
        DMat C, A, B;
        C.ptr = d_out; C.ld = n; C.rows = n; C.cols = n;
        A.ptr = U; A.ld = r; A.rows = n; A.cols = r;
        B.ptr = V; B.ld = r; B.rows = n; B.cols = r;
        gemm(f, st, GEMM_SET, C, A, false, B, true, n, n, r);
        FFB_CUDA(cudaStreamSynchronize(st));
        cudaFree(U);
        cudaFree(V);
        if (ia) cudaFree(ia);
        if (ib) cudaFree(ib);
        return FFB_OK;
    } catch (const Status& e) {
        return e.code;
    }
}

}  // extern "C"
