// ffldl_b200 -- command line front end of the B200 library.
//
// Mirrors the reference CLI (proj/tools/ffldl_main.cpp:172-262): the subcommands gen,
// factor, verify and bench, their options, the RPM_LDLT_THRESHOLD fallback (:33-47) and the
// exit codes (:20-25).  Differences: files may also be binary (--binary; readers detect the
// format), `gen` draws the BASELINE.json families (--kind config1..config5) on the device,
// and `bench` times the device factorization.  Everything goes through the C-ABI of
// include/ffldl_b200.h; the factorization runs on the GPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "ffldl_b200.h"

namespace {

constexpr int exit_ok = 0;
constexpr int exit_verify_failed = 1;
constexpr int exit_usage = 2;
constexpr int exit_not_symmetric = 3;
constexpr int exit_parse = 4;
constexpr int exit_bench = 5;

struct Failure {
    int status;
    std::string msg;
};

void check(int s) {
    if (s != FFB_OK) {
        const char* d = ffb_last_error();
        throw Failure{s, std::string(ffb_status_string(s)) + (d && *d ? std::string(": ") + d : "")};
    }
}
void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw Failure{FFB_CUDA_ERROR, cudaGetErrorString(e)};
}

int usage(const std::string& msg) {
    std::cerr << msg << "\n"
              << "usage: ffldl_b200 gen --kind K -n N [--rank R] [--modulus P] [--seed S] [-o FILE] [--binary]\n"
              << "       ffldl_b200 factor -i FILE [-o FILE] [--variant V] [--threshold T] [--binary]\n"
              << "       ffldl_b200 verify -i FILE -f FILE [--check-rpm]\n"
              << "       ffldl_b200 bench --kind K -n N [N ...] [--modulus P] [--seed S] [--variant V]\n"
              << "                        [--threshold T] [-o FILE]\n"
              << "kinds: config1..config5 (BASELINE.json families), dense, hollow, rpm-half, generic\n";
    return exit_usage;
}

struct Args {
    std::string cmd;
    std::map<std::string, std::vector<std::string>> opt;
    bool has(const std::string& k) const { return opt.count(k) > 0; }
    std::string get(const std::string& k, const std::string& dflt) const {
        auto it = opt.find(k);
        return it == opt.end() || it->second.empty() ? dflt : it->second.back();
    }
};

bool parse_u64(const std::string& s, uint64_t& v) {
    if (s.empty() || s.find_first_not_of("0123456789") != std::string::npos) return false;
    v = std::strtoull(s.c_str(), nullptr, 10);
    return true;
}

int variant_from_name(const std::string& name) {
    if (name == "recursive") return FFB_VARIANT_RECURSIVE;
    if (name == "crout") return FFB_VARIANT_CROUT;
    return FFB_VARIANT_CASCADE;
}

// --threshold wins; otherwise RPM_LDLT_THRESHOLD; a malformed value is a usage error
// (ffldl_main.cpp:33-47).  Default 64 (sytrf.hpp:14-17).
bool resolve_threshold(const Args& a, uint64_t& t) {
    t = 64;
    if (a.has("--threshold")) return parse_u64(a.get("--threshold", ""), t);
    const char* env = std::getenv("RPM_LDLT_THRESHOLD");
    if (!env) return true;
    if (!parse_u64(env, t)) {
        std::cerr << "RPM_LDLT_THRESHOLD is not a nonnegative integer: '" << env << "'\n";
        return false;
    }
    return true;
}

// kind -> (config family of csrc/ffb_gen.cu, rank parameter)
bool kind_config(const std::string& kind, uint64_t n, uint64_t rank, int& config, uint64_t& r) {
    r = 0;
    if (kind.size() == 7 && kind.rfind("config", 0) == 0 && kind[6] >= '1' && kind[6] <= '5') {
        config = kind[6] - '0';
        if (config == 2 || config == 5) r = rank ? rank : n / 2;
        return true;
    }
    if (kind == "dense" || kind == "dense-random") config = 1;
    else if (kind == "hollow") config = 4;
    else if (kind == "rpm-half" || kind == "rpm-random") { config = 5; r = rank ? rank : n / 2; }
    else if (kind == "rpm-full") { config = 5; r = n; }
    else if (kind == "generic") { config = 2; r = rank ? rank : n; }
    else return false;
    return true;
}

int elem_type_for(uint64_t p) { return p <= 256 ? FFB_U8 : p <= 65536 ? FFB_U16 : FFB_U32; }

struct Ctx {
    ffb_context* c = nullptr;
    Ctx() { check(ffb_create(&c, 0)); }
    ~Ctx() { ffb_destroy(c); }
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { cuda(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
    ~DevBuf() { cudaFree(p); }
};

// device matrix of the family, downloaded as uint32 residues
std::vector<uint32_t> generate(Ctx& ctx, int config, uint64_t n, uint64_t r, uint64_t p, uint64_t seed) {
    DevBuf<uint32_t> d(n * n);
    check(ffb_generate_device(ctx.c, config, n, r, p, seed, d.p));
    std::vector<uint32_t> h(n * n);
    cuda(cudaMemcpy(h.data(), d.p, n * n * 4, cudaMemcpyDeviceToHost));
    return h;
}

int run_gen(const Args& a) {
    uint64_t n = 0, rank = 0, p = 8388593, seed = 1;  // modulus default as ffldl_main.cpp:179
    if (!parse_u64(a.get("-n", ""), n)) return usage("gen: -n is required");
    if (a.has("--rank") && !parse_u64(a.get("--rank", ""), rank)) return usage("gen: bad --rank");
    if (a.has("--modulus") && !parse_u64(a.get("--modulus", ""), p)) return usage("gen: bad --modulus");
    if (a.has("--seed") && !parse_u64(a.get("--seed", ""), seed)) return usage("gen: bad --seed");
    if (rank > n) {
        std::cerr << "requested rank " << rank << " exceeds dimension " << n << '\n';
        return exit_usage;
    }
    int config = 0;
    uint64_t r = 0;
    if (!kind_config(a.get("--kind", ""), n, rank, config, r)) return usage("gen: unknown --kind");
    Ctx ctx;
    std::vector<uint32_t> h = generate(ctx, config, n, r, p, seed);
    check(ffb_matrix_write(a.get("-o", "-").c_str(), a.has("--binary"), n, n, p, 1, h.data(), FFB_U32));
    return exit_ok;
}

int run_factor(const Args& a) {
    if (!a.has("-i")) return usage("factor: -i is required");
    uint64_t t = 64;
    if (!resolve_threshold(a, t)) return exit_usage;
    const std::string in = a.get("-i", "");
    uint64_t rows = 0, cols = 0, p = 0;
    int sym = 0;
    check(ffb_matrix_read(in.c_str(), &rows, &cols, &p, &sym, nullptr, FFB_U64));
    const int et = elem_type_for(p);
    std::vector<char> vals((size_t)(rows * cols * et) + 1);
    check(ffb_matrix_read(in.c_str(), &rows, &cols, &p, &sym, vals.data(), et));
    if (rows != cols) throw Failure{FFB_DIMENSION_MISMATCH, "ldlt: matrix must be square"};
    Ctx ctx;
    const size_t n = rows;
    std::vector<int64_t> perm(std::max<size_t>(n, 1));
    std::vector<char> lower(std::max<size_t>(n * n * et, 1));
    std::vector<int32_t> kind(std::max<size_t>(n, 1));
    std::vector<uint64_t> v(std::max<size_t>(n, 1)), v2(std::max<size_t>(n, 1));
    size_t r = 0;
    check(ffb_ldlt_compact(ctx.c, p, n, vals.data(), et, variant_from_name(a.get("--variant", "cascade")), t,
                           perm.data(), lower.data(), et, kind.data(), v.data(), v2.data(), &r));
    check(ffb_factorization_write(a.get("-o", "-").c_str(), a.has("--binary"), n, p, r, perm.data(), lower.data(),
                                  et, kind.data(), v.data(), v2.data()));
    return exit_ok;
}

// Rank profile matrix of A by incremental row echelon form (verification only): the
// column rank profile of the first i rows grows by at most the leading column c_i of
// row i reduced against the reduced basis, and R(i, c_i) = 1 (rpmtools.cpp:43-59's
// inclusion-exclusion on leading ranks, in O(n^3)).
std::vector<int64_t> rpm_partners(const std::vector<uint64_t>& A, size_t n, uint64_t p) {
    auto mul = [p](uint64_t x, uint64_t y) { return (uint64_t)((unsigned __int128)x * y % p); };
    auto inv = [&](uint64_t x) {
        uint64_t r = 1, b = x, e = p - 2;
        while (e) {
            if (e & 1) r = mul(r, b);
            b = mul(b, b);
            e >>= 1;
        }
        return r;
    };
    std::vector<std::vector<uint64_t>> basis;
    std::vector<size_t> piv;
    std::vector<int64_t> partner(n, -1);
    for (size_t i = 0; i < n; ++i) {
        std::vector<uint64_t> row(A.begin() + i * n, A.begin() + (i + 1) * n);
        for (size_t b = 0; b < basis.size(); ++b) {
            const uint64_t f = row[piv[b]];
            if (!f) continue;
            for (size_t j = 0; j < n; ++j) row[j] = (row[j] + p - mul(f, basis[b][j])) % p;
        }
        size_t c = 0;
        while (c < n && row[c] == 0) ++c;
        if (c == n) continue;
        const uint64_t s = inv(row[c]);
        for (auto& x : row) x = mul(x, s);
        for (size_t b = 0; b < basis.size(); ++b) {  // keep the basis reduced at c
            const uint64_t f = basis[b][c];
            if (!f) continue;
            for (size_t j = 0; j < n; ++j) basis[b][j] = (basis[b][j] + p - mul(f, row[j])) % p;
        }
        basis.push_back(row);
        piv.push_back(c);
        partner[i] = (int64_t)c;
    }
    return partner;
}

int run_verify(const Args& a) {
    if (!a.has("-i") || !a.has("-f")) return usage("verify: -i and -f are required");
    const std::string mp = a.get("-i", ""), fp = a.get("-f", "");
    uint64_t rows = 0, cols = 0, p = 0, n = 0, pf = 0, r = 0;
    int sym = 0;
    check(ffb_matrix_read(mp.c_str(), &rows, &cols, &p, &sym, nullptr, FFB_U64));
    check(ffb_factorization_read(fp.c_str(), &n, &pf, &r, nullptr, nullptr, FFB_U64, nullptr, nullptr, nullptr));
    if (rows != cols || n != rows) throw Failure{FFB_PARSE_ERROR, "matrix and factorization dimensions disagree"};
    if (pf != p) throw Failure{FFB_PARSE_ERROR, "factorization bound to a field with another modulus"};
    std::vector<uint64_t> A(n * n);
    check(ffb_matrix_read(mp.c_str(), &rows, &cols, &p, &sym, A.data(), FFB_U64));
    std::vector<int64_t> perm(std::max<uint64_t>(n, 1));
    std::vector<uint64_t> L(std::max<uint64_t>(n * r, 1)), v(std::max<uint64_t>(r, 1)), v2(std::max<uint64_t>(r, 1));
    std::vector<int32_t> kind(std::max<uint64_t>(r, 1));
    check(ffb_factorization_read(fp.c_str(), &n, &pf, &r, perm.data(), L.data(), FFB_U64, kind.data(), v.data(),
                                 v2.data()));
    // unit lower triangular in the top rank rows (ffldl_main.cpp:111-120)
    for (size_t i = 0; i < r; ++i)
        for (size_t j = i; j < r; ++j)
            if (L[i * r + j] != (i == j ? 1 % p : 0)) {
                std::cout << "FAIL: L is not unit lower triangular in its top rank rows\n";
                return exit_verify_failed;
            }
    if (p >= (1ull << 31)) throw Failure{FFB_UNSUPPORTED, "verify: device residues need p < 2^31"};
    Ctx ctx;
    std::vector<uint32_t> A32(A.begin(), A.end()), L32(L.begin(), L.end()), v32(v.begin(), v.end()),
        v232(v2.begin(), v2.end());
    std::vector<int32_t> perm32(perm.begin(), perm.end());
    DevBuf<uint32_t> dA(n * n), dL(n * std::max<uint64_t>(r, 1)), dv(r), dv2(r);
    DevBuf<int32_t> dp(n), dk(r), dpart(n);
    cuda(cudaMemcpy(dA.p, A32.data(), n * n * 4, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(dL.p, L32.data(), n * r * 4, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(dp.p, perm32.data(), n * 4, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(dk.p, kind.data(), r * 4, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(dv.p, v32.data(), r * 4, cudaMemcpyHostToDevice));
    cuda(cudaMemcpy(dv2.p, v232.data(), r * 4, cudaMemcpyHostToDevice));
    uint64_t bad = 0;
    check(ffb_verify_device(ctx.c, p, n, dA.p, n, dp.p, dL.p, std::max<uint64_t>(r, 1), dk.p, dv.p, dv2.p, r, &bad));
    if (bad) {
        std::cout << "FAIL: factorization does not reconstruct the matrix\n";
        return exit_verify_failed;
    }
    const bool check_rpm = a.has("--check-rpm");
    if (check_rpm) {
        check(ffb_pivoting_partners_device(ctx.c, n, dp.p, dk.p, r, dpart.p));
        std::vector<int32_t> got(n);
        cuda(cudaMemcpy(got.data(), dpart.p, n * 4, cudaMemcpyDeviceToHost));
        const std::vector<int64_t> want = rpm_partners(A, n, p);
        for (size_t i = 0; i < n; ++i)
            if (got[i] != want[i]) {
                std::cout << "FAIL: pivoting matrix does not match the rank profile matrix\n";
                return exit_verify_failed;
            }
    }
    std::cout << "OK: rank " << r << (check_rpm ? ", rank profile matrix revealed" : "") << '\n';
    return exit_ok;
}

// CSV like write_csv (genbench.cpp:187-196); mul_count is not kept on the device (0).
int run_bench(const Args& a) {
    uint64_t p = 8388593, seed = 1, t = 64;
    if (a.has("--modulus") && !parse_u64(a.get("--modulus", ""), p)) return usage("bench: bad --modulus");
    if (a.has("--seed") && !parse_u64(a.get("--seed", ""), seed)) return usage("bench: bad --seed");
    if (!resolve_threshold(a, t)) return exit_usage;
    auto it = a.opt.find("-n");
    if (it == a.opt.end() || it->second.empty()) return usage("bench: -n is required");
    const std::string vname = a.get("--variant", "cascade");
    std::ostringstream csv;
    csv << "n,r,field,variant,seconds,mul_count,effective_gfops\n";
    try {
        Ctx ctx;
        for (const std::string& s : it->second) {
            uint64_t n = 0, r = 0;
            int config = 0;
            if (!parse_u64(s, n)) return usage("bench: bad -n");
            if (!kind_config(a.get("--kind", ""), n, 0, config, r)) return usage("bench: unknown --kind");
            DevBuf<uint32_t> A(n * n), L(n * n);
            DevBuf<int32_t> perm(n), kind(n);
            DevBuf<uint32_t> v(n), v2(n);
            check(ffb_generate_device(ctx.c, config, n, r, p, seed, A.p));
            size_t rank = 0;
            cuda(cudaDeviceSynchronize());
            const auto t0 = std::chrono::steady_clock::now();
            check(ffb_ldlt_device(ctx.c, p, n, A.p, n, variant_from_name(vname), t, perm.p, L.p, n, kind.p, v.p,
                                  v2.p, &rank));
            const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            const double rr = (double)rank, nn = (double)n;
            const double gf = (rr * rr * rr / 3 + nn * nn * rr - rr * rr * nn) / 1e9 / sec;  // genbench.cpp
            char line[256];
            snprintf(line, sizeof line, "%llu,%zu,%llu,%s,%.6e,0,%.6e\n", (unsigned long long)n, rank,
                     (unsigned long long)p, vname == "crout" ? "Crout" : vname == "recursive" ? "Recursive" : "Cascade",
                     sec, gf);
            csv << line;
        }
    } catch (const Failure& f) {
        std::cerr << "bench failed: " << f.msg << '\n';
        return exit_bench;
    }
    const std::string out = a.get("-o", "-");
    if (out == "-") {
        std::cout << csv.str();
    } else {
        FILE* fh = std::fopen(out.c_str(), "wb");
        if (!fh) {
            std::cerr << "cannot open '" << out << "' for writing\n";
            return exit_usage;
        }
        std::fputs(csv.str().c_str(), fh);
        std::fclose(fh);
    }
    return exit_ok;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage("a subcommand is required");
    Args a;
    a.cmd = argv[1];
    static const char* flags[] = {"--binary", "--check-rpm"};
    std::string key;
    for (int i = 2; i < argc; ++i) {
        std::string s = argv[i];
        if (s == "--output") s = "-o";
        if (s == "--input") s = "-i";
        if (s == "--size") s = "-n";
        if (s == "--factorization") s = "-f";
        if (s.size() > 1 && s[0] == '-' && !(s.size() > 1 && std::isdigit((unsigned char)s[1]))) {
            bool flag = false;
            for (const char* f : flags) flag |= s == f;
            a.opt[s];
            key = flag ? "" : s;
        } else if (!key.empty()) {
            a.opt[key].push_back(s);
            if (key != "-n") key.clear();
        } else {
            return usage("unexpected argument '" + s + "'");
        }
    }
    try {
        if (a.cmd == "gen") return run_gen(a);
        if (a.cmd == "factor") return run_factor(a);
        if (a.cmd == "verify") return run_verify(a);
        if (a.cmd == "bench") return run_bench(a);
        return usage("unknown subcommand '" + a.cmd + "'");
    } catch (const Failure& f) {
        std::cerr << f.msg << '\n';
        if (f.status == FFB_NOT_SYMMETRIC) return exit_not_symmetric;
        return exit_parse;  // ParseError, NotPrime and other ffldl::Error (ffldl_main.cpp:252-261)
    }
}
