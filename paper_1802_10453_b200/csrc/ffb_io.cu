// ffb_io.cu -- matrix and factorization files.
//
// Two formats behind one C-ABI (include/ffldl_b200.h):
//   * text: byte-compatible with the reference's MatrixFile / FactorizationFile
//     (proj/include/ffldl/io.hpp:10-62, proj/src/io.cpp:39-222) -- "SymMat n p" / "Mat m n p"
//     and "Factorization n p / rank r / P ... / L ... / D ..." -- so files move between the
//     reference CLI and this one.  Parsing applies the same checks and raises the same
//     ParseError cases (io.cpp:15-36,39-67,104-146).
//   * binary: the same content without the decimal expansion (≈ 10 GB of text for L at
//     n = 32768 becomes n*r bytes at p <= 255).  Little-endian:
//       matrix:         "FFBMAT1\n" u64 rows u64 cols u64 modulus u32 symmetric u32 eb
//                       values[rows*cols] (eb bytes each) u64 fnv1a64(values)
//       factorization:  "FFBFAC1\n" u64 n u64 modulus u64 rank u32 eb u32 0
//                       perm int64[n]  L[n*rank] (eb bytes each)  dkind int32[rank]
//                       dval u64[rank]  dval2 u64[rank]  u64 fnv1a64(everything after the header)
//     eb is the smallest of 1/2/4/8 bytes holding modulus-1.
// Readers accept both formats (by the first bytes).  Host code only: files are host data.
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/ffldl_b200.h"

extern thread_local std::string g_last_error;  // ffb_engine.cu (ffb_last_error)

namespace {

struct IoError {
    int code;
    std::string msg;
};

[[noreturn]] void parse_error(const std::string& m) { throw IoError{FFB_PARSE_ERROR, m}; }

int eb_for(uint64_t modulus) {
    const uint64_t m = modulus - 1;
    return m < (1ull << 8) ? 1 : m < (1ull << 16) ? 2 : m < (1ull << 32) ? 4 : 8;
}

uint64_t get_elem(const void* base, size_t i, int eb) {
    switch (eb) {
    case 1: return ((const uint8_t*)base)[i];
    case 2: return ((const uint16_t*)base)[i];
    case 4: return ((const uint32_t*)base)[i];
    default: return ((const uint64_t*)base)[i];
    }
}
void put_elem(void* base, size_t i, int eb, uint64_t v) {
    switch (eb) {
    case 1: ((uint8_t*)base)[i] = (uint8_t)v; break;
    case 2: ((uint16_t*)base)[i] = (uint16_t)v; break;
    case 4: ((uint32_t*)base)[i] = (uint32_t)v; break;
    default: ((uint64_t*)base)[i] = v; break;
    }
}
int check_type(int t) {
    if (t == FFB_U8 || t == FFB_U16 || t == FFB_U32 || t == FFB_U64) return t;
    throw IoError{FFB_ERROR, "unknown element type"};
}

struct Fnv {
    uint64_t h = 0xcbf29ce484222325ull;
    void add(const void* p, size_t n) {
        const uint8_t* b = (const uint8_t*)p;
        for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
    }
};

// ---- whole-file input with a token scanner -------------------------------------------
struct Input {
    std::vector<char> buf;
    size_t pos = 0;

    explicit Input(const char* path) {
        FILE* f = strcmp(path, "-") == 0 ? stdin : fopen(path, "rb");
        if (!f) parse_error(std::string("cannot open '") + path + "' for reading");
        char tmp[1 << 16];
        size_t got;
        while ((got = fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
        if (f != stdin) fclose(f);
    }
    bool starts_with(const char* magic) const {
        const size_t n = strlen(magic);
        return buf.size() >= n && memcmp(buf.data(), magic, n) == 0;
    }
    void skip_ws() {
        while (pos < buf.size() && (buf[pos] == ' ' || buf[pos] == '\n' || buf[pos] == '\t' || buf[pos] == '\r'))
            ++pos;
    }
    std::string word(const char* what) {
        skip_ws();
        const size_t b = pos;
        while (pos < buf.size() && !(buf[pos] == ' ' || buf[pos] == '\n' || buf[pos] == '\t' || buf[pos] == '\r'))
            ++pos;
        if (b == pos) parse_error(std::string("expected ") + what);
        return std::string(buf.data() + b, pos - b);
    }
    // a decimal number like `in >> uint64_t` (io.cpp:15-20): digits only, no sign
    uint64_t number(const char* what) {
        skip_ws();
        if (pos >= buf.size() || buf[pos] < '0' || buf[pos] > '9') parse_error(std::string("expected ") + what);
        uint64_t v = 0;
        while (pos < buf.size() && buf[pos] >= '0' && buf[pos] <= '9') {
            const uint64_t d = (uint64_t)(buf[pos] - '0');
            if (v > (UINT64_MAX - d) / 10) parse_error(std::string("expected ") + what);
            v = v * 10 + d;
            ++pos;
        }
        return v;
    }
    void keyword(const char* kw) {
        const std::string w = word(kw);
        if (w != kw) parse_error(std::string("expected '") + kw + "', got '" + w + "'");
    }
    template <class T>
    T raw() {
        if (pos + sizeof(T) > buf.size()) parse_error("truncated binary file");
        T v;
        memcpy(&v, buf.data() + pos, sizeof(T));
        pos += sizeof(T);
        return v;
    }
    const char* bytes(size_t n) {
        if (pos + n > buf.size() || pos + n < pos) parse_error("truncated binary file");
        const char* p = buf.data() + pos;
        pos += n;
        return p;
    }
};

void check_residue(uint64_t v, uint64_t modulus, const char* what) {
    if (v >= modulus) parse_error(std::string(what) + " is not a canonical residue");
}

// ---- buffered output -------------------------------------------------------------------
struct Output {
    FILE* f;
    bool own;
    std::vector<char> buf;
    explicit Output(const char* path) {
        own = strcmp(path, "-") != 0;
        f = own ? fopen(path, "wb") : stdout;
        if (!f) throw IoError{FFB_ERROR, std::string("cannot open '") + path + "' for writing"};
        buf.reserve(1 << 20);
    }
    ~Output() {  // only reached without close() on an error path: never throw here
        if (f) {
            if (!buf.empty()) (void)!fwrite(buf.data(), 1, buf.size(), f);
            if (own) fclose(f);
        }
    }
    void flush() {
        if (!buf.empty() && fwrite(buf.data(), 1, buf.size(), f) != buf.size())
            throw IoError{FFB_ERROR, "write failed"};
        buf.clear();
    }
    void put(const char* s, size_t n) {
        buf.insert(buf.end(), s, s + n);
        if (buf.size() >= (1 << 20)) flush();
    }
    void str(const char* s) { put(s, strlen(s)); }
    void ch(char c) { put(&c, 1); }
    void num(uint64_t v) {
        char t[24];
        int k = 0;
        do {
            t[k++] = (char)('0' + v % 10);
            v /= 10;
        } while (v);
        char o[24];
        for (int i = 0; i < k; ++i) o[i] = t[k - 1 - i];
        put(o, (size_t)k);
    }
    template <class T>
    void raw(const T& v) { put((const char*)&v, sizeof(T)); }
    void close() {
        flush();
        if (own && fclose(f) != 0) {
            f = nullptr;
            throw IoError{FFB_ERROR, "close failed"};
        }
        f = nullptr;
    }
};

template <class F>
int io_guarded(F&& fn) {
    try {
        fn();
        return FFB_OK;
    } catch (const IoError& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return FFB_NO_MEMORY;
    }
}

void check_dkind(size_t r, const int32_t* dkind, const uint64_t* dval, const uint64_t* dval2, uint64_t modulus) {
    // the D block rules of io.cpp:125-145 on the per-column encoding
    size_t t = 0;
    while (t < r) {
        const int32_t k = dkind[t];
        if (k != FFB_D_SCALAR && k != FFB_D_ANTIDIAG_HEAD && k != FFB_D_ANTITRI_HEAD)
            parse_error("unknown D block tag");
        check_residue(dval[t], modulus, "D block value");
        if (dval[t] == 0) parse_error("D block pivot must be nonzero");
        if (k == FFB_D_ANTITRI_HEAD) {
            check_residue(dval2[t], modulus, "D block value");
            if (dval2[t] == 0) parse_error("AntiTri diagonal must be nonzero");
        }
        if (k == FFB_D_SCALAR) {
            ++t;
            continue;
        }
        if (t + 1 >= r) parse_error("D block orders exceed the rank");
        if (dkind[t + 1] != k + 1 || dval[t + 1] != dval[t] || (k == FFB_D_ANTITRI_HEAD && dval2[t + 1] != dval2[t]))
            parse_error("malformed two-column D block");
        t += 2;
    }
}

void check_perm(size_t n, const int64_t* perm) {
    std::vector<char> seen(n, 0);
    for (size_t i = 0; i < n; ++i) {
        if (perm[i] < 0 || (uint64_t)perm[i] >= n) parse_error("permutation image out of range");
        if (seen[(size_t)perm[i]]) parse_error("permutation images do not form a bijection");
        seen[(size_t)perm[i]] = 1;
    }
}

}  // namespace

extern "C" {

int ffb_matrix_read(const char* path, uint64_t* rows, uint64_t* cols, uint64_t* modulus, int* symmetric,
                    void* values, int elem_type) {
    return io_guarded([&] {
        Input in(path);
        uint64_t r = 0, c = 0, m = 0;
        int sym = 0;
        if (in.starts_with("FFBMAT1\n")) {
            in.pos = 8;
            r = in.raw<uint64_t>();
            c = in.raw<uint64_t>();
            m = in.raw<uint64_t>();
            sym = (int)in.raw<uint32_t>();
            const int eb = (int)in.raw<uint32_t>();
            if (m < 2) parse_error("modulus must be at least 2");
            if (eb != 1 && eb != 2 && eb != 4 && eb != 8) parse_error("bad element size");
            *rows = r, *cols = c, *modulus = m, *symmetric = sym;
            if (!values) return;
            const int et = check_type(elem_type);
            const char* data = in.bytes((size_t)(r * c * eb));
            Fnv h;
            h.add(data, (size_t)(r * c * eb));
            if (in.raw<uint64_t>() != h.h) parse_error("checksum mismatch");
            for (size_t i = 0; i < r * c; ++i) {
                const uint64_t v = get_elem(data, i, eb);
                check_residue(v, m, "matrix entry");
                put_elem(values, i, et, v);
            }
        } else {  // MatrixFile::parse, io.cpp:39-67
            const std::string head = in.word("matrix header");
            if (head == "SymMat") {
                sym = 1;
                r = c = in.number("dimension");
            } else if (head == "Mat") {
                r = in.number("row count");
                c = in.number("column count");
            } else {
                parse_error("unknown matrix header '" + head + "'");
            }
            m = in.number("modulus");
            if (m < 2) parse_error("modulus must be at least 2");
            *rows = r, *cols = c, *modulus = m, *symmetric = sym;
            if (!values) return;
            const int et = check_type(elem_type);
            for (size_t i = 0; i < r * c; ++i) {
                const uint64_t v = in.number("matrix entry");
                check_residue(v, m, "matrix entry");
                put_elem(values, i, et, v);
            }
        }
        if (sym)
            for (size_t i = 0; i < r; ++i)
                for (size_t j = 0; j < i; ++j)
                    if (get_elem(values, i * c + j, elem_type) != get_elem(values, j * c + i, elem_type))
                        parse_error("SymMat contents are not symmetric");
    });
}

int ffb_matrix_write(const char* path, int binary, uint64_t rows, uint64_t cols, uint64_t modulus, int symmetric,
                     const void* values, int elem_type) {
    return io_guarded([&] {
        const int et = check_type(elem_type);
        if (modulus < 2) throw IoError{FFB_ERROR, "modulus must be at least 2"};
        for (size_t i = 0; i < rows * cols; ++i)
            if (get_elem(values, i, et) >= modulus) throw IoError{FFB_ERROR, "matrix entry is not a canonical residue"};
        if (symmetric) {  // MatrixFile::from refuses an asymmetric SymMat (io.cpp:70-72)
            if (rows != cols) throw IoError{FFB_DIMENSION_MISMATCH, "SymMat must be square"};
            for (size_t i = 0; i < rows; ++i)
                for (size_t j = 0; j < i; ++j)
                    if (get_elem(values, i * cols + j, et) != get_elem(values, j * cols + i, et))
                        throw IoError{FFB_NOT_SYMMETRIC, "MatrixFile: SymMat requested for an asymmetric matrix"};
        }
        Output out(path);
        if (binary) {
            const int eb = eb_for(modulus);
            out.put("FFBMAT1\n", 8);
            out.raw(rows);
            out.raw(cols);
            out.raw(modulus);
            out.raw((uint32_t)(symmetric != 0));
            out.raw((uint32_t)eb);
            Fnv h;
            std::vector<char> row((size_t)cols * eb);
            for (size_t i = 0; i < rows; ++i) {
                for (size_t j = 0; j < cols; ++j) put_elem(row.data(), j, eb, get_elem(values, i * cols + j, et));
                h.add(row.data(), row.size());
                out.put(row.data(), row.size());
            }
            out.raw(h.h);
        } else {  // MatrixFile::emit, io.cpp:83-95
            if (symmetric) {
                out.str("SymMat ");
                out.num(rows);
            } else {
                out.str("Mat ");
                out.num(rows);
                out.ch(' ');
                out.num(cols);
            }
            out.ch(' ');
            out.num(modulus);
            out.ch('\n');
            for (size_t i = 0; i < rows; ++i) {
                for (size_t j = 0; j < cols; ++j) {
                    if (j) out.ch(' ');
                    out.num(get_elem(values, i * cols + j, et));
                }
                out.ch('\n');
            }
        }
        out.close();
    });
}

int ffb_factorization_read(const char* path, uint64_t* n, uint64_t* modulus, uint64_t* rank, int64_t* perm,
                           void* lower, int lower_type, int32_t* dkind, uint64_t* dval, uint64_t* dval2) {
    return io_guarded([&] {
        Input in(path);
        if (in.starts_with("FFBFAC1\n")) {
            in.pos = 8;
            const uint64_t N = in.raw<uint64_t>(), M = in.raw<uint64_t>(), R = in.raw<uint64_t>();
            const int eb = (int)in.raw<uint32_t>();
            in.raw<uint32_t>();
            if (M < 2) parse_error("modulus must be at least 2");
            if (R > N) parse_error("rank exceeds dimension");
            if (eb != 1 && eb != 2 && eb != 4 && eb != 8) parse_error("bad element size");
            *n = N, *modulus = M, *rank = R;
            if (!perm) return;
            const int et = check_type(lower_type);
            const size_t body = (size_t)(N * 8 + N * R * eb + R * 4 + R * 16);
            const char* data = in.bytes(body);
            Fnv h;
            h.add(data, body);
            if (in.raw<uint64_t>() != h.h) parse_error("checksum mismatch");
            memcpy(perm, data, N * 8);
            const char* L = data + N * 8;
            for (size_t i = 0; i < N * R; ++i) {
                const uint64_t v = get_elem(L, i, eb);
                check_residue(v, M, "L entry");
                put_elem(lower, i, et, v);
            }
            const char* d = L + N * R * eb;
            memcpy(dkind, d, R * 4);
            memcpy(dval, d + R * 4, R * 8);
            memcpy(dval2, d + R * 12, R * 8);
            check_perm(N, perm);
            check_dkind(R, dkind, dval, dval2, M);
            return;
        }
        // FactorizationFile::parse, io.cpp:104-146
        in.keyword("Factorization");
        const uint64_t N = in.number("dimension");
        const uint64_t M = in.number("modulus");
        if (M < 2) parse_error("modulus must be at least 2");
        in.keyword("rank");
        const uint64_t R = in.number("rank");
        if (R > N) parse_error("rank exceeds dimension");
        *n = N, *modulus = M, *rank = R;
        if (!perm) return;
        const int et = check_type(lower_type);
        in.keyword("P");
        for (size_t i = 0; i < N; ++i) {
            const uint64_t v = in.number("permutation image");
            if (v >= N) parse_error("permutation image out of range");
            perm[i] = (int64_t)v;
        }
        in.keyword("L");
        for (size_t i = 0; i < N * R; ++i) {
            const uint64_t v = in.number("L entry");
            check_residue(v, M, "L entry");
            put_elem(lower, i, et, v);
        }
        in.keyword("D");
        size_t order = 0;
        while (order < R) {
            const std::string tag = in.word("D block tag");
            if (tag.size() != 1 || (tag[0] != 'S' && tag[0] != 'A' && tag[0] != 'T'))
                parse_error("unknown D block tag '" + tag + "'");
            const uint64_t a = in.number("D block value");
            check_residue(a, M, "D block value");
            if (a == 0) parse_error("D block pivot must be nonzero");
            uint64_t b = 0;
            if (tag[0] == 'T') {
                b = in.number("D block value");
                check_residue(b, M, "D block value");
                if (b == 0) parse_error("AntiTri diagonal must be nonzero");
            }
            const size_t w = tag[0] == 'S' ? 1 : 2;
            if (order + w > R) parse_error("D block orders exceed the rank");
            const int32_t k0 = tag[0] == 'S' ? FFB_D_SCALAR : tag[0] == 'A' ? FFB_D_ANTIDIAG_HEAD : FFB_D_ANTITRI_HEAD;
            for (size_t u = 0; u < w; ++u) {
                dkind[order + u] = k0 + (int32_t)u;
                dval[order + u] = a;
                dval2[order + u] = b;
            }
            order += w;
        }
        check_perm(N, perm);  // Permutation::from_image (io.cpp:205-213)
    });
}

int ffb_factorization_write(const char* path, int binary, uint64_t n, uint64_t modulus, uint64_t rank,
                            const int64_t* perm, const void* lower, int lower_type, const int32_t* dkind,
                            const uint64_t* dval, const uint64_t* dval2) {
    return io_guarded([&] {
        const int et = check_type(lower_type);
        if (rank > n) throw IoError{FFB_DIMENSION_MISMATCH, "rank exceeds dimension"};
        Output out(path);
        if (binary) {
            const int eb = eb_for(modulus);
            out.put("FFBFAC1\n", 8);
            out.raw(n);
            out.raw(modulus);
            out.raw(rank);
            out.raw((uint32_t)eb);
            out.raw((uint32_t)0);
            Fnv h;
            h.add(perm, n * 8);
            out.put((const char*)perm, n * 8);
            std::vector<char> row((size_t)std::max<uint64_t>(rank, 1) * eb);
            for (size_t i = 0; i < n; ++i) {
                for (size_t j = 0; j < rank; ++j) put_elem(row.data(), j, eb, get_elem(lower, i * rank + j, et));
                h.add(row.data(), (size_t)rank * eb);
                out.put(row.data(), (size_t)rank * eb);
            }
            h.add(dkind, rank * 4);
            out.put((const char*)dkind, rank * 4);
            h.add(dval, rank * 8);
            out.put((const char*)dval, rank * 8);
            h.add(dval2, rank * 8);
            out.put((const char*)dval2, rank * 8);
            out.raw(h.h);
        } else {  // FactorizationFile::emit, io.cpp:177-198
            out.str("Factorization ");
            out.num(n);
            out.ch(' ');
            out.num(modulus);
            out.str("\nrank ");
            out.num(rank);
            out.str("\nP");
            for (size_t i = 0; i < n; ++i) {
                out.ch(' ');
                out.num((uint64_t)perm[i]);
            }
            out.str("\nL\n");
            for (size_t i = 0; i < n; ++i) {
                for (size_t j = 0; j < rank; ++j) {
                    if (j) out.ch(' ');
                    out.num(get_elem(lower, i * rank + j, et));
                }
                out.ch('\n');
            }
            out.str("D\n");
            for (size_t t = 0; t < rank;) {
                const int32_t k = dkind[t];
                out.ch(k == FFB_D_SCALAR ? 'S' : k == FFB_D_ANTIDIAG_HEAD ? 'A' : 'T');
                out.ch(' ');
                out.num(dval[t]);
                if (k == FFB_D_ANTITRI_HEAD) {
                    out.ch(' ');
                    out.num(dval2[t]);
                }
                out.ch('\n');
                t += k == FFB_D_SCALAR ? 1 : 2;
            }
        }
        out.close();
    });
}

}  // extern "C"
