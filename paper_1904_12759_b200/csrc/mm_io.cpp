// §8f rows f1 and f3, host side.
//
//  * Matrix Market coordinate I/O: load_matrix_market / write_matrix_market
//    (proj/src/matrix_market.cpp:51-207, contract in
//    proj/include/expmc/matrix_market.hpp:9-18).  Same header rules, skip
//    rules, number syntax (std::from_chars after skipping ' ', '\t', '\r')
//    and messages ("path:line: what").  The body is parsed by all host
//    cores: pass 1 counts lines and entry lines per byte range, a prefix sum
//    gives each range its first line number and entry index, pass 2 parses
//    in place.  The earliest failing line wins, so the reported error is the
//    sequential reader's.  The general-symmetry fold and from_entries run on
//    the GPU (from_entries.cu, driven from api.cu).
//  * Binary CSR cache (f3: "a binary CSR cache format" for generated
//    inputs): a 64-byte header plus row_ptr, col, val and diag, with a
//    block-parallel 64-bit checksum.
//
// Deviation: node ids are 32-bit on the device, so dimensions >= 2^32 are
// rejected at the size line (the reference would truncate its NodeId casts).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <system_error>
#include <thread>
#include <vector>

#include "host_io.h"

namespace expmc_b200 {

std::string mm_message(const std::string& path, uint64_t line, const std::string& what) {
    return path + ":" + std::to_string(line) + ": " + what;
}

namespace {

unsigned pick_threads(unsigned req, uint64_t work, uint64_t grain) {
    unsigned t = req ? req : std::max(1u, std::thread::hardware_concurrency());
    const uint64_t useful = work / grain + 1;
    return (unsigned)std::min<uint64_t>(t, useful);
}

template <class F>
void run_parallel(unsigned T, F&& f) {
    if (T <= 1) {
        f(0u);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T);
    for (unsigned k = 0; k < T; ++k) th.emplace_back([&f, k] { f(k); });
    for (auto& t : th) t.join();
}

struct Mapped {
    const char* p = nullptr;
    size_t size = 0;
    int fd = -1;
    ~Mapped() {
        if (p) munmap(const_cast<char*>(p), size);
        if (fd >= 0) close(fd);
    }
};

void map_file(const char* path, Mapped& m) {
    m.fd = open(path, O_RDONLY);
    if (m.fd < 0) throw std::runtime_error(std::string("cannot open ") + path);
    struct stat st;
    if (fstat(m.fd, &st) != 0) throw std::runtime_error(std::string("cannot open ") + path);
    if (!S_ISREG(st.st_mode)) return;  // a directory reads as an empty stream
    m.size = (size_t)st.st_size;
    if (!m.size) return;
    void* p = mmap(nullptr, m.size, PROT_READ, MAP_PRIVATE, m.fd, 0);
    if (p == MAP_FAILED) throw std::runtime_error(std::string("cannot open ") + path);
    madvise(p, m.size, MADV_SEQUENTIAL);
    m.p = static_cast<const char*>(p);
}

// std::getline over [pos, end): false at end of input.
bool next_line(const char* base, size_t end, size_t& pos, const char*& b, const char*& e) {
    if (pos >= end) return false;
    b = base + pos;
    const void* nl = memchr(b, '\n', end - pos);
    e = nl ? static_cast<const char*>(nl) : base + end;
    pos = (size_t)(e - base) + (nl ? 1 : 0);
    return true;
}

// skip_ws / parse_u64 / parse_double, matrix_market.cpp:28-47
const char* skip_ws(const char* p, const char* end) {
    while (p != end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
    return p;
}
bool parse_u64(const char*& p, const char* end, uint64_t& out) {
    p = skip_ws(p, end);
    auto [next, ec] = std::from_chars(p, end, out);
    if (ec != std::errc{} || next == p) return false;
    p = next;
    return true;
}
bool parse_double(const char*& p, const char* end, double& out) {
    p = skip_ws(p, end);
    auto [next, ec] = std::from_chars(p, end, out);
    if (ec != std::errc{} || next == p) return false;
    p = next;
    return true;
}

// banner tokens: lower-cased (C locale), split on isspace like operator>>
std::vector<std::string> banner_tokens(const char* b, const char* e) {
    std::vector<std::string> t;
    std::string cur;
    for (const char* p = b; p != e; ++p) {
        const unsigned char ch = (unsigned char)*p;
        if (ch == ' ' || ch == '\t' || ch == '\n' || ch == '\v' || ch == '\f' || ch == '\r') {
            if (!cur.empty()) t.push_back(cur), cur.clear();
        } else {
            cur.push_back((ch >= 'A' && ch <= 'Z') ? (char)(ch + 32) : (char)ch);
        }
    }
    if (!cur.empty()) t.push_back(cur);
    t.resize(std::max<size_t>(t.size(), 5));
    return t;
}

inline bool entry_line(const char* b, const char* e) { return b != e && *b != '%'; }

}  // namespace

void mm_parse(const char* path, expmc_mm& out, unsigned threads) {
    const std::string P = path ? path : "";
    if (!path) throw std::runtime_error("cannot open ");
    Mapped m;
    map_file(path, m);
    auto fail = [&](uint64_t line, const std::string& what) {
        throw std::runtime_error(mm_message(P, line, what));
    };
    const char* base = m.p;
    const size_t size = m.size;
    size_t pos = 0;
    uint64_t lineno = 0;
    const char *b = nullptr, *e = nullptr;

    // banner (matrix_market.cpp:58-79)
    if (!next_line(base, size, pos, b, e)) fail(1, "empty file");
    ++lineno;
    const auto tok = banner_tokens(b, e);
    const std::string &magic = tok[0], &object = tok[1], &format = tok[2], &field = tok[3],
                      &symmetry = tok[4];
    if (magic != "%%matrixmarket" || object != "matrix")
        fail(lineno, "not a MatrixMarket matrix file");
    if (format != "coordinate")
        fail(lineno, "unsupported format '" + format + "' (coordinate only)");
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer")
        fail(lineno, "unsupported field '" + field + "'");
    const bool general = symmetry == "general";
    if (!general && symmetry != "symmetric")
        fail(lineno, "unsupported symmetry '" + symmetry + "'");

    // size line after any comments (matrix_market.cpp:81-104)
    uint64_t rows = 0, cols = 0, nnz = 0;
    for (;;) {
        if (!next_line(base, size, pos, b, e)) fail(lineno + 1, "missing size line");
        ++lineno;
        if (!entry_line(b, e)) continue;
        const char* p = b;
        if (!parse_u64(p, e, rows) || !parse_u64(p, e, cols) || !parse_u64(p, e, nnz))
            fail(lineno, "malformed size line");
        break;
    }
    if (rows == 0 || cols == 0) fail(lineno, "zero dimension");
    if (rows != cols)
        fail(lineno, "matrix is not square (" + std::to_string(rows) + " x " +
                         std::to_string(cols) + ")");
    if (rows >= (1ull << 32)) fail(lineno, "dimension exceeds 32-bit node ids");
    const uint64_t n = rows;

    // body: ranges starting at line starts
    const size_t body = pos, blen = size - pos;
    const unsigned T = pick_threads(threads, blen, 1u << 20);
    std::vector<size_t> cut(T + 1);
    cut[0] = body;
    cut[T] = size;
    for (unsigned k = 1; k < T; ++k) {
        size_t c = body + blen / T * k;
        if (c < cut[k - 1]) c = cut[k - 1];
        if (c > body && c < size && base[c - 1] != '\n') {
            const void* nl = memchr(base + c, '\n', size - c);
            c = nl ? (size_t)(static_cast<const char*>(nl) - base) + 1 : size;
        }
        cut[k] = c;
    }
    std::vector<uint64_t> nlines(T, 0), nent(T, 0);
    run_parallel(T, [&](unsigned k) {
        size_t q = cut[k];
        const char *lb, *le;
        uint64_t L = 0, E = 0;
        while (q < cut[k + 1] && next_line(base, cut[k + 1], q, lb, le)) {
            ++L;
            E += entry_line(lb, le);
        }
        nlines[k] = L;
        nent[k] = E;
    });
    std::vector<uint64_t> line0(T), ent0(T);
    uint64_t L = lineno, E = 0;
    for (unsigned k = 0; k < T; ++k) {
        line0[k] = L;
        ent0[k] = E;
        L += nlines[k];
        E += nent[k];
    }
    const uint64_t take = std::min(nnz, E);
    out.r.assign(take, 0);
    out.c.assign(take, 0);
    out.w.assign(take, 1.0);
    std::vector<uint64_t> err_line(T, ~0ull), last(T, 0);
    std::vector<const char*> err_what(T, nullptr);
    run_parallel(T, [&](unsigned k) {
        if (ent0[k] >= take) return;
        size_t q = cut[k];
        const char *lb, *le;
        uint64_t line = line0[k], idx = ent0[k];
        while (idx < take && next_line(base, cut[k + 1], q, lb, le)) {
            ++line;
            if (!entry_line(lb, le)) continue;
            // one entry (matrix_market.cpp:119-130)
            const char* p = lb;
            uint64_t i = 0, j = 0;
            double w = 1.0;
            const char* what = nullptr;
            if (!parse_u64(p, le, i) || !parse_u64(p, le, j))
                what = "malformed entry";
            else if (!pattern && !parse_double(p, le, w))
                what = "malformed entry value";
            else if (i == 0 || j == 0 || i > n || j > n)
                what = "index out of range";
            if (what) {
                err_line[k] = line;
                err_what[k] = what;
                return;
            }
            out.r[idx] = (uint32_t)(i - 1);
            out.c[idx] = (uint32_t)(j - 1);
            out.w[idx] = w;
            if (++idx == take) last[k] = line;
        }
    });
    for (unsigned k = 0; k < T; ++k)  // ranges are in file order: first hit is earliest
        if (err_line[k] != ~0ull) fail(err_line[k], err_what[k]);
    if (E < nnz)
        fail(L + 1, "unexpected end of file: expected " + std::to_string(nnz) +
                        " entries, got " + std::to_string(E));
    uint64_t last_line = lineno;
    for (unsigned k = 0; k < T; ++k)
        if (last[k]) last_line = last[k];
    out.path = P;
    out.n = n;
    out.general = general;
    out.pattern = pattern;
    out.last_line = last_line;
}

namespace {

// ---------------------------------------------------------------- writer
void write_mm(const char* path, uint64_t n, const uint64_t* rp, const uint32_t* col,
              const double* val, const double* diag) {
    const std::string P = path;
    if (n && !rp) throw std::invalid_argument("row_ptr is null");
    const uint64_t nnz = n ? rp[n] : 0;
    if (nnz && (!col || !val)) throw std::invalid_argument("col / val are null");
    // entries = diagonal + upper triangle, sorted by (row, col)
    // (SparseSymmetric::entries_, sparse_matrix.cpp:41-48)
    uint64_t count = 0;
    bool pattern = true;
    for (uint64_t i = 0; i < n; ++i) {
        if (diag && diag[i] != 0.0) {
            ++count;
            pattern &= diag[i] == 1.0;
        }
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (col[k] > i) {
                ++count;
                pattern &= val[k] == 1.0;
            }
    }
    FILE* f = fopen(path, "wb");
    if (!f) throw std::runtime_error("cannot open " + P + " for write");
    bool ok = fprintf(f, "%%%%MatrixMarket matrix coordinate %s symmetric\n%llu %llu %llu\n",
                      pattern ? "pattern" : "real", (unsigned long long)n,
                      (unsigned long long)n, (unsigned long long)count) > 0;
    // rows in blocks of ~2^22 stored entries, formatted by all cores, written in order
    const unsigned T = pick_threads(0, nnz, 1u << 18);
    const uint64_t grain = 1ull << 22;
    uint64_t i0 = 0;
    std::vector<std::string> buf(T);
    while (ok && i0 < n) {
        std::vector<uint64_t> lo(T + 1, n);
        lo[0] = i0;
        for (unsigned k = 1; k <= T; ++k) {
            uint64_t i = lo[k - 1];
            const uint64_t stop = rp[i] + grain;
            while (i < n && rp[i] < stop) ++i;
            if (i == lo[k - 1] && i < n) ++i;
            lo[k] = i;
        }
        run_parallel(T, [&](unsigned k) {
            std::string& s = buf[k];
            s.clear();
            char tmp[96];
            auto emit = [&](uint64_t r, uint64_t c, double w) {  // lower triangle, 1-based
                char* p = tmp;
                p = std::to_chars(p, tmp + sizeof(tmp), c + 1).ptr;
                *p++ = ' ';
                p = std::to_chars(p, tmp + sizeof(tmp), r + 1).ptr;
                if (!pattern) {
                    *p++ = ' ';
                    p = std::to_chars(p, tmp + sizeof(tmp), w).ptr;
                }
                *p++ = '\n';
                s.append(tmp, p);
            };
            for (uint64_t i = lo[k]; i < lo[k + 1]; ++i) {
                if (diag && diag[i] != 0.0) emit(i, i, diag[i]);
                for (uint64_t q = rp[i]; q < rp[i + 1]; ++q)
                    if (col[q] > i) emit(i, col[q], val[q]);
            }
        });
        for (unsigned k = 0; k < T && ok; ++k)
            ok = fwrite(buf[k].data(), 1, buf[k].size(), f) == buf[k].size();
        i0 = lo[T];
    }
    ok = (fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write failed for " + P);
}

// ------------------------------------------------------- binary CSR cache
constexpr char kMagic[8] = {'E', 'X', 'P', 'M', 'C', 'C', 'S', 'R'};
constexpr uint32_t kVersion = 1;

struct CacheHeader {
    char magic[8];
    uint32_t version;
    uint32_t flags;
    uint64_t n, nnz, checksum;
    uint64_t reserved[3];
};
static_assert(sizeof(CacheHeader) == 64, "header size");

inline uint64_t mix(uint64_t h, uint64_t x) {
    h ^= x * 0x9E3779B97F4A7C15ull;
    h = (h ^ (h >> 29)) * 0xBF58476D1CE4E5B9ull;
    return h ^ (h >> 32);
}

// hash of a byte range as zero-padded 64-bit words, in fixed 1 MiB blocks
// (independent of the thread count)
uint64_t hash_bytes(const void* data, uint64_t bytes) {
    const uint64_t block = 1ull << 20;
    const uint64_t nb = (bytes + block - 1) / block;
    std::vector<uint64_t> bh(nb);
    const unsigned T = pick_threads(0, bytes, 1u << 24);
    run_parallel(T, [&](unsigned k) {
        for (uint64_t b = k; b < nb; b += T) {
            const char* p = static_cast<const char*>(data) + b * block;
            const uint64_t len = std::min(block, bytes - b * block);
            uint64_t h = 0x243F6A8885A308D3ull ^ b;
            uint64_t q = 0;
            for (; q + 8 <= len; q += 8) {
                uint64_t x;
                memcpy(&x, p + q, 8);
                h = mix(h, x);
            }
            if (q < len) {
                uint64_t x = 0;
                memcpy(&x, p + q, len - q);
                h = mix(h, x);
            }
            bh[b] = mix(h, len);
        }
    });
    uint64_t h = mix(0x13198A2E03707344ull, bytes);
    for (uint64_t x : bh) h = mix(h, x);
    return h;
}

uint64_t csr_checksum(uint64_t n, uint64_t nnz, const uint64_t* rp, const uint32_t* col,
                      const double* val, const double* diag) {
    uint64_t h = mix(mix(0, n), nnz);
    h = mix(h, hash_bytes(rp, (n + 1) * 8));
    h = mix(h, hash_bytes(col, nnz * 4));
    h = mix(h, hash_bytes(val, nnz * 8));
    h = mix(h, hash_bytes(diag, n * 8));
    return h;
}

void save_csr(const char* path, uint64_t n, const uint64_t* rp, const uint32_t* col,
              const double* val, const double* diag) {
    const std::string P = path;
    if (!rp) throw std::invalid_argument("row_ptr is null");
    const uint64_t nnz = rp[n];
    if (nnz && (!col || !val)) throw std::invalid_argument("col / val are null");
    std::vector<double> zero;
    if (!diag) {
        zero.assign(n, 0.0);
        diag = zero.data();
    }
    CacheHeader h{};
    memcpy(h.magic, kMagic, 8);
    h.version = kVersion;
    h.n = n;
    h.nnz = nnz;
    h.checksum = csr_checksum(n, nnz, rp, col, val, diag);
    FILE* f = fopen(path, "wb");
    if (!f) throw std::runtime_error("cannot open " + P + " for write");
    const uint64_t pad = (8 - (nnz * 4) % 8) % 8, zeros = 0;
    bool ok = fwrite(&h, sizeof h, 1, f) == 1 && fwrite(rp, 8, n + 1, f) == n + 1 &&
              fwrite(col, 4, nnz, f) == nnz && fwrite(&zeros, 1, pad, f) == pad &&
              fwrite(val, 8, nnz, f) == nnz && fwrite(diag, 8, n, f) == n;
    ok = (fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write failed for " + P);
}

expmc_csr* load_csr(const char* path) {
    const std::string P = path;
    FILE* f = fopen(path, "rb");
    if (!f) throw std::runtime_error("cannot open " + P);
    struct Closer {
        FILE* f;
        ~Closer() { fclose(f); }
    } closer{f};
    CacheHeader h{};
    if (fread(&h, sizeof h, 1, f) != 1 || memcmp(h.magic, kMagic, 8) != 0)
        throw std::runtime_error(P + ": not an expmc CSR cache file");
    if (h.version != kVersion)
        throw std::runtime_error(P + ": unsupported CSR cache version " +
                                 std::to_string(h.version));
    struct stat st;
    if (fstat(fileno(f), &st) != 0) throw std::runtime_error("cannot open " + P);
    const uint64_t fsize = (uint64_t)st.st_size;
    if (h.n >= (1ull << 32) || h.nnz >= (1ull << 36)) throw std::runtime_error(P + ": corrupt header");
    const uint64_t pad = (8 - (h.nnz * 4) % 8) % 8;
    const uint64_t want = 64 + (h.n + 1) * 8 + h.nnz * 4 + pad + h.nnz * 8 + h.n * 8;
    if (fsize != want)
        throw std::runtime_error(P + ": truncated or oversized CSR cache (" +
                                 std::to_string(fsize) + " bytes, expected " +
                                 std::to_string(want) + ")");
    auto* c = new expmc_csr;
    try {
        c->n = h.n;
        c->row_ptr.resize(h.n + 1);
        c->col.resize(h.nnz);
        c->val.resize(h.nnz);
        c->diag.resize(h.n);
        uint64_t skip = 0;
        bool ok = fread(c->row_ptr.data(), 8, h.n + 1, f) == h.n + 1 &&
                  fread(c->col.data(), 4, h.nnz, f) == h.nnz &&
                  fread(&skip, 1, pad, f) == pad &&
                  fread(c->val.data(), 8, h.nnz, f) == h.nnz &&
                  fread(c->diag.data(), 8, h.n, f) == h.n;
        if (!ok) throw std::runtime_error(P + ": short read");
        if (csr_checksum(h.n, h.nnz, c->row_ptr.data(), c->col.data(), c->val.data(),
                         c->diag.data()) != h.checksum)
            throw std::runtime_error(P + ": checksum mismatch");
        if (c->row_ptr[0] != 0 || c->row_ptr[h.n] != h.nnz)
            throw std::runtime_error(P + ": corrupt row_ptr");
        for (uint64_t i = 0; i < h.n; ++i)
            if (c->row_ptr[i + 1] < c->row_ptr[i]) throw std::runtime_error(P + ": corrupt row_ptr");
    } catch (...) {
        delete c;
        throw;
    }
    return c;
}

}  // namespace
}  // namespace expmc_b200

using namespace expmc_b200;

extern "C" {

int expmc_mm_parse(const char* path, expmc_mm** out) {
    return host_guarded([&] {
        if (!out) throw std::invalid_argument("out is null");
        auto* m = new expmc_mm;
        try {
            mm_parse(path, *m);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

int expmc_mm_info(const expmc_mm* m, uint64_t* n, uint64_t* n_entries, int32_t* general,
                  int32_t* pattern, uint64_t* last_line) {
    return host_guarded([&] {
        if (!m) throw std::invalid_argument("null handle");
        if (n) *n = m->n;
        if (n_entries) *n_entries = m->r.size();
        if (general) *general = m->general;
        if (pattern) *pattern = m->pattern;
        if (last_line) *last_line = m->last_line;
    });
}

int expmc_mm_view(const expmc_mm* m, const uint32_t** rows, const uint32_t** cols,
                  const double** weights) {
    return host_guarded([&] {
        if (!m) throw std::invalid_argument("null handle");
        if (rows) *rows = m->r.data();
        if (cols) *cols = m->c.data();
        if (weights) *weights = m->w.data();
    });
}

void expmc_mm_free(expmc_mm* m) { delete m; }

int expmc_mm_write(const char* path, uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                   const double* val, const double* diag) {
    return host_guarded([&] {
        if (!path) throw std::invalid_argument("path is null");
        write_mm(path, n, row_ptr, col, val, diag);
    });
}

int expmc_csr_save(const char* path, uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                   const double* val, const double* diag) {
    return host_guarded([&] {
        if (!path) throw std::invalid_argument("path is null");
        save_csr(path, n, row_ptr, col, val, diag);
    });
}

int expmc_csr_load(const char* path, expmc_csr** out) {
    return host_guarded([&] {
        if (!path || !out) throw std::invalid_argument("null argument");
        *out = load_csr(path);
    });
}

}  // extern "C"
