// Corpus IO for the B200 core: the reference's text matrix
// format (corpus.cpp:182-272) read and written natively, plus a binary CSR
// format that loads at disk speed. Host code; not on the clustering hot path.
//
// Text format (corpus.hpp:74-80):
//   %%sparse-unit-matrix <n_rows> <n_dims> <nnz>
//   <row> <dim> <weight>     (0-based, rows then dims ascending, %.17g weights)
// with doc ids in the sidecar <path>.ids. The loader applies the reference's
// checks with the reference's messages ("<path>:<line>: <what>"): header,
// bounds, row / dim order, zero weights, declared nnz, unit row norm (fp64,
// tolerance 1e-9 by default), id count. It parses in parallel (chunks split at
// line boundaries, std::from_chars) and hands back CSR with fp32 values (the
// device storage type) and the parsed fp64 values.
//
// Binary format "SSKMCSR1": magic[8], int64 n_rows, uint32 dims, uint32 pad,
// int64 nnz, then indptr int64[n+1], indices int32[nnz], values fp32[nnz].
#include <stdint.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

struct Loaded {
    int64_t n = 0;
    uint32_t dims = 0;
    std::vector<int64_t> indptr;
    std::vector<int32_t> idx;
    std::vector<double> val;
    std::vector<std::string> ids;
};

std::runtime_error format_error(const std::string& path, size_t line, const std::string& what) {
    return std::runtime_error(path + ":" + std::to_string(line) + ": " + what);
}

struct Triple {
    uint64_t row;
    uint32_t dim;
    uint32_t line;  // 1-based line within its chunk (exact error positions)
    double w;
};

struct ChunkOut {
    std::vector<Triple> t;
    size_t lines = 0;     // newlines consumed in this chunk
    size_t bad_line = 0;  // 1-based line within the chunk of the first malformed line (0 = none)
};

// Parse "<row> <dim> <weight>" lines of [b, e) (e is at a line boundary).
void parse_chunk(const char* b, const char* e, ChunkOut& out) {
    const char* p = b;
    size_t line = 0;
    while (p < e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
        const char* le = nl ? nl : e;
        ++line;
        const char* q = p;
        while (q < le && (*q == ' ' || *q == '\r' || *q == '\t')) ++q;
        if (q < le) {
            uint64_t row = 0;
            uint32_t dim = 0;
            double w = 0.0;
            auto r1 = std::from_chars(q, le, row);
            const char* s = r1.ptr;
            while (s < le && *s == ' ') ++s;
            auto r2 = std::from_chars(s, le, dim);
            const char* s2 = r2.ptr;
            while (s2 < le && *s2 == ' ') ++s2;
            auto r3 = std::from_chars(s2, le, w);
            if (r1.ec != std::errc() || r2.ec != std::errc() || r3.ec != std::errc() || r1.ptr == q ||
                r2.ptr == s || r3.ptr == s2) {
                if (!out.bad_line) out.bad_line = line;
            } else {
                out.t.push_back({row, dim, static_cast<uint32_t>(line), w});
            }
        }
        p = nl ? nl + 1 : e;
    }
    out.lines = line;
}

Loaded* load_text(const std::string& path, double norm_tol, int threads) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open " + path);
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    std::string buf(static_cast<size_t>(std::max(size, 0L)), '\0');
    if (size > 0 && std::fread(buf.data(), 1, buf.size(), f) != buf.size()) {
        std::fclose(f);
        throw std::runtime_error("read failed: " + path);
    }
    std::fclose(f);
    if (buf.empty()) throw std::runtime_error(path + ": empty file");
    const char* data = buf.data();
    const char* end = data + buf.size();
    const char* nl = static_cast<const char*>(std::memchr(data, '\n', buf.size()));
    const std::string header(data, nl ? nl : end);
    char magic[64] = {0};
    unsigned long long n_rows = 0, nnz = 0;
    unsigned int n_dims = 0;
    if (std::sscanf(header.c_str(), "%63s %llu %u %llu", magic, &n_rows, &n_dims, &nnz) != 4 ||
        std::string(magic) != "%%sparse-unit-matrix")
        throw format_error(path, 1, "bad header, expected '%%sparse-unit-matrix <n_rows> <n_dims> <nnz>'");
    const char* body = nl ? nl + 1 : end;

    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const size_t span = static_cast<size_t>(end - body);
    threads = static_cast<int>(std::min<size_t>(threads, std::max<size_t>(1, span / (1 << 20) + 1)));
    std::vector<const char*> cut(threads + 1, end);
    cut[0] = body;
    for (int t = 1; t < threads; ++t) {
        const char* c = body + span * t / threads;
        if (c < cut[t - 1]) c = cut[t - 1];
        const char* n2 = static_cast<const char*>(std::memchr(c, '\n', static_cast<size_t>(end - c)));
        cut[t] = n2 ? n2 + 1 : end;
    }
    std::vector<ChunkOut> outs(threads);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < threads; ++t) th.emplace_back(parse_chunk, cut[t], cut[t + 1], std::ref(outs[t]));
        for (auto& x : th) x.join();
    }
    // validation in file order, with the reference's messages (corpus.cpp:221-262)
    auto* L = new Loaded();
    std::unique_ptr<Loaded> guard(L);
    L->n = static_cast<int64_t>(n_rows);
    L->dims = n_dims;
    L->indptr.assign(n_rows + 1, 0);
    L->idx.reserve(nnz);
    L->val.reserve(nnz);
    size_t line_base = 1;  // header is line 1
    uint64_t current_row = 0;
    bool have = false;
    uint32_t last_dim = 0;
    size_t seen = 0;
    for (int t = 0; t < threads; ++t) {
        const ChunkOut& o = outs[t];
        if (o.bad_line) throw format_error(path, line_base + o.bad_line, "expected '<row> <dim> <weight>'");
        for (const Triple& x : o.t) {
            auto where = [&] { return line_base + x.line; };
            if (x.row >= n_rows) throw format_error(path, where(), "row index out of bounds");
            if (x.dim >= n_dims) throw format_error(path, where(), "dim index out of bounds");
            if (have && x.row < current_row) throw format_error(path, where(), "rows out of order");
            if (have && x.row == current_row && last_dim >= x.dim)
                throw format_error(path, where(), "dims out of order within row");
            if (x.w == 0.0) throw format_error(path, where(), "zero weight");
            while (current_row < x.row) L->indptr[++current_row] = static_cast<int64_t>(L->idx.size());
            L->idx.push_back(static_cast<int32_t>(x.dim));
            L->val.push_back(x.w);
            have = true;
            last_dim = x.dim;
            ++seen;
        }
        line_base += o.lines;
    }
    while (current_row < n_rows) L->indptr[++current_row] = static_cast<int64_t>(L->idx.size());
    if (seen != nnz)
        throw std::runtime_error(path + ": header declares " + std::to_string(nnz) + " entries but file has " +
                                 std::to_string(seen));
    for (uint64_t r = 0; r < n_rows; ++r) {
        double s = 0.0;
        for (int64_t p = L->indptr[r]; p < L->indptr[r + 1]; ++p) s += L->val[p] * L->val[p];
        const double nrm = std::sqrt(s);
        if (std::abs(nrm - 1.0) > norm_tol)
            throw std::runtime_error(path + ": row " + std::to_string(r) + " is not unit length (norm " +
                                     std::to_string(nrm) + ")");
    }
    std::ifstream ids(path + ".ids");
    if (!ids) throw std::runtime_error("cannot open " + path + ".ids");
    std::string line;
    while (std::getline(ids, line)) L->ids.push_back(line);
    if (L->ids.size() != n_rows)
        throw std::runtime_error(path + ".ids: has " + std::to_string(L->ids.size()) + " ids for " +
                                 std::to_string(n_rows) + " rows");
    return guard.release();
}

}  // namespace

extern "C" {

const char* sskm_io_last_error(void) { return g_err.c_str(); }

// Returns a handle (NULL on error; message in sskm_io_last_error).
void* sskm_io_load_matrix(const char* path, double norm_tol, int threads) {
    try {
        return load_text(path, norm_tol, threads);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void sskm_io_sizes(void* h, int64_t* n, uint32_t* dims, int64_t* nnz, int64_t* ids_bytes) {
    auto* L = static_cast<Loaded*>(h);
    *n = L->n;
    *dims = L->dims;
    *nnz = static_cast<int64_t>(L->idx.size());
    int64_t b = 0;
    for (const auto& s : L->ids) b += static_cast<int64_t>(s.size()) + 1;
    *ids_bytes = b;
}

// values_f32: the device storage type; values_f64 (may be NULL): as parsed.
// ids: '\n'-joined doc ids (ids_bytes from sskm_io_sizes).
void sskm_io_export(void* h, int64_t* indptr, int32_t* idx, float* values_f32, double* values_f64, char* ids) {
    auto* L = static_cast<Loaded*>(h);
    std::memcpy(indptr, L->indptr.data(), L->indptr.size() * 8);
    if (!L->idx.empty()) std::memcpy(idx, L->idx.data(), L->idx.size() * 4);
    for (size_t p = 0; p < L->val.size(); ++p) values_f32[p] = static_cast<float>(L->val[p]);
    if (values_f64 && !L->val.empty()) std::memcpy(values_f64, L->val.data(), L->val.size() * 8);
    if (ids) {
        char* o = ids;
        for (const auto& s : L->ids) {
            std::memcpy(o, s.data(), s.size());
            o += s.size();
            *o++ = '\n';
        }
    }
}

void sskm_io_free(void* h) { delete static_cast<Loaded*>(h); }

// write_matrix (corpus.cpp:182-199): %.17g of the stored (fp32) weights.
int sskm_io_write_matrix(const char* path, int64_t n, uint32_t dims, const int64_t* indptr, const int32_t* idx,
                         const float* val, const char* ids_joined) {
    try {
        std::FILE* f = std::fopen(path, "w");
        if (!f) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
        std::fprintf(f, "%%%%sparse-unit-matrix %lld %u %lld\n", static_cast<long long>(n), dims,
                     static_cast<long long>(indptr[n]));
        for (int64_t r = 0; r < n; ++r)
            for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p)
                std::fprintf(f, "%lld %d %.17g\n", static_cast<long long>(r), idx[p], static_cast<double>(val[p]));
        if (std::fclose(f) != 0) throw std::runtime_error(std::string("write failed: ") + path);
        std::ofstream ids(std::string(path) + ".ids");
        if (!ids) throw std::runtime_error(std::string("cannot open ") + path + ".ids for writing");
        if (ids_joined) {
            ids << ids_joined;
        } else {
            for (int64_t r = 0; r < n; ++r) ids << r << '\n';
        }
        if (!ids) throw std::runtime_error(std::string("write failed: ") + path + ".ids");
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

int sskm_io_save_csr(const char* path, int64_t n, uint32_t dims, const int64_t* indptr, const int32_t* idx,
                     const float* val) {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) {
        g_err = std::string("cannot open ") + path + " for writing";
        return 2;
    }
    const int64_t nnz = indptr[n];
    const uint32_t pad = 0;
    bool ok = std::fwrite("SSKMCSR1", 1, 8, f) == 8 && std::fwrite(&n, 8, 1, f) == 1 && std::fwrite(&dims, 4, 1, f) == 1 &&
              std::fwrite(&pad, 4, 1, f) == 1 && std::fwrite(&nnz, 8, 1, f) == 1 &&
              std::fwrite(indptr, 8, static_cast<size_t>(n + 1), f) == static_cast<size_t>(n + 1) &&
              (nnz == 0 || (std::fwrite(idx, 4, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz) &&
                            std::fwrite(val, 4, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz)));
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) {
        g_err = std::string("write failed: ") + path;
        return 2;
    }
    return 0;
}

// Two-phase binary load: header (sizes), then the arrays into caller buffers.
int sskm_io_csr_header(const char* path, int64_t* n, uint32_t* dims, int64_t* nnz) {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) {
        g_err = std::string("cannot open ") + path;
        return 2;
    }
    char magic[8];
    uint32_t pad;
    const bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, "SSKMCSR1", 8) == 0 &&
                    std::fread(n, 8, 1, f) == 1 && std::fread(dims, 4, 1, f) == 1 && std::fread(&pad, 4, 1, f) == 1 &&
                    std::fread(nnz, 8, 1, f) == 1;
    std::fclose(f);
    if (!ok) {
        g_err = std::string(path) + ": not an SSKMCSR1 file";
        return 1;
    }
    return 0;
}

int sskm_io_csr_read(const char* path, int64_t* indptr, int32_t* idx, float* val) {
    int64_t n, nnz;
    uint32_t dims;
    if (int rc = sskm_io_csr_header(path, &n, &dims, &nnz)) return rc;
    std::FILE* f = std::fopen(path, "rb");
    std::fseek(f, 32, SEEK_SET);
    bool ok = std::fread(indptr, 8, static_cast<size_t>(n + 1), f) == static_cast<size_t>(n + 1) &&
              (nnz == 0 || (std::fread(idx, 4, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz) &&
                            std::fread(val, 4, static_cast<size_t>(nnz), f) == static_cast<size_t>(nnz)));
    std::fclose(f);
    if (!ok || indptr[0] != 0 || indptr[n] != nnz) {
        g_err = std::string(path) + ": truncated or inconsistent CSR";
        return 1;
    }
    return 0;
}

}  // extern "C"
