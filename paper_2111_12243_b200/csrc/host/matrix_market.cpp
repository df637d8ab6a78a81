// Matrix Market coordinate files, the reference's
// read_matrix_market / write_matrix_market (matrix_market.hpp:24-34) with its
// semantics: real, integer or pattern fields; general or symmetric symmetry
// (symmetric inputs mirrored, must be square); pattern entries get 1.0;
// duplicates summed and indices made 0-based by csr_from_triplets; comment
// ('%') and blank lines skipped; the declared entry count must match
// exactly; every error names its 1-based line. Parsing is one buffered pass
// with strtoll / strtod rather than stream extraction.
#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "capi_types.hpp"
#include "common.hpp"
#include "csr.hpp"

namespace pscb {
namespace {

[[noreturn]] void parse_error(int64_t line, const std::string& what) {
    throw std::invalid_argument("line " + std::to_string(line) + ": " + what);
}

std::string lower(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

struct Lines {  // the file as lines, with 1-based physical numbers
    std::vector<char> buf;
    size_t pos = 0;
    int64_t line_no = 0;
    // next line (NUL-terminated in place); false at end of input
    bool next(char*& s) {
        if (pos >= buf.size()) return false;
        s = buf.data() + pos;
        char* nl = static_cast<char*>(std::memchr(s, '\n', buf.size() - pos));
        if (nl) {
            *nl = '\0';
            pos = static_cast<size_t>(nl - buf.data()) + 1;
        } else {
            buf.push_back('\0');
            s = buf.data() + pos;
            pos = buf.size();
        }
        ++line_no;
        const size_t n = std::strlen(s);
        if (n && s[n - 1] == '\r') s[n - 1] = '\0';
        return true;
    }
    // next non-blank, non-comment line
    bool next_data(char*& s) {
        while (next(s)) {
            const char* p = s;
            while (*p && std::isspace(static_cast<unsigned char>(*p))) ++p;
            if (*p && s[0] != '%') return true;
        }
        ++line_no;  // the reference reports end of input as the line after the last
        return false;
    }
};

bool only_space(const char* p) {
    while (*p && std::isspace(static_cast<unsigned char>(*p))) ++p;
    return *p == '\0';
}

}  // namespace

Csr read_matrix_market(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    require(f != nullptr, "cannot open '" + path + "'");
    Lines in;
    {
        char chunk[1 << 16];
        size_t n;
        while ((n = std::fread(chunk, 1, sizeof chunk, f)) > 0) in.buf.insert(in.buf.end(), chunk, chunk + n);
        std::fclose(f);
    }
    char* s = nullptr;
    if (!in.next(s)) parse_error(1, "empty input");
    char banner[64] = {0}, object[64] = {0}, format[64] = {0}, field[64] = {0}, sym[64] = {0};
    std::sscanf(s, "%63s %63s %63s %63s %63s", banner, object, format, field, sym);
    if (std::string(banner) != "%%MatrixMarket" || lower(object) != "matrix")
        parse_error(1, "not a MatrixMarket matrix header");
    if (lower(format) != "coordinate")
        parse_error(1, "unsupported format '" + std::string(format) + "' (expected coordinate)");
    const std::string fl = lower(field), sy = lower(sym);
    const int kind = fl == "real" ? 0 : fl == "integer" ? 1 : fl == "pattern" ? 2 : -1;
    if (kind < 0) parse_error(1, "unsupported field '" + fl + "'");
    if (sy != "general" && sy != "symmetric") parse_error(1, "unsupported symmetry '" + sy + "'");
    const bool symmetric = sy == "symmetric";

    if (!in.next_data(s)) parse_error(in.line_no, "missing size line");
    char* e = nullptr;
    errno = 0;
    const long long rows = std::strtoll(s, &e, 10);
    char* e2 = nullptr;
    const long long cols = std::strtoll(e, &e2, 10);
    char* e3 = nullptr;
    const long long declared = std::strtoll(e2, &e3, 10);
    if (e == s || e2 == e || e3 == e2 || errno || rows < 0 || cols < 0 || declared < 0)
        parse_error(in.line_no, "malformed size line");
    if (!only_space(e3)) parse_error(in.line_no, "trailing characters on size line");
    if (symmetric && rows != cols) parse_error(in.line_no, "symmetric matrix must be square");
    require(rows <= INT32_MAX && cols <= INT32_MAX, "matrix dimensions exceed int32");

    std::vector<Triplet> t;
    t.reserve(static_cast<size_t>(declared) * (symmetric ? 2 : 1));
    for (long long k = 0; k < declared; ++k) {
        if (!in.next_data(s))
            parse_error(in.line_no, "expected " + std::to_string(declared) + " entries, got " + std::to_string(k));
        const int64_t line = in.line_no;
        char *p1 = nullptr, *p2 = nullptr;
        errno = 0;
        const long long r = std::strtoll(s, &p1, 10);
        const long long c = std::strtoll(p1, &p2, 10);
        if (p1 == s || p2 == p1 || errno) parse_error(line, "malformed entry");
        double v = 1.0;
        char* p3 = p2;
        if (kind == 0) {
            v = std::strtod(p2, &p3);
            if (p3 == p2) parse_error(line, "malformed real value");
        } else if (kind == 1) {
            const long long iv = std::strtoll(p2, &p3, 10);
            if (p3 == p2) parse_error(line, "malformed integer value");
            v = static_cast<double>(iv);
        }
        if (!only_space(p3)) parse_error(line, "trailing characters on entry");
        if (r < 1 || r > rows || c < 1 || c > cols)
            parse_error(line, "entry (" + std::to_string(r) + ", " + std::to_string(c) + ") out of range");
        t.push_back({static_cast<int32_t>(r - 1), static_cast<int32_t>(c - 1), v});
        if (symmetric && r != c) t.push_back({static_cast<int32_t>(c - 1), static_cast<int32_t>(r - 1), v});
    }
    if (in.next_data(s)) parse_error(in.line_no, "more entries than declared");
    return csr_from_triplets(static_cast<int32_t>(rows), static_cast<int32_t>(cols), std::move(t));
}

void write_matrix_market(const psc_csr_view& a, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    require(f != nullptr, "cannot open '" + path + "'");
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%d %d %" PRId64 "\n", a.n_rows, a.n_cols, a.nnz);
    for (int32_t r = 0; r < a.n_rows; ++r)
        for (int32_t k = a.row_offsets[r]; k < a.row_offsets[r + 1]; ++k)
            std::fprintf(f, "%d %d %.17g\n", r + 1, a.col_indices[k] + 1, a.values[k]);
    const bool ok = std::fclose(f) == 0;
    require(ok, "write failed: '" + path + "'");
}

}  // namespace pscb

using namespace pscb;

PSC_API psc_status psc_csr_read_matrix_market(const char* path, psc_csr** out) {
    return guarded([&] {
        require(path && out, "read_matrix_market: null argument");
        *out = new psc_csr{read_matrix_market(path)};
    });
}

PSC_API psc_status psc_csr_write_matrix_market(const psc_csr_view* a, const char* path) {
    return guarded([&] {
        require(a && path, "write_matrix_market: null argument");
        write_matrix_market(*a, path);
    });
}
