// Native readers for the reference's input files (pkg/src/deflamg/mmio.py):
// MatrixMarket coordinate matrices (real / integer, general / symmetric),
// plain vector files (one float per line) and mask files (one 0/1 per line).
//
// The whole file is read into memory once and walked line by line with a
// cursor; numbers are parsed with strtoll / strtod (the same correctly
// rounded decimal -> binary64 conversion Python's float() performs, so the
// values are bit-identical).  Coordinate entries are sorted by (row, col)
// with a stable sort and duplicates summed in file order, then laid out as
// CSR -- SparseMatrix.from_coo's result (sparse.py:72-96).  Every failure
// returns DFL_E_PARSE with "<path>:<line>: <reason>" (1-based line) in
// dfl_last_setup_error, the reference's ParseError contract.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "host_setup.hpp"

#define RC_PARSE(x)                  \
    do {                             \
        const int rc_ = (x);         \
        if (rc_ != DFL_OK) return rc_; \
    } while (0)

namespace {

struct Text {
    std::string path;
    std::vector<char> buf;           // file bytes + '\0'
    std::vector<size_t> line_start;  // offset of every line
};

int fail(const Text &t, size_t line, const std::string &why) {
    dfl::set_setup_error(t.path + ":" + std::to_string(line) + ": " + why);
    return DFL_E_PARSE;
}

int load(const char *path, Text &t) {
    t.path = path;
    FILE *f = std::fopen(path, "rb");
    if (!f) {
        dfl::set_setup_error(t.path + ": cannot open: " + std::strerror(errno));
        return DFL_E_PARSE;
    }
    char chunk[1 << 16];
    size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) t.buf.insert(t.buf.end(), chunk, chunk + got);
    std::fclose(f);
    for (char c : t.buf)
        if ((unsigned char)c > 127) {
            dfl::set_setup_error(t.path + ": cannot open: not an ASCII file");
            return DFL_E_PARSE;
        }
    t.buf.push_back('\0');
    const size_t n = t.buf.size() - 1;
    if (n > 0) t.line_start.push_back(0);
    for (size_t i = 0; i < n; ++i)
        if (t.buf[i] == '\n' && i + 1 < n) t.line_start.push_back(i + 1);
    return DFL_OK;
}

// the whitespace-separated fields of line k (0-based)
std::vector<std::string> fields(const Text &t, size_t k) {
    std::vector<std::string> out;
    const char *p = t.buf.data() + t.line_start[k];
    while (*p && *p != '\n') {
        while (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\f' || *p == '\v') ++p;
        if (!*p || *p == '\n') break;
        const char *q = p;
        while (*q && *q != '\n' && *q != ' ' && *q != '\t' && *q != '\r' && *q != '\f' && *q != '\v') ++q;
        out.emplace_back(p, q);
        p = q;
    }
    return out;
}

// line k stripped of surrounding whitespace
std::string stripped(const Text &t, size_t k) {
    const char *b = t.buf.data() + t.line_start[k];
    const char *e = b;
    while (*e && *e != '\n') ++e;
    while (b < e && std::isspace((unsigned char)*b)) ++b;
    while (e > b && std::isspace((unsigned char)e[-1])) --e;
    return std::string(b, e);
}

bool skip_line(const Text &t, size_t k) {
    const std::string s = stripped(t, k);
    return s.empty() || s[0] == '%';
}

bool to_int(const std::string &s, int64_t &v) {
    if (s.empty()) return false;
    size_t i = (s[0] == '+' || s[0] == '-') ? 1 : 0;
    if (i == s.size()) return false;
    for (size_t j = i; j < s.size(); ++j)
        if (s[j] < '0' || s[j] > '9') return false;
    errno = 0;
    char *end = nullptr;
    v = std::strtoll(s.c_str(), &end, 10);
    return errno == 0 && *end == '\0';
}

// Python float(): decimal / exponent forms, inf / nan spellings
bool to_float(const std::string &s, double &v) {
    if (s.empty()) return false;
    for (char c : s)
        if (!(std::isdigit((unsigned char)c) || c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-' ||
              std::isalpha((unsigned char)c)))
            return false;
    if (s.find_first_of("xXpP") != std::string::npos) return false;  // no hex floats
    char *end = nullptr;
    v = std::strtod(s.c_str(), &end);
    return end != s.c_str() && *end == '\0';
}

std::string lower(std::string s) {
    for (char &c : s) c = (char)std::tolower((unsigned char)c);
    return s;
}

std::string quoted(const std::string &s) { return "'" + s + "'"; }

// triplets -> CSR: stable (row, col) order, duplicates summed in file order
void coo_to_csr(int64_t nrows, int64_t ncols, std::vector<int64_t> &r, std::vector<int64_t> &c,
                std::vector<double> &v, dfl::Csr &out) {
    std::vector<int64_t> ord(r.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        return r[a] != r[b] ? r[a] < r[b] : c[a] < c[b];
    });
    out.nrows = nrows;
    out.ncols = ncols;
    out.ptr.assign(nrows + 1, 0);
    out.col.clear();
    out.val.clear();
    for (size_t q = 0; q < ord.size(); ++q) {
        const int64_t e = ord[q];
        if (q > 0 && r[ord[q - 1]] == r[e] && c[ord[q - 1]] == c[e]) {
            out.val.back() += v[e];
            continue;
        }
        out.col.push_back(c[e]);
        out.val.push_back(v[e]);
        out.ptr[r[e] + 1]++;
    }
    for (int64_t i = 0; i < nrows; ++i) out.ptr[i + 1] += out.ptr[i];
}

}  // namespace

extern "C" {

int dfl_mm_read(const char *path, dfl_matrix **out) {
    if (!path || !out) return DFL_E_STATE;
    *out = nullptr;
    Text t;
    RC_PARSE(load(path, t));
    const size_t nl = t.line_start.size();
    if (nl == 0) return fail(t, 1, "empty file");
    const std::vector<std::string> h = fields(t, 0);
    if (h.size() != 5 || h[0] != "%%MatrixMarket")
        return fail(t, 1, "expected '%%MatrixMarket matrix coordinate <field> <symmetry>' header");
    const std::string obj = lower(h[1]), fmt = lower(h[2]), field = lower(h[3]), sym = lower(h[4]);
    if (obj != "matrix" || fmt != "coordinate")
        return fail(t, 1, "unsupported object/format '" + obj + " " + fmt + "' (need matrix coordinate)");
    if (field != "real" && field != "integer")
        return fail(t, 1, "unsupported field '" + field + "' (need real or integer)");
    if (sym != "general" && sym != "symmetric")
        return fail(t, 1, "unsupported symmetry '" + sym + "' (need general or symmetric)");
    size_t k = 1;
    while (k < nl && (t.buf[t.line_start[k]] == '%' || stripped(t, k).empty())) ++k;
    if (k == nl) return fail(t, nl, "missing size line");
    const std::vector<std::string> sz = fields(t, k);
    if (sz.size() != 3)
        return fail(t, k + 1, "size line needs 3 integers, got " + std::to_string(sz.size()) + " tokens");
    int64_t nrows, ncols, nnz;
    if (!to_int(sz[0], nrows) || !to_int(sz[1], ncols) || !to_int(sz[2], nnz))
        return fail(t, k + 1, "bad size line " + quoted(stripped(t, k)));
    if (nrows < 0 || ncols < 0 || nnz < 0) return fail(t, k + 1, "negative dimensions");
    if (sym == "symmetric" && nrows != ncols) return fail(t, k + 1, "symmetric matrix must be square");
    std::vector<int64_t> r, c;
    std::vector<double> v;
    r.reserve(nnz);
    c.reserve(nnz);
    v.reserve(nnz);
    for (size_t q = k + 1; q < nl; ++q) {
        if (skip_line(t, q)) continue;
        if ((int64_t)v.size() == nnz)
            return fail(t, q + 1, "more than the declared " + std::to_string(nnz) + " entries");
        const std::vector<std::string> e = fields(t, q);
        if (e.size() != 3)
            return fail(t, q + 1, "entry needs 'row col value', got " + std::to_string(e.size()) + " tokens");
        int64_t i, j;
        double x;
        if (!to_int(e[0], i) || !to_int(e[1], j) || !to_float(e[2], x))
            return fail(t, q + 1, "cannot parse entry " + quoted(stripped(t, q)));
        if (i < 1 || i > nrows || j < 1 || j > ncols)
            return fail(t, q + 1, "index (" + std::to_string(i) + ", " + std::to_string(j) + ") outside " +
                                      std::to_string(nrows) + "x" + std::to_string(ncols));
        r.push_back(i - 1);
        c.push_back(j - 1);
        v.push_back(x);
    }
    if ((int64_t)v.size() != nnz)
        return fail(t, nl, "expected " + std::to_string(nnz) + " entries, found " + std::to_string(v.size()));
    if (sym == "symmetric") {  // mirror the strictly off-diagonal entries after the file's own
        const size_t m = v.size();
        for (size_t q = 0; q < m; ++q)
            if (r[q] != c[q]) {
                r.push_back(c[q]);
                c.push_back(r[q]);
                v.push_back(v[q]);
            }
    }
    auto *mat = new dfl_matrix;
    coo_to_csr(nrows, ncols, r, c, v, mat->m);
    *out = mat;
    return DFL_OK;
}

// mask == 0: one float per line (vector file); mask != 0: one 0 / 1 per line.
// Blank lines and lines starting with '%' are skipped.  The values come back
// as an n x 1 matrix (one entry per row).
int dfl_vec_read(const char *path, int32_t mask, dfl_matrix **out) {
    if (!path || !out) return DFL_E_STATE;
    *out = nullptr;
    Text t;
    RC_PARSE(load(path, t));
    std::vector<double> vals;
    for (size_t q = 0; q < t.line_start.size(); ++q) {
        const std::string s = stripped(t, q);
        if (s.empty() || s[0] == '%') continue;
        if (mask) {
            if (s != "0" && s != "1") return fail(t, q + 1, "mask entries must be 0 or 1, got " + quoted(s));
            vals.push_back(s == "1" ? 1.0 : 0.0);
        } else {
            double x;
            if (!to_float(s, x)) return fail(t, q + 1, "cannot parse vector entry " + quoted(s));
            vals.push_back(x);
        }
    }
    auto *mat = new dfl_matrix;
    const int64_t n = (int64_t)vals.size();
    mat->m.nrows = n;
    mat->m.ncols = 1;
    mat->m.ptr.resize(n + 1);
    std::iota(mat->m.ptr.begin(), mat->m.ptr.end(), 0);
    mat->m.col.assign(n, 0);
    mat->m.val = std::move(vals);
    *out = mat;
    return DFL_OK;
}

}  // extern "C"
