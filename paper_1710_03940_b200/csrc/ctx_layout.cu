#include <thread>
// Device layouts: format selection and upload of every matrix of the solve
// phase, subdomain grouping of the V-cycle levels and row tiles of the operator.
#include "ctx_impl.cuh"

// colscale != nullptr: also upload the column-scaled values a_ij * colscale_j
// in the same layout (shares the index arrays) into *scaled.
// FMT_CODE encoder: every row <= 8 entries and <= 255 distinct (column - row,
// value-bits) pairs; returns false when the matrix does not qualify
static int try_upload_code(dfl_ctx *ctx, const HostRows &h, DMat &m, bool &ok) {
    ok = false;
    struct Key {
        int64_t d;
        uint64_t v;
        bool operator==(const Key &o) const { return d == o.d && v == o.v; }
    };
    struct KH {
        size_t operator()(const Key &k) const { return std::hash<int64_t>()(k.d) * 1000003u ^ std::hash<uint64_t>()(k.v); }
    };
    std::unordered_map<Key, int, KH> dict;
    std::vector<int> delta;
    std::vector<double> val;
    std::vector<uint8_t> codes((size_t)h.nrows * 8, (uint8_t)kCodePad);
    for (int64_t i = 0; i < h.nrows; ++i) {
        const int64_t b = h.ptr[i], e = h.ptr[i + 1];
        if (e - b > 8) return DFL_OK;
        for (int64_t k = b; k < e; ++k) {
            uint64_t bits;
            std::memcpy(&bits, &h.val[k], 8);
            const int64_t d = h.col[k] - i;
            if (d < INT32_MIN || d > INT32_MAX) return DFL_OK;
            auto it = dict.find(Key{d, bits});
            int code;
            if (it == dict.end()) {
                if (dict.size() >= kCodePad) return DFL_OK;
                code = (int)dict.size();
                dict.emplace(Key{d, bits}, code);
                delta.push_back((int)d);
                val.push_back(h.val[k]);
            } else {
                code = it->second;
            }
            codes[(size_t)i * 8 + (k - b)] = (uint8_t)code;
        }
    }
    m.fmt = FMT_CODE;
    m.stored = m.nnz;
    m.ncodes = (int)delta.size();
    m.code_lead = 0;
    for (int d : delta) m.code_lead = std::max(m.code_lead, d);
    uint8_t *d_codes;
    int *d_delta;
    double *d_val;
    RC(upload(ctx, &d_codes, codes.data(), (int64_t)codes.size()));
    RC(upload(ctx, &d_delta, delta.data(), (int64_t)std::max<size_t>(1, delta.size())));
    RC(upload(ctx, &d_val, val.data(), (int64_t)std::max<size_t>(1, val.size())));
    m.codes = reinterpret_cast<const uint2 *>(d_codes);
    m.ctab_delta = d_delta;
    m.ctab_val = d_val;
    ok = true;
    return DFL_OK;
}

// a row as (column - row, value bits) pairs, <= 8 entries
struct ClsRow {
    int len = 0;
    int d[8];
    uint64_t v[8];
    bool operator==(const ClsRow &o) const {
        if (len != o.len) return false;
        for (int k = 0; k < len; ++k)
            if (d[k] != o.d[k] || v[k] != o.v[k]) return false;
        return true;
    }
};
struct ClsRowHash {
    size_t operator()(const ClsRow &r) const {
        uint64_t x = (uint64_t)r.len * 0x9e3779b97f4a7c15ull;
        for (int k = 0; k < r.len; ++k)
            x = (x ^ ((uint64_t)(uint32_t)r.d[k] * 0x100000001b3ull) ^ r.v[k]) * 0xff51afd7ed558ccdull;
        return (size_t)x;
    }
};
// deterministic order for ties of the dominant row (hash-map order is not)
static bool cls_row_less(const ClsRow &a, const ClsRow &b) {
    if (a.len != b.len) return a.len < b.len;
    for (int k = 0; k < a.len; ++k) {
        if (a.d[k] != b.d[k]) return a.d[k] < b.d[k];
        if (a.v[k] != b.v[k]) return a.v[k] < b.v[k];
    }
    return false;
}
static bool cls_row_of(const HostRows &h, int64_t i, ClsRow &r) {
    const int64_t b = h.ptr[i], e = h.ptr[i + 1];
    if (e - b > 8) return false;
    r.len = (int)(e - b);
    for (int64_t k = b; k < e; ++k) {
        const int64_t d = h.col[k] - i;
        if (d < INT32_MIN || d > INT32_MAX) return false;
        r.d[k - b] = (int)d;
        std::memcpy(&r.v[k - b], &h.val[k], 8);
    }
    return true;
}

// Rows that keep a matrix from class-coding only because it has more than
// kMaxClass generic rows: with the dominant row (and its subsets) and the
// kMaxClass most frequent other rows coded, the rows of the rarer ones are
// flagged (1 per row) for the operator's boundary pass.  Rows with
// skip(i) are ignored (they are in that pass already).  Empty result: not
// needed (the rows fit), or hopeless (> 4096 distinct rows, long rows, or
// more than 5% of the rows would be flagged).
std::vector<uint8_t> class_exceptions(const HostRows &h, const std::function<bool(int64_t)> &skip) {
    std::unordered_map<ClsRow, int64_t, ClsRowHash> count;
    ClsRow r;
    for (int64_t i = 0; i < h.nrows; ++i) {
        if (skip(i)) continue;
        if (!cls_row_of(h, i, r)) return {};
        auto it = count.find(r);
        if (it == count.end()) {
            if (count.size() >= 4096) return {};
            count.emplace(r, 1);
        } else {
            it->second++;
        }
    }
    ClsRow dom;
    int64_t best = -1;
    for (auto &kv : count)
        if (kv.second > best || (kv.second == best && cls_row_less(kv.first, dom))) best = kv.second, dom = kv.first;
    bool have_dom = dom.len <= 7;
    for (int k = 0; k < dom.len && have_dom; ++k) have_dom = std::isfinite(*reinterpret_cast<const double *>(&dom.v[k]));
    auto subset = [&](const ClsRow &x) {
        if (!have_dom) return false;
        int k = 0;
        for (int e = 0; e < x.len; ++e) {
            while (k < dom.len && dom.d[k] != x.d[e]) ++k;
            if (k == dom.len || dom.v[k] != x.v[e]) return false;
            ++k;
        }
        return true;
    };
    std::vector<std::pair<int64_t, const ClsRow *>> gen;
    for (auto &kv : count)
        if (!subset(kv.first)) gen.emplace_back(kv.second, &kv.first);
    if ((int)gen.size() <= kMaxClass) return {};
    std::sort(gen.begin(), gen.end(), [](const auto &a, const auto &b) { return a.first > b.first; });
    std::unordered_map<ClsRow, int, ClsRowHash> rare;
    int64_t nrare = 0;
    for (size_t q = kMaxClass; q < gen.size(); ++q) {
        rare.emplace(*gen[q].second, 1);
        nrare += gen[q].first;
    }
    if (nrare * 20 > h.nrows) return {};
    std::vector<uint8_t> flag((size_t)h.nrows, 0);
    for (int64_t i = 0; i < h.nrows; ++i) {
        if (skip(i)) continue;
        cls_row_of(h, i, r);
        if (rare.count(r)) flag[(size_t)i] = 1;
    }
    return flag;
}

// FMT_CLASS encoder (kernels.cuh ClassTab): the dominant row (most frequent,
// <= 7 entries) and its subsets as presence masks, <= kMaxClass generic
// classes for the rest, every row <= 8 entries.  ok = false leaves m
// untouched for the next format.
static int try_upload_class(dfl_ctx *ctx, const HostRows &h, DMat &m, bool &ok) {
    ok = false;
    auto row_of = [&](int64_t i, ClsRow &r) -> bool { return cls_row_of(h, i, r); };
    using Row = ClsRow;
    using RH = ClsRowHash;
    // pass 1: the dominant row (count distinct rows, give up beyond a bound)
    std::unordered_map<Row, int64_t, RH> count;
    Row r;
    for (int64_t i = 0; i < h.nrows; ++i) {
        if (!row_of(i, r)) return DFL_OK;
        auto it = count.find(r);
        if (it == count.end()) {
            if (count.size() >= 4096) return DFL_OK;
            count.emplace(r, 1);
        } else {
            it->second++;
        }
    }
    Row dom;
    int64_t best = -1;
    for (auto &kv : count)
        if (kv.second > best || (kv.second == best && cls_row_less(kv.first, dom))) best = kv.second, dom = kv.first;
    // the masked dominant-row sum adds dval * 0.0 for absent entries: finite values only
    bool have_dom = dom.len <= 7;
    for (int k = 0; k < dom.len && have_dom; ++k) {
        double v;
        std::memcpy(&v, &dom.v[k], 8);  // v[] holds the value bits
        have_dom = std::isfinite(v);
    }
    // pass 2: masks for subsets of the dominant row, generic classes for the rest
    std::unordered_map<Row, int, RH> dict;
    std::vector<Row> rows;
    std::vector<uint8_t> cls((size_t)h.nrows);
    for (int64_t i = 0; i < h.nrows; ++i) {
        row_of(i, r);
        if (have_dom) {
            unsigned mask = 0;
            int k = 0;
            bool sub = true;
            for (int e = 0; e < r.len && sub; ++e) {
                while (k < dom.len && dom.d[k] != r.d[e]) ++k;
                if (k == dom.len || dom.v[k] != r.v[e]) sub = false;
                else mask |= 1u << k++;
            }
            if (sub) {
                cls[(size_t)i] = (uint8_t)(0x80u | mask);
                continue;
            }
        }
        auto it = dict.find(r);
        if (it == dict.end()) {
            if ((int)rows.size() >= kMaxClass) return DFL_OK;
            it = dict.emplace(r, (int)rows.size()).first;
            rows.push_back(r);
        }
        cls[(size_t)i] = (uint8_t)it->second;
    }
    auto tab = std::make_unique<ClassTab>();
    std::memset(tab.get(), 0, sizeof(ClassTab));
    tab->n = (int)rows.size();
    tab->dom = -1;
    tab->lead = 0;
    if (have_dom) {
        tab->dlen = dom.len;
        for (int k = 0; k < dom.len; ++k) {
            tab->ddelta[k] = dom.d[k];
            std::memcpy(&tab->dval[k], &dom.v[k], 8);
            tab->lead = std::max(tab->lead, dom.d[k]);
        }
    }
    for (int c = 0; c < tab->n; ++c) {
        tab->len[c] = rows[c].len;
        for (int k = 0; k < rows[c].len; ++k) {
            tab->delta[c][k] = rows[c].d[k];
            std::memcpy(&tab->val[c][k], &rows[c].v[k], 8);
            tab->lead = std::max(tab->lead, rows[c].d[k]);
        }
    }
    uint8_t *d_cls;
    RC(upload(ctx, &d_cls, cls.data(), std::max<int64_t>(1, h.nrows)));
    m.fmt = FMT_CLASS;
    m.stored = m.nnz;
    m.cls = d_cls;
    {
        std::lock_guard<std::mutex> lk(ctx->setup_mu);
        m.class_id = (int)ctx->class_tabs.size();
        ctx->class_tabs.push_back(std::move(tab));
    }
    ok = true;
    return DFL_OK;
}

// FMT_PCODE encoder (kernels.cuh): ok = false leaves m untouched
static int try_upload_pcode(dfl_ctx *ctx, const HostRows &h, DMat &m, bool &ok) {
    ok = false;
    const int64_t n = h.nrows;
    std::unordered_map<uint64_t, int> dict;
    std::vector<double> tab;
    std::vector<int> c0(n, 0);
    std::vector<uint32_t> d((size_t)3 * n, 0u);
    std::vector<uint8_t> code((size_t)n * kPcMaxLen, 0);
    std::vector<uint8_t> len((size_t)n, 0);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t b = h.ptr[i], e = h.ptr[i + 1];
        if (e - b > kPcMaxLen) return DFL_OK;
        len[(size_t)i] = (uint8_t)(e - b);
        if (e > b) c0[i] = (int)h.col[b];
        for (int64_t k = b; k < e; ++k) {
            const int64_t j = k - b;
            if (j > 0) {
                const int64_t dl = h.col[k] - h.col[b];
                if (dl <= 0 || dl > 65535) return DFL_OK;  // unsorted or too spread
                d[(size_t)((j - 1) >> 1) * n + i] |= (uint32_t)dl << (16 * ((j - 1) & 1));
            }
            uint64_t bits;
            std::memcpy(&bits, &h.val[k], 8);
            auto it = dict.find(bits);
            if (it == dict.end()) {
                if (dict.size() >= 256) return DFL_OK;
                it = dict.emplace(bits, (int)tab.size()).first;
                tab.push_back(h.val[k]);
            }
            code[(size_t)i * kPcMaxLen + j] = (uint8_t)it->second;
        }
    }
    // up to 16 values: 4-bit codes in one word; else 8-bit codes in two
    const bool wide = tab.size() > 16;
    std::vector<uint32_t> v((size_t)(wide ? 2 : 1) * n, 0u);
    for (int64_t i = 0; i < n; ++i) {
        const uint8_t *c = &code[(size_t)i * kPcMaxLen];
        uint32_t w = len[(size_t)i], w2 = 0;
        for (int j = 0; j < len[(size_t)i]; ++j) {
            if (!wide) w |= (uint32_t)c[j] << (3 + 4 * j);
            else if (j < 3) w |= (uint32_t)c[j] << (8 * (j + 1));
            else w2 |= (uint32_t)c[j] << (8 * (j - 3));
        }
        v[(size_t)i] = w;
        if (wide) v[(size_t)(n + i)] = w2;
    }
    tab.resize(wide ? 256 : 16, 0.0);
    int *d_c0;
    uint32_t *d_d, *d_v;
    double *d_tab;
    RC(upload(ctx, &d_c0, c0.data(), std::max<int64_t>(1, n)));
    RC(upload(ctx, &d_d, d.data(), std::max<int64_t>(1, 3 * n)));
    RC(upload(ctx, &d_v, v.data(), std::max<int64_t>(1, (int64_t)v.size())));
    RC(upload(ctx, &d_tab, tab.data(), (int64_t)tab.size()));
    m.pc_wide = wide ? 1 : 0;
    m.fmt = FMT_PCODE;
    m.stored = m.nnz;
    m.pc_c0 = d_c0;
    m.pc_d = d_d;
    m.pc_v = d_v;
    m.pc_tab = d_tab;
    ok = true;
    return DFL_OK;
}


static constexpr int64_t kSigma = 1024;  // SELL-C-sigma sorting window
// SELL-32-1024 for long-row matrices with enough rows to hide the per-warp
// width imbalance (measured: L0 restriction and L1 operator, profiles/r01);
// short-row (P) and small coarse matrices stay CSR-vector
static constexpr int64_t kSellMinRows = 100000;
static constexpr double kSellMinMean = 12.0;
static constexpr double kShortRowMean = 8.0;
static constexpr double kShortRowPad = 1.7;     // short rows: padding is cheaper than CSR up to this
static constexpr double kCsrPerLane = 12.0;     // CSR-vector: target entries per lane
static constexpr int64_t kCsrTinyRows = 5000;   // levels below: kCsrPerLaneTiny (profiles/r02/README.md)
static constexpr double kCsrPerLaneTiny = 3.0;

int upload_matrix(dfl_ctx *ctx, const HostRows &h, DMat &m, const std::vector<int64_t> &bounds,
                  std::vector<int64_t> *bound_tiles, bool allow_ell, const double *colscale, DMat *scaled,
                  bool allow_sell, bool allow_code, bool allow_class) {
    m = DMat{};
    m.nrows = h.nrows;
    m.ncols = h.ncols;
    m.nnz = h.ptr[h.nrows] - h.ptr[0];
    if (h.ncols >= INT32_MAX || m.nnz >= INT32_MAX) {
        ctx->err = "matrix too large for int32 device indices";
        return DFL_E_DIMENSION;
    }
    if (g_use_class && allow_class && allow_ell && h.nrows > 0) {
        bool ok = false;
        RC(try_upload_class(ctx, h, m, ok));
        if (ok) {
            if (colscale) *scaled = m;  // RESID on a class-coded matrix gathers w .* r
            return DFL_OK;
        }
    }
    if (g_use_code && allow_code && allow_ell && h.nrows > 0) {
        bool ok = false;
        RC(try_upload_code(ctx, h, m, ok));
        if (ok) {
            if (colscale) *scaled = m;  // RESID on a coded matrix gathers w .* r
            return DFL_OK;
        }
    }
    // delta/value-coded rows: only where no pre-scaled copy is needed (P, R)
    if (g_use_pcode && allow_code && allow_ell && !colscale && h.nrows > 0) {
        bool ok = false;
        RC(try_upload_pcode(ctx, h, m, ok));
        if (ok) return DFL_OK;
    }
    const int64_t nsl = cdiv(h.nrows, 32);
    auto rlen = [&](int64_t i) { return h.ptr[i + 1] - h.ptr[i]; };
    // slot -> row: identity, or (SELL-C-sigma) rows sorted by length,
    // descending and stable, inside windows of kSigma rows
    std::vector<int> perm;
    auto slice_offsets = [&](const std::vector<int> &pm, int64_t &maxlen) {
        std::vector<int64_t> so(nsl + 1, 0);
        maxlen = 0;
        for (int64_t s = 0; s < nsl; ++s) {
            int64_t wmax = 0;
            for (int64_t j = s * 32; j < std::min(h.nrows, s * 32 + 32); ++j)
                wmax = std::max(wmax, rlen(pm.empty() ? j : pm[j]));
            maxlen = std::max(maxlen, wmax);
            so[s + 1] = so[s] + 32 * wmax;
        }
        return so;
    };
    int64_t maxlen = 0;
    std::vector<int64_t> soff = slice_offsets(perm, maxlen);
    const double mean = h.nrows ? (double)m.nnz / (double)h.nrows : 0.0;
    const double nnzd = (double)m.nnz + 64.0;
    bool ell = false;
    const double upad = mean <= kShortRowMean ? kShortRowPad : 1.03;
    if (allow_ell && maxlen <= 8 && (double)(nsl * 32 * maxlen) <= upad * nnzd) {
        // uniform slice width: the kernels compute slice offsets instead of loading them
        ell = true;
        m.ell_w = (int)maxlen;
        for (int64_t s = 0; s <= nsl; ++s) soff[s] = s * 32 * maxlen;
    } else if (allow_ell && (double)soff[nsl] <= 1.03 * nnzd) {
        ell = true;
    } else if (allow_ell && allow_sell && maxlen <= 1024 &&
               !g_no_sell && h.nrows >= kSellMinRows && mean >= kSellMinMean) {
        perm.resize(h.nrows);
        for (int64_t w0 = 0; w0 < h.nrows; w0 += kSigma) {
            const int64_t w1 = std::min(h.nrows, w0 + kSigma);
            for (int64_t j = w0; j < w1; ++j) perm[j] = (int)j;
            std::stable_sort(perm.begin() + w0, perm.begin() + w1, [&](int a, int b) { return rlen(a) > rlen(b); });
        }
        int64_t ml = 0;
        std::vector<int64_t> ss = slice_offsets(perm, ml);
        if ((double)ss[nsl] <= 1.25 * nnzd) {
            ell = true;
            soff = ss;
            maxlen = ml;
        } else {
            perm.clear();
        }
    }
    if (!ell && allow_ell && maxlen <= 32 && (double)soff[nsl] <= 1.2 * nnzd) ell = true;
    // short rows (prolongation, ~4 entries): coalesced sliced ELL beats 1-lane
    // CSR even with ~40% padding (profiles/r01)
    if (!ell && allow_ell && mean <= kShortRowMean && maxlen <= 16 && (double)soff[nsl] <= kShortRowPad * nnzd) {
        ell = true;
        perm.clear();
        soff = slice_offsets(perm, maxlen);
    }
    if (ell) {
        m.fmt = FMT_ELL;
        m.stored = soff[nsl];
        std::vector<int> col(m.stored, 0);
        std::vector<double> val(m.stored, 0.0);
        std::vector<double> sval(colscale ? m.stored : 0, 0.0);
        for (int64_t s = 0; s < nsl; ++s) {
            const int64_t wdt = (soff[s + 1] - soff[s]) / 32;
            for (int64_t j = s * 32; j < std::min(h.nrows, s * 32 + 32); ++j) {
                const int lane = (int)(j - s * 32);
                const int64_t i = perm.empty() ? j : perm[j];
                const int64_t b = h.ptr[i], e = h.ptr[i + 1];
                const int pad_col = e > b ? (int)h.col[e - 1] : 0;
                for (int64_t k = 0; k < wdt; ++k) {
                    const int64_t dst = soff[s] + k * 32 + lane;
                    if (b + k < e) {
                        col[dst] = (int)h.col[b + k];
                        val[dst] = h.val[b + k];
                        if (colscale) sval[dst] = h.val[b + k] * colscale[h.col[b + k]];
                    } else {
                        col[dst] = pad_col;
                    }
                }
            }
        }
        int64_t *d_soff;
        int *d_col;
        double *d_val;
        RC(upload(ctx, &d_soff, soff.data(), nsl + 1));
        RC(upload(ctx, &d_col, col.data(), m.stored));
        RC(upload(ctx, &d_val, val.data(), m.stored));
        m.slice_off = d_soff;
        m.col = d_col;
        m.val = d_val;
        if (!perm.empty()) {
            int *d_perm;
            RC(upload(ctx, &d_perm, perm.data(), h.nrows));
            m.perm = d_perm;
        }
        if (colscale) {
            double *d_sval;
            RC(upload(ctx, &d_sval, sval.data(), m.stored));
            *scaled = m;
            scaled->val = d_sval;
        }
    } else {
        m.fmt = FMT_CSR;
        m.stored = m.nnz;
        // lanes per row: about kCsrPerLane entries per lane, batched kCsrUnroll deep
        int g = 1;
        // tiny levels (< kCsrTinyRows rows: the last AMG levels, the coarsest
        // restriction) are latency chains: more lanes, fewer entries each
        const int want = (int)std::ceil(mean / (h.nrows < kCsrTinyRows ? kCsrPerLaneTiny : kCsrPerLane));
        while (g < want && g < 32) g *= 2;
        m.group = g;
        // padded by 4 entries (aligned vector loads may overrun the last row)
        std::vector<int> ptr(h.nrows + 1), col(m.nnz + 4, 0);
        std::vector<double> val(m.nnz + 4, 0.0);
        for (int64_t i = 0; i <= h.nrows; ++i) ptr[i] = (int)(h.ptr[i] - h.ptr[0]);
        for (int64_t k = 0; k < m.nnz; ++k) col[k] = (int)h.col[h.ptr[0] + k];
        std::memcpy(val.data(), h.val + h.ptr[0], sizeof(double) * m.nnz);
        int *d_ptr, *d_col;
        double *d_val;
        RC(upload(ctx, &d_ptr, ptr.data(), h.nrows + 1));
        RC(upload(ctx, &d_col, col.data(), m.nnz + 4));
        RC(upload(ctx, &d_val, val.data(), m.nnz + 4));
        m.ptr = d_ptr;
        m.col = d_col;
        m.val = d_val;
        if (colscale) {
            std::vector<double> sval(m.nnz + 4, 0.0);
            for (int64_t k = 0; k < m.nnz; ++k) sval[k] = h.val[h.ptr[0] + k] * colscale[h.col[h.ptr[0] + k]];
            double *d_sval;
            RC(upload(ctx, &d_sval, sval.data(), m.nnz + 4));
            *scaled = m;
            scaled->val = d_sval;
        }
    }
    return DFL_OK;
}

// ---------------------------------------------------------------------------
// upload helpers for finalize

struct OwnedRows {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> ptr{0}, col;
    std::vector<double> val;
    HostRows view() const { return HostRows{nrows, ncols, ptr.data(), col.data(), val.data()}; }
};

// block-diagonal concatenation: part j contributes rows at row offset, columns
// shifted by col offset
static OwnedRows merge_blocks(const std::vector<const dfl::Csr *> &parts, const std::vector<int64_t> &coff) {
    OwnedRows m;
    int64_t nnz = 0;
    for (auto *p : parts) nnz += p->nnz(), m.nrows += p->nrows;
    m.ncols = coff.back();
    m.ptr.reserve(m.nrows + 1);
    m.col.reserve(nnz);
    m.val.reserve(nnz);
    for (size_t j = 0; j < parts.size(); ++j) {
        const dfl::Csr &p = *parts[j];
        for (int64_t i = 0; i < p.nrows; ++i) {
            for (int64_t k = p.ptr[i]; k < p.ptr[i + 1]; ++k) {
                m.col.push_back(p.col[k] + coff[j]);
                m.val.push_back(p.val[k]);
            }
            m.ptr.push_back((int64_t)m.col.size());
        }
    }
    return m;
}

int build_groups(dfl_ctx *ctx) {
    ctx->groups.clear();
    int s = 0;
    while (s < ctx->nsub) {
        const size_t depth = ctx->pending[s]->levels.size();
        int e = s + 1;
        while (e < ctx->nsub && ctx->pending[e]->levels.size() == depth) ++e;
        VGroup g;
        g.sub0 = s;
        g.nsub = e - s;
        g.row0 = ctx->sub_off[s];
        g.row1 = ctx->sub_off[e];
        const int L = (int)depth - 1;
        for (int j = s; j < e; ++j)
            if (ctx->pending[j]->levels[0].A.nrows != ctx->sub_off[j + 1] - ctx->sub_off[j]) {
                ctx->err = "hierarchy of subdomain " + std::to_string(j) + " does not match its row range";
                return DFL_E_DIMENSION;
            }
        // the levels' A / P / R layouts are converted and uploaded concurrently
        // (independent host work; allocations are serialised by setup_mu)
        std::vector<DLevel> vs(L);
        std::vector<OwnedRows> Am(L), Pm(L), Rm(L);
        std::vector<std::vector<double>> wl(L);
        std::vector<std::vector<int64_t>> fol(L), col(L);
        std::vector<std::vector<const dfl::Csr *>> As(L), Ps(L), Rs(L);
        for (int l = 0; l < L; ++l) {
            fol[l] = {0};
            col[l] = {0};
            for (int j = s; j < e; ++j) {
                const dfl::Level &lv = ctx->pending[j]->levels[l];
                As[l].push_back(&lv.A);
                Ps[l].push_back(&lv.P);
                Rs[l].push_back(&lv.R);
                fol[l].push_back(fol[l].back() + lv.A.nrows);
                col[l].push_back(col[l].back() + lv.P.ncols);
                wl[l].insert(wl[l].end(), lv.w.begin(), lv.w.end());
            }
        }
        std::vector<int> rcs(3 * L, DFL_OK);
        {
            std::vector<std::thread> th;
            for (int l = 0; l < L; ++l)
                for (int which = 0; which < 3; ++which)
                    th.emplace_back([&, l, which] {
                        cudaSetDevice(ctx->device);
                        DLevel &v = vs[l];
                        int &rc = rcs[3 * l + which];
                        if (which == 0) Am[l] = merge_blocks(As[l], fol[l]);
                        else if (which == 1) Pm[l] = merge_blocks(Ps[l], col[l]);
                        else Rm[l] = merge_blocks(Rs[l], fol[l]);
                        if (which == 0)
                            rc = upload_matrix(ctx, Am[l].view(), v.A, {0, Am[l].nrows}, nullptr, true, wl[l].data(),
                                               &v.Aw, true, true, true);
                        else if (which == 1)
                            rc = upload_matrix(ctx, Pm[l].view(), v.P, {0, Pm[l].nrows}, nullptr, true, nullptr,
                                               nullptr, true, true, true);
                        else
                            rc = upload_matrix(ctx, Rm[l].view(), v.R, {0, Rm[l].nrows}, nullptr, true, nullptr,
                                               nullptr, true, true, true);
                    });
            for (auto &t : th) t.join();
        }
        for (int rc : rcs) RC(rc);
        for (int l = 0; l < L; ++l) {
            DLevel &v = vs[l];
            RC(upload(ctx, &v.w, wl[l].data(), (int64_t)wl[l].size()));
            v.n = fol[l].back();
            v.nc = col[l].back();
            RC(dalloc(ctx, &v.t, v.n));
            if (l > 0) {
                RC(dalloc(ctx, &v.rv, v.n));
                RC(dalloc(ctx, &v.xv, v.n));
            }
            g.nnzA.push_back(Am[l].ptr.back());
            g.nnzP.push_back(Pm[l].ptr.back());
            g.rows.push_back(v.n);
            g.lv.push_back(v);
        }
        // bottom level
        std::vector<int64_t> boff{0}, ioff{0};
        std::vector<double> invT;
        for (int j = s; j < e; ++j) {
            const dfl::Level &bl = ctx->pending[j]->levels.back();
            const int64_t nb = bl.A.nrows;
            boff.push_back(boff.back() + nb);
            ioff.push_back(ioff.back() + nb * nb);
            g.max_nb = std::max<int>(g.max_nb, (int)nb);
            for (int64_t c = 0; c < nb; ++c)
                for (int64_t i = 0; i < nb; ++i) invT.push_back(bl.bottom_inv[i * nb + c]);
        }
        g.nb = boff.back();
        g.rows.push_back(g.nb);
        RC(upload(ctx, &g.binvT, invT.data(), (int64_t)invT.size()));
        RC(upload(ctx, &g.binv_off, ioff.data(), (int64_t)ioff.size()));
        RC(upload(ctx, &g.b_off, boff.data(), (int64_t)boff.size()));
        if (L > 0) {
            RC(dalloc(ctx, &g.rb, g.nb));
            RC(dalloc(ctx, &g.xb, g.nb));
        }
        if (g.max_nb > (1 << 20)) {
            ctx->err = "bottom level too large for shared-memory staging";
            return DFL_E_DIMENSION;
        }
        ctx->groups.push_back(std::move(g));
        s = e;
    }
    return DFL_OK;
}

int build_tiles(dfl_ctx *ctx) {
    const int rpt = rows_per_block(ctx->Aop);
    std::vector<int64_t> r0, r1, subt{0};
    std::vector<int> ts;
    for (int s = 0; s < ctx->nsub; ++s) {
        for (int64_t i = ctx->sub_off[s]; i < ctx->sub_off[s + 1]; i += rpt) {
            r0.push_back(i);
            r1.push_back(std::min(i + rpt, ctx->sub_off[s + 1]));
            ts.push_back(s);
        }
        subt.push_back((int64_t)r0.size());
    }
    ctx->ntiles = (int64_t)r0.size();
    int64_t *d0, *d1;
    RC(upload(ctx, &d0, r0.data(), ctx->ntiles));
    RC(upload(ctx, &d1, r1.data(), ctx->ntiles));
    RC(upload(ctx, &ctx->tile_sub, ts.data(), ctx->ntiles));
    RC(upload(ctx, &ctx->sub_tiles, subt.data(), (int64_t)subt.size()));
    ctx->h_sub_tiles = subt;
    ctx->tiles = Tiles{d0, d1, ctx->ntiles};
    ctx->subtab = SubTable{};
    if (ctx->nsub <= kSubTab) {
        ctx->subtab.n = ctx->nsub;
        ctx->subtab.rows_per_tile = rpt;
        for (int s = 0; s <= ctx->nsub; ++s) {
            ctx->subtab.sub_off[s] = ctx->sub_off[s];
            ctx->subtab.tile_start[s] = subt[s];
        }
    }
    return DFL_OK;
}

