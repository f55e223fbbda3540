// Host-side setup of the B200 solve phase (native C++, runs once per solver,
// timed separately from the solve as in the paper).
//
// Produces a smoothed-aggregation hierarchy that is label-for-label and
// bit-for-bit identical to the reference's (amg.py:217-250): same strength
// test, same greedy aggregation order, same Gustavson product summation
// order, no FMA contraction (compiled with -ffp-contract=off).  Only the
// bottom-level dense factorisation differs in rounding (own LU vs LAPACK).
#include "host_setup.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <thread>
#include <string>
#include <vector>

namespace dfl {

static thread_local std::string g_setup_error;

void set_setup_error(const std::string &s) { g_setup_error = s; }
const char *setup_error() { return g_setup_error.c_str(); }

// ---------------------------------------------------------------------------
// CSR primitives

Csr csr_from_view(const dfl_csr *v) {
    Csr m;
    m.nrows = v->nrows;
    m.ncols = v->ncols;
    m.ptr.assign(v->row_ptr, v->row_ptr + v->nrows + 1);
    const int64_t nnz = m.ptr.back();
    m.col.assign(v->col_idx, v->col_idx + nnz);
    m.val.assign(v->values, v->values + nnz);
    return m;
}

// counting-sort transpose, stable in row order (reference _kernels.pyx:26-52)
Csr transpose(const Csr &a) {
    Csr t;
    t.nrows = a.ncols;
    t.ncols = a.nrows;
    t.ptr.assign(a.ncols + 1, 0);
    const int64_t nnz = a.nnz();
    t.col.resize(nnz);
    t.val.resize(nnz);
    for (int64_t k = 0; k < nnz; ++k) t.ptr[a.col[k] + 1]++;
    for (int64_t c = 0; c < a.ncols; ++c) t.ptr[c + 1] += t.ptr[c];
    std::vector<int64_t> next(t.ptr.begin(), t.ptr.end() - 1);
    for (int64_t i = 0; i < a.nrows; ++i)
        for (int64_t k = a.ptr[i]; k < a.ptr[i + 1]; ++k) {
            const int64_t d = next[a.col[k]]++;
            t.col[d] = i;
            t.val[d] = a.val[k];
        }
    return t;
}

// Host threads for the row-parallel setup kernels (every output row is
// computed by exactly one thread with the sequential per-row arithmetic, so
// the result does not depend on the thread count).  DFL_SETUP_THREADS
// overrides the default (hardware concurrency).
static int setup_threads() {
    static int t = [] {
        const char *e = std::getenv("DFL_SETUP_THREADS");
        int v = e ? std::atoi(e) : (int)std::thread::hardware_concurrency();
        return std::max(1, std::min(v, 64));
    }();
    return t;
}

template <class F>
static void parallel_rows(int64_t n, int64_t min_chunk, F &&f) {
    const int T = (int)std::min<int64_t>(setup_threads(), std::max<int64_t>(1, n / std::max<int64_t>(1, min_chunk)));
    if (T <= 1) {
        f(0, (int64_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back([&, t] { f(t, n * t / T, n * (t + 1) / T); });
    for (auto &x : th) x.join();
}

// Gustavson product; per output row the values accumulate in (A entry,
// B entry) order into a dense scratch row and the touched columns are
// insertion-sorted (reference _kernels.pyx:55-115).  Row-parallel.
Csr spgemm(const Csr &a, const Csr &b) {
    Csr c;
    c.nrows = a.nrows;
    c.ncols = b.ncols;
    c.ptr.assign(a.nrows + 1, 0);
    parallel_rows(a.nrows, 4096, [&](int, int64_t r0, int64_t r1) {
        std::vector<int64_t> mark(b.ncols, -1);
        for (int64_t i = r0; i < r1; ++i) {
            int64_t cnt = 0;
            for (int64_t ka = a.ptr[i]; ka < a.ptr[i + 1]; ++ka) {
                const int64_t r = a.col[ka];
                for (int64_t kb = b.ptr[r]; kb < b.ptr[r + 1]; ++kb) {
                    const int64_t j = b.col[kb];
                    if (mark[j] != i) {
                        mark[j] = i;
                        ++cnt;
                    }
                }
            }
            c.ptr[i + 1] = cnt;
        }
    });
    for (int64_t i = 0; i < a.nrows; ++i) c.ptr[i + 1] += c.ptr[i];
    c.col.resize(c.ptr.back());
    c.val.resize(c.ptr.back());
    parallel_rows(a.nrows, 4096, [&](int, int64_t r0, int64_t r1) {
        std::vector<double> acc(b.ncols, 0.0);
        std::vector<int64_t> mark(b.ncols, -1);
        for (int64_t i = r0; i < r1; ++i) {
            int64_t *cols = c.col.data() + c.ptr[i];
            int64_t len = 0;
            for (int64_t ka = a.ptr[i]; ka < a.ptr[i + 1]; ++ka) {
                const int64_t r = a.col[ka];
                const double av = a.val[ka];
                for (int64_t kb = b.ptr[r]; kb < b.ptr[r + 1]; ++kb) {
                    const int64_t j = b.col[kb];
                    acc[j] = acc[j] + av * b.val[kb];
                    if (mark[j] != i) {
                        mark[j] = i;
                        cols[len++] = j;
                    }
                }
            }
            for (int64_t p = 1; p < len; ++p) {
                const int64_t key = cols[p];
                int64_t q = p - 1;
                while (q >= 0 && cols[q] > key) {
                    cols[q + 1] = cols[q];
                    --q;
                }
                cols[q + 1] = key;
            }
            double *vals = c.val.data() + c.ptr[i];
            for (int64_t p = 0; p < len; ++p) {
                vals[p] = acc[cols[p]];
                acc[cols[p]] = 0.0;
            }
        }
    });
    return c;
}

// diagonal with the reference's zero/missing check (sparse.py:153-161)
bool diagonal(const Csr &a, std::vector<double> &d, const char *what) {
    if (a.nrows != a.ncols) {
        set_setup_error(std::string(what) + " must be square");
        return false;
    }
    d.assign(a.nrows, 0.0);
    for (int64_t i = 0; i < a.nrows; ++i)
        for (int64_t k = a.ptr[i]; k < a.ptr[i + 1]; ++k)
            if (a.col[k] == i) d[i] = a.val[k];
    for (int64_t i = 0; i < a.nrows; ++i)
        if (d[i] == 0.0) {
            set_setup_error(std::string(what) + " has zero/missing diagonal at row " +
                            std::to_string(i));
            return false;
        }
    return true;
}

// |a_ij| > eps * sqrt(|a_ii| |a_jj|) or i == j  (amg.py:70-84)
static Csr strength(const Csr &a, const std::vector<double> &d, double eps) {
    Csr s;
    s.nrows = a.nrows;
    s.ncols = a.ncols;
    s.ptr.assign(a.nrows + 1, 0);
    s.col.reserve(a.nnz());
    s.val.reserve(a.nnz());
    for (int64_t i = 0; i < a.nrows; ++i) {
        const double di = std::fabs(d[i]);
        for (int64_t k = a.ptr[i]; k < a.ptr[i + 1]; ++k) {
            const int64_t j = a.col[k];
            const double th = eps * std::sqrt(di * std::fabs(d[j]));
            if (j == i || std::fabs(a.val[k]) > th) {
                s.col.push_back(j);
                s.val.push_back(a.val[k]);
            }
        }
        s.ptr[i + 1] = (int64_t)s.col.size();
    }
    return s;
}

// greedy distance-2 aggregation, ascending node order (amg.py:87-125)
int64_t aggregate(const Csr &s, std::vector<int64_t> &label) {
    const int64_t n = s.nrows;
    label.assign(n, -1);
    int64_t naggr = 0;
    std::vector<int64_t> freeset;
    for (int64_t i = 0; i < n; ++i) {
        if (label[i] != -1) continue;
        int64_t nb = 0;
        freeset.clear();
        for (int64_t k = s.ptr[i]; k < s.ptr[i + 1]; ++k) {
            const int64_t j = s.col[k];
            if (j == i) continue;
            ++nb;
            if (label[j] == -1) freeset.push_back(j);
        }
        if (freeset.empty() && nb != 0) continue;
        const int64_t id = naggr++;
        label[i] = id;
        for (int64_t j : freeset) label[j] = id;
        for (int64_t j : freeset)
            for (int64_t k = s.ptr[j]; k < s.ptr[j + 1]; ++k)
                if (label[s.col[k]] == -1) label[s.col[k]] = id;
    }
    for (int64_t i = 0; i < n; ++i) {
        if (label[i] != -1) continue;
        for (int64_t k = s.ptr[i]; k < s.ptr[i + 1]; ++k) {
            const int64_t j = s.col[k];
            if (j != i && label[j] != -1) {
                label[i] = label[j];
                break;
            }
        }
    }
    return naggr;
}

// P = (I - omega D^-1 S) T with T the piecewise-constant interpolation.
// The reference builds it with from_coo over [T entries; scaled S*T entries]
// (amg.py:136-157); the duplicate at (i, label_i) sums as 1.0 + scaled.
static Csr smoothed_prolongation(const Csr &s, const std::vector<double> &d,
                                 const std::vector<int64_t> &label, int64_t naggr, double omega) {
    Csr t;
    t.nrows = s.nrows;
    t.ncols = naggr;
    t.ptr.resize(s.nrows + 1);
    t.col.resize(s.nrows);
    t.val.assign(s.nrows, 1.0);
    for (int64_t i = 0; i <= s.nrows; ++i) t.ptr[i] = i;
    for (int64_t i = 0; i < s.nrows; ++i) t.col[i] = label[i];
    Csr st = spgemm(s, t);
    Csr p;
    p.nrows = s.nrows;
    p.ncols = naggr;
    p.ptr.assign(s.nrows + 1, 0);
    p.col.reserve(st.nnz() + s.nrows);
    p.val.reserve(st.nnz() + s.nrows);
    for (int64_t i = 0; i < s.nrows; ++i) {
        const double neg = -(omega / d[i]);
        bool placed = false;
        for (int64_t k = st.ptr[i]; k < st.ptr[i + 1]; ++k) {
            const int64_t j = st.col[k];
            const double scaled = neg * st.val[k];
            if (!placed && j > label[i]) {
                p.col.push_back(label[i]);
                p.val.push_back(1.0);
                placed = true;
            }
            if (j == label[i]) {
                p.col.push_back(j);
                p.val.push_back(1.0 + scaled);
                placed = true;
            } else {
                p.col.push_back(j);
                p.val.push_back(scaled);
            }
        }
        if (!placed) {
            p.col.push_back(label[i]);
            p.val.push_back(1.0);
        }
        p.ptr[i + 1] = (int64_t)p.col.size();
    }
    return p;
}

// LU with partial pivoting, in place on a row-major n x n matrix.
// Singularity criterion of sparse.py:236-241.
int lu_inverse(int64_t n, const double *a, double *inv) {
    if (n == 0) return DFL_OK;
    std::vector<double> lu(a, a + n * n);
    std::vector<int64_t> piv(n);
    for (int64_t k = 0; k < n; ++k) {
        int64_t p = k;
        double best = std::fabs(lu[k * n + k]);
        for (int64_t i = k + 1; i < n; ++i) {
            const double v = std::fabs(lu[i * n + k]);
            if (v > best) {
                best = v;
                p = i;
            }
        }
        piv[k] = p;
        if (p != k)
            for (int64_t j = 0; j < n; ++j) std::swap(lu[k * n + j], lu[p * n + j]);
        const double pivot = lu[k * n + k];
        if (pivot != 0.0)
            for (int64_t i = k + 1; i < n; ++i) {
                const double f = lu[i * n + k] / pivot;
                lu[i * n + k] = f;
                if (f != 0.0)
                    for (int64_t j = k + 1; j < n; ++j) lu[i * n + j] -= f * lu[k * n + j];
            }
    }
    double dmax = 0.0, dmin = INFINITY;
    bool finite = true;
    for (int64_t i = 0; i < n * n; ++i)
        if (!std::isfinite(lu[i])) finite = false;
    for (int64_t i = 0; i < n; ++i) {
        const double v = std::fabs(lu[i * n + i]);
        dmax = std::max(dmax, v);
        dmin = std::min(dmin, v);
    }
    const double scale = std::max(dmax, 1e-300);
    if (!finite || dmin <= 1e-14 * scale) {
        char buf[160];
        snprintf(buf, sizeof buf, "matrix is singular to working precision (pivot ratio %.2e)",
                 dmin / scale);
        set_setup_error(buf);
        return DFL_E_SINGULAR;
    }
    // solve A X = I column by column
    std::vector<double> col(n);
    for (int64_t c = 0; c < n; ++c) {
        std::fill(col.begin(), col.end(), 0.0);
        col[c] = 1.0;
        for (int64_t k = 0; k < n; ++k)
            if (piv[k] != k) std::swap(col[k], col[piv[k]]);
        for (int64_t i = 1; i < n; ++i) {
            double s = col[i];
            for (int64_t j = 0; j < i; ++j) s -= lu[i * n + j] * col[j];
            col[i] = s;
        }
        for (int64_t i = n - 1; i >= 0; --i) {
            double s = col[i];
            for (int64_t j = i + 1; j < n; ++j) s -= lu[i * n + j] * col[j];
            col[i] = s / lu[i * n + i];
        }
        for (int64_t i = 0; i < n; ++i) inv[i * n + c] = col[i];
    }
    return DFL_OK;
}

static std::vector<double> to_dense(const Csr &a) {
    std::vector<double> d(a.nrows * a.ncols, 0.0);
    for (int64_t i = 0; i < a.nrows; ++i)
        for (int64_t k = a.ptr[i]; k < a.ptr[i + 1]; ++k) d[i * a.ncols + a.col[k]] = a.val[k];
    return d;
}

int close_bottom(Hierarchy &h, Csr &&a) {
    Level lv;
    lv.A = std::move(a);
    lv.bottom = true;
    const int64_t n = lv.A.nrows;
    lv.bottom_inv.resize(n * n);
    std::vector<double> dense = to_dense(lv.A);
    int rc = lu_inverse(n, dense.data(), lv.bottom_inv.data());
    h.levels.push_back(std::move(lv));
    return rc;
}

// amg.py:217-250
int build_hierarchy(const Csr &a0, const dfl_amg_options &o, Hierarchy &h) {
    if (o.relax != DFL_RELAX_DAMPED_JACOBI && o.relax != DFL_RELAX_SPAI0) {
        set_setup_error("relaxation must be damped_jacobi or spai0 on the B200 path");
        return DFL_E_CONFIG;
    }
    if (setup_device() >= 0) return build_hierarchy_dev(a0, o, h);
    h.levels.clear();
    h.relax = o.relax;
    Csr cur = a0;
    int li = 0;
    for (;;) {
        if (cur.nrows <= o.coarse_enough || li + 1 >= o.max_levels) return close_bottom(h, std::move(cur));
        const bool verbose = std::getenv("DFL_SETUP_VERBOSE") != nullptr;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        auto t0 = now();
        std::vector<double> d;
        if (!diagonal(cur, d, "strength graph")) return DFL_E_STRUCTURE;
        const double eps = o.eps_strong * std::ldexp(1.0, -li);
        Csr s = strength(cur, d, eps);
        auto t1 = now();
        std::vector<int64_t> label;
        const int64_t naggr = aggregate(s, label);
        auto t2 = now();
        if (verbose) fprintf(stderr, "L%d strength %.0f ms aggregate %.0f ms\n", li, ms(t0, t1), ms(t1, t2));
        if (naggr == cur.nrows) return close_bottom(h, std::move(cur));
        for (int64_t i = 0; i < cur.nrows; ++i)
            if (label[i] < 0) {
                set_setup_error("aggregation left an unassigned node");
                return DFL_E_STRUCTURE;
            }
        Level lv;
        lv.P = smoothed_prolongation(s, d, label, naggr, o.omega);
        lv.R = transpose(lv.P);
        lv.w.resize(cur.nrows);
        if (o.relax == DFL_RELAX_DAMPED_JACOBI) {
            // (damping * inv_diag) * r  (amg.py:193, inv_diag amg.py:242)
            for (int64_t i = 0; i < cur.nrows; ++i) lv.w[i] = o.damping * (1.0 / d[i]);
        } else {
            // a_ii / sum_j a_ij^2 with the sum in CSR order (amg.py:160-166)
            for (int64_t i = 0; i < cur.nrows; ++i) {
                double sq = 0.0;
                for (int64_t k = cur.ptr[i]; k < cur.ptr[i + 1]; ++k) sq = sq + cur.val[k] * cur.val[k];
                lv.w[i] = d[i] / sq;
            }
        }
        auto t3 = now();
        Csr ap = spgemm(cur, lv.P);
        Csr next = spgemm(lv.R, ap);
        if (verbose)
            fprintf(stderr, "L%d P+R+w %.0f ms RAP %.0f ms\n", li, ms(t2, t3), ms(t3, now()));
        lv.A = std::move(cur);
        h.levels.push_back(std::move(lv));
        cur = std::move(next);
        ++li;
    }
}

// AZ = A Z restricted to this rank's rows (deflation.py:140) and the rank's
// rows of E (deflation.py:144-149).
int basis_az(const dfl_csr *A, int k, const double *zext, const int32_t *owner,
             const int32_t *rowsub, int64_t K, int sub0, int nsub, int keep_zeros, Csr &az,
             double *E_rows) {
    const int64_t n = A->nrows;
    std::vector<double> acc(K, 0.0);
    std::vector<int64_t> mark(K, -1);
    std::vector<int64_t> cols;
    az.nrows = n;
    az.ncols = K;
    az.ptr.assign(n + 1, 0);
    az.col.clear();
    az.val.clear();
    // E = Z'AZ sums ~10^6 products per entry whose linear-column parts
    // cancel almost completely (A applied to a linear function vanishes in
    // the interior); a naive double sum leaves errors of ~1e-6 relative in
    // the small entries, which makes the projector inconsistent with the
    // device's Z' sums and stalls CG (200^3 jump problem, m=8: 130 vs 65
    // iterations).  Accumulate in extended precision and round once: E is
    // then Z'AZ of the stored AZ values to within an ulp, at least as
    // accurate as the reference's blocked dgemm (deflation.py:144-149).
    std::vector<long double> Eacc((size_t)nsub * k * K, 0.0L);
    for (int64_t i = 0; i < n; ++i) {
        cols.clear();
        for (int64_t e = A->row_ptr[i]; e < A->row_ptr[i + 1]; ++e) {
            const int64_t j = A->col_idx[e];
            const double av = A->values[e];
            const int64_t base = (int64_t)owner[j] * k;
            for (int c = 0; c < k; ++c) {
                const int64_t cc = base + c;
                acc[cc] = acc[cc] + av * zext[j * k + c];
                if (mark[cc] != i) {
                    mark[cc] = i;
                    cols.push_back(cc);
                }
            }
        }
        std::sort(cols.begin(), cols.end());
        // E rows: Z(i, a) * AZ(i, :) accumulated over the subdomain's rows
        const int ls = rowsub[i] - sub0;
        for (int64_t cc : cols) {
            const double v = acc[cc];
            for (int a = 0; a < k; ++a)
                Eacc[((int64_t)ls * k + a) * K + cc] += (long double)zext[i * k + a] * (long double)v;
            if (keep_zeros || v != 0.0) {
                az.col.push_back(cc);
                az.val.push_back(v);
            }
            acc[cc] = 0.0;
        }
        az.ptr[i + 1] = (int64_t)az.col.size();
    }
    for (size_t q = 0; q < Eacc.size(); ++q) E_rows[q] = (double)Eacc[q];
    return DFL_OK;
}

}  // namespace dfl

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

int dfl_abi_version(void) { return DFLB200_ABI_VERSION; }
const char *dfl_last_setup_error(void) { return dfl::setup_error(); }

int dfl_hier_build(const dfl_csr *A, const dfl_amg_options *opts, dfl_hier **out) {
    dfl::NvtxRange nv("dfl.setup.hierarchy");
    if (!A || !opts || !out) return DFL_E_STATE;
    *out = nullptr;
    if (A->nrows != A->ncols) {
        dfl::set_setup_error("matrix must be square");
        return DFL_E_DIMENSION;
    }
    try {
        auto *h = new dfl_hier;
        int rc = dfl::build_hierarchy(dfl::csr_from_view(A), *opts, h->h);
        if (rc != DFL_OK) {
            delete h;
            return rc;
        }
        *out = h;
        return DFL_OK;
    } catch (const std::bad_alloc &) {
        dfl::set_setup_error("host out of memory in hierarchy setup");
        return DFL_E_STATE;
    }
}

int dfl_hier_num_levels(const dfl_hier *h) { return h ? (int)h->h.levels.size() : 0; }

static const dfl::Csr *level_matrix(const dfl_hier *h, int level, int which) {
    if (!h || level < 0 || level >= (int)h->h.levels.size()) return nullptr;
    const dfl::Level &lv = h->h.levels[level];
    if (which == DFL_LEVEL_A) return &lv.A;
    if (lv.bottom) return nullptr;
    return which == DFL_LEVEL_P ? &lv.P : which == DFL_LEVEL_R ? &lv.R : nullptr;
}

int dfl_hier_level_shape(const dfl_hier *h, int level, int which, int64_t *nrows, int64_t *ncols,
                         int64_t *nnz) {
    const dfl::Csr *m = level_matrix(h, level, which);
    if (!m) {
        *nrows = *ncols = 0;
        *nnz = -1;
        return (h && level >= 0 && level < (int)h->h.levels.size()) ? DFL_OK : DFL_E_DIMENSION;
    }
    *nrows = m->nrows;
    *ncols = m->ncols;
    *nnz = m->nnz();
    return DFL_OK;
}

int dfl_hier_level_copy(const dfl_hier *h, int level, int which, int64_t *row_ptr,
                        int64_t *col_idx, double *values) {
    const dfl::Csr *m = level_matrix(h, level, which);
    if (!m) return DFL_E_DIMENSION;
    std::memcpy(row_ptr, m->ptr.data(), sizeof(int64_t) * m->ptr.size());
    std::memcpy(col_idx, m->col.data(), sizeof(int64_t) * m->col.size());
    std::memcpy(values, m->val.data(), sizeof(double) * m->val.size());
    return DFL_OK;
}

int dfl_hier_level_weights(const dfl_hier *h, int level, double *w) {
    if (!h || level < 0 || level >= (int)h->h.levels.size() || h->h.levels[level].bottom)
        return DFL_E_DIMENSION;
    const auto &v = h->h.levels[level].w;
    std::memcpy(w, v.data(), sizeof(double) * v.size());
    return DFL_OK;
}

int dfl_hier_bottom_inverse(const dfl_hier *h, double *inv) {
    if (!h || h->h.levels.empty()) return DFL_E_STATE;
    const auto &v = h->h.levels.back().bottom_inv;
    std::memcpy(inv, v.data(), sizeof(double) * v.size());
    return DFL_OK;
}

void dfl_hier_free(dfl_hier *h) { delete h; }

int dfl_basis_az(const dfl_csr *A, int32_t k, const double *zext, const int32_t *owner,
                 const int32_t *rowsub, int64_t K, int32_t sub0, int32_t nsub, int32_t keep_zeros,
                 dfl_matrix **AZ, double *E_rows) {
    dfl::NvtxRange nv("dfl.setup.basis");
    if (!A || !zext || !owner || !rowsub || !AZ || !E_rows || k < 1) return DFL_E_STATE;
    auto *m = new dfl_matrix;
    int rc = dfl::basis_az(A, k, zext, owner, rowsub, K, sub0, nsub, keep_zeros, m->m, E_rows);
    if (rc != DFL_OK) {
        delete m;
        return rc;
    }
    *AZ = m;
    return DFL_OK;
}

int dfl_matrix_shape(const dfl_matrix *m, int64_t *nrows, int64_t *ncols, int64_t *nnz) {
    if (!m) return DFL_E_STATE;
    *nrows = m->m.nrows;
    *ncols = m->m.ncols;
    *nnz = m->m.nnz();
    return DFL_OK;
}

int dfl_matrix_copy(const dfl_matrix *m, int64_t *row_ptr, int64_t *col_idx, double *values) {
    if (!m) return DFL_E_STATE;
    std::memcpy(row_ptr, m->m.ptr.data(), sizeof(int64_t) * m->m.ptr.size());
    std::memcpy(col_idx, m->m.col.data(), sizeof(int64_t) * m->m.col.size());
    std::memcpy(values, m->m.val.data(), sizeof(double) * m->m.val.size());
    return DFL_OK;
}

void dfl_matrix_free(dfl_matrix *m) { delete m; }

int dfl_dense_inverse(int64_t n, const double *a, double *inv) {
    if (n < 0 || (n > 0 && (!a || !inv))) return DFL_E_DIMENSION;
    return dfl::lu_inverse(n, a, inv);
}

}  // extern "C"
