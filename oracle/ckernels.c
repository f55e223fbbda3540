/*
 * TEST INFRASTRUCTURE ONLY -- never linked into the product.
 *
 * Plain-C restatement of the reference's compiled CSR loops and of its
 * greedy aggregation, used by oracle/port.py as the CPU checker for the
 * B200 solve path (and as the CPU baseline arm of bench.py).
 *
 *   csr_spmv        <- pkg/src/deflamg/_kernels.pyx:11-23  (spmv_rows)
 *   csr_transpose   <- pkg/src/deflamg/_kernels.pyx:26-52  (transpose)
 *   csr_spgemm_*    <- pkg/src/deflamg/_kernels.pyx:55-115 (spgemm)
 *   greedy_aggregate<- pkg/src/deflamg/amg.py:87-125       (aggregate)
 *
 * Summation orders follow the reference exactly (sequential, CSR order,
 * no FMA contraction: built with -ffp-contract=off).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* out[i] = sum_k val[k] * x[col[k]] for i in [lo, hi), accumulated from 0.0
 * in storage order. */
void csr_spmv(const int64_t *ptr, const int64_t *col, const double *val,
              const double *x, double *out, int64_t lo, int64_t hi)
{
    for (int64_t i = lo; i < hi; ++i) {
        double s = 0.0;
        const int64_t e = ptr[i + 1];
        for (int64_t k = ptr[i]; k < e; ++k)
            s = s + val[k] * x[col[k]];
        out[i] = s;
    }
}

/* Counting-sort transpose. tptr must be zeroed, length ncols+1. */
void csr_transpose(int64_t nrows, int64_t ncols, const int64_t *ptr,
                   const int64_t *col, const double *val, int64_t *tptr,
                   int64_t *tcol, double *tval)
{
    const int64_t nnz = ptr[nrows];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncols > 0 ? ncols : 1));
    for (int64_t k = 0; k < nnz; ++k) tptr[col[k] + 1] += 1;
    for (int64_t c = 0; c < ncols; ++c) {
        tptr[c + 1] += tptr[c];
        cursor[c] = tptr[c];
    }
    for (int64_t i = 0; i < nrows; ++i)
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            int64_t d = cursor[col[k]]++;
            tcol[d] = i;
            tval[d] = val[k];
        }
    free(cursor);
}

/* Pass 1 of the Gustavson product: row counts of C = A B into cptr
 * (length anrows+1, cptr[0] = 0 on return). */
void csr_spgemm_count(int64_t anrows, const int64_t *aptr, const int64_t *acol,
                      int64_t bncols, const int64_t *bptr, const int64_t *bcol,
                      int64_t *cptr)
{
    int64_t *mark = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bncols > 0 ? bncols : 1));
    for (int64_t j = 0; j < bncols; ++j) mark[j] = -1;
    cptr[0] = 0;
    for (int64_t i = 0; i < anrows; ++i) {
        int64_t cnt = 0;
        for (int64_t ka = aptr[i]; ka < aptr[i + 1]; ++ka) {
            const int64_t r = acol[ka];
            for (int64_t kb = bptr[r]; kb < bptr[r + 1]; ++kb) {
                const int64_t j = bcol[kb];
                if (mark[j] != i) { mark[j] = i; ++cnt; }
            }
        }
        cptr[i + 1] = cptr[i] + cnt;
    }
    free(mark);
}

/* Pass 2: accumulate in A-entry then B-entry order into a dense row buffer,
 * insertion-sort the touched columns, gather the sums. */
void csr_spgemm_fill(int64_t anrows, const int64_t *aptr, const int64_t *acol,
                     const double *aval, int64_t bncols, const int64_t *bptr,
                     const int64_t *bcol, const double *bval, const int64_t *cptr,
                     int64_t *ccol, double *cval)
{
    double *acc = (double *)calloc((size_t)(bncols > 0 ? bncols : 1), sizeof(double));
    int64_t *mark = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bncols > 0 ? bncols : 1));
    for (int64_t j = 0; j < bncols; ++j) mark[j] = -1;
    for (int64_t i = 0; i < anrows; ++i) {
        int64_t *cols = ccol + cptr[i];
        int64_t len = 0;
        for (int64_t ka = aptr[i]; ka < aptr[i + 1]; ++ka) {
            const int64_t r = acol[ka];
            const double a = aval[ka];
            for (int64_t kb = bptr[r]; kb < bptr[r + 1]; ++kb) {
                const int64_t j = bcol[kb];
                acc[j] += a * bval[kb];
                if (mark[j] != i) { mark[j] = i; cols[len++] = j; }
            }
        }
        for (int64_t p = 1; p < len; ++p) {
            int64_t key = cols[p], q = p - 1;
            while (q >= 0 && cols[q] > key) { cols[q + 1] = cols[q]; --q; }
            cols[q + 1] = key;
        }
        for (int64_t p = 0; p < len; ++p) {
            cval[cptr[i] + p] = acc[cols[p]];
            acc[cols[p]] = 0.0;
        }
    }
    free(acc);
    free(mark);
}

/* Greedy distance-2 aggregation over a strength graph (ptr/col include the
 * diagonal). labels has length n; returns the number of aggregates. */
int64_t greedy_aggregate(int64_t n, const int64_t *ptr, const int64_t *col, int64_t *labels)
{
    int64_t naggr = 0;
    for (int64_t i = 0; i < n; ++i) labels[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (labels[i] != -1) continue;
        int64_t nb = 0, nfree = 0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            const int64_t j = col[k];
            if (j == i) continue;
            ++nb;
            if (labels[j] == -1) ++nfree;
        }
        if (nfree == 0 && nb != 0) continue; /* second pass */
        const int64_t a = naggr++;
        labels[i] = a;
        /* the reference snapshots the free set before labelling it */
        int64_t *freeset = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nfree > 0 ? nfree : 1));
        int64_t f = 0;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            const int64_t j = col[k];
            if (j != i && labels[j] == -1) freeset[f++] = j;
        }
        for (int64_t q = 0; q < f; ++q) labels[freeset[q]] = a;
        for (int64_t q = 0; q < f; ++q) {
            const int64_t j = freeset[q];
            for (int64_t k = ptr[j]; k < ptr[j + 1]; ++k)
                if (labels[col[k]] == -1) labels[col[k]] = a;
        }
        free(freeset);
    }
    for (int64_t i = 0; i < n; ++i) {
        if (labels[i] != -1) continue;
        for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
            const int64_t j = col[k];
            if (j != i && labels[j] != -1) { labels[i] = labels[j]; break; }
        }
    }
    return naggr;
}
