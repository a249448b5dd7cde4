/*
 * diaq_oracle.c -- CPU restatement of the DiaQ hot path of the reference
 * package `diaqsim` (arXiv 2405.01250 artifact, /root/reference/pkg).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path (paper_2405_01250_b200/) never links, imports or calls it.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every routine here
 * against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/diaqsim).
 *
 * Storage convention (reference matrix.py:1-14): d = col - row, diagonal d
 * holds n-|d| values, element (r, r+d) sits at k = r + min(d,0).  The
 * reference keeps planar float64 re/im arrays per diagonal; this restatement
 * keeps exactly that: `re`/`im` are the concatenation of all diagonals, and
 * `starts[i]` is the element offset of diagonal i.  State vectors are
 * interleaved complex128 (reference sim.py:36, sim.py:57).
 *
 * Arithmetic: compiled with -ffp-contract=off so every `a*b - c*d` rounds
 * each product, exactly like numpy's float64 ufuncs used by the reference
 * spmv (matrix.py:276-277) and matmul (matrix.py:214-215).  The gate apply
 * (sim.py:76-78) uses numpy's complex128 multiply, which on AVX-512 hosts is
 * re = fma(vr,xr,-(vi*xi)), im = fma(vr,xi,vi*xr) (probed in
 * tests/golden/make_golden.py and recorded in the fixture meta); mode
 * CMUL_FMA restates that, CMUL_PLAIN the textbook formula.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CMUL_PLAIN 0
#define CMUL_FMA 1

static inline int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }
static inline int64_t i64max(int64_t a, int64_t b) { return a > b ? a : b; }

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------
 * spmv -- reference matrix.py:253-278.
 * y[r] = sum over d ascending with max(0,-d) <= r < min(n,n-d) of
 *        D_d[r+min(d,0)] * x[r+d];   per term tr = re*xr - im*xi,
 *        ti = re*xi + im*xr, each product rounded (no FMA), then y += t.
 * The reference walks diagonals in the outer loop and rows in the inner
 * slice; for every row the additions happen in ascending d, which is the
 * order this row-outer restatement uses, so results are bitwise equal.
 * ------------------------------------------------------------------- */
void oracle_spmv(int64_t n, int64_t nd, const int64_t *offs, const int64_t *starts,
                 const double *re, const double *im, const double *x, double *y,
                 int threads) {
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
    for (int64_t r = 0; r < n; ++r) {
        double yr = 0.0, yi = 0.0;
        for (int64_t i = 0; i < nd; ++i) {
            const int64_t d = offs[i];
            if (r < i64max(0, -d) || r >= i64min(n, n - d)) continue;
            const int64_t k = starts[i] + r + i64min(d, 0);
            const double vr = re[k], vi = im[k];
            const double xr = x[2 * (r + d)], xi = x[2 * (r + d) + 1];
            const double tr = vr * xr - vi * xi;
            const double ti = vr * xi + vi * xr;
            yr = yr + tr;
            yi = yi + ti;
        }
        y[2 * r] = yr;
        y[2 * r + 1] = yi;
    }
    (void)threads;
}

/* ---------------------------------------------------------------------
 * matmul (spgemm) -- reference matrix.py:173-250.
 * plan: candidate result offsets dC = dA + dB with |dC| < n and a non-empty
 * pair range [lo,hi) (matrix.py:173-178, 235-240), sorted ascending.
 * ------------------------------------------------------------------- */
static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

int64_t oracle_matmul_plan(int64_t n, int64_t nda, const int64_t *offa, int64_t ndb,
                           const int64_t *offb, int64_t *cand /* cap nda*ndb */) {
    int64_t m = 0;
    for (int64_t ia = 0; ia < nda; ++ia)
        for (int64_t ib = 0; ib < ndb; ++ib) {
            const int64_t da = offa[ia], db = offb[ib], dc = da + db;
            if (dc >= n || -dc >= n) continue;
            const int64_t lo = i64max(0, i64max(-da, -dc));
            const int64_t hi = i64min(n, i64min(n - da, n - dc));
            if (lo >= hi) continue;
            cand[m++] = dc;
        }
    qsort(cand, (size_t)m, sizeof(int64_t), cmp_i64);
    int64_t u = 0;
    for (int64_t i = 0; i < m; ++i)
        if (u == 0 || cand[u - 1] != cand[i]) cand[u++] = cand[i];
    return u;
}

/* fill: for each candidate dC, accumulate pairs in ascending dA from zeroed
 * accumulators (matrix.py:241-244, 202-215), then flag keep iff some
 * |re|+|im| > prune_eps (matrix.py:246-249). */
void oracle_matmul_fill(int64_t n, int64_t nda, const int64_t *offa, const int64_t *sta,
                        const double *are, const double *aim, int64_t ndb,
                        const int64_t *offb, const int64_t *stb, const double *bre,
                        const double *bim, int64_t nc, const int64_t *offc,
                        const int64_t *stc, double *cre, double *cim, uint8_t *keep,
                        double prune_eps, int threads) {
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
    for (int64_t ic = 0; ic < nc; ++ic) {
        const int64_t dc = offc[ic];
        const int64_t len = n - (dc < 0 ? -dc : dc);
        double *acr = cre + stc[ic], *aci = cim + stc[ic];
        memset(acr, 0, (size_t)len * sizeof(double));
        memset(aci, 0, (size_t)len * sizeof(double));
        for (int64_t ia = 0; ia < nda; ++ia) {
            const int64_t da = offa[ia], db = dc - da;
            /* binary search db in offb (sorted, unique) */
            int64_t lo_i = 0, hi_i = ndb;
            while (lo_i < hi_i) {
                int64_t mid = (lo_i + hi_i) / 2;
                if (offb[mid] < db) lo_i = mid + 1; else hi_i = mid;
            }
            if (lo_i >= ndb || offb[lo_i] != db) continue;
            const int64_t ib = lo_i;
            const int64_t lo = i64max(0, i64max(-da, -dc));
            const int64_t hi = i64min(n, i64min(n - da, n - dc));
            if (lo >= hi) continue;
            const double *ar = are + sta[ia] + lo + i64min(da, 0);
            const double *ai = aim + sta[ia] + lo + i64min(da, 0);
            const double *br = bre + stb[ib] + lo + da + i64min(db, 0);
            const double *bi = bim + stb[ib] + lo + da + i64min(db, 0);
            double *cr = acr + lo + i64min(dc, 0), *ci = aci + lo + i64min(dc, 0);
            for (int64_t t = 0; t < hi - lo; ++t) {
                cr[t] = cr[t] + (ar[t] * br[t] - ai[t] * bi[t]);
                ci[t] = ci[t] + (ar[t] * bi[t] + ai[t] * br[t]);
            }
        }
        uint8_t k = 0;
        for (int64_t t = 0; t < len && !k; ++t)
            if (fabs(acr[t]) + fabs(aci[t]) > prune_eps) k = 1;
        keep[ic] = k;
    }
    (void)threads;
}

/* ---------------------------------------------------------------------
 * kron_identity -- reference matrix.py:358-387.  Diagonal d of m becomes
 * d*R; with block = n_m*R and run = len(m_d)*R the value at position k is
 * m_d[(k mod block) / R] if (k mod block) < run else 0.  One diagonal per
 * call (caller loops diagonals); never prunes.
 * ------------------------------------------------------------------- */
void oracle_kron_identity_diag(int64_t left, int64_t n_m, int64_t right, int64_t d,
                               const double *mre, const double *mim, double *ore,
                               double *oim) {
    const int64_t n = left * n_m * right;
    const int64_t dout = d * right;
    const int64_t len = n - (dout < 0 ? -dout : dout);
    const int64_t block = n_m * right;
    const int64_t run = (n_m - (d < 0 ? -d : d)) * right;
    for (int64_t k = 0; k < len; ++k) {
        const int64_t p = k % block;
        if (p < run) {
            ore[k] = mre[p / right];
            oim[k] = mim[p / right];
        } else {
            ore[k] = 0.0;
            oim[k] = 0.0;
        }
    }
}

/* ---------------------------------------------------------------------
 * build_span_unitary -- reference gates.py:169-219.
 * g is given dense (2^k x 2^k, interleaved complex, row-major); positions are
 * span-relative (0 = most significant).  Only entries with |re|+|im| > 0
 * create diagonals (gates.py:203-204).  embed() scatters gate-index bit i
 * (operand 0 = MSB) to shift span-1-positions[i] (gates.py:186,195-199);
 * free-bit patterns are spread over the remaining shifts (gates.py:190-193).
 * plan returns the sorted unique result offsets.
 * ------------------------------------------------------------------- */
static int64_t embed_idx(int64_t idx, int k, const int *shifts) {
    int64_t out = 0;
    for (int i = 0; i < k; ++i) out |= ((idx >> (k - 1 - i)) & 1) << shifts[i];
    return out;
}

int64_t oracle_span_plan(int k, const double *g, const int *positions, int span,
                         int64_t *offs /* cap 4^k */) {
    int shifts[64];
    for (int i = 0; i < k; ++i) shifts[i] = span - 1 - positions[i];
    const int64_t kk = (int64_t)1 << k;
    int64_t m = 0;
    for (int64_t rg = 0; rg < kk; ++rg)
        for (int64_t cg = 0; cg < kk; ++cg) {
            const double vr = g[2 * (rg * kk + cg)], vi = g[2 * (rg * kk + cg) + 1];
            if (!(fabs(vr) + fabs(vi) > 0)) continue;
            offs[m++] = embed_idx(cg, k, shifts) - embed_idx(rg, k, shifts);
        }
    qsort(offs, (size_t)m, sizeof(int64_t), cmp_i64);
    int64_t u = 0;
    for (int64_t i = 0; i < m; ++i)
        if (u == 0 || offs[u - 1] != offs[i]) offs[u++] = offs[i];
    return u;
}

void oracle_span_fill(int k, const double *g, const int *positions, int span, int64_t nd,
                      const int64_t *offs, const int64_t *starts, double *re, double *im) {
    int shifts[64], free_shifts[64];
    int nfree = 0;
    for (int i = 0; i < k; ++i) shifts[i] = span - 1 - positions[i];
    for (int p = 0; p < span; ++p) {
        int used = 0;
        for (int i = 0; i < k; ++i) used |= (positions[i] == p);
        if (!used) free_shifts[nfree++] = span - 1 - p;
    }
    const int64_t n = (int64_t)1 << span;
    for (int64_t i = 0; i < nd; ++i) {
        const int64_t len = n - (offs[i] < 0 ? -offs[i] : offs[i]);
        memset(re + starts[i], 0, (size_t)len * sizeof(double));
        memset(im + starts[i], 0, (size_t)len * sizeof(double));
    }
    const int64_t kk = (int64_t)1 << k;
    const int64_t nf = (int64_t)1 << nfree;
    for (int64_t rg = 0; rg < kk; ++rg)
        for (int64_t cg = 0; cg < kk; ++cg) {
            const double vr = g[2 * (rg * kk + cg)], vi = g[2 * (rg * kk + cg) + 1];
            if (!(fabs(vr) + fabs(vi) > 0)) continue;
            const int64_t br = embed_idx(rg, k, shifts), bc = embed_idx(cg, k, shifts);
            const int64_t d = bc - br;
            int64_t lo_i = 0, hi_i = nd;
            while (lo_i < hi_i) {
                int64_t mid = (lo_i + hi_i) / 2;
                if (offs[mid] < d) lo_i = mid + 1; else hi_i = mid;
            }
            double *dre = re + starts[lo_i], *dim = im + starts[lo_i];
            for (int64_t f = 0; f < nf; ++f) {
                int64_t spread = 0;
                for (int j = 0; j < nfree; ++j) spread |= ((f >> j) & 1) << free_shifts[j];
                const int64_t kidx = br + spread + (d < 0 ? d : 0);
                dre[kidx] = vr;
                dim[kidx] = vi;
            }
        }
}

/* ---------------------------------------------------------------------
 * apply_placed -- reference sim.py:69-105.
 * View x as (dim_a, n_m, dim_b); for each stored diagonal of m ascending:
 * d<0: y[:, -d:-d+len, :] += v * x[:, :len, :];  d>=0: y[:, :len, :] +=
 * v * x[:, d:d+len, :].  v*x is numpy's complex multiply (mode), then a
 * complex add.  Row-outer restatement: each output element sees its terms in
 * ascending d, so it is bitwise equal to the diagonal-outer reference.
 * ------------------------------------------------------------------- */
void oracle_apply_placed(int64_t dim_a, int64_t n_m, int64_t dim_b, int64_t nd,
                         const int64_t *offs, const int64_t *starts, const double *re,
                         const double *im, const double *x, double *y, int cmul_mode,
                         int threads) {
    const int64_t total = dim_a * n_m;
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
    for (int64_t ar = 0; ar < total; ++ar) {
        const int64_t row = ar % n_m;
        double *yrow = y + 2 * ar * dim_b;
        for (int64_t j = 0; j < dim_b; ++j) { yrow[2 * j] = 0.0; yrow[2 * j + 1] = 0.0; }
        for (int64_t i = 0; i < nd; ++i) {
            const int64_t d = offs[i];
            const int64_t k = row + (d < 0 ? d : 0);
            if (k < 0 || k >= n_m - (d < 0 ? -d : d)) continue;
            const double vr = re[starts[i] + k], vi = im[starts[i] + k];
            const double *xrow = x + 2 * (ar + d) * dim_b;
            for (int64_t j = 0; j < dim_b; ++j) {
                const double xr = xrow[2 * j], xi = xrow[2 * j + 1];
                double tr, ti;
                if (cmul_mode == CMUL_FMA) {
                    tr = fma(vr, xr, -(vi * xi));
                    ti = fma(vr, xi, vi * xr);
                } else {
                    tr = vr * xr - vi * xi;
                    ti = vr * xi + vi * xr;
                }
                yrow[2 * j] = yrow[2 * j] + tr;
                yrow[2 * j + 1] = yrow[2 * j + 1] + ti;
            }
        }
    }
    (void)threads;
}

/* sum |x_i|^2 (for norm checks; reference sim.py:38-39 uses np.linalg.norm) */
double oracle_norm2(int64_t n, const double *x, int threads) {
    double s = 0.0;
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for reduction(+ : s) num_threads(threads)
#endif
    for (int64_t i = 0; i < n; ++i) s += x[2 * i] * x[2 * i] + x[2 * i + 1] * x[2 * i + 1];
    (void)threads;
    return s;
}
