/*
 * oracle.c -- CPU restatement of the reference nested recursive
 * mixed-precision Cholesky (arXiv 2601.08082, /root/reference/proj).
 *
 * TEST INFRASTRUCTURE ONLY -- the checker and the timed CPU baseline.  The
 * product library (paper_2601_08082_b200/libtreechol_b200.so) never links or
 * calls this code; see oracle.h for who may.
 *
 * Bit-exactness contract: every scalar is computed with the same operation
 * sequence as the reference, so results are identical bit for bit (pinned
 * against oracle/_ref by tests/test_oracle.py).  Two things differ only in
 * *how* the same arithmetic is scheduled:
 *   - operand rows are staged into contiguous, pre-rounded scratch arrays
 *     (round_to is a pure function, so rounding once and reusing is exact);
 *   - independent output elements run on OpenMP threads (each element's
 *     k-loop stays sequential, so the sums are unchanged).
 * Build with -ffp-contract=off and no -march.
 */
#include "oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 0;

void or_set_threads(int t) { g_threads = t; }

int or_get_threads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* precision.hpp:41-76 -- rounding                                          */
/* ------------------------------------------------------------------------ */

/* Nearest binary16 value (ties to even), widened back to double.
 * Restates precision.hpp:41-62: inf/nan pass through, double subnormals
 * flush to a signed zero, |x| >= 2^16 overflows, the quantum is 2^(e-10)
 * floored at 2^-24, and a rounded magnitude above 65504 overflows. */
double or_round_half(double x) {
    if (isnan(x) || isinf(x)) return x;
    if (x == 0.0 || fpclassify(x) == FP_SUBNORMAL) return copysign(0.0, x);
    int e2;
    (void)frexp(x, &e2);  /* x = f * 2^e2, f in [0.5,1) => unbiased exp e2-1 */
    const int e = e2 - 1;
    if (e > 15) return copysign(INFINITY, x);
    const int qe = (e < -14 ? -14 : e) - 10;
    /* |x| * 2^-qe is an exact scaling; rint is round-half-even */
    const double r = ldexp(rint(ldexp(fabs(x), -qe)), qe);
    if (r > 65504.0) return copysign(INFINITY, x);
    return copysign(r, x);
}

double or_round_to(double x, int p) {
    switch (p) {
        case OR_HALF: return or_round_half(x);
        case OR_SINGLE: return (double)(float)x; /* precision.hpp:64-66 */
        default: return x;
    }
}

static inline double rt(double x, int p) { return or_round_to(x, p); }

static inline void fl_add(or_flops* f, int level, int kernel, uint64_t n) {
    if (!f) return;
    f->by_level[level] += n;
    f->by_kernel[kernel] += n;
    f->calls[kernel] += 1;
}

/* ------------------------------------------------------------------------ */
/* kernels.cpp:23-38 -- dot_update, split into its k-loop and its epilogue  */
/* ------------------------------------------------------------------------ */

/* accumulator level: Single for Half (half_accumulator default, kernels.hpp:14),
 * the level itself otherwise (kernels.cpp:45-46) */
static inline int acc_of(int level) { return level == OR_HALF ? OR_SINGLE : level; }

/* s = sum_t x[t]*y[t] with the reference's per-term rounding; x and y are
 * already rounded to `level`.  Half: products exact, sum rounded to Single.
 * Single: product and sum rounded to Single.  Double: plain. */
static inline double dot_acc(int k, const double* x, const double* y, int level) {
    double s = 0.0;
    if (level == OR_HALF) {
        for (int t = 0; t < k; ++t) s = (double)(float)(s + x[t] * y[t]);
    } else if (level == OR_SINGLE) {
        for (int t = 0; t < k; ++t) {
            const double p = (double)(float)(x[t] * y[t]);
            s = (double)(float)(s + p);
        }
    } else {
        for (int t = 0; t < k; ++t) {
            const double p = x[t] * y[t];
            s = s + p;
        }
    }
    return s;
}

/* tail of dot_update (kernels.cpp:33-37) */
static inline double dot_finish(double s, double alpha, double beta, double c,
                                int level) {
    const int acc = acc_of(level);
    double r = rt(alpha * s, acc);
    if (beta != 0.0) r = rt(r + rt(beta * rt(c, level), acc), acc);
    return rt(r, level);
}

/* copy rows r of a column-major view into contiguous row-major scratch,
 * rounded to level: out[i*k + t] = rt(a(i, t), level) */
static double* stage_rows(const double* a, int rows, int k, int lda, int level) {
    double* out = (double*)malloc(sizeof(double) * (size_t)(rows > 0 ? rows : 1) *
                                  (size_t)(k > 0 ? k : 1));
    for (int t = 0; t < k; ++t) {
        const double* col = a + (size_t)t * lda;
        for (int i = 0; i < rows; ++i) out[(size_t)i * k + t] = rt(col[i], level);
    }
    return out;
}

/* ------------------------------------------------------------------------ */
/* kernels.cpp:9-16 round_matrix, tree.cpp:33-40 round_lower                */
/* ------------------------------------------------------------------------ */

static void round_rect(double* a, int m, int n, int ld, int level, int lower) {
    if (level == OR_DOUBLE) return;
    for (int j = 0; j < n; ++j)
        for (int i = lower ? j : 0; i < m; ++i)
            a[(size_t)j * ld + i] = rt(a[(size_t)j * ld + i], level);
}

/* ------------------------------------------------------------------------ */
/* kernels.cpp:42-69 potrf_leaf                                              */
/* ------------------------------------------------------------------------ */

int or_potrf_leaf(double* a, int n, int ld, int row0, int level, or_flops* f,
                  int* index) {
    uint64_t fl = 0;
    /* row-major rounded mirror of the solved part: row i at lr[i*n] */
    double* lr = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(n ? n : 1));
    for (int j = 0; j < n; ++j) {
        for (int i = j; i < n; ++i) {
            /* operands a(i,t), a(j,t), t < j: already final for this leaf */
            const double s = dot_acc(j, lr + (size_t)i * n, lr + (size_t)j * n, level);
            a[(size_t)j * ld + i] = dot_finish(s, -1.0, 1.0, a[(size_t)j * ld + i], level);
        }
        fl += 2ull * (uint64_t)j * (uint64_t)(n - j);
        const double piv = a[(size_t)j * ld + j];
        if (!isfinite(piv) || piv <= 0.0) {
            if (index) *index = row0 + j;
            free(lr);
            return OR_NOT_POSITIVE_DEFINITE;
        }
        const double d = rt(sqrt(piv), level);
        a[(size_t)j * ld + j] = d;
        for (int i = j + 1; i < n; ++i)
            a[(size_t)j * ld + i] = rt(a[(size_t)j * ld + i] / d, level);
        fl += 1ull + (uint64_t)(n - j - 1);
        /* publish column j into the mirror, rounded as dot_update reads it */
        for (int i = j; i < n; ++i) lr[(size_t)i * n + j] = rt(a[(size_t)j * ld + i], level);
    }
    fl_add(f, level, OR_POTRF, fl);
    free(lr);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* kernels.cpp:71-92 trsm_leaf: B <- B L^-T by column substitution          */
/* ------------------------------------------------------------------------ */

int or_trsm_leaf(double* b, int m, int n, int ldb, const double* l, int ldl,
                 int lrow0, int level, or_flops* f, int* index) {
    /* L rows rounded to level (dot_update rounds bv(t) = l(j,t)) */
    double* lrow = stage_rows(l, n, n, ldl, level);
    /* singular check order: column j is checked before any row of column j
     * is touched; rows never influence the check, so pre-scan is exact */
    int bad = -1;
    for (int j = 0; j < n; ++j) {
        const double ljj = rt(l[(size_t)j * ldl + j], level);
        if (ljj == 0.0 || !isfinite(ljj)) { bad = j; break; }
    }
    const int ncols = bad < 0 ? n : bad; /* columns fully processed */
    int i;
#pragma omp parallel for schedule(static) num_threads(or_get_threads())
    for (i = 0; i < m; ++i) {
        double* row = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
        for (int j = 0; j < ncols; ++j) {
            const double ljj = rt(l[(size_t)j * ldl + j], level);
            const double s = dot_acc(j, row, lrow + (size_t)j * n, level);
            const double r = dot_finish(s, -1.0, 1.0, b[(size_t)j * ldb + i], level);
            const double x = rt(r / ljj, level);
            b[(size_t)j * ldb + i] = x;
            row[j] = rt(x, level);
        }
        free(row);
    }
    free(lrow);
    if (bad >= 0) {
        if (index) *index = lrow0 + bad;
        return OR_SINGULAR_DIAGONAL;
    }
    uint64_t fl = 0;
    for (int j = 0; j < n; ++j) fl += (uint64_t)m * (2ull * (uint64_t)j + 1ull);
    fl_add(f, level, OR_TRSM, fl);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* kernels.cpp:94-112 syrk_leaf and kernels.cpp:114-132 gemm_mixed          */
/* ------------------------------------------------------------------------ */

void or_syrk_leaf(double* c, int n, int ldc, const double* a, int k, int lda,
                  double alpha, double beta, int level, or_flops* f) {
    double* ar = stage_rows(a, n, k, lda, level);
    int j;
#pragma omp parallel for schedule(dynamic, 1) num_threads(or_get_threads())
    for (j = 0; j < n; ++j)
        for (int i = j; i < n; ++i) {
            const double s = dot_acc(k, ar + (size_t)i * k, ar + (size_t)j * k, level);
            c[(size_t)j * ldc + i] = dot_finish(s, alpha, beta, c[(size_t)j * ldc + i], level);
        }
    free(ar);
    fl_add(f, level, OR_SYRK, (uint64_t)n * (uint64_t)(n + 1) * (uint64_t)k);
}

void or_gemm_mixed(double* c, int m, int n, int ldc, const double* a, int k,
                   int lda, const double* b, int ldb, double alpha, double beta,
                   int level, or_flops* f) {
    double* ar = stage_rows(a, m, k, lda, level);
    double* br = stage_rows(b, n, k, ldb, level);
    int j;
#pragma omp parallel for schedule(static) num_threads(or_get_threads())
    for (j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) {
            const double s = dot_acc(k, ar + (size_t)i * k, br + (size_t)j * k, level);
            c[(size_t)j * ldc + i] = dot_finish(s, alpha, beta, c[(size_t)j * ldc + i], level);
        }
    free(ar);
    free(br);
    fl_add(f, level, OR_GEMM, 2ull * (uint64_t)m * (uint64_t)n * (uint64_t)k);
}

/* ------------------------------------------------------------------------ */
/* tree.cpp:80-104 quantize / dequantize                                     */
/* ------------------------------------------------------------------------ */

static double range_max(int p) {
    return p == OR_HALF ? 65504.0 : p == OR_SINGLE ? 3.4028234663852886e38
                                                   : 1.7976931348623157e308;
}

double or_quantize_block(double* b, int m, int n, int ld, int target) {
    double amax = 0.0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) {
            const double v = fabs(b[(size_t)j * ld + i]);
            if (amax < v) amax = v; /* std::max(amax, v) keeps amax on NaN */
        }
    double alpha = amax / range_max(target);
    if (!(alpha > 1.0)) alpha = 1.0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i)
            b[(size_t)j * ld + i] = rt(b[(size_t)j * ld + i] / alpha, target);
    return alpha;
}

void or_dequantize_block(double* b, int m, int n, int ld, double alpha, int level) {
    if (alpha == 1.0) return;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i)
            b[(size_t)j * ld + i] = rt(b[(size_t)j * ld + i] * alpha, level);
}

/* ------------------------------------------------------------------------ */
/* tree.cpp:42-152 -- the recursion.  A node is (offset r0, order n, depth) */
/* inside one buffer; the tree is implicit (n1 = n/2, leaf iff n <= b).      */
/* ------------------------------------------------------------------------ */

typedef struct {
    double* a;
    int lda;
    int b;          /* leaf size used to build */
    int leaf_size;  /* SolveOptions::leaf_size (== b via factor_matrix) */
    const int* levels;
    int nlevels;
    int quantize;
    or_flops* fl;
    char* detail;
    int detail_len;
    int index;
} ctx_t;

static int at_depth(const ctx_t* c, int d) {
    return c->levels[d < c->nlevels ? d : c->nlevels - 1];
}
static int leaf_level(const ctx_t* c) { return c->levels[c->nlevels - 1]; }
static double* at(const ctx_t* c, int i, int j) { return c->a + (size_t)j * c->lda + i; }

/* build_node rounding (tree.cpp:42-66): leaves to the leaf level (lower
 * triangle), off-diagonals too when quantization is off */
static void build_node(ctx_t* c, int r0, int n, int depth) {
    if (n <= c->b) {
        round_rect(at(c, r0, r0), n, n, c->lda, leaf_level(c), 1);
        return;
    }
    const int n1 = n / 2, n2 = n - n1;
    if (!c->quantize) round_rect(at(c, r0 + n1, r0), n2, n1, c->lda, at_depth(c, depth), 0);
    build_node(c, r0, n1, depth + 1);
    build_node(c, r0 + n1, n2, depth + 1);
}

/* require_finite (tree.cpp:19-31), exact what() text */
static int require_finite(ctx_t* c, int r0, int c0, int m, int n, int lower,
                          const char* what) {
    for (int j = 0; j < n; ++j)
        for (int i = lower ? j : 0; i < m; ++i)
            if (!isfinite(*at(c, r0 + i, c0 + j))) {
                if (c->detail && c->detail_len > 0)
                    snprintf(c->detail, (size_t)c->detail_len,
                             "non-finite value in %s block (rows %d..%d, cols %d..%d) "
                             "at element (%d, %d)",
                             what, r0, r0 + m - 1, c0, c0 + n - 1, r0 + i, c0 + j);
                return OR_NUMERICAL_BREAKDOWN;
            }
    return OR_OK;
}

/* tree_trsm (tree.cpp:127-138): B (rows x cols at (br, bc)) against the L
 * subtree rooted at (lr0, ln, ldepth) */
static int tree_trsm(ctx_t* c, int br, int bc, int rows, int cols, int p,
                     int lr0, int ln, int ldepth) {
    const int lleaf = ln <= c->b;
    const int mn = rows < cols ? rows : cols;
    if (lleaf || mn <= c->leaf_size) {
        int idx = 0;
        const int st = or_trsm_leaf(at(c, br, bc), rows, cols, c->lda, at(c, lr0, lr0),
                                    c->lda, lr0, p, c->fl, &idx);
        if (st != OR_OK) c->index = idx;
        return st;
    }
    const int n1 = ln / 2, n2 = ln - n1;
    int st = tree_trsm(c, br, bc, rows, n1, p, lr0, n1, ldepth + 1);
    if (st) return st;
    or_gemm_mixed(at(c, br, bc + n1), rows, cols - n1, c->lda, at(c, br, bc), n1, c->lda,
                  at(c, lr0 + n1, lr0), c->lda, -1.0, 1.0, p, c->fl);
    return tree_trsm(c, br, bc + n1, rows, cols - n1, p, lr0 + n1, n2, ldepth + 1);
}

/* tree_syrk (tree.cpp:140-152): C subtree (cr0, cn, cdepth), A rows x k at (ar, ac) */
static void tree_syrk(ctx_t* c, int cr0, int cn, int cdepth, int ar, int ac,
                      int arows, int k, double alpha, double beta, int p) {
    if (cn <= c->b) {
        or_syrk_leaf(at(c, cr0, cr0), cn, c->lda, at(c, ar, ac), k, c->lda, alpha, beta,
                     leaf_level(c), c->fl);
        return;
    }
    const int n1 = cn / 2, n2 = cn - n1;
    tree_syrk(c, cr0, n1, cdepth + 1, ar, ac, n1, k, alpha, beta, p);
    or_gemm_mixed(at(c, cr0 + n1, cr0), n2, n1, c->lda, at(c, ar + n1, ac), k, c->lda,
                  at(c, ar, ac), c->lda, alpha, beta, at_depth(c, cdepth), c->fl);
    tree_syrk(c, cr0 + n1, n2, cdepth + 1, ar + n1, ac, arows - n1, k, alpha, beta, p);
}

/* tree_potrf (tree.cpp:106-125) */
static int tree_potrf(ctx_t* c, int r0, int n, int depth) {
    if (n <= c->b) {
        int st = require_finite(c, r0, r0, n, n, 1, "diagonal");
        if (st) return st;
        int idx = 0;
        st = or_potrf_leaf(at(c, r0, r0), n, c->lda, r0, leaf_level(c), c->fl, &idx);
        if (st) c->index = idx;
        return st;
    }
    const int n1 = n / 2, n2 = n - n1;
    const int p = at_depth(c, depth);
    int st = tree_potrf(c, r0, n1, depth + 1);
    if (st) return st;
    st = require_finite(c, r0 + n1, r0, n2, n1, 0, "off-diagonal");
    if (st) return st;
    double alpha = 1.0;
    if (c->quantize) alpha = or_quantize_block(at(c, r0 + n1, r0), n2, n1, c->lda, p);
    st = tree_trsm(c, r0 + n1, r0, n2, n1, p, r0, n1, depth + 1);
    if (st) return st;
    or_dequantize_block(at(c, r0 + n1, r0), n2, n1, c->lda, alpha, p);
    st = require_finite(c, r0 + n1, r0, n2, n1, 0, "off-diagonal");
    if (st) return st;
    tree_syrk(c, r0 + n1, n2, depth + 1, r0 + n1, r0, n2, n1, -1.0, 1.0, p);
    return tree_potrf(c, r0 + n1, n2, depth + 1);
}

static void set_detail(char* d, int len, const char* msg) {
    if (d && len > 0) snprintf(d, (size_t)len, "%s", msg);
}

int or_tree_potrf(int n, double* a, int lda, int b, const int* levels,
                  int nlevels, int quantize, or_flops* fl, char* detail,
                  int detail_len) {
    if (detail && detail_len > 0) detail[0] = '\0';
    /* build_tree argument checks (tree.cpp:70-78) */
    if (b < 1) { set_detail(detail, detail_len, "leaf size must be >= 1"); return OR_INVALID_ARGUMENT; }
    if (nlevels < 1) { set_detail(detail, detail_len, "empty precision config"); return OR_INVALID_ARGUMENT; }
    if (n < 1) { set_detail(detail, detail_len, "tree requires a square matrix of order >= 1"); return OR_INVALID_ARGUMENT; }
    ctx_t c = {a, lda, b, b, levels, nlevels, quantize, fl, detail, detail_len, 0};
    build_node(&c, 0, n, 0);
    const int st = tree_potrf(&c, 0, n, 0);
    if (st == OR_NOT_POSITIVE_DEFINITE && detail && detail_len > 0)
        snprintf(detail, (size_t)detail_len,
                 "matrix is not positive definite: pivot %d is non-positive or non-finite",
                 c.index);
    if (st == OR_SINGULAR_DIAGONAL && detail && detail_len > 0)
        snprintf(detail, (size_t)detail_len,
                 "singular triangular factor: diagonal entry %d is zero or non-finite", c.index);
    return st;
}

/* ------------------------------------------------------------------------ */
/* analysis.cpp:12-28 spd_generate -- mt19937_64 written out                 */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    static const uint64_t MATA = 0xB5026F5AA96619E9ULL;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= MATA;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

void or_spd_generate(int n, uint64_t seed, double* a) {
    /* R drawn column-major over the full square; A = (R + R^T)/2, A_jj += n */
    double* r = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
    mt64 s;
    mt64_seed(&s, seed);
    for (size_t t = 0; t < (size_t)n * (size_t)n; ++t)
        r[t] = (double)(mt64_next(&s) >> 11) * 0x1p-53;
    for (int j = 0; j < n; ++j) {
        for (int i = 0; i < n; ++i)
            a[(size_t)j * n + i] = 0.5 * (r[(size_t)j * n + i] + r[(size_t)i * n + j]);
        a[(size_t)j * n + j] += (double)n;
    }
    free(r);
}

/* ------------------------------------------------------------------------ */
/* analysis.cpp:30-62 factorization_error                                    */
/* ------------------------------------------------------------------------ */

double or_factorization_error(int n, const double* a, int lda, const double* l, int ldl) {
    for (int j = 0; j < n; ++j)
        for (int i = j; i < n; ++i)
            if (!isfinite(a[(size_t)j * lda + i]) || !isfinite(l[(size_t)j * ldl + i]))
                return NAN;
    /* lrow[i*n + k] = l(i,k) for k <= i (lower only is ever read) */
    double* lrow = (double*)calloc((size_t)n * (size_t)n, sizeof(double));
    for (int k = 0; k < n; ++k)
        for (int i = k; i < n; ++i) lrow[(size_t)i * n + k] = l[(size_t)k * ldl + i];
    double* e = (double*)malloc(sizeof(double) * (size_t)n * (size_t)n);
    int j;
    /* per element, e(i,j) -= l(i,k)*l(j,k) for k = 0..j in increasing k,
     * skipping l(j,k) == 0 -- the reference's k-outer loop order per element */
#pragma omp parallel for schedule(dynamic, 4) num_threads(or_get_threads())
    for (j = 0; j < n; ++j) {
        const double* lj = lrow + (size_t)j * n;
        for (int i = j; i < n; ++i) {
            const double* li = lrow + (size_t)i * n;
            double v = a[(size_t)j * lda + i];
            for (int k = 0; k <= j; ++k) {
                const double ljk = lj[k];
                if (ljk == 0.0) continue;
                const double p = li[k] * ljk;
                v -= p;
            }
            e[(size_t)j * n + i] = v;
        }
    }
    double num = 0.0, den = 0.0;
    for (j = 0; j < n; ++j)
        for (int i = j; i < n; ++i) {
            const double w = (i == j) ? 1.0 : 2.0;
            const double ev = e[(size_t)j * n + i], av = a[(size_t)j * lda + i];
            num += w * ev * ev;
            den += w * av * av;
        }
    free(lrow);
    free(e);
    return sqrt(num / den);
}

/* ------------------------------------------------------------------------ */
/* analysis.cpp:64-120 flop_breakdown (StaticCounter)                        */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t b;
    const int* levels;
    int nlevels;
    or_flops* f;
} sc_t;

static int sc_level(const sc_t* s, int d) { return s->levels[d < s->nlevels ? d : s->nlevels - 1]; }

static void sc_trsm(sc_t* s, uint64_t m, uint64_t n, int d, int p) {
    if (n <= s->b || m <= s->b) { fl_add(s->f, p, OR_TRSM, m * n * n); return; }
    const uint64_t n1 = n / 2, n2 = n - n1;
    sc_trsm(s, m, n1, d + 1, p);
    fl_add(s->f, p, OR_GEMM, 2 * m * n2 * n1);
    sc_trsm(s, m, n2, d + 1, p);
}

static void sc_syrk(sc_t* s, uint64_t n, uint64_t k, int d, int p) {
    if (n <= s->b) { fl_add(s->f, s->levels[s->nlevels - 1], OR_SYRK, n * (n + 1) * k); return; }
    const uint64_t n1 = n / 2, n2 = n - n1;
    sc_syrk(s, n1, k, d + 1, p);
    fl_add(s->f, sc_level(s, d), OR_GEMM, 2 * n2 * n1 * k);
    sc_syrk(s, n2, k, d + 1, p);
}

static void sc_potrf(sc_t* s, uint64_t n, int d) {
    if (n <= s->b) {
        fl_add(s->f, s->levels[s->nlevels - 1], OR_POTRF, n * (n + 1) * (2 * n + 1) / 6);
        return;
    }
    const uint64_t n1 = n / 2, n2 = n - n1;
    const int p = sc_level(s, d);
    sc_potrf(s, n1, d + 1);
    sc_trsm(s, n2, n1, d + 1, p);
    sc_syrk(s, n2, n1, d + 1, p);
    sc_potrf(s, n2, d + 1);
}

void or_flop_breakdown(int n, int b, const int* levels, int nlevels, or_flops* out) {
    memset(out, 0, sizeof(*out));
    if (n < 1 || b < 1 || nlevels < 1) return;
    sc_t s = {(uint64_t)b, levels, nlevels, out};
    sc_potrf(&s, (uint64_t)n, 0);
}

/* ------------------------------------------------------------------------ */
/* analysis.cpp:122-155 factor_matrix                                        */
/* ------------------------------------------------------------------------ */

int or_factor_matrix(int n, const double* a, int b, const int* levels, int nlevels,
                     int quantize, double* l, double* rel_error, or_flops* fl,
                     char* detail, int detail_len) {
    memcpy(l, a, sizeof(double) * (size_t)n * (size_t)n);
    if (fl) memset(fl, 0, sizeof(*fl));
    const int st = or_tree_potrf(n, l, n, b, levels, nlevels, quantize, fl, detail, detail_len);
    if (rel_error) *rel_error = (st == OR_OK) ? or_factorization_error(n, a, n, l, n) : NAN;
    return st;
}

/* ------------------------------------------------------------------------ */
/* POTRS restatement (no reference counterpart)                  */
/* ------------------------------------------------------------------------ */

void or_potrs(int n, const double* l, int ldl, double* rhs, int ldb, int nrhs) {
    for (int r = 0; r < nrhs; ++r) {
        double* y = rhs + (size_t)r * ldb;
        /* forward: trsm_leaf at Double on the 1 x n row b^T (kernels.cpp:71-92) */
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int t = 0; t < j; ++t) {
                const double p = y[t] * l[(size_t)t * ldl + j];
                s = s + p;
            }
            double v = -1.0 * s;
            v = v + 1.0 * y[j];
            y[j] = v / l[(size_t)j * ldl + j];
        }
        /* backward: L^T x = y, t descending */
        for (int j = n - 1; j >= 0; --j) {
            double s = 0.0;
            for (int t = j + 1; t < n; ++t) {
                const double p = l[(size_t)j * ldl + t] * y[t];
                s = s + p;
            }
            y[j] = (y[j] - s) / l[(size_t)j * ldl + j];
        }
    }
}
