/*
 * oracle.h -- CPU restatement of the reference tree-Cholesky path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product library links this file;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * liboracle.so, and only as the checker or the timed CPU baseline.
 *
 * Every function restates one reference function (file:line relative to
 * /root/reference/proj).  The restatement is bit-exact against the compiled
 * reference (oracle/_ref, see tests/test_oracle.py), which itself reproduces
 * proj/test_output.txt.  Parity is therefore PINNED for the factorization,
 * the flop accounting, the generator and the error metric.  POTRS has no
 * reference implementation: or_potrs is a restatement defined in SURVEY 8(c)
 * and its parity is UNPINNED.
 *
 * Conventions: matrices are column-major doubles, element (i,j) at
 * a[j*ld + i], exactly like TileView (include/treechol/matrix.hpp:11-24).
 * Precision tags: 0 = Half, 1 = Single, 2 = Double (precision.hpp:14).
 */
#ifndef TREECHOL_ORACLE_H
#define TREECHOL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_HALF = 0, OR_SINGLE = 1, OR_DOUBLE = 2 };
enum { OR_POTRF = 0, OR_TRSM = 1, OR_SYRK = 2, OR_GEMM = 3 };
/* status codes (mirrors analysis.cpp:139-146 plus the kernel exceptions) */
enum {
    OR_OK = 0,
    OR_NOT_POSITIVE_DEFINITE = 1,
    OR_NUMERICAL_BREAKDOWN = 2,
    OR_SINGULAR_DIAGONAL = 3,
    OR_INVALID_ARGUMENT = 4
};

/* flop record: by_level[3], by_kernel[4], calls[4] (flops.hpp:17-48) */
typedef struct {
    uint64_t by_level[3];
    uint64_t by_kernel[4];
    uint64_t calls[4];
} or_flops;

double or_round_half(double x);
double or_round_to(double x, int p);

void or_spd_generate(int n, uint64_t seed, double* a);
double or_factorization_error(int n, const double* a, int lda,
                              const double* l, int ldl);
void or_flop_breakdown(int n, int b, const int* levels, int nlevels,
                       or_flops* out);

/* leaf kernels; views are (ptr, rows, cols, ld, row0, col0). Return a status;
 * *index receives the global index for NPD / singular diagonal. */
int or_potrf_leaf(double* a, int n, int ld, int row0, int level,
                  or_flops* fl, int* index);
int or_trsm_leaf(double* b, int m, int n, int ldb, const double* l, int ldl,
                 int lrow0, int level, or_flops* fl, int* index);
void or_syrk_leaf(double* c, int n, int ldc, const double* a, int k, int lda,
                  double alpha, double beta, int level, or_flops* fl);
void or_gemm_mixed(double* c, int m, int n, int ldc, const double* a,
                   int k, int lda, const double* b, int ldb, double alpha,
                   double beta, int level, or_flops* fl);
double or_quantize_block(double* b, int m, int n, int ld, int target);
void or_dequantize_block(double* b, int m, int n, int ld, double alpha,
                         int level);

/* Whole factorization in place on a (build_tree + tree_potrf).  detail gets
 * the exact what() text of the reference exception on failure. */
int or_tree_potrf(int n, double* a, int lda, int b, const int* levels,
                  int nlevels, int quantize, or_flops* fl, char* detail,
                  int detail_len);

/* factor_matrix restatement (analysis.cpp:122-155): copies A, factors the
 * copy into l (n*n col-major), fills rel_error (NaN unless ok). */
int or_factor_matrix(int n, const double* a, int b, const int* levels,
                     int nlevels, int quantize, double* l, double* rel_error,
                     or_flops* fl, char* detail, int detail_len);

/* POTRS restatement (no reference counterpart): forward substitution is
 * trsm_leaf at Double with B = b^T (kernels.cpp:71-92); backward
 * substitution L^T x = y in plain double.  Overwrites rhs (n x nrhs). */
void or_potrs(int n, const double* l, int ldl, double* rhs, int ldb,
              int nrhs);

/* threads used by the OpenMP loops (0 = library default) */
void or_set_threads(int t);
int or_get_threads(void);

#ifdef __cplusplus
}
#endif

#endif
