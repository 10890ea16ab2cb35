/*
 * treechol_c.h -- C ABI of the B200-native nested recursive mixed-precision
 * Cholesky (libtreechol_b200.so).
 *
 * This is the drop-in boundary: plain pointers, sizes and int status codes,
 * no C++ or torch types.  Each entry point names the reference interface it
 * replaces (file:line under /root/reference/proj).  The C++ headers in
 * include/treechol/ (same API as the reference's proj/include/treechol) are
 * implemented on top of these calls; INTEGRATION.md shows the ctypes and C++
 * bindings a maintainer would add.
 *
 * Storage contract (matrix.hpp:11-24): matrices are column-major doubles,
 * element (i,j) at a[j*lda + i].  The factor L overwrites the lower
 * triangle; the strict upper triangle is never read or written.  Every value
 * written is a double holding a value of its block's precision level.
 */
#ifndef TREECHOL_C_H
#define TREECHOL_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The C++ shim maps them back onto the reference exception
 * types (errors.hpp:8-62) with identical what() text. */
typedef enum {
    TC_OK = 0,
    TC_NOT_POSITIVE_DEFINITE = 1, /* NotPositiveDefinite, kernels.cpp:57-60  */
    TC_NUMERICAL_BREAKDOWN = 2,   /* NumericalBreakdown, tree.cpp:19-31     */
    TC_SINGULAR_DIAGONAL = 3,     /* SingularDiagonal, kernels.cpp:79-81    */
    TC_INVALID_ARGUMENT = 4,      /* InvalidArgument, tree.cpp:72-76        */
    TC_SYNTAX_ERROR = 5,          /* SyntaxError, precision.cpp:52-100      */
    TC_VALIDATION_ERROR = 6,      /* ValidationError, precision.cpp:103-109 */
    TC_CUDA_ERROR = 7,            /* device/runtime failure (no reference)  */
    TC_NO_DEVICE = 8              /* no CUDA device: there is no CPU path   */
} tc_status;

/* Precision tags, identical to treechol::Precision (precision.hpp:14). */
enum { TC_F16 = 0, TC_F32 = 1, TC_F64 = 2 };
/* Kernel tags, identical to treechol::Kernel (flops.hpp:10). */
enum { TC_K_POTRF = 0, TC_K_TRSM = 1, TC_K_SYRK = 2, TC_K_GEMM = 3 };

/* FlopBreakdown (flops.hpp:17-48) */
typedef struct {
    uint64_t by_level[3];
    uint64_t by_kernel[4];
    uint64_t calls[4];
} tc_flops;

/* Failure details of the last factorization on a plan. */
typedef struct {
    int status;      /* tc_status */
    int index;       /* NPD / singular: global row index (errors.hpp:27-43) */
    int row0, row1;  /* breakdown: block rows a..b, cols c..d (tree.cpp:23-27) */
    int col0, col1;
    int elem_row;    /* breakdown: global element (i, j) */
    int elem_col;
    int diagonal;    /* breakdown: 1 = "diagonal" block, 0 = "off-diagonal" */
} tc_info;

typedef struct tc_plan tc_plan;

/* ---- configuration (precision.hpp:81-99, precision.cpp:17-111) -------- */

/* PrecisionConfig::parse.  levels must hold >= 16 ints. */
int tc_config_parse(const char* text, int* levels, int* nlevels);
/* PrecisionConfig::to_string into buf (NUL-terminated). */
int tc_config_to_string(const int* levels, int nlevels, char* buf, int buflen);

/* ---- planning (build_tree, tree.cpp:42-78; flop_breakdown, analysis.cpp:64-120) */

/* flop_breakdown(n, b, config): static count, no device needed. */
int tc_flop_breakdown(int n, int b, const int* levels, int nlevels, tc_flops* out);

/* build_tree(view, config, b, quantize) + SolveOptions{leaf_size}: plans
 * the factorization of an order-n matrix.  Pure host work: no device memory
 * is touched until the first factorization.  leaf_size <= 0 means b. */
int tc_plan_create(int n, int b, const int* levels, int nlevels, int quantize,
                   int leaf_size, tc_plan** out);
void tc_plan_destroy(tc_plan* plan);
/* the flops tree_potrf adds to SolveOptions::flops (tree.cpp:106-152) */
int tc_plan_flops(const tc_plan* plan, tc_flops* out);
/* plan statistics: number of device ops / kernel launches per factorization */
int tc_plan_stats(const tc_plan* plan, int* n_ops, int* n_launches, int* n_gemm_problems);
/* execution knobs: use_graph (default 1), n_streams (default 6),
 * use_tc (default 1: tcgen05 for FP16-operand GEMMs; 0 = SIMT path),
 * use_tc32 (default 1: three-pass TF32 tcgen05 for FP32 x FP32 GEMMs),
 * dag_graph (1: explicit DAG graph; 0: stream capture), inverse_trsm,
 * fuse_checks, syrk_split_min, bulk_tiles_per_cta, bulk_max_ctas,
 * mma32_max_log2 (FP32 GEMMs with m*n*k <= 2^v on mma.sync, default 24),
 * mma32w_max_log2 (in-place FP32 leaf solves on full-width mma.sync tiles,
 * default 28); the plan-shaping ones before the first run */
int tc_plan_set_option(tc_plan* plan, const char* key, int value);

/* ---- factorization (tree_potrf, tree.cpp:106-125) ---------------------- */

/* Device-resident factorization.  Reads A (column-major doubles, lda) from
 * device memory dA_in and writes L's lower triangle into dL_out (may equal
 * dA_in for the in-place drop-in).  stream: a cudaStream_t or NULL.
 * If info != NULL the call synchronizes and reports the outcome; with
 * info == NULL it only enqueues (read the outcome with tc_plan_status). */
int tc_potrf_device(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out,
                    int lda_out, void* stream, tc_info* info);
/* Host buffers, in place on A (the reference's TileView contract): the lower
 * triangle is copied to the device in leaf-column strips, factored, and every
 * block is copied back as soon as it is final, so the copies overlap the
 * factorization (one captured graph per (A, lda) when A is pinned).  The
 * strict upper triangle is returned bit-for-bit unchanged. */
int tc_potrf_host(tc_plan* plan, double* A, int lda, tc_info* info);
/* Serialized, eagerly launched run with a CUDA event after every op:
 * op_ms[i] = device time of op i (cap entries).  For roofline accounting. */
int tc_plan_profile(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out,
                    int lda_out, void* stream, float* op_ms, int cap);
/* Eager multi-stream run with timing events around every op: t_start[i],
 * t_end[i] = ms from the run's start (the concurrency timeline). */
int tc_plan_timeline(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out, int lda_out,
                     void* stream, float* t_start, float* t_end, int cap);
/* development: the same for the host entry point (eager, pinned host buffer
 * factored in place): op start/end plus the completion time of each H2D copy
 * (block order) and each D2H copy (export order), ms from the first copy */
int tc_plan_timeline_host(tc_plan* plan, double* host, int lda, void* stream, float* t_start, float* t_end,
                          int cap_ops, float* t_h2d, int cap_h2d, float* t_d2h, int cap_d2h);
/* development: one run of the host entry point's own CUDA graph with a
 * global-timer stamp after every op / H2D / D2H node: completion times in ms
 * from the graph's root (ops in op order, H2D in block order, D2H in export
 * order; -1 = not run) */
int tc_plan_trace_host(tc_plan* plan, double* host, int lda, void* stream, float* t_ops, int cap_ops, float* t_h2d,
                       int cap_h2d, float* t_d2h, int cap_d2h);
/* development: the same for the device entry point's DAG graph: completion
 * time of every op in ms from the graph's root (-1e9 = not run) */
int tc_plan_trace_device(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out, int lda_out, void* stream,
                         float* t_ops, int cap_ops);
/* op i of the plan: type (0 import, 1 export, 2 check, 3 quant, 4 dequant,
 * 5 shadow, 6 potrf leaf, 7 trsm leaf, 8 gemm), gemm class (0 = tcgen05
 * FP16, 1..5 SIMT classes, -1 otherwise), level, algorithmic flops, rect */
int tc_plan_op_info(const tc_plan* plan, int i, int* type, int* gclass, int* level,
                    double* flops, int* rect4);
/* development: the GEMM problems of op i (0 for other ops), 13 ints each --
 * m, n, k, a_r0, a_c0, a_kwrap, b_buf, b_r0, b_c0, c_r0, c_c0, exec_level,
 * lower -- up to cap problems; returns the count */
int tc_plan_op_probs(const tc_plan* plan, int i, int* out, int cap);
/* dependencies of op i (indices of earlier ops); returns their count
 * (entries beyond cap are not written), -1 on a bad index */
int tc_plan_op_deps(const tc_plan* plan, int i, int* deps, int cap);
/* flops of the last run as SolveOptions::flops would hold them: the full
 * plan on success, the calls completed before the failure otherwise */
int tc_plan_run_flops(const tc_plan* plan, tc_flops* out);
/* Synchronize the plan's last factorization and decode its status. */
int tc_plan_status(tc_plan* plan, tc_info* info);
/* Human-readable text identical to the reference exception's what(). */
int tc_info_message(const tc_plan* plan, const tc_info* info, char* buf, int buflen);

/* ---- solve (no reference counterpart) -------------- */

/* Solves A X = B with the factor in dL (column-major doubles, lower
 * triangle), B overwritten by X (n x nrhs, ldb).  Forward then backward
 * substitution in FP64 on the device. */
int tc_potrs_device(int n, const double* dL, int ldl, double* dB, int ldb, int nrhs,
                    void* stream);

/* The solves of nsys independent systems in one launch sequence: system k
 * has its factor at dL[k] and right-hand sides at dB[k] (arrays of device
 * pointers on the host; common n, ldl, ldb, nrhs).  Synchronous. */
int tc_potrs_batch_device(int n, int nsys, const double* const* dL, int ldl, double* const* dB, int ldb,
                          int nrhs, void* stream);

/* ---- distributed single factorization (BASELINE config C5) ------------- */

/* Compact forms of the two distributed pieces (BASELINE config C5 at
 * N = 131072; paper_2601_08082_b200/distributed.py):
 *  _trsm_ext: L11 is not imported from doubles -- the caller writes rn_p(L11)
 *    (p = the panel level) into the plan's level buffer rows [0, n1)
 *    (tc_plan_level_buffer, tc_level_image_device); the caller's doubles hold
 *    only the m panel rows.
 *  _syrk_rows_ext: the solved panel is written by the caller into the level
 *    buffer rows [row_hi, row_hi + n2); the caller's doubles hold only A22's
 *    rows [row_lo, row_hi).
 * tc_plan_input_rows gives the caller operand's first row (its pointer refers
 * to that row) and row count (the leading dimension must be at least that). */
int tc_plan_create_trsm_ext(int n1, int m, int b, const int* levels, int nlevels, int leaf_size, tc_plan** out);
int tc_plan_create_syrk_rows_ext(int n2, int k, int b, const int* levels, int nlevels, int row_lo, int row_hi,
                                 tc_plan** out);
int tc_plan_input_rows(const tc_plan* plan, int* row0, int* rows);
/* device bytes the plan's workspace takes (level-buffer windows, leaf
 * inverses); no device needed */
int tc_plan_device_bytes(const tc_plan* plan, unsigned long long* bytes);
/* the allocated window of a level buffer (row-major, ld elements): *ptr is
 * row *row_lo; rows [*row_lo, *row_hi) exist.  Allocates on first use. */
int tc_plan_level_buffer(tc_plan* plan, int level, void** ptr, long long* ld, int* row_lo, int* row_hi);
/* dst (row-major, ldd) = rn_level(src) of an m x n column-major double
 * block, strict upper triangle zero when lower != 0 (asynchronous) */
int tc_level_image_device(int m, int n, const double* src, int lds, int level, int lower, void* dst, long long ldd,
                          void* stream);

/* The two pieces a rank runs for the top split of an order-N factorization
 * (n1 = N/2, n2 = N - n1) besides whole factorizations; levels are the big
 * tree's (the split's subtrees sit at depth 1, its panel at depth 0).
 * tc_plan_create_trsm: the caller's buffer (device, column-major doubles,
 *   lda >= n1 + m) holds the factored L11 in rows [0, n1) and a row block of
 *   A21 in rows [n1, n1 + m); the run quantizes the block with the alpha of
 *   tc_plan_set_external_absmax (the max |A21| over ALL ranks' rows),
 *   solves it against L11 (tree_trsm, tree.cpp:127-138), dequantizes and
 *   writes it back in place (rows [n1, n1 + m) only).
 * tc_plan_create_syrk_rows: the buffer (lda >= 2 n2) holds A22 in rows
 *   [0, n2) (columns [0, n2)) and the solved A21 in rows [n2, 2 n2)
 *   (columns [0, n1)); the run applies tree_syrk(A22, A21) (tree.cpp:
 *   140-152) to A22's rows [row_lo, row_hi) and writes those rows back.
 * Both run through tc_potrf_device like a factorization plan.  Row blocks
 * of a GEMM are independent, so the distributed factor equals the
 * single-device one bit for bit (tests/test_distributed.py). */
int tc_plan_create_trsm(int n1, int m, int b, const int* levels, int nlevels, int leaf_size, tc_plan** out);
int tc_plan_create_syrk_rows(int n2, int k, int b, const int* levels, int nlevels, int row_lo, int row_hi,
                             tc_plan** out);
int tc_plan_set_external_absmax(tc_plan* plan, double absmax);
/* storage extent (rows, cols) a plan's caller buffer must cover */
int tc_plan_extent(const tc_plan* plan, int* rows, int* cols);
/* max |A(i,j)| over an m x n device block (NaN skipped, like quantize_block) */
int tc_absmax_device(int m, int n, const double* dA, int lda, double* out, void* stream);

/* ---- batched POTRF + POTRS (BASELINE config C4) ------------------------ */

/* A batch driver for independent order-n systems with one precision tree:
 * `concurrency` plans (own workspace, graph and stream each) run systems
 * side by side on the current device. */
typedef struct tc_batch tc_batch;
int tc_batch_create(int n, int b, const int* levels, int nlevels, int quantize, int concurrency,
                    tc_batch** out);
void tc_batch_destroy(tc_batch* batch);
/* execution knobs of every plan of the batch (bulk_tiles_per_cta, dag_graph,
 * use_graph; see tc_plan_set_option), before the first run; and
 * "solve_order" (any time): 0 (default) every factorization first, then the
 * solves; 1 each system's POTRS right behind its factorization */
int tc_batch_set_option(tc_batch* batch, const char* key, int value);
/* Factors dA[k] in place (device, column-major, lda) for k < count and, if
 * dB && dB[k], solves A X = B for its nrhs right-hand sides (dB[k], ldb,
 * overwritten by X).  status[k] = tc_status of system k; index[k] (optional)
 * = its failing row.  Returns TC_OK, the first failing status, or an
 * argument / device error. */
int tc_batch_run(tc_batch* batch, int count, double* const* dA, int lda, double* const* dB, int ldb,
                 int nrhs, int* status, int* index);

/* device milliseconds of the last tc_batch_run's batched solve phase (every
 * POTRS of the call in one launch sequence; solve_order 0), 0 if none ran */
int tc_batch_solve_ms(const tc_batch* batch, float* ms);

/* ---- analysis (analysis.cpp) ------------------------------------------- */

/* spd_generate(n, seed) into a host column-major buffer (lda >= n);
 * bit-identical to analysis.cpp:12-28 (mt19937_64). */
int tc_spd_generate_host(int n, uint64_t seed, double* A, int lda);
/* the same matrix straight into device memory: the host streams the raw
 * mt19937_64 draws, the device symmetrizes them (bit-identical) */
int tc_spd_generate_device(int n, uint64_t seed, double* dA, int lda, void* stream);
/* ||A - L L^T||_F / ||A||_F on the device in FP64 (analysis.cpp:30-62):
 * only lower triangles are read; NaN if any lower entry is non-finite. */
int tc_factorization_error_device(int n, const double* dA, int lda, const double* dL,
                                  int ldl, double* out, void* stream);
/* the same metric on host buffers (staged through device memory) */
int tc_factorization_error_host(int n, const double* A, int lda, const double* L, int ldl, double* out);
/* ||b - A x||_2 / (||A||_F ||x||_2 + ||b||_2) with A symmetric (lower read) */
int tc_solve_residual_device(int n, const double* dA, int lda, const double* dX,
                             const double* dB, double* out, void* stream);

/* ---- standalone block operations (kernels.hpp:20-40, tree.hpp:47-51) ---
 * The reference's kernel-level API on column-major doubles, executed on the
 * device with the reference's scalar operation order (bit-identical).  Not
 * used by the factorization path.  `acc` is the accumulator level of Half
 * GEMM-style sums (KernelContext::half_accumulator; ignored at F32/F64).
 * *_device: device pointers, enqueued on `stream`.  *_host: host pointers;
 * the call stages the block through device memory and synchronizes.
 * Failures: *fail_index = the block-local index (pivot / diagonal entry),
 * status TC_NOT_POSITIVE_DEFINITE / TC_SINGULAR_DIAGONAL. */

/* round_matrix (kernels.cpp:9-16); lower != 0: lower triangle only
 * (round_lower, tree.cpp:33-40) */
int tc_round_host(int m, int n, double* A, int lda, int level, int lower);
/* quantize_block (tree.cpp:80-95): returns alpha in *alpha */
int tc_quantize_host(int m, int n, double* B, int ldb, int level, double* alpha);
/* dequantize_block (tree.cpp:97-104) */
int tc_dequantize_host(int m, int n, double* B, int ldb, int level, double alpha);
/* potrf_leaf (kernels.cpp:42-69) on the n x n lower triangle */
int tc_potrf_leaf_host(int n, double* A, int lda, int level, int acc, int* fail_index);
/* trsm_leaf (kernels.cpp:71-92): B (m x n) <- B L^-T, L n x n */
int tc_trsm_leaf_host(int m, int n, double* B, int ldb, const double* L, int ldl, int level, int acc,
                      int* fail_index);
/* gemm_mixed (kernels.cpp:114-132): C (m x n) <- beta C + alpha A B^T, k
 * columns; lower != 0: syrk_leaf (kernels.cpp:94-112), m == n, B may be A */
int tc_gemm_mixed_host(int m, int n, int k, double* C, int ldc, const double* A, int lda, const double* B, int ldb,
                       double alpha, double beta, int level, int acc, int lower);
int tc_gemm_mixed_device(int m, int n, int k, double* dC, int ldc, const double* dA, int lda, const double* dB,
                         int ldb, double alpha, double beta, int level, int acc, int lower, void* stream);

/* ---- development ------------------------------------------------------- */

/* one launch of the grouped GEMM of class gclass (0 tcgen05 FP16, 6 tcgen05
 * three-pass TF32, 1..5 SIMT) on scratch buffers: C (m x n) -= A (m x k) B^T
 * (n x k), exec level exec_level, optional lower mask (SYRK leaf) and beta;
 * *avg_us = mean device time of `iters` back-to-back launches */
int tc_debug_gemm(int gclass, int m, int n, int k, int lower, double beta, int exec_level, int iters,
                  float* avg_us);

/* one problem of grouped-GEMM class gclass on caller device level buffers
 * (row-major, ld = ldw; the engine's layout): C(c_r0.., c_c0..) =
 * epi(C, alpha * A(a_r0.., a_c0..) B(b_r0.., b_c0..)^T) with the dot_update
 * tail of kernels.cpp:23-38 at exec_level, optional lower mask (syrk_leaf).
 * prob = {m, n, k, a_r0, a_c0, b_r0, b_c0, c_r0, c_c0, exec_level, lower}.
 * Operands come from the operand level's buffer (b16 for FP16 classes, b32
 * for FP32 classes, b64 for SIMT F64), C from the exec level's buffer.
 * Synchronous.  Kernel-level parity tests (tests/test_gpu_kernels.py). */
/* development: 15 %globaltimer stamps (ns) of CTA 0 of the last
 * tc_debug_gemm launch (tcgen05 classes; 0 = not reached): entry, after
 * setup, first TMA issued, first stage landed, accumulator ready, epilogue
 * done, exit, then epilogue detail (C staged, computed, synced, stores
 * issued) */
int tc_debug_gemm_stamps(unsigned long long* out15);

/* development: FP64 FLOP/s of the whole GPU, `ctas` CTAs of 256 threads
 * issuing `iters` x 4 independent instructions per warp: kind 0 DMMA
 * (mma.sync m8n8k4 f64, the FP64 tensor pipe), 1 DFMA (SIMT).  The
 * denominator of the FP64 rooflines (profiles/r02_fp64_peak.json). */
double tc_debug_fp64_probe(int kind, int iters, int ctas);
/* development: accumulated phase cycles of the leaf kernels since the last
 * reset (CTA 0 of each launch).  potrf: load, a, b1, b2, store, launches;
 * inverse: load, reciprocals, diagonal inverses, products, triangular
 * multiplies, store, launches */
int tc_debug_potrf_clocks(long long* out8, int reset);
int tc_debug_inv_clocks(long long* out8, int reset);
/* development: FMA/s of one SM on mma.sync (0 tf32 m16n8k8, 1 f16 m16n8k16) */
double tc_debug_mma_probe(int kind, int iters);

/* process-wide kernel settings for measurements: "tc_kchunk" = K chunk
 * (elements) of FP32-exec tensor-core accumulations, 0 = one accumulation.
 * Applies to plans built (graphs captured) afterwards. */
int tc_set_global_option(const char* key, int value);

int tc_gemm_problem_device(int gclass, void* b16, void* b32, void* b64, long long ldw, const int* prob,
                           double alpha, double beta, void* stream);

/* ---- misc --------------------------------------------------------------- */

/* thread-local text of the last error (argument / CUDA failures) */
const char* tc_last_error(void);
/* 1 if a CUDA device is usable */
int tc_device_available(void);
/* library build tag */
const char* tc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TREECHOL_C_H */
