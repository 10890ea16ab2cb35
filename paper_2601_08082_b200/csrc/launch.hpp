// launch.hpp -- host-side launchers of the sm_100a kernels (internal).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "device.cuh"
#include "plan.hpp"

#include <string>

namespace tcb {

struct BlockDescHost {
    int r0, c0, m, n, level, lower;
};

// elementwise (k_elementwise.cu)
int make_block_table(const std::vector<BlockDescHost>& in, std::vector<BlockDesc>& out);
void launch_import(const DevCtx& c, const BlockDesc* d_blocks, int nb, int tiles, cudaStream_t s);
void launch_export(const DevCtx& c, const BlockDesc* d_blocks, int nb, int tiles, cudaStream_t s);
void launch_shadow(const DevCtx& c, const BlockDesc* d_blocks, int nb, int tiles, int p, cudaStream_t s);
void launch_check(const DevCtx& c, int lv, int r0, int c0, int m, int n, int lower, uint32_t seq,
                  cudaStream_t s);
void launch_quant(const DevCtx& c, int lv, int r0, int c0, int m, int n, int slot, uint32_t seq,
                  cudaStream_t s);
// chk_dr, chk_dc: offset of (r0, c0) from the checked block's origin (the
// failure element is reported relative to that block)
void launch_dequant(const DevCtx& c, int lv, int r0, int c0, int m, int n, int slot, uint32_t chk_seq, int chk_dr,
                    int chk_dc, cudaStream_t s);

// spin until *host_flag (mapped pinned memory) becomes non-zero (profiling)
void launch_noop(cudaStream_t s);
void launch_gate(volatile int* host_flag, cudaStream_t s);
void launch_stamp(unsigned long long* out, cudaStream_t s);

// row-major level image of a column-major double block (k_elementwise.cu)
void launch_level_image(int m, int n, const double* src, long long lds, int level, int lower, void* dst,
                        long long ldd, cudaStream_t s);
// spd_generate symmetrization of raw draws (k_elementwise.cu)
void launch_symmetrize(double* a, long long lda, int n, cudaStream_t s);

// one-time kernel attributes (before any graph capture)
void init_leaf_attributes();
void init_tc_attributes();

// leaves (k_leaf.cu)
void launch_potrf_leaf(const DevCtx& c, int lv, int r0, int n, uint32_t seq, uint32_t chk_seq, cudaStream_t s,
                       uint32_t inv_seq = 0, int fuse_inv = 0, int shadow16 = 0);
void launch_trsm_leaf(const DevCtx& c, int lv, int br0, int bc0, int m, int n, int lr0, uint32_t seq,
                      uint32_t chk_seq, int chk_r0, int chk_c0, cudaStream_t s);
// latency-optimised F16/F32 leaves, n % 32 == 0, n <= 256 (k_leaf_cm.cu)
bool leaf_cm_ok(int lv, int n);
void init_leaf_cm_attributes();
void launch_potrf_cm(const DevCtx& c, int lv, int r0, int n, uint32_t seq, uint32_t chk, cudaStream_t s);
void launch_trsm_cm(const DevCtx& c, int lv, int br0, int bc0, int m, int n, int lr0, uint32_t seq,
                    uint32_t chk_seq, int chk_r0, int chk_c0, cudaStream_t s);
void launch_leaf_inverse(const DevCtx& c, int r0, int n, uint32_t seq, cudaStream_t s);
// leaf inverse W = inv(L), n % 32 == 0, n <= 256: mode 0 -> W16 pair, 1 -> W32 (k_inverse.cu)
bool inv2_ok(int n);
void init_inv2_attributes();
void launch_leaf_inv2(const DevCtx& c, int mode, int r0, int n, uint32_t seq, cudaStream_t s);
// 512-thread F16/F32 leaf POTRF, n % 32 == 0, n <= 256 (k_potrf.cu)
bool potrf_v2_ok(int lv, int n);
void init_potrf_v2_attributes();
// fuse_inv (F32 leaves): also W = inv(L) into the FP32 inverse workspace,
// reporting a singular diagonal under inv_seq (the leaf's OP_INVERSE)
// shadow16 (F32 leaves): also the binary16 copy into the F16 level buffer
void launch_potrf_v2(const DevCtx& c, int lv, int r0, int n, uint32_t seq, uint32_t chk, cudaStream_t s,
                     uint32_t inv_seq = 0, int fuse_inv = 0, int shadow16 = 0);

// grouped GEMM (k_gemm_simt.cu / k_gemm_tc.cu)
// problems must already be in device memory with tile0 / tiles_n filled by
// the matching *_tiles() helper
constexpr int M32_TILE = 32;  // output tile of the mma.sync FP32 kernel (GC_MMA32)
constexpr int M32W_ROWS = 16; // rows per CTA of its full-width in-place variant (GC_MMA32W; k_gemm_simt.cu WM)
int simt_tiles(std::vector<DevProb>& probs, int tile = 0, int tile_n = 0);  // 0: the 64x64 SIMT tile
void init_mma32w_attributes();
void launch_gemm_simt(const DevCtx& c, int gclass, const DevProb* d_probs, int nprob, int tiles,
                      cudaStream_t s);

struct TcProb;  // defined in k_gemm_tc.cu (holds TMA descriptors)
size_t tc_prob_size();
// fills host-side TcProb records (tensor maps over the F16 buffer)
// operand kinds of the tensor-core GEMM (k_gemm_tc.cu)
// tcgen05 GEMM kinds: FP16 (128x256 tiles), three-pass TF32 (128x128),
// FP16 on 128x128 tiles (lists too small to fill the SMs with 128x256 ones)
enum { KIND_F16 = 0, KIND_TF32X3 = 1, KIND_F16N = 2 };
int tc_build_probs(const DevCtx& c, int kind, const std::vector<DevProb>& probs, std::vector<unsigned char>& out,
                   std::string* err,
                   int pair = 0);
// FP16 kind on CTA pairs (tcgen05 cta_group::2, 256x256 tiles); the table
// built with tc_build_probs(..., pair = 1)
int tc_pair_min_tiles();
// process-wide copy-kernel setting ("elem_tiles_per_cta"); false: unknown key
bool elem_set_option(const std::string& key, int value);
// FP16 lists of fewer 128x256 tiles than this run on 128x128 tiles (0 = never)
int tc_narrow_max_tiles();
// the kernel variant and table for one problem list (tf32: the three-pass
// kind): CTA pairs at >= pair_min tiles (0 = never), the narrow FP16 kind
// below narrow_max tiles (-1: the process-wide tc_narrow_max_tiles); returns
// the tile count (< 0: error) and sets *kind, *pair
int tc_select_tables(const DevCtx& c, bool tf32, const std::vector<DevProb>& probs, std::vector<unsigned char>& out,
                     std::string* err, int pair_min, int narrow_max, int* kind, int* pair);
void launch_gemm_tc_pair(const DevCtx& c, int kind, const void* d_probs, int nprob, int tiles, cudaStream_t s,
                         int tiles_per_pair = 0, int max_ctas = 0);
void launch_gemm_tc(const DevCtx& c, int kind, const void* d_probs, int nprob, int tiles, cudaStream_t s,
                    int max_ctas = 0, int tiles_per_cta = 0);
bool tc_supported();
// process-wide tensor-core GEMM settings ("tc_kchunk"); false: unknown key
bool tc_set_option(const std::string& key, int value);
bool potrs_set_option(const std::string& key, int value);  // "potrs_poll" (k_verify.cu)

// standalone block operations on column-major doubles (k_blockops.cu)
void bo_round(double* a, long long lda, int m, int n, int lv, int lower, cudaStream_t s);
void bo_quantize(double* a, long long lda, int m, int n, int lv, unsigned long long* d_amax, double* d_alpha,
                 cudaStream_t s);
void bo_absmax(const double* a, long long lda, int m, int n, unsigned long long* d_amax, cudaStream_t s);
void bo_dequantize(double* a, long long lda, int m, int n, int lv, double alpha, cudaStream_t s);
void bo_gemm(double* c, long long ldc, const double* a, long long lda, const double* b, long long ldb, int m, int n,
             int k, double alpha, double beta, int lv, int acc, int lower, cudaStream_t s);
void bo_potrf(double* a, long long lda, int n, int lv, int acc, int* d_status, cudaStream_t s);
void bo_trsm(double* b, long long ldb, const double* l, long long ldl, int m, int n, int lv, int acc, int* d_status,
             cudaStream_t s);

// verification (k_verify.cu)
void launch_fact_error(int n, const double* dA, long long lda, const double* dL, long long ldl,
                       double* d_partials, int* d_nonfinite, int tiles_per_side, cudaStream_t s);
int fact_error_partials(int n, int* tiles_per_side);
void launch_potrs(int n, const double* dL, long long ldl, double* dB, long long ldb, int nrhs,
                  int* d_counters, double* d_work, cudaStream_t s, int max_ctas = 0);
size_t potrs_work_doubles(int n, int nrhs);  // incl. the flag / ticket words
size_t potrs_batch_work_bytes(int n, int nsys, int nrhs);
// the POTRS of nsys systems in one launch sequence (device pointer tables)
void launch_potrs_batch(int n, int nsys, const double* const* d_Ltab, long long ldl, double* const* d_Btab,
                        long long ldb, int nrhs, void* d_work, int max_ctas, cudaStream_t s);
void launch_residual(int n, const double* dA, long long lda, const double* dX, const double* dB,
                     double* d_partials, cudaStream_t s);
int residual_partials(int n);

}  // namespace tcb
