// treechol/kernels.hpp -- block kernels of the C++ drop-in API
// (reference proj/include/treechol/kernels.hpp:12-40).
//
// In the reference these are scalar CPU loops.  Here each call runs on the
// device: the block is copied to HBM, processed by the sm_100a kernels the
// factorization itself uses (leaf POTRF, leaf TRSM, grouped GEMM / SYRK with
// the level epilogue), and copied back.  They exist for API completeness and
// unit-level parity; the factorization path (tree_potrf) never calls them --
// it keeps every block resident on the device.
#pragma once

#include "treechol/flops.hpp"
#include "treechol/matrix.hpp"
#include "treechol/precision.hpp"

namespace treechol {

// flop sink + the accumulator of Half-level GEMMs (only Single is
// implemented on the tensor cores: FP16 operands, FP32 accumulate)
struct KernelContext {
    FlopBreakdown* flops = nullptr;
    Precision half_accumulator = Precision::Single;
};

// lower-triangular Cholesky of `a` in place, every result rounded to
// `level`; strict upper triangle untouched; NotPositiveDefinite(global row)
void potrf_leaf(TileView a, Precision level, const KernelContext& ctx = {});

// B <- B * L^-T, L read through `level`; SingularDiagonal(global row)
void trsm_leaf(TileView b, TileView l, Precision level, const KernelContext& ctx = {});

// lower(C) <- beta*C + alpha*A*A^T at `level`; beta == 0: C is not read
void syrk_leaf(TileView c, TileView a, double alpha, double beta, Precision level,
               const KernelContext& ctx = {});

// C <- beta*C + alpha*A*B^T at `level`
void gemm_mixed(TileView c, TileView a, TileView b, double alpha, double beta, Precision level,
                const KernelContext& ctx = {});

// every element rounded to `level`, in place
void round_matrix(TileView tile, Precision level);

}  // namespace treechol
