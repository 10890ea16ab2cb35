// core.cpp -- precision / matrix / flops / kernels layer of the C++ drop-in
// API (include/treechol/*.hpp) over the C ABI of libtreechol_b200.so.
// Every numeric call goes to the device; this file only marshals arguments
// and turns tc_status codes into the reference's exception types.
#include <cstring>
#include <string>

#include "abi.hpp"
#include "treechol/errors.hpp"
#include "treechol/flops.hpp"
#include "treechol/kernels.hpp"
#include "treechol/matrix.hpp"
#include "treechol/precision.hpp"

namespace treechol {

// ---------------------------------------------------------------- precision

const char* precision_name(Precision p) {
    static const char* names[3] = {"F16", "F32", "F64"};
    const int i = static_cast<int>(p);
    return names[i >= 0 && i < 3 ? i : 2];
}

double round_to_half(double x) {
    // GCC's double -> _Float16 conversion is a single correctly rounded
    // (RNE) step with IEEE overflow / gradual underflow -- the contract of
    // the reference's round_to_half; widening back is exact
    return static_cast<double>(static_cast<_Float16>(x));
}

std::string PrecisionConfig::to_string() const {
    int lv[16];
    const int n = int(levels.size());
    if (n < 1 || n > 16) throw InvalidArgument("empty precision config");
    for (int i = 0; i < n; ++i) lv[i] = static_cast<int>(levels[i]);
    char buf[160];
    abi::check(tc_config_to_string(lv, n, buf, int(sizeof buf)));
    return buf;
}

PrecisionConfig PrecisionConfig::parse(const std::string& text) {
    int lv[16];
    int n = 0;
    abi::check(tc_config_parse(text.c_str(), lv, &n));
    PrecisionConfig c;
    for (int i = 0; i < n; ++i) c.levels.push_back(static_cast<Precision>(lv[i]));
    return c;
}

// ---------------------------------------------------------------- matrix

std::atomic<long> Matrix::created_{0};

Matrix::Matrix(int rows, int cols) : rows_(rows), cols_(cols), buf_(std::size_t(rows) * std::size_t(cols)) {
    created_.fetch_add(1, std::memory_order_relaxed);
}

Matrix::Matrix(const Matrix& other) : rows_(other.rows_), cols_(other.cols_), buf_(other.buf_) {
    created_.fetch_add(1, std::memory_order_relaxed);
}

long Matrix::allocations() { return created_.load(std::memory_order_relaxed); }

// ---------------------------------------------------------------- flops

const char* kernel_name(Kernel k) {
    switch (k) {
        case Kernel::Potrf: return "POTRF-leaf";
        case Kernel::Trsm: return "TRSM-leaf";
        case Kernel::Syrk: return "SYRK-leaf";
        case Kernel::Gemm: return "GEMM";
    }
    return "?";
}

// ---------------------------------------------------------------- kernels
// flop formulas of kernels.cpp:56-66, 89, 107-110, 127-130

namespace {
int acc_of(Precision level, const KernelContext& ctx) {
    return static_cast<int>(level == Precision::Half ? ctx.half_accumulator : level);
}
}  // namespace

void round_matrix(TileView tile, Precision level) {
    abi::check(tc_round_host(tile.rows, tile.cols, tile.data, tile.ld, static_cast<int>(level), 0));
}

void potrf_leaf(TileView a, Precision level, const KernelContext& ctx) {
    int bad = -1;
    const int st = tc_potrf_leaf_host(a.rows, a.data, a.ld, static_cast<int>(level), acc_of(level, ctx), &bad);
    if (st == TC_NOT_POSITIVE_DEFINITE) throw NotPositiveDefinite(a.row0 + bad);
    abi::check(st);
    if (ctx.flops) {
        const std::uint64_t n = std::uint64_t(a.rows);
        // sum_j 2 j (n - j) + 1 + (n - j - 1) = n(n+1)(2n+1)/6 - n(n+1)/2 ... as
        // accumulated column by column in the reference
        std::uint64_t fl = 0;
        for (std::uint64_t j = 0; j < n; ++j) fl += 2 * j * (n - j) + 1 + (n - j - 1);
        ctx.flops->add(level, Kernel::Potrf, fl);
    }
}

void trsm_leaf(TileView b, TileView l, Precision level, const KernelContext& ctx) {
    int bad = -1;
    const int st =
        tc_trsm_leaf_host(b.rows, b.cols, b.data, b.ld, l.data, l.ld, static_cast<int>(level), acc_of(level, ctx), &bad);
    if (st == TC_SINGULAR_DIAGONAL) throw SingularDiagonal(l.row0 + bad);
    abi::check(st);
    if (ctx.flops) ctx.flops->add(level, Kernel::Trsm, std::uint64_t(b.rows) * b.cols * b.cols);
}

void syrk_leaf(TileView c, TileView a, double alpha, double beta, Precision level, const KernelContext& ctx) {
    abi::check(tc_gemm_mixed_host(c.rows, c.rows, a.cols, c.data, c.ld, a.data, a.ld, a.data, a.ld, alpha, beta,
                                  static_cast<int>(level), acc_of(level, ctx), 1));
    if (ctx.flops)
        ctx.flops->add(level, Kernel::Syrk, std::uint64_t(c.rows) * std::uint64_t(c.rows + 1) * std::uint64_t(a.cols));
}

void gemm_mixed(TileView c, TileView a, TileView b, double alpha, double beta, Precision level,
                const KernelContext& ctx) {
    abi::check(tc_gemm_mixed_host(c.rows, c.cols, a.cols, c.data, c.ld, a.data, a.ld, b.data, b.ld, alpha, beta,
                                  static_cast<int>(level), acc_of(level, ctx), 0));
    if (ctx.flops)
        ctx.flops->add(level, Kernel::Gemm, 2ull * std::uint64_t(c.rows) * std::uint64_t(c.cols) * std::uint64_t(a.cols));
}

}  // namespace treechol
