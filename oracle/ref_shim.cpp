// ref_shim.cpp -- extern "C" face of the *compiled reference* (oracle/_ref).
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles the reference's own
// sources where they lie under /root/reference/proj/src (nothing is copied)
// together with this shim into oracle/_ref/libtreechol_ref.so.  Tests use it
// to pin the C restatement (oracle.c) bit for bit and to produce the golden
// fixtures in tests/golden/.  Signatures mirror oracle.h with a ref_ prefix.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "treechol/analysis.hpp"
#include "treechol/errors.hpp"
#include "treechol/kernels.hpp"
#include "treechol/tree.hpp"

using namespace treechol;

namespace {

PrecisionConfig make_cfg(const int* levels, int nlevels) {
    PrecisionConfig c;
    for (int i = 0; i < nlevels; ++i) c.levels.push_back(Precision(levels[i]));
    return c;
}

void copy_flops(const FlopBreakdown& fb, std::uint64_t* out) {
    if (!out) return;
    for (int i = 0; i < 3; ++i) out[i] = fb.by_level[i];
    for (int i = 0; i < 4; ++i) out[3 + i] = fb.by_kernel[i];
    for (int i = 0; i < 4; ++i) out[7 + i] = fb.calls[i];
}

void put(char* dst, int len, const std::string& s) {
    if (dst && len > 0) std::snprintf(dst, std::size_t(len), "%s", s.c_str());
}

}  // namespace

extern "C" {

double ref_round_to(double x, int p) { return round_to(x, Precision(p)); }

void ref_spd_generate(int n, std::uint64_t seed, double* a) {
    Matrix m = spd_generate(n, seed);
    std::memcpy(a, m.data(), sizeof(double) * std::size_t(n) * n);
}

double ref_factorization_error(int n, const double* a, const double* l) {
    Matrix ma(n, n), ml(n, n);
    std::memcpy(ma.data(), a, sizeof(double) * std::size_t(n) * n);
    std::memcpy(ml.data(), l, sizeof(double) * std::size_t(n) * n);
    return factorization_error(ma, ml);
}

void ref_flop_breakdown(int n, int b, const int* levels, int nlevels, std::uint64_t* out) {
    copy_flops(flop_breakdown(n, b, make_cfg(levels, nlevels)), out);
}

// build_tree + tree_potrf in place; status 0 ok, 1 NPD, 2 breakdown,
// 3 singular, 4 invalid argument (same numbering as oracle.h)
int ref_tree_potrf(int n, double* a, int lda, int b, const int* levels, int nlevels,
                   int quantize, std::uint64_t* flops, char* detail, int detail_len) {
    if (detail && detail_len > 0) detail[0] = '\0';
    FlopBreakdown fb;
    int st = 0;
    try {
        TileView v{a, n, n, lda, 0, 0};
        PrecisionTreeNode t = build_tree(v, make_cfg(levels, nlevels), b, quantize != 0);
        SolveOptions opt;
        opt.leaf_size = b;
        opt.quantize = quantize != 0;
        opt.flops = &fb;
        tree_potrf(t, opt);
    } catch (const NotPositiveDefinite& e) {
        st = 1;
        put(detail, detail_len, e.what());
    } catch (const NumericalBreakdown& e) {
        st = 2;
        put(detail, detail_len, e.what());
    } catch (const SingularDiagonal& e) {
        st = 3;
        put(detail, detail_len, e.what());
    } catch (const InvalidArgument& e) {
        st = 4;
        put(detail, detail_len, e.what());
    }
    copy_flops(fb, flops);
    return st;
}

int ref_factor_matrix(int n, const double* a, int b, const int* levels, int nlevels,
                      int quantize, double* l, double* rel_error, std::uint64_t* flops,
                      char* detail, int detail_len, double* wall_ms) {
    Matrix m(n, n);
    std::memcpy(m.data(), a, sizeof(double) * std::size_t(n) * n);
    FactorReport r = factor_matrix(m, make_cfg(levels, nlevels), b, quantize != 0);
    // factor_matrix keeps its factor internal; refactor for the caller's L
    if (l) {
        std::memcpy(l, a, sizeof(double) * std::size_t(n) * n);
        char scratch[8];
        ref_tree_potrf(n, l, n, b, levels, nlevels, quantize, nullptr, scratch, 0);
    }
    if (rel_error) *rel_error = r.rel_error;
    copy_flops(r.flops, flops);
    put(detail, detail_len, r.detail);
    if (wall_ms) *wall_ms = r.wall_ms;
    if (r.status == "ok") return 0;
    if (r.status == "not-positive-definite") return 1;
    return 2;
}

// factor only (no copy of L, no error eval): the timed CPU baseline unit
double ref_time_factor(int n, const double* a, int b, const int* levels, int nlevels,
                       int quantize) {
    Matrix m(n, n);
    std::memcpy(m.data(), a, sizeof(double) * std::size_t(n) * n);
    FactorReport r = factor_matrix(m, make_cfg(levels, nlevels), b, quantize != 0);
    return r.wall_ms;
}

void ref_gemm_mixed(double* c, int m, int n, int ldc, const double* a, int k, int lda,
                    const double* b, int ldb, double alpha, double beta, int level) {
    TileView vc{c, m, n, ldc, 0, 0};
    TileView va{const_cast<double*>(a), m, k, lda, 0, 0};
    TileView vb{const_cast<double*>(b), n, k, ldb, 0, 0};
    gemm_mixed(vc, va, vb, alpha, beta, Precision(level));
}

int ref_trsm_leaf(double* b, int m, int n, int ldb, const double* l, int ldl, int level) {
    TileView vb{b, m, n, ldb, 0, 0};
    TileView vl{const_cast<double*>(l), n, n, ldl, 0, 0};
    try {
        trsm_leaf(vb, vl, Precision(level));
    } catch (const SingularDiagonal& e) {
        return 3;
    }
    return 0;
}

int ref_potrf_leaf(double* a, int n, int ld, int level) {
    TileView v{a, n, n, ld, 0, 0};
    try {
        potrf_leaf(v, Precision(level));
    } catch (const NotPositiveDefinite&) {
        return 1;
    }
    return 0;
}

void ref_syrk_leaf(double* c, int n, int ldc, const double* a, int k, int lda, double alpha,
                   double beta, int level) {
    TileView vc{c, n, n, ldc, 0, 0};
    TileView va{const_cast<double*>(a), n, k, lda, 0, 0};
    syrk_leaf(vc, va, alpha, beta, Precision(level));
}

}  // extern "C"
