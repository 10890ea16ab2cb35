// analysis.cpp -- driver, generator and metric of the C++ drop-in API
// (reference analysis.hpp:15-55).  factor_matrix keeps the reference's
// status mapping (analysis.cpp:139-146); the factorization and the
// ||A - LL^T||_F / ||A||_F metric run on the device.
#include <chrono>
#include <cmath>

#include "abi.hpp"
#include "treechol/analysis.hpp"
#include "treechol/errors.hpp"
#include "treechol/tree.hpp"

namespace treechol {

Matrix spd_generate(int n, std::uint64_t seed) {
    Matrix a(n, n);
    if (n > 0) abi::check(tc_spd_generate_host(n, seed, a.data(), n));
    return a;
}

double factorization_error(const Matrix& a, const Matrix& lfac) {
    const int n = a.rows();
    if (n < 1) return std::nan("");
    double out = 0.0;
    abi::check(tc_factorization_error_host(n, a.data(), n, lfac.data(), lfac.rows(), &out));
    return out;
}

FlopBreakdown flop_breakdown(int n, int b, const PrecisionConfig& config) {
    std::vector<int> lv;
    for (Precision p : config.levels) lv.push_back(static_cast<int>(p));
    tc_flops f{};
    abi::check(tc_flop_breakdown(n, b, lv.data(), int(lv.size()), &f));
    FlopBreakdown fb;
    for (int i = 0; i < 3; ++i) fb.by_level[size_t(i)] = f.by_level[i];
    for (int i = 0; i < 4; ++i) {
        fb.by_kernel[size_t(i)] = f.by_kernel[i];
        fb.calls[size_t(i)] = f.calls[i];
    }
    return fb;
}

FactorReport factor_matrix(const Matrix& a, const PrecisionConfig& config, int b, bool quantize) {
    FactorReport rep;
    rep.n = a.rows();
    rep.config = config.to_string();
    rep.b = b;
    rep.quantize = quantize;
    Matrix work = a;  // the one permitted copy (analysis.cpp:130)
    const auto t0 = std::chrono::steady_clock::now();
    try {
        PrecisionTreeNode tree = build_tree(work.view(), config, b, quantize);
        SolveOptions opt;
        opt.leaf_size = b;
        opt.quantize = quantize;
        opt.flops = &rep.flops;
        tree_potrf(tree, opt);
        rep.status = "ok";
    } catch (const NotPositiveDefinite& e) {
        rep.status = "not-positive-definite";
        rep.detail = e.what();
    } catch (const NumericalBreakdown& e) {
        rep.status = "numerical-breakdown";
        rep.detail = e.what();
    }
    rep.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (rep.status == "ok") {
        rep.rel_error = factorization_error(a, work);
        rep.digits = -std::log10(rep.rel_error);
    }
    return rep;
}

std::vector<FactorReport> accuracy_sweep(const std::vector<int>& sizes, const std::vector<PrecisionConfig>& configs,
                                         int b, const std::vector<std::uint64_t>& seeds, bool quantize) {
    std::vector<FactorReport> out;
    out.reserve(sizes.size() * configs.size() * seeds.size());
    for (int n : sizes)
        for (const PrecisionConfig& cfg : configs)
            for (std::uint64_t s : seeds) {
                FactorReport r = factor_matrix(spd_generate(n, s), cfg, b, quantize);
                r.seed = s;
                out.push_back(std::move(r));
            }
    return out;
}

}  // namespace treechol
