// report.cpp -- the reference's CSV / plan report formats (treechol/cli.hpp).
#include <cmath>
#include <cstdio>
#include <ostream>
#include <string>

#include "treechol/cli.hpp"
#include "treechol/flops.hpp"

namespace treechol {

namespace {

std::string g17(double v) {
    if (std::isnan(v)) return "nan";
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

}  // namespace

void write_csv(const std::vector<FactorReport>& reports, std::ostream& out) {
    out << "n,config,leaf,quantize,seed,status,rel_error,digits,flops_f16,flops_f32,flops_f64,flops_total,wall_ms\n";
    for (const FactorReport& r : reports) {
        out << r.n << ",\"" << r.config << "\"," << r.b << ',' << (r.quantize ? 1 : 0) << ',' << r.seed << ','
            << r.status << ',' << g17(r.rel_error) << ',' << g17(r.digits) << ',' << r.flops.by_level[0] << ','
            << r.flops.by_level[1] << ',' << r.flops.by_level[2] << ',' << r.flops.total() << ',' << g17(r.wall_ms)
            << '\n';
    }
}

void print_plan(int n, int b, const PrecisionConfig& cfg, const FlopBreakdown& fb, std::ostream& out) {
    const double t = double(fb.total());
    auto pct = [&](double f) { return t > 0 ? 100.0 * f / t : 0.0; };
    out << "n=" << n << " leaf=" << b << " config=" << cfg.to_string() << " total_flops=" << fb.total() << "\n\n";
    out << "per precision:\n";
    char line[96];
    for (Precision p : {Precision::Half, Precision::Single, Precision::Double}) {
        const auto f = fb.by_level[static_cast<int>(p)];
        std::snprintf(line, sizeof line, "  %-4s %20llu  %6.2f%%\n", precision_name(p), (unsigned long long)f,
                      pct(double(f)));
        out << line;
    }
    out << "per kernel:\n";
    for (Kernel k : {Kernel::Potrf, Kernel::Trsm, Kernel::Syrk, Kernel::Gemm}) {
        const auto f = fb.by_kernel[static_cast<int>(k)];
        std::snprintf(line, sizeof line, "  %-10s %14llu  %6.2f%%  (%llu calls)\n", kernel_name(k),
                      (unsigned long long)f, pct(double(f)), (unsigned long long)fb.calls[static_cast<int>(k)]);
        out << line;
    }
    const double off = double(fb.by_kernel[static_cast<int>(Kernel::Trsm)] +
                              fb.by_kernel[static_cast<int>(Kernel::Syrk)] +
                              fb.by_kernel[static_cast<int>(Kernel::Gemm)]);
    std::snprintf(line, sizeof line, "off-diagonal share (TRSM+SYRK+GEMM): %.2f%%\n", pct(off));
    out << line;
}

}  // namespace treechol
