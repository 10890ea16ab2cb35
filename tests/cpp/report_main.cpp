// tests/cpp/report_main.cpp -- the C++ report writers (treechol/cli.hpp) on
// fixed inputs, compared with the Python mirror by tests/test_cpu.py.  Host
// only: flop_breakdown is the planner's static count.
#include <iostream>
#include <limits>
#include <vector>

#include "treechol/cli.hpp"

using namespace treechol;

int main() {
    FactorReport a;
    a.n = 1024;
    a.config = "[F16, F64]";
    a.b = 128;
    a.quantize = true;
    a.seed = 3;
    a.status = "ok";
    a.rel_error = 1.2345678901234567e-06;
    a.digits = 5.9084850188786495;
    a.flops = flop_breakdown(1024, 128, PrecisionConfig::parse("[F16, F64]"));
    a.wall_ms = 12.5;
    FactorReport b = a;
    b.status = "not-positive-definite";
    b.quantize = false;
    b.rel_error = std::numeric_limits<double>::quiet_NaN();
    b.digits = std::numeric_limits<double>::quiet_NaN();
    write_csv({a, b}, std::cout);
    std::cout << "--\n";
    print_plan(65536, 256, PrecisionConfig::parse("[F16, F16, F16, F32]"),
               flop_breakdown(65536, 256, PrecisionConfig::parse("[F16, F16, F16, F32]")), std::cout);
    return 0;
}
