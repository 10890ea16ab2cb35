// Host-only checks of the C++ drop-in API (include/treechol/*.hpp) that need
// no device: config grammar, the rounding contract, flop accounting, the
// Matrix Market reader and the exception mapping.  Known answers follow the
// reference's unit tests (test_precision.cpp:75-94, test_analysis.cpp:158-171,
// test_tree.cpp:58-85 shapes are covered by the python planner tests).
#include <cmath>
#include <cstdio>
#include <sstream>
#include <string>

#include "treechol/analysis.hpp"
#include "treechol/errors.hpp"
#include "treechol/mtx.hpp"
#include "treechol/precision.hpp"
#include "treechol/tree.hpp"

using namespace treechol;

static int fails = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                               \
        }                                                          \
    } while (0)

template <typename E, typename F>
static bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // grammar (precision.cpp:52-111)
    CHECK(PrecisionConfig::parse("[F16, F32]").to_string() == "[F16, F32]");
    CHECK(PrecisionConfig::parse(" pure fp64 ").to_string() == "Pure F64");
    CHECK(PrecisionConfig::parse("[fp16,F16 , f16,F32]").levels.size() == 4);
    CHECK(throws<SyntaxError>([] { PrecisionConfig::parse("[F16, F8]"); }));
    CHECK(throws<SyntaxError>([] { PrecisionConfig::parse("[]"); }));
    CHECK(throws<ValidationError>([] { PrecisionConfig::parse("[F32, F16]"); }));
    const auto c = PrecisionConfig::parse("[F16, F32]");
    CHECK(c.at_depth(0) == Precision::Half && c.at_depth(7) == Precision::Single && c.leaf() == Precision::Single);

    // rounding contract (test_precision.cpp:75-94)
    CHECK(round_to_half(65519.0) == 65504.0);
    CHECK(std::isinf(round_to_half(65520.0)) && round_to_half(-65520.0) < 0);
    CHECK(round_to_half(0x1p-25) == 0.0);
    CHECK(round_to_half(0x1.0000001p-25) == 0x1p-24);
    CHECK(std::signbit(round_to_half(-0x1p-1074)) && round_to_half(-0x1p-1074) == 0.0);
    CHECK(round_to_half(1.0 + 0x1p-11) == 1.0);            // tie to even
    CHECK(round_to_half(1.0 + 3 * 0x1p-11) == 1.0 + 0x1p-9);  // tie to even (up)
    CHECK(std::isnan(round_to_half(std::nan(""))));
    CHECK(round_to(1.0 + 0x1p-30, Precision::Single) == 1.0);
    CHECK(round_to(1.0 + 0x1p-30, Precision::Double) == 1.0 + 0x1p-30);
    CHECK(std::string(precision_name(Precision::Single)) == "F32");
    CHECK(range_max(Precision::Half) == 65504.0 && unit_roundoff(Precision::Double) == 0x1p-53);

    // flop accounting (test_analysis.cpp:119-128, 158-171)
    const auto fb = flop_breakdown(4, 2, PrecisionConfig::parse("Pure F64"));
    CHECK(fb.total() == 30);
    CHECK(fb.by_kernel[0] == 10 && fb.by_kernel[1] == 8 && fb.by_kernel[2] == 12);
    for (int n = 1; n <= 40; ++n)
        for (int b = 1; b <= n; b += 3) {
            const auto f = flop_breakdown(n, b, PrecisionConfig::parse("[F16, F32, F64]"));
            CHECK(f.total() == std::uint64_t(n) * (n + 1) * (2 * n + 1) / 6);
        }
    CHECK(std::string(kernel_name(Kernel::Gemm)) == "GEMM");

    // Matrix Market reader
    {
        std::istringstream in("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 4\n1 1 4\n2 1 1\n2 2 5\n3 3 6\n");
        Matrix m = load_matrix_market(in);
        CHECK(m.rows() == 3 && m.at(0, 1) == 1.0 && m.at(1, 0) == 1.0 && m.at(2, 2) == 6.0 && m.at(2, 0) == 0.0);
        std::istringstream arr("%%MatrixMarket matrix array integer general\n2 2\n1\n2\n3\n4\n");
        Matrix g = load_matrix_market(arr);
        CHECK(g.at(1, 0) == 2.0 && g.at(0, 1) == 3.0);
        std::istringstream cx("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n");
        CHECK(throws<UnsupportedFormat>([&] { load_matrix_market(cx); }));
        std::istringstream big("%%MatrixMarket matrix coordinate real general\n100 100 0\n");
        CHECK(throws<TooLarge>([&] { load_matrix_market(big, 64); }));
        std::istringstream bad("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n");
        CHECK(throws<ParseError>([&] { load_matrix_market(bad); }));
    }

    // argument errors of build_tree (tree.cpp:72-76) need no device
    {
        Matrix a(4, 4);
        CHECK(throws<InvalidArgument>([&] { build_tree(a.view(), PrecisionConfig::parse("Pure F64"), 0); }));
        Matrix r(3, 4);
        CHECK(throws<InvalidArgument>([&] { build_tree(r.view(), PrecisionConfig::parse("Pure F64"), 2); }));
    }
    // Matrix allocation counter (matrix.hpp:53-55)
    {
        const long a0 = Matrix::allocations();
        Matrix x(2, 2);
        Matrix y = x;
        CHECK(Matrix::allocations() == a0 + 2);
    }
    std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
    return fails ? 1 : 0;
}
