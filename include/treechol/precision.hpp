// treechol/precision.hpp -- precision tags, rounding contract and the
// precision-tree configuration of the B200 library.
//
// Drop-in for /root/reference/proj/include/treechol/precision.hpp: same
// names and semantics (precision.hpp:14-99 there).  The host-side rounding
// helpers are provided for callers and tests; the factorization itself
// rounds on the device (cvt.rn.f16.f64 / cvt.rn.f32.f64 in the kernels).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace treechol {

// storage formats, ordered by precision (values = the C ABI's TC_F16..F64)
enum class Precision : int { Half = 0, Single = 1, Double = 2 };

inline constexpr double kHalfMax = 65504.0;
inline constexpr double kSingleMax = 3.4028234663852886e38;
inline constexpr double kDoubleMax = 1.7976931348623157e308;

// largest finite value of a format (reference precision.hpp:20-26)
inline double range_max(Precision p) {
    return p == Precision::Half ? kHalfMax : p == Precision::Single ? kSingleMax : kDoubleMax;
}

// unit roundoff 2^-(t) of a format (reference precision.hpp:28-34)
inline double unit_roundoff(Precision p) {
    return p == Precision::Half ? 0x1p-11 : p == Precision::Single ? 0x1p-24 : 0x1p-53;
}

// "F16" / "F32" / "F64"
const char* precision_name(Precision p);

// binary16 round-to-nearest-even of a double, widened back: one rounding
// straight from double (no binary32 hop), |x| >= 65520 -> +-inf, binary16
// subnormals kept, double subnormals -> signed zero, inf/NaN unchanged.
// Implemented out of line with the compiler's correctly rounded
// double -> _Float16 conversion (reference precision.hpp:41-62).
double round_to_half(double x);

inline double round_to_single(double x) { return double(static_cast<float>(x)); }

inline double round_to(double x, Precision p) {
    if (p == Precision::Half) return round_to_half(x);
    if (p == Precision::Single) return round_to_single(x);
    return x;
}

// Outer -> inner level list; depth d uses levels[min(d, size-1)], leaves
// use the last entry (reference precision.hpp:81-99).
struct PrecisionConfig {
    std::vector<Precision> levels;

    Precision at_depth(std::size_t d) const { return levels[std::min(d, levels.size() - 1)]; }
    Precision leaf() const { return levels.back(); }
    bool operator==(const PrecisionConfig&) const = default;

    // "Pure F32" for one level, "[F16, F32]" otherwise
    std::string to_string() const;
    // grammar of precision.cpp:52-111: "[F16, F32]", "Pure FP32", any case
    // and spacing; SyntaxError when malformed, ValidationError when the
    // precision decreases outer -> inner
    static PrecisionConfig parse(const std::string& text);
};

}  // namespace treechol
