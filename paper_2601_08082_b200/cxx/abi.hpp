// abi.hpp -- C ABI status -> C++ exception mapping for the drop-in layer.
#pragma once

#include <string>

#include "treechol/errors.hpp"
#include "treechol_c.h"

namespace treechol::abi {

// throws the reference exception type of a failed tc_* call (argument,
// grammar and device errors; numerical failures carry indices and are
// mapped by the callers that know the view's origin)
inline void check(int status) {
    if (status == TC_OK) return;
    const std::string msg = tc_last_error();
    switch (status) {
        case TC_SYNTAX_ERROR: throw SyntaxError(msg);
        case TC_VALIDATION_ERROR: throw ValidationError(msg);
        case TC_INVALID_ARGUMENT: throw InvalidArgument(msg);
        case TC_NUMERICAL_BREAKDOWN: throw NumericalBreakdown(msg);
        case TC_NOT_POSITIVE_DEFINITE: throw NotPositiveDefinite(-1);
        case TC_SINGULAR_DIAGONAL: throw SingularDiagonal(-1);
        default: throw DeviceError(msg.empty() ? std::string("device error") : msg);
    }
}

}  // namespace treechol::abi
