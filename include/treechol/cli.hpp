#pragma once
// treechol/cli.hpp -- result reporting of the reference's command-line front
// end (proj/include/treechol/cli.hpp), kept so results stay diffable with the
// reference's schema.  The CLI itself (run_cli, built on CLI11) is out of
// scope; the report writers are here.

#include <iosfwd>
#include <vector>

#include "treechol/analysis.hpp"

namespace treechol {

// Fixed-schema CSV emission, header row included, LF endings (reference
// cli.cpp:123-127 with the row format of cli.cpp:26-33): doubles as %.17g,
// NaN as "nan", the config quoted.
void write_csv(const std::vector<FactorReport>& reports, std::ostream& out);

// The `plan` subcommand's flop report (reference cli.cpp:52-86): totals per
// precision and per kernel with shares and call counts, and the off-diagonal
// (TRSM + SYRK + GEMM) share.
void print_plan(int n, int b, const PrecisionConfig& cfg, const FlopBreakdown& fb, std::ostream& out);

}  // namespace treechol
