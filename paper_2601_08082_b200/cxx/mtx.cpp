// mtx.cpp -- Matrix Market reader of the C++ drop-in API (reference
// mtx.hpp:17-20).  Off the factorization path: it exists
// so callers and the reference's acceptance gate link unchanged.  Errors are
// only the documented treechol types.
#include <cctype>
#include <cmath>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "treechol/errors.hpp"
#include "treechol/mtx.hpp"

namespace treechol {

namespace {

std::string lower(std::string s) {
    for (char& c : s) c = char(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

// next line that is not a comment and not blank; false at EOF
bool data_line(std::istream& in, std::string& line) {
    while (std::getline(in, line)) {
        size_t i = 0;
        while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
        if (i == line.size() || line[i] == '%') continue;
        return true;
    }
    return false;
}

long long parse_int(const std::string& tok, const char* what) {
    if (tok.empty()) throw ParseError(std::string("missing ") + what);
    size_t used = 0;
    long long v = 0;
    try {
        v = std::stoll(tok, &used);
    } catch (...) {
        throw ParseError(std::string("malformed ") + what + " '" + tok + "'");
    }
    if (used != tok.size()) throw ParseError(std::string("malformed ") + what + " '" + tok + "'");
    return v;
}

double parse_real(const std::string& tok, bool integer_field) {
    if (integer_field) return double(parse_int(tok, "integer entry"));
    size_t used = 0;
    double v = 0;
    try {
        v = std::stod(tok, &used);
    } catch (const std::out_of_range&) {
        throw ParseError("entry out of range '" + tok + "'");
    } catch (...) {
        throw ParseError("malformed entry '" + tok + "'");
    }
    if (used != tok.size()) throw ParseError("malformed entry '" + tok + "'");
    if (!std::isfinite(v)) throw ParseError("non-finite entry '" + tok + "'");
    return v;
}

std::vector<std::string> split(const std::string& line) {
    std::istringstream ss(line);
    std::vector<std::string> out;
    std::string t;
    while (ss >> t) out.push_back(t);
    return out;
}

}  // namespace

Matrix load_matrix_market(std::istream& in, int densify_limit) {
    std::string line;
    if (!std::getline(in, line)) throw ParseError("empty input");
    const std::vector<std::string> hdr = split(line);
    if (hdr.size() != 5 || lower(hdr[0]) != "%%matrixmarket" || lower(hdr[1]) != "matrix")
        throw ParseError("missing '%%MatrixMarket matrix <format> <field> <symmetry>' header");
    const std::string format = lower(hdr[2]), field = lower(hdr[3]), sym = lower(hdr[4]);
    if (format != "coordinate" && format != "array") throw ParseError("unknown format '" + hdr[2] + "'");
    if (field == "complex" || field == "pattern") throw UnsupportedFormat("field '" + field + "' is not supported");
    if (field != "real" && field != "integer" && field != "double") throw ParseError("unknown field '" + hdr[3] + "'");
    if (sym == "skew-symmetric" || sym == "hermitian")
        throw UnsupportedFormat("symmetry '" + sym + "' is not supported");
    if (sym != "general" && sym != "symmetric") throw ParseError("unknown symmetry '" + hdr[4] + "'");
    const bool integer_field = field == "integer";
    const bool symmetric = sym == "symmetric";

    if (!data_line(in, line)) throw ParseError("missing size line");
    const std::vector<std::string> sz = split(line);
    const bool coord = format == "coordinate";
    if (sz.size() != (coord ? 3u : 2u)) throw ParseError("malformed size line");
    const long long rows = parse_int(sz[0], "row count"), cols = parse_int(sz[1], "column count");
    if (rows < 1 || cols < 1) throw ParseError("matrix dimensions must be positive");
    if (rows != cols) throw UnsupportedFormat("matrix is not square");
    if (rows > densify_limit) throw TooLarge("order " + std::to_string(rows) + " exceeds the densify limit");
    const int n = int(rows);
    Matrix a(n, n);

    if (coord) {
        const long long nnz = parse_int(sz[2], "entry count");
        if (nnz < 0 || nnz > rows * cols) throw ParseError("invalid entry count");
        for (long long e = 0; e < nnz; ++e) {
            if (!data_line(in, line)) throw ParseError("fewer entries than declared");
            const std::vector<std::string> t = split(line);
            if (t.size() != 3) throw ParseError("malformed entry line");
            const long long i = parse_int(t[0], "row index"), j = parse_int(t[1], "column index");
            if (i < 1 || i > n || j < 1 || j > n) throw ParseError("index out of range");
            const double v = parse_real(t[2], integer_field);
            if (symmetric && j > i) throw ParseError("symmetric input lists an upper-triangle entry");
            a.at(int(i - 1), int(j - 1)) = v;
            if (symmetric) a.at(int(j - 1), int(i - 1)) = v;
        }
    } else {
        // column-major values; symmetric arrays list the lower triangle only
        for (int j = 0; j < n; ++j)
            for (int i = symmetric ? j : 0; i < n; ++i) {
                if (!data_line(in, line)) throw ParseError("fewer entries than declared");
                const std::vector<std::string> t = split(line);
                if (t.size() != 1) throw ParseError("malformed entry line");
                const double v = parse_real(t[0], integer_field);
                a.at(i, j) = v;
                if (symmetric) a.at(j, i) = v;
            }
    }
    if (data_line(in, line)) throw ParseError("more entries than declared");
    return a;
}

Matrix load_matrix_market(const std::string& path, int densify_limit) {
    std::ifstream f(path);
    if (!f) throw ParseError("cannot open '" + path + "'");
    return load_matrix_market(f, densify_limit);
}

}  // namespace treechol
