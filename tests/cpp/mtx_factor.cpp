// Matrix Market -> device: the reference's public API path on a .mtx file.
// load_matrix_market (mtx.hpp) reads and densifies it, factor_matrix
// (analysis.hpp:48) copies it and factors the copy through build_tree /
// tree_potrf -- on this library, tc_potrf_host: H2D, the CUDA graph, D2H --
// then measures ||A - LL^T||_F / ||A||_F.  Prints one line per config:
//   <config>|<status>|<rel_error %.17g>|<flops total>
// Usage: mtx_factor <file.mtx> <b> <config>...
//        mtx_factor <file.mtx> --checksum   (host only: n, sum, sum of
//        squares and sum of (i+1)(j+2)a(i,j) of the dense matrix)
#include <cstdio>
#include <cstdlib>

#include "treechol/analysis.hpp"
#include "treechol/mtx.hpp"

using namespace treechol;

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s file.mtx b config...\n", argv[0]);
        return 2;
    }
    const Matrix a = load_matrix_market(std::string(argv[1]));
    if (std::string(argv[2]) == "--checksum") {
        double s = 0, s2 = 0, w = 0;
        for (int j = 0; j < a.cols(); ++j)
            for (int i = 0; i < a.rows(); ++i) {
                const double v = a.at(i, j);
                s += v;
                s2 += v * v;
                w += double(i + 1) * double(j + 2) * v;
            }
        std::printf("n=%d|%.17g|%.17g|%.17g\n", a.rows(), s, s2, w);
        return 0;
    }
    const int b = std::atoi(argv[2]);
    std::printf("n=%d\n", a.rows());
    for (int i = 3; i < argc; ++i) {
        const FactorReport r = factor_matrix(a, PrecisionConfig::parse(argv[i]), b, true);
        std::printf("%s|%s|%.17g|%llu\n", r.config.c_str(), r.status.c_str(), r.rel_error,
                    static_cast<unsigned long long>(r.flops.total()));
    }
    return 0;
}
