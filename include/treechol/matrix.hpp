// treechol/matrix.hpp -- the host-side storage boundary of the B200 library.
//
// Drop-in for /root/reference/proj/include/treechol/matrix.hpp:11-62.  A
// TileView is a non-owning column-major window (element (i,j) at
// data[j*ld + i]); the factorization reads the window's lower triangle,
// runs on the device and writes L back in place.  Matrix owns a host buffer
// and counts how many numeric buffers were ever created, so callers can
// check the solver allocates none (the device workspace is not a Matrix).
#pragma once

#include <atomic>
#include <cstddef>
#include <vector>

namespace treechol {

struct TileView {
    double* data = nullptr;
    int rows = 0;
    int cols = 0;
    int ld = 0;    // column stride
    int row0 = 0;  // origin inside the full matrix (diagnostics, error indices)
    int col0 = 0;

    double& at(int i, int j) const { return *(data + (std::size_t(j) * std::size_t(ld) + std::size_t(i))); }

    // the m x n window starting at local (r, c)
    TileView sub(int r, int c, int m, int n) const {
        TileView v;
        v.data = data + (std::size_t(c) * std::size_t(ld) + std::size_t(r));
        v.rows = m;
        v.cols = n;
        v.ld = ld;
        v.row0 = row0 + r;
        v.col0 = col0 + c;
        return v;
    }
};

class Matrix {
   public:
    Matrix(int rows, int cols);
    Matrix(const Matrix& other);
    Matrix(Matrix&&) noexcept = default;
    Matrix& operator=(const Matrix&) = default;
    Matrix& operator=(Matrix&&) noexcept = default;

    int rows() const { return rows_; }
    int cols() const { return cols_; }
    double& at(int i, int j) { return buf_[std::size_t(j) * std::size_t(rows_) + std::size_t(i)]; }
    double at(int i, int j) const { return buf_[std::size_t(j) * std::size_t(rows_) + std::size_t(i)]; }
    double* data() { return buf_.data(); }
    const double* data() const { return buf_.data(); }

    // full-matrix window (ld = rows)
    TileView view() {
        TileView v;
        v.data = buf_.data();
        v.rows = rows_;
        v.cols = cols_;
        v.ld = rows_;
        return v;
    }

    // numeric buffers created since process start
    static long allocations();

   private:
    int rows_;
    int cols_;
    std::vector<double> buf_;
    static std::atomic<long> created_;
};

}  // namespace treechol
