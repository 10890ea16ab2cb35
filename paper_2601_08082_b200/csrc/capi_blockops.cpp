// capi_blockops.cpp -- C ABI of the standalone block operations
// (treechol_c.h "standalone block operations"; kernels in k_blockops.cu).
// Host variants stage the caller's column-major block through device memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "../../include/treechol_c.h"
#include "launch.hpp"

using namespace tcb;

namespace tcb {
void set_last_error(const std::string& msg);  // capi.cpp
}

namespace {

int bo_fail(int code, const std::string& msg) {
    set_last_error(msg);
    return code;
}

// device staging of one column-major block (ld = rows on the device)
struct Stage {
    double* d = nullptr;
    ~Stage() {
        if (d) cudaFree(d);
    }
};

bool lv_ok(int lv) { return lv >= 0 && lv <= 2; }

cudaError_t h2d(double* d, const double* h, int lda, int m, int n) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    return cudaMemcpy2D(d, sizeof(double) * size_t(m), h, sizeof(double) * size_t(lda), sizeof(double) * size_t(m),
                        size_t(n), cudaMemcpyHostToDevice);
}
cudaError_t d2h(double* h, int lda, const double* d, int m, int n) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    return cudaMemcpy2D(h, sizeof(double) * size_t(lda), d, sizeof(double) * size_t(m), sizeof(double) * size_t(m),
                        size_t(n), cudaMemcpyDeviceToHost);
}
// lower trapezoid of an m x n block back to the host (strict upper untouched)
cudaError_t d2h_lower(double* h, int lda, const double* d, int m, int n) {
    for (int j0 = 0; j0 < n; j0 += 64) {
        const int w = std::min(64, n - j0);
        if (j0 >= m) break;
        const cudaError_t e =
            cudaMemcpy2D(h + size_t(j0) * lda + j0, sizeof(double) * size_t(lda), d + size_t(j0) * m + j0,
                         sizeof(double) * size_t(m), sizeof(double) * size_t(m - j0), size_t(w),
                         cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int no_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
        cudaGetLastError();
        return 1;
    }
    return 0;
}

#define BO_CUDA(expr)                                                                       \
    do {                                                                                    \
        const cudaError_t e_ = (expr);                                                      \
        if (e_ != cudaSuccess) return bo_fail(TC_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

}  // namespace

extern "C" {

int tc_round_host(int m, int n, double* A, int lda, int level, int lower) {
    if (!A || m < 0 || n < 0 || lda < m || !lv_ok(level)) return bo_fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (level == TC_F64 || m == 0 || n == 0) return TC_OK;
    if (no_device()) return bo_fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    Stage s;
    BO_CUDA(cudaMalloc(&s.d, sizeof(double) * size_t(m) * size_t(n)));
    BO_CUDA(h2d(s.d, A, lda, m, n));
    bo_round(s.d, m, m, n, level, lower, nullptr);
    BO_CUDA(cudaGetLastError());
    BO_CUDA(lower ? d2h_lower(A, lda, s.d, m, n) : d2h(A, lda, s.d, m, n));
    return TC_OK;
}

int tc_quantize_host(int m, int n, double* B, int ldb, int level, double* alpha) {
    if (!B || !alpha || m < 0 || n < 0 || ldb < m || !lv_ok(level))
        return bo_fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (no_device()) return bo_fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    Stage s;
    BO_CUDA(cudaMalloc(&s.d, sizeof(double) * (size_t(m) * size_t(n) + 2)));
    double* d_alpha = s.d + size_t(m) * size_t(n);
    auto* d_amax = reinterpret_cast<unsigned long long*>(d_alpha + 1);
    BO_CUDA(h2d(s.d, B, ldb, m, n));
    bo_quantize(s.d, m, m, n, level, d_amax, d_alpha, nullptr);
    BO_CUDA(cudaGetLastError());
    BO_CUDA(cudaMemcpy(alpha, d_alpha, sizeof(double), cudaMemcpyDeviceToHost));
    BO_CUDA(d2h(B, ldb, s.d, m, n));
    return TC_OK;
}

int tc_dequantize_host(int m, int n, double* B, int ldb, int level, double alpha) {
    if (!B || m < 0 || n < 0 || ldb < m || !lv_ok(level)) return bo_fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (alpha == 1.0 || m == 0 || n == 0) return TC_OK;  // tree.cpp:98
    if (no_device()) return bo_fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    Stage s;
    BO_CUDA(cudaMalloc(&s.d, sizeof(double) * size_t(m) * size_t(n)));
    BO_CUDA(h2d(s.d, B, ldb, m, n));
    bo_dequantize(s.d, m, m, n, level, alpha, nullptr);
    BO_CUDA(cudaGetLastError());
    BO_CUDA(d2h(B, ldb, s.d, m, n));
    return TC_OK;
}

int tc_potrf_leaf_host(int n, double* A, int lda, int level, int acc, int* fail_index) {
    if (!A || n < 0 || lda < n || !lv_ok(level) || !lv_ok(acc)) return bo_fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (fail_index) *fail_index = -1;
    if (n == 0) return TC_OK;
    if (no_device()) return bo_fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    Stage s;
    BO_CUDA(cudaMalloc(&s.d, sizeof(double) * (size_t(n) * size_t(n) + 1)));
    int* d_status = reinterpret_cast<int*>(s.d + size_t(n) * size_t(n));
    BO_CUDA(h2d(s.d, A, lda, n, n));
    bo_potrf(s.d, n, n, level, level == TC_F16 ? acc : level, d_status, nullptr);
    BO_CUDA(cudaGetLastError());
    int st = -1;
    BO_CUDA(cudaMemcpy(&st, d_status, sizeof(int), cudaMemcpyDeviceToHost));
    BO_CUDA(d2h_lower(A, lda, s.d, n, n));
    if (st >= 0) {
        if (fail_index) *fail_index = st;
        return bo_fail(TC_NOT_POSITIVE_DEFINITE, "pivot " + std::to_string(st) + " is non-positive or non-finite");
    }
    return TC_OK;
}

int tc_trsm_leaf_host(int m, int n, double* B, int ldb, const double* L, int ldl, int level, int acc,
                      int* fail_index) {
    if (!B || !L || m < 0 || n < 0 || ldb < m || ldl < n || !lv_ok(level) || !lv_ok(acc))
        return bo_fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (fail_index) *fail_index = -1;
    if (n == 0) return TC_OK;
    if (no_device()) return bo_fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    Stage s;
    const size_t nb = size_t(m) * size_t(n), nl = size_t(n) * size_t(n);
    BO_CUDA(cudaMalloc(&s.d, sizeof(double) * (nb + nl + 1)));
    double* dL = s.d + nb;
    int* d_status = reinterpret_cast<int*>(dL + nl);
    BO_CUDA(h2d(s.d, B, ldb, m, n));
    BO_CUDA(h2d(dL, L, ldl, n, n));
    bo_trsm(s.d, m, dL, n, m, n, level, level == TC_F16 ? acc : level, d_status, nullptr);
    BO_CUDA(cudaGetLastError());
    int st = -1;
    BO_CUDA(cudaMemcpy(&st, d_status, sizeof(int), cudaMemcpyDeviceToHost));
    BO_CUDA(d2h(B, ldb, s.d, m, n));
    if (st >= 0) {
        if (fail_index) *fail_index = st;
        return bo_fail(TC_SINGULAR_DIAGONAL, "diagonal entry " + std::to_string(st) + " is zero or non-finite");
    }
    return TC_OK;
}

int tc_gemm_mixed_device(int m, int n, int k, double* dC, int ldc, const double* dA, int lda, const double* dB,
                         int ldb, double alpha, double beta, int level, int acc, int lower, void* stream) {
    if (!dC || (k > 0 && (!dA || !dB)) || m < 0 || n < 0 || k < 0 || ldc < m || !lv_ok(level) || !lv_ok(acc))
        return bo_fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (m == 0 || n == 0) return TC_OK;
    bo_gemm(dC, ldc, dA, lda, dB, ldb, m, n, k, alpha, beta, level, level == TC_F16 ? acc : level, lower,
            static_cast<cudaStream_t>(stream));
    BO_CUDA(cudaGetLastError());
    return TC_OK;
}

int tc_gemm_mixed_host(int m, int n, int k, double* C, int ldc, const double* A, int lda, const double* B, int ldb,
                       double alpha, double beta, int level, int acc, int lower) {
    if (!C || (k > 0 && (!A || !B)) || m < 0 || n < 0 || k < 0 || ldc < m || (k > 0 && (lda < m || ldb < n)) ||
        !lv_ok(level) || !lv_ok(acc))
        return bo_fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (m == 0 || n == 0) return TC_OK;
    if (no_device()) return bo_fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    const bool same = A == B && lda == ldb && m == n;
    Stage s;
    const size_t nc = size_t(m) * n, na = size_t(m) * k, nb = same ? 0 : size_t(n) * k;
    BO_CUDA(cudaMalloc(&s.d, sizeof(double) * (nc + na + nb + 1)));
    double* dA = s.d + nc;
    double* dB = same ? dA : dA + na;
    // beta == 0: C is not read (kernels.cpp:34); stage it anyway for the
    // lower-triangle SYRK whose strict upper part must come back unchanged
    BO_CUDA(h2d(s.d, C, ldc, m, n));
    BO_CUDA(h2d(dA, A, lda, m, k));
    if (!same) BO_CUDA(h2d(dB, B, ldb, n, k));
    bo_gemm(s.d, m, dA, m, dB, same ? m : n, m, n, k, alpha, beta, level, level == TC_F16 ? acc : level, lower,
            nullptr);
    BO_CUDA(cudaGetLastError());
    BO_CUDA(lower ? d2h_lower(C, ldc, s.d, m, n) : d2h(C, ldc, s.d, m, n));
    return TC_OK;
}

}  // extern "C"
