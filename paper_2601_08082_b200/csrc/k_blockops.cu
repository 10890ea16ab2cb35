// k_blockops.cu -- standalone block operations on column-major doubles:
// the device side of the reference's kernel-level API (kernels.hpp:20-40,
// tree.hpp:47-51), used by the C++ drop-in layer for potrf_leaf / trsm_leaf /
// syrk_leaf / gemm_mixed / round_matrix / quantize_block / dequantize_block.
//
// These are NOT on the factorization path (tree_potrf keeps every block
// resident in the level buffers and uses k_leaf*/k_gemm_*).  They follow the
// reference's scalar contract operation by operation -- dot_update
// (kernels.cpp:23-38): level-rounded operands, products rounded to the level
// (exact at Half), a running sum rounded to the accumulator after every add,
// alpha/beta epilogue, final round -- in double with explicit _rn intrinsics
// (no FMA contraction), so their results are bit-identical to the reference.
// One thread owns one output element (or one row for TRSM), the k loop is
// sequential in t like the reference's.
#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

// round_to(x, level) of precision.hpp:70-76 (double in, double out)
__device__ __forceinline__ double rt(double x, int lv) {
    if (lv == 0) return double(__half2float(d2h(x)));
    if (lv == 1) return double(__double2float_rn(x));
    return x;
}

// dot_update (kernels.cpp:23-38), strided operands
__device__ double dot_update(int k, const double* a, long long sa, const double* b, long long sb, double alpha,
                             double beta, double c, int lv, int acc) {
    const bool half = lv == 0;
    double s = 0.0;
    for (int t = 0; t < k; ++t) {
        double p = __dmul_rn(rt(a[t * sa], lv), rt(b[t * sb], lv));
        if (!half) p = rt(p, lv);
        s = rt(__dadd_rn(s, p), acc);
    }
    double r = rt(__dmul_rn(alpha, s), acc);
    if (beta != 0.0) r = rt(__dadd_rn(r, rt(__dmul_rn(beta, rt(c, lv)), acc)), acc);
    return rt(r, lv);
}

__global__ void k_bo_round(double* a, long long lda, int m, int n, int lv, int lower) {
    const long long total = (long long)m * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = int(e % m), j = int(e / m);
        if (lower && i < j) continue;
        double* p = a + (long long)j * lda + i;
        *p = rt(*p, lv);
    }
}

// max |x| over the block, NaN skipped (std::max(amax, NaN) keeps amax,
// tree.cpp:82-86); non-negative doubles order like their bit patterns
__global__ void k_bo_absmax(const double* a, long long lda, int m, int n, unsigned long long* out) {
    const long long total = (long long)m * n;
    unsigned long long best = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const double v = fabs(a[(e / m) * lda + e % m]);
        if (!(v != v)) {
            const unsigned long long u = __double_as_longlong(v);
            best = u > best ? u : best;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x > best ? x : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

// quantize (mode 0): alpha = max|B|/range_max, !(alpha > 1) -> 1,
// B <- rn(B / alpha); dequantize (mode 1): B <- rn(B * alpha) unless alpha == 1
__global__ void k_bo_scale(double* a, long long lda, int m, int n, int lv, int mode, const unsigned long long* amax,
                           double alpha_in, double* alpha_out) {
    double alpha = alpha_in;
    if (mode == 0) {
        alpha = __ddiv_rn(__longlong_as_double(*amax), range_max(lv));
        if (!(alpha > 1.0)) alpha = 1.0;
        if (blockIdx.x == 0 && threadIdx.x == 0) *alpha_out = alpha;
    } else if (alpha == 1.0) {
        return;
    }
    const long long total = (long long)m * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        double* p = a + (e / m) * lda + e % m;
        *p = rt(mode == 0 ? __ddiv_rn(*p, alpha) : __dmul_rn(*p, alpha), lv);
    }
}

// C <- dot_update over k for every (i, j) (gemm_mixed) or j <= i (syrk_leaf)
__global__ void k_bo_gemm(double* c, long long ldc, const double* a, long long lda, const double* b, long long ldb,
                          int m, int n, int k, double alpha, double beta, int lv, int acc, int lower) {
    const long long total = (long long)m * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = int(e % m), j = int(e / m);
        if (lower && i < j) continue;
        double* cp = c + (long long)j * ldc + i;
        *cp = dot_update(k, a + i, lda, b + j, ldb, alpha, beta, *cp, lv, acc);
    }
}

// potrf_leaf (kernels.cpp:42-69): left-looking, one CTA, column by column;
// status = first failing pivot j (NotPositiveDefinite), else -1
__global__ void k_bo_potrf(double* a, long long lda, int n, int lv, int acc, int* status) {
    __shared__ double s_d;
    __shared__ int s_bad;
    for (int j = 0; j < n; ++j) {
        for (int i = j + threadIdx.x; i < n; i += blockDim.x) {
            double* p = a + (long long)j * lda + i;
            *p = dot_update(j, a + i, lda, a + j, lda, -1.0, 1.0, *p, lv, acc);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const double piv = a[(long long)j * lda + j];
            s_bad = !isfinite(piv) || piv <= 0.0;
            if (s_bad) *status = j;
            else {
                s_d = rt(__dsqrt_rn(piv), lv);
                a[(long long)j * lda + j] = s_d;
            }
        }
        __syncthreads();
        if (s_bad) return;
        const double d = s_d;
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
            double* p = a + (long long)j * lda + i;
            *p = rt(__ddiv_rn(*p, d), lv);
        }
        __syncthreads();
    }
}

// trsm_leaf (kernels.cpp:71-92): B <- B L^-T, one thread per row of B;
// status = first j whose rn(L(j,j)) is zero / non-finite (SingularDiagonal)
__global__ void k_bo_trsm(double* b, long long ldb, const double* l, long long ldl, int m, int n, int lv, int acc,
                          int* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    for (int j = 0; j < n; ++j) {
        const double ljj = rt(l[(long long)j * ldl + j], lv);
        if (ljj == 0.0 || !isfinite(ljj)) {
            if (i == 0) *status = j;
            return;
        }
        if (i < m) {
            double* p = b + (long long)j * ldb + i;
            const double r = dot_update(j, b + i, ldb, l + j, ldl, -1.0, 1.0, *p, lv, acc);
            *p = rt(__ddiv_rn(r, ljj), lv);
        }
    }
}

int grid_for(long long work, int threads) {
    long long g = (work + threads - 1) / threads;
    if (g > 148 * 16) g = 148 * 16;
    return int(g < 1 ? 1 : g);
}

}  // namespace

void bo_round(double* a, long long lda, int m, int n, int lv, int lower, cudaStream_t s) {
    k_bo_round<<<grid_for((long long)m * n, 256), 256, 0, s>>>(a, lda, m, n, lv, lower);
}

void bo_quantize(double* a, long long lda, int m, int n, int lv, unsigned long long* d_amax, double* d_alpha,
                 cudaStream_t s) {
    cudaMemsetAsync(d_amax, 0, sizeof(unsigned long long), s);
    k_bo_absmax<<<grid_for((long long)m * n, 256), 256, 0, s>>>(a, lda, m, n, d_amax);
    k_bo_scale<<<grid_for((long long)m * n, 256), 256, 0, s>>>(a, lda, m, n, lv, 0, d_amax, 1.0, d_alpha);
}

void bo_absmax(const double* a, long long lda, int m, int n, unsigned long long* d_amax, cudaStream_t s) {
    cudaMemsetAsync(d_amax, 0, sizeof(unsigned long long), s);
    k_bo_absmax<<<grid_for((long long)m * n, 256), 256, 0, s>>>(a, lda, m, n, d_amax);
}

void bo_dequantize(double* a, long long lda, int m, int n, int lv, double alpha, cudaStream_t s) {
    k_bo_scale<<<grid_for((long long)m * n, 256), 256, 0, s>>>(a, lda, m, n, lv, 1, nullptr, alpha, nullptr);
}

void bo_gemm(double* c, long long ldc, const double* a, long long lda, const double* b, long long ldb, int m, int n,
             int k, double alpha, double beta, int lv, int acc, int lower, cudaStream_t s) {
    k_bo_gemm<<<grid_for((long long)m * n, 128), 128, 0, s>>>(c, ldc, a, lda, b, ldb, m, n, k, alpha, beta, lv, acc,
                                                              lower);
}

void bo_potrf(double* a, long long lda, int n, int lv, int acc, int* d_status, cudaStream_t s) {
    cudaMemsetAsync(d_status, 0xFF, sizeof(int), s);
    k_bo_potrf<<<1, 512, 0, s>>>(a, lda, n, lv, acc, d_status);
}

void bo_trsm(double* b, long long ldb, const double* l, long long ldl, int m, int n, int lv, int acc, int* d_status,
             cudaStream_t s) {
    cudaMemsetAsync(d_status, 0xFF, sizeof(int), s);
    k_bo_trsm<<<grid_for(m, 128), 128, 0, s>>>(b, ldb, l, ldl, m, n, lv, acc, d_status);
}

}  // namespace tcb
