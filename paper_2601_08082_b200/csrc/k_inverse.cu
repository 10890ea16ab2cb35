// k_inverse.cu -- W = inv(L) of one diagonal leaf (n % 32 == 0, n <= 256),
// the operand of the inverse-based leaf solves: trsm_leaf (kernels.cpp:
// 71-92) of a tall panel B becomes the tensor-core GEMM X = rn_p(B W^T).
//
//   MODE 0 (F16 panels): W = inv(rn16(L)) in FP32, written as the FP16 pair
//          W 2^-e = hi + lo into W16 (row r0+i: hi at [0,n), lo at
//          [kW16Lo, kW16Lo+n)), 2^e to wscale[r0] (e from the largest
//          |1/L(j,j)| of the leaf, so every CTA of the leaf agrees);
//   MODE 1 (F32 panels): W = inv(L) in FP32 into W32 (row r0+i, ld 256),
//          consumed by the three-pass TF32 GEMM.
//
// CTA c computes column block c of W by block forward substitution:
//   W(I,c) = inv(L(I,I)) (delta_Ic - sum_{c<=K<I} L(I,K) W(K,c)),  I >= c
// -- the 32x32x32 products on all 16 warps, the 32x32 triangular solve on
// one warp (lane = column, right-looking, reciprocal + Newton correction).
// The first solve's singular-diagonal check (kernels.cpp:79-81) is reported
// here: the first j with L(j,j) zero or non-finite.
#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

constexpr int IT = 512;

__device__ __forceinline__ int isw(int r, int c) { return (c << 5) + (r ^ ((c & 7) << 2)); }

template <int MODE>
__global__ void __launch_bounds__(IT, 1) k_leaf_inv2(DevCtx c, int r0, int n, uint32_t seq) {
    using T = typename LvT<MODE == 0 ? 0 : 1>::T;
    extern __shared__ __align__(16) float ism[];
    const int NT = n >> 5, cb = blockIdx.x;
    const int NB = NT - cb;  // row blocks I = cb .. NT-1
    // tiles (I, K), cb <= K <= I, local index (I-cb)(I-cb+1)/2 + (K-cb)
    float* Ls = ism;
    float* Wb = Ls + ((NB * (NB + 1)) >> 1) * 1024;  // [NB][32][32] row-major W(I, cb)
    float* Rd = Wb + NB * 1024;                       // [NB*32] reciprocal diagonal
    const T* g = lvbuf<MODE == 0 ? 0 : 1>(c) + (long long)r0 * c.ldw + r0;
    const long long ld = c.ldw;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto tl = [&](int I, int K) { return Ls + ((((I - cb) * (I - cb + 1)) >> 1) + (K - cb)) * 1024; };

    // load the needed lower part (coalesced rows)
    const int ntile = (NB * (NB + 1)) >> 1;
    for (int k = warp; k < ntile; k += IT / 32) {
        int a = 0;
        while (((a + 1) * (a + 2)) / 2 <= k) ++a;
        const int I = cb + a, K = cb + (k - ((a * (a + 1)) >> 1));
        float v[32];
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) v[rr] = to_f(g[(long long)(I * 32 + rr) * ld + K * 32 + lane]);
        float* t = Ls + k * 1024;
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) t[isw(rr, lane)] = v[rr];
    }
    __syncthreads();
    for (int j = tid; j < NB * 32; j += IT) {
        const int I = cb + (j >> 5), r = j & 31;
        Rd[j] = 1.0f / tl(I, I)[isw(r, r)];
    }
    if (tid < 32) {  // singular diagonal in this column block
        const float d = tl(cb, cb)[isw(tid, tid)];
        const unsigned bad = __ballot_sync(0xffffffffu, d == 0.f || !isfinite(d));
        if (tid == 0 && bad) report(c, seq, uint64_t(cb * 32 + __ffs(bad) - 1));
    }
    __syncthreads();

    for (int I = cb; I < NT; ++I) {
        // rhs = delta - sum_K L(I,K) W(K,cb); thread: rows warp, warp+16; col lane
        float* Wi = Wb + (I - cb) * 1024;
        {
            float s0 = 0.f, s1 = 0.f;
            for (int K = cb; K < I; ++K) {
                const float* Lt = tl(I, K);
                const float* Wk = Wb + (K - cb) * 1024;
#pragma unroll 8
                for (int k = 0; k < 32; ++k) {
                    const float w = Wk[k * 32 + lane];
                    s0 = fmaf(Lt[isw(warp, k)], w, s0);
                    s1 = fmaf(Lt[isw(warp + 16, k)], w, s1);
                }
            }
            const float d0 = (I == cb && warp == lane) ? 1.f : 0.f;
            const float d1 = (I == cb && warp + 16 == lane) ? 1.f : 0.f;
            Wi[warp * 32 + lane] = d0 - s0;
            Wi[(warp + 16) * 32 + lane] = d1 - s1;
        }
        __syncthreads();
        if (warp == 0) {
            // W(I,cb)(:, lane) = inv(L(I,I)) rhs(:, lane), right-looking
            const float* Lt = tl(I, I);
            float w[32];
#pragma unroll
            for (int r = 0; r < 32; ++r) w[r] = Wi[r * 32 + lane];
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                const float d = Lt[isw(r, r)], rd = Rd[(I - cb) * 32 + r];
                const float q = w[r] * rd;
                w[r] = fmaf(fmaf(-q, d, w[r]), rd, q);
#pragma unroll
                for (int k = r + 1; k < 32; ++k) w[k] = fmaf(-Lt[isw(k, r)], w[r], w[k]);
            }
#pragma unroll
            for (int r = 0; r < 32; ++r) Wi[r * 32 + lane] = w[r];
        }
        __syncthreads();
    }

    // write column block cb of W (rows < 32 cb are zero)
    if constexpr (MODE == 0) {
        float dmax = 0.f;
        for (int j = lane; j < n; j += 32) dmax = fmaxf(dmax, fabsf(1.0f / __half2float(c.b16[(long long)(r0 + j) * ld + r0 + j])));
#pragma unroll
        for (int o = 16; o; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        int e = 0;
        if (dmax > 0.f && isfinite(dmax)) (void)frexpf(dmax, &e);
        const float up = ldexpf(1.0f, -e);
        if (cb == 0 && tid == 0) c.wscale[r0] = ldexpf(1.0f, e);
        __half* W = c.w16 + (long long)r0 * kW16Ld;
        for (int e2 = tid; e2 < n * 32; e2 += IT) {
            const int i = e2 >> 5, j = e2 & 31, t = cb * 32 + j;
            const float w = (i >= cb * 32) ? Wb[((i >> 5) - cb) * 1024 + (i & 31) * 32 + j] * up : 0.f;
            const float wz = i >= t ? w : 0.f;
            const __half hi = __float2half_rn(wz);
            const __half lo = __float2half_rn(wz - __half2float(hi));
            W[(long long)i * kW16Ld + t] = hi;
            W[(long long)i * kW16Ld + kW16Lo + t] = lo;
        }
    } else {
        float* W = c.w32 + (long long)r0 * kW32Ld;
        for (int e2 = tid; e2 < n * 32; e2 += IT) {
            const int i = e2 >> 5, j = e2 & 31, t = cb * 32 + j;
            const float w = (i >= cb * 32) ? Wb[((i >> 5) - cb) * 1024 + (i & 31) * 32 + j] : 0.f;
            W[(long long)i * kW32Ld + t] = i >= t ? w : 0.f;
        }
    }
}

size_t inv2_smem(int n) {
    const int NB = n / 32;
    return (size_t(NB * (NB + 1) / 2) * 1024 + size_t(NB) * 1024 + size_t(NB) * 32) * sizeof(float);
}

}  // namespace

bool inv2_ok(int n) { return n % 32 == 0 && n >= 32 && n <= 256; }

void init_inv2_attributes() {
    cudaFuncSetAttribute(k_leaf_inv2<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_leaf_inv2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}

void launch_leaf_inv2(const DevCtx& c, int mode, int r0, int n, uint32_t seq, cudaStream_t s) {
    if (mode == 0) k_leaf_inv2<0><<<n / 32, IT, inv2_smem(n), s>>>(c, r0, n, seq);
    else k_leaf_inv2<1><<<n / 32, IT, inv2_smem(n), s>>>(c, r0, n, seq);
}

}  // namespace tcb
