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
// -- both products on the warp-level tensor path (mma.sync TF32, three-pass
// hi/lo split: FP32-accurate); the 32x32 diagonal inverses up front, one
// warp each (lane = column, right-looking substitution).
// The first solve's singular-diagonal check (kernels.cpp:79-81) is reported
// here: the first j with L(j,j) zero or non-finite.
#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

constexpr int IT = 512;

// development counters (CTA 0 of every launch): cycles in load, reciprocals,
// diagonal inverses, products, triangular multiplies, store; launches
__device__ unsigned long long g_inv_clk[8];
constexpr int WLD = 36, WBS = 32 * WLD;  // W / inverse / partial blocks: row-major, padded rows

__device__ __forceinline__ void mma_tf32_i(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// x = hi + lo, hi = x truncated to TF32 (exact), lo = x - hi (exact)
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(x) & 0xFFFFE000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ int isw(int r, int c) { return (c << 5) + (r ^ ((c & 7) << 2)); }

template <int MODE>
__global__ void __launch_bounds__(IT, 1) k_leaf_inv2(DevCtx c, int r0, int n, uint32_t seq) {
    pdl_wait();
    using T = typename LvT<MODE == 0 ? 0 : 1>::T;
    extern __shared__ __align__(16) float ism[];
    const int NT = n >> 5, cb = blockIdx.x;
    const int NB = NT - cb;  // row blocks I = cb .. NT-1
    // tiles (I, K), cb <= K <= I, local index (I-cb)(I-cb+1)/2 + (K-cb)
    float* Ls = ism;
    float* Wb = Ls + ((NB * (NB + 1)) >> 1) * 1024;  // [NB][32][WLD] row-major W(I, cb)
    float* Pq = Wb + NB * WBS;                        // [4][32][WLD] K-split partials of the product
    float* Rd = Pq + 4 * WBS;                         // [NB*32] reciprocal diagonal
    const T* g = lvbuf<MODE == 0 ? 0 : 1>(c) + (long long)r0 * c.ldw + r0;
    const long long ld = c.ldw;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto tl = [&](int I, int K) { return Ls + ((((I - cb) * (I - cb + 1)) >> 1) + (K - cb)) * 1024; };

    long long ck0 = clock64(), ck_prod = 0, ck_tri = 0, ck1, ck2, ck3;
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
    ck1 = clock64();
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
    ck2 = clock64();

    // inv(L(I,I)) of every diagonal block, one warp each, in place (the
    // diagonal tiles are read only as these inverses afterwards): lane =
    // column, right-looking forward substitution, reciprocal + Newton step
    if (warp < NB) {
        const int I = cb + warp;
        float* Lt = tl(I, I);
        float x[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) x[r] = r == lane ? 1.f : 0.f;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            const float d = Lt[isw(r, r)], rd = Rd[(I - cb) * 32 + r];
            const float q = x[r] * rd;
            x[r] = fmaf(fmaf(-q, d, x[r]), rd, q);
#pragma unroll
            for (int k = r + 1; k < 32; ++k) x[k] = fmaf(-Lt[isw(k, r)], x[r], x[k]);
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) Lt[isw(r, lane)] = x[r];
    }
    __syncthreads();
    ck3 = clock64();

    const int gq = lane >> 2, tq = lane & 3;
    for (int I = cb; I < NT; ++I) {
        const long long ca = clock64();
        float* Wi = Wb + (I - cb) * WBS;
        const float* Dc = tl(I, I);  // inv(L(I,I)), tile layout
        // (1) P = sum_{cb <= K < I} L(I,K) W(K,cb) on the tensor cores: the
        //     K range split over 4 warp groups, each warp a 16x16 output
        //     block (two n8 tiles sharing the A fragment), one accumulator
        //     per hi/lo term (independent MMA chains)
        if (I > cb) {
            const int kg = warp >> 2, wt = warp & 3;
            const int mt = wt >> 1, np = wt & 1;
            float acc[2][4] = {}, acc1[2][4] = {}, acc2[2][4] = {};
            const int nk = 4 * (I - cb);  // k-steps of 8
            const int k0 = kg * nk / 4, k1 = (kg + 1) * nk / 4;
            const int r = mt * 16 + gq;
#pragma unroll 2
            for (int ks = k0; ks < k1; ++ks) {
                const int K = cb + (ks >> 2), kk = (ks & 3) * 8;
                const float* Lt = tl(I, K);
                const float* Wk = Wb + (K - cb) * WBS;
                uint32_t ah[4], al[4];
                tf32_split(Lt[isw(r, kk + tq)], ah[0], al[0]);
                tf32_split(Lt[isw(r + 8, kk + tq)], ah[1], al[1]);
                tf32_split(Lt[isw(r, kk + tq + 4)], ah[2], al[2]);
                tf32_split(Lt[isw(r + 8, kk + tq + 4)], ah[3], al[3]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = np * 16 + h * 8 + gq;
                    uint32_t bh[2], bl[2];
                    tf32_split(Wk[(kk + tq) * WLD + col], bh[0], bl[0]);
                    tf32_split(Wk[(kk + tq + 4) * WLD + col], bh[1], bl[1]);
                    mma_tf32_i(acc1[h], al, bh);
                    mma_tf32_i(acc2[h], ah, bl);
                    mma_tf32_i(acc[h], ah, bh);
                }
            }
            float* P = Pq + kg * WBS;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = np * 16 + h * 8 + 2 * tq;
                P[r * WLD + col] = acc[h][0] + (acc1[h][0] + acc2[h][0]);  // small terms first
                P[r * WLD + col + 1] = acc[h][1] + (acc1[h][1] + acc2[h][1]);
                P[(r + 8) * WLD + col] = acc[h][2] + (acc1[h][2] + acc2[h][2]);
                P[(r + 8) * WLD + col + 1] = acc[h][3] + (acc1[h][3] + acc2[h][3]);
            }
        }
        __syncthreads();
        const long long cb2 = clock64();
        ck_prod += cb2 - ca;
        // (2) W(I,cb) = inv(L(I,I)) (delta - P) on warps 0-7
        if (warp < 8) {
            const int mt = warp >> 2, nb = warp & 3;
            auto rhs = [&](int rr, int cc) {
                const float dl = (I == cb && rr == cc) ? 1.f : 0.f;
                return I > cb ? dl - ((Pq[rr * WLD + cc] + Pq[WBS + rr * WLD + cc]) +
                                      (Pq[2 * WBS + rr * WLD + cc] + Pq[3 * WBS + rr * WLD + cc]))
                              : dl;
            };
            float acc[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int kk = 0; kk < 32; kk += 8) {
                const int r = mt * 16 + gq;
                uint32_t ah[4], al[4], bh[2], bl[2];
                tf32_split(Dc[isw(r, kk + tq)], ah[0], al[0]);
                tf32_split(Dc[isw(r + 8, kk + tq)], ah[1], al[1]);
                tf32_split(Dc[isw(r, kk + tq + 4)], ah[2], al[2]);
                tf32_split(Dc[isw(r + 8, kk + tq + 4)], ah[3], al[3]);
                tf32_split(rhs(kk + tq, nb * 8 + gq), bh[0], bl[0]);
                tf32_split(rhs(kk + tq + 4, nb * 8 + gq), bh[1], bl[1]);
                mma_tf32_i(acc1, al, bh);
                mma_tf32_i(acc2, ah, bl);
                mma_tf32_i(acc, ah, bh);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] += acc1[e] + acc2[e];
            const int r = mt * 16 + gq, col = nb * 8 + 2 * tq;
            Wi[r * WLD + col] = acc[0];
            Wi[r * WLD + col + 1] = acc[1];
            Wi[(r + 8) * WLD + col] = acc[2];
            Wi[(r + 8) * WLD + col + 1] = acc[3];
        }
        __syncthreads();
        ck_tri += clock64() - cb2;
    }
    const long long ck4 = clock64();
    pdl_trigger();  // only the stores remain

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
            const float w = (i >= cb * 32) ? Wb[((i >> 5) - cb) * WBS + (i & 31) * WLD + j] * up : 0.f;
            const float wz = i >= t ? w : 0.f;
            const __half hi = __float2half_rn(wz);
            const __half lo = __float2half_rn(wz - __half2float(hi));
            W[(long long)i * kW16Ld + t] = hi;
            W[(long long)i * kW16Ld + kW16Lo + t] = lo;
        }
    } else {
        // rows of column block cb: 16-byte chunks (4 columns), zero above
        // the diagonal
        float* W = c.w32 + (long long)r0 * kW32Ld + cb * 32;
        for (int e2 = tid; e2 < n * 8; e2 += IT) {
            const int i = e2 >> 3, j = (e2 & 7) * 4, t = cb * 32 + j;
            float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i >= cb * 32) {
                w = *reinterpret_cast<const float4*>(&Wb[((i >> 5) - cb) * WBS + (i & 31) * WLD + j]);
                if (i < t + 3) {  // the diagonal tile: strict upper part zero
                    w.x = i >= t ? w.x : 0.f;
                    w.y = i >= t + 1 ? w.y : 0.f;
                    w.z = i >= t + 2 ? w.z : 0.f;
                    w.w = 0.f;
                }
            }
            *reinterpret_cast<float4*>(W + (long long)i * kW32Ld + j) = w;
        }
    }
    if (cb == 0 && tid == 0) {
        atomicAdd(&g_inv_clk[0], (unsigned long long)(ck1 - ck0));
        atomicAdd(&g_inv_clk[1], (unsigned long long)(ck2 - ck1));
        atomicAdd(&g_inv_clk[2], (unsigned long long)(ck3 - ck2));
        atomicAdd(&g_inv_clk[3], (unsigned long long)ck_prod);
        atomicAdd(&g_inv_clk[4], (unsigned long long)ck_tri);
        atomicAdd(&g_inv_clk[5], (unsigned long long)(clock64() - ck4));
        atomicAdd(&g_inv_clk[6], 1ull);
    }
}

size_t inv2_smem(int n) {
    const int NB = n / 32;
    return (size_t(NB * (NB + 1) / 2) * 1024 + size_t(NB + 4) * WBS + size_t(NB) * 32) * sizeof(float);
}

}  // namespace

void inv_debug_clocks(long long* out, bool reset) {
    cudaMemcpyFromSymbol(out, g_inv_clk, sizeof(long long) * 8);
    if (reset) {
        long long z[8] = {0};
        cudaMemcpyToSymbol(g_inv_clk, z, sizeof(z));
    }
}

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
