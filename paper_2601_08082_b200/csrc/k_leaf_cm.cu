// k_leaf_cm.cu -- latency-optimised diagonal-leaf kernels for the common case:
// F16/F32 levels (FP32 arithmetic), n % 32 == 0, n <= 256 -- every leaf of the
// BASELINE configs C3..C5 (b = 256).  k_leaf.cu keeps the general kernels.
//
// The leaf lives in shared memory in a column-major packed layout whose
// columns start on 16-byte boundaries (cm_off): rows r..r+31 (r % 4 == 0) of
// column t are 8 float4 broadcast loads.  That removes every staging pass and
// every barrier from the inner loops:
//   potrf  (a) partial dot products against the finished columns read the
//              leaf in place (split over the t range for the short panels,
//              reduced in a fixed order: deterministic),
//          (b1) 32x32 diagonal block on one warp, (b2) rows below, one thread
//              per row -- right-looking schedule, reference summation order.
//   trsm   B rows staged once, L resident; per 32-column chunk the finished-
//          column sums are 8 float4 broadcasts per column, then the in-chunk
//          substitution with a reciprocal + one Newton correction division.
// Arithmetic follows dot_update (kernels.cpp:23-38): FP32 sums never rounded
// to the level mid-way, rn_level(rn_f32(c - s)), then the pivot / divide.
#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

constexpr int PW = 32;
constexpr int POT_THREADS = 256;
constexpr int TR_TPR = 8;                     // threads per row of B
constexpr int TR_ROWS = 16;                   // rows per trsm CTA
constexpr int TR_THREADS = TR_TPR * TR_ROWS;  // 128

// start of column t minus (t & ~3): element (r, t), r >= (t & ~3), of an n x n
// lower triangle (n % 4 == 0) sits at cm_off(t, n) + r, 16-byte aligned when
// r % 4 == 0.  Column t holds rows [t & ~3, n).
__host__ __device__ __forceinline__ int cm_off(int t, int n) {
    const int G = t >> 2, k = t & 3;
    return t * n - 8 * G * (G - 1) - 4 * G * k - (t & ~3);
}
__host__ __device__ __forceinline__ int cm_size(int n) {
    const int G = n >> 2;
    return n * n - 8 * G * (G - 1);
}

// correctly rounded in all but overflow / underflow corner cases: q = v*rd
// refined by one FMA residual (rd = rn(1/d))
__device__ __forceinline__ float div_nr(float v, float d, float rd) {
    const float q = v * rd;
    const float r = fmaf(-q, d, v);
    return fmaf(r, rd, q);
}

// global row-major lower triangle (T at level L) <-> smem CM layout, one warp
// per 32x32 tile through a warp-private padded tile (coalesced both sides)
template <typename T>
__device__ void cm_load(float* S, const T* g, long long ld, int n, float* tiles, int warp, int nwarps, int lane) {
    float* tile = tiles + warp * 32 * 33;
    const int nt = n / 32;
    for (int k = warp; k < nt * (nt + 1) / 2; k += nwarps) {
        int I = 0;
        while ((I + 1) * (I + 2) / 2 <= k) ++I;
        const int J = k - I * (I + 1) / 2;
        float v[32];  // 32 independent loads in flight per lane
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) v[rr] = to_f(g[(long long)(I * 32 + rr) * ld + J * 32 + lane]);
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) tile[rr * 33 + lane] = v[rr];
        __syncwarp();
#pragma unroll 8
        for (int cc = 0; cc < 32; ++cc) {
            const int t = J * 32 + cc, r = I * 32 + lane;
            if (r >= t) S[cm_off(t, n) + r] = tile[lane * 33 + cc];
        }
        __syncwarp();
    }
}

template <typename T>
__device__ void cm_store(const float* S, T* g, long long ld, int n, float* tiles, int warp, int nwarps, int lane) {
    float* tile = tiles + warp * 32 * 33;
    const int nt = n / 32;
    for (int k = warp; k < nt * (nt + 1) / 2; k += nwarps) {
        int I = 0;
        while ((I + 1) * (I + 2) / 2 <= k) ++I;
        const int J = k - I * (I + 1) / 2;
        for (int cc = 0; cc < 32; ++cc) {
            const int t = J * 32 + cc, r = I * 32 + lane;
            tile[lane * 33 + cc] = r >= t ? S[cm_off(t, n) + r] : 0.f;
        }
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
            const int r = I * 32 + rr, t = J * 32 + lane;
            if (r >= t) g[(long long)r * ld + t] = from_float<T>(tile[rr * 33 + lane]);
        }
        __syncwarp();
    }
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// ------------------------------------------------------------------ POTRF
template <int L>
__global__ void __launch_bounds__(POT_THREADS, 1) k_potrf_cm(DevCtx c, int r0, int n, uint32_t seq,
                                                            uint32_t chk_seq) {
    pdl_wait();
    using T = typename LvT<L>::T;
    extern __shared__ __align__(16) float sm[];
    float* S = sm;                              // cm_size(n)
    float* P = S + cm_size(n);                  // [n][PW] partial sums
    float* Pp = P + n * PW;                     // [4096] split-K partials / load tiles
    float* Dt = Pp + 8 * 32 * 33;               // [PW][PW+4] Dt[jj][j2] = L(J+j2, J+jj)
    T* g = lvbuf<L>(c) + (long long)r0 * c.ldw + r0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = POT_THREADS / 32;

    cm_load(S, g, c.ldw, n, Pp, warp, NW, lane);
    __syncthreads();
    if (chk_seq) {  // leaf require_finite (tree.cpp:107-108), lower triangle
        unsigned long long bad = ~0ull;
        for (int t = warp; t < n; t += NW)
            for (int r = t + lane; r < n; r += 32)
                if (!isfinite(S[cm_off(t, n) + r])) {
                    const unsigned long long k = fail_key(chk_seq, elem_local(r, t));
                    bad = k < bad ? k : bad;
                }
        warp_report_min(c, bad);
    }

    for (int J = 0; J < n; J += PW) {
        const int R = n - J;
        // (a) P[r][jj] = sum_{t<J} L(J+r, t) L(J+jj, t), 4x4 micro-tiles; the
        // t range is split over G groups when the panel is short
        if (J > 0) {
            const int units = 8 * (R / 4);
            int G = 1;
            while (2 * G * units <= POT_THREADS && G < 8) G *= 2;
            for (int ub = 0; ub < units; ub += POT_THREADS / G) {
                const int u = ub + tid % (POT_THREADS / G);
                const int grp = tid / (POT_THREADS / G);
                const bool mine = u < units && grp < G;
                const int cb = u & 7, rb = u >> 3;
                float acc[4][4];
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 4; ++y) acc[x][y] = 0.f;
                if (mine) {
                    const int tl = (J * grp) / G, th = (J * (grp + 1)) / G;
                    for (int t = tl; t < th; ++t) {
                        const float* col = S + cm_off(t, n) + J;
                        const float4 a = ld4(col + 4 * rb);
                        const float4 b = ld4(col + 4 * cb);
                        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                        for (int x = 0; x < 4; ++x)
#pragma unroll
                            for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
                    }
                }
                if (G == 1) {
                    if (mine)
#pragma unroll
                        for (int x = 0; x < 4; ++x)
#pragma unroll
                            for (int y = 0; y < 4; ++y) P[(4 * rb + x) * PW + 4 * cb + y] = acc[x][y];
                } else {
                    if (mine)
#pragma unroll
                        for (int x = 0; x < 4; ++x)
#pragma unroll
                            for (int y = 0; y < 4; ++y) Pp[(grp * R + 4 * rb + x) * PW + 4 * cb + y] = acc[x][y];
                    __syncthreads();
                    for (int e = tid; e < R * PW; e += POT_THREADS) {
                        float sum = Pp[e];
                        for (int gg = 1; gg < G; ++gg) sum += Pp[gg * R * PW + e];
                        P[e] = sum;
                    }
                }
            }
        } else {
            for (int e = tid; e < R * PW; e += POT_THREADS) P[e] = 0.f;
        }
        __syncthreads();
        // (b1) diagonal block on warp 0, lane l = row J + l: a[] = c, s[] the
        // running sum (reference order), c - s formed once per element
        if (warp == 0) {
            float a[PW], s[PW];
#pragma unroll
            for (int tt = 0; tt < PW; ++tt) {
                const bool in = tt <= lane;
                a[tt] = in ? S[cm_off(J + tt, n) + J + lane] : 0.f;
                s[tt] = in ? P[lane * PW + tt] : 0.f;
            }
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) {
                const float v = rnd<L>(a[jj] - s[jj]);
                const float piv = __shfl_sync(0xffffffffu, v, jj);
                if (lane == 0 && !(isfinite(piv) && piv > 0.f)) report(c, seq, uint64_t(J + jj));
                const float d = rnd<L>(sqrtf(piv));
                const float lij = lane == jj ? d : rnd<L>(v / d);
                a[jj] = lij;
                float* col = Dt + jj * (PW + 4);
                col[lane] = lane >= jj ? lij : 0.f;
                __syncwarp();
#pragma unroll
                for (int j2 = jj + 1; j2 < PW; ++j2) s[j2] = fmaf(lij, col[j2], s[j2]);
            }
#pragma unroll
            for (int tt = 0; tt < PW; ++tt)
                if (tt <= lane) S[cm_off(J + tt, n) + J + lane] = a[tt];
        }
        __syncthreads();
        // (b2) rows below, one thread per row, same scheme
        for (int r = PW + tid; r < R; r += POT_THREADS) {
            const int i = J + r;
            float s[PW];
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) s[jj] = P[r * PW + jj];
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) {
                asm volatile("" ::: "memory");  // keep the block's loads per iteration
                const float* col = Dt + jj * (PW + 4);
                float* dst = S + cm_off(J + jj, n) + i;
                const float x = rnd<L>(rnd<L>(*dst - s[jj]) / col[jj]);
                *dst = x;
#pragma unroll
                for (int j2 = jj + 1; j2 < PW; ++j2) s[j2] = fmaf(x, col[j2], s[j2]);
            }
        }
        __syncthreads();
    }
    cm_store(S, g, c.ldw, n, Pp, warp, NW, lane);
}

// ------------------------------------------------------------------ TRSM
// B (m x n at (br0, bc0), level L) <- B L^-T, L the n x n leaf at lr0 (its
// level-L copy).  16 rows of B per CTA, 8 threads per row.
template <int L>
__global__ void __launch_bounds__(TR_THREADS, 1) k_trsm_cm(DevCtx c, int br0, int bc0, int m, int n, int lr0,
                                                          uint32_t seq, uint32_t chk_seq, int chk_r0, int chk_c0) {
    pdl_wait();
    using T = typename LvT<L>::T;
    extern __shared__ __align__(16) float sm[];
    float* S = sm;                         // leaf, CM layout
    float* rd = S + cm_size(n);            // [n] reciprocal diagonal
    float* Bs = rd + n;                    // [TR_ROWS][n + 4]
    float* tiles = Bs + TR_ROWS * (n + 4); // 4 x 32 x 33 load tiles
    const int ldb = n + 4;
    const T* Lg = lvbuf<L>(c) + (long long)lr0 * c.ldw + lr0;
    T* Bg = lvbuf<L>(c) + (long long)br0 * c.ldw + bc0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = tid % TR_TPR, r = tid / TR_TPR;
    const int i0 = blockIdx.x * TR_ROWS, i = i0 + r;
    const bool live = i < m;
    const int rows = min(TR_ROWS, m - i0);

    cm_load(S, Lg, c.ldw, n, tiles, warp, TR_THREADS / 32, lane);
    for (int rr = warp; rr < rows; rr += TR_THREADS / 32) {
        float v[8];  // n <= 256: one row in 8 independent loads per lane
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = lane + 32 * k < n ? to_f(Bg[(long long)(i0 + rr) * c.ldw + lane + 32 * k]) : 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (lane + 32 * k < n) Bs[rr * ldb + lane + 32 * k] = v[k];
    }
    __syncthreads();
    for (int j = tid; j < n; j += TR_THREADS) rd[j] = 1.0f / S[cm_off(j, n) + j];
    if (blockIdx.x == 0 && tid == 0)  // singular diagonal (kernels.cpp:78-81), first column
        for (int j = 0; j < n; ++j) {
            const float ljj = S[cm_off(j, n) + j];
            if (ljj == 0.f || !isfinite(ljj)) {
                report(c, seq, uint64_t(j));
                break;
            }
        }
    __syncthreads();
    unsigned long long bad = ~0ull;
    const float* brow = Bs + r * ldb;

    for (int J = 0; J < n; J += PW) {
        float acc[PW];
#pragma unroll
        for (int jj = 0; jj < PW; ++jj) acc[jj] = 0.f;
        if (live)
            for (int t = q; t < J; t += TR_TPR) {
                const float xv = brow[t];
                const float* col = S + cm_off(t, n) + J;
#pragma unroll
                for (int k = 0; k < PW / 4; ++k) {
                    const float4 l4 = ld4(col + 4 * k);
                    acc[4 * k + 0] = fmaf(xv, l4.x, acc[4 * k + 0]);
                    acc[4 * k + 1] = fmaf(xv, l4.y, acc[4 * k + 1]);
                    acc[4 * k + 2] = fmaf(xv, l4.z, acc[4 * k + 2]);
                    acc[4 * k + 3] = fmaf(xv, l4.w, acc[4 * k + 3]);
                }
            }
#pragma unroll
        for (int jj = 0; jj < PW; ++jj)
#pragma unroll
            for (int o = 1; o < TR_TPR; o <<= 1) acc[jj] += __shfl_xor_sync(0xffffffffu, acc[jj], o);
        float x[PW];
        if (live) {
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) {
                asm volatile("" ::: "memory");
                const float* col = S + cm_off(J + jj, n) + J;  // col[j2] = L(J+j2, J+jj)
                const float v = rnd<L>(brow[J + jj] - acc[jj]);  // rn_level(rn_f32(c - s))
                x[jj] = rnd<L>(div_nr(v, col[jj], rd[J + jj]));
#pragma unroll
                for (int j2 = jj + 1; j2 < PW; ++j2) acc[j2] = fmaf(x[jj], col[j2], acc[j2]);
                if (chk_seq && !isfinite(x[jj])) {
                    const unsigned long long k = fail_key(chk_seq, elem_local(br0 + i - chk_r0, bc0 + J + jj - chk_c0));
                    bad = k < bad ? k : bad;
                }
            }
        }
        __syncwarp();
        if (live && q == 0)
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) Bs[r * ldb + J + jj] = x[jj];
        __syncwarp();
    }
    __syncthreads();
    for (int rr = warp; rr < rows; rr += TR_THREADS / 32)
        for (int t = lane; t < n; t += 32) Bg[(long long)(i0 + rr) * c.ldw + t] = from_float<T>(Bs[rr * ldb + t]);
    if (chk_seq) warp_report_min(c, bad);
}

size_t potrf_cm_smem(int n) {
    return (size_t(cm_size(n)) + size_t(n) * PW + 8 * 32 * 33 + PW * (PW + 4)) * sizeof(float);
}
size_t trsm_cm_smem(int n) {
    return (size_t(cm_size(n)) + n + size_t(TR_ROWS) * (n + 4) + 4 * 32 * 33) * sizeof(float);
}

}  // namespace

void init_leaf_cm_attributes() {
    const int cap = 227 * 1024;
    cudaFuncSetAttribute(k_potrf_cm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_cm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_trsm_cm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_trsm_cm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
}

bool leaf_cm_ok(int lv, int n) {
    return (lv == LV_F16 || lv == LV_F32) && n % 32 == 0 && n >= 32 && n <= 256 &&
           potrf_cm_smem(n) <= 227 * 1024 && trsm_cm_smem(n) <= 227 * 1024;
}

void launch_potrf_cm(const DevCtx& c, int lv, int r0, int n, uint32_t seq, uint32_t chk, cudaStream_t s) {
    if (lv == LV_F16) k_potrf_cm<0><<<1, POT_THREADS, potrf_cm_smem(n), s>>>(c, r0, n, seq, chk);
    else k_potrf_cm<1><<<1, POT_THREADS, potrf_cm_smem(n), s>>>(c, r0, n, seq, chk);
}

void launch_trsm_cm(const DevCtx& c, int lv, int br0, int bc0, int m, int n, int lr0, uint32_t seq,
                    uint32_t chk_seq, int chk_r0, int chk_c0, cudaStream_t s) {
    const int grid = (m + TR_ROWS - 1) / TR_ROWS;
    if (lv == LV_F16)
        k_trsm_cm<0><<<grid, TR_THREADS, trsm_cm_smem(n), s>>>(c, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0);
    else
        k_trsm_cm<1><<<grid, TR_THREADS, trsm_cm_smem(n), s>>>(c, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0);
}

}  // namespace tcb
