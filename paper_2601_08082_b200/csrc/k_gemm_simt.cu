// k_gemm_simt.cu -- grouped GEMMs for the operand classes the tcgen05
// kernel does not cover: every F64 exec class on DMMA (the FP64 tensor pipe),
// where the reference sums exact products in double (kernels.cpp:26-31) and
// an FP32 accumulator would lose accuracy; plus SIMT FP32 instantiations
// (the FP16 / FP32 classes with use_tc off), used to cross-check tcgen05.
//
// C(i,j) <- epi(C, sum_t A(i,t) B(j,t)), A/B rows K-major in the operand
// level's row-major buffer; epi is dot_update's tail (kernels.cpp:33-37).
// 64x64 output tile per CTA, BK = 16, 4x4 register block per thread.
#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__device__ __forceinline__ int find_prob(const DevProb* p, int np, int tile) {
    int lo = 0, hi = np - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p[mid].tile0 <= tile) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// epilogue of dot_update for an FP32 accumulator (exec level F16 / F32);
// returns whether the stored (level-rounded) value is non-finite
__device__ __forceinline__ bool epi_store_f(const DevCtx& c, const DevProb& p, long long off, float s) {
    float r = p.alpha == -1.0 ? -s : __double2float_rn(p.alpha * double(s));
    if (p.beta != 0.0) {
        const float cv = float(load_level(c, p.exec_level, off));
        const float t = p.beta == 1.0 ? cv : __double2float_rn(p.beta * double(cv));
        r = r + t;
    }
    store_level(c, p.exec_level, off, double(r));
    return !isfinite(round_level(p.exec_level, double(r)));
}
// FP64 accumulator (exec level F64)
__device__ __forceinline__ bool epi_store_d(const DevCtx& c, const DevProb& p, long long off, double s) {
    double r = p.alpha * s;
    if (p.beta != 0.0) r = r + p.beta * load_level(c, p.exec_level, off);
    store_level(c, p.exec_level, off, r);
    return !isfinite(round_level(p.exec_level, r));
}

template <int OPL, typename Acc>
__global__ void __launch_bounds__(256) k_gemm_simt(DevCtx c, const DevProb* probs, int np) {
    using T = typename LvT<OPL>::T;
    __shared__ Acc As[BK][BM + 4];
    __shared__ Acc Bs[BK][BN + 4];
    const DevProb p = probs[find_prob(probs, np, blockIdx.x)];
    const int lt = blockIdx.x - p.tile0;
    const int tm = lt / p.tiles_n, tn = lt % p.tiles_n;
    const int i0 = tm * BM, j0 = tn * BN;
    if (p.lower && p.c_c0 + j0 > p.c_r0 + i0 + BM - 1) return;  // tile above the diagonal
    const T* buf = lvbuf<OPL>(c);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    Acc acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = Acc(0);

    for (int k0 = 0; k0 < p.k; k0 += BK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + 256 * q;
            const int r = e >> 4, kk = e & 15;
            const int kg = k0 + kk;
            const int ia = i0 + r, jb = j0 + r;
            As[kk][r] = (ia < p.m && kg < p.k)
                            ? Acc(to_d(buf[(long long)(p.a_r0 + ia) * c.ldw + p.a_c0 + kg])) : Acc(0);
            Bs[kk][r] = (jb < p.n && kg < p.k)
                            ? Acc(to_d(buf[(long long)(p.b_r0 + jb) * c.ldw + p.b_c0 + kg])) : Acc(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            Acc a[4], b[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) a[x] = As[kk][ty * 4 + x];
#pragma unroll
            for (int y = 0; y < 4; ++y) b[y] = Bs[kk][tx * 4 + y];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
        }
        __syncthreads();
    }
    unsigned long long bad = ~0ull;  // fused require_finite (first bad element)
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int i = i0 + ty * 4 + x, j = j0 + tx * 4 + y;
            if (i >= p.m || j >= p.n) continue;
            if (p.lower && p.c_c0 + j > p.c_r0 + i) continue;
            const long long off = (long long)(p.c_r0 + i) * c.ldw + p.c_c0 + j;
            bool nb;
            if constexpr (sizeof(Acc) == 4) nb = epi_store_f(c, p, off, acc[x][y]);
            else nb = epi_store_d(c, p, off, acc[x][y]);
            if (nb && p.check_seq) {
                const unsigned long long k =
                    fail_key(p.check_seq, elem_local(p.c_r0 + i - p.chk_r0, p.c_c0 + j - p.chk_c0));
                bad = k < bad ? k : bad;
            }
        }
    if (p.check_seq) warp_report_min(c, bad);
}

// FP64-accumulating classes (F16 -> F64, F32 -> F64, F64 x F64 exec F64) on
// the FP64 tensor pipe: mma.sync.m8n8k4.f64 (DMMA).  Same 64x64 tiles and
// problem tables as the SIMT kernel; 8 warps as 2 (rows) x 4 (columns), each
// a 32x16 block of 4x2 8x8 MMA tiles.  Operands are converted to double
// exactly (half/float -> double) when staged; the reference sums exact
// products in double at F64 exec (kernels.cpp:26-31) -- only the order of
// the double sums differs.
constexpr int DBK = 16, DLD = DBK + 4;  // stride 20 doubles: conflict-free fragment reads

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <int OPL>
__global__ void __launch_bounds__(256) k_gemm_dmma(DevCtx c, const DevProb* probs, int np) {
    using T = typename LvT<OPL>::T;
    __shared__ double As[BM][DLD];
    __shared__ double Bs[BN][DLD];
    const DevProb p = probs[find_prob(probs, np, blockIdx.x)];
    const int lt = blockIdx.x - p.tile0;
    const int tm = lt / p.tiles_n, tn = lt % p.tiles_n;
    const int i0 = tm * BM, j0 = tn * BN;
    if (p.lower && p.c_c0 + j0 > p.c_r0 + i0 + BM - 1) return;  // tile above the diagonal
    const T* buf = lvbuf<OPL>(c);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
    const int g = lane >> 2, t = lane & 3;
    double acc[4][2][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

    for (int k0 = 0; k0 < p.k; k0 += DBK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + 256 * q;
            const int r = e >> 4, kk = e & 15;
            const int kg = k0 + kk;
            const int ia = i0 + r, jb = j0 + r;
            As[r][kk] = (ia < p.m && kg < p.k) ? to_d(buf[(long long)(p.a_r0 + ia) * c.ldw + p.a_c0 + kg]) : 0.0;
            Bs[r][kk] = (jb < p.n && kg < p.k) ? to_d(buf[(long long)(p.b_r0 + jb) * c.ldw + p.b_c0 + kg]) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kq = 0; kq < DBK; kq += 4) {
            double a[4], b[2];
#pragma unroll
            for (int x = 0; x < 4; ++x) a[x] = As[wm * 32 + x * 8 + g][kq + t];
#pragma unroll
            for (int y = 0; y < 2; ++y) b[y] = Bs[wn * 16 + y * 8 + g][kq + t];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) dmma(acc[x][y], a[x], b[y]);
        }
        __syncthreads();
    }
    unsigned long long bad = ~0ull;  // fused require_finite (first bad element)
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int i = i0 + wm * 32 + x * 8 + g, j = j0 + wn * 16 + y * 8 + 2 * t + h;
                if (i >= p.m || j >= p.n) continue;
                if (p.lower && p.c_c0 + j > p.c_r0 + i) continue;
                const long long off = (long long)(p.c_r0 + i) * c.ldw + p.c_c0 + j;
                if (epi_store_d(c, p, off, acc[x][y][h]) && p.check_seq) {
                    const unsigned long long k =
                        fail_key(p.check_seq, elem_local(p.c_r0 + i - p.chk_r0, p.c_c0 + j - p.chk_c0));
                    bad = k < bad ? k : bad;
                }
            }
    if (p.check_seq) warp_report_min(c, bad);
}

}  // namespace

int simt_tiles(std::vector<DevProb>& probs) {
    int tiles = 0;
    for (auto& p : probs) {
        p.tile0 = tiles;
        p.tiles_n = (p.n + BN - 1) / BN;
        tiles += ((p.m + BM - 1) / BM) * p.tiles_n;
    }
    return tiles;
}

void launch_gemm_simt(const DevCtx& c, int gclass, const DevProb* d_probs, int nprob, int tiles,
                      cudaStream_t s) {
    if (tiles <= 0) return;
    switch (gclass) {
        case GC_SIMT_F16: k_gemm_simt<0, float><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        case GC_SIMT_F32: k_gemm_simt<1, float><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        // FP64 accumulation on the FP64 tensor pipe (DMMA)
        case GC_SIMT_F16D: k_gemm_dmma<0><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        case GC_SIMT_F32D: k_gemm_dmma<1><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        default: k_gemm_dmma<2><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
    }
}

}  // namespace tcb
