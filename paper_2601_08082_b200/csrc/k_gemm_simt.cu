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
    pdl_wait();
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
    pdl_wait();
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

// Small FP32 x FP32 problems (F32 exec) on the warp-level tensor path:
// mma.sync m16n8k8 TF32 with a three-pass hi/lo split (hi = x truncated to
// TF32, lo = x - hi; lo*hi + hi*lo + hi*hi, FP32 accumulate) -- the same
// arithmetic as the tcgen05 TF32X3 kernel, without its per-launch setup
// (TMEM allocation, descriptors, pipeline fill), which dominates the
// 256-wide leaf-level solves and updates on the factorization's chain.
// 32x32 output tiles (simt_tiles with M32_TILE), 4 warps of 16x16.
constexpr int MK = 32, MLD = MK + 4;  // k-slab, padded row (conflict-free fragments)
// its own 32x32 output tiles (4x the CTAs of the 64x64 SIMT tiles: these
// problems are latency-bound, the chain waits on each)

__device__ __forceinline__ void mma_tf32x(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(x) & 0xFFFFE000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}

__global__ void __launch_bounds__(128) k_gemm_mma32(DevCtx c, const DevProb* probs, int np) {
    pdl_wait();
    pdl_trigger();  // short kernel: let the dependents launch right away
    constexpr int TM = M32_TILE, TN = M32_TILE;  // 32 x 32 output tile: 4 warps of 16 x 16
    __shared__ __align__(16) float As[2][TM][MLD];
    __shared__ __align__(16) float Bs[2][TN][MLD];
    const DevProb p = probs[find_prob(probs, np, blockIdx.x)];
    const int lt = blockIdx.x - p.tile0;
    const int tm = lt / p.tiles_n, tn = lt % p.tiles_n;
    const int i0 = tm * TM, j0 = tn * TN;
    if (p.lower && p.c_c0 + j0 > p.c_r0 + i0 + TM - 1) return;  // tile above the diagonal
    const float* buf = c.b32;
    // B from the FP32 leaf inverses for inverse-based solves (plan.hpp kW32Ld)
    const float* bbuf = p.b_buf == BUF_W32 ? c.w32 : c.b32;
    const long long bld = p.b_buf == BUF_W32 ? kW32Ld : c.ldw;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 1, wn = warp & 1;  // 2 x 2 warps of 16 x 16
    const int g = lane >> 2, tq = lane & 3;
    float acc[2][4];
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[y][e] = 0.f;
    // 32 x 32 slabs of A and B, double-buffered with cp.async (zero-filled
    // outside the problem): the next slab loads while this one multiplies
    auto load = [&](int k0, int sb) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int e = threadIdx.x + 128 * q;  // 256 x 16 B per operand
            const int r = e >> 3, kq = (e & 7) * 4;
            const int kg = k0 + kq;
            const int kb = min(16, max(0, (p.k - kg) * 4));
            const int ia = i0 + r, jb = j0 + r;
            cp_async16(&As[sb][r][kq], buf + (long long)(p.a_r0 + (ia < p.m ? ia : 0)) * c.ldw + p.a_c0 + (kb ? kg : 0),
                       ia < p.m ? kb : 0);
            cp_async16(&Bs[sb][r][kq], bbuf + (long long)(p.b_r0 + (jb < p.n ? jb : 0)) * bld + p.b_c0 + (kb ? kg : 0),
                       jb < p.n ? kb : 0);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int ns = (p.k + MK - 1) / MK;
    load(0, 0);
    for (int st = 0; st < ns; ++st) {
        const int sb = st & 1;
        if (st + 1 < ns) {
            load((st + 1) * MK, sb ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < MK; kk += 8) {
            uint32_t ah[4], al[4];
            const int rb = wm * 16;
            split_tf32(As[sb][rb + g][kk + tq], ah[0], al[0]);
            split_tf32(As[sb][rb + g + 8][kk + tq], ah[1], al[1]);
            split_tf32(As[sb][rb + g][kk + tq + 4], ah[2], al[2]);
            split_tf32(As[sb][rb + g + 8][kk + tq + 4], ah[3], al[3]);
#pragma unroll
            for (int y = 0; y < 2; ++y) {
                const int cb = wn * 16 + y * 8;
                uint32_t bh[2], bl[2];
                split_tf32(Bs[sb][cb + g][kk + tq], bh[0], bl[0]);
                split_tf32(Bs[sb][cb + g][kk + tq + 4], bh[1], bl[1]);
                mma_tf32x(acc[y], al, bh);
                mma_tf32x(acc[y], ah, bl);
                mma_tf32x(acc[y], ah, bh);
            }
        }
        __syncthreads();
    }
    unsigned long long bad = ~0ull;
#pragma unroll
    for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int i = i0 + wm * 16 + g + (e >= 2 ? 8 : 0);
            const int j = j0 + wn * 16 + y * 8 + 2 * tq + (e & 1);
            if (i >= p.m || j >= p.n) continue;
            if (p.lower && p.c_c0 + j > p.c_r0 + i) continue;
            const long long off = (long long)(p.c_r0 + i) * c.ldw + p.c_c0 + j;
            if (epi_store_f(c, p, off, acc[y][e]) && p.check_seq) {
                const unsigned long long k =
                    fail_key(p.check_seq, elem_local(p.c_r0 + i - p.chk_r0, p.c_c0 + j - p.chk_c0));
                bad = k < bad ? k : bad;
            }
        }
    if (p.check_seq) warp_report_min(c, bad);
}

// In-place inverse leaf solves X = rn32(B W^T) (GC_MMA32W): one CTA owns
// WM full rows (all n <= 256 output columns), so it reads every K column of
// its rows before it writes any of them -- no other CTA touches those rows.
// 8 warps, each WM rows x 32 columns (WM/16 m16 x 4 n8 fragments).
constexpr int WN = 256;  // widest n
constexpr int WM = M32W_ROWS;  // rows per CTA (16: twice the CTAs of 32 rows for the 256-row solves on the chain)
__global__ void __launch_bounds__(256) k_gemm_mma32w(DevCtx c, const DevProb* probs, int np) {
    pdl_wait();
    pdl_trigger();  // short kernel: let the dependents launch right away
    extern __shared__ __align__(16) float wsm[];
    float (*As)[WM][MLD] = reinterpret_cast<float (*)[WM][MLD]>(wsm);            // [2][WM][MLD]
    float (*Bs)[WN][MLD] = reinterpret_cast<float (*)[WN][MLD]>(wsm + 2 * WM * MLD);  // [2][256][MLD]
    const DevProb p = probs[find_prob(probs, np, blockIdx.x)];
    const int lt = blockIdx.x - p.tile0;
    const int i0 = lt * WM;  // tiles_n == 1
    const float* buf = c.b32;
    const float* bbuf = p.b_buf == BUF_W32 ? c.w32 : c.b32;
    const long long bld = p.b_buf == BUF_W32 ? kW32Ld : c.ldw;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    constexpr int XM = WM / 16;
    float acc[XM][4][4];
#pragma unroll
    for (int x = 0; x < XM; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[x][y][e] = 0.f;
    auto load = [&](int k0, int sb) {
        if (threadIdx.x < WM * 8) {  // A: WM rows x 32 k, 16 B per thread
            const int e = threadIdx.x;
            const int r = e >> 3, kq = (e & 7) * 4;
            const int kg = k0 + kq;
            const int kb = min(16, max(0, (p.k - kg) * 4));
            const int ia = i0 + r;
            cp_async16(&As[sb][r][kq], buf + (long long)(p.a_r0 + (ia < p.m ? ia : 0)) * c.ldw + p.a_c0 + (kb ? kg : 0),
                       ia < p.m ? kb : 0);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {  // B: 256 rows x 32 k = 2048 x 16 B
            const int e = threadIdx.x + 256 * q;
            const int r = e >> 3, kq = (e & 7) * 4;
            const int kg = k0 + kq;
            const int kb = min(16, max(0, (p.k - kg) * 4));
            cp_async16(&Bs[sb][r][kq], bbuf + (long long)(p.b_r0 + (r < p.n ? r : 0)) * bld + p.b_c0 + (kb ? kg : 0),
                       r < p.n ? kb : 0);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int ns = (p.k + MK - 1) / MK;
    load(0, 0);
    for (int st = 0; st < ns; ++st) {
        const int sb = st & 1;
        if (st + 1 < ns) {
            load((st + 1) * MK, sb ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < MK; kk += 8) {
            uint32_t ah[XM][4], al[XM][4];
#pragma unroll
            for (int x = 0; x < XM; ++x) {
                const int rb = x * 16;
                split_tf32(As[sb][rb + g][kk + tq], ah[x][0], al[x][0]);
                split_tf32(As[sb][rb + g + 8][kk + tq], ah[x][1], al[x][1]);
                split_tf32(As[sb][rb + g][kk + tq + 4], ah[x][2], al[x][2]);
                split_tf32(As[sb][rb + g + 8][kk + tq + 4], ah[x][3], al[x][3]);
            }
#pragma unroll
            for (int y = 0; y < 4; ++y) {
                const int cb = warp * 32 + y * 8;
                uint32_t bh[2], bl[2];
                split_tf32(Bs[sb][cb + g][kk + tq], bh[0], bl[0]);
                split_tf32(Bs[sb][cb + g][kk + tq + 4], bh[1], bl[1]);
#pragma unroll
                for (int x = 0; x < XM; ++x) {
                    mma_tf32x(acc[x][y], al[x], bh);
                    mma_tf32x(acc[x][y], ah[x], bl);
                    mma_tf32x(acc[x][y], ah[x], bh);
                }
            }
        }
        __syncthreads();
    }
    // every K column of these rows has been read (the loop's last barrier):
    // the in-place write is safe
    unsigned long long bad = ~0ull;
#pragma unroll
    for (int x = 0; x < XM; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = i0 + x * 16 + g + (e >= 2 ? 8 : 0);
                const int j = warp * 32 + y * 8 + 2 * tq + (e & 1);
                if (i >= p.m || j >= p.n) continue;
                const long long off = (long long)(p.c_r0 + i) * c.ldw + p.c_c0 + j;
                if (epi_store_f(c, p, off, acc[x][y][e]) && p.check_seq) {
                    const unsigned long long k =
                        fail_key(p.check_seq, elem_local(p.c_r0 + i - p.chk_r0, p.c_c0 + j - p.chk_c0));
                    bad = k < bad ? k : bad;
                }
            }
    if (p.check_seq) warp_report_min(c, bad);
}
constexpr size_t kMma32wSmem = sizeof(float) * 2 * (WM + WN) * MLD;

}  // namespace

int simt_tiles(std::vector<DevProb>& probs, int tile, int tile_n) {
    const int tm = tile > 0 ? tile : BM, tn = tile_n > 0 ? tile_n : tile > 0 ? tile : BN;
    int tiles = 0;
    for (auto& p : probs) {
        p.tile0 = tiles;
        p.tiles_n = (p.n + tn - 1) / tn;
        tiles += ((p.m + tm - 1) / tm) * p.tiles_n;
    }
    return tiles;
}

void init_mma32w_attributes() {
    cudaFuncSetAttribute(k_gemm_mma32w, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMma32wSmem));
}

void launch_gemm_simt(const DevCtx& c, int gclass, const DevProb* d_probs, int nprob, int tiles,
                      cudaStream_t s) {
    if (tiles <= 0) return;
    switch (gclass) {
        case GC_SIMT_F16: k_gemm_simt<0, float><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        case GC_SIMT_F32: k_gemm_simt<1, float><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        case GC_MMA32: k_gemm_mma32<<<tiles, 128, 0, s>>>(c, d_probs, nprob); break;
        case GC_MMA32W: k_gemm_mma32w<<<tiles, 256, kMma32wSmem, s>>>(c, d_probs, nprob); break;
        // FP64 accumulation on the FP64 tensor pipe (DMMA)
        case GC_SIMT_F16D: k_gemm_dmma<0><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        case GC_SIMT_F32D: k_gemm_dmma<1><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
        default: k_gemm_dmma<2><<<tiles, 256, 0, s>>>(c, d_probs, nprob); break;
    }
}

}  // namespace tcb
