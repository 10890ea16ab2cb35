// k_leaf.cu -- diagonal leaf POTRF and leaf TRSM (kernels.cpp:42-92).
//
// Both keep the reference's per-element arithmetic (dot_update, kernels.cpp:
// 23-38): the dot product accumulates in Acc (FP32 for the F16/F32 levels,
// FP64 for F64) and is never rounded to the level mid-way; the result is
// rn_level(rn_acc(c - s)), then pivots / divisions round to the level.  Only
// the summation order differs (blocked by 32 columns).
//
// potrf_leaf: one CTA per leaf.  The lower triangle lives in shared memory
// (packed rows) when it fits, else it is worked on in place in global memory
// (L2-resident).  Columns are processed in 32-wide panels:
//   a) P = partial dot products against all finished columns (register-
//      blocked 4x4 per thread),
//   b1) the 32x32 diagonal block factored by one warp with shuffles,
//   b2) rows below solved against it, one thread per row, no barriers.
// trsm_leaf: one thread per row of B, 128 rows per CTA; the current 32-column
// chunk of L is staged (transposed) in shared memory and broadcast.
#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

constexpr int PW = 32;  // panel width
__device__ long long g_leaf_clk[8];  // debug: cycles per potrf phase (a, b1, b2), count
constexpr int TRSM_TPR = 8;                    // threads per row of B
constexpr int TRSM_ROWS = 128 / TRSM_TPR;      // rows per trsm CTA
constexpr int POTRF_THREADS = 256;
constexpr int KT = 16;  // potrf phase (a): finished columns staged per step

template <typename Acc>
constexpr size_t potrf_smem(int n, bool smem) {
    return (size_t(n) * PW + size_t(KT) * (n + 4) + size_t(KT) * (PW + 4) + size_t(PW) * (PW + 4) +
            (smem ? size_t(n) * (n + 1) / 2 : 0)) * sizeof(Acc);
}

template <int L, bool SMEM>
struct LeafAcc {
    using T = typename LvT<L>::T;
    using Acc = typename LvT<L>::Acc;
    Acc* s;             // packed rows (SMEM)
    T* g;               // global leaf origin (row-major, ld)
    long long ld;
    __device__ __forceinline__ Acc get(int i, int j) const {
        if constexpr (SMEM) return s[(i * (i + 1)) / 2 + j];
        else return Acc(to_d(g[(long long)i * ld + j]));
    }
    __device__ __forceinline__ void set(int i, int j, Acc v) const {
        if constexpr (SMEM) s[(i * (i + 1)) / 2 + j] = v;
        else g[(long long)i * ld + j] = from_double<T>(double(v));
    }
};

// (b1) factor the diagonal block at (J, J) on one warp, lane l = row J + l.
// a[] holds c, s[] the running dot product in the reference's order
// (kernels.cpp:28-32); c - s is formed once per element (kernels.cpp:33-37)
// -- subtracting products from c directly would round relative to the
// large diagonal.  Each solved column is broadcast through Dt (also kept for
// the rows below: Dt[jj][j2] = L(J+j2, J+jj)).
template <int L, bool FULL, typename Acc, typename AccT>
__device__ __forceinline__ void diag_block(const AccT& A, const Acc* P, Acc* Dt, int J, int w, int lane,
                                           const DevCtx& c, uint32_t seq) {
    Acc a[PW], s[PW];
    const bool live = lane < w;
#pragma unroll
    for (int tt = 0; tt < PW; ++tt) {
        const bool in = live && tt <= lane && (FULL || tt < w);
        a[tt] = in ? A.get(J + lane, J + tt) : Acc(0);
        s[tt] = in ? P[lane * PW + tt] : Acc(0);
    }
#pragma unroll
    for (int jj = 0; jj < PW; ++jj) {
        if (FULL || jj < w) {
            const Acc v = rnd<L>(a[jj] - s[jj]);  // rn_level(rn_acc(c - s))
            const Acc piv = __shfl_sync(0xffffffffu, v, jj);
            if (lane == 0 && !(isfinite(piv) && piv > Acc(0))) report(c, seq, uint64_t(J + jj));
            const Acc d = rnd<L>(sqrt(piv));
            const Acc lij = lane == jj ? d : rnd<L>(v / d);
            a[jj] = lij;
            Acc* col = Dt + jj * (PW + 4);
            col[lane] = lane >= jj ? lij : Acc(0);
            __syncwarp();
#pragma unroll
            for (int j2 = jj + 1; j2 < PW; ++j2) s[j2] = fma(lij, col[j2], s[j2]);
        }
    }
    if (live)
#pragma unroll
        for (int tt = 0; tt < PW; ++tt)
            if (tt <= lane && (FULL || tt < w)) A.set(J + lane, J + tt, a[tt]);
}

// (b2) rows J+PW .. J+R-1 against the factored diagonal block: one thread
// per row, right-looking over the block's columns with the same separate
// running sum; the block comes from Dt (vector broadcast reads).
template <int L, bool FULL, typename Acc, typename AccT>
__device__ __forceinline__ void below_rows(const AccT& A, const Acc* P, const Acc* Dt, int J, int R, int w,
                                           int tid) {
    for (int r = PW + tid; r < R; r += POTRF_THREADS) {
        const int i = J + r;
        Acc s[PW];
#pragma unroll
        for (int jj = 0; jj < PW; ++jj) s[jj] = (FULL || jj < w) ? P[r * PW + jj] : Acc(0);
#pragma unroll
        for (int jj = 0; jj < PW; ++jj) {
            if (FULL || jj < w) {
                // compiler fence: keep the block's loads inside their
                // iteration (hoisting all 496 would explode register use)
                asm volatile("" ::: "memory");
                const Acc* col = Dt + jj * (PW + 4);
                const Acc x = rnd<L>(rnd<L>(A.get(i, J + jj) - s[jj]) / col[jj]);
                A.set(i, J + jj, x);
#pragma unroll
                for (int j2 = jj + 1; j2 < PW; ++j2) s[j2] = fma(x, col[j2], s[j2]);
            }
        }
    }
}

template <int L, bool SMEM>
__global__ void __launch_bounds__(POTRF_THREADS, 1) k_potrf_leaf(DevCtx c, int r0, int n, uint32_t seq,
                                                              uint32_t chk_seq) {
    pdl_wait();
    using T = typename LvT<L>::T;
    using Acc = typename LvT<L>::Acc;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ldS = n + 4;                        // staged rows, padded
    Acc* P = reinterpret_cast<Acc*>(smem_raw);    // [n][PW] partial sums
    Acc* As = P + size_t(n) * PW;                 // [KT][ldS]  A(J+r, t0+tt) transposed
    Acc* Bs = As + size_t(KT) * ldS;              // [KT][PW+4] A(J+jj, t0+tt)
    Acc* Dt = Bs + size_t(KT) * (PW + 4);         // [PW][PW+4] Dt[jj][j2] = L(J+j2, J+jj)
    Acc* S = Dt + size_t(PW) * (PW + 4);          // packed lower triangle (SMEM)
    T* g = lvbuf<L>(c) + (long long)r0 * c.ldw + r0;
    LeafAcc<L, SMEM> A{S, g, c.ldw};
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = POTRF_THREADS / 32;

    // leaf require_finite (tree.cpp:107-108) fused into the load: the first
    // non-finite element of the lower triangle in column-major order
    if (chk_seq) {
        unsigned long long bad = ~0ull;
        for (int i = warp; i < n; i += NW)
            for (int j = lane; j <= i; j += 32) {
                const Acc v = Acc(to_d(g[(long long)i * c.ldw + j]));
                if constexpr (SMEM) S[(i * (i + 1)) / 2 + j] = v;
                if (!isfinite(v)) {
                    const unsigned long long k = fail_key(chk_seq, elem_local(i, j));
                    bad = k < bad ? k : bad;
                }
            }
        warp_report_min(c, bad);
        __syncthreads();
    } else if constexpr (SMEM) {
        for (int i = warp; i < n; i += NW)
            for (int j = lane; j <= i; j += 32) S[(i * (i + 1)) / 2 + j] = Acc(to_d(g[(long long)i * c.ldw + j]));
        __syncthreads();
    }

    long long t_ph = clock64();
    long long* clk = g_leaf_clk;
    for (int J = 0; J < n; J += PW) {
        const int w = min(PW, n - J);
        const int R = n - J;  // rows of this panel
        // (a) P[r][jj] = sum_{t<J} A(J+r, t) * A(J+jj, t): a small SIMT GEMM,
        // KT finished columns at a time staged transposed (conflict-free
        // float4 reads), one 4x4 register block per thread
        const int units = 8 * ((R + 3) / 4);
        for (int ub = 0; ub < units; ub += POTRF_THREADS) {  // one pass for n <= 256
        const int cb = tid & 7, rb = (ub + tid) >> 3;
        const bool mine = ub + tid < units;
        Acc acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = Acc(0);
        for (int t0 = 0; t0 < J; t0 += KT) {
            for (int e = tid; e < R * KT; e += POTRF_THREADS) {
                const int r = e / KT, tt = e % KT;
                As[tt * ldS + r] = A.get(J + r, t0 + tt);
            }
            for (int e = tid; e < PW * KT; e += POTRF_THREADS) {
                const int jj = e / KT, tt = e % KT;
                Bs[tt * (PW + 4) + jj] = jj < w ? A.get(J + jj, t0 + tt) : Acc(0);
            }
            __syncthreads();
            if (mine)
#pragma unroll 4
                for (int tt = 0; tt < KT; ++tt) {
                    Acc a[4], bb[4];
#pragma unroll
                    for (int x = 0; x < 4; ++x) a[x] = As[tt * ldS + 4 * rb + x];
#pragma unroll
                    for (int y = 0; y < 4; ++y) bb[y] = Bs[tt * (PW + 4) + 4 * cb + y];
#pragma unroll
                    for (int x = 0; x < 4; ++x)
#pragma unroll
                        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], bb[y], acc[x][y]);
                }
            __syncthreads();
        }
        if (mine)
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) {
                    const int r = 4 * rb + x;
                    if (r < R) P[r * PW + 4 * cb + y] = acc[x][y];
                }
        }
        __syncthreads();
        if (threadIdx.x == 0) { const long long t = clock64(); clk[0] += t - t_ph; t_ph = t; }
        // (b1) diagonal block by warp 0 (lane l owns row J + l), then (b2)
        // the rows below, one thread per row.  Right-looking schedule in the
        // reference's summation order (see diag_block / below_rows).
        if (w == PW) {
            if (warp == 0) diag_block<L, true>(A, P, Dt, J, w, lane, c, seq);
            __syncthreads();
            if (threadIdx.x == 0) { const long long t = clock64(); clk[1] += t - t_ph; t_ph = t; }
            below_rows<L, true>(A, P, Dt, J, R, w, tid);
        } else {
            if (warp == 0) diag_block<L, false>(A, P, Dt, J, w, lane, c, seq);
            __syncthreads();
            if (threadIdx.x == 0) { const long long t = clock64(); clk[1] += t - t_ph; t_ph = t; }
            below_rows<L, false>(A, P, Dt, J, R, w, tid);
        }
        __syncthreads();
        if (threadIdx.x == 0) { const long long t = clock64(); clk[2] += t - t_ph; t_ph = t; }
    }
    if (threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&clk[3]), 1ull);
    if constexpr (SMEM) {
        for (int i = warp; i < n; i += NW)
            for (int j = lane; j <= i; j += 32)
                g[(long long)i * c.ldw + j] = from_double<T>(double(S[(i * (i + 1)) / 2 + j]));
    }
}

// ---------------------------------------------------------------------------
// F64 leaves (BASELINE C1 [F16, F64] b=128, C2 [F16, F32, F64] b=256):
// potrf_leaf in FP64 with the panel products on the FP64 tensor pipe.  The
// leaf stays in global memory (L2-resident: a 256 F64 triangle is 264 KB);
// per 32-column panel J:
//   (a) P = A(J.., 0:J) A(J:J+32, 0:J)^T by DMMA (mma.sync m8n8k4 f64), the
//       K range staged through shared memory 32 columns at a time (the B
//       operand is the first 32 staged rows); 8x8 output tiles, a warp owns
//       row tiles warp, warp+8, ... and all four column tiles;
//   (b1) the diagonal block on warp 0 (diag_block: the reference's per-
//       element order, IEEE sqrt and division);
//   (b2) the rows below, one thread per row: the row's 32 entries loaded
//       before the substitution chain, quotients v/d by Markstein's
//       correctly rounded scheme from y = rn(1/d) (q = rn(v y), the exact
//       FMA residual, one correction: rn(v/d) in the normal range).
// Only the summation order differs from kernels.cpp:42-69.
// ---------------------------------------------------------------------------
constexpr int F64T = 256;     // threads

// (b1) on its own register allocation: inlined into the kernel beside the
// DMMA phase and the unrolled rows-below loop it measured 3.5x slower
__device__ __noinline__ void diag_block_f64(double* g, long long ld, const double* P, double* Dt, int J, int lane,
                                            const DevCtx& c, uint32_t seq) {
    LeafAcc<2, false> A{nullptr, g, ld};
    diag_block<2, true>(A, P, Dt, J, PW, lane, c, seq);
}
constexpr int F64LD = 36;     // staged slice row pitch (doubles)

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(F64T, 1) k_potrf_f64(DevCtx c, int r0, int n, uint32_t seq, uint32_t chk_seq) {
    pdl_wait();
    extern __shared__ __align__(16) double f64sm[];
    double* P = f64sm;                          // [n][PW] partial sums
    double* As = P + size_t(n) * PW;            // [n][F64LD] staged K-slice, rows J..n-1
    double* Dt = As + size_t(n) * F64LD;        // [PW][PW+4] Dt[jj][j2] = L(J+j2, J+jj)
    double* Dr = Dt + PW * (PW + 4);            // [PW] rn(1 / L(J+jj, J+jj))
    double* g = c.b64 + (long long)r0 * c.ldw + r0;
    const long long ld = c.ldw;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = F64T / 32;

    if (chk_seq) {  // leaf require_finite (tree.cpp:107-108)
        unsigned long long bad = ~0ull;
        for (int i = warp; i < n; i += NW)
            for (int j = lane; j <= i; j += 32)
                if (!isfinite(g[(long long)i * ld + j])) {
                    const unsigned long long k = fail_key(chk_seq, elem_local(i, j));
                    bad = k < bad ? k : bad;
                }
        warp_report_min(c, bad);
    }

    long long t_ph = clock64();
    long long* clk = g_leaf_clk;
    for (int J = 0; J < n; J += PW) {
        const int R = n - J;        // rows of this panel (multiple of 32)
        const int mtiles = R >> 3;  // 8-row tiles
        // ---- (a) the panel's partial sums on DMMA
        double acc[4][4][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) acc[mi][nt][0] = acc[mi][nt][1] = 0.0;
        for (int t0 = 0; t0 < J; t0 += PW) {
            __syncthreads();
            for (int e = tid; e < R * (PW / 2); e += F64T) {  // 16-byte loads, lanes along the row
                const int r = e >> 4, c2 = (e & 15) * 2;
                const double2 v = *reinterpret_cast<const double2*>(g + (long long)(J + r) * ld + t0 + c2);
                *reinterpret_cast<double2*>(As + r * F64LD + c2) = v;
            }
            __syncthreads();
#pragma unroll 2
            for (int kk = 0; kk < PW; kk += 4) {
                double b[4];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) b[nt] = As[(nt * 8 + (lane >> 2)) * F64LD + kk + (lane & 3)];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) {
                    const int mt = warp + NW * mi;
                    if (mt < mtiles) {
                        const double a = As[(mt * 8 + (lane >> 2)) * F64LD + kk + (lane & 3)];
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mi][nt], a, b[nt]);
                    }
                }
            }
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const int mt = warp + NW * mi;
            if (mt < mtiles)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    const int r = mt * 8 + (lane >> 2), col = nt * 8 + 2 * (lane & 3);
                    P[r * PW + col] = acc[mi][nt][0];
                    P[r * PW + col + 1] = acc[mi][nt][1];
                }
        }
        __syncthreads();
        if (threadIdx.x == 0) { const long long t = clock64(); clk[0] += t - t_ph; t_ph = t; }
        // ---- (b1) the diagonal block
        if (warp == 0) {
            diag_block_f64(g, ld, P, Dt, J, lane, c, seq);
            __syncwarp();
            Dr[lane] = __drcp_rn(Dt[lane * (PW + 4) + lane]);  // y = rn(1/d) for the rows below
        }
        __syncthreads();
        if (threadIdx.x == 0) { const long long t = clock64(); clk[1] += t - t_ph; t_ph = t; }
        // ---- (b2) the rows below: staged through shared memory (16-byte
        // loads), one thread per row, written back the same way
        for (int e = tid; e < (R - PW) * (PW / 2); e += F64T) {
            const int r = PW + (e >> 4), c2 = (e & 15) * 2;
            *reinterpret_cast<double2*>(As + r * F64LD + c2) =
                *reinterpret_cast<const double2*>(g + (long long)(J + r) * ld + J + c2);
        }
        __syncthreads();
        for (int r = PW + tid; r < R; r += F64T) {
            double s[PW];
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) s[jj] = P[r * PW + jj];
            double* row = As + r * F64LD;
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) {
                // keep the block's loads inside their iteration (hoisting
                // them all would exhaust the registers)
                asm volatile("" ::: "memory");
                const double* col = Dt + jj * (PW + 4);
                const double a = row[jj] - s[jj];                     // rn(c - s)
                const double d = col[jj], y = Dr[jj];
                const double q0 = a * y;
                const double x = fma(fma(-q0, d, a), y, q0);        // rn(a / d) (Markstein)
                row[jj] = x;
#pragma unroll
                for (int j2 = jj + 1; j2 < PW; ++j2) s[j2] = fma(x, col[j2], s[j2]);
            }
        }
        __syncthreads();
        for (int e = tid; e < (R - PW) * (PW / 2); e += F64T) {
            const int r = PW + (e >> 4), c2 = (e & 15) * 2;
            *reinterpret_cast<double2*>(g + (long long)(J + r) * ld + J + c2) =
                *reinterpret_cast<const double2*>(As + r * F64LD + c2);
        }
        __syncthreads();
        if (threadIdx.x == 0) { const long long t = clock64(); clk[2] += t - t_ph; t_ph = t; }
    }
    if (threadIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&clk[3]), 1ull);
}

size_t potrf_f64_smem(int n) { return (size_t(n) * PW + size_t(n) * F64LD + PW * (PW + 4) + PW) * sizeof(double); }

// trsm_leaf: B (m x n at (br0, bc0)) <- B * L^-T, L the n x n square at lr0
// The CTA's 32 rows of B are staged in shared memory (BS) so the
// finished-column sums read them at smem latency; the in-chunk substitution
// is right-looking (each new x immediately updates the later partial sums),
// which leaves one short dependent chain per column.  Fused require_finite
// (tree.cpp:121) on the values written, relative to the panel origin.
template <int L, bool BS>
__global__ void __launch_bounds__(128) k_trsm_leaf(DevCtx c, int br0, int bc0, int m, int n, int lr0,
                                                  uint32_t seq, uint32_t chk_seq, int chk_r0, int chk_c0) {
    pdl_wait();
    using T = typename LvT<L>::T;
    using Acc = typename LvT<L>::Acc;
    constexpr int TSL = 128;  // staged slice of finished columns
    __shared__ __align__(16) Acc Lc[TSL][PW + 4];  // 16-byte rows: vector broadcast reads
    __shared__ __align__(16) Acc D[PW][PW + 4];
    extern __shared__ __align__(16) unsigned char trsm_smem[];
    Acc* Bs = reinterpret_cast<Acc*>(trsm_smem);  // [TRSM_ROWS][n + 1]
    const int ldb = n + 1;
    const T* Lg = lvbuf<L>(c) + (long long)lr0 * c.ldw + lr0;
    T* Bg = lvbuf<L>(c) + (long long)br0 * c.ldw + bc0;
    // a quad of threads per row: the finished-column sums are split over the
    // quad (t = q, q+4, ...) and reduced with shuffles; the in-chunk
    // substitution is run redundantly by the quad, quad lane 0 stores
    const int q = threadIdx.x % TRSM_TPR;
    const int r = threadIdx.x / TRSM_TPR;
    const int i0 = blockIdx.x * TRSM_ROWS;
    const int i = i0 + r;
    const bool live = i < m;
    T* row = Bg + (long long)(live ? i : 0) * c.ldw;
    if constexpr (BS) {
        const int rows = min(TRSM_ROWS, m - i0);
        for (int rr = threadIdx.x >> 5; rr < rows; rr += 4)
            for (int t = threadIdx.x & 31; t < n; t += 32)
                Bs[rr * ldb + t] = Acc(to_d(Bg[(long long)(i0 + rr) * c.ldw + t]));
        __syncthreads();
    }
    auto getx = [&](int t) -> Acc {
        if constexpr (BS) return Bs[r * ldb + t];
        else return Acc(to_d(row[t]));
    };
    unsigned long long bad = ~0ull;

    long long t_tr = clock64();
    for (int J = 0; J < n; J += PW) {
        const int w = min(PW, n - J);
        Acc acc[PW];
#pragma unroll
        for (int jj = 0; jj < PW; ++jj) acc[jj] = Acc(0);
        for (int t0 = 0; t0 < J; t0 += TSL) {
            const int tw = min(TSL, J - t0);
            __syncthreads();
            for (int e = threadIdx.x; e < tw * PW; e += 128) {
                const int tt = e % tw, jj = e / tw;
                Lc[tt][jj] = jj < w ? Acc(to_d(Lg[(long long)(J + jj) * c.ldw + t0 + tt])) : Acc(0);
            }
            __syncthreads();
            if (live)
                for (int tt = q; tt < tw; tt += TRSM_TPR) {
                    const Acc xv = getx(t0 + tt);
#pragma unroll
                    for (int jj = 0; jj < PW; ++jj) acc[jj] = fma(xv, Lc[tt][jj], acc[jj]);
                }
        }
#pragma unroll
        for (int jj = 0; jj < PW; ++jj) {
            for (int o = 1; o < TRSM_TPR; o <<= 1) acc[jj] += __shfl_xor_sync(0xffffffffu, acc[jj], o);
        }
        __syncthreads();
        for (int e = threadIdx.x; e < PW * PW; e += 128) {
            const int tt = e % PW, jj = e / PW;
            D[tt][jj] = (jj < w && tt < w) ? Acc(to_d(Lg[(long long)(J + jj) * c.ldw + J + tt])) : Acc(1);
        }
        __syncthreads();
        if (blockIdx.x == 0 && threadIdx.x == 0)
            for (int jj = 0; jj < w; ++jj) {
                const Acc ljj = D[jj][jj];
                if (ljj == Acc(0) || !isfinite(ljj)) {
                    report(c, seq, uint64_t(J + jj));
                    break;
                }
            }
        if (threadIdx.x == 0 && blockIdx.x == 0) { const long long t = clock64(); g_leaf_clk[4] += t - t_tr; t_tr = t; }
        Acc x[PW];
        if (live) {
#pragma unroll
            for (int jj = 0; jj < PW; ++jj) {
                if (jj < w) {
                    asm volatile("" ::: "memory");  // keep D loads in their iteration
                    const Acc v = rnd<L>(getx(J + jj) - acc[jj]);  // rn_level(rn_acc(c - s))
                    x[jj] = rnd<L>(v / D[jj][jj]);
#pragma unroll
                    for (int j2 = jj + 1; j2 < PW; ++j2) acc[j2] = fma(x[jj], D[jj][j2], acc[j2]);
                    if (chk_seq && !isfinite(x[jj])) {
                        const unsigned long long k =
                            fail_key(chk_seq, elem_local(br0 + i - chk_r0, bc0 + J + jj - chk_c0));
                        bad = k < bad ? k : bad;
                    }
                }
            }
        }
        __syncwarp();  // every quad lane has read its row's [J, J+w) before lane 0 stores
        if (live && q == 0)
#pragma unroll
            for (int jj = 0; jj < PW; ++jj)
                if (jj < w) {
                    if constexpr (BS) Bs[r * ldb + J + jj] = x[jj];
                    else row[J + jj] = from_double<T>(double(x[jj]));
                }
        __syncwarp();
        if (threadIdx.x == 0 && blockIdx.x == 0) { const long long t = clock64(); g_leaf_clk[5] += t - t_tr; t_tr = t; }
    }
    if constexpr (BS) {
        __syncthreads();
        const int rows = min(TRSM_ROWS, m - i0);
        for (int rr = threadIdx.x >> 5; rr < rows; rr += 4)
            for (int t = threadIdx.x & 31; t < n; t += 32)
                Bg[(long long)(i0 + rr) * c.ldw + t] = from_double<T>(double(Bs[rr * ldb + t]));
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&g_leaf_clk[7]), 1ull);
    if (chk_seq) warp_report_min(c, bad);
}

// W = inv(rn16(L)) for one leaf (L the F16-level copy: the leaf itself or its
// shadow), FP32 arithmetic, written as an FP16 pair W*2^e = hi + lo into the
// W16 workspace (row r0+i: hi at [0,n), lo at [kW16Lo, kW16Lo+n)); 2^-e goes
// to wscale[r0].  Column t of W is a forward substitution L w = e_t that only
// reads L and its own earlier entries, so columns are independent: a quad of
// threads per column splits each dot product.  CTA = 32 columns.
// Also the singular-diagonal check of the first solve against this leaf
// (kernels.cpp:79-81: rn16(l(j,j)) zero or non-finite).
constexpr int INV_COLS = 32;

__global__ void __launch_bounds__(128) k_leaf_inverse(DevCtx c, int r0, int n, uint32_t seq) {
    pdl_wait();
    extern __shared__ __align__(16) float inv_smem[];
    float* Ls = inv_smem;                          // packed lower triangle, n(n+1)/2
    float* Wc = Ls + (n * (n + 1)) / 2;            // [INV_COLS][n] this CTA's columns
    __shared__ float colmax[INV_COLS];
    const __half* g = c.b16 + (long long)r0 * c.ldw + r0;
    const int c0 = blockIdx.x * INV_COLS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = c0 + warp; i < n; i += 4)
        for (int j = c0 + lane; j <= i; j += 32) Ls[(i * (i + 1)) / 2 + j] = __half2float(g[(long long)i * c.ldw + j]);
    __syncthreads();
    const int q = threadIdx.x & 3;
    const int tl = threadIdx.x >> 2;  // local column
    const int t = c0 + tl;
    const bool live = t < n;
    float amax = 0.f;
    if (threadIdx.x == 0)
        for (int j = c0; j < min(n, c0 + INV_COLS); ++j) {
            const float d = Ls[(j * (j + 1)) / 2 + j];
            if (d == 0.f || !isfinite(d)) {
                report(c, seq, uint64_t(j));
                break;
            }
        }
    for (int i = c0; i < n; ++i) {
        float s = 0.f;
        if (live && i > t) {
            const float* Li = Ls + (i * (i + 1)) / 2;
            const float* Wt = Wc + tl * n;
            for (int k = t + q; k < i; k += 4) s = fmaf(Li[k], Wt[k], s);
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (live && i >= t) {
            const float lii = Ls[(i * (i + 1)) / 2 + i];
            const float w = i == t ? 1.0f / lii : -s / lii;
            if (q == 0) Wc[tl * n + i] = w;
            amax = fmaxf(amax, fabsf(w));
        }
        __syncwarp();
    }
    if (q == 0 && tl < INV_COLS) colmax[tl] = live ? amax : 0.f;
    __syncthreads();
    // per-leaf scale: all CTAs of the leaf must agree, so it is derived from
    // the diagonal (|W(t,t)| = 1/|L(t,t)| dominates a diagonally dominant
    // leaf) of the whole leaf, not from this CTA's columns
    float dmax = 0.f;  // from global: this CTA only staged rows/cols >= c0
    for (int j = lane; j < n; j += 32) dmax = fmaxf(dmax, fabsf(1.0f / __half2float(g[(long long)j * c.ldw + j])));
#pragma unroll
    for (int o = 16; o; o >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    int e = 0;
    if (dmax > 0.f && isfinite(dmax)) (void)frexpf(dmax, &e);  // dmax = f * 2^e, f in [0.5, 1)
    const float up = ldexpf(1.0f, -e), down = ldexpf(1.0f, e);
    if (blockIdx.x == 0 && threadIdx.x == 0) c.wscale[r0] = down;
    __half* W = c.w16 + (long long)r0 * kW16Ld;
    // write rows i = 0..n-1 of this CTA's columns: hi, lo (upper part zero)
    for (int e2 = threadIdx.x; e2 < n * INV_COLS; e2 += 128) {
        const int i = e2 / INV_COLS, tc = e2 % INV_COLS, tt = c0 + tc;
        if (tt >= n) continue;
        const float w = i >= tt ? Wc[tc * n + i] * up : 0.f;
        const __half hi = __float2half_rn(w);
        const __half lo = __float2half_rn(w - __half2float(hi));
        W[(long long)i * kW16Ld + tt] = hi;
        W[(long long)i * kW16Ld + kW16Lo + tt] = lo;
    }
}

size_t inverse_smem(int n) { return (size_t(n) * (n + 1) / 2 + size_t(INV_COLS) * n) * sizeof(float); }

template <int L, bool SMEM>
void potrf_launch(const DevCtx& c, int r0, int n, uint32_t seq, uint32_t chk, cudaStream_t s) {
    using Acc = typename LvT<L>::Acc;
    const size_t smem = potrf_smem<Acc>(n, SMEM);
    k_potrf_leaf<L, SMEM><<<1, POTRF_THREADS, smem, s>>>(c, r0, n, seq, chk);
}

}  // namespace

void launch_leaf_inverse(const DevCtx& c, int r0, int n, uint32_t seq, cudaStream_t s) {
    k_leaf_inverse<<<(n + INV_COLS - 1) / INV_COLS, 128, inverse_smem(n), s>>>(c, r0, n, seq);
}

void init_trsm_attributes();

void init_leaf_attributes() {
    const int cap = 227 * 1024;
    init_leaf_cm_attributes();
    init_potrf_v2_attributes();
    init_inv2_attributes();
    init_trsm_attributes();
    cudaFuncSetAttribute(k_leaf_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_leaf<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_leaf<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_leaf<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_leaf<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_leaf<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_leaf<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
    cudaFuncSetAttribute(k_potrf_f64, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
}

constexpr size_t kLeafSmemCap = 220 * 1024;

void launch_potrf_leaf(const DevCtx& c, int lv, int r0, int n, uint32_t seq, uint32_t chk, cudaStream_t s,
                       uint32_t inv_seq, int fuse_inv, int shadow16) {
    if (potrf_v2_ok(lv, n)) return launch_potrf_v2(c, lv, r0, n, seq, chk, s, inv_seq, fuse_inv, shadow16);
    if (leaf_cm_ok(lv, n)) return launch_potrf_cm(c, lv, r0, n, seq, chk, s);
    const bool d = lv == LV_F64;
    if (d && n % 32 == 0 && n > 128 && n <= 256 && (c.ldw % 2) == 0 && (r0 % 2) == 0) {
        // FP64 leaves whose triangle does not fit shared memory (C2's 256):
        // the DMMA kernel (a 227k -> 153k cycles, b2 245k -> 69k, b1 105k ->
        // 349k -- net even, 323 vs 327 us).  Smaller leaves (C1's 128) keep
        // the shared-memory SIMT kernel, 1.09 vs 1.52 ms for C1.
        k_potrf_f64<<<1, F64T, potrf_f64_smem(n), s>>>(c, r0, n, seq, chk);
        return;
    }
    const bool fits = (d ? potrf_smem<double>(n, true) : potrf_smem<float>(n, true)) <= kLeafSmemCap;
    const bool pfits = (d ? potrf_smem<double>(n, false) : potrf_smem<float>(n, false)) <= kLeafSmemCap;
    if (!pfits) {
        // the partial-sum panel alone exceeds shared memory: n > ~860 (F64)
        // -- not reachable with the supported leaf sizes; guard anyway
        return;
    }
    switch (lv) {
        case LV_F16: fits ? potrf_launch<0, true>(c, r0, n, seq, chk, s) : potrf_launch<0, false>(c, r0, n, seq, chk, s); break;
        case LV_F32: fits ? potrf_launch<1, true>(c, r0, n, seq, chk, s) : potrf_launch<1, false>(c, r0, n, seq, chk, s); break;
        default: fits ? potrf_launch<2, true>(c, r0, n, seq, chk, s) : potrf_launch<2, false>(c, r0, n, seq, chk, s); break;
    }
}

constexpr size_t kTrsmRowsSmemCap = 100 * 1024;

template <int L>
void trsm_launch(const DevCtx& c, int br0, int bc0, int m, int n, int lr0, uint32_t seq, uint32_t chk_seq,
                 int chk_r0, int chk_c0, cudaStream_t s) {
    using Acc = typename LvT<L>::Acc;
    const int grid = (m + TRSM_ROWS - 1) / TRSM_ROWS;
    const size_t rows_smem = size_t(TRSM_ROWS) * (n + 1) * sizeof(Acc);
    if (rows_smem <= kTrsmRowsSmemCap)
        k_trsm_leaf<L, true><<<grid, 128, rows_smem, s>>>(c, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0);
    else
        k_trsm_leaf<L, false><<<grid, 128, 0, s>>>(c, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0);
}

void init_trsm_attributes() {
    cudaFuncSetAttribute(k_trsm_leaf<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmRowsSmemCap);
    cudaFuncSetAttribute(k_trsm_leaf<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmRowsSmemCap);
    cudaFuncSetAttribute(k_trsm_leaf<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTrsmRowsSmemCap);
}

void launch_trsm_leaf(const DevCtx& c, int lv, int br0, int bc0, int m, int n, int lr0, uint32_t seq,
                      uint32_t chk_seq, int chk_r0, int chk_c0, cudaStream_t s) {
    if (m <= 0) return;
    if (leaf_cm_ok(lv, n)) return launch_trsm_cm(c, lv, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0, s);
    switch (lv) {
        case LV_F16: trsm_launch<0>(c, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0, s); break;
        case LV_F32: trsm_launch<1>(c, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0, s); break;
        default: trsm_launch<2>(c, br0, bc0, m, n, lr0, seq, chk_seq, chk_r0, chk_c0, s); break;
    }
}

}  // namespace tcb

namespace tcb {
// debug: accumulated potrf-leaf phase cycles since the last call (a, b1, b2, launches)
void leaf_debug_clocks(long long* out, bool reset) {
    cudaMemcpyFromSymbol(out, g_leaf_clk, sizeof(long long) * 8);
    if (reset) {
        long long z[8] = {0};
        cudaMemcpyToSymbol(g_leaf_clk, z, sizeof(z));
    }
}
}  // namespace tcb
