// k_verify.cu -- accuracy metrics and the solve, all FP64 on the device.
//
//   fact_error   ||A - L L^T||_F / ||A||_F over the symmetric matrix
//                (factorization_error, analysis.cpp:30-62): lower triangles
//                only, weight 2 off the diagonal, NaN on non-finite input.
//                64x64 lower tiles of E = A - L L^T; per-tile partial sums
//                reduced in a fixed order (deterministic).
//   potrs        L y = b then L^T x = y (no reference counterpart; SURVEY
//                8(a) row 25).  Bandwidth-bound wavefront: one CTA per
//                64-row block, blocks claim logical indices from an atomic
//                ticket so a block only ever waits on blocks already
//                running; finished blocks publish a flag.  L is streamed
//                once per direction with coalesced column reads.
//   residual     ||b - A x||_2 / (||A||_F ||x||_2 + ||b||_2), A symmetric
//                with only its lower triangle read.
#include <string>

#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

constexpr int VT = 64;  // tile / block size

// ---------------------------------------------------------------- fact_error
__global__ void __launch_bounds__(256) k_fact_error(int n, const double* __restrict__ A, long long lda,
                                                    const double* __restrict__ Lm, long long ldl, double* partials,
                                                    int* nonfinite, int T) {
    // tile index -> (I, J), I >= J, row-major over the lower tile triangle
    const int t = blockIdx.x;
    int I = int((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    const int J = t - I * (I + 1) / 2;
    const int i0 = I * VT, j0 = J * VT;
    __shared__ double Li[16][VT + 1];
    __shared__ double Lj[16][VT + 1];
    __shared__ double red[2][8];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 4x4 each
    double acc[4][4] = {};
    const int kmax = min(j0 + VT, n);  // k <= j <= i for lower elements
    for (int k0 = 0; k0 < kmax; k0 += 16) {
        for (int e = threadIdx.x; e < 16 * VT; e += 256) {
            const int r = e % VT, kk = e / VT;
            const int k = k0 + kk, gi = i0 + r, gj = j0 + r;
            Li[kk][r] = (gi < n && k < n && k <= gi) ? Lm[(long long)k * ldl + gi] : 0.0;
            Lj[kk][r] = (gj < n && k < n && k <= gj) ? Lm[(long long)k * ldl + gj] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) a[x] = Li[kk][ty * 4 + x];
#pragma unroll
            for (int y = 0; y < 4; ++y) b[y] = Lj[kk][tx * 4 + y];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
        }
        __syncthreads();
    }
    double num = 0.0, den = 0.0;
    int bad = 0;
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int i = i0 + ty * 4 + x, j = j0 + tx * 4 + y;
            if (i >= n || j > i) continue;
            const double a = A[(long long)j * lda + i];
            const double l = Lm[(long long)j * ldl + i];
            if (!isfinite(a) || !isfinite(l)) bad = 1;
            const double e = a - acc[x][y];
            const double w = i == j ? 1.0 : 2.0;
            num += w * e * e;
            den += w * a * a;
        }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = num;
        red[1][threadIdx.x >> 5] = den;
    }
    if (bad && (threadIdx.x & 31) == 0) atomicExch(nonfinite, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < 8; ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
        }
        partials[2 * t] = s0;
        partials[2 * t + 1] = s1;
    }
}

__global__ void k_fact_error_final(const double* partials, int count, const int* nonfinite, double* out) {
    __shared__ double s0[256], s1[256];
    double a = 0.0, b = 0.0;
    for (int t = threadIdx.x; t < count; t += 256) {
        a += partials[2 * t];
        b += partials[2 * t + 1];
    }
    s0[threadIdx.x] = a;
    s1[threadIdx.x] = b;
    __syncthreads();
    for (int w = 128; w; w >>= 1) {
        if (threadIdx.x < w) {
            s0[threadIdx.x] += s0[threadIdx.x + w];
            s1[threadIdx.x] += s1[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = *nonfinite ? __longlong_as_double(0x7ff8000000000000ll) : sqrt(s0[0] / s1[0]);
}

// ---------------------------------------------------------------- potrs
// The solves of a set of problems (system s, right-hand side r) -- one, or
// a whole batch in one launch.  System s: factor Ls[s] (ld ldl), right-hand
// sides Bs[s] + r*ldb; tables null: the single system L0 / B0.
struct PotrsArgs {
    int n, nsys, nrhs;
    const double* const* Ls;
    double* const* Bs;
    const double* L0;
    double* B0;
    long long ldl, ldb;
    int* ticket;  // one word per direction: the next (block, problem) pair
    double* W;    // [system][nb][VT][VT] diagonal-block inverses
    // published y / x per problem ([problem][nb * VT]), pre-filled with the
    // sentinel: a consumer polls the values it needs until they are real
    double* Yw;
    double* Xw;
    int poll;     // 0: every thread polls its values; >0: with that ns backoff;
                  // -1: warp 0 polls the whole block, then a CTA barrier
};

// "not yet written" marker of Yw / Xw: a NaN bit pattern no arithmetic
// produces; a computed value with exactly these bits is stored as the
// canonical NaN instead (publish), so the marker never means data
constexpr unsigned long long kPotrsPending = 0xFFFFFFFFFFFFFFFFull;
__device__ __forceinline__ void publish(double* p, double v) {
    if (static_cast<unsigned long long>(__double_as_longlong(v)) == kPotrsPending) v = __longlong_as_double(0x7ff8000000000000ll);
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ bool pending(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v)) == kPotrsPending;
}
__device__ __forceinline__ double2 ld_relaxed2(const double* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}
// spin until the published value at p is real (relaxed, L2-coherent reads);
// backoff > 0: sleep that many ns between polls
__device__ __forceinline__ double await_value(const double* p, int backoff) {
    for (;;) {
        const double v = ld_relaxed(p);
        if (!pending(v)) return v;
        if (backoff) __nanosleep(backoff);
    }
}
__device__ __forceinline__ const double* potrs_L(const PotrsArgs& a, int s) { return a.Ls ? a.Ls[s] : a.L0; }
__device__ __forceinline__ double* potrs_B(const PotrsArgs& a, int s) { return a.Bs ? a.Bs[s] : a.B0; }

// diagonal-block inverses W_I = inv(L(I,I)) (64 x 64, row-major), one CTA
// per (block, system), one thread per column (independent forward
// substitutions): they take the 64-step dependent solve off the block chain
// of the substitutions below
__global__ void __launch_bounds__(VT) k_potrs_diaginv(PotrsArgs a) {
    __shared__ double Ls[VT][VT + 1];
    const int n = a.n, nb = (n + VT - 1) / VT;
    const int I = blockIdx.x, sys = blockIdx.y, i0 = I * VT, rows = min(VT, n - i0), t = threadIdx.x;
    const double* Lm = potrs_L(a, sys);
    const long long ldl = a.ldl;
    for (int c = 0; c < VT; ++c) Ls[t][c] = (t < rows && c < rows && t >= c) ? Lm[(long long)(i0 + c) * ldl + i0 + t] : 0.0;
    __syncthreads();
    double* Wi = a.W + (size_t(sys) * nb + I) * VT * VT;
    double w[VT];
#pragma unroll
    for (int i = 0; i < VT; ++i) {
        double s = (i == t) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < i; ++k) s = fma(-Ls[i][k], w[k], s);
        w[i] = (i >= t && i < rows) ? s / Ls[i][i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < VT; ++i) Wi[i * VT + t] = w[i];
}

// forward y = L^-1 b / backward x = L^-T y.  Persistent CTAs claim tickets
// t -> (block index t / P, problem t % P): every problem's blocks are claimed
// in chain order, so a CTA only ever waits on blocks already claimed by
// running CTAs.  Block I accumulates L(I,J) y_J (forward) or L(J,I)^T x_J
// (backward) over J in chain order -- the L tile of the next J is in flight
// while the threads wait for the current one -- then y_I = W_I (b_I - sum) /
// x_I = W_I^T (y_I - sum): a 64x64 product from shared memory (W_I staged off
// the chain), no dependent chain.
//
// Links carry no flags or fences: a finished block publishes its 64 values
// into a sentinel-filled buffer (Yw forward, Xw backward) and each consumer
// thread polls exactly the values it multiplies, all of them in flight at
// once (16-byte relaxed L2 loads), so one store-to-load trip through L2 is
// the whole link.  The forward sweep writes y to Yw only; the backward sweep
// reads y from Yw and writes x to B (the result) and Xw (for its consumers).
// (Measured alternatives: one flag per block behind a fence, 1.6 ms per
// N=16384 solve; polling with nanosleep backoff or by one warp behind a CTA
// barrier, 1.5-1.8 ms; precomputing W_I L(I,I-1) so the last link is a bare
// matvec, 1.8 ms (the 64^3 product per block costs more than it saves);
// this form, 1.0 ms.)
//
// HBM access (L read once per sweep, n(n+1)/2 * 8 bytes): every
// warp load instruction reads 512 contiguous bytes of one column of L as 16-
// byte vectors.  Forward: the block's rows are contiguous within a column, so
// lanes run along the rows (thread = 2 rows x 8 columns of the 64-wide tile).
// Backward: the tile L(J, I) is read along its columns too -- lanes run along
// J's rows (k), each warp owns 8 of I's columns and reduces them with
// shuffles at the end -- instead of striding by ldl across lanes.
constexpr int VP = VT + 2;  // padded smem row (16-byte aligned)

template <bool BWD>
__global__ void __launch_bounds__(256, 2) k_potrs_sweep(PotrsArgs a) {
    const int n = a.n, nb = (n + VT - 1) / VT, P = a.nsys * a.nrhs;
    const long long ldp = (long long)nb * VT;  // Yw / Xw stride per problem
    extern __shared__ __align__(16) double sm[];
    double(*Ws)[VP] = reinterpret_cast<double(*)[VP]>(sm);  // W_I
    double(*part)[VT] = reinterpret_cast<double(*)[VT]>(sm + VT * VP);
    double* rhs = sm + VT * VP + 8 * VT;
    int* sT = reinterpret_cast<int*>(rhs + VT);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // forward: rows 2*rp, 2*rp+1 of the block x columns kq*8 .. +8 of a tile;
    // backward: rows 2*lane, 2*lane+1 of tile J x columns warp*8 .. +8 of block I
    const int rp = tid & 31, kq = tid >> 5;
    const long long ldl = a.ldl;
    const int bo = a.poll > 0 ? a.poll : 0;
    for (;;) {
        if (tid == 0) *sT = atomicAdd(a.ticket, 1);
        __syncthreads();
        const int t = *sT;
        if (t >= nb * P) break;
        const int p = t % P, sys = p / a.nrhs, rr = p % a.nrhs;
        const int I = BWD ? nb - 1 - t / P : t / P;
        const double* __restrict__ Lm = potrs_L(a, sys);
        double* bx = potrs_B(a, sys) + rr * a.ldb;  // b (forward input) / x (backward output)
        double* Y = a.Yw + p * ldp;
        double* X = a.Xw + p * ldp;
        const double* src = BWD ? X : Y;            // the values this sweep consumes
        const int i0 = I * VT, rows = min(VT, n - i0);
        const bool vec = ((ldl & 1) == 0) && ((reinterpret_cast<uintptr_t>(Lm) & 15) == 0);
        // this block's own right-hand side (b_I, or y_I from the forward sweep)
        const double own = tid < rows ? (BWD ? __ldcg(Y + i0 + tid) : __ldcg(bx + i0 + tid)) : 0.0;
        // W_I into shared memory (off the chain; read after the last wait)
        {
            const double* Wi = a.W + (size_t(sys) * nb + I) * VT * VT;
            for (int e = tid; e < VT * VT / 2; e += 256) {
                const double2 w = reinterpret_cast<const double2*>(Wi)[e];
                const int r = (2 * e) / VT, c = (2 * e) % VT;
                *reinterpret_cast<double2*>(&Ws[r][c]) = w;
            }
        }
        const int nsteps = BWD ? nb - 1 - I : I;
        // one 64x64 tile of L as 8 double2 per thread
        auto load_tile = [&](int J, double2* lv) {
            const int k0 = J * VT;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                // forward: L(i0 + 2rp + {0,1}, k0 + kq*8 + kk); backward: L(k0 + 2lane + {0,1}, i0 + warp*8 + kk)
                const int row = BWD ? k0 + 2 * lane : i0 + 2 * rp;
                const int col = BWD ? i0 + warp * 8 + kk : k0 + kq * 8 + kk;
                const double* q = Lm + (long long)col * ldl + row;
                if (col < n && row + 1 < n && vec) {
                    lv[kk] = __ldcs(reinterpret_cast<const double2*>(q));
                } else {
                    lv[kk].x = (col < n && row < n) ? __ldcs(q) : 0.0;
                    lv[kk].y = (col < n && row + 1 < n) ? __ldcs(q + 1) : 0.0;
                }
            }
        };
        double acc0 = 0.0, acc1 = 0.0;  // forward: rows 2rp, 2rp+1
        double accb[8];                 // backward: columns warp*8 + kk
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) accb[kk] = 0.0;
        double2 cur[8], nxt[8];
        if (nsteps > 0) load_tile(BWD ? nb - 1 : 0, cur);
        for (int step = 0; step < nsteps; ++step) {
            const int J = BWD ? nb - 1 - step : step;
            if (step + 1 < nsteps) load_tile(BWD ? J - 1 : J + 1, nxt);
            const int k0 = J * VT;
            if (!BWD) {
                double yk[8];
                const int kb = k0 + kq * 8;  // a full block (only the last block is ragged)
                for (;;) {
                    bool wait = false;
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const double2 v = ld_relaxed2(src + kb + 2 * h);
                        yk[2 * h] = v.x;
                        yk[2 * h + 1] = v.y;
                        wait |= pending(v.x) | pending(v.y);
                    }
                    if (!wait) break;
                    if (bo) __nanosleep(bo);
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    acc0 = fma(cur[kk].x, yk[kk], acc0);
                    acc1 = fma(cur[kk].y, yk[kk], acc1);
                }
            } else {
                const int k = k0 + 2 * lane;
                double x0, x1;
                if (k + 1 < n) {
                    for (;;) {
                        const double2 v = ld_relaxed2(src + k);
                        x0 = v.x;
                        x1 = v.y;
                        if (!(pending(x0) | pending(x1))) break;
                        if (bo) __nanosleep(bo);
                    }
                } else {
                    x0 = k < n ? await_value(src + k, bo) : 0.0;
                    x1 = 0.0;
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) accb[kk] = fma(cur[kk].y, x1, fma(cur[kk].x, x0, accb[kk]));
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) cur[kk] = nxt[kk];
        }
        if (!BWD) {
            part[kq][2 * rp] = acc0;
            part[kq][2 * rp + 1] = acc1;
        } else {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                double v = accb[kk];
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) part[0][warp * 8 + kk] = v;
            }
        }
        __syncthreads();
        if (tid < VT) {
            double sum = 0.0;
            if (!BWD) {
#pragma unroll
                for (int g = 0; g < 8; ++g) sum += part[g][tid];
            } else {
                sum = part[0][tid];
            }
            rhs[tid] = tid < rows ? own - sum : 0.0;
        }
        __syncthreads();
        // y_I = W_I rhs (forward) / x_I = W_I^T rhs (backward); thread: rows
        // 2rp, 2rp+1, terms kq*8 .. +8
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const int c = kq * 8 + kk;
            const double r = rhs[c];
            s0 = fma(BWD ? Ws[c][2 * rp] : Ws[2 * rp][c], r, s0);
            s1 = fma(BWD ? Ws[c][2 * rp + 1] : Ws[2 * rp + 1][c], r, s1);
        }
        __syncthreads();
        part[kq][2 * rp] = s0;
        part[kq][2 * rp + 1] = s1;
        __syncthreads();
        if (tid < rows) {
            double v = 0.0;
#pragma unroll
            for (int g = 0; g < 8; ++g) v += part[g][tid];
            if (BWD) {
                bx[i0 + tid] = v;
                publish(X + i0 + tid, v);
            } else {
                publish(Y + i0 + tid, v);
            }
        }
    }
}

constexpr size_t kSweepSmem = sizeof(double) * (VT * VP + 8 * VT + VT) + 16;

// ---------------------------------------------------------------- residual
// per 64-row block I: r_I = b_I - sum_J A(I,J) x_J with A(I,J) = A(J,I)^T above
__global__ void __launch_bounds__(256) k_residual(int n, const double* __restrict__ A, long long lda,
                                                  const double* __restrict__ X, const double* __restrict__ Bv,
                                                  double* partials) {
    const int I = blockIdx.x, i0 = I * VT;
    const int r = threadIdx.x & 63, q = threadIdx.x >> 6;
    const int gi = i0 + r;
    __shared__ double part[4][VT];
    __shared__ double red[4][8];
    double acc = 0.0, anorm = 0.0;
    if (gi < n)
        for (int j = q; j < n; j += 4) {
            // lower element A(max, min)
            const double a = j <= gi ? A[(long long)j * lda + gi] : A[(long long)gi * lda + j];
            acc = fma(a, X[j], acc);
            if (j <= gi) anorm += (j == gi ? 1.0 : 2.0) * a * a;
        }
    part[q][r] = acc;
    __syncthreads();
    double rr = 0.0, xx = 0.0, bb = 0.0, aa = anorm;
    if (threadIdx.x < VT && gi < n) {
        const double ax = part[0][r] + part[1][r] + part[2][r] + part[3][r];
        const double res = Bv[gi] - ax;
        rr = res * res;
        xx = X[gi] * X[gi];
        bb = Bv[gi] * Bv[gi];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        rr += __shfl_xor_sync(0xffffffffu, rr, o);
        xx += __shfl_xor_sync(0xffffffffu, xx, o);
        bb += __shfl_xor_sync(0xffffffffu, bb, o);
        aa += __shfl_xor_sync(0xffffffffu, aa, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = rr;
        red[1][threadIdx.x >> 5] = xx;
        red[2][threadIdx.x >> 5] = bb;
        red[3][threadIdx.x >> 5] = aa;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += red[threadIdx.x][w];
        partials[4 * I + threadIdx.x] = s;
    }
}

__global__ void k_residual_final(const double* partials, int count, double* out) {
    if (threadIdx.x != 0) return;
    double s[4] = {0, 0, 0, 0};
    for (int t = 0; t < count; ++t)
        for (int k = 0; k < 4; ++k) s[k] += partials[4 * t + k];
    *out = sqrt(s[0]) / (sqrt(s[3]) * sqrt(s[1]) + sqrt(s[2]));
}

}  // namespace

int fact_error_partials(int n, int* tiles_per_side) {
    const int T = (n + VT - 1) / VT;
    *tiles_per_side = T;
    return T * (T + 1) / 2;
}

void launch_fact_error(int n, const double* dA, long long lda, const double* dL, long long ldl, double* d_partials,
                       int* d_nonfinite, int T, cudaStream_t s) {
    const int tiles = T * (T + 1) / 2;
    cudaMemsetAsync(d_nonfinite, 0, sizeof(int), s);
    k_fact_error<<<tiles, 256, 0, s>>>(n, dA, lda, dL, ldl, d_partials, d_nonfinite, T);
    k_fact_error_final<<<1, 256, 0, s>>>(d_partials, tiles, d_nonfinite, d_partials + 2 * size_t(tiles));
}

size_t potrs_work_doubles(int n, int nrhs) { return potrs_batch_work_bytes(n, 1, nrhs) / sizeof(double) + 1; }

// workspace of nsys systems: W, Yw, Xw, then the two tickets
size_t potrs_batch_work_bytes(int n, int nsys, int nrhs) {
    const size_t nb = size_t((n + VT - 1) / VT);
    return sizeof(double) * (size_t(nsys) * nb * VT * VT + 2 * size_t(nsys) * size_t(nrhs) * nb * VT) +
           2 * sizeof(int);
}

static int g_potrs_poll = 0;

bool potrs_set_option(const std::string& key, int value) {
    if (key == "potrs_poll") {
        g_potrs_poll = value;
        return true;
    }
    return false;
}

static void potrs_run(PotrsArgs a, void* work, int max_ctas, cudaStream_t s) {
    static const bool attr = [] {
        cudaFuncSetAttribute(k_potrs_sweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSweepSmem));
        cudaFuncSetAttribute(k_potrs_sweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSweepSmem));
        return true;
    }();
    (void)attr;
    a.poll = g_potrs_poll;
    const int nb = (a.n + VT - 1) / VT;
    const size_t pub = size_t(a.nsys) * size_t(a.nrhs) * size_t(nb) * VT;  // doubles per published buffer
    a.W = static_cast<double*>(work);
    a.Yw = a.W + size_t(a.nsys) * nb * VT * VT;
    a.Xw = a.Yw + pub;
    int* words = reinterpret_cast<int*>(a.Xw + pub);
    k_potrs_diaginv<<<dim3(nb, a.nsys), VT, 0, s>>>(a);
    const long long work_items = (long long)nb * a.nsys * a.nrhs;
    const int g = int(max_ctas > 0 && max_ctas < work_items ? max_ctas : work_items);
    cudaMemsetAsync(a.Yw, 0xFF, 2 * pub * sizeof(double), s);  // kPotrsPending
    cudaMemsetAsync(words, 0, 2 * sizeof(int), s);
    a.ticket = words;
    k_potrs_sweep<false><<<g, 256, kSweepSmem, s>>>(a);
    a.ticket = words + 1;
    k_potrs_sweep<true><<<g, 256, kSweepSmem, s>>>(a);
}

void launch_potrs(int n, const double* dL, long long ldl, double* dB, long long ldb, int nrhs, int* /*d_counters*/,
                  double* d_work, cudaStream_t s, int max_ctas) {
    PotrsArgs a{};
    a.n = n;
    a.nsys = 1;
    a.nrhs = nrhs;
    a.L0 = dL;
    a.B0 = dB;
    a.ldl = ldl;
    a.ldb = ldb;
    potrs_run(a, d_work, max_ctas, s);
}

void launch_potrs_batch(int n, int nsys, const double* const* d_Ltab, long long ldl, double* const* d_Btab,
                        long long ldb, int nrhs, void* d_work, int max_ctas, cudaStream_t s) {
    PotrsArgs a{};
    a.n = n;
    a.nsys = nsys;
    a.nrhs = nrhs;
    a.Ls = d_Ltab;
    a.Bs = d_Btab;
    a.ldl = ldl;
    a.ldb = ldb;
    potrs_run(a, d_work, max_ctas, s);
}

int residual_partials(int n) { return (n + VT - 1) / VT; }

void launch_residual(int n, const double* dA, long long lda, const double* dX, const double* dB, double* d_partials,
                     cudaStream_t s) {
    const int nb = (n + VT - 1) / VT;
    k_residual<<<nb, 256, 0, s>>>(n, dA, lda, dX, dB, d_partials);
    k_residual_final<<<1, 32, 0, s>>>(d_partials, nb, d_partials + 4 * size_t(nb));
}

}  // namespace tcb
