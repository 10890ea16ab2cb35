// device.cuh -- structures and numerics shared by every sm_100a kernel.
//
// Storage layout in HBM: each precision level has
// its own ROW-MAJOR n x ldw buffer (element (i,j) at buf[i*ldw + j]).  Row
// major turns every update of the algorithm, C -= A * B^T with A, B row
// blocks of the one lower-triangular matrix, into a GEMM whose operands are
// both K-major -- the native tcgen05 / TMA SWIZZLE_128B layout.  A block
// lives in the buffer of its level; a final L block read by a lower-level
// TRSM additionally gets a rounded copy in that level's buffer (planner
// OP_SHADOW).  The caller's column-major doubles are touched only by
// import / quantize (read) and export (write).
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace tcb {

// per-launch pointers to the caller's matrix (read through one indirection
// so a captured CUDA graph serves every call of a plan)
struct RunArgs {
    const double* a_in;
    double* l_out;
    long long lda_in;
    long long lda_out;
};

struct DevCtx {
    __half* b16;   // F16 level buffer (row-major, ld = ldw)
    float* b32;    // F32 level buffer
    double* b64;   // F64 level buffer
    long long ldw;
    const RunArgs* ra;
    unsigned long long* status;      // first failure key (atomicMin)
    unsigned long long* alpha_bits;  // per quantize slot: bits of max|B| (atomicMax)
    __half* w16;      // leaf inverses, hi | lo (ld kW16Ld), for inverse FP16 solves
    float* wscale;    // per leaf (indexed by its first row): 2^-e the W16 entries carry
    float* w32;       // FP32 leaf inverses (ld kW32Ld), for inverse FP32 solves
    unsigned long long* stamps;  // development: %globaltimer stamps of CTA 0 (null = off)
    // first allocated row of each level buffer (b16/b32/b64 are virtual bases:
    // rows below are never accessed, but TMA descriptors need real addresses)
    int win_lo[3];
};

// failure key: seq in the high 24 bits, a position inside the op below.
// Smaller key == earlier in the reference's sequential order.
__host__ __device__ inline unsigned long long fail_key(uint32_t seq, uint64_t local) {
    return (uint64_t(seq) << 40) | (local & ((1ull << 40) - 1));
}
// element (i, j) of a block, first in column-major order (tree.cpp:20-21)
__host__ __device__ inline uint64_t elem_local(int i, int j) {
    return (uint64_t(j) << 20) | uint64_t(i);
}

#ifdef __CUDACC__
__device__ inline void report(const DevCtx& c, uint32_t seq, uint64_t local) {
    atomicMin(c.status, fail_key(seq, local));
}

// ---------------------------------------------------------------------------
// level types and rounding (precision.hpp:41-76)
// ---------------------------------------------------------------------------

template <int L> struct LvT;
template <> struct LvT<0> { using T = __half; using Acc = float; };
template <> struct LvT<1> { using T = float; using Acc = float; };
template <> struct LvT<2> { using T = double; using Acc = double; };

// binary16 round-to-nearest-even directly from double: one rounding, overflow
// to +-inf, half subnormals kept, double subnormals to signed zero -- the
// exact contract of round_to_half (precision.hpp:41-62).  No FP32 hop.
__device__ __forceinline__ __half d2h(double x) {
    unsigned short r;
    asm("cvt.rn.f16.f64 %0, %1;" : "=h"(r) : "d"(x));
    return __ushort_as_half(r);
}
__device__ __forceinline__ __half f2h(float x) { return __float2half_rn(x); }

template <typename T> __device__ __forceinline__ T from_double(double x);
template <> __device__ __forceinline__ __half from_double<__half>(double x) { return d2h(x); }
template <> __device__ __forceinline__ float from_double<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ double from_double<double>(double x) { return x; }

template <typename T> __device__ __forceinline__ T from_float(float x);
template <> __device__ __forceinline__ __half from_float<__half>(float x) { return f2h(x); }
template <> __device__ __forceinline__ float from_float<float>(float x) { return x; }
template <> __device__ __forceinline__ double from_float<double>(float x) { return double(x); }

__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ double to_d(__half x) { return double(__half2float(x)); }
__device__ __forceinline__ double to_d(float x) { return double(x); }
__device__ __forceinline__ double to_d(double x) { return x; }

// round an accumulator-type value to level L, staying in Acc
template <int L> __device__ __forceinline__ typename LvT<L>::Acc rnd(typename LvT<L>::Acc v);
template <> __device__ __forceinline__ float rnd<0>(float v) { return __half2float(f2h(v)); }
template <> __device__ __forceinline__ float rnd<1>(float v) { return v; }
template <> __device__ __forceinline__ double rnd<2>(double v) { return v; }

template <int L> __device__ __forceinline__ typename LvT<L>::T* lvbuf(const DevCtx& c);
template <> __device__ __forceinline__ __half* lvbuf<0>(const DevCtx& c) { return c.b16; }
template <> __device__ __forceinline__ float* lvbuf<1>(const DevCtx& c) { return c.b32; }
template <> __device__ __forceinline__ double* lvbuf<2>(const DevCtx& c) { return c.b64; }

// read element (i,j) of level buffer `lv` as double (runtime level)
__device__ __forceinline__ double load_level(const DevCtx& c, int lv, long long off) {
    if (lv == 0) return to_d(c.b16[off]);
    if (lv == 1) return to_d(c.b32[off]);
    return c.b64[off];
}
// store double x rounded to level lv
__device__ __forceinline__ void store_level(const DevCtx& c, int lv, long long off, double x) {
    if (lv == 0) c.b16[off] = d2h(x);
    else if (lv == 1) c.b32[off] = __double2float_rn(x);
    else c.b64[off] = x;
}
__device__ __forceinline__ double round_level(int lv, double x) {
    if (lv == 0) return double(__half2float(d2h(x)));
    if (lv == 1) return double(__double2float_rn(x));
    return x;
}

// ---------------------------------------------------------------------------
// leaf kernels' shared-memory tiles: a lower triangle of nt x nt blocks of
// 32 x 32, tile k = a(a+1)/2 + b holding block (off + a, off + b), each tile
// column-major with the row index XOR-swizzled by 4 (c & 7): one column
// across a warp's 32 rows and 4 consecutive rows of one column are both
// bank-conflict free.  (k_potrf.cu, k_inverse.cu)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int tri_sw(int r, int c) { return (c << 5) + (r ^ ((c & 7) << 2)); }
__device__ __forceinline__ void tri_tile_ab(int k, int& a, int& b) {
    a = 0;
    while (((a + 1) * (a + 2)) / 2 <= k) ++a;
    b = k - ((a * (a + 1)) >> 1);
}
// tiles -> global, whole tiles as 16-byte row chunks (a diagonal tile's
// strict upper part goes back as loaded); g16 (F32 tiles only, may be null):
// also the binary16-rounded copy at the same coordinates (a fused OP_SHADOW)
template <typename T, int NTHREADS>
__device__ __forceinline__ void tri_store_vec(const float* S, T* g, long long ld, int nt, int off, int tid,
                                              __half* g16 = nullptr) {
    constexpr int VEC = 16 / int(sizeof(T)), CPR = 32 / VEC, CPT = 32 * CPR, KSTEP = NTHREADS / CPT;
    const int ntile = (nt * (nt + 1)) >> 1;
    const int row = (tid % CPT) / CPR, col = (tid % CPR) * VEC;
#pragma unroll 1
    for (int k = tid / CPT; k < ntile; k += KSTEP) {
        int a, b;
        tri_tile_ab(k, a, b);
        const float* t = S + k * 1024;
        uint4 w;
        T* e = reinterpret_cast<T*>(&w);
#pragma unroll
        for (int u = 0; u < VEC; ++u) e[u] = from_float<T>(t[tri_sw(row, col + u)]);
        const long long o = (long long)((off + a) * 32 + row) * ld + (off + b) * 32 + col;
        *reinterpret_cast<uint4*>(g + o) = w;
        if constexpr (VEC == 4) {
            if (g16) {
                const float* f = reinterpret_cast<const float*>(&w);
                __half2 h[2] = {__floats2half2_rn(f[0], f[1]), __floats2half2_rn(f[2], f[3])};
                *reinterpret_cast<uint2*>(g16 + o) = *reinterpret_cast<const uint2*>(h);
            }
        }
    }
}
__device__ __forceinline__ bool vec16_ok(const void* g, long long ld_bytes) {
    return (reinterpret_cast<uintptr_t>(g) & 15) == 0 && (ld_bytes & 15) == 0;
}

// programmatic dependent launch: every factorization kernel waits here
// before it reads anything a preceding kernel wrote (a no-op unless it was
// launched through a programmatic graph edge); chain kernels signal their
// dependents near their end so those are scheduled while they finish
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ double range_max(int lv) {
    return lv == 0 ? 65504.0 : lv == 1 ? 3.4028234663852886e38 : 1.7976931348623157e308;
}

#endif  // __CUDACC__

// ---------------------------------------------------------------------------
// block tables for the elementwise kernels (import / export / shadow /
// check): a CTA handles one 32x32 tile of one block; blocks are located by a
// binary search over the tiles' prefix sums
// ---------------------------------------------------------------------------

struct BlockDesc {
    int r0, c0, m, n;
    int level;      // storage level of the block
    int lower;      // diagonal leaf: lower triangle only
    int tile0;      // first tile index of this block
    int tiles_n;    // tiles across (n direction)
};

#ifdef __CUDACC__
__device__ __forceinline__ int find_block(const BlockDesc* b, int nb, int tile) {
    int lo = 0, hi = nb - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b[mid].tile0 <= tile) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

#endif

// one grouped-GEMM problem as seen by the device
struct DevProb {
    int m, n, k;
    int a_r0, a_c0, b_r0, b_c0, c_r0, c_c0;
    int exec_level;
    int lower;
    int tile0;      // first tile of this problem in the launch
    int tiles_n;    // tiles across n
    double alpha, beta;
    int a_kwrap;    // A's K coordinate wraps (inverse solve); 0 = no
    int b_buf;      // B operand buffer (BUF_W16 for inverse solves), -1 = operand level
    uint32_t check_seq;  // fused require_finite on the stored values (0 = none)
    int chk_r0, chk_c0;  // origin of the checked block
};

#ifdef __CUDACC__
// fused require_finite helpers: the first bad element in column-major order
__device__ __forceinline__ bool h_bad(__half h) { return (__half_as_ushort(h) & 0x7c00) == 0x7c00; }
__device__ __forceinline__ void warp_report_min(const DevCtx& c, unsigned long long key) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, key, o);
        key = x < key ? x : key;
    }
    if ((threadIdx.x & 31) == 0 && key != ~0ull) atomicMin(c.status, key);
}
#endif

}  // namespace tcb
