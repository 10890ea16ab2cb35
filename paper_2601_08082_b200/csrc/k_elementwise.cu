// k_elementwise.cu -- HBM-bound passes over blocks of the matrix:
//   import   caller doubles (col-major) -> level buffers (row-major), rounding
//            to each block's level (build_tree rounding, tree.cpp:47-60)
//   export   level buffers -> caller doubles, lower triangle only
//   shadow   final L block -> p-rounded copy in buffer p (kernels.cpp:29,78)
//   check    require_finite (tree.cpp:19-31) -> first bad element
//   quant    quantize_block of a spine panel (tree.cpp:80-95), fused with its
//            require_finite and the absmax reduction
//   dequant  dequantize_block (tree.cpp:97-104)
// Transposing kernels stage a 32x32 tile in shared memory so both the
// column-major and the row-major side are coalesced.
#include "device.cuh"
#include "launch.hpp"

namespace tcb {

namespace {

constexpr int TS = 32;  // tile side

// grid-stride over 64x64 tiles (a few thousand CTAs, not one per tile);
// every thread issues all 16 of its loads before touching shared memory
constexpr int TB = 64;  // block-table tile side (import / export / shadow)
constexpr int TBR = (TB * TB) / 256;  // elements per thread per tile

__global__ void __launch_bounds__(256) k_import(DevCtx c, const BlockDesc* blocks, int nb, int tiles) {
    pdl_wait();
    __shared__ double tile[TB][TB + 1];
    const int tx = threadIdx.x & (TB - 1), ty = threadIdx.x / TB;  // ty in [0, 4)
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const BlockDesc bd = blocks[find_block(blocks, nb, t)];
        const int lt = t - bd.tile0;
        const int i0 = (lt / bd.tiles_n) * TB, j0 = (lt % bd.tiles_n) * TB;
        const double* a = c.ra->a_in;
        const long long lda = c.ra->lda_in;
        double v[TBR];
#pragma unroll
        for (int r = 0; r < TBR; ++r) {  // column-major source: lanes along i
            const int i = i0 + tx, j = j0 + ty + 4 * r;
            v[r] = (i < bd.m && j < bd.n) ? a[(long long)(bd.c0 + j) * lda + bd.r0 + i] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < TBR; ++r) tile[ty + 4 * r][tx] = v[r];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < TBR; ++r) {  // row-major level buffer: lanes along j
            const int i = i0 + ty + 4 * r, j = j0 + tx;
            if (i < bd.m && j < bd.n) {
                double x = tile[tx][ty + 4 * r];
                if (bd.lower && j > i) x = 0.0;  // strict upper of a leaf square: unused
                store_level(c, bd.level, (long long)(bd.r0 + i) * c.ldw + bd.c0 + j, x);
            }
        }
        __syncthreads();
    }
}

// export: 64x64 tiles, 16-byte accesses on both sides.  Thread (r, q) =
// (tid / 4, tid % 4) reads 16 consecutive row-major elements of row r
// (2 / 4 / 8 vector loads for F16 / F32 / F64, all issued before the first
// shared-memory store), converts them to double and stores them transposed
// (tile[col][row], an even row pitch so double2 reads stay aligned; rows
// offset by 8 per 16-column quarter so the 32 lanes of a store hit every
// bank pair twice, the minimum for doubles); then each warp
// writes 8 columns as 512-byte runs of double2 (lanes along the rows).
// Edge and diagonal tiles (and unaligned operands) take per-element paths.
constexpr int EX_LD = TB + 2;
__device__ __forceinline__ int ex_phys(int c, int r) { return c * EX_LD + ((r + 8 * (c >> 4)) & (TB - 1)); }

__global__ void __launch_bounds__(256) k_export(DevCtx c, const BlockDesc* blocks, int nb, int tiles) {
    pdl_wait();
    __shared__ __align__(16) double tile[TB * EX_LD];
    const int tid = threadIdx.x, r = tid >> 2, q = tid & 3, lane = tid & 31, warp = tid >> 5;
    double* l = c.ra->l_out;
    const long long ldl = c.ra->lda_out;
    const bool out_vec = (ldl % 2 == 0) && ((reinterpret_cast<uintptr_t>(l) & 15) == 0);
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const BlockDesc bd = blocks[find_block(blocks, nb, t)];
        const int lt = t - bd.tile0;
        const int i0 = (lt / bd.tiles_n) * TB, j0 = (lt % bd.tiles_n) * TB;
        const int mi = min(TB, bd.m - i0), nj = min(TB, bd.n - j0);
        // ---- row-major level buffer -> registers (16 elements per thread)
        double v[16];
        const int i = i0 + r, jq = j0 + 16 * q;
        const long long off = (long long)(bd.r0 + i) * c.ldw + bd.c0 + jq;
        const bool row_in = r < mi;
        const int cnt = row_in ? max(0, min(16, nj - 16 * q)) : 0;
        if (bd.level == 0) {
            const __half* p = c.b16 + off;
            if (cnt == 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
                uint4 w[2];
                w[0] = __ldcs(reinterpret_cast<const uint4*>(p));
                w[1] = __ldcs(reinterpret_cast<const uint4*>(p) + 1);
                const __half2* h = reinterpret_cast<const __half2*>(w);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float2 f = __half22float2(h[e]);
                    v[2 * e] = f.x;
                    v[2 * e + 1] = f.y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = e < cnt ? to_d(p[e]) : 0.0;
            }
        } else if (bd.level == 1) {
            const float* p = c.b32 + off;
            if (cnt == 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
                float4 w[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = __ldcs(reinterpret_cast<const float4*>(p) + k);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    v[4 * k] = w[k].x;
                    v[4 * k + 1] = w[k].y;
                    v[4 * k + 2] = w[k].z;
                    v[4 * k + 3] = w[k].w;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = e < cnt ? double(p[e]) : 0.0;
            }
        } else {
            const double* p = c.b64 + off;
            if (cnt == 16 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
                double2 w[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) w[k] = __ldcs(reinterpret_cast<const double2*>(p) + k);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    v[2 * k] = w[k].x;
                    v[2 * k + 1] = w[k].y;
                }
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = e < cnt ? p[e] : 0.0;
            }
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) tile[ex_phys(16 * q + e, r)] = v[e];
        __syncthreads();
        // ---- column-major doubles: warp w writes columns 8w .. 8w+7
        const bool full = mi == TB && nj == TB && !(bd.lower && j0 + TB - 1 > i0);
        const long long base = (long long)(bd.c0 + j0) * ldl + bd.r0 + i0;
        if (full && out_vec && ((bd.r0 + i0) & 1) == 0) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int cc = 8 * warp + k;
                const double2 x = *reinterpret_cast<const double2*>(&tile[ex_phys(cc, 2 * lane)]);
                __stcs(reinterpret_cast<double2*>(l + base + (long long)cc * ldl) + lane, x);
            }
        } else {
            for (int k = 0; k < 8; ++k) {
                const int cc = 8 * warp + k;
                if (cc >= nj) break;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rr = lane + 32 * h;
                    if (rr < mi && !(bd.lower && j0 + cc > i0 + rr))
                        l[base + (long long)cc * ldl + rr] = tile[ex_phys(cc, rr)];
                }
            }
        }
        __syncthreads();
    }
}

// shadow: blocks carry their source level; target is `p`
__global__ void __launch_bounds__(256) k_shadow(DevCtx c, const BlockDesc* blocks, int nb, int p, int tiles) {
    pdl_wait();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const BlockDesc bd = blocks[find_block(blocks, nb, t)];
        const int lt = t - bd.tile0;
        const int i0 = (lt / bd.tiles_n) * TB, j0 = (lt % bd.tiles_n) * TB;
        // all 16 loads of a thread first (the level buffers may alias as far
        // as the compiler knows, so an interleaved load / store loop would
        // pay one L2 round trip per element)
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int i = i0 + ty + 8 * (k >> 1), j = j0 + 32 * (k & 1) + tx;
            v[k] = (i < bd.m && j < bd.n) ? load_level(c, bd.level, (long long)(bd.r0 + i) * c.ldw + bd.c0 + j) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int i = i0 + ty + 8 * (k >> 1), j = j0 + 32 * (k & 1) + tx;
            if (i < bd.m && j < bd.n)
                store_level(c, p, (long long)(bd.r0 + i) * c.ldw + bd.c0 + j, (bd.lower && j > i) ? 0.0 : v[k]);
        }
    }
}

// require_finite over rect (lower: leaf lower triangle) of buffer `lv`
__global__ void __launch_bounds__(256) k_check(DevCtx c, int lv, int r0, int c0, int m, int n, int lower,
                                               uint32_t seq) {
    pdl_wait();
    const int j = blockIdx.x * 256 + threadIdx.x;
    const int ib = blockIdx.y * 16;
    unsigned long long best = ~0ull;
    if (j < n) {
        for (int ii = 0; ii < 16; ++ii) {
            const int i = ib + ii;
            if (i >= m) break;
            if (lower && j > i) continue;
            const double v = load_level(c, lv, (long long)(r0 + i) * c.ldw + c0 + j);
            if (!isfinite(v)) {
                best = fail_key(seq, elem_local(i, j));
                break;
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
        best = x < best ? x : best;
    }
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(c.status, best);
}

// quantize pass 1: require_finite on the caller's doubles, max|B| into the
// alpha slot, and a speculative alpha == 1 conversion into buffer lv
__global__ void __launch_bounds__(256) k_quant1(DevCtx c, int lv, int r0, int c0, int m, int n, int slot,
                                                uint32_t seq) {
    pdl_wait();
    // 64x64 transposing tiles, all 16 loads of a thread in flight (k_import)
    __shared__ double tile[TB][TB + 1];
    __shared__ unsigned long long smax[8], skey[8];
    const int tiles_n = (n + TB - 1) / TB;
    const int tiles = tiles_n * ((m + TB - 1) / TB);
    const double* a = c.ra->a_in;
    const long long lda = c.ra->lda_in;
    const int tx = threadIdx.x & (TB - 1), ty = threadIdx.x / TB;
    unsigned long long mx = 0, key = ~0ull;
    // grid-stride over the tiles; one reduction per CTA at the end
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int i0 = (t / tiles_n) * TB, j0 = (t % tiles_n) * TB;
        double v[TBR];
#pragma unroll
        for (int r = 0; r < TBR; ++r) {
            const int i = i0 + tx, j = j0 + ty + 4 * r;
            v[r] = (i < m && j < n) ? a[(long long)(c0 + j) * lda + r0 + i] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < TBR; ++r) {
            const int i = i0 + tx, j = j0 + ty + 4 * r;
            if (i < m && j < n && !isfinite(v[r])) {
                const unsigned long long k = fail_key(seq, elem_local(i, j));
                key = k < key ? k : key;
            }
            const unsigned long long bits = __double_as_longlong(fabs(v[r]));
            mx = (bits > mx && bits <= 0x7ff0000000000000ull) ? bits : mx;  // NaN skipped (tree.cpp:82-86)
            tile[ty + 4 * r][tx] = v[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < TBR; ++r) {
            const int i = i0 + ty + 4 * r, j = j0 + tx;
            if (i < m && j < n) store_level(c, lv, (long long)(r0 + i) * c.ldw + c0 + j, tile[tx][ty + 4 * r]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, mx, o);
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
        mx = x > mx ? x : mx;
        key = y < key ? y : key;
    }
    if ((threadIdx.x & 31) == 0) {
        smax[threadIdx.x >> 5] = mx;
        skey[threadIdx.x >> 5] = key;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long M = 0, K = ~0ull;
        for (int w = 0; w < 8; ++w) {
            M = smax[w] > M ? smax[w] : M;
            K = skey[w] < K ? skey[w] : K;
        }
        if (M) atomicMax(c.alpha_bits + slot, M);
        if (K != ~0ull) atomicMin(c.status, K);
    }
}

__device__ __forceinline__ double slot_alpha(const DevCtx& c, int lv, int slot) {
    const double amax = __longlong_as_double((long long)c.alpha_bits[slot]);
    double alpha = amax / range_max(lv);
    if (!(alpha > 1.0)) alpha = 1.0;
    return alpha;
}

// quantize pass 2: only when alpha != 1, B <- rn(B / alpha) from the doubles
__global__ void __launch_bounds__(256) k_quant2(DevCtx c, int lv, int r0, int c0, int m, int n, int slot) {
    pdl_wait();
    const double alpha = slot_alpha(c, lv, slot);
    if (alpha == 1.0) return;
    __shared__ double tile[TS][TS + 1];
    const int tiles_n = (n + TS - 1) / TS;
    const int tiles = tiles_n * ((m + TS - 1) / TS);
    const double* a = c.ra->a_in;
    const long long lda = c.ra->lda_in;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int i0 = (t / tiles_n) * TS, j0 = (t % tiles_n) * TS;
#pragma unroll
        for (int r = 0; r < TS; r += 8) {
            const int i = i0 + tx, j = j0 + ty + r;
            tile[ty + r][tx] = (i < m && j < n) ? a[(long long)(c0 + j) * lda + r0 + i] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < TS; r += 8) {
            const int i = i0 + ty + r, j = j0 + tx;
            if (i < m && j < n) store_level(c, lv, (long long)(r0 + i) * c.ldw + c0 + j, tile[tx][ty + r] / alpha);
        }
        __syncthreads();
    }
}

// dequantize_block; when alpha != 1 it is the panel's last writer, so the
// post-dequantize require_finite (tree.cpp:121) is fused here too
__global__ void __launch_bounds__(256) k_dequant(DevCtx c, int lv, int r0, int c0, int m, int n, int slot,
                                                 uint32_t chk_seq, int chk_dr, int chk_dc) {
    pdl_wait();
    const double alpha = slot_alpha(c, lv, slot);
    if (alpha == 1.0) return;  // tree.cpp:98 (the common case: a bounded grid, so the no-op launch is short)
    unsigned long long bad = ~0ull;
    const int cols = (n + 255) / 256, items = cols * ((m + 15) / 16);
    for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int j = (it % cols) * 256 + threadIdx.x, i0 = (it / cols) * 16;
        if (j < n)
            for (int ii = 0; ii < 16; ++ii) {
                const int i = i0 + ii;
                if (i >= m) break;
                const long long off = (long long)(r0 + i) * c.ldw + c0 + j;
                const double v = load_level(c, lv, off) * alpha;
                store_level(c, lv, off, v);
                if (!isfinite(round_level(lv, v))) {
                    const unsigned long long k = fail_key(chk_seq, elem_local(i + chk_dr, j + chk_dc));
                    bad = k < bad ? k : bad;
                }
            }
    }
    if (chk_seq) warp_report_min(c, bad);
}

int tiles_of(int m, int n) { return ((m + TS - 1) / TS) * ((n + TS - 1) / TS); }

// spd_generate's symmetrization (analysis.cpp:22-26) in place on the raw
// column-major draws R: A(i,j) = A(j,i) = 0.5 * (R(i,j) + R(j,i)), A(j,j) +=
// n.  One CTA per lower tile pair; explicit _rn ops forbid contraction, so
// the result is bit-identical to the host reference.
__global__ void __launch_bounds__(256) k_symmetrize(double* a, long long lda, int n) {
    __shared__ double t1[TS][TS + 1], t2[TS][TS + 1];
    const int t = blockIdx.x;
    int I = int((sqrt(8.0 * t + 1.0) - 1.0) / 2.0);
    while ((I + 1) * (I + 2) / 2 <= t) ++I;
    while (I * (I + 1) / 2 > t) --I;
    const int J = t - I * (I + 1) / 2;  // I >= J
    const int i0 = I * TS, j0 = J * TS;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int r = 0; r < TS; r += 8) {
        const int i = i0 + tx, j = j0 + ty + r;  // tile (I,J): rows i, cols j
        t1[ty + r][tx] = (i < n && j < n) ? a[(long long)j * lda + i] : 0.0;
        const int i2 = j0 + tx, j2 = i0 + ty + r;  // tile (J,I)
        t2[ty + r][tx] = (i2 < n && j2 < n) ? a[(long long)j2 * lda + i2] : 0.0;
    }
    __syncthreads();
    const double dn = double(n);
    for (int r = 0; r < TS; r += 8) {
        // element (i, j) of tile (I,J) pairs with (j, i) of tile (J,I)
        const int jl = ty + r, il = tx;
        const int i = i0 + il, j = j0 + jl;
        if (i < n && j < n) {
            double v = __dmul_rn(0.5, __dadd_rn(t1[jl][il], t2[il][jl]));
            if (i == j) v = __dadd_rn(v, dn);
            a[(long long)j * lda + i] = v;
            a[(long long)i * lda + j] = v;
        }
    }
}

}  // namespace

// row-major level image of a column-major double block: dst[i * ldd + j] =
// rn_L(src[j * lds + i]) (direct RNE, d2h for binary16), strict upper
// triangle zero when `lower` -- how a distributed piece receives a factor
// block it reads through rn_p (kernels.cpp:29, 78)
template <typename T>
__global__ void __launch_bounds__(256) k_level_image(int m, int n, const double* __restrict__ src, long long lds,
                                                     int lower, T* __restrict__ dst, long long ldd) {
    __shared__ double t[32][33];
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + tx, j = j0 + r;  // coalesced down a column
        t[r][tx] = (i < m && j < n) ? src[(long long)j * lds + i] : 0.0;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int i = i0 + r, j = j0 + tx;  // coalesced along a row
        if (i < m && j < n) dst[(long long)i * ldd + j] = (lower && j > i) ? from_double<T>(0.0) : from_double<T>(t[tx][r]);
    }
}

void launch_level_image(int m, int n, const double* src, long long lds, int level, int lower, void* dst,
                        long long ldd, cudaStream_t s) {
    const dim3 grid((n + 31) / 32, (m + 31) / 32);
    if (level == 0)
        k_level_image<__half><<<grid, 256, 0, s>>>(m, n, src, lds, lower, static_cast<__half*>(dst), ldd);
    else if (level == 1)
        k_level_image<float><<<grid, 256, 0, s>>>(m, n, src, lds, lower, static_cast<float*>(dst), ldd);
    else
        k_level_image<double><<<grid, 256, 0, s>>>(m, n, src, lds, lower, static_cast<double*>(dst), ldd);
}

void launch_symmetrize(double* a, long long lda, int n, cudaStream_t s) {
    const int T = (n + TS - 1) / TS;
    k_symmetrize<<<T * (T + 1) / 2, 256, 0, s>>>(a, lda, n);
}

// host-side block table construction
int make_block_table(const std::vector<BlockDescHost>& in, std::vector<BlockDesc>& out) {
    out.clear();
    int tiles = 0;
    for (const auto& h : in) {
        BlockDesc d;
        d.r0 = h.r0;
        d.c0 = h.c0;
        d.m = h.m;
        d.n = h.n;
        d.level = h.level;
        d.lower = h.lower;
        d.tile0 = tiles;
        d.tiles_n = (h.n + TB - 1) / TB;
        out.push_back(d);
        tiles += ((h.m + TB - 1) / TB) * d.tiles_n;
    }
    return tiles;
}

// grid of the tiled copy kernels: grid-stride over at most 8 CTAs per SM
// (default), or a fixed number of tiles per CTA (option elem_tiles_per_cta),
// so their CTAs turn over and higher-priority work gets SMs between tiles
static int g_elem_tiles_per_cta = 0;
bool elem_set_option(const std::string& key, int value) {
    if (key != "elem_tiles_per_cta") return false;
    g_elem_tiles_per_cta = value < 0 ? 0 : value;
    return true;
}
static int tile_grid(int tiles) {
    if (g_elem_tiles_per_cta > 0) return (tiles + g_elem_tiles_per_cta - 1) / g_elem_tiles_per_cta;
    return tiles < 148 * 8 ? tiles : 148 * 8;
}
void launch_import(const DevCtx& c, const BlockDesc* d_blocks, int nb, int tiles, cudaStream_t s) {
    if (tiles > 0) k_import<<<tile_grid(tiles), 256, 0, s>>>(c, d_blocks, nb, tiles);
}
void launch_export(const DevCtx& c, const BlockDesc* d_blocks, int nb, int tiles, cudaStream_t s) {
    if (tiles > 0) k_export<<<tile_grid(tiles), 256, 0, s>>>(c, d_blocks, nb, tiles);
}
void launch_shadow(const DevCtx& c, const BlockDesc* d_blocks, int nb, int tiles, int p, cudaStream_t s) {
    if (tiles > 0) k_shadow<<<tile_grid(tiles), 256, 0, s>>>(c, d_blocks, nb, p, tiles);
}
void launch_check(const DevCtx& c, int lv, int r0, int c0, int m, int n, int lower, uint32_t seq,
                  cudaStream_t s) {
    dim3 g((n + 255) / 256, (m + 15) / 16);
    k_check<<<g, 256, 0, s>>>(c, lv, r0, c0, m, n, lower, seq);
}
void launch_quant(const DevCtx& c, int lv, int r0, int c0, int m, int n, int slot, uint32_t seq,
                  cudaStream_t s) {
    const int t = tiles_of(m, n);
    const int g = t < 148 * 8 ? t : 148 * 8;
    k_quant1<<<g, 256, 0, s>>>(c, lv, r0, c0, m, n, slot, seq);
    k_quant2<<<g, 256, 0, s>>>(c, lv, r0, c0, m, n, slot);
}
void launch_dequant(const DevCtx& c, int lv, int r0, int c0, int m, int n, int slot, uint32_t chk_seq,
                    int chk_dr, int chk_dc, cudaStream_t s) {
    const long long items = (long long)((n + 255) / 256) * ((m + 15) / 16);
    const int g = int(items < 148 * 8 ? items : 148 * 8);
    k_dequant<<<g, 256, 0, s>>>(c, lv, r0, c0, m, n, slot, chk_seq, chk_dr, chk_dc);
}

}  // namespace tcb

namespace tcb {
namespace {
// holds the stream until the host has enqueued everything behind it, so the
// per-op events of a profiling run measure device time, not launch gaps
__global__ void k_gate(volatile int* flag) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {  // never longer than 5 s, whatever the host does
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (*flag == 0 && t - t0 < 5000000000ull);
}
__global__ void k_noop() {}
// development trace: the global timer (ns) when this node runs
__global__ void k_stamp(unsigned long long* out) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *out = t;
}
}  // namespace
void launch_gate(volatile int* host_flag, cudaStream_t s) { k_gate<<<1, 1, 0, s>>>(host_flag); }
void launch_noop(cudaStream_t s) { k_noop<<<1, 32, 0, s>>>(); }
void launch_stamp(unsigned long long* out, cudaStream_t s) { k_stamp<<<1, 1, 0, s>>>(out); }
}  // namespace tcb
