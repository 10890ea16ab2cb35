// k_gemm_tc.cu -- grouped FP16 GEMM on the 5th-generation tensor cores.
//
//   C(i,j) <- rn_exec( rn_f32(alpha*s) + rn_f32(beta*C(i,j)) ),
//   s = sum_t A(i,t) * B(j,t)   (FP16 operands, exact products, FP32 sums)
//
// This is gemm_mixed / syrk_leaf (kernels.cpp:94-132) for every call whose
// operands are FP16-valued: exec level F16 (82% of the flops at N=65536
// [F16,F16,F16,F32]) and F32 exec on FP16 panels (16.4%) -- the products of
// two binary16 values are exact in binary32, so the reference's
// rn_f32(a*b) is the identity and an FP32 tensor-core accumulator implements
// the same arithmetic model (SURVEY headline fact 3).
//
// Structure (one persistent CTA per SM, 192 threads, warp-specialised):
//   warp 0      TMA producer: 128x64 A and 256x64 B tiles, SWIZZLE_128B,
//               4-stage smem ring guarded by full/empty mbarriers
//   warp 1      TMEM allocator + MMA issuer: one elected lane issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=256, K=16) into
//               a double-buffered FP32 accumulator (2 x 256 TMEM columns)
//   warps 2-5   epilogue: tcgen05.ld 32x32b -> registers -> rounding to the
//               destination level -> global (row-major C)
// A problem list (one tree_syrk = all its output blocks, or one trsm GEMM)
// is flattened into 128x256 tiles; each problem has its own pair of TMA
// descriptors whose extents end at the problem's edge, so partial tiles are
// zero-filled by the TMA unit and K need not be a multiple of 64.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <string>

#include "device.cuh"
#include "launch.hpp"

namespace tcb {

struct alignas(128) TcProb {
    CUtensorMap ta;  // A rows [a_r0, a_r0+m) x cols [a_c0, a_c0+k) (extents end there)
    CUtensorMap tb;  // B rows [b_r0, b_r0+n) x cols [b_c0, b_c0+k)
    int m, n, k;
    int a_r0, a_c0, b_r0, b_c0, c_r0, c_c0;
    int exec_level, lower, tile0, tiles_n;
    double alpha, beta;
    int a_kwrap;  // inverse solve: A columns repeat with this period (B = [W_hi | W_lo])
    uint32_t check_seq;  // fused require_finite (0 = none), element relative to chk origin
    int chk_r0, chk_c0;
};

size_t tc_prob_size() { return sizeof(TcProb); }

namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int NTHREADS = 192;
constexpr uint32_t TMEM_COLS = 512;  // 2 accumulators x 256 columns

// instruction descriptor, kind::f16: D=F32 (bits 4-5 = 1), A=B=F16 (0),
// both K-major, N>>3 at bits 17-22, M>>4 at bits 24-28
constexpr uint32_t IDESC = (1u << 4) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B (layout type 2 at
// bits 61-63), SBO = 1024 B between 8-row groups, LBO unused (1), version 1
__device__ __forceinline__ uint64_t sdesc(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ int find_tc_prob(const TcProb* p, int np, int tile) {
    int lo = 0, hi = np - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p[mid].tile0 <= tile) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// tile -> (problem, tm, tn); false for a lower problem's tile strictly above
// the diagonal (nothing to write).  Every role evaluates the same predicate.
__device__ __forceinline__ bool tile_coords(const TcProb* probs, int np, int t, int& pi, int& tm, int& tn) {
    pi = find_tc_prob(probs, np, t);
    const TcProb& p = probs[pi];
    const int lt = t - p.tile0;
    tm = lt / p.tiles_n;
    tn = lt % p.tiles_n;
    return !(p.lower && p.c_c0 + tn * BN > p.c_r0 + tm * BM + BM - 1);
}

__device__ __forceinline__ float epi_f(float s, float cv, double alpha, double beta) {
    float r = alpha == -1.0 ? -s : __double2float_rn(alpha * double(s));
    if (beta != 0.0) r = r + (beta == 1.0 ? cv : __double2float_rn(beta * double(cv)));
    return r;
}

__global__ void __launch_bounds__(NTHREADS, 1) k_gemm_tc(DevCtx c, const TcProb* __restrict__ probs, int np,
                                                        int tiles) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                           ~uintptr_t(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                int pi, tm, tn;
                if (!tile_coords(probs, np, t, pi, tm, tn)) continue;
                const TcProb* p = probs + pi;
                prefetch_map(&p->ta);
                prefetch_map(&p->tb);
                const int nk = (p->k + BK - 1) / BK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], STAGE_BYTES);
                    const int ka = p->a_kwrap ? (kb * BK) % p->a_kwrap : kb * BK;
                    tma_load_2d(sA + stage * A_BYTES, &p->ta, &full[stage], p->a_c0 + ka, p->a_r0 + tm * BM);
                    tma_load_2d(sB + stage * B_BYTES, &p->tb, &full[stage], p->b_c0 + kb * BK, p->b_r0 + tn * BN);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        int stage = 0;
        uint32_t phase = 0;
        int as = 0;
        uint32_t aphase = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            int pi, tm, tn;
            if (!tile_coords(probs, np, t, pi, tm, tn)) continue;
            const int nk = (probs[pi].k + BK - 1) / BK;
            mbar_wait(&tempty[as], aphase ^ 1);
            tc_fence_after();
            const uint32_t dcol = tmem + uint32_t(as * BN);
            for (int kb = 0; kb < nk; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint64_t da = sdesc(sA + stage * A_BYTES);
                    const uint64_t db = sdesc(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)  // +32 bytes per K=16 step inside the swizzled row
                        mma_f16(dcol, da + uint64_t(2 * k), db + uint64_t(2 * k), (kb | k) != 0);
                    mma_commit(&empty[stage]);
                    if (kb == nk - 1) mma_commit(&tfull[as]);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (++as == 2) {
                as = 0;
                aphase ^= 1;
            }
        }
    } else {
        // ---------------- epilogue (warps 2..5) ----------------
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int as = 0;
        uint32_t aphase = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            int pi, tm, tn;
            if (!tile_coords(probs, np, t, pi, tm, tn)) continue;
            const TcProb& p = probs[pi];
            mbar_wait(&tfull[as], aphase);
            tc_fence_after();
            const int i = tm * BM + q * 32 + lane;  // row of C inside the problem
            const bool row_ok = i < p.m;
            const long long rowoff = (long long)(p.c_r0 + (row_ok ? i : 0)) * c.ldw + p.c_c0;
            const int lvl = p.exec_level;
            // inverse solves carry W scaled by 2^e; undo it exactly here
            const double alpha = p.a_kwrap ? double(c.wscale[p.b_r0]) : p.alpha;
            // fused require_finite: track the first non-finite stored value
            const bool chk = p.check_seq != 0;
            unsigned long long bad = ~0ull;
            const int iloc = p.c_r0 + i - p.chk_r0;
            auto note = [&](bool isbad, int j) {
                if (chk && isbad) {
                    const unsigned long long k = fail_key(p.check_seq, elem_local(iloc, p.c_c0 + j - p.chk_c0));
                    bad = k < bad ? k : bad;
                }
            };
            for (int cc = 0; cc < BN; cc += 32) {
                float v[32];
                __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge first
                tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(as * BN + cc), v);
                if (cc == BN - 32) {
                    // accumulator drained: hand it back to the MMA warp
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[as]);
                }
                const int j0 = tn * BN + cc;
                if (!row_ok || j0 >= p.n) continue;
                // columns allowed in this chunk: bounds and the lower mask
                int jmax = min(32, p.n - j0);
                if (p.lower) jmax = min(jmax, (p.c_r0 + i) - (p.c_c0 + j0) + 1);
                if (jmax <= 0) continue;
                if (lvl == LV_F16) {
                    __half* C = c.b16 + rowoff + j0;
                    const bool vec = jmax == 32 && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
                    if (vec) {
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            uint4 raw = p.beta != 0.0 ? *reinterpret_cast<const uint4*>(C + 8 * g) : make_uint4(0, 0, 0, 0);
                            __half2* h = reinterpret_cast<__half2*>(&raw);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 cf = __half22float2(h[e]);
                                const __half o0 = f2h(epi_f(v[8 * g + 2 * e], cf.x, alpha, p.beta));
                                const __half o1 = f2h(epi_f(v[8 * g + 2 * e + 1], cf.y, alpha, p.beta));
                                note(h_bad(o0), j0 + 8 * g + 2 * e);
                                note(h_bad(o1), j0 + 8 * g + 2 * e + 1);
                                h[e] = __halves2half2(o0, o1);
                            }
                            *reinterpret_cast<uint4*>(C + 8 * g) = raw;
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (e < jmax) {
                                const float cv = p.beta != 0.0 ? __half2float(C[e]) : 0.f;
                                const __half o = f2h(epi_f(v[e], cv, alpha, p.beta));
                                note(h_bad(o), j0 + e);
                                C[e] = o;
                            }
                    }
                } else {
                    float* C = c.b32 + rowoff + j0;
                    const bool vec = jmax == 32 && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
                    if (vec) {
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            float4 cv = p.beta != 0.0 ? *reinterpret_cast<const float4*>(C + 4 * g) : make_float4(0, 0, 0, 0);
                            cv.x = epi_f(v[4 * g + 0], cv.x, alpha, p.beta);
                            cv.y = epi_f(v[4 * g + 1], cv.y, alpha, p.beta);
                            cv.z = epi_f(v[4 * g + 2], cv.z, alpha, p.beta);
                            cv.w = epi_f(v[4 * g + 3], cv.w, alpha, p.beta);
                            note(!isfinite(cv.x), j0 + 4 * g);
                            note(!isfinite(cv.y), j0 + 4 * g + 1);
                            note(!isfinite(cv.z), j0 + 4 * g + 2);
                            note(!isfinite(cv.w), j0 + 4 * g + 3);
                            *reinterpret_cast<float4*>(C + 4 * g) = cv;
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (e < jmax) {
                                const float cv = p.beta != 0.0 ? C[e] : 0.f;
                                const float o = epi_f(v[e], cv, alpha, p.beta);
                                note(!isfinite(o), j0 + e);
                                C[e] = o;
                            }
                    }
                }
            }
            __syncwarp();
            if (chk) warp_report_min(c, bad);
            if (++as == 2) {
                as = 0;
                aphase ^= 1;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool make_map(CUtensorMap* m, const __half* base, long long ldw, int rows_end, int cols_end, int box_rows,
              std::string* err) {
    auto enc = get_encode();
    if (!enc) {
        if (err) *err = "cuTensorMapEncodeTiled unavailable";
        return false;
    }
    cuuint64_t dims[2] = {cuuint64_t(cols_end), cuuint64_t(rows_end)};
    cuuint64_t strides[1] = {cuuint64_t(ldw) * 2};
    cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        if (err) *err = "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")";
        return false;
    }
    return true;
}

}  // namespace

bool tc_supported() {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major == 10 && minor == 0 && get_encode() != nullptr;
}

int tc_build_probs(const DevCtx& c, const std::vector<DevProb>& probs, std::vector<unsigned char>& out,
                   std::string* err) {
    out.assign(probs.size() * sizeof(TcProb), 0);
    TcProb* tp = reinterpret_cast<TcProb*>(out.data());
    int tiles = 0;
    for (size_t i = 0; i < probs.size(); ++i) {
        const DevProb& d = probs[i];
        TcProb& p = tp[i];
        // A extent ends at the problem's K edge (an inverse solve's A is the
        // n-wide leaf column block read twice: its extent is n, period a_kwrap)
        if (!make_map(&p.ta, c.b16, c.ldw, d.a_r0 + d.m, d.a_c0 + (d.a_kwrap ? d.n : d.k), BM, err)) return -1;
        const bool w = d.b_buf == BUF_W16;
        if (!make_map(&p.tb, w ? c.w16 : c.b16, w ? kW16Ld : c.ldw, d.b_r0 + d.n, d.b_c0 + d.k, BN, err))
            return -1;
        p.a_kwrap = d.a_kwrap;
        p.check_seq = d.check_seq;
        p.chk_r0 = d.chk_r0;
        p.chk_c0 = d.chk_c0;
        p.m = d.m;
        p.n = d.n;
        p.k = d.k;
        p.a_r0 = d.a_r0;
        p.a_c0 = d.a_c0;
        p.b_r0 = d.b_r0;
        p.b_c0 = d.b_c0;
        p.c_r0 = d.c_r0;
        p.c_c0 = d.c_c0;
        p.exec_level = d.exec_level;
        p.lower = d.lower;
        p.alpha = d.alpha;
        p.beta = d.beta;
        p.tile0 = tiles;
        p.tiles_n = (d.n + BN - 1) / BN;
        tiles += ((d.m + BM - 1) / BM) * p.tiles_n;
    }
    return tiles;
}

static int g_sms = 148;

void init_tc_attributes() {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
}

void launch_gemm_tc(const DevCtx& c, const void* d_probs, int nprob, int tiles, cudaStream_t s) {
    if (tiles <= 0) return;
    const int grid = tiles < g_sms ? tiles : g_sms;
    k_gemm_tc<<<grid, NTHREADS, SMEM_BYTES, s>>>(c, static_cast<const TcProb*>(d_probs), nprob, tiles);
}

}  // namespace tcb
