// k_gemm_tc.cu -- grouped GEMM on the 5th-generation tensor cores.
//
//   C(i,j) <- rn_exec( rn_f32(alpha*s) + rn_f32(beta*C(i,j)) ),
//   s = sum_t A(i,t) * B(j,t)   (FP32 sums in TMEM)
//
// This is gemm_mixed / syrk_leaf (kernels.cpp:94-132) for two operand
// classes, one template:
//
//  KIND_F16   FP16-valued operands, tcgen05 kind::f16 -- exec level F16 (82%
//             of the flops at N=65536 [F16,F16,F16,F32]) and F32 exec on FP16
//             panels (16.4%): products of two binary16 values are exact in
//             binary32, so the reference's rn_f32(a*b) is the identity and an
//             FP32 accumulator implements the same arithmetic model (SURVEY
//             headline fact 3).
//  KIND_TF32X3  FP32 x FP32 operands (F32 exec, 1.6%): each operand is split
//             x = hi + lo with hi = x truncated to TF32 (exact) and lo = x - hi
//             (exact in FP32), and s = sum lo_a*hi_b + hi_a*lo_b + hi_a*hi_b
//             on kind::tf32 -- ~22 significant bits per operand, FP32 sums
//             (the reference rounds each product to FP32, kernels.cpp:29-30).
//             The tensor core reads the staged FP32 x as its TF32 hi (it drops
//             the 13 low mantissa bits); converter warps write lo = x - hi
//             next to it in shared memory, so the operands are read from HBM
//             once.
//
// Structure (one persistent CTA per SM, warp-specialised):
//   warp 0      TMA producer: 128x(128 B) A and BNx(128 B) B tiles, SWIZZLE_128B,
//               STAGES-deep smem ring guarded by full/empty mbarriers
//   warp 1      TMEM allocator + MMA issuer: one elected lane issues
//               tcgen05.mma.cta_group::1 (M=128, N=BN) into a double-buffered
//               FP32 accumulator (2 x BN TMEM columns)
//   warps 2-9   epilogue, two warps per TMEM lane quarter (one per column
//               half): C prefetched one 32-column chunk ahead, tcgen05.ld
//               32x32b -> registers -> dot_update tail -> rounding to the
//               destination level -> global (row-major C); fused
//               require_finite as one OR per element, located only on failure
//   warps 10-13 (TF32X3 only) lo half of each stage, then a
//               fence.proxy.async so the tensor core sees the generic writes
// A problem list (one tree_syrk = all its output blocks, or one trsm GEMM)
// is flattened into 128xBN tiles; each problem has its own pair of TMA
// descriptors whose extents end at the problem's edge, so partial tiles are
// zero-filled by the TMA unit and K need not be a multiple of the k-block.
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
    CUtensorMap tcm; // C rows [c_r0, c_r0+m) x cols [c_c0, c_c0+n) at the exec level (128 x 128-byte boxes)
    CUtensorMap tbh; // B as tb, 128-row boxes: one CTA's half of a CTA pair's 256-row B tile (FP16 kind)
    int m, n, k;
    int a_r0, a_c0, b_r0, b_c0, c_r0, c_c0;
    int exec_level, lower, tile0, tiles_n;
    double alpha, beta;
    int a_kwrap;  // inverse solve: A columns repeat with this period (B = [W_hi | W_lo])
    uint32_t check_seq;  // fused require_finite (0 = none), element relative to chk origin
    int chk_r0, chk_c0;
    int nkc, kb_per_chunk;  // FP32-exec K chunks (1, 0: one accumulation)
    int c_tma;              // C's columns start 16-byte aligned: epilogue through TMA boxes
    int ya, yb, yc;         // first row of each map (the level buffer window): TMA y = row - y*
};

size_t tc_prob_size() { return sizeof(TcProb); }

namespace {

constexpr int BM = 128;

// Optional K chunking of FP32-exec accumulations (tc_set_global_option
// "tc_kchunk", in K elements; 0 = off, the default).  The tensor core
// truncates when it adds into its FP32 accumulator, so one long accumulation
// drifts with the sign of the sum: at k = 32768 the drift is ~17x the RMS
// error of the reference's sequential round-to-nearest sum
// (tools/gemm_acc_probe.py).  With chunks, each chunk's TMEM sum is added
// into C by the epilogue.  On the factorization's diagonally dominant inputs
// |C| >> |s| (the diagonal carries n), so those extra roundings at C's
// magnitude cost more than the drift saves: C3's backward error goes from
// 8.65e-7 to 1.18e-6 and the step from 137 to 158 ms with 1024-chunks, while
// without them the N=16384 factor is already within the oracle's error
// (1.5745e-6 vs 1.5766e-6).  Hence off by default.
int g_tc_kchunk = 0;

// per operand kind: tile width, k-block (one 128-byte swizzled row), ring
// depth, threads, TMEM columns and the instruction descriptor
//   idesc: D=F32 (bits 4-5 = 1), A/B format at bits 7-9 / 10-12 (F16 = 0,
//   TF32 = 2), both K-major, N>>3 at bits 17-22, M>>4 at bits 24-28
template <int KIND> struct Cfg;
#ifndef TC_F16_STAGES
#define TC_F16_STAGES 4  // smem ring depth of the FP16 kind (3: 16384^3 1371 vs 1592 TF/s)
#endif
#ifndef TC_F16_STG
#define TC_F16_STG 2     // C staging boxes (16 KB each) of the FP16 kind
#endif
template <> struct Cfg<KIND_F16> {
    static constexpr int BN = 256, ESZ = 2, BK = 64, STAGES = TC_F16_STAGES, NTHREADS = 320, PASSES = 1,
                         STG_BOXES = TC_F16_STG;
    static constexpr uint32_t FMT = 0;
};
// the FP16 kind on 128x128 tiles: twice the CTAs of a 128x256 tiling for the
// skinny TRSM updates (m x 256 x 512 and the like), whose 64-128 tiles leave
// most SMs idle; same K order per element as KIND_F16 (bit-identical)
template <> struct Cfg<KIND_F16N> {
    static constexpr int BN = 128, ESZ = 2, BK = 64, STAGES = 6, NTHREADS = 320, PASSES = 1, STG_BOXES = 2;
    static constexpr uint32_t FMT = 0;
};
template <> struct Cfg<KIND_TF32X3> {
    static constexpr int BN = 128, ESZ = 4, BK = 32, STAGES = 3, NTHREADS = 448, PASSES = 3, STG_BOXES = 2;
    static constexpr uint32_t FMT = 2;
};
template <int KIND> struct Geo {
    using C = Cfg<KIND>;
    static constexpr int BN = C::BN, BK = C::BK, STAGES = C::STAGES;
    static constexpr int A_BYTES = BM * 128;  // one 128-byte row per tile row
    static constexpr int B_BYTES = BN * 128;
    static constexpr int TILE_BYTES = A_BYTES + B_BYTES;  // TMA bytes per stage
    // TF32X3 keeps a lo copy of both tiles next to the (hi) TMA tiles
    static constexpr int STAGE_BYTES = TILE_BYTES * (C::PASSES > 1 ? 2 : 1);
    // C staging for the epilogue: STG_BOXES boxes of 128 rows x 128 bytes
    // (SWIZZLE_128B, the TMA load / store layout of C)
    static constexpr int STG_BYTES = C::STG_BOXES * BM * 128;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + STG_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulators
    static constexpr uint32_t IDESC = (1u << 4) | (C::FMT << 7) | (C::FMT << 10) | (uint32_t(BN >> 3) << 17) |
                                      (uint32_t(BM >> 4) << 24);
    static_assert(STAGES * STAGE_BYTES + STG_BYTES + 1024 + 256 <= 227 * 1024, "shared memory");
};

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

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// the 8 epilogue warps only (named barrier 1)
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B (layout type 2 at
// bits 61-63), SBO = 1024 B between 8-row groups, LBO unused (1), version 1
__device__ __forceinline__ uint64_t sdesc(const void* p) {
    const uint64_t a = smem_u32(p);
    return ((a >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

template <int KIND>
__device__ __forceinline__ void mma_issue(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    if constexpr (KIND != KIND_TF32X3)
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(Geo<KIND>::IDESC), "r"(accum));
    else
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(Geo<KIND>::IDESC), "r"(accum));
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

__device__ __forceinline__ void stamp(const DevCtx& c, int slot) {
    if (c.stamps && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        c.stamps[slot] = t;
    }
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
template <int BN, int BMT = BM>
__device__ __forceinline__ bool tile_coords(const TcProb* probs, int np, int t, int& pi, int& tm, int& tn) {
    pi = find_tc_prob(probs, np, t);
    const TcProb& p = probs[pi];
    const int lt = t - p.tile0;
    // grouped raster: bands of GROUP tile rows, column-major inside a band,
    // so the CTAs resident at once share a few A and B panels per k-block
    // (L2 reuse; a plain row-major order streams ~tiles_n B panels from DRAM)
    constexpr int GROUP = 16 * BM / BMT;
    const int tiles_m = (p.m + BMT - 1) / BMT;
    const int band = GROUP * p.tiles_n;
    const int g = lt / band, r = lt - g * band;
    const int rows = min(GROUP, tiles_m - g * GROUP);
    tm = g * GROUP + r % rows;
    tn = r / rows;
    return !(p.lower && p.c_c0 + tn * BN > p.c_r0 + tm * BMT + BMT - 1);
}

// dot_update's tail (kernels.cpp:33-37) for an FP32 accumulator s:
// r = rn_f32(alpha*s); if beta != 0: r = rn_f32(r + rn_f32(beta*c)).  The
// fast form covers alpha = +-2^e (alpha*s exact in FP32 exactly when it is
// in double, then rounded once) and beta in {0, 1}; the rest goes through
// double like the reference.
struct Epi {
    bool fast;
    float af;
    double alpha, beta;
    __device__ __forceinline__ float operator()(float s, float cv) const {
        if (fast) return beta != 0.0 ? af * s + cv : af * s;
        float r = __double2float_rn(alpha * double(s));
        if (beta != 0.0) r = r + (beta == 1.0 ? cv : __double2float_rn(beta * double(cv)));
        return r;
    }
};
__device__ __forceinline__ bool pow2_or_one(double a) {
    const unsigned long long b = __double_as_longlong(a) & 0x7fffffffffffffffull;
    const int e = int(b >> 52);
    return (b & 0xfffffffffffffull) == 0 && e > 1023 - 100 && e < 1023 + 100;
}

// one 32-column chunk of C for one row: 32 halves (4 x uint4) or 32 floats
// (8 x float4); prefetched a chunk ahead of its use
struct CChunk {
    uint4 r[8];
};
__device__ __forceinline__ void load_chunk(CChunk& ch, const void* p, bool f16) {
    const uint4* q = static_cast<const uint4*>(p);
#pragma unroll
    for (int g = 0; g < 8; ++g)
        if (!f16 || g < 4) ch.r[g] = __ldcg(q + g);
}

// lo half of one staged tile pair for the three-pass TF32 product: the
// tensor core reads an FP32 element as TF32 by dropping its 13 low mantissa
// bits, so the staged x already is hi; lo = x - hi (exact) goes next to it.
// Elementwise, so the TMA swizzle is preserved.  128 threads.  (Writing hi
// back as well measured 23% slower on 4096^3, bit-identical results: the
// stage is shared-memory-bandwidth bound.)
__device__ __forceinline__ void split_tf32(const unsigned char* hi, unsigned char* lo, int bytes, int t) {
    const float4* h = reinterpret_cast<const float4*>(hi);
    float4* l = reinterpret_cast<float4*>(lo);
    const int n4 = bytes / 16;
#pragma unroll 4
    for (int e = t; e < n4; e += 128) {
        const float4 x = h[e];
        float4 y;
        y.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
        y.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
        y.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
        y.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
        l[e] = y;
    }
}

template <int KIND>
__global__ void __launch_bounds__(Cfg<KIND>::NTHREADS, 1) k_gemm_tc(DevCtx c, const TcProb* __restrict__ probs,
                                                                    int np, int tiles) {
    using G = Geo<KIND>;
    constexpr int BN = G::BN, STAGES = G::STAGES;
    constexpr bool SPLIT = Cfg<KIND>::PASSES > 1;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                           ~uintptr_t(1023));
    // stage s: A (hi) | B (hi) [| A lo | B lo]
    auto sA = [&](int s) { return smem + s * G::STAGE_BYTES; };
    auto sB = [&](int s) { return smem + s * G::STAGE_BYTES + G::A_BYTES; };
    auto sAl = [&](int s) { return smem + s * G::STAGE_BYTES + G::TILE_BYTES; };
    auto sBl = [&](int s) { return smem + s * G::STAGE_BYTES + G::TILE_BYTES + G::A_BYTES; };
    unsigned char* stg = smem + STAGES * G::STAGE_BYTES;  // C staging (1024-aligned)
    uint64_t* full = reinterpret_cast<uint64_t*>(stg + G::STG_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* split = empty + STAGES;  // TF32X3: hi/lo ready
    uint64_t* tfull = split + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* cfull = tempty + 2;      // C staged
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) stamp(c, 0);

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
            mbar_init(&split[s], 4);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 8);
        }
        mbar_init(cfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(G::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) stamp(c, 1);
    // setup done: from here on operands written by the preceding kernels are read
    pdl_wait();

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer ----------------
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                int pi, tm, tn;
                if (!tile_coords<BN>(probs, np, t, pi, tm, tn)) continue;
                const TcProb* p = probs + pi;
                prefetch_map(&p->ta);
                prefetch_map(&p->tb);
                prefetch_map(&p->tcm);  // the epilogue's C loads / stores
                const int nk = (p->k + G::BK - 1) / G::BK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], G::TILE_BYTES);
                    const int ka = p->a_kwrap ? (kb * G::BK) % p->a_kwrap : kb * G::BK;
                    tma_load_2d(sA(stage), &p->ta, &full[stage], p->a_c0 + ka, p->a_r0 - p->ya + tm * BM);
                    tma_load_2d(sB(stage), &p->tb, &full[stage], p->b_c0 + kb * G::BK, p->b_r0 - p->yb + tn * BN);
                    if (kb == 0) stamp(c, 2);
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
            if (!tile_coords<BN>(probs, np, t, pi, tm, tn)) continue;
            const int nk = (probs[pi].k + G::BK - 1) / G::BK;
            const int nkc = probs[pi].nkc;
            const int KB_PER_CHUNK = probs[pi].kb_per_chunk;
            for (int kc = 0; kc < nkc; ++kc) {
            mbar_wait(&tempty[as], aphase ^ 1);
            tc_fence_after();
            const uint32_t dcol = tmem + uint32_t(as * BN);
            const int kb0 = nkc > 1 ? kc * KB_PER_CHUNK : 0;
            const int kb1 = nkc > 1 ? min(nk, kb0 + KB_PER_CHUNK) : nk;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(SPLIT ? &split[stage] : &full[stage], phase);
                tc_fence_after();
                if (lane == 0 && kb == kb0) stamp(c, 3);
                if (lane == 0) {
                    const uint64_t da = sdesc(sA(stage));
                    const uint64_t db = sdesc(sB(stage));
                    // 4 MMAs per 128-byte k-block: +32 bytes (2 in the >>4
                    // address field) per K=16 (f16) / K=8 (tf32) step
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t o = uint64_t(2 * k);
                        if constexpr (SPLIT) {
                            // small terms first: lo*hi + hi*lo + hi*hi
                            const uint64_t dal = sdesc(sAl(stage)), dbl = sdesc(sBl(stage));
                            mma_issue<KIND>(dcol, dal + o, db + o, ((kb - kb0) | k) != 0);
                            mma_issue<KIND>(dcol, da + o, dbl + o, 1);
                            mma_issue<KIND>(dcol, da + o, db + o, 1);
                        } else {
                            mma_issue<KIND>(dcol, da + o, db + o, ((kb - kb0) | k) != 0);
                        }
                    }
                    mma_commit(&empty[stage]);
                    if (kb == kb1 - 1) mma_commit(&tfull[as]);
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
            }  // chunks
        }
        // every MMA issued: the dependents may be scheduled (they wait for
        // this grid's completion in pdl_wait)
        pdl_trigger();
    } else if (warp >= 10) {
        // ---------------- lo halves (TF32X3) ----------------
        if constexpr (SPLIT) {
            const int t128 = threadIdx.x - 10 * 32;
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                int pi, tm, tn;
                if (!tile_coords<BN>(probs, np, t, pi, tm, tn)) continue;
                const int nk = (probs[pi].k + G::BK - 1) / G::BK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    split_tf32(sA(stage), sAl(stage), G::A_BYTES, t128);
                    split_tf32(sB(stage), sBl(stage), G::B_BYTES, t128);
                    // generic-proxy smem writes -> visible to the tensor core
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&split[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else {
        // ---------------- epilogue (warps 2..9) ----------------
        // C goes through shared memory in TMA boxes (128 rows x 128 bytes,
        // SWIZZLE_128B): loaded by one bulk-tensor copy, updated in place by
        // the thread that owns each row (TMEM lane = row), stored back by one
        // bulk-tensor copy.  Direct per-thread global access would touch 32
        // rows -- 32 separate sectors -- per warp instruction.  A round covers
        // the columns the staging holds (256 F16 / 128 F32 for the FP16 kind,
        // 64 for TF32X3); warp (q, h) takes rows q*32.., half h of the round.
        const int q = warp & 3;             // TMEM lane quarter this warp may access
        const int half = (warp - 2) >> 2;   // column half of the round
        const bool leader = warp == 2 && lane == 0;
        const int row_l = q * 32 + lane;    // row inside the tile
        int as = 0;
        uint32_t aphase = 0, cphase = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            int pi, tm, tn;
            if (!tile_coords<BN>(probs, np, t, pi, tm, tn)) continue;
            const TcProb& p = probs[pi];
            if (!p.c_tma) {
                // C columns not 16-byte aligned in global memory (ragged
                // leaf sizes): direct per-thread access, C prefetched one
                // 32-column chunk ahead
                constexpr int HW = BN / 2;          // columns per epilogue warp
                const int nkc = p.nkc;
                for (int kc = 0; kc < nkc; ++kc) {
                const bool last_chunk = kc == nkc - 1;
                const int i = tm * BM + q * 32 + lane;  // row of C inside the problem
                const bool row_ok = i < p.m;
                const bool f16 = p.exec_level == LV_F16;
                const long long rowoff = (long long)(p.c_r0 + (row_ok ? i : 0)) * c.ldw + p.c_c0;
                Epi epi;
                // inverse solves carry W scaled by 2^e; undo it exactly here
                epi.alpha = p.a_kwrap ? double(c.wscale[p.b_r0]) : p.alpha;
                // later K chunks add into the C the previous chunk wrote (FP32)
                epi.beta = kc == 0 ? p.beta : 1.0;
                epi.fast = pow2_or_one(epi.alpha) && (epi.beta == 0.0 || epi.beta == 1.0);
                epi.af = float(epi.alpha);
                const bool has_c = epi.beta != 0.0;
                // columns [jlo, jhi) of this row are written (bounds, lower mask)
                const int jbase = tn * BN + half * HW;
                int jhi = min(p.n, jbase + HW);
                if (p.lower) jhi = min(jhi, (p.c_r0 + i) - p.c_c0 + 1);
                const int nch = row_ok && jhi > jbase ? (jhi - jbase + 31) >> 5 : 0;  // live chunks
                auto cptr = [&](int j0) -> const void* {
                    return f16 ? static_cast<const void*>(c.b16 + rowoff + j0) : static_cast<const void*>(c.b32 + rowoff + j0);
                };
                auto full_chunk = [&](int j0) {
                    return j0 + 32 <= jhi && ((reinterpret_cast<uintptr_t>(cptr(j0)) & 15) == 0);
                };
                // C of the first chunk does not depend on the accumulator: load it
                // before waiting for the MMA
                CChunk cur, nxt;
                if (has_c && nch > 0 && full_chunk(jbase)) load_chunk(cur, cptr(jbase), f16);
                mbar_wait(&tfull[as], aphase);
                tc_fence_after();
                uint32_t anybad = 0;
                int badj = -1;
                for (int cc = 0; cc < HW; cc += 32) {
                    float v[32];
                    __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge first
                    tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(as * BN + half * HW + cc), v);
                    if (cc == HW - 32) {
                        // accumulator drained: hand it back to the MMA warp
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[as]);
                    }
                    const int ch = cc >> 5;
                    if (ch >= nch) continue;
                    const int j0 = jbase + cc;
                    if (has_c && ch + 1 < nch && full_chunk(j0 + 32)) load_chunk(nxt, cptr(j0 + 32), f16);
                    uint32_t bad = 0;
                    if (full_chunk(j0)) {
                        if (f16) {
                            uint4* C = reinterpret_cast<uint4*>(c.b16 + rowoff + j0);
    #pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                uint4 raw = has_c ? cur.r[g] : make_uint4(0, 0, 0, 0);
                                uint32_t* w = reinterpret_cast<uint32_t*>(&raw);
    #pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const float2 cf = __half22float2(*reinterpret_cast<__half2*>(&w[e]));
                                    const __half2 o = __floats2half2_rn(epi(v[8 * g + 2 * e], cf.x),
                                                                        epi(v[8 * g + 2 * e + 1], cf.y));
                                    w[e] = *reinterpret_cast<const uint32_t*>(&o);
                                    bad |= ((w[e] & 0x7c00u) == 0x7c00u) | ((w[e] & 0x7c000000u) == 0x7c000000u);
                                }
                                C[g] = raw;
                            }
                        } else {
                            float4* C = reinterpret_cast<float4*>(c.b32 + rowoff + j0);
    #pragma unroll
                            for (int g = 0; g < 8; ++g) {
                                float4 cv = has_c ? *reinterpret_cast<const float4*>(&cur.r[g]) : make_float4(0, 0, 0, 0);
                                cv.x = epi(v[4 * g + 0], cv.x);
                                cv.y = epi(v[4 * g + 1], cv.y);
                                cv.z = epi(v[4 * g + 2], cv.z);
                                cv.w = epi(v[4 * g + 3], cv.w);
                                bad |= ((__float_as_uint(cv.x) & 0x7f800000u) == 0x7f800000u) |
                                       ((__float_as_uint(cv.y) & 0x7f800000u) == 0x7f800000u) |
                                       ((__float_as_uint(cv.z) & 0x7f800000u) == 0x7f800000u) |
                                       ((__float_as_uint(cv.w) & 0x7f800000u) == 0x7f800000u);
                                C[g] = cv;
                            }
                        }
                    } else {
                        // ragged / unaligned chunk: element by element
                        const int jm = min(32, jhi - j0);
    #pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (e < jm) {
                                if (f16) {
                                    __half* C = c.b16 + rowoff + j0 + e;
                                    const __half o = f2h(epi(v[e], has_c ? __half2float(*C) : 0.f));
                                    bad |= h_bad(o);
                                    *C = o;
                                } else {
                                    float* C = c.b32 + rowoff + j0 + e;
                                    const float o = epi(v[e], has_c ? *C : 0.f);
                                    bad |= !isfinite(o);
                                    *C = o;
                                }
                            }
                    }
                    if (bad && badj < 0) {
                        // locate the first non-finite value of this chunk (rare path)
                        const int jm = min(32, jhi - j0);
                        for (int e = 0; e < jm && badj < 0; ++e) {
                            const bool b = f16 ? h_bad(c.b16[rowoff + j0 + e]) : !isfinite(c.b32[rowoff + j0 + e]);
                            if (b) badj = j0 + e;
                        }
                    }
                    anybad |= bad;
                    cur = nxt;
                }
                if (p.check_seq != 0 && last_chunk) {
                    // fused require_finite: first bad element in column-major order
                    unsigned long long key = ~0ull;
                    if (badj >= 0)
                        key = fail_key(p.check_seq, elem_local(p.c_r0 + i - p.chk_r0, p.c_c0 + badj - p.chk_c0));
                    __syncwarp();
                    warp_report_min(c, key);
                }
                (void)anybad;
                if (++as == 2) {
                    as = 0;
                    aphase ^= 1;
                }
                }  // chunks
                continue;
            }
            const int nkc = p.nkc;
            const bool f16 = p.exec_level == LV_F16;
            const int box_cols = f16 ? 64 : 32;                 // columns per 128-byte box
            const int rc = min(BN, Cfg<KIND>::STG_BOXES * box_cols);  // columns per round
            const int rounds = BN / rc;
            const int hw = rc / 2;                              // columns per warp per round
            const int i = tm * BM + row_l;                      // row of C inside the problem
            const bool row_ok = i < p.m;
            for (int kc = 0; kc < nkc; ++kc) {
            const bool last_chunk = kc == nkc - 1;
            Epi epi;
            // inverse solves carry W scaled by 2^e; undo it exactly here
            epi.alpha = p.a_kwrap ? double(c.wscale[p.b_r0]) : p.alpha;
            // later K chunks add into the C the previous chunk wrote (FP32)
            epi.beta = kc == 0 ? p.beta : 1.0;
            epi.fast = pow2_or_one(epi.alpha) && (epi.beta == 0.0 || epi.beta == 1.0);
            epi.af = float(epi.alpha);
            const bool has_c = epi.beta != 0.0;
            // lower tiles write back the staged C above the diagonal untouched
            const bool load_c = has_c || p.lower;
            // columns [.., jhi) of this row are computed (bounds, lower mask)
            int jhi = p.n;
            if (p.lower) jhi = min(jhi, (p.c_r0 + i) - p.c_c0 + 1);
            if (!row_ok) jhi = 0;
            int badj = -1;
            for (int rd = 0; rd < rounds; ++rd) {
                const int col0 = tn * BN + rd * rc;  // first column of the round (in the problem)
                // boxes with columns inside the problem (0: a round past its
                // edge -- its TMEM columns are still read, for the hand-back)
                const int nbox = col0 < p.n ? min(Cfg<KIND>::STG_BOXES, (p.n - col0 + box_cols - 1) / box_cols) : 0;
                const bool do_load = load_c && nbox > 0;
                // the staging is free once the previous round's store has read it
                if (leader) {
                    bulk_wait_read0();
                    if (do_load) {
                        mbar_expect_tx(cfull, uint32_t(nbox) * BM * 128);
                        for (int bx = 0; bx < nbox; ++bx)
                            tma_load_2d(stg + bx * BM * 128, &p.tcm, cfull, p.c_c0 + col0 + bx * box_cols,
                                        p.c_r0 - p.yc + tm * BM);
                    }
                }
                if (rd == 0) {
                    mbar_wait(&tfull[as], aphase);
                    tc_fence_after();
                    if (warp == 2 && lane == 0) stamp(c, 4);
                }
                if (do_load) {
                    mbar_wait(cfull, cphase);
                    cphase ^= 1;
                    if (leader) stamp(c, 7);
                } else {
                    epi_sync();  // nobody writes the staging before the leader's wait above
                }
                for (int cc = 0; cc < hw; cc += 32) {
                    float v[32];
                    const int jt = rd * rc + half * hw + cc;   // column inside the tile
                    __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge first
                    if (leader && cc == 0) stamp(c, 11);
                    tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(as * BN + jt), v);
                    if (leader && cc == 0) stamp(c, 12);
                    if (leader && cc == 32) stamp(c, 14);
                    if (rd == rounds - 1 && cc == hw - 32) {
                        // accumulator drained: hand it back to the MMA warp
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tempty[as]);
                    }
                    const int j0 = tn * BN + jt;               // column inside the problem
                    if (j0 >= jhi) continue;
                    const int jm = min(32, jhi - j0);          // live columns of this chunk
                    // swizzled 16-byte chunks of this row inside its box
                    const int bx = (jt - rd * rc) / box_cols;
                    unsigned char* rowp = stg + bx * BM * 128 + row_l * 128;
                    const int c16 = ((jt - rd * rc) % box_cols) * (f16 ? 2 : 4) / 16;  // first 16-byte chunk
                    uint32_t bad = 0;
                    if (epi.fast && jm == 32) {
                        // common case (alpha = +-2^e, beta in {0, 1}, a full
                        // chunk): straight-line FP32, no per-element branches
                        const float af = epi.af;
                        if (f16) {
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                uint4* cp = reinterpret_cast<uint4*>(rowp + (((c16 + g) ^ (row_l & 7)) << 4));
                                uint4 raw = has_c ? *cp : make_uint4(0, 0, 0, 0);
                                uint32_t* w = reinterpret_cast<uint32_t*>(&raw);
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const float2 cf = __half22float2(*reinterpret_cast<__half2*>(&w[e]));
                                    const __half2 o = __floats2half2_rn(fmaf(af, v[8 * g + 2 * e], cf.x),
                                                                        fmaf(af, v[8 * g + 2 * e + 1], cf.y));
                                    w[e] = *reinterpret_cast<const uint32_t*>(&o);
                                    bad |= ((w[e] & 0x7c00u) == 0x7c00u) | ((w[e] & 0x7c000000u) == 0x7c000000u);
                                }
                                *cp = raw;
                            }
                        } else {
#pragma unroll
                            for (int g = 0; g < 8; ++g) {
                                float4* cp = reinterpret_cast<float4*>(rowp + (((c16 + g) ^ (row_l & 7)) << 4));
                                float4 o = has_c ? *cp : make_float4(0.f, 0.f, 0.f, 0.f);
                                o.x = fmaf(af, v[4 * g + 0], o.x);
                                o.y = fmaf(af, v[4 * g + 1], o.y);
                                o.z = fmaf(af, v[4 * g + 2], o.z);
                                o.w = fmaf(af, v[4 * g + 3], o.w);
                                bad |= ((__float_as_uint(o.x) & 0x7f800000u) == 0x7f800000u) |
                                       ((__float_as_uint(o.y) & 0x7f800000u) == 0x7f800000u) |
                                       ((__float_as_uint(o.z) & 0x7f800000u) == 0x7f800000u) |
                                       ((__float_as_uint(o.w) & 0x7f800000u) == 0x7f800000u);
                                *cp = o;
                            }
                        }
                    } else if (f16) {
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            uint4* cp = reinterpret_cast<uint4*>(rowp + (((c16 + g) ^ (row_l & 7)) << 4));
                            uint4 orig = load_c ? *cp : make_uint4(0, 0, 0, 0);  // staged (masked columns)
                            uint4 raw = has_c ? orig : make_uint4(0, 0, 0, 0);
                            uint32_t* w = reinterpret_cast<uint32_t*>(&raw);
                            uint32_t* wo = reinterpret_cast<uint32_t*>(&orig);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int jj = 8 * g + 2 * e;
                                const float2 cf = __half22float2(*reinterpret_cast<__half2*>(&w[e]));
                                const __half2 o = __floats2half2_rn(epi(v[jj], cf.x), epi(v[jj + 1], cf.y));
                                uint32_t ou = *reinterpret_cast<const uint32_t*>(&o);
                                // masked columns keep the staged C
                                if (jj >= jm) ou = (ou & 0xFFFF0000u) | (wo[e] & 0xFFFFu);
                                if (jj + 1 >= jm) ou = (ou & 0xFFFFu) | (wo[e] & 0xFFFF0000u);
                                w[e] = ou;
                                bad |= (jj < jm && (ou & 0x7c00u) == 0x7c00u) |
                                       (jj + 1 < jm && (ou & 0x7c000000u) == 0x7c000000u);
                            }
                            *cp = raw;
                        }
                    } else {
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            float4* cp = reinterpret_cast<float4*>(rowp + (((c16 + g) ^ (row_l & 7)) << 4));
                            const float4 co = has_c ? *cp : make_float4(0, 0, 0, 0);
                            const float4 cm = p.lower ? *cp : co;  // staged values (masked columns)
                            float4 o;
                            const int jj = 4 * g;
                            o.x = jj + 0 < jm ? epi(v[jj + 0], co.x) : cm.x;
                            o.y = jj + 1 < jm ? epi(v[jj + 1], co.y) : cm.y;
                            o.z = jj + 2 < jm ? epi(v[jj + 2], co.z) : cm.z;
                            o.w = jj + 3 < jm ? epi(v[jj + 3], co.w) : cm.w;
                            bad |= (jj + 0 < jm && (__float_as_uint(o.x) & 0x7f800000u) == 0x7f800000u) |
                                   (jj + 1 < jm && (__float_as_uint(o.y) & 0x7f800000u) == 0x7f800000u) |
                                   (jj + 2 < jm && (__float_as_uint(o.z) & 0x7f800000u) == 0x7f800000u) |
                                   (jj + 3 < jm && (__float_as_uint(o.w) & 0x7f800000u) == 0x7f800000u);
                            *cp = o;
                        }
                    }
                    if (leader && cc == 0) stamp(c, 13);
                    if (bad && badj < 0) {
                        // locate the first non-finite value of this chunk (rare path)
                        for (int e = 0; e < jm && badj < 0; ++e) {
                            const int cb = (c16 * 16 + e * (f16 ? 2 : 4)) / 16, off = (e * (f16 ? 2 : 4)) % 16;
                            const unsigned char* ep = rowp + ((cb ^ (row_l & 7)) << 4) + off;
                            const bool b = f16 ? h_bad(*reinterpret_cast<const __half*>(ep))
                                               : !isfinite(*reinterpret_cast<const float*>(ep));
                            if (b) badj = j0 + e;
                        }
                    }
                }
                // generic-proxy smem writes -> visible to the bulk copy; then
                // one thread stores the round's boxes
                if (leader) stamp(c, 8);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                epi_sync();
                if (leader) stamp(c, 9);
                if (leader && nbox > 0) {
                    for (int bx = 0; bx < nbox; ++bx)
                        tma_store_2d(&p.tcm, stg + bx * BM * 128, p.c_c0 + col0 + bx * box_cols,
                                     p.c_r0 - p.yc + tm * BM);
                    bulk_commit();
                }
            }
            if (p.check_seq != 0 && last_chunk) {
                // fused require_finite: first bad element in column-major order
                unsigned long long key = ~0ull;
                if (badj >= 0)
                    key = fail_key(p.check_seq, elem_local(p.c_r0 + i - p.chk_r0, p.c_c0 + badj - p.chk_c0));
                __syncwarp();
                warp_report_min(c, key);
            }
            if (++as == 2) {
                as = 0;
                aphase ^= 1;
            }
            }  // chunks
            // the next tile's staging loads wait for these stores (leader)
        }
        if (leader) stamp(c, 10);
        if (leader) bulk_wait0();  // every store complete before the CTA exits
    }

    if (warp == 2 && lane == 0) stamp(c, 5);
    tc_fence_before();
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(G::TMEM_COLS));
    if (threadIdx.x == 32) stamp(c, 6);
}

// ---------------------------------------------------------------------------
// CTA-pair variant of the FP16 kind (tcgen05.mma.cta_group::2): a cluster of
// two CTAs computes 256 x 256 tiles.  Each CTA stages its own 128 rows of A
// and one 128-row half of B per k-block (32 KB instead of 48 KB), the
// leader (rank 0) issues M=256, N=256 MMAs that read A from both CTAs' own
// halves and B from both halves, and each CTA's TMEM holds its 128 rows of
// the accumulator.  Per SM the operand bytes per flop fall by a third, and
// the ring holds 6 stages (1.1 us of MMA at full rate) instead of 4: the big
// trailing updates are short of operand latency hiding with 128x256 tiles.
// Barriers: full[s] in the leader (its expect_tx covers both CTAs' loads,
// which complete on it through .cta_group::2), empty[s] / tfull in both
// (the leader's commits multicast), tempty in the leader (both CTAs'
// epilogue warps arrive).  Epilogue as in k_gemm_tc (TMA-staged C only).
// ---------------------------------------------------------------------------
// per operand kind: FP16 (6 stages of A + half B) or TF32X3 (3 stages of A +
// half B + their lo halves, converter warps 10-13 in both CTAs)
template <int KIND> struct PairCfg;
template <> struct PairCfg<KIND_F16> {
    static constexpr int STAGES = 6, NTHREADS = 320, PASSES = 1, BK = 64;
    static constexpr uint32_t FMT = 0;
};
template <> struct PairCfg<KIND_TF32X3> {
    static constexpr int STAGES = 3, NTHREADS = 448, PASSES = 3, BK = 32;
    static constexpr uint32_t FMT = 2;
};
constexpr int P_BN = 256;                       // pair tile columns (N of the MMA)
constexpr int P_A_BYTES = BM * 128;             // this CTA's A rows, one k-block
constexpr int P_B_BYTES = BM * 128;             // this CTA's half of B
constexpr int P_TILE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr int P_STG_BYTES = 2 * BM * 128;
template <int KIND> struct PairGeo {
    using C = PairCfg<KIND>;
    static constexpr int STAGE_BYTES = P_TILE_BYTES * (C::PASSES > 1 ? 2 : 1);
    static constexpr int SMEM_BYTES = C::STAGES * STAGE_BYTES + P_STG_BYTES + 1024 + 256;
    static constexpr uint32_t IDESC = (1u << 4) | (C::FMT << 7) | (C::FMT << 10) | (uint32_t(P_BN >> 3) << 17) |
                                      (uint32_t((2 * BM) >> 4) << 24);
    static_assert(SMEM_BYTES <= 227 * 1024, "pair shared memory");
};
constexpr uint32_t P_TMEM_COLS = 2 * P_BN;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose completion goes to the leader's barrier (cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t mbar_cluster, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar_cluster), "r"(x), "r"(y)
        : "memory");
}
template <int KIND>
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    if constexpr (KIND == KIND_F16)
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(PairGeo<KIND>::IDESC), "r"(accum));
    else
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "setp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
            "}\n" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(PairGeo<KIND>::IDESC), "r"(accum));
}
// arrive on the barrier at this offset in both CTAs of the pair once the
// leader's MMAs so far have completed
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n"
        ".reg .b16 m;\n"
        "mov.b16 m, 3;\n"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
        "}\n" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(PairCfg<KIND>::NTHREADS, 1) k_gemm_tc2(DevCtx c, const TcProb* __restrict__ probs,
                                                                         int np, int tiles) {
    using G = PairGeo<KIND>;
    constexpr int P_STAGES = PairCfg<KIND>::STAGES, BKK = PairCfg<KIND>::BK;
    constexpr bool SPLIT = PairCfg<KIND>::PASSES > 1;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                           ~uintptr_t(1023));
    // stage: A | B half [| A lo | B half lo]
    auto sA = [&](int st) { return smem + st * G::STAGE_BYTES; };
    auto sB = [&](int st) { return smem + st * G::STAGE_BYTES + P_A_BYTES; };
    auto sAl = [&](int st) { return smem + st * G::STAGE_BYTES + P_TILE_BYTES; };
    auto sBl = [&](int st) { return smem + st * G::STAGE_BYTES + P_TILE_BYTES + P_A_BYTES; };
    unsigned char* stg = smem + P_STAGES * G::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(stg + P_STG_BYTES);
    uint64_t* empty = full + P_STAGES;
    uint64_t* split = empty + P_STAGES;  // TF32X3: both CTAs' lo halves written (leader's copy)
    uint64_t* tfull = split + P_STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* cfull = tempty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        for (int st = 0; st < P_STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], 1);
            mbar_init(&split[st], 8);  // 4 converter warps x 2 CTAs
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 16);  // 8 epilogue warps x 2 CTAs (leader's copy)
        }
        mbar_init(cfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(P_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();  // both CTAs' barriers initialised, TMEM allocated
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs) ----------------
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair; t < tiles; t += npairs) {
                int pi, tm, tn;
                if (!tile_coords<P_BN, 2 * BM>(probs, np, t, pi, tm, tn)) continue;
                const TcProb* p = probs + pi;
                prefetch_map(&p->ta);
                prefetch_map(&p->tbh);
                prefetch_map(&p->tcm);
                const int nk = (p->k + BKK - 1) / BKK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const int ka = p->a_kwrap ? (kb * BKK) % p->a_kwrap : kb * BKK;
                    const int ya = p->a_r0 - p->ya + tm * 2 * BM + int(rank) * BM;
                    const int yb = p->b_r0 - p->yb + tn * P_BN + int(rank) * BM;
                    if constexpr (SPLIT) {
                        // each CTA's loads complete on its own barrier: its
                        // converter warps need them before the leader's MMA
                        mbar_expect_tx(&full[stage], P_TILE_BYTES);
                        tma_load_2d(sA(stage), &p->ta, &full[stage], p->a_c0 + ka, ya);
                        tma_load_2d(sB(stage), &p->tbh, &full[stage], p->b_c0 + kb * BKK, yb);
                    } else {
                        if (leader) mbar_expect_tx(&full[stage], 2 * P_TILE_BYTES);
                        const uint32_t fb = mapa_rank(smem_u32(&full[stage]), 0);
                        tma_load_2d_pair(sA(stage), &p->ta, fb, p->a_c0 + ka, ya);
                        tma_load_2d_pair(sB(stage), &p->tbh, fb, p->b_c0 + kb * BKK, yb);
                    }
                    if (++stage == P_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader only) ----------------
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            int as = 0;
            uint32_t aphase = 0;
            for (int t = pair; t < tiles; t += npairs) {
                int pi, tm, tn;
                if (!tile_coords<P_BN, 2 * BM>(probs, np, t, pi, tm, tn)) continue;
                const int nk = (probs[pi].k + BKK - 1) / BKK;
                mbar_wait(&tempty[as], aphase ^ 1);
                tc_fence_after();
                const uint32_t dcol = tmem + uint32_t(as * P_BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(SPLIT ? &split[stage] : &full[stage], phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint64_t da = sdesc(sA(stage));
                        const uint64_t db = sdesc(sB(stage));
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint64_t o = uint64_t(2 * k);
                            if constexpr (SPLIT) {
                                // small terms first: lo*hi + hi*lo + hi*hi
                                const uint64_t dal = sdesc(sAl(stage)), dbl = sdesc(sBl(stage));
                                mma_pair<KIND>(dcol, dal + o, db + o, (kb | k) != 0);
                                mma_pair<KIND>(dcol, da + o, dbl + o, 1);
                                mma_pair<KIND>(dcol, da + o, db + o, 1);
                            } else {
                                mma_pair<KIND>(dcol, da + o, db + o, (kb | k) != 0);
                            }
                        }
                        mma_commit_pair(&empty[stage]);
                        if (kb == nk - 1) mma_commit_pair(&tfull[as]);
                    }
                    __syncwarp();
                    if (++stage == P_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (++as == 2) {
                    as = 0;
                    aphase ^= 1;
                }
            }
        }
    } else if (warp >= 10) {
        // ---------------- lo halves (TF32X3, both CTAs) ----------------
        if constexpr (SPLIT) {
            const int t128 = threadIdx.x - 10 * 32;
            const uint32_t split_leader = mapa_rank(smem_u32(&split[0]), 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair; t < tiles; t += npairs) {
                int pi, tm, tn;
                if (!tile_coords<P_BN, 2 * BM>(probs, np, t, pi, tm, tn)) continue;
                const int nk = (probs[pi].k + BKK - 1) / BKK;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(&full[stage], phase);
                    split_tf32(sA(stage), sAl(stage), P_A_BYTES, t128);
                    split_tf32(sB(stage), sBl(stage), P_B_BYTES, t128);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(split_leader + uint32_t(stage) * 8u);
                    if (++stage == P_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else {
        // ---------------- epilogue (warps 2..9, both CTAs) ----------------
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const bool ldr = warp == 2 && lane == 0;
        const int row_l = q * 32 + lane;
        const uint32_t tempty_leader0 = mapa_rank(smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa_rank(smem_u32(&tempty[1]), 0);
        int as = 0;
        uint32_t aphase = 0, cphase = 0;
        for (int t = pair; t < tiles; t += npairs) {
            int pi, tm, tn;
            if (!tile_coords<P_BN, 2 * BM>(probs, np, t, pi, tm, tn)) continue;
            const TcProb& p = probs[pi];
            const bool f16 = p.exec_level == LV_F16;
            const int box_cols = f16 ? 64 : 32;
            const int rc = min(P_BN, 2 * box_cols);  // columns per round
            const int rounds = P_BN / rc;
            const int hw = rc / 2;
            const int i = tm * 2 * BM + int(rank) * BM + row_l;  // row of C inside the problem
            const int crow = tm * 2 * BM + int(rank) * BM;        // first row of this CTA's half tile
            const bool row_ok = i < p.m;
            Epi epi;
            epi.alpha = p.a_kwrap ? double(c.wscale[p.b_r0]) : p.alpha;
            epi.beta = p.beta;
            epi.fast = pow2_or_one(epi.alpha) && (epi.beta == 0.0 || epi.beta == 1.0);
            epi.af = float(epi.alpha);
            const bool has_c = epi.beta != 0.0;
            const bool load_c = has_c || p.lower;
            int jhi = p.n;
            if (p.lower) jhi = min(jhi, (p.c_r0 + i) - p.c_c0 + 1);
            if (!row_ok) jhi = 0;
            const bool half_live = crow < p.m;  // this CTA's rows exist in the problem
            int badj = -1;
            for (int rd = 0; rd < rounds; ++rd) {
                const int col0 = tn * P_BN + rd * rc;
                const int nbox = (col0 < p.n && half_live) ? min(2, (p.n - col0 + box_cols - 1) / box_cols) : 0;
                const bool do_load = load_c && nbox > 0;
                if (ldr) {
                    bulk_wait_read0();
                    if (do_load) {
                        mbar_expect_tx(cfull, uint32_t(nbox) * BM * 128);
                        for (int bx = 0; bx < nbox; ++bx)
                            tma_load_2d(stg + bx * BM * 128, &p.tcm, cfull, p.c_c0 + col0 + bx * box_cols,
                                        p.c_r0 - p.yc + crow);
                    }
                }
                if (rd == 0) {
                    mbar_wait(&tfull[as], aphase);
                    tc_fence_after();
                }
                if (do_load) {
                    mbar_wait(cfull, cphase);
                    cphase ^= 1;
                } else {
                    epi_sync();
                }
                for (int cc = 0; cc < hw; cc += 32) {
                    float v[32];
                    const int jt = rd * rc + half * hw + cc;
                    __syncwarp();
                    tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(as * P_BN + jt), v);
                    if (rd == rounds - 1 && cc == hw - 32) {
                        // accumulator drained: tell the leader's MMA warp
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(as == 0 ? tempty_leader0 : tempty_leader1);
                    }
                    const int j0 = tn * P_BN + jt;
                    if (j0 >= jhi) continue;
                    const int jm = min(32, jhi - j0);
                    const int bx = (jt - rd * rc) / box_cols;
                    unsigned char* rowp = stg + bx * BM * 128 + row_l * 128;
                    const int c16 = ((jt - rd * rc) % box_cols) * (f16 ? 2 : 4) / 16;
                    uint32_t bad = 0;
                    if (f16) {
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            uint4* cp = reinterpret_cast<uint4*>(rowp + (((c16 + g) ^ (row_l & 7)) << 4));
                            uint4 orig = load_c ? *cp : make_uint4(0, 0, 0, 0);
                            uint4 raw = has_c ? orig : make_uint4(0, 0, 0, 0);
                            uint32_t* w = reinterpret_cast<uint32_t*>(&raw);
                            uint32_t* wo = reinterpret_cast<uint32_t*>(&orig);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int jj = 8 * g + 2 * e;
                                const float2 cf = __half22float2(*reinterpret_cast<__half2*>(&w[e]));
                                const __half2 o = epi.fast
                                                      ? __floats2half2_rn(fmaf(epi.af, v[jj], cf.x), fmaf(epi.af, v[jj + 1], cf.y))
                                                      : __floats2half2_rn(epi(v[jj], cf.x), epi(v[jj + 1], cf.y));
                                uint32_t ou = *reinterpret_cast<const uint32_t*>(&o);
                                if (jj >= jm) ou = (ou & 0xFFFF0000u) | (wo[e] & 0xFFFFu);
                                if (jj + 1 >= jm) ou = (ou & 0xFFFFu) | (wo[e] & 0xFFFF0000u);
                                w[e] = ou;
                                bad |= (jj < jm && (ou & 0x7c00u) == 0x7c00u) |
                                       (jj + 1 < jm && (ou & 0x7c000000u) == 0x7c000000u);
                            }
                            *cp = raw;
                        }
                    } else {
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            float4* cp = reinterpret_cast<float4*>(rowp + (((c16 + g) ^ (row_l & 7)) << 4));
                            const float4 co = has_c ? *cp : make_float4(0, 0, 0, 0);
                            const float4 cm = p.lower ? *cp : co;
                            float4 o;
                            const int jj = 4 * g;
                            o.x = jj + 0 < jm ? epi(v[jj + 0], co.x) : cm.x;
                            o.y = jj + 1 < jm ? epi(v[jj + 1], co.y) : cm.y;
                            o.z = jj + 2 < jm ? epi(v[jj + 2], co.z) : cm.z;
                            o.w = jj + 3 < jm ? epi(v[jj + 3], co.w) : cm.w;
                            bad |= (jj + 0 < jm && (__float_as_uint(o.x) & 0x7f800000u) == 0x7f800000u) |
                                   (jj + 1 < jm && (__float_as_uint(o.y) & 0x7f800000u) == 0x7f800000u) |
                                   (jj + 2 < jm && (__float_as_uint(o.z) & 0x7f800000u) == 0x7f800000u) |
                                   (jj + 3 < jm && (__float_as_uint(o.w) & 0x7f800000u) == 0x7f800000u);
                            *cp = o;
                        }
                    }
                    if (bad && badj < 0) {
                        for (int e = 0; e < jm && badj < 0; ++e) {
                            const int cb = (c16 * 16 + e * (f16 ? 2 : 4)) / 16, off = (e * (f16 ? 2 : 4)) % 16;
                            const unsigned char* ep = rowp + ((cb ^ (row_l & 7)) << 4) + off;
                            const bool b = f16 ? h_bad(*reinterpret_cast<const __half*>(ep))
                                               : !isfinite(*reinterpret_cast<const float*>(ep));
                            if (b) badj = j0 + e;
                        }
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                epi_sync();
                if (ldr && nbox > 0) {
                    for (int bx = 0; bx < nbox; ++bx)
                        tma_store_2d(&p.tcm, stg + bx * BM * 128, p.c_c0 + col0 + bx * box_cols, p.c_r0 - p.yc + crow);
                    bulk_commit();
                }
            }
            if (p.check_seq != 0) {
                unsigned long long key = ~0ull;
                if (badj >= 0)
                    key = fail_key(p.check_seq, elem_local(p.c_r0 + i - p.chk_r0, p.c_c0 + badj - p.chk_c0));
                __syncwarp();
                warp_report_min(c, key);
            }
            if (++as == 2) {
                as = 0;
                aphase ^= 1;
            }
        }
        if (ldr) bulk_wait0();
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer's last arrivals and TMEM reads are done
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P_TMEM_COLS));
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

// 2-D map over a row-major buffer, k-block wide (one 128-byte row) boxes
bool make_map(CUtensorMap* m, const void* base, bool f32, long long ldw, int rows_end, int cols_end, int box_rows,
              std::string* err) {
    auto enc = get_encode();
    if (!enc) {
        if (err) *err = "cuTensorMapEncodeTiled unavailable";
        return false;
    }
    const int esz = f32 ? 4 : 2;
    cuuint64_t dims[2] = {cuuint64_t(cols_end), cuuint64_t(rows_end)};
    cuuint64_t strides[1] = {cuuint64_t(ldw) * esz};
    cuuint32_t box[2] = {cuuint32_t(128 / esz), cuuint32_t(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                     const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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

int tc_build_probs(const DevCtx& c, int kind, const std::vector<DevProb>& probs, std::vector<unsigned char>& out,
                   std::string* err, int pair) {
    out.assign(probs.size() * sizeof(TcProb), 0);
    TcProb* tp = reinterpret_cast<TcProb*>(out.data());
    const bool f32 = kind == KIND_TF32X3;
    const int BN = f32 ? Cfg<KIND_TF32X3>::BN : kind == KIND_F16N ? Cfg<KIND_F16N>::BN : Cfg<KIND_F16>::BN;
    const void* obuf = f32 ? static_cast<const void*>(c.b32) : static_cast<const void*>(c.b16);
    int tiles = 0;
    for (size_t i = 0; i < probs.size(); ++i) {
        const DevProb& d = probs[i];
        TcProb& p = tp[i];
        // A extent ends at the problem's K edge (an inverse solve's A is the
        // n-wide leaf column block read twice: its extent is n, period a_kwrap)
        // maps start at the level buffer's first allocated row (the context's
        // bases are virtual: rows below the window are not memory)
        const int olv = f32 ? LV_F32 : LV_F16;
        const int ylo = c.win_lo[olv];
        const size_t oesz = f32 ? 4 : 2;
        const void* obase = static_cast<const unsigned char*>(obuf) + size_t(ylo) * size_t(c.ldw) * oesz;
        p.ya = ylo;
        if (!make_map(&p.ta, obase, f32, c.ldw, d.a_r0 + d.m - ylo, d.a_c0 + (d.a_kwrap ? d.n : d.k), BM, err))
            return -1;
        const bool bw = d.b_buf == BUF_W16 || d.b_buf == BUF_W32;
        const void* bbuf = d.b_buf == BUF_W16 ? static_cast<const void*>(c.w16)
                           : d.b_buf == BUF_W32 ? static_cast<const void*>(c.w32)
                                                : obase;
        const long long bld = d.b_buf == BUF_W16 ? kW16Ld : d.b_buf == BUF_W32 ? kW32Ld : c.ldw;
        const bool bf32 = d.b_buf == BUF_W32 || (f32 && d.b_buf != BUF_W16);
        p.yb = bw ? 0 : ylo;
        if (!make_map(&p.tb, bbuf, bf32, bld, d.b_r0 + d.n - p.yb, d.b_c0 + d.k, BN, err)) return -1;
        if (!make_map(&p.tbh, bbuf, bf32, bld, d.b_r0 + d.n - p.yb, d.b_c0 + d.k, BM, err)) return -1;
        {
            const bool cf32 = d.exec_level == LV_F32;
            const void* cbuf = cf32 ? static_cast<const void*>(c.b32) : static_cast<const void*>(c.b16);
            if (d.exec_level != LV_F16 && !cf32) {
                if (err) *err = "tensor-core GEMM: exec level must be F16 or F32";
                return -1;
            }
            p.yc = c.win_lo[cf32 ? LV_F32 : LV_F16];
            const void* cbase = static_cast<const unsigned char*>(cbuf) + size_t(p.yc) * size_t(c.ldw) * (cf32 ? 4 : 2);
            if (!make_map(&p.tcm, cbase, cf32, c.ldw, d.c_r0 + d.m - p.yc, d.c_c0 + d.n, BM, err)) return -1;
            // bulk-tensor boxes must start 16-byte aligned in global memory
            p.c_tma = (d.c_c0 * (cf32 ? 4 : 2)) % 16 == 0 && (c.ldw * (cf32 ? 4 : 2)) % 16 == 0;
        }
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
        p.tiles_n = (d.n + (pair ? P_BN : BN) - 1) / (pair ? P_BN : BN);
        {
            const int bk = f32 ? Cfg<KIND_TF32X3>::BK : Cfg<KIND_F16>::BK;
            const int kc = (g_tc_kchunk / bk) * bk;
            p.nkc = d.exec_level == LV_F32 && kc > 0 && d.k > kc ? (d.k + kc - 1) / kc : 1;
            p.kb_per_chunk = kc / bk;
        }
        const int bmt = pair ? 2 * BM : BM;  // CTA pairs: 256-row tiles
        tiles += ((d.m + bmt - 1) / bmt) * p.tiles_n;
        if (pair && (!p.c_tma || p.nkc != 1)) return -2;  // the pair kernel: TMA-staged C, one K chunk
    }
    return tiles;
}

// CTA pairs for FP16-kind problem lists of at least this many 128x256 tiles
// (0 = never); process-wide, read when a plan's tables are built.  Below ~2
// waves the pair's 256x256 tiles leave SMs idle (8192x1024x1024: 22 -> 26 us)
static int g_tc_pair_min_tiles = 512;
int tc_pair_min_tiles() { return g_tc_pair_min_tiles; }
static int g_tc_narrow_max_tiles = 0;
int tc_narrow_max_tiles() { return g_tc_narrow_max_tiles; }

int tc_select_tables(const DevCtx& c, bool tf32, const std::vector<DevProb>& probs, std::vector<unsigned char>& out,
                     std::string* err, int pair_min, int narrow_max, int* kind, int* pair) {
    *kind = tf32 ? KIND_TF32X3 : KIND_F16;
    *pair = 0;
    int tiles = tc_build_probs(c, *kind, probs, out, err);
    if (tiles < 0) return tiles;
    if (pair_min > 0 && tiles >= pair_min) {
        std::vector<unsigned char> t2;
        const int n2 = tc_build_probs(c, *kind, probs, t2, nullptr, 1);
        if (n2 > 0) {
            out.swap(t2);
            *pair = 1;
            return n2;
        }
    }
    // narrow tiles pay off for short K (latency-bound launches: 2048..8192 x
    // 256 x 512 12.8 -> 9.2 us); at K >= 2048 or >= 128 wide tiles they lose
    // (4096 x 2048 x 2048 37 -> 52 us: A is read twice per output column)
    const int nmax = narrow_max >= 0 ? narrow_max : g_tc_narrow_max_tiles;
    // never for in-place inverse solves (a_kwrap: C overwrites A, so one tile
    // must cover every column of its rows)
    int kmax = 0;
    bool inplace = false;
    for (const DevProb& d : probs) {
        kmax = d.k > kmax ? d.k : kmax;
        inplace |= d.a_kwrap != 0;
    }
    if (!tf32 && nmax > 0 && tiles < nmax && kmax <= 1024 && !inplace) {
        std::vector<unsigned char> t2;
        const int n2 = tc_build_probs(c, KIND_F16N, probs, t2, err);
        if (n2 < 0) return n2;
        out.swap(t2);
        *kind = KIND_F16N;
        return n2;
    }
    return tiles;
}

static int g_sms = 148;

bool tc_set_option(const std::string& key, int value) {
    if (key == "tc_kchunk") {
        g_tc_kchunk = value < 0 ? 0 : value;
        return true;
    }
    if (key == "tc_pair_min_tiles") {
        g_tc_pair_min_tiles = value < 0 ? 0 : value;
        return true;
    }
    if (key == "tc_narrow_max_tiles") {
        g_tc_narrow_max_tiles = value < 0 ? 0 : value;
        return true;
    }
    return false;
}

void init_tc_attributes() {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_gemm_tc2<KIND_F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, PairGeo<KIND_F16>::SMEM_BYTES);
    cudaFuncSetAttribute(k_gemm_tc2<KIND_TF32X3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PairGeo<KIND_TF32X3>::SMEM_BYTES);
    cudaFuncSetAttribute(k_gemm_tc<KIND_F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<KIND_F16>::SMEM_BYTES);
    cudaFuncSetAttribute(k_gemm_tc<KIND_F16N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Geo<KIND_F16N>::SMEM_BYTES);
    cudaFuncSetAttribute(k_gemm_tc<KIND_TF32X3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Geo<KIND_TF32X3>::SMEM_BYTES);
}

void launch_gemm_tc(const DevCtx& c, int kind, const void* d_probs, int nprob, int tiles, cudaStream_t s,
                    int max_ctas, int tiles_per_cta) {
    if (tiles <= 0) return;
    // persistent (tiles_per_cta = 0: one CTA per SM) or a bounded number of
    // tiles per CTA, so SMs free up between tiles and work on higher-priority
    // streams is not locked out; max_ctas caps the CTAs resident at once
    int grid = tiles_per_cta > 0 ? (tiles + tiles_per_cta - 1) / tiles_per_cta : g_sms;
    if (grid < g_sms && tiles_per_cta > 0) grid = g_sms;
    if (max_ctas > 0 && grid > max_ctas && tiles_per_cta == 0) grid = max_ctas;
    if (grid > tiles) grid = tiles;
    const TcProb* p = static_cast<const TcProb*>(d_probs);
    if (kind == KIND_TF32X3)
        k_gemm_tc<KIND_TF32X3><<<grid, Cfg<KIND_TF32X3>::NTHREADS, Geo<KIND_TF32X3>::SMEM_BYTES, s>>>(c, p, nprob,
                                                                                                    tiles);
    else if (kind == KIND_F16N)
        k_gemm_tc<KIND_F16N><<<grid, Cfg<KIND_F16N>::NTHREADS, Geo<KIND_F16N>::SMEM_BYTES, s>>>(c, p, nprob, tiles);
    else
        k_gemm_tc<KIND_F16><<<grid, Cfg<KIND_F16>::NTHREADS, Geo<KIND_F16>::SMEM_BYTES, s>>>(c, p, nprob, tiles);
}

// CTA-pair launch (k_gemm_tc2): problem table built with pair = 1; persistent
// pairs (one per two SMs, or fewer when there are fewer tiles)
void launch_gemm_tc_pair(const DevCtx& c, int kind, const void* d_probs, int nprob, int tiles, cudaStream_t s,
                         int tiles_per_pair, int max_ctas) {
    if (tiles <= 0) return;
    // persistent (tiles_per_pair = 0; at most max_ctas / 2 pairs when
    // max_ctas > 0, leaving SMs to the chain) or a bounded number of tiles
    // per pair, so SMs free up between tiles for concurrent work
    int pairs = tiles_per_pair > 0 ? (tiles + tiles_per_pair - 1) / tiles_per_pair : g_sms / 2;
    if (tiles_per_pair == 0 && max_ctas > 1 && pairs > max_ctas / 2) pairs = max_ctas / 2;
    if (pairs > tiles) pairs = tiles;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    const bool tf = kind == KIND_TF32X3;
    cfg.blockDim = dim3(tf ? PairCfg<KIND_TF32X3>::NTHREADS : PairCfg<KIND_F16>::NTHREADS, 1, 1);
    cfg.dynamicSmemBytes = tf ? PairGeo<KIND_TF32X3>::SMEM_BYTES : PairGeo<KIND_F16>::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (tf) cudaLaunchKernelEx(&cfg, k_gemm_tc2<KIND_TF32X3>, c, static_cast<const TcProb*>(d_probs), nprob, tiles);
    else cudaLaunchKernelEx(&cfg, k_gemm_tc2<KIND_F16>, c, static_cast<const TcProb*>(d_probs), nprob, tiles);
}

}  // namespace tcb
