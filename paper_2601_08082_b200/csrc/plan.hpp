// plan.hpp -- host planner: the reference recursion unrolled into a flat op
// list with explicit data dependencies (SURVEY 7.1 "planner", Appendix B).
//
// The reference drives tree_potrf / tree_trsm / tree_syrk recursively at run
// time (tree.cpp:106-152).  Here the same recursion runs once, on the host,
// at plan time, and emits device ops in the reference's sequential order:
//   * every reference kernel call (potrf_leaf, trsm_leaf, syrk_leaf,
//     gemm_mixed) and every check point (require_finite, pivot, singular
//     diagonal) gets a sequence number `seq` in that order, so the device can
//     report the FIRST failure the reference would have thrown;
//   * the flops each call adds to SolveOptions::flops are recorded with its
//     seq (static == instrumented, criterion 6);
//   * ops carry (buffer, rect, read/write) accesses; dependencies are
//     derived from conflicts, which preserves every block's update order
//      while letting independent updates overlap.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace tcb {

enum Level : int { LV_F16 = 0, LV_F32 = 1, LV_F64 = 2 };
enum Buf : int { BUF_F16 = 0, BUF_F32 = 1, BUF_F64 = 2, BUF_USER = 3, BUF_ALPHA = 4, BUF_W16 = 5, BUF_W32 = 6,
                 BUF_COUNT = 7 };

// inverse-based FP16 leaf solves: W = inv(rn16(L_leaf)) as an FP16 hi/lo pair
// in the W16 workspace (row r0+j of a leaf at columns [0,n) hi, [256, 256+n) lo)
constexpr int kW16Ld = 512;
constexpr int kW16Lo = 256;
constexpr int kInvMinRows = 512;  // below this the substitution kernel is used (F16)
// FP32 leaf inverses W = inv(L) (row r0+i of a leaf, columns [0, n)), for
// inverse-based FP32 leaf solves on the three-pass TF32 tensor-core GEMM
constexpr int kW32Ld = 256;
constexpr int kTc32TileN = 128;  // output tile width of the TF32X3 tcgen05 GEMM (k_gemm_tc.cu Cfg)
enum RefKernel : int { K_POTRF = 0, K_TRSM = 1, K_SYRK = 2, K_GEMM = 3 };

struct Rect {
    int r0 = 0, c0 = 0, m = 0, n = 0;
    bool overlaps(const Rect& o) const {
        return m > 0 && n > 0 && o.m > 0 && o.n > 0 && r0 < o.r0 + o.m && o.r0 < r0 + m &&
               c0 < o.c0 + o.n && o.c0 < c0 + n;
    }
    Rect unite(const Rect& o) const;
};

// one node of the precision tree (PrecisionTreeNode, tree.hpp:14-26)
struct Node {
    int r0 = 0, n = 0, depth = 0;
    bool leaf = false;
    int level = LV_F64;  // leaf_level (leaves) / offdiag_level (splits)
    int n1 = 0;
    int d1 = -1, d2 = -1;  // child node ids
    int block = -1;        // storage block: the leaf square or the off-diagonal
};

// a storage block: every lower-triangle element belongs to exactly one
struct Block {
    Rect rect;
    int level = LV_F64;
    bool leaf = false;         // diagonal leaf (lower triangle only)
    bool spine_quant = false;  // quantized from the caller's doubles (see planner)
    bool external = false;     // values placed in the level buffer by the caller (no import / export)
    int node = -1;
};

// one reference-level GEMM-shaped call: C(m x n) = epi(C, sum_t A(i,t) B(j,t))
struct GemmProb {
    int m = 0, n = 0, k = 0;
    int a_r0 = 0, a_c0 = 0;
    int b_r0 = 0, b_c0 = 0;
    int c_r0 = 0, c_c0 = 0;
    int exec_level = LV_F64;  // rounding level of the result (= C's level)
    int lower = 0;            // syrk_leaf: only C(i,j) with global col <= row
    double alpha = -1.0, beta = 1.0;
    uint32_t seq = 0;
    int ref_kernel = K_GEMM;
    int a_kwrap = 0;        // A's K coordinate wraps at this period (inverse solve: hi|lo)
    int b_buf = -1;         // buffer of the B operand (-1: the operand level's)
    // fused require_finite on the values this call writes (0 = none): the
    // element position is reported relative to the checked block's origin
    uint32_t check_seq = 0;
    int chk_r0 = 0, chk_c0 = 0;
};

enum OpType : int {
    OP_IMPORT = 0,  // caller doubles -> level buffers (build-time rounding, tree.cpp:47-60)
    OP_EXPORT,      // level buffers -> caller doubles (lower triangle)
    OP_CHECK,       // require_finite (tree.cpp:19-31)
    OP_QUANT,       // quantize_block of a spine panel from the caller's doubles (tree.cpp:80-95)
    OP_DEQUANT,     // dequantize_block (tree.cpp:97-104)
    OP_SHADOW,      // round final L blocks down to a TRSM's level p (kernels.cpp:29, 78)
    OP_POTRF,       // potrf_leaf (kernels.cpp:42-69)
    OP_TRSM,        // trsm_leaf (kernels.cpp:71-92)
    OP_GEMM,        // grouped gemm_mixed / syrk_leaf calls of one operand class
    OP_INVERSE,     // W16 = inv(rn16(L_leaf)) hi/lo, for inverse-based FP16 leaf solves
};

// GEMM launch classes
enum GemmClass : int {
    GC_TC16 = 0,      // FP16 operands, FP32 accumulate, tcgen05 (exec F16/F32)
    GC_SIMT_F16 = 1,  // FP16 operands, FP32 accumulate, SIMT (validation / fallback)
    GC_SIMT_F32 = 2,  // FP32 operands, FP32 accumulate
    GC_SIMT_F16D = 3, // FP16 operands, FP64 accumulate (F64 exec)
    GC_SIMT_F32D = 4, // FP32 operands, FP64 accumulate
    GC_SIMT_F64 = 5,  // FP64 operands, FP64 accumulate
    GC_TC32 = 6,      // FP32 operands, three-pass TF32 split on tcgen05, FP32 accumulate (exec F32)
    GC_MMA32 = 7,     // the same arithmetic on mma.sync, for problems too small for tcgen05's setup
    GC_MMA32W = 8,    // GC_MMA32 with full-width (32 x n) tiles: in-place inverse leaf solves X = B W^T,
                      // where a tile must not overwrite columns another tile still reads as K
};

struct Access {
    int buf;
    Rect rect;
    bool write;
};

struct Op {
    OpType type = OP_CHECK;
    int level = LV_F64;   // storage/exec level of the op's target
    int src = BUF_F64;    // OP_CHECK: buffer read; OP_SHADOW: unused (per block)
    Rect rect;            // target rect (check / quant / potrf square / trsm B)
    Rect lrect;           // OP_TRSM: the L square (r0 == c0)
    int lower = 0;        // OP_CHECK: lower triangle only
    int diagonal = 0;     // OP_CHECK: "diagonal" vs "off-diagonal" wording
    int slot = -1;        // OP_QUANT / OP_DEQUANT: alpha slot
    uint32_t seq = 0;     // status sequence number (0 = op never fails)
    // fused require_finite: POTRF leaf entry check (lower triangle of rect),
    // TRSM / DEQUANT: post-dequantize check of the panel at chk (origin)
    uint32_t check_seq = 0;
    Rect chk;
    int gclass = GC_TC16; // OP_GEMM
    int prob_begin = 0, prob_end = 0;  // OP_GEMM: range in Plan::probs
    std::vector<int> blocks;           // OP_IMPORT / EXPORT / SHADOW
    std::vector<Access> acc;
    std::vector<int> deps;
    double flops = 0;      // algorithmic flops executed (for per-op timing)
    int bulk = 0;          // 1: trailing (SYRK) update, off the factorization's critical chain
    // OP_POTRF of an F32 leaf: also computes W32 = inv(L) (the leaf's
    // OP_INVERSE is then `fused`: kept only to decode a singular diagonal
    // reported under its seq, launches nothing)
    int fuse_inv = 0;
    uint32_t inv_seq = 0;
    int fused = 0;         // OP_INVERSE done by the leaf's POTRF
    int shadow16 = 0;      // OP_POTRF of an F32 leaf: also writes the leaf's F16 shadow (its OP_SHADOW removed)
};

// a require_finite point of the reference (tree.cpp:108, 114, 121): a
// failure key with this seq is a NumericalBreakdown in `rect`, element
// position relative to its origin
struct CheckRec {
    uint32_t seq;
    Rect rect;
    int diagonal;
};

struct FlopRec {
    uint32_t seq;
    int level, kernel;
    uint64_t flops;
};

struct PlanOptions {
    bool use_tc = true;      // FP16-operand GEMMs on tcgen05
    bool use_tc32 = true;    // FP32 x FP32 GEMMs on tcgen05 (three-pass TF32)
    double mma32w_max = 268435456.0;  // in-place inverse solves at or below this m*n*k on mma.sync (2^28: panels up to 4096 rows)
    double mma32_max = 16777216.0;  // m*n*k at or below which they run on mma.sync instead (2^24: the 256^3 leaf-level ones; 2^26 is 3% faster for one N=16384 factorization but 5% slower for the C4 batch)
    bool inverse_trsm = true; // FP16 leaf solves with m >= kInvMinRows as tcgen05 GEMMs
    bool fuse_checks = true;  // require_finite inside the producing kernels
    int sub32_max_rows = 0;  // F32 leaf solves of at most this many rows by substitution (k_trsm_cm) instead of inverse + GEMM
    bool lookahead_prio = true;   // with the splits below: the first row part / the diag1 chain of a split SYRK at high priority, the rest low
    int trsm_row_split_min = 0;   // off-diagonal panels with at least this many rows: TRSM ops split at diag2's first split (lookahead: diag2.diag1's SYRK and factorization start after the first row part)
    bool fuse_shadow = true;      // F32 leaves: their F16 shadow written by the leaf POTRF's store phase
    bool fuse_inverse = false;    // F32 leaves: W = inv(L) inside the leaf POTRF kernel (no separate inverse launch on the chain); measured slower: 99.5k extra cycles per leaf on one SM vs the 8-CTA inverse's 25 us (N=16384 11.7 vs 9.3 ms)
    bool shadow_per_block = true;  // one OP_SHADOW per block of L (pipelines the lower-level TRSM with the factorization it reads)
    int syrk_split_min = 1 << 30; // tree_syrk nodes at least this large launch per region (lookahead; off by default: it shortens the critical path but adds launches, a net loss for batches)
};

struct Plan {
    int n = 0, b = 0, leaf_size = 0;
    // storage extent of the level buffers (rows x cols); n x n for a
    // factorization, larger for the distributed panel plans below
    int rows = 0, cols = 0;
    int ext_alpha_slot = -1;  // alpha slot filled from outside before every run (distributed TRSM)
    // the caller's operand pointer refers to this row: rows below it are
    // never touched (the compact distributed pieces pass only their rows)
    int user_row0 = 0;
    int user_rows = 0;  // rows of the caller's operand (0: rows - user_row0)
    int caller_rows() const { return user_rows > 0 ? user_rows : (rows > 0 ? rows : n) - user_row0; }
    // rows [win_lo, win_hi) of each level buffer that any op or external
    // block touches: only that window is allocated (a virtual base keeps
    // absolute row coordinates in every kernel)
    int win_lo[3] = {0, 0, 0}, win_hi[3] = {0, 0, 0};
    std::vector<int> levels;
    bool quantize = true;
    PlanOptions opt;

    std::vector<Node> nodes;
    std::vector<Block> blocks;
    std::vector<GemmProb> probs;
    std::vector<Op> ops;
    std::vector<FlopRec> flops;  // in seq order
    std::vector<CheckRec> checks;  // in seq order
    std::vector<int> block_order;  // depth-first (first use / finalization) order
    int n_alpha_slots = 0;
    uint32_t n_seq = 0;
    bool needs_buf[3] = {false, false, false};
    bool needs_w16 = false;
    bool needs_w32 = false;

    // build + plan (throws std::invalid_argument on bad input)
    static Plan make(int n, int b, const std::vector<int>& levels, bool quantize,
                     int leaf_size, const PlanOptions& opt);

    // Distributed single factorization (BASELINE config C5), the two pieces
    // a rank runs besides whole factorizations.  Both use the big tree's
    // levels: the top split's diag1 / diag2 subtrees sit at depth 1, its
    // off-diagonal panel at depth 0.
    //  make_trsm: rows [0, n1) hold the factored L11 (tree of order n1),
    //    rows [n1, n1 + m) a row block of the panel A21; quantize it with an
    //    external alpha (the all-reduced max over every rank's rows), solve
    //    against L11 (tree_trsm), dequantize; only the panel is exported.
    //  make_syrk_rows: rows [0, n2) hold A22 (tree of order n2), rows
    //    [n2, 2 n2) the solved panel A21 (k = n1 columns, stored values);
    //    tree_syrk(A22, A21) restricted to output rows [row_lo, row_hi)
    //    (GEMM rows are independent: the restriction changes no element's
    //    arithmetic); only those rows of A22 are imported and exported.
    //  compact (ext) forms, for N = 131072 on 8 GPUs:
    //  make_trsm ext: L11 is supplied by the caller directly as its
    //    panel-level image (rn_p(L11), what tree_trsm reads: kernels.cpp:29,
    //    78) in the F16/F32 level buffer rows [0, n1); the caller's doubles
    //    hold only the m panel rows (user_row0 = n1).
    //  make_syrk_rows ext: the solved panel is supplied by the caller as its
    //    level image at rows [row_hi, row_hi + n2) (only rows < 2 row_hi are
    //    read); the caller's doubles hold only A22's rows [row_lo, row_hi)
    //    (user_row0 = row_lo).
    static Plan make_trsm(int n1, int m, int b, const std::vector<int>& levels, int leaf_size,
                          const PlanOptions& opt, bool ext = false);
    static Plan make_syrk_rows(int n2, int k, int b, const std::vector<int>& levels, int row_lo, int row_hi,
                               const PlanOptions& opt, bool ext = false);

    // device bytes the engine allocates for this plan (level windows, leaf
    // inverses, status words; excludes the launch tables, a few MB)
    size_t device_bytes() const;
    long long ldw() const { return (long long)((((cols > 0 ? cols : n) + 63) / 64) * 64); }

    int at_depth(int d) const { return levels[d < int(levels.size()) ? d : int(levels.size()) - 1]; }
    int leaf_level() const { return levels.back(); }

    // total flops (optionally only of calls with seq < limit)
    void flop_totals(uint64_t by_level[3], uint64_t by_kernel[4], uint64_t calls[4],
                     uint32_t seq_limit = 0xffffffffu) const;

    // which op owns a sequence number
    int op_of_seq(uint32_t seq) const;

   private:
    std::vector<std::vector<uint8_t>> has_shadow;  // [block][level]
    std::vector<uint8_t> has_inverse;              // [block] bit 0: W16 ready, bit 1: W32 ready
    int build_node(int r0, int n, int depth);
    void emit_potrf(int node);
    // row ranges [r0, r0 + m) of a TRSM's B emitted as separate device ops
    // (rows are independent, tree.cpp:133-134); the reference's calls, their
    // flops and sequence numbers stay one per call
    using RowSplit = std::vector<std::pair<int, int>>;
    void fuse_leaf_inverses();
    void fuse_leaf_shadows();
    void emit_panel(int block, int lnode, int ext_slot, int d2node = -1);
    void emit_trsm(Rect brect, int p, int lnode, const RowSplit* rows = nullptr);
    void emit_syrk(int cnode, Rect arect, int p, bool critical = true, bool via_split = false);
    void collect_syrk(int cnode, Rect arect, int p, std::vector<GemmProb>& out);
    GemmProb syrk_offdiag(int cnode, Rect arect);
    void push_gemm_group(const std::vector<GemmProb>& all, int p, int bulk = 1);
    void ensure_shadows(int node, int p);
    int push(Op op);
    uint32_t next_seq() { return ++n_seq; }
    void add_flops(uint32_t seq, int level, int kernel, uint64_t f) {
        flops.push_back({seq, level, kernel, f});
    }
    int gemm_class(int op_level, int exec_level, const GemmProb* g) const;
    void finalize_accesses();
    void build_deps();
    void compute_windows();
};

// static flop count (analysis.cpp:64-120 StaticCounter restated)
void static_flop_breakdown(int n, int b, const std::vector<int>& levels, uint64_t by_level[3],
                           uint64_t by_kernel[4], uint64_t calls[4]);

// PrecisionConfig grammar (precision.cpp:52-111); returns 0 ok, 1 syntax, 2 validation
int parse_config(const std::string& text, std::vector<int>& out, std::string& err);
std::string config_to_string(const std::vector<int>& levels);

}  // namespace tcb
