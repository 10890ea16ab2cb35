// tree.cpp -- the precision tree and tree_potrf of the C++ drop-in API.
//
// build_tree reproduces the reference's partition on the host (views only;
// the build-time rounding of tree.cpp:47-60 runs on the device).  tree_potrf
// does not walk the tree: it recovers (n, b, levels) from it, fetches a
// cached device plan (tc_plan_create: the same recursion unrolled into a DAG
// of sm_100a kernels, captured as one CUDA graph) and runs it on the node's
// view with tc_potrf_host.  tree_trsm / tree_syrk (not used by tree_potrf)
// drive the reference recursion over the device block operations.
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "abi.hpp"
#include "treechol/errors.hpp"
#include "treechol/tree.hpp"

namespace treechol {

namespace {

int lv(Precision p) { return static_cast<int>(p); }

PrecisionTreeNode make_node(TileView a, const PrecisionConfig& cfg, int b, bool quantize, int depth) {
    PrecisionTreeNode nd;
    nd.block = a;
    nd.depth = depth;
    if (a.rows <= b) {
        nd.is_leaf = true;
        nd.leaf_level = cfg.leaf();
        // leaf input down-conversion, lower triangle (tree.cpp:47-51)
        abi::check(tc_round_host(a.rows, a.cols, a.data, a.ld, lv(nd.leaf_level), 1));
        return nd;
    }
    nd.n1 = a.rows / 2;
    const int n2 = a.rows - nd.n1;
    nd.offdiag = a.sub(nd.n1, 0, n2, nd.n1);
    nd.offdiag_level = cfg.at_depth(std::size_t(depth));
    if (!quantize)  // converted plainly at build when not quantized (tree.cpp:58-60)
        abi::check(tc_round_host(n2, nd.n1, nd.offdiag.data, nd.offdiag.ld, lv(nd.offdiag_level), 0));
    nd.diag1 = std::make_unique<PrecisionTreeNode>(make_node(a.sub(0, 0, nd.n1, nd.n1), cfg, b, quantize, depth + 1));
    nd.diag2 = std::make_unique<PrecisionTreeNode>(make_node(a.sub(nd.n1, nd.n1, n2, n2), cfg, b, quantize, depth + 1));
    return nd;
}

// (b, levels) that rebuild exactly this tree: b = the largest leaf order
// (every split is larger), levels = the split level of each depth followed
// by the leaf level (at_depth saturates at the last entry)
void tree_shape(const PrecisionTreeNode& t, int& b, std::vector<int>& levels) {
    b = 0;
    std::vector<int> split_lv;
    int leaf_lv = lv(Precision::Double);
    std::vector<const PrecisionTreeNode*> todo{&t};
    while (!todo.empty()) {
        const PrecisionTreeNode* nd = todo.back();
        todo.pop_back();
        const int d = nd->depth - t.depth;
        if (nd->is_leaf) {
            b = std::max(b, nd->block.rows);
            leaf_lv = lv(nd->leaf_level);
            continue;
        }
        if (int(split_lv.size()) <= d) split_lv.resize(size_t(d) + 1, -1);
        split_lv[size_t(d)] = lv(nd->offdiag_level);
        todo.push_back(nd->diag1.get());
        todo.push_back(nd->diag2.get());
    }
    levels = split_lv;
    levels.push_back(leaf_lv);
}

// device plans, cached per (n, b, levels, quantize, leaf_size); a plan owns
// HBM workspace, so only a few are kept
struct PlanCache {
    using Key = std::tuple<int, int, std::vector<int>, bool, int>;
    std::mutex mu;
    std::vector<std::pair<Key, tc_plan*>> lru;  // most recent last
    static constexpr size_t kMax = 4;

    tc_plan* get(const Key& k) {
        for (size_t i = 0; i < lru.size(); ++i)
            if (lru[i].first == k) {
                auto e = lru[i];
                lru.erase(lru.begin() + long(i));
                lru.push_back(e);
                return e.second;
            }
        const auto& lvls = std::get<2>(k);
        tc_plan* p = nullptr;
        abi::check(tc_plan_create(std::get<0>(k), std::get<1>(k), lvls.data(), int(lvls.size()),
                                  std::get<3>(k) ? 1 : 0, std::get<4>(k), &p));
        if (lru.size() >= kMax) {
            tc_plan_destroy(lru.front().second);
            lru.erase(lru.begin());
        }
        lru.emplace_back(k, p);
        return p;
    }
    ~PlanCache() {
        for (auto& e : lru) tc_plan_destroy(e.second);
    }
};

PlanCache& cache() {
    static PlanCache c;
    return c;
}

void add_flops(FlopBreakdown* fb, const tc_flops& f) {
    if (!fb) return;
    for (int i = 0; i < 3; ++i) fb->by_level[size_t(i)] += f.by_level[i];
    for (int i = 0; i < 4; ++i) {
        fb->by_kernel[size_t(i)] += f.by_kernel[i];
        fb->calls[size_t(i)] += f.calls[i];
    }
}

}  // namespace

PrecisionTreeNode build_tree(TileView a, const PrecisionConfig& config, int b, bool quantize) {
    if (b < 1) throw InvalidArgument("leaf size must be >= 1");
    if (config.levels.empty()) throw InvalidArgument("empty precision config");
    if (a.rows < 1 || a.rows != a.cols) throw InvalidArgument("tree requires a square matrix of order >= 1");
    return make_node(a, config, b, quantize, 0);
}

double quantize_block(TileView b, Precision target) {
    double alpha = 1.0;
    abi::check(tc_quantize_host(b.rows, b.cols, b.data, b.ld, lv(target), &alpha));
    return alpha;
}

void dequantize_block(TileView b, double alpha, Precision level) {
    abi::check(tc_dequantize_host(b.rows, b.cols, b.data, b.ld, lv(level), alpha));
}

void tree_potrf(PrecisionTreeNode& node, const SolveOptions& opt) {
    if (opt.half_accumulator != Precision::Single)
        throw InvalidArgument("the device factorization accumulates Half-level sums in Single (FP32 tensor-core "
                              "accumulators); half_accumulator must be Single");
    int b = 0;
    std::vector<int> levels;
    tree_shape(node, b, levels);
    const int n = node.block.rows;
    tc_plan* plan = nullptr;
    tc_info info{};
    int st;
    {
        std::lock_guard<std::mutex> g(cache().mu);
        plan = cache().get({n, b, levels, opt.quantize, opt.leaf_size});
        st = tc_potrf_host(plan, node.block.data, node.block.ld, &info);
        tc_flops f{};
        if (st == TC_OK || st == TC_NOT_POSITIVE_DEFINITE || st == TC_NUMERICAL_BREAKDOWN ||
            st == TC_SINGULAR_DIAGONAL) {
            tc_plan_run_flops(plan, &f);
            add_flops(opt.flops, f);
        }
    }
    const int r0 = node.block.row0, c0 = node.block.col0;
    switch (st) {
        case TC_OK: return;
        case TC_NOT_POSITIVE_DEFINITE: throw NotPositiveDefinite(r0 + info.index);
        case TC_SINGULAR_DIAGONAL: throw SingularDiagonal(r0 + info.index);
        case TC_NUMERICAL_BREAKDOWN: {
            // tree.cpp:19-31 wording, global coordinates
            throw NumericalBreakdown(std::string("non-finite value in ") +
                                     (info.diagonal ? "diagonal" : "off-diagonal") + " block (rows " +
                                     std::to_string(r0 + info.row0) + ".." + std::to_string(r0 + info.row1) +
                                     ", cols " + std::to_string(c0 + info.col0) + ".." +
                                     std::to_string(c0 + info.col1) + ") at element (" +
                                     std::to_string(r0 + info.elem_row) + ", " + std::to_string(c0 + info.elem_col) +
                                     ")");
        }
        default: abi::check(st);
    }
}

// tree.cpp:127-138 over the device block operations: split B's columns along
// L's tree, solve the left part, update the right part, solve it
void tree_trsm(TileView b, Precision p, const PrecisionTreeNode& l, const SolveOptions& opt) {
    const bool base = l.is_leaf || std::min(b.rows, b.cols) <= opt.leaf_size;
    if (base) return trsm_leaf(b, l.block, p, opt.kernel_ctx());
    const TileView left = b.sub(0, 0, b.rows, l.n1);
    const TileView right = b.sub(0, l.n1, b.rows, b.cols - l.n1);
    tree_trsm(left, p, *l.diag1, opt);
    gemm_mixed(right, left, l.offdiag, -1.0, 1.0, p, opt.kernel_ctx());
    tree_trsm(right, p, *l.diag2, opt);
}

// tree.cpp:140-152: leaves at their own level, the off-diagonal update at the
// destination block's level, the two halves recursively
void tree_syrk(PrecisionTreeNode& c, TileView a, double alpha, double beta, Precision p, const SolveOptions& opt) {
    if (c.is_leaf) return syrk_leaf(c.block, a, alpha, beta, c.leaf_level, opt.kernel_ctx());
    const TileView top = a.sub(0, 0, c.n1, a.cols);
    const TileView bottom = a.sub(c.n1, 0, a.rows - c.n1, a.cols);
    tree_syrk(*c.diag1, top, alpha, beta, p, opt);
    gemm_mixed(c.offdiag, bottom, top, alpha, beta, c.offdiag_level, opt.kernel_ctx());
    tree_syrk(*c.diag2, bottom, alpha, beta, p, opt);
}

}  // namespace treechol
