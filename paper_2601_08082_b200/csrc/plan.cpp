// plan.cpp -- see plan.hpp.  Reference recursion: tree.cpp:42-152,
// static counter: analysis.cpp:64-120, config grammar: precision.cpp:17-111.
#include "plan.hpp"

#include <algorithm>
#include <array>
#include <cctype>
#include <stdexcept>

namespace tcb {

Rect Rect::unite(const Rect& o) const {
    if (m <= 0 || n <= 0) return o;
    if (o.m <= 0 || o.n <= 0) return *this;
    Rect r;
    r.r0 = std::min(r0, o.r0);
    r.c0 = std::min(c0, o.c0);
    r.m = std::max(r0 + m, o.r0 + o.m) - r.r0;
    r.n = std::max(c0 + n, o.c0 + o.n) - r.c0;
    return r;
}

// ---------------------------------------------------------------------------
// tree construction (build_node, tree.cpp:42-66): n1 = floor(n/2), leaf iff
// n <= b, levels by depth with saturation (precision.hpp:84-86)
// ---------------------------------------------------------------------------

int Plan::build_node(int r0, int n, int depth) {
    const int id = int(nodes.size());
    nodes.push_back(Node{});
    nodes[id].r0 = r0;
    nodes[id].n = n;
    nodes[id].depth = depth;
    if (n <= b) {
        nodes[id].leaf = true;
        nodes[id].level = leaf_level();
        Block blk;
        blk.rect = {r0, r0, n, n};
        blk.level = leaf_level();
        blk.leaf = true;
        blk.node = id;
        nodes[id].block = int(blocks.size());
        blocks.push_back(blk);
        return id;
    }
    const int n1 = n / 2, n2 = n - n1;
    nodes[id].n1 = n1;
    nodes[id].level = at_depth(depth);
    Block blk;
    blk.rect = {r0 + n1, r0, n2, n1};
    blk.level = at_depth(depth);
    blk.node = id;
    nodes[id].block = int(blocks.size());
    blocks.push_back(blk);
    const int d1 = build_node(r0, n1, depth + 1);
    const int d2 = build_node(r0 + n1, n2, depth + 1);
    nodes[id].d1 = d1;
    nodes[id].d2 = d2;
    return id;
}

int Plan::gemm_class(int op_level, int exec_level, const GemmProb* g) const {
    if (op_level == LV_F16) {
        if (exec_level == LV_F64) return GC_SIMT_F16D;
        // TMA needs 16-byte aligned rows: column offsets and K multiples of 8
        // halves (always true for power-of-two n and b >= 8)
        const bool aligned = !g || (g->a_c0 % 8 == 0 && g->b_c0 % 8 == 0 && g->k % 8 == 0);
        return (opt.use_tc && aligned) ? GC_TC16 : GC_SIMT_F16;
    }
    if (op_level == LV_F32) {
        if (exec_level == LV_F64) return GC_SIMT_F32D;
        // TMA: 16-byte aligned rows (column offsets multiples of 4 floats)
        const bool aligned = !g || (g->a_c0 % 4 == 0 && g->b_c0 % 4 == 0 && g->k % 4 == 0);
        if (!(opt.use_tc && opt.use_tc32)) return GC_SIMT_F32;
        // small problems: the warp-level path (float4 loads need the same alignment)
        if (g && aligned && g->b_buf < 0 && double(g->m) * g->n * g->k <= opt.mma32_max) return GC_MMA32;
        return aligned ? GC_TC32 : GC_SIMT_F32;
    }
    return GC_SIMT_F64;
}

int Plan::push(Op op) {
    ops.push_back(std::move(op));
    return int(ops.size()) - 1;
}

// ---------------------------------------------------------------------------
// level conversion of final L blocks: trsm_leaf / gemm_mixed read L through
// round_to(., p) (kernels.cpp:29, kernels.cpp:78).  Blocks stored above p get
// a p-rounded copy in buffer p, made once, right after they became final.
// ---------------------------------------------------------------------------

void Plan::ensure_shadows(int node, int p) {
    std::vector<int> todo;
    std::vector<int> stack{node};
    while (!stack.empty()) {
        const int id = stack.back();
        stack.pop_back();
        const Node& nd = nodes[id];
        const int blk = nd.block;
        if (blocks[blk].level > p && !has_shadow[blk][p]) {
            todo.push_back(blk);
            has_shadow[blk][p] = 1;
        }
        if (!nd.leaf) {
            stack.push_back(nd.d1);
            stack.push_back(nd.d2);
        }
    }
    if (todo.empty()) return;
    std::sort(todo.begin(), todo.end());
    needs_buf[p] = true;
    if (opt.shadow_per_block) {
        // one op per block: the TRSM that reads the shadow (its leaf solves
        // and GEMMs walk lnode's tree block by block) starts on a block as
        // soon as that block of L is final, i.e. it pipelines with the
        // factorization of lnode instead of waiting for all of it
        for (int blk : todo) {
            Op op;
            op.type = OP_SHADOW;
            op.level = p;
            op.blocks = {blk};
            op.rect = blocks[blk].rect;
            push(std::move(op));
        }
        return;
    }
    Op op;
    op.type = OP_SHADOW;
    op.level = p;
    op.blocks = todo;
    for (int blk : todo) op.rect = op.rect.unite(blocks[blk].rect);
    push(std::move(op));
}

// ---------------------------------------------------------------------------
// tree_trsm (tree.cpp:127-138)
// ---------------------------------------------------------------------------

void Plan::emit_trsm(Rect B, int p, int lnode, const RowSplit* rows) {
    const Node& L = nodes[lnode];
    // the row parts of B this call's device ops cover
    RowSplit parts = rows ? *rows : RowSplit{{B.r0, B.m}};
    if (L.leaf || std::min(B.m, B.n) <= leaf_size) {
        const uint32_t seq = next_seq();
        const uint64_t f = uint64_t(B.m) * uint64_t(B.n) * uint64_t(B.n);
        add_flops(seq, p, K_TRSM, f);
        // large FP16 leaf solve on the tensor cores: X = rn16(B (W_hi + W_lo)^T)
        // with W = inv(rn16(L)) from the leaf's inverse op.  Rows are
        // independent, so the tile owning a row block reads and overwrites it.
        // (F16: X = rn16(B (W_hi + W_lo)^T), W = inv(rn16(L)) as an FP16 pair;
        //  F32: X = rn32(B W^T) on the three-pass TF32 kernel, W = inv(L))
        const bool inv16 = opt.use_tc && opt.inverse_trsm && p == LV_F16 && L.leaf && L.n <= kW16Lo &&
                           B.m >= kInvMinRows && B.c0 % 8 == 0 && L.r0 % 8 == 0;
        const bool inv32 = opt.use_tc && opt.use_tc32 && opt.inverse_trsm && p == LV_F32 && L.leaf &&
                           L.n <= kW32Ld && L.n % 32 == 0 && B.c0 % 4 == 0 && L.r0 % 4 == 0 &&
                           B.m > opt.sub32_max_rows;
        if (inv16 || inv32) {
            const int lb = nodes[lnode].block;
            const uint8_t bit = inv16 ? 1 : 2;
            if (!(has_inverse[lb] & bit)) {
                has_inverse[lb] |= bit;
                (inv16 ? needs_w16 : needs_w32) = true;
                Op iv;
                iv.type = OP_INVERSE;
                iv.level = p;
                iv.rect = {L.r0, L.r0, L.n, L.n};
                iv.seq = seq;  // singular diagonal is reported for its first solve
                push(std::move(iv));
            }
            for (const auto& part : parts) {
            GemmProb g;
            g.m = part.second;
            g.n = L.n;
            g.k = inv16 ? 2 * kW16Lo : L.n;
            g.a_r0 = part.first;
            g.a_c0 = B.c0;
            g.a_kwrap = inv16 ? kW16Lo : 0;
            g.b_r0 = L.r0;
            g.b_c0 = 0;
            g.b_buf = inv16 ? BUF_W16 : BUF_W32;
            g.c_r0 = part.first;
            g.c_c0 = B.c0;
            g.exec_level = p;
            g.alpha = 1.0;
            g.beta = 0.0;
            g.seq = seq;
            g.ref_kernel = K_TRSM;
            // X overwrites B in place, so no output tile may be written while
            // another tile still reads those columns as K.  FP16: one 256-wide
            // column tile covers n.  FP32 on mma.sync: full-width tiles
            // (GC_MMA32W).  FP32 on tcgen05 (128-wide tiles): two ops in
            // sequence -- columns [128, n) first (they read all of B), then
            // [0, 128), which need only B[:, 0:128) (W is lower triangular)
            const bool later_part = opt.lookahead_prio && &part != &parts.front();  // lookahead: low priority
            auto emit = [&](const GemmProb& gp, int gclass, double fl) {
                Op op;
                op.type = OP_GEMM;
                op.level = p;
                op.gclass = gclass;
                op.bulk = later_part ? 1 : 0;
                op.prob_begin = int(probs.size());
                probs.push_back(gp);
                op.prob_end = int(probs.size());
                op.rect = {gp.c_r0, gp.c_c0, gp.m, gp.n};
                op.flops = fl;
                push(std::move(op));
            };
            const double fp = double(f) * double(g.m) / double(B.m);  // this part's share
            if (inv16) {
                emit(g, GC_TC16, fp);
            } else if (double(g.m) * g.n * g.k <= opt.mma32w_max) {
                emit(g, GC_MMA32W, fp);
            } else if (g.n <= kTc32TileN) {
                emit(g, GC_TC32, fp);
            } else {
                GemmProb r = g, l = g;
                r.n = g.n - kTc32TileN;  // right columns [128, n): B rows of W from 128 on
                r.b_r0 = g.b_r0 + kTc32TileN;
                r.c_c0 = g.c_c0 + kTc32TileN;
                l.n = kTc32TileN;        // left columns [0, 128): K = 128
                l.k = kTc32TileN;
                const double fr = fp * double(r.n) / double(g.n);
                emit(r, GC_TC32, fr);
                emit(l, GC_TC32, fp - fr);
            }
            }  // row parts
            return;
        }
        for (const auto& part : parts) {
            Op op;
            op.type = OP_TRSM;
            op.level = p;
            op.bulk = (opt.lookahead_prio && &part != &parts.front()) ? 1 : 0;
            op.rect = {part.first, B.c0, part.second, B.n};
            op.lrect = {L.r0, L.r0, L.n, L.n};
            op.seq = seq;
            op.flops = double(f) * double(part.second) / double(B.m);
            push(std::move(op));
        }
        return;
    }
    const int n1 = L.n1;
    const int d1 = L.d1, d2 = L.d2;
    const Rect off = blocks[L.block].rect;
    Rect B1{B.r0, B.c0, B.m, n1};
    Rect B2{B.r0, B.c0 + n1, B.m, B.n - n1};
    emit_trsm(B1, p, d1, rows);
    const uint32_t gseq = next_seq();
    const uint64_t f = 2ull * uint64_t(B.m) * uint64_t(B.n - n1) * uint64_t(n1);
    add_flops(gseq, p, K_GEMM, f);
    for (const auto& part : parts) {
        GemmProb g;
        g.m = part.second;
        g.n = B.n - n1;
        g.k = n1;
        g.a_r0 = part.first;
        g.a_c0 = B1.c0;
        g.b_r0 = off.r0;
        g.b_c0 = off.c0;
        g.c_r0 = part.first;
        g.c_c0 = B2.c0;
        g.exec_level = p;
        g.seq = gseq;
        g.ref_kernel = K_GEMM;
        Op op;
        op.type = OP_GEMM;
        op.level = p;
        op.gclass = gemm_class(p, p, &g);
        op.bulk = (opt.lookahead_prio && &part != &parts.front()) ? 1 : 0;
        op.prob_begin = int(probs.size());
        probs.push_back(g);
        op.prob_end = int(probs.size());
        op.rect = {part.first, B2.c0, part.second, B2.n};
        op.flops = double(f) * double(part.second) / double(B.m);
        push(std::move(op));
    }
    emit_trsm(B2, p, d2, rows);
}

// ---------------------------------------------------------------------------
// tree_syrk (tree.cpp:140-152): leaves via syrk_leaf at the leaf level, the
// off-diagonal contributions via gemm_mixed at the destination's level.  All
// sub-updates of one tree_syrk write disjoint blocks, so they are grouped
// into one launch per operand class.
// ---------------------------------------------------------------------------

// the off-diagonal update C21 -= A2 A1^T of one tree_syrk split, at the
// destination's level (tree.cpp:149)
GemmProb Plan::syrk_offdiag(int cnode, Rect A) {
    const Node& C = nodes[cnode];
    const int n1 = C.n1;
    const Rect off = blocks[C.block].rect;
    GemmProb g;
    g.m = off.m;
    g.n = off.n;
    g.k = A.n;
    g.a_r0 = A.r0 + n1;
    g.a_c0 = A.c0;
    g.b_r0 = A.r0;
    g.b_c0 = A.c0;
    g.c_r0 = off.r0;
    g.c_c0 = off.c0;
    g.exec_level = C.level;
    g.seq = next_seq();
    g.ref_kernel = K_GEMM;
    add_flops(g.seq, C.level, K_GEMM, 2ull * uint64_t(g.m) * uint64_t(g.n) * uint64_t(g.k));
    return g;
}

void Plan::collect_syrk(int cnode, Rect A, int p, std::vector<GemmProb>& out) {
    const Node& C = nodes[cnode];
    if (C.leaf) {
        GemmProb g;
        g.m = g.n = C.n;
        g.k = A.n;
        g.a_r0 = A.r0;
        g.a_c0 = A.c0;
        g.b_r0 = A.r0;
        g.b_c0 = A.c0;
        g.c_r0 = C.r0;
        g.c_c0 = C.r0;
        g.exec_level = leaf_level();
        g.lower = 1;
        g.seq = next_seq();
        g.ref_kernel = K_SYRK;
        add_flops(g.seq, g.exec_level, K_SYRK,
                  uint64_t(C.n) * uint64_t(C.n + 1) * uint64_t(A.n));
        out.push_back(g);
        return;
    }
    const int n1 = C.n1;
    const int d1 = C.d1, d2 = C.d2;
    Rect A1{A.r0, A.c0, n1, A.n};
    Rect A2{A.r0 + n1, A.c0, A.m - n1, A.n};
    collect_syrk(d1, A1, p, out);
    out.push_back(syrk_offdiag(cnode, A));
    collect_syrk(d2, A2, p, out);
}

// one launch per operand class, classes in order of first appearance
void Plan::push_gemm_group(const std::vector<GemmProb>& all, int p, int bulk) {
    std::vector<int> classes;
    for (const auto& g : all) {
        const int c = gemm_class(p, g.exec_level, &g);
        if (std::find(classes.begin(), classes.end(), c) == classes.end()) classes.push_back(c);
    }
    for (int c : classes) {
        Op op;
        op.type = OP_GEMM;
        op.level = p;
        op.gclass = c;
        op.prob_begin = int(probs.size());
        for (const auto& g : all)
            if (gemm_class(p, g.exec_level, &g) == c) {
                probs.push_back(g);
                op.rect = op.rect.unite({g.c_r0, g.c_c0, g.m, g.n});
                op.flops += double(g.lower ? 2.0 * g.m * g.n * g.k / 2.0 : 2.0 * g.m * g.n * g.k);
            }
        op.prob_end = int(probs.size());
        op.bulk = bulk;
        push(std::move(op));
    }
}

// A large tree_syrk is emitted as separate launches for its diag1 part, its
// off-diagonal GEMM and its diag2 part (recursively, down to
// opt.syrk_split_min): the recursion that follows (tree_potrf(diag2) ->
// tree_potrf(diag2.diag1) -> ...) then starts as soon as the region it reads
// is updated, while the rest of the update runs beside it (lookahead).  The
// sequence numbers keep the reference's order either way.
void Plan::emit_syrk(int cnode, Rect A, int p, bool critical, bool via_split) {
    const Node& C = nodes[cnode];
    if (!C.leaf && C.n >= opt.syrk_split_min) {
        // lookahead_prio: the diag1 chain of the split regions is what the
        // factorization that follows waits for first -- high priority; the
        // off-diagonal and diag2 regions low
        const int n1 = C.n1, d1 = C.d1, d2 = C.d2;
        emit_syrk(d1, Rect{A.r0, A.c0, n1, A.n}, p, critical, true);
        push_gemm_group({syrk_offdiag(cnode, A)}, p);
        emit_syrk(d2, Rect{A.r0 + n1, A.c0, A.m - n1, A.n}, p, false, true);
        return;
    }
    std::vector<GemmProb> all;
    collect_syrk(cnode, A, p, all);
    push_gemm_group(all, p, (opt.lookahead_prio && critical && via_split) ? 0 : 1);
}

// ---------------------------------------------------------------------------
// tree_potrf (tree.cpp:106-125)
// ---------------------------------------------------------------------------

// the off-diagonal panel of a split (tree.cpp:113-121): require_finite,
// quantize (spine panels; ext_slot >= 0: an alpha slot already allocated,
// e.g. filled from outside by a distributed driver), tree_trsm against the
// factored diag1 tree rooted at lnode, dequantize, require_finite
void Plan::emit_panel(int bi, int lnode, int ext_slot, int d2node) {
    const Block blk = blocks[bi];
    const int p = blk.level;
    int slot = -1;
    if (blk.spine_quant) {
        slot = ext_slot >= 0 ? ext_slot : n_alpha_slots++;
        Op q;
        q.type = OP_QUANT;
        q.level = p;
        q.rect = blk.rect;
        q.blocks.push_back(bi);
        q.slot = slot;
        q.seq = next_seq();  // the require_finite that precedes quantize
        checks.push_back({q.seq, blk.rect, 0});
        push(std::move(q));
    } else {
        const uint32_t seq = next_seq();
        checks.push_back({seq, blk.rect, 0});
        // require_finite before quantize (tree.cpp:114): a non-spine panel's
        // last writer is the SYRK update of its nearest ancestor, which wrote
        // the whole block -- its epilogue checks what it stores
        int last = -1;
        if (opt.fuse_checks)
            for (int i = int(probs.size()) - 1; i >= 0; --i) {
                const GemmProb& g = probs[i];
                if (g.c_r0 == blk.rect.r0 && g.c_c0 == blk.rect.c0 && g.m == blk.rect.m && g.n == blk.rect.n &&
                    g.ref_kernel == K_GEMM && g.exec_level == p) {
                    last = i;
                    break;
                }
            }
        if (last >= 0) {
            probs[last].check_seq = seq;
            probs[last].chk_r0 = blk.rect.r0;
            probs[last].chk_c0 = blk.rect.c0;
        } else {
            Op chk;
            chk.type = OP_CHECK;
            chk.level = p;
            chk.src = p;
            chk.rect = blk.rect;
            chk.seq = seq;
            push(std::move(chk));
        }
    }
    ensure_shadows(lnode, p);
    // lookahead: a tall panel's TRSM as two row parts split where diag2
    // splits, so diag2.diag1's SYRK part and factorization wait only for the
    // first (the SYRK below is then emitted per region, syrk_split_min)
    RowSplit split;
    if (opt.trsm_row_split_min > 0 && d2node >= 0 && blk.rect.m >= opt.trsm_row_split_min &&
        !nodes[d2node].leaf) {
        const int h = nodes[d2node].n1;
        split = {{blk.rect.r0, h}, {blk.rect.r0 + h, blk.rect.m - h}};
    }
    const int op0 = int(ops.size()), pr0 = int(probs.size());
    emit_trsm(blk.rect, p, lnode, split.empty() ? nullptr : &split);
    const int op1 = int(ops.size()), pr1 = int(probs.size());
    std::vector<int> dq_ops;
    if (blk.spine_quant) {
        const RowSplit dparts = split.empty() ? RowSplit{{blk.rect.r0, blk.rect.m}} : split;
        for (const auto& part : dparts) {
            Op dq;
            dq.type = OP_DEQUANT;
            dq.level = p;
            dq.rect = {part.first, blk.rect.c0, part.second, blk.rect.n};
            dq.slot = slot;
            dq_ops.push_back(push(std::move(dq)));
        }
    }
    // require_finite after dequantize (tree.cpp:121): every panel element's
    // last writer is the leaf solve of its column block (or the dequantize
    // when alpha != 1), so those kernels check their outputs
    const uint32_t post = next_seq();
    checks.push_back({post, blk.rect, 0});
    if (opt.fuse_checks) {
        for (int i = op0; i < op1; ++i)
            if (ops[i].type == OP_TRSM) {
                ops[i].check_seq = post;
                ops[i].chk = blk.rect;
            }
        for (int i = pr0; i < pr1; ++i)
            if (probs[i].ref_kernel == K_TRSM) {
                probs[i].check_seq = post;
                probs[i].chk_r0 = blk.rect.r0;
                probs[i].chk_c0 = blk.rect.c0;
            }
        for (int dq_op : dq_ops) {
            ops[dq_op].check_seq = post;
            ops[dq_op].chk = blk.rect;
        }
    } else {
        Op chk;
        chk.type = OP_CHECK;
        chk.level = p;
        chk.src = p;
        chk.rect = blk.rect;
        chk.seq = post;
        push(std::move(chk));
    }
}

void Plan::emit_potrf(int node) {
    const Node nd = nodes[node];
    if (nd.leaf) {
        Op chk;
        chk.type = OP_CHECK;
        chk.level = nd.level;
        chk.src = nd.level;
        chk.rect = blocks[nd.block].rect;
        chk.lower = 1;
        chk.diagonal = 1;
        chk.seq = next_seq();
        checks.push_back({chk.seq, chk.rect, 1});
        // the leaf's require_finite (tree.cpp:108) runs inside the POTRF
        // kernel, which loads the lower triangle anyway
        const uint32_t chk_seq = chk.seq;
        if (!opt.fuse_checks) push(std::move(chk));
        Op op;
        op.type = OP_POTRF;
        op.level = nd.level;
        op.rect = blocks[nd.block].rect;
        if (opt.fuse_checks) {
            op.check_seq = chk_seq;
            op.chk = op.rect;
        }
        op.seq = next_seq();
        const uint64_t n = uint64_t(nd.n);
        add_flops(op.seq, nd.level, K_POTRF, n * (n + 1) * (2 * n + 1) / 6);
        op.flops = double(n) * n * n / 3.0;
        push(std::move(op));
        return;
    }
    emit_potrf(nd.d1);
    const Block blk = blocks[nd.block];
    const int p = blk.level;
    emit_panel(nd.block, nd.d1, -1, nd.d2);
    emit_syrk(nd.d2, blk.rect, p);
    emit_potrf(nd.d2);
}

// ---------------------------------------------------------------------------
// dependencies
// ---------------------------------------------------------------------------

bool potrf_v2_ok(int lv, int n);  // k_potrf.cu: the shared-memory leaf kernel handles (lv, n)

// an F32 leaf's inverse (W32, for the FP32 panel solves) is computed by its
// POTRF kernel from the factor still in shared memory
void Plan::fuse_leaf_inverses() {
    if (!opt.fuse_inverse) return;
    for (Op& iv : ops) {
        if (iv.type != OP_INVERSE || iv.level != LV_F32) continue;
        for (Op& pf : ops)
            if (pf.type == OP_POTRF && pf.level == LV_F32 && pf.rect.r0 == iv.rect.r0 && pf.rect.m == iv.rect.m &&
                potrf_v2_ok(pf.level, pf.rect.m)) {
                pf.fuse_inv = 1;
                pf.inv_seq = iv.seq;
                iv.fused = 1;
                break;
            }
    }
}

// an F32 leaf's F16 shadow (the rn16 copy the F16 panel solves read,
// kernels.cpp:29/78) is written by its POTRF kernel next to the factor: the
// leaf's OP_SHADOW disappears from the chain
void Plan::fuse_leaf_shadows() {
    if (!opt.fuse_shadow) return;
    std::vector<char> drop(ops.size(), 0);
    for (size_t i = 0; i < ops.size(); ++i) {
        Op& sh = ops[i];
        if (sh.type != OP_SHADOW || sh.level != LV_F16 || sh.blocks.size() != 1) continue;
        const Block& blk = blocks[sh.blocks[0]];
        if (!blk.leaf || blk.level != LV_F32) continue;
        for (Op& pf : ops)
            if (pf.type == OP_POTRF && pf.level == LV_F32 && pf.rect.r0 == blk.rect.r0 && pf.rect.m == blk.rect.m &&
                potrf_v2_ok(pf.level, pf.rect.m)) {
                pf.shadow16 = 1;
                drop[i] = 1;
                break;
            }
    }
    std::vector<Op> kept;
    kept.reserve(ops.size());
    for (size_t i = 0; i < ops.size(); ++i)
        if (!drop[i]) kept.push_back(std::move(ops[i]));
    ops.swap(kept);
}

void Plan::finalize_accesses() {
    for (Op& op : ops) {
        op.acc.clear();
        switch (op.type) {
            case OP_IMPORT:
                for (int blk : op.blocks) {
                    op.acc.push_back({BUF_USER, blocks[blk].rect, false});
                    op.acc.push_back({blocks[blk].level, blocks[blk].rect, true});
                }
                break;
            case OP_EXPORT:
                for (int blk : op.blocks) {
                    op.acc.push_back({BUF_USER, blocks[blk].rect, true});
                    op.acc.push_back({blocks[blk].level, blocks[blk].rect, false});
                }
                break;
            case OP_CHECK:
                op.acc.push_back({op.src, op.rect, false});
                break;
            case OP_QUANT:
                op.acc.push_back({BUF_USER, op.rect, false});
                op.acc.push_back({op.level, op.rect, true});
                op.acc.push_back({BUF_ALPHA, {op.slot, 0, 1, 1}, true});
                break;
            case OP_DEQUANT:
                op.acc.push_back({BUF_ALPHA, {op.slot, 0, 1, 1}, false});
                op.acc.push_back({op.level, op.rect, true});
                break;
            case OP_SHADOW:
                for (int blk : op.blocks) {
                    op.acc.push_back({blocks[blk].level, blocks[blk].rect, false});
                    op.acc.push_back({op.level, blocks[blk].rect, true});
                }
                break;
            case OP_POTRF:
                op.acc.push_back({op.level, op.rect, true});
                if (op.fuse_inv) op.acc.push_back({BUF_W32, {op.rect.r0, 0, op.rect.m, kW32Ld}, true});
                if (op.shadow16) op.acc.push_back({LV_F16, op.rect, true});
                break;
            case OP_INVERSE:
                if (op.fused) break;  // no accesses: nothing waits on it
                op.acc.push_back({op.level, op.rect, false});
                if (op.level == LV_F16) op.acc.push_back({BUF_W16, {op.rect.r0, 0, op.rect.m, kW16Ld}, true});
                else op.acc.push_back({BUF_W32, {op.rect.r0, 0, op.rect.m, kW32Ld}, true});
                break;
            case OP_TRSM:
                op.acc.push_back({op.level, op.rect, true});
                op.acc.push_back({op.level, op.lrect, false});
                break;
            case OP_GEMM: {
                Rect rd;
                std::vector<Rect> rds;
                for (int i = op.prob_begin; i < op.prob_end; ++i) {
                    const GemmProb& g = probs[i];
                    rds.push_back({g.a_r0, g.a_c0, g.m, g.a_kwrap ? g.a_kwrap : g.k});
                    if (g.b_buf >= 0) op.acc.push_back({g.b_buf, {g.b_r0, g.b_c0, g.n, g.k}, false});
                    else rds.push_back({g.b_r0, g.b_c0, g.n, g.k});
                    op.acc.push_back({g.exec_level, {g.c_r0, g.c_c0, g.m, g.n}, true});
                }
                // drop read rects contained in another (SYRK reads sub-rows of one panel)
                std::vector<Rect> keep;
                for (size_t i = 0; i < rds.size(); ++i) {
                    bool contained = false;
                    for (size_t j = 0; j < rds.size() && !contained; ++j) {
                        if (i == j) continue;
                        const Rect& a = rds[i];
                        const Rect& b = rds[j];
                        const bool inside = a.r0 >= b.r0 && a.c0 >= b.c0 && a.r0 + a.m <= b.r0 + b.m &&
                                            a.c0 + a.n <= b.c0 + b.n;
                        const bool same = a.r0 == b.r0 && a.c0 == b.c0 && a.m == b.m && a.n == b.n;
                        if (inside && !(same && j > i)) contained = true;
                    }
                    if (!contained) keep.push_back(rds[i]);
                }
                for (const Rect& r : keep) op.acc.push_back({op.level, r, false});
                break;
            }
        }
    }
}

void Plan::build_deps() {
    const int N = int(ops.size());
    // per-op, per-buffer bounding boxes for a fast reject
    std::vector<std::array<Rect, BUF_COUNT>> bb(N);
    for (int i = 0; i < N; ++i)
        for (const Access& a : ops[i].acc) bb[i][a.buf] = bb[i][a.buf].unite(a.rect);
    const int W = (N + 63) / 64;
    std::vector<uint64_t> anc(size_t(N) * W, 0);
    auto conflict = [&](int i, int j) {
        bool any = false;
        for (int b = 0; b < BUF_COUNT && !any; ++b) any = bb[i][b].overlaps(bb[j][b]);
        if (!any) return false;
        for (const Access& x : ops[i].acc)
            for (const Access& y : ops[j].acc)
                if (x.buf == y.buf && (x.write || y.write) && x.rect.overlaps(y.rect)) return true;
        return false;
    };
    for (int i = 0; i < N; ++i) {
        uint64_t* ai = &anc[size_t(i) * W];
        for (int j = i - 1; j >= 0; --j) {
            if (ai[j / 64] >> (j % 64) & 1ull) continue;  // already ordered transitively
            if (!conflict(i, j)) continue;
            ops[i].deps.push_back(j);
            const uint64_t* aj = &anc[size_t(j) * W];
            for (int w = 0; w < W; ++w) ai[w] |= aj[w];
            ai[j / 64] |= 1ull << (j % 64);
        }
    }
}

void Plan::compute_windows() {
    for (int l = 0; l < 3; ++l) {
        win_lo[l] = 1 << 30;
        win_hi[l] = 0;
    }
    auto touch = [&](int buf, const Rect& r) {
        if (buf < 0 || buf > 2 || r.m <= 0) return;
        win_lo[buf] = std::min(win_lo[buf], r.r0);
        win_hi[buf] = std::max(win_hi[buf], r.r0 + r.m);
    };
    for (const Op& op : ops)
        for (const Access& a : op.acc) touch(a.buf, a.rect);
    for (const Block& blk : blocks)
        if (blk.external) touch(blk.level, blk.rect);
    for (int l = 0; l < 3; ++l) {
        if (win_hi[l] <= win_lo[l]) {
            win_lo[l] = win_hi[l] = 0;
        } else {
            needs_buf[l] = true;
        }
    }
}

size_t Plan::device_bytes() const {
    const size_t esz[3] = {2, 4, 8};
    const int nr = rows > 0 ? rows : n;
    size_t total = 0;
    for (int l = 0; l < 3; ++l)
        if (needs_buf[l]) total += ((size_t(win_hi[l] - win_lo[l]) * size_t(ldw()) * esz[l] + 255) / 256) * 256;
    if (needs_w16) total += sizeof(uint16_t) * size_t(nr) * kW16Ld + sizeof(float) * size_t(nr);
    if (needs_w32) total += sizeof(float) * size_t(nr) * kW32Ld;
    return total;
}

Plan Plan::make(int n, int b, const std::vector<int>& levels, bool quantize, int leaf_size,
                const PlanOptions& opt) {
    if (b < 1) throw std::invalid_argument("leaf size must be >= 1");
    if (levels.empty()) throw std::invalid_argument("empty precision config");
    if (n < 1) throw std::invalid_argument("tree requires a square matrix of order >= 1");
    for (int l : levels)
        if (l < LV_F16 || l > LV_F64) throw std::invalid_argument("precision level out of range");
    Plan P;
    P.n = n;
    P.rows = P.cols = n;
    P.b = b;
    P.leaf_size = leaf_size > 0 ? leaf_size : b;
    P.levels = levels;
    P.quantize = quantize;
    P.opt = opt;
    P.build_node(0, n, 0);
    // spine: nodes reached from the root through diag1 links only.  Their
    // off-diagonal panels get no SYRK update before their quantize, so the
    // scale is computed from the caller's original doubles (tree.cpp:117).
    // Every other panel receives >= 1 update rounded to its level first, so
    // max|B| <= range_max(level) and alpha == 1 exactly.  F64 spine panels
    // also have alpha == 1 (max|B| <= DBL_MAX).
    if (quantize)
        for (int id = 0; id >= 0 && !P.nodes[id].leaf; id = P.nodes[id].d1) {
            Block& blk = P.blocks[P.nodes[id].block];
            if (blk.level != LV_F64) blk.spine_quant = true;
        }
    P.has_shadow.assign(P.blocks.size(), std::vector<uint8_t>(3, 0));
    P.has_inverse.assign(P.blocks.size(), 0);
    for (const Block& blk : P.blocks) P.needs_buf[blk.level] = true;

    // one import / export op per storage block, in the order the recursion
    // first touches / finalizes them (depth first: diag1, the off-diagonal,
    // diag2): a block is imported right before its first use and exported as
    // soon as it is final, so with host buffers the copies overlap the
    // factorization in that order (Engine::enqueue_host)
    std::vector<int> order;
    {
        std::vector<int> stack{0};
        while (!stack.empty()) {
            const int id = stack.back();
            stack.pop_back();
            if (id < 0) {  // marker: emit the split's off-diagonal block
                order.push_back(P.nodes[-id - 1].block);
                continue;
            }
            const Node& nd = P.nodes[id];
            if (nd.leaf) {
                order.push_back(nd.block);
                continue;
            }
            stack.push_back(nd.d2);
            stack.push_back(-id - 1);
            stack.push_back(nd.d1);
        }
    }
    P.block_order = order;
    for (int i : order)
        if (!P.blocks[i].spine_quant) {
            Op imp;
            imp.type = OP_IMPORT;
            imp.blocks.push_back(i);
            imp.rect = P.blocks[i].rect;
            P.push(std::move(imp));
        }
    P.emit_potrf(0);
    P.fuse_leaf_inverses();
    P.fuse_leaf_shadows();
    for (int i : order) {
        Op exp;
        exp.type = OP_EXPORT;
        exp.blocks.push_back(i);
        exp.rect = P.blocks[i].rect;
        P.push(std::move(exp));
    }
    P.finalize_accesses();
    P.build_deps();
    P.compute_windows();
    return P;
}

void Plan::flop_totals(uint64_t by_level[3], uint64_t by_kernel[4], uint64_t calls[4],
                       uint32_t seq_limit) const {
    for (int i = 0; i < 3; ++i) by_level[i] = 0;
    for (int i = 0; i < 4; ++i) by_kernel[i] = calls[i] = 0;
    for (const FlopRec& r : flops) {
        if (r.seq >= seq_limit) continue;
        by_level[r.level] += r.flops;
        by_kernel[r.kernel] += r.flops;
        calls[r.kernel] += 1;
    }
}

int Plan::op_of_seq(uint32_t seq) const {
    for (int i = 0; i < int(ops.size()); ++i) {
        const Op& op = ops[i];
        if (op.seq == seq) return i;
        if (op.type == OP_GEMM)
            for (int p = op.prob_begin; p < op.prob_end; ++p)
                if (probs[p].seq == seq) return i;
    }
    return -1;
}

// ---------------------------------------------------------------------------
// StaticCounter (analysis.cpp:70-111) restated
// ---------------------------------------------------------------------------

namespace {
struct Counter {
    uint64_t b;
    const std::vector<int>& lv;
    uint64_t *L, *K, *C;
    int at(int d) const { return lv[d < int(lv.size()) ? d : int(lv.size()) - 1]; }
    void add(int level, int kernel, uint64_t f) {
        L[level] += f;
        K[kernel] += f;
        C[kernel] += 1;
    }
    void trsm(uint64_t m, uint64_t n, int d, int p) {
        if (n <= b || m <= b) return add(p, K_TRSM, m * n * n);
        const uint64_t n1 = n / 2, n2 = n - n1;
        trsm(m, n1, d + 1, p);
        add(p, K_GEMM, 2 * m * n2 * n1);
        trsm(m, n2, d + 1, p);
    }
    void syrk(uint64_t n, uint64_t k, int d, int p) {
        if (n <= b) return add(lv.back(), K_SYRK, n * (n + 1) * k);
        const uint64_t n1 = n / 2, n2 = n - n1;
        syrk(n1, k, d + 1, p);
        add(at(d), K_GEMM, 2 * n2 * n1 * k);
        syrk(n2, k, d + 1, p);
    }
    void potrf(uint64_t n, int d) {
        if (n <= b) return add(lv.back(), K_POTRF, n * (n + 1) * (2 * n + 1) / 6);
        const uint64_t n1 = n / 2, n2 = n - n1;
        const int p = at(d);
        potrf(n1, d + 1);
        trsm(n2, n1, d + 1, p);
        syrk(n2, n1, d + 1, p);
        potrf(n2, d + 1);
    }
};
}  // namespace

// depth-first block order of the subtree at `root` (first use / finalization)
static std::vector<int> dfs_blocks(const Plan& P, int root) {
    std::vector<int> order, stack{root};
    while (!stack.empty()) {
        const int id = stack.back();
        stack.pop_back();
        if (id < 0) {
            order.push_back(P.nodes[-id - 1].block);
            continue;
        }
        const Node& nd = P.nodes[id];
        if (nd.leaf) {
            order.push_back(nd.block);
            continue;
        }
        stack.push_back(nd.d2);
        stack.push_back(-id - 1);
        stack.push_back(nd.d1);
    }
    return order;
}

static void check_args(int b, const std::vector<int>& levels) {
    if (b < 1) throw std::invalid_argument("leaf size must be >= 1");
    if (levels.empty()) throw std::invalid_argument("empty precision config");
    for (int l : levels)
        if (l < LV_F16 || l > LV_F64) throw std::invalid_argument("precision level out of range");
}

Plan Plan::make_trsm(int n1, int m, int b, const std::vector<int>& levels, int leaf_size, const PlanOptions& opt,
                     bool ext) {
    check_args(b, levels);
    if (n1 < 1 || m < 1) throw std::invalid_argument("panel TRSM needs n1, m >= 1");
    Plan P;
    P.n = n1;
    P.rows = n1 + m;
    P.cols = n1;
    P.b = b;
    P.leaf_size = leaf_size > 0 ? leaf_size : b;
    P.levels = levels;
    P.quantize = true;
    P.opt = opt;
    P.build_node(0, n1, 1);  // L11 = the big tree's diag1
    if (ext) {
        // tree_trsm reads L only through rn_p (kernels.cpp:29, 78): L11 is
        // supplied as that image, every block at the panel level p, so no
        // import and no shadow copies; the caller's doubles start at row n1
        for (Block& blk : P.blocks) {
            blk.level = P.at_depth(0);
            blk.external = true;
        }
        P.user_row0 = n1;
    }
    Block pb;
    pb.rect = {n1, 0, m, n1};
    pb.level = P.at_depth(0);
    pb.spine_quant = pb.level != LV_F64;  // the top panel: quantized from the caller's doubles
    const int pbi = int(P.blocks.size());
    P.blocks.push_back(pb);
    P.has_shadow.assign(P.blocks.size(), std::vector<uint8_t>(3, 0));
    P.has_inverse.assign(P.blocks.size(), 0);
    for (const Block& blk : P.blocks) P.needs_buf[blk.level] = true;
    P.block_order = dfs_blocks(P, 0);
    P.block_order.push_back(pbi);
    for (int i : P.block_order)
        if (!P.blocks[i].spine_quant && !P.blocks[i].external) {
            Op imp;
            imp.type = OP_IMPORT;
            imp.blocks.push_back(i);
            imp.rect = P.blocks[i].rect;
            P.push(std::move(imp));
        }
    int slot = -1;
    if (pb.spine_quant) {
        slot = P.n_alpha_slots++;
        P.ext_alpha_slot = slot;
    }
    P.emit_panel(pbi, 0, slot);
    Op exp;
    exp.type = OP_EXPORT;
    exp.blocks.push_back(pbi);
    exp.rect = pb.rect;
    P.push(std::move(exp));
    P.finalize_accesses();
    P.build_deps();
    P.compute_windows();
    return P;
}

Plan Plan::make_syrk_rows(int n2, int k, int b, const std::vector<int>& levels, int row_lo, int row_hi,
                          const PlanOptions& opt, bool ext) {
    check_args(b, levels);
    if (n2 < 1 || k < 1 || k > n2 || row_lo < 0 || row_hi > n2 || row_lo >= row_hi)
        throw std::invalid_argument("panel SYRK: bad sizes or row range");
    Plan P;
    P.n = n2;
    P.rows = 2 * n2;
    P.cols = n2;
    P.b = b;
    P.leaf_size = b;
    P.levels = levels;
    P.quantize = true;
    P.opt = opt;
    P.build_node(0, n2, 1);  // A22 = the big tree's diag2
    const int ntree = int(P.blocks.size());
    const int p = P.at_depth(0);
    // A22's blocks restricted to the rows (a leaf may not straddle a bound)
    std::vector<int> mine;
    for (int i = 0; i < ntree; ++i) {
        const Rect r = P.blocks[i].rect;
        const int lo = std::max(r.r0, row_lo), hi = std::min(r.r0 + r.m, row_hi);
        if (lo >= hi) continue;
        if (P.blocks[i].leaf && (lo != r.r0 || hi != r.r0 + r.m))
            throw std::invalid_argument("panel SYRK: row range splits a diagonal leaf");
        Block pb = P.blocks[i];
        pb.rect = {lo, r.c0, hi - lo, r.n};
        pb.node = -1;
        mine.push_back(int(P.blocks.size()));
        P.blocks.push_back(pb);
    }
    // the solved panel: rows [n2, 2 n2) (ext: rows [row_hi, row_hi + n2),
    // supplied by the caller as its level image; the problems clipped to
    // output rows < row_hi read only its rows < row_hi)
    const int pr0 = ext ? row_hi : n2;
    Block ab;
    ab.rect = {pr0, 0, n2, k};
    ab.level = p;
    ab.external = ext;
    const int abi = int(P.blocks.size());
    P.blocks.push_back(ab);
    if (ext) {
        P.rows = row_hi + n2;
        P.user_row0 = row_lo;
        P.user_rows = row_hi - row_lo;
    }
    P.has_shadow.assign(P.blocks.size(), std::vector<uint8_t>(3, 0));
    P.has_inverse.assign(P.blocks.size(), 0);
    P.needs_buf[p] = true;
    for (int i : mine) P.needs_buf[P.blocks[i].level] = true;
    P.block_order = mine;
    if (!ext) P.block_order.push_back(abi);
    for (int i : P.block_order) {
        Op imp;
        imp.type = OP_IMPORT;
        imp.blocks.push_back(i);
        imp.rect = P.blocks[i].rect;
        P.push(std::move(imp));
    }
    // tree_syrk(A22, A21, -1, 1, p) with every problem clipped to the rows
    std::vector<GemmProb> all, kept;
    P.collect_syrk(0, ab.rect, p, all);
    P.flops.clear();
    for (GemmProb g : all) {
        const int lo = std::max(g.c_r0, row_lo), hi = std::min(g.c_r0 + g.m, row_hi);
        if (lo >= hi) continue;
        const int d = lo - g.c_r0;
        if (g.lower && (d != 0 || hi - lo != g.m))
            throw std::invalid_argument("panel SYRK: row range splits a diagonal leaf");
        g.c_r0 += d;
        g.a_r0 += d;
        g.m = hi - lo;
        // flops of the rows kept (informational: the distributed parts sum
        // to the reference's totals)
        const uint64_t f = g.lower ? uint64_t(g.m) * uint64_t(g.m + 1) * uint64_t(g.k)
                                   : 2ull * uint64_t(g.m) * uint64_t(g.n) * uint64_t(g.k);
        P.add_flops(g.seq, g.exec_level, g.lower ? K_SYRK : K_GEMM, f);
        kept.push_back(g);
    }
    if (!kept.empty()) P.push_gemm_group(kept, p);
    for (int i : mine) {
        Op exp;
        exp.type = OP_EXPORT;
        exp.blocks.push_back(i);
        exp.rect = P.blocks[i].rect;
        P.push(std::move(exp));
    }
    P.finalize_accesses();
    P.build_deps();
    P.compute_windows();
    return P;
}

void static_flop_breakdown(int n, int b, const std::vector<int>& levels, uint64_t by_level[3],
                           uint64_t by_kernel[4], uint64_t calls[4]) {
    for (int i = 0; i < 3; ++i) by_level[i] = 0;
    for (int i = 0; i < 4; ++i) by_kernel[i] = calls[i] = 0;
    if (n < 1 || b < 1 || levels.empty()) throw std::invalid_argument("flop_breakdown: n, b >= 1");
    Counter c{uint64_t(b), levels, by_level, by_kernel, calls};
    c.potrf(uint64_t(n), 0);
}

// ---------------------------------------------------------------------------
// PrecisionConfig grammar (precision.cpp:17-111):
//   config := '[' fmt (',' fmt)* ']' | ['Pure'] fmt ;  fmt := ('F'|'FP')('16'|'32'|'64')
// case-insensitive, whitespace anywhere, monotone outer -> inner.
// ---------------------------------------------------------------------------

namespace {
struct Scan {
    const std::string& s;
    size_t i = 0;
    void ws() {
        while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
    }
    bool end() {
        ws();
        return i >= s.size();
    }
    char peek() {
        ws();
        return i < s.size() ? s[i] : '\0';
    }
};

int read_format(Scan& sc, int& out, std::string& err) {
    sc.ws();
    std::string tok;
    while (sc.i < sc.s.size() && std::isalnum((unsigned char)sc.s[sc.i]))
        tok += char(std::toupper((unsigned char)sc.s[sc.i++]));
    const std::string norm = tok.rfind("FP", 0) == 0 ? "F" + tok.substr(2) : tok;
    if (norm == "F16") out = LV_F16;
    else if (norm == "F32") out = LV_F32;
    else if (norm == "F64") out = LV_F64;
    else {
        err = "unknown precision token '" + norm + "'";
        return 1;
    }
    return 0;
}
}  // namespace

int parse_config(const std::string& text, std::vector<int>& out, std::string& err) {
    out.clear();
    Scan sc{text};
    if (sc.end()) {
        err = "empty precision config";
        return 1;
    }
    int lv = 0;
    if (sc.peek() == '[') {
        ++sc.i;
        if (sc.peek() == ']') {
            err = "empty precision config";
            return 1;
        }
        if (read_format(sc, lv, err)) return 1;
        out.push_back(lv);
        while (sc.peek() == ',') {
            ++sc.i;
            if (read_format(sc, lv, err)) return 1;
            out.push_back(lv);
        }
        if (sc.peek() != ']') {
            err = "expected ',' or ']' in precision config";
            return 1;
        }
        ++sc.i;
    } else {
        const size_t save = sc.i;
        std::string word;
        while (sc.i < text.size() && std::isalpha((unsigned char)text[sc.i]))
            word += char(std::toupper((unsigned char)text[sc.i++]));
        if (word != "PURE") sc.i = save;
        if (read_format(sc, lv, err)) return 1;
        out.push_back(lv);
    }
    if (!sc.end()) {
        err = "trailing characters in precision config";
        return 1;
    }
    for (size_t i = 1; i < out.size(); ++i)
        if (out[i] < out[i - 1]) {
            err = "precision must be non-decreasing from outer to inner: " + text;
            return 2;
        }
    return 0;
}

std::string config_to_string(const std::vector<int>& levels) {
    static const char* names[3] = {"F16", "F32", "F64"};
    if (levels.size() == 1) return std::string("Pure ") + names[levels[0]];
    std::string s = "[";
    for (size_t i = 0; i < levels.size(); ++i) {
        if (i) s += ", ";
        s += names[levels[i]];
    }
    return s + "]";
}

}  // namespace tcb
