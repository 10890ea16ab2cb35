// engine.cu -- see engine.hpp.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <thread>

#include "launch.hpp"

namespace tcb {

namespace {

constexpr int kRaRing = 16;

#define TC_TRY(expr)                                                        \
    do {                                                                    \
        cudaError_t e_ = (expr);                                            \
        if (e_ != cudaSuccess) {                                            \
            if (err) *err = std::string(#expr) + ": " + cudaGetErrorString(e_); \
            return false;                                                   \
        }                                                                   \
    } while (0)

// split a column-major rect into column ranges of at most kChunkBytes (the
// copy in flight is the longest any other work queued behind it on a shared
// hardware channel can wait)
void chunk_rect(const Rect& r, std::vector<Rect>& out) {
    constexpr double kChunkBytes = 64.0 * 1024 * 1024;
    const int w = std::max(1, int(kChunkBytes / (8.0 * std::max(1, r.m))));
    for (int c = 0; c < r.n; c += w) out.push_back({r.r0, r.c0 + c, r.m, std::min(w, r.n - c)});
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

Engine::~Engine() {
    if (gexec_) cudaGraphExecDestroy(gexec_);
    if (graph_) cudaGraphDestroy(graph_);
    if (hexec_) cudaGraphExecDestroy(hexec_);
    if (hgraph_) cudaGraphDestroy(hgraph_);
    drop_host_phases();
    for (auto e : ev_hc_) cudaEventDestroy(e);
    for (auto e : ev_dc_) cudaEventDestroy(e);
    for (auto e : ev_h2d_) cudaEventDestroy(e);
    for (auto e : ra_ev_) cudaEventDestroy(e);
    for (auto e : ev_d2h_) cudaEventDestroy(e);
    if (cs_h2d_) cudaStreamDestroy(cs_h2d_);
    if (cs_d2h_) cudaStreamDestroy(cs_d2h_);
    if (d_stage_) cudaFree(d_stage_);
    for (auto e : events_) cudaEventDestroy(e);
    if (fork_) cudaEventDestroy(fork_);
    for (auto s : streams_) cudaStreamDestroy(s);
    if (d_bufs_) cudaFree(d_bufs_);
    if (d_words_) cudaFree(d_words_);
    if (d_w16_) cudaFree(d_w16_);
    if (d_w32_) cudaFree(d_w32_);
    if (d_arena_) cudaFree(d_arena_);
    if (d_ra_) cudaFree(d_ra_);
    if (h_ra_) cudaFreeHost(h_ra_);
    if (h_status_) cudaFreeHost(h_status_);
    if (h_ext_) cudaFreeHost(h_ext_);
}

int Engine::launches_per_run() const {
    int k = 2;  // status / alpha resets
    for (const Op& op : plan.ops) k += op.type == OP_QUANT ? 2 : 1;
    return k;
}

bool Engine::prepare(std::string* err) {
    if (ready_) return true;
    TC_TRY(cudaGetDevice(&device_));
    init_leaf_attributes();
    init_tc_attributes();
    init_mma32w_attributes();
    // level buffers: rows [win_lo, win_hi) x ldw of each level the plan
    // touches (all n rows for a factorization plan), one allocation with
    // 256-byte aligned sub-buffers.  The context holds VIRTUAL bases (the
    // allocation minus win_lo rows), so every kernel keeps addressing
    // base + row * ldw + col with absolute rows; no op touches a row
    // outside its level's window (Plan::compute_windows).
    const int n = plan.rows > 0 ? plan.rows : plan.n;
    const long long ldw = plan.ldw();
    ctx_.ldw = ldw;
    size_t sz[3] = {0, 0, 0}, total = 0;
    const size_t esz[3] = {2, 4, 8};
    for (int l = 0; l < 3; ++l)
        if (plan.needs_buf[l]) {
            sz[l] = size_t(plan.win_hi[l] - plan.win_lo[l]) * size_t(ldw) * esz[l];
            buf_off_[l] = total;
            total = align_up(total + sz[l], 256);
        }
    if (total) TC_TRY(cudaMalloc(&d_bufs_, total));
    unsigned char* base = static_cast<unsigned char*>(d_bufs_);
    auto vbase = [&](int l) -> unsigned char* {
        return plan.needs_buf[l] ? base + buf_off_[l] - ptrdiff_t(plan.win_lo[l]) * ptrdiff_t(ldw) * ptrdiff_t(esz[l])
                                 : nullptr;
    };
    for (int l = 0; l < 3; ++l) ctx_.win_lo[l] = plan.needs_buf[l] ? plan.win_lo[l] : 0;
    ctx_.b16 = reinterpret_cast<__half*>(vbase(0));
    ctx_.b32 = reinterpret_cast<float*>(vbase(1));
    ctx_.b64 = reinterpret_cast<double*>(vbase(2));
    if (plan.needs_w16) {
        // leaf inverses (hi | lo, zero outside the written triangles) + scales
        TC_TRY(cudaMalloc(&d_w16_, sizeof(__half) * size_t(n) * kW16Ld + sizeof(float) * size_t(n)));
        TC_TRY(cudaMemset(d_w16_, 0, sizeof(__half) * size_t(n) * kW16Ld + sizeof(float) * size_t(n)));
        ctx_.w16 = static_cast<__half*>(d_w16_);
        ctx_.wscale = reinterpret_cast<float*>(ctx_.w16 + size_t(n) * kW16Ld);
    }
    if (plan.needs_w32) {
        TC_TRY(cudaMalloc(&d_w32_, sizeof(float) * size_t(n) * kW32Ld));
        TC_TRY(cudaMemset(d_w32_, 0, sizeof(float) * size_t(n) * kW32Ld));
        ctx_.w32 = static_cast<float*>(d_w32_);
    }
    TC_TRY(cudaMalloc(&d_words_, sizeof(unsigned long long) * size_t(1 + std::max(1, plan.n_alpha_slots))));
    ctx_.status = d_words_;
    ctx_.alpha_bits = d_words_ + 1;
    TC_TRY(cudaMalloc(&d_ra_, sizeof(RunArgs)));
    ctx_.ra = d_ra_;
    TC_TRY(cudaMallocHost(&h_ra_, sizeof(RunArgs) * kRaRing));
    TC_TRY(cudaMallocHost(&h_status_, sizeof(unsigned long long)));

    // launch tables
    std::vector<unsigned char> host;
    launch_.assign(plan.ops.size(), OpLaunch{});
    auto append = [&](const void* p, size_t bytes) {
        const size_t o = align_up(host.size(), 128);
        host.resize(o + bytes);
        if (bytes) std::memcpy(host.data() + o, p, bytes);
        return o;
    };
    for (size_t i = 0; i < plan.ops.size(); ++i) {
        const Op& op = plan.ops[i];
        OpLaunch& L = launch_[i];
        if (op.type == OP_IMPORT || op.type == OP_EXPORT || op.type == OP_SHADOW) {
            std::vector<BlockDescHost> bh;
            for (int b : op.blocks) {
                const Block& blk = plan.blocks[b];
                bh.push_back({blk.rect.r0, blk.rect.c0, blk.rect.m, blk.rect.n, blk.level, blk.leaf ? 1 : 0});
            }
            std::vector<BlockDesc> bd;
            L.tiles = make_block_table(bh, bd);
            L.count = int(bd.size());
            L.offset = append(bd.data(), bd.size() * sizeof(BlockDesc));
        } else if (op.type == OP_GEMM) {
            std::vector<DevProb> dp;
            for (int p = op.prob_begin; p < op.prob_end; ++p) {
                const GemmProb& g = plan.probs[p];
                DevProb d{};
                d.m = g.m;
                d.n = g.n;
                d.k = g.k;
                d.a_r0 = g.a_r0;
                d.a_c0 = g.a_c0;
                d.b_r0 = g.b_r0;
                d.b_c0 = g.b_c0;
                d.c_r0 = g.c_r0;
                d.c_c0 = g.c_c0;
                d.exec_level = g.exec_level;
                d.lower = g.lower;
                d.alpha = g.alpha;
                d.beta = g.beta;
                d.a_kwrap = g.a_kwrap;
                d.b_buf = g.b_buf;
                d.check_seq = g.check_seq;
                d.chk_r0 = g.chk_r0;
                d.chk_c0 = g.chk_c0;
                dp.push_back(d);
            }
            L.count = int(dp.size());
            if (op.gclass == GC_TC16 || op.gclass == GC_TC32) {
                std::vector<unsigned char> tp;
                const int pmin = pair_min_tiles >= 0 ? pair_min_tiles : tc_pair_min_tiles();
                L.tiles = tc_select_tables(ctx_, op.gclass == GC_TC32, dp, tp, err, pmin, narrow_max_tiles, &L.kind,
                                           &L.pair);
                if (L.tiles < 0) return false;
                L.offset = append(tp.data(), tp.size());
            } else {
                L.tiles = op.gclass == GC_MMA32W ? simt_tiles(dp, M32W_ROWS, 256)
                                                 : simt_tiles(dp, op.gclass == GC_MMA32 ? M32_TILE : 0);
                L.offset = append(dp.data(), dp.size() * sizeof(DevProb));
            }
        }
    }
    if (!host.empty()) {
        TC_TRY(cudaMalloc(&d_arena_, host.size()));
        TC_TRY(cudaMemcpy(d_arena_, host.data(), host.size(), cudaMemcpyHostToDevice));
    }
    seq_op_.assign(size_t(plan.n_seq) + 1, -1);
    for (size_t i = 0; i < plan.ops.size(); ++i) {
        const Op& op = plan.ops[i];
        if (op.seq) seq_op_[op.seq] = int(i);
        if (op.type == OP_GEMM)  // GEMMs never fail: keep a failing op's claim on a shared seq
            for (int p = op.prob_begin; p < op.prob_end; ++p)
                if (seq_op_[plan.probs[p].seq] < 0) seq_op_[plan.probs[p].seq] = int(i);
    }
    ready_ = true;
    return true;
}

void Engine::launch_op(int i, cudaStream_t s) {
    const Op& op = plan.ops[i];
    const OpLaunch& L = launch_[i];
    const Rect& r = op.rect;
    unsigned char* tab = d_arena_ + L.offset;
    if (dev_skip && ((dev_skip >> op.type) & 1 || (op.type == OP_GEMM && (dev_skip >> (16 + op.gclass)) & 1))) {
        launch_noop(s);
        return;
    }
    switch (op.type) {
        case OP_IMPORT: launch_import(ctx_, reinterpret_cast<BlockDesc*>(tab), L.count, L.tiles, s); break;
        case OP_EXPORT: launch_export(ctx_, reinterpret_cast<BlockDesc*>(tab), L.count, L.tiles, s); break;
        case OP_SHADOW: launch_shadow(ctx_, reinterpret_cast<BlockDesc*>(tab), L.count, L.tiles, op.level, s); break;
        case OP_CHECK: launch_check(ctx_, op.src, r.r0, r.c0, r.m, r.n, op.lower, op.seq, s); break;
        case OP_QUANT: launch_quant(ctx_, op.level, r.r0, r.c0, r.m, r.n, op.slot, op.seq, s); break;
        case OP_DEQUANT:
            launch_dequant(ctx_, op.level, r.r0, r.c0, r.m, r.n, op.slot, op.check_seq,
                           op.check_seq ? r.r0 - op.chk.r0 : 0, op.check_seq ? r.c0 - op.chk.c0 : 0, s);
            break;
        case OP_POTRF:
            launch_potrf_leaf(ctx_, op.level, r.r0, r.m, op.seq, op.check_seq, s, op.inv_seq, op.fuse_inv, op.shadow16);
            break;
        case OP_TRSM:
            launch_trsm_leaf(ctx_, op.level, r.r0, r.c0, r.m, r.n, op.lrect.r0, op.seq, op.check_seq, op.chk.r0,
                             op.chk.c0, s);
            break;
        case OP_INVERSE:
            if (op.fused) launch_noop(s);  // computed by the leaf's POTRF
            else if (inv2_ok(r.m)) launch_leaf_inv2(ctx_, op.level == LV_F16 ? 0 : 1, r.r0, r.m, op.seq, s);
            else launch_leaf_inverse(ctx_, r.r0, r.m, op.seq, s);
            break;
        case OP_GEMM:
            if (L.pair)
                launch_gemm_tc_pair(ctx_, L.kind, tab, L.count, L.tiles, s,
                                    op.bulk ? bulk_tiles_per_cta : crit_tiles_per_cta,
                                    op.bulk ? bulk_max_ctas : crit_max_ctas);
            else if (op.gclass == GC_TC16 || op.gclass == GC_TC32)
                launch_gemm_tc(ctx_, L.kind, tab, L.count, L.tiles, s, op.bulk ? bulk_max_ctas : crit_max_ctas,
                               op.bulk ? bulk_tiles_per_cta : crit_tiles_per_cta);
            else launch_gemm_simt(ctx_, op.gclass, reinterpret_cast<DevProb*>(tab), L.count, L.tiles, s);
            break;
    }
}

void Engine::reset_words(cudaStream_t s) {
    cudaMemsetAsync(d_words_, 0xFF, sizeof(unsigned long long), s);
    if (plan.n_alpha_slots > 0)
        cudaMemsetAsync(d_words_ + 1, 0, sizeof(unsigned long long) * size_t(plan.n_alpha_slots), s);
    // an externally reduced max|B| (distributed panel): the slot starts at
    // it, so the local atomicMax leaves it unchanged and the quantize uses
    // the global alpha (read from pinned memory when the copy executes)
    if (plan.ext_alpha_slot >= 0 && h_ext_)
        cudaMemcpyAsync(d_words_ + 1 + plan.ext_alpha_slot, h_ext_, sizeof(unsigned long long),
                        cudaMemcpyHostToDevice, s);
}

bool Engine::level_buffer(int level, void** ptr, long long* ld, int* row_lo, int* row_hi, std::string* err) {
    if (!prepare(err)) return false;
    if (level < 0 || level > 2 || !plan.needs_buf[level]) {
        if (err) *err = "the plan has no buffer at that level";
        return false;
    }
    *ptr = static_cast<unsigned char*>(d_bufs_) + buf_off_[level];
    *ld = ctx_.ldw;
    *row_lo = plan.win_lo[level];
    *row_hi = plan.win_hi[level];
    return true;
}

bool Engine::set_external_absmax(double amax, std::string* err) {
    if (plan.ext_alpha_slot < 0) {
        if (err) *err = "plan has no external alpha slot";
        return false;
    }
    if (!h_ext_) TC_TRY(cudaMallocHost(&h_ext_, sizeof(unsigned long long)));
    const double a = std::fabs(amax);
    unsigned long long bits;
    std::memcpy(&bits, &a, sizeof bits);
    *h_ext_ = (a != a) ? 0ull : bits;  // NaN skipped like the local max
    return true;
}

// enqueue every op on the stream pool (works eagerly or under capture)
bool Engine::enqueue_ops(cudaStream_t origin, std::string* err, const HostIO* io, std::vector<cudaEvent_t>* tl) {
    const int N = int(plan.ops.size());
    // compute streams 0..C-1, then one stream for the imports and one for the
    // exports: a transfer-side op never sits in front of unrelated compute
    // (in-order streams would otherwise turn a wait for the caller's data
    // into a wait for everything queued behind it)
    const int C = std::max(2, n_streams);
    // compute streams: [0, CH) high priority -- the leaf chain, TRSMs, checks,
    // quantization (the factorization's critical path) -- and [CH, C) low
    // priority -- the trailing SYRK updates, whose CTAs yield SMs to the
    // chain as they finish tiles
    const int CH = C / 2;
    const int S = C + 2, SI = C, SE = C + 1;
    if (int(streams_.size()) < S) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi = greatest priority (numerically lowest)
        for (int s = int(streams_.size()); s < S; ++s) {
            cudaStream_t st;
            const int prio = s < CH ? hi : lo;
            TC_TRY(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, prio));
            streams_.push_back(st);
        }
    }
    if (int(events_.size()) < N + S) {
        for (int e = int(events_.size()); e < N + S; ++e) {
            cudaEvent_t ev;
            TC_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            events_.push_back(ev);
        }
    }
    if (!fork_) TC_TRY(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
    // stream assignment: continue a dep's stream of the same class when that
    // dep is its tail, else the least recently used stream of the class
    std::vector<int> sid(N, 0), tail(S, -1), last_use(S, -1);
    std::vector<char> need_ev(N, 0);
    std::vector<std::vector<int>> waits(N);
    for (int i = 0; i < N; ++i) {
        const Op& op = plan.ops[i];
        const OpType ty = op.type;
        const int b0 = op.bulk ? CH : 0, b1 = op.bulk ? C : CH;
        int pick = ty == OP_IMPORT ? SI : ty == OP_EXPORT ? SE : -1;
        if (pick < 0) {
            for (int d : op.deps)
                if (sid[d] >= b0 && sid[d] < b1 && tail[sid[d]] == d) {
                    pick = sid[d];
                    break;
                }
        }
        if (pick < 0) {
            pick = b0;
            for (int s = b0 + 1; s < b1; ++s)
                if (last_use[s] < last_use[pick]) pick = s;
        }
        sid[i] = pick;
        for (int d : op.deps)
            if (sid[d] != pick) {  // same-stream deps are ordered already
                waits[i].push_back(d);
                need_ev[d] = 1;
            }
        tail[pick] = i;
        last_use[pick] = i;
    }
    reset_words(origin);
    TC_TRY(cudaEventRecord(fork_, origin));
    for (int s = 0; s < S; ++s) TC_TRY(cudaStreamWaitEvent(streams_[s], fork_, 0));
    const int n = plan.n;
    const size_t esz = sizeof(double);
    if (io) {
        // H2D of every block in the order the recursion first needs them
        // (the diagonal leaf squares whole, so their upper halves come back
        // unchanged with the per-block D2H)
        TC_TRY(cudaStreamWaitEvent(cs_h2d_, fork_, 0));
        TC_TRY(cudaStreamWaitEvent(cs_d2h_, fork_, 0));
        for (int b : plan.block_order) {
            const Rect& r = plan.blocks[b].rect;
            TC_TRY(cudaMemcpy2DAsync(d_stage_ + size_t(r.c0) * n + r.r0, esz * n, io->host + size_t(r.c0) * io->lda + r.r0,
                                     esz * io->lda, esz * size_t(r.m), size_t(r.n), cudaMemcpyHostToDevice, cs_h2d_));
            TC_TRY(cudaEventRecord(ev_h2d_[b], cs_h2d_));
            if (tl_h2d_) {
                tl_h2d_->emplace_back();
                TC_TRY(cudaEventCreate(&tl_h2d_->back()));
                TC_TRY(cudaEventRecord(tl_h2d_->back(), cs_h2d_));
            }
        }
    }
    int n_d2h = 0;
    for (int i = 0; i < N; ++i) {
        cudaStream_t st = streams_[sid[i]];
        for (int d : waits[i]) TC_TRY(cudaStreamWaitEvent(st, events_[d], 0));
        const Op& op = plan.ops[i];
        if (io && (op.type == OP_IMPORT || op.type == OP_QUANT))  // the caller's doubles have arrived
            for (int b : op.blocks) TC_TRY(cudaStreamWaitEvent(st, ev_h2d_[b], 0));
        if (tl) TC_TRY(cudaEventRecord((*tl)[2 * i], st));
        launch_op(i, st);
        if (tl) TC_TRY(cudaEventRecord((*tl)[2 * i + 1], st));
        if (need_ev[i]) TC_TRY(cudaEventRecord(events_[i], st));
        if (io && op.type == OP_EXPORT) {
            // this block is final: copy it back while the rest computes
            cudaEvent_t e = ev_d2h_[n_d2h++];
            TC_TRY(cudaEventRecord(e, st));
            TC_TRY(cudaStreamWaitEvent(cs_d2h_, e, 0));
            const Rect& r = op.rect;
            TC_TRY(cudaMemcpy2DAsync(io->host + size_t(r.c0) * io->lda + r.r0, esz * io->lda,
                                     d_stage_ + size_t(r.c0) * n + r.r0, esz * n, esz * size_t(r.m), size_t(r.n),
                                     cudaMemcpyDeviceToHost, cs_d2h_));
            if (tl_d2h_) {
                tl_d2h_->emplace_back();
                TC_TRY(cudaEventCreate(&tl_d2h_->back()));
                TC_TRY(cudaEventRecord(tl_d2h_->back(), cs_d2h_));
            }
        }
    }
    for (int s = 0; s < S; ++s) {
        TC_TRY(cudaEventRecord(events_[N + s], streams_[s]));
        TC_TRY(cudaStreamWaitEvent(origin, events_[N + s], 0));
    }
    if (io) {
        TC_TRY(cudaEventRecord(ev_d2h_[n_d2h], cs_d2h_));
        TC_TRY(cudaStreamWaitEvent(origin, ev_d2h_[n_d2h], 0));
        TC_TRY(cudaEventRecord(ev_d2h_[n_d2h + 1], cs_h2d_));
        TC_TRY(cudaStreamWaitEvent(origin, ev_d2h_[n_d2h + 1], 0));
    }
    TC_TRY(cudaGetLastError());
    return true;
}

// a pinned RunArgs slot whose previous H2D copy has executed (the copies
// read the host slot asynchronously, in stream order)
RunArgs* Engine::next_args(std::string* err) {
    const int k = ra_next_++ % kRaRing;
    if (ra_ev_.empty()) {
        ra_ev_.resize(kRaRing);
        for (auto& e : ra_ev_)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
                if (err) *err = "cudaEventCreate";
                return nullptr;
            }
    }
    if (cudaEventSynchronize(ra_ev_[size_t(k)]) != cudaSuccess) {
        if (err) *err = "cudaEventSynchronize";
        return nullptr;
    }
    return h_ra_ + k;
}

bool Engine::enqueue(const double* a_in, long long lda_in, double* l_out, long long lda_out, cudaStream_t stream,
                     std::string* err) {
    if (!prepare(err)) return false;
    RunArgs* slot = next_args(err);
    if (!slot) return false;
    // the caller's pointers refer to row plan.user_row0 (compact pieces)
    slot->a_in = a_in - plan.user_row0;
    slot->l_out = l_out - plan.user_row0;
    slot->lda_in = lda_in;
    slot->lda_out = lda_out;
    TC_TRY(cudaMemcpyAsync(d_ra_, slot, sizeof(RunArgs), cudaMemcpyHostToDevice, stream));
    TC_TRY(cudaEventRecord(ra_ev_[size_t(slot - h_ra_)], stream));
    if (use_graph) {
        if (!gexec_ && dag_graph) {
            if (!build_dag_graph(&graph_, -1, err)) return false;
            TC_TRY(cudaGraphInstantiate(&gexec_, graph_, inst_flags()));
        }
        if (!gexec_) {
            cudaStream_t cap;
            TC_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            TC_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            std::string e2;
            const bool ok = enqueue_ops(cap, &e2);
            cudaGraph_t g = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(cap, &g);
            cudaStreamDestroy(cap);
            if (!ok) {
                if (err) *err = e2;
                if (g) cudaGraphDestroy(g);
                return false;
            }
            TC_TRY(ce);
            graph_ = g;
            TC_TRY(cudaGraphInstantiate(&gexec_, graph_, 0));
        }
        TC_TRY(cudaGraphLaunch(gexec_, stream));
    } else {
        if (!enqueue_ops(stream, err)) return false;
    }
    last_stream_ = stream;
    return true;
}

// any kernel may be the source of a programmatic edge (it triggers its
// dependents explicitly near its end, or implicitly when it exits)
bool Engine::pdl_src_ok(int) const { return true; }

bool Engine::build_dag_graph(cudaGraph_t* out, int phase, std::string* err) {
    *out = nullptr;
    // phase >= 0: only the ops of that host-path phase (edges to earlier
    // phases are satisfied by the launch order); the root only in phase 0
    auto in = [&](int i) { return phase < 0 || ph_op_[size_t(i)] == phase; };
    const int N = int(plan.ops.size());
    cudaGraph_t g = nullptr;
    TC_TRY(cudaGraphCreate(&g, 0));
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    // prio_levels 3: the leaf chain above the critical GEMMs (numerically
    // lower = greater priority)
    const int mid = prio_levels >= 3 && hi < lo ? hi + 1 : hi;
    cudaStream_t cap_top = nullptr, cap_hi = nullptr, cap_lo = nullptr;
    TC_TRY(cudaStreamCreateWithPriority(&cap_top, cudaStreamNonBlocking, hi));
    TC_TRY(cudaStreamCreateWithPriority(&cap_hi, cudaStreamNonBlocking, mid));
    TC_TRY(cudaStreamCreateWithPriority(&cap_lo, cudaStreamNonBlocking, lo));
    bool ok = true;
    std::string e2;
    // op index -> 1 if its node is a plain kernel node (programmatic edges
    // need a kernel node on both ends)
    std::vector<char> is_kernel(size_t(N), 0);
    // capture fn on stream s and add it with deps: a single kernel launch
    // becomes a kernel node of g (its parameters copied from the capture),
    // anything else a child-graph node.  pdl[j] != 0: the edge from deps[j]
    // is programmatic (the kernel may launch while deps[j] finishes and
    // waits for it in griddepcontrol.wait)
    auto add = [&](cudaStream_t s, const std::vector<cudaGraphNode_t>& deps, auto&& fn, cudaGraphNode_t* node,
                   const std::vector<char>* pdl = nullptr, bool* kernel_node = nullptr) -> bool {
        cudaGraph_t child = nullptr;
        if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return false;
        fn(s);
        if (cudaStreamEndCapture(s, &child) != cudaSuccess || !child) return false;
        // the scheduling priority of the capture stream, made explicit on
        // every kernel node: the chain's CTAs go first when SMs free up
        cudaKernelNodeAttrValue pv{};
        pv.priority = s == cap_top ? hi : s == cap_hi ? mid : lo;
        size_t nn = 0;
        cudaGraphGetNodes(child, nullptr, &nn);
        std::vector<cudaGraphNode_t> kids(nn);
        if (nn) cudaGraphGetNodes(child, kids.data(), &nn);
        int nk = 0;
        for (cudaGraphNode_t k : kids) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(k, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel) {
                ++nk;
                cudaGraphKernelNodeSetAttribute(k, cudaKernelNodeAttributePriority, &pv);
            }
        }
        cudaGetLastError();
        cudaError_t e = cudaErrorUnknown;
        if (use_pdl && nn == 1 && nk == 1) {
            cudaKernelNodeParams kp{};
            e = cudaGraphKernelNodeGetParams(kids[0], &kp);
            if (e == cudaSuccess) e = cudaGraphAddKernelNode(node, g, nullptr, 0, &kp);
            if (e == cudaSuccess) e = cudaGraphKernelNodeSetAttribute(*node, cudaKernelNodeAttributePriority, &pv);
            for (size_t j = 0; e == cudaSuccess && j < deps.size(); ++j) {
                cudaGraphEdgeData ed{};
                if (pdl && (*pdl)[j]) {
                    ed.from_port = cudaGraphKernelNodePortProgrammatic;
                    ed.type = cudaGraphDependencyTypeProgrammatic;
                }
                e = cudaGraphAddDependencies_v2(g, &deps[j], node, &ed, 1);
            }
            if (kernel_node) *kernel_node = e == cudaSuccess;
        } else {
            e = cudaGraphAddChildGraphNode(node, g, deps.empty() ? nullptr : deps.data(), deps.size(), child);
            if (kernel_node) *kernel_node = false;
        }
        cudaGraphDestroy(child);
        return e == cudaSuccess;
    };
    cudaGraphNode_t root = nullptr;
    if (phase <= 0) ok = add(cap_hi, {}, [&](cudaStream_t s) { reset_words(s); }, &root);
    // trace mode: slot 0 root, 1 + i op i
    auto stamp = [&](cudaGraphNode_t after, int k) {
        if (!d_trace_ || !ok || !after) return;
        cudaGraphNode_t sn = nullptr;
        unsigned long long* slot = d_trace_ + k;
        // greatest priority: a stamp queued behind bulk CTAs would report
        // their dispatch, not the op's end (one thread, co-resides anywhere)
        ok = add(cap_top, {after}, [&](cudaStream_t s) { launch_stamp(slot, s); }, &sn);
    };
    stamp(root, 0);
    std::vector<cudaGraphNode_t> node(size_t(N), nullptr);
    // startup_order (device graph): the spine quantizes of panels up to
    // 8192 wide (read by the first leaves' solves) go first, then the
    // imports, then the big spine quantizes (needed ~10+ ms in): otherwise
    // all of them start at once and the small quantize the chain waits on
    // gets a 1/500 share of HBM (4.8 ms instead of ~0.1 ms)
    std::vector<int> order, first_q, imports;
    const bool startup = (startup_order || import_chain > 0) && phase < 0;
    for (int i = 0; i < N; ++i) {
        const Op& op = plan.ops[size_t(i)];
        if (startup_order && phase < 0 && op.type == OP_QUANT && op.deps.empty() &&
            (long long)op.rect.m * op.rect.n <= 8192LL * 8192)
            first_q.push_back(i);
        if (startup && op.type == OP_IMPORT && op.deps.empty()) imports.push_back(i);
    }
    order = first_q;
    for (int i = 0; i < N; ++i)
        if (std::find(first_q.begin(), first_q.end(), i) == first_q.end()) order.push_back(i);
    for (int i : order) {
        if (!ok) break;
        if (!in(i)) continue;
        const Op& op = plan.ops[i];
        std::vector<cudaGraphNode_t> deps;
        std::vector<char> pdl;
        if (startup && op.deps.empty()) {
            if (op.type == OP_IMPORT) {
                for (int q : first_q) deps.push_back(node[size_t(q)]);
                // import_chain W: at most W imports in flight, in the
                // depth-first block order (the first leaves' blocks land first)
                if (import_chain > 0) {
                    const size_t k = size_t(std::find(imports.begin(), imports.end(), i) - imports.begin());
                    if (k >= size_t(import_chain)) deps.push_back(node[size_t(imports[k - size_t(import_chain)])]);
                }
            } else if (startup_order && op.type == OP_QUANT &&
                       std::find(first_q.begin(), first_q.end(), i) == first_q.end()) {
                for (int m : imports) deps.push_back(node[size_t(m)]);
            }
            pdl.assign(deps.size(), 0);
        }
        // programmatic edges into the chain's ops (not the bulk trailing
        // updates, whose waiting CTAs would hold SMs the chain needs), from
        // kernel nodes only
        const bool pdl_dst = use_pdl && !op.bulk && !d_trace_;
        for (int d : op.deps)
            if (in(d)) {
                deps.push_back(node[size_t(d)]);
                pdl.push_back(pdl_dst && is_kernel[size_t(d)] && pdl_src_ok(d));
            }
        if (deps.empty() && root) {
            deps.push_back(root);
            pdl.push_back(0);
        }
        bool kn = false;
        const bool chain = prio_levels >= 3 && !op.bulk && !(op.type == OP_GEMM && op.gclass == GC_TC16);
        const bool low = op.bulk || (import_low && op.type == OP_IMPORT);
        ok = add(low ? cap_lo : chain ? cap_top : cap_hi, deps, [&](cudaStream_t s) { launch_op(i, s); }, &node[size_t(i)], &pdl,
                 &kn);
        is_kernel[size_t(i)] = kn;
        // host phases: an event after each export, which the copy pipeline
        // polls to start that block's D2H
        if (ok && phase >= 0 && op.type == OP_EXPORT && size_t(i) < ev_ex_.size() && ev_ex_[size_t(i)]) {
            cudaGraphNode_t en = nullptr;
            ok = cudaGraphAddEventRecordNode(&en, g, &node[size_t(i)], 1, ev_ex_[size_t(i)]) == cudaSuccess;
        }
    }
    if (d_trace_)
        for (int i = 0; i < N; ++i) stamp(node[size_t(i)], 1 + i);
    cudaStreamDestroy(cap_top);
    cudaStreamDestroy(cap_hi);
    cudaStreamDestroy(cap_lo);
    if (!ok) {
        cudaGetLastError();
        cudaGraphDestroy(g);
        if (err) *err = "building the DAG graph failed";
        return false;
    }
    *out = g;
    return true;
}

bool Engine::ensure_stage(std::string* err) {
    if (d_stage_) return true;
    const int n = plan.n;
    TC_TRY(cudaMalloc(&d_stage_, sizeof(double) * size_t(n) * size_t(n)));
    TC_TRY(cudaStreamCreateWithFlags(&cs_h2d_, cudaStreamNonBlocking));
    TC_TRY(cudaStreamCreateWithFlags(&cs_d2h_, cudaStreamNonBlocking));
    ev_h2d_.resize(plan.blocks.size());
    for (auto& e : ev_h2d_) TC_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int n_exp = 0;
    for (const Op& op : plan.ops) n_exp += op.type == OP_EXPORT;
    ev_d2h_.resize(size_t(n_exp) + 2);
    for (auto& e : ev_d2h_) TC_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return true;
}

bool Engine::enqueue_host(double* host, long long lda, cudaStream_t stream, std::string* err) {
    if (!prepare(err) || !ensure_stage(err)) return false;
    const int n = plan.n;
    RunArgs* slot = next_args(err);
    if (!slot) return false;
    slot->a_in = d_stage_;
    slot->l_out = d_stage_;
    slot->lda_in = n;
    slot->lda_out = n;
    TC_TRY(cudaMemcpyAsync(d_ra_, slot, sizeof(RunArgs), cudaMemcpyHostToDevice, stream));
    TC_TRY(cudaEventRecord(ra_ev_[size_t(slot - h_ra_)], stream));
    HostIO io{host, lda};
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    // the copy pipeline serves pageable buffers too: their H2D calls return
    // once staged, their D2H calls once done -- issued only when the phase
    // that exports the block has finished, so nothing deadlocks
    if (use_graph && dag_graph) {
        if (hph_exec_.empty() && !build_host_phases(err)) return false;
        if (!run_host(io, stream, err)) return false;
    } else if (use_graph && pinned) {
        if (!hexec_ || hkey_ != host || hkey_lda_ != lda) {
            if (hexec_) cudaGraphExecDestroy(hexec_);
            if (hgraph_) cudaGraphDestroy(hgraph_);
            hexec_ = nullptr;
            hgraph_ = nullptr;
            cudaGraph_t g = nullptr;
            cudaStream_t cap;
            TC_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            TC_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            std::string e2;
            const bool ok = enqueue_ops(cap, &e2, &io);
            const cudaError_t ce = cudaStreamEndCapture(cap, &g);
            cudaStreamDestroy(cap);
            if (!ok) {
                if (err) *err = e2;
                if (g) cudaGraphDestroy(g);
                return false;
            }
            TC_TRY(ce);
            hgraph_ = g;
            TC_TRY(cudaGraphInstantiate(&hexec_, hgraph_, 0));
            hkey_ = host;
            hkey_lda_ = lda;
        }
        TC_TRY(cudaGraphLaunch(hexec_, stream));
    } else {
        if (!enqueue_ops(stream, err, &io)) return false;
    }
    last_stream_ = stream;
    return true;
}

// host-path phases: op i's phase follows the last H2D it needs (its own
// block for an import / quant, else the latest of its dependencies), the H2D
// stream cut into ~kPhases equal byte ranges (empty ranges dropped)
bool Engine::build_host_phases(std::string* err) {
    constexpr int kPhases = 32;  // measured: 32 phases 0.528 s, 16 phases 0.537-0.543 s (C3 e2e)
    const int N = int(plan.ops.size()), B = int(plan.block_order.size());
    std::vector<int> pos(plan.blocks.size(), -1);
    std::vector<double> cum(size_t(B), 0.0);
    double tot = 0.0;
    for (int k = 0; k < B; ++k) {
        const Rect& r = plan.blocks[size_t(plan.block_order[size_t(k)])].rect;
        pos[size_t(plan.block_order[size_t(k)])] = k;
        tot += double(r.m) * double(r.n);
        cum[size_t(k)] = tot;
    }
    std::vector<int> need(size_t(N), -1);
    for (int i = 0; i < N; ++i) {
        const Op& op = plan.ops[size_t(i)];
        int m = -1;
        for (int d : op.deps) m = std::max(m, need[size_t(d)]);
        if (op.type == OP_IMPORT || op.type == OP_QUANT)
            for (int b : op.blocks) m = std::max(m, pos[size_t(b)]);
        need[size_t(i)] = m;
    }
    // raw phase of an H2D position: its byte range; then compact
    auto raw = [&](int k) { return k < 0 ? 0 : std::min(kPhases - 1, int(cum[size_t(k)] * kPhases / tot)); };
    std::vector<int> used(kPhases, 0), wait(kPhases, -1);
    for (int i = 0; i < N; ++i) used[size_t(raw(need[size_t(i)]))] = 1;
    std::vector<int> remap(kPhases, -1);
    int P = 0;
    for (int q = 0; q < kPhases; ++q)
        if (used[size_t(q)]) remap[size_t(q)] = P++;
    ph_op_.assign(size_t(N), 0);
    ph_wait_.assign(size_t(P), -1);
    for (int i = 0; i < N; ++i) {
        const int p = remap[size_t(raw(need[size_t(i)]))];
        ph_op_[size_t(i)] = p;
        if (need[size_t(i)] >= 0)
            ph_wait_[size_t(p)] = std::max(ph_wait_[size_t(p)], need[size_t(i)]);
    }
    // H2D chunks in block order; a phase needs every chunk up to the last
    // one of its latest block.  D2H chunks of the exports, ordered by phase
    hc_rect_.clear();
    std::vector<int> last_chunk(size_t(B), -1);
    for (int k = 0; k < B; ++k) {
        chunk_rect(plan.blocks[size_t(plan.block_order[size_t(k)])].rect, hc_rect_);
        last_chunk[size_t(k)] = int(hc_rect_.size()) - 1;
    }
    ph_need_.assign(size_t(P), -1);
    for (int p = 0; p < P; ++p)
        if (ph_wait_[size_t(p)] >= 0) ph_need_[size_t(p)] = last_chunk[size_t(ph_wait_[size_t(p)])];
    struct DC {
        int phase, op;
        Rect r;
    };
    std::vector<DC> dl;
    ev_ex_.assign(size_t(N), nullptr);
    for (int i = 0; i < N; ++i)
        if (plan.ops[size_t(i)].type == OP_EXPORT) {
            std::vector<Rect> rs;
            chunk_rect(plan.ops[size_t(i)].rect, rs);
            for (const Rect& r : rs) dl.push_back({ph_op_[size_t(i)], i, r});
            if (export_events) TC_TRY(cudaEventCreateWithFlags(&ev_ex_[size_t(i)], cudaEventDisableTiming));
        }
    std::stable_sort(dl.begin(), dl.end(), [](const DC& x, const DC& y) { return x.phase < y.phase; });
    dc_rect_.clear();
    dc_phase_.clear();
    dc_op_.clear();
    for (auto& x : dl) {
        dc_phase_.push_back(x.phase);
        dc_op_.push_back(x.op);
        dc_rect_.push_back(x.r);
    }
    for (int p = 0; p < P; ++p) {
        cudaGraph_t g = nullptr;
        if (!build_dag_graph(&g, p, err)) return false;
        cudaGraphExec_t x = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&x, g, inst_flags());
        cudaGraphDestroy(g);
        TC_TRY(e);
        hph_exec_.push_back(x);
        cudaEvent_t ev;
        TC_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        ev_ph_.push_back(ev);
    }
    return true;
}

void Engine::drop_host_phases() {
    for (auto x : hph_exec_) cudaGraphExecDestroy(x);
    for (auto e : ev_ph_) cudaEventDestroy(e);
    for (auto e : ev_ex_)
        if (e) cudaEventDestroy(e);
    hph_exec_.clear();
    ev_ph_.clear();
    ev_ex_.clear();
}


// host entry point with the DAG graphs (synchronous): the calling thread
// feeds the copy engines and launches each phase's graph once the blocks it
// reads have landed and the previous phase has finished, and copies every
// exported block back once its phase has finished.  Nothing on the device
// ever waits on a copy or on a later phase (a waiting stream head would also
// stall unrelated work sharing its hardware channel); at most kDepth copies
// per direction are in flight.
bool Engine::run_host(const HostIO& io, cudaStream_t stream, std::string* err) {
    if (run_host_pipeline(io, stream, err)) return true;
    // error path: up to kDepth copies per direction may still read from or
    // write into the caller's host buffer; drain them (errors ignored) so the
    // caller may free or reuse it once this returns
    cudaStreamSynchronize(cs_h2d_);
    cudaStreamSynchronize(cs_d2h_);
    cudaStreamSynchronize(stream);
    return false;
}

bool Engine::run_host_pipeline(const HostIO& io, cudaStream_t stream, std::string* err) {
    constexpr int kDepth = 6;
    const int n = plan.n, N = int(plan.ops.size());
    const int P = int(hph_exec_.size()), H = int(hc_rect_.size()), D = int(dc_rect_.size());
    const size_t esz = sizeof(double);
    while (int(ev_hc_.size()) < H) {
        cudaEvent_t e;
        TC_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev_hc_.push_back(e);
    }
    while (int(ev_dc_.size()) < D) {
        cudaEvent_t e;
        TC_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev_dc_.push_back(e);
    }
    // earlier work on `stream` (the RunArgs upload, a previous run) first
    if (!fork_) TC_TRY(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
    TC_TRY(cudaEventRecord(fork_, stream));
    TC_TRY(cudaEventSynchronize(fork_));
    auto done = [&](cudaEvent_t e, bool* ok) {
        const cudaError_t q = cudaEventQuery(e);
        if (q == cudaSuccess) return true;
        if (q != cudaErrorNotReady) *ok = false;
        return false;
    };
    int h_iss = 0, h_done = 0, p_iss = 0, p_done = 0, d_iss = 0, d_done = 0;
    bool ok = true;
    while (ok && (h_done < H || p_done < P || d_done < D)) {
        bool moved = false;
        while (h_done < h_iss && done(ev_hc_[size_t(h_done)], &ok)) ++h_done, moved = true;
        while (ok && h_iss < H && h_iss - h_done < kDepth) {
            const Rect& r = hc_rect_[size_t(h_iss)];
            TC_TRY(cudaMemcpy2DAsync(d_stage_ + size_t(r.c0) * n + r.r0, esz * n,
                                     io.host + size_t(r.c0) * io.lda + r.r0, esz * io.lda, esz * size_t(r.m),
                                     size_t(r.n), cudaMemcpyHostToDevice, cs_h2d_));
            if (d_trace_) launch_stamp(d_trace_ + 1 + N + h_iss, cs_h2d_);
            TC_TRY(cudaEventRecord(ev_hc_[size_t(h_iss)], cs_h2d_));
            ++h_iss;
            moved = true;
        }
        while (p_done < p_iss && done(ev_ph_[size_t(p_done)], &ok)) ++p_done, moved = true;
        if (ok && p_iss < P && p_iss == p_done && h_done > ph_need_[size_t(p_iss)]) {
            TC_TRY(cudaGraphLaunch(hph_exec_[size_t(p_iss)], stream));
            TC_TRY(cudaEventRecord(ev_ph_[size_t(p_iss)], stream));
            ++p_iss;
            moved = true;
        }
        while (d_done < d_iss && done(ev_dc_[size_t(d_done)], &ok)) ++d_done, moved = true;
        // a D2H chunk goes once its phase has finished, or (export_events)
        // once its phase is running and its export op's event has fired
        auto d2h_ready = [&](int d) {
            const int ph = dc_phase_[size_t(d)];
            if (p_done > ph) return true;
            if (p_iss <= ph || ev_ex_.empty()) return false;
            const cudaEvent_t e = ev_ex_[size_t(dc_op_[size_t(d)])];
            return e != nullptr && done(e, &ok);
        };
        while (ok && d_iss < D && d_iss - d_done < kDepth && d2h_ready(d_iss)) {
            const Rect& r = dc_rect_[size_t(d_iss)];
            TC_TRY(cudaMemcpy2DAsync(io.host + size_t(r.c0) * io.lda + r.r0, esz * io.lda,
                                     d_stage_ + size_t(r.c0) * n + r.r0, esz * n, esz * size_t(r.m), size_t(r.n),
                                     cudaMemcpyDeviceToHost, cs_d2h_));
            if (d_trace_) launch_stamp(d_trace_ + 1 + N + H + d_iss, cs_d2h_);
            TC_TRY(cudaEventRecord(ev_dc_[size_t(d_iss)], cs_d2h_));
            ++d_iss;
            moved = true;
        }
        if (!moved) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    if (!ok) {
        if (err) *err = std::string("host pipeline: ") + cudaGetErrorString(cudaGetLastError());
        return false;
    }
    return true;
}

bool Engine::result(Failure* f, std::string* err) {
    TC_TRY(cudaMemcpyAsync(h_status_, d_words_, sizeof(unsigned long long), cudaMemcpyDeviceToHost, last_stream_));
    TC_TRY(cudaStreamSynchronize(last_stream_));
    return decode(*h_status_, f, err);
}

bool Engine::copy_status(unsigned long long* host_slot, cudaStream_t s, std::string* err) {
    TC_TRY(cudaMemcpyAsync(host_slot, d_words_, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    return true;
}

bool Engine::decode(unsigned long long key, Failure* f, std::string* err) const {
    *f = Failure{};
    if (key == ~0ull) return true;
    const uint32_t seq = uint32_t(key >> 40);
    const uint64_t local = key & ((1ull << 40) - 1);
    f->seq = seq;
    // a require_finite point (fused into a producing kernel or standalone)?
    {
        const auto& ck = plan.checks;
        auto it = std::lower_bound(ck.begin(), ck.end(), seq,
                                   [](const CheckRec& r, uint32_t s) { return r.seq < s; });
        if (it != ck.end() && it->seq == seq) {
            f->status = 2;
            f->block = it->rect;
            f->elem_row = it->rect.r0 + int(local & 0xFFFFF);
            f->elem_col = it->rect.c0 + int(local >> 20);
            f->diagonal = it->diagonal;
            return true;
        }
    }
    const int oi = seq < seq_op_.size() ? seq_op_[seq] : -1;
    if (oi < 0) {
        if (err) *err = "corrupt status word";
        return false;
    }
    const Op& op = plan.ops[oi];
    switch (op.type) {
        case OP_CHECK:
        case OP_QUANT:
            f->status = 2;
            f->block = op.rect;
            f->elem_row = op.rect.r0 + int(local & 0xFFFFF);
            f->elem_col = op.rect.c0 + int(local >> 20);
            f->diagonal = op.type == OP_CHECK ? op.diagonal : 0;
            break;
        case OP_POTRF:
            f->status = 1;
            f->index = op.rect.r0 + int(local);
            break;
        case OP_TRSM:
            f->status = 3;
            f->index = op.lrect.r0 + int(local);
            break;
        case OP_INVERSE:
            f->status = 3;
            f->index = op.rect.r0 + int(local);
            break;
        default:
            if (err) *err = "status from an op that cannot fail";
            return false;
    }
    return true;
}

bool Engine::timeline(const double* a_in, long long lda_in, double* l_out, long long lda_out, cudaStream_t stream,
                      std::vector<float>& t0, std::vector<float>& t1, std::string* err) {
    if (!prepare(err)) return false;
    RunArgs* slot = next_args(err);
    if (!slot) return false;
    // the caller's pointers refer to row plan.user_row0 (compact pieces)
    slot->a_in = a_in - plan.user_row0;
    slot->l_out = l_out - plan.user_row0;
    slot->lda_in = lda_in;
    slot->lda_out = lda_out;
    TC_TRY(cudaMemcpyAsync(d_ra_, slot, sizeof(RunArgs), cudaMemcpyHostToDevice, stream));
    TC_TRY(cudaEventRecord(ra_ev_[size_t(slot - h_ra_)], stream));
    const int N = int(plan.ops.size());
    std::vector<cudaEvent_t> tl(2 * size_t(N));
    for (auto& e : tl) TC_TRY(cudaEventCreate(&e));
    int* flag = nullptr;
    TC_TRY(cudaHostAlloc(&flag, sizeof(int), cudaHostAllocMapped));
    *reinterpret_cast<volatile int*>(flag) = 0;
    int* dflag = nullptr;
    TC_TRY(cudaHostGetDevicePointer(&dflag, flag, 0));
    launch_gate(dflag, stream);  // hold the device until most of the work is queued
    cudaEvent_t origin_ev;
    TC_TRY(cudaEventCreate(&origin_ev));
    TC_TRY(cudaEventRecord(origin_ev, stream));
    std::thread release([flag] {
        std::this_thread::sleep_for(std::chrono::milliseconds(300));
        __sync_synchronize();
        *reinterpret_cast<volatile int*>(flag) = 1;
    });
    const bool ok = enqueue_ops(stream, err, nullptr, &tl);
    release.join();
    if (!ok) return false;
    TC_TRY(cudaStreamSynchronize(stream));
    TC_TRY(cudaDeviceSynchronize());
    t0.assign(N, 0.f);
    t1.assign(N, 0.f);
    for (int i = 0; i < N; ++i) {
        cudaEventElapsedTime(&t0[i], origin_ev, tl[2 * i]);
        cudaEventElapsedTime(&t1[i], origin_ev, tl[2 * i + 1]);
    }
    for (auto& e : tl) cudaEventDestroy(e);
    cudaEventDestroy(origin_ev);
    cudaFreeHost(flag);
    last_stream_ = stream;
    return true;
}

bool Engine::timeline_host(double* host, long long lda, cudaStream_t stream, std::vector<float>& t0,
                           std::vector<float>& t1, std::vector<float>& th2d, std::vector<float>& td2h,
                           std::string* err) {
    if (!prepare(err) || !ensure_stage(err)) return false;
    const int n = plan.n;
    RunArgs* slot = next_args(err);
    if (!slot) return false;
    slot->a_in = d_stage_;
    slot->l_out = d_stage_;
    slot->lda_in = n;
    slot->lda_out = n;
    TC_TRY(cudaMemcpyAsync(d_ra_, slot, sizeof(RunArgs), cudaMemcpyHostToDevice, stream));
    TC_TRY(cudaEventRecord(ra_ev_[size_t(slot - h_ra_)], stream));
    const int N = int(plan.ops.size());
    std::vector<cudaEvent_t> tl(2 * size_t(N)), eh, ed;
    for (auto& e : tl) TC_TRY(cudaEventCreate(&e));
    int* flag = nullptr;
    TC_TRY(cudaHostAlloc(&flag, sizeof(int), cudaHostAllocMapped));
    *reinterpret_cast<volatile int*>(flag) = 0;
    int* dflag = nullptr;
    TC_TRY(cudaHostGetDevicePointer(&dflag, flag, 0));
    launch_gate(dflag, stream);
    cudaEvent_t origin_ev;
    TC_TRY(cudaEventCreate(&origin_ev));
    TC_TRY(cudaEventRecord(origin_ev, stream));
    std::thread release([flag] {
        std::this_thread::sleep_for(std::chrono::milliseconds(300));
        __sync_synchronize();
        *reinterpret_cast<volatile int*>(flag) = 1;
    });
    HostIO io{host, lda};
    tl_h2d_ = &eh;
    tl_d2h_ = &ed;
    const bool ok = enqueue_ops(stream, err, &io, &tl);
    tl_h2d_ = tl_d2h_ = nullptr;
    release.join();
    if (!ok) return false;
    TC_TRY(cudaStreamSynchronize(stream));
    TC_TRY(cudaDeviceSynchronize());
    auto rd = [&](std::vector<cudaEvent_t>& ev, std::vector<float>& out) {
        out.assign(ev.size(), 0.f);
        for (size_t i = 0; i < ev.size(); ++i) cudaEventElapsedTime(&out[i], origin_ev, ev[i]);
        for (auto& e : ev) cudaEventDestroy(e);
    };
    t0.assign(N, 0.f);
    t1.assign(N, 0.f);
    for (int i = 0; i < N; ++i) {
        cudaEventElapsedTime(&t0[i], origin_ev, tl[2 * i]);
        cudaEventElapsedTime(&t1[i], origin_ev, tl[2 * i + 1]);
    }
    for (auto& e : tl) cudaEventDestroy(e);
    rd(eh, th2d);
    rd(ed, td2h);
    cudaEventDestroy(origin_ev);
    cudaFreeHost(flag);
    return true;
}

bool Engine::trace_device(const double* a_in, long long lda_in, double* l_out, long long lda_out,
                          cudaStream_t stream, std::vector<float>& top, std::string* err) {
    if (!prepare(err)) return false;
    if (!use_graph || !dag_graph) {
        if (err) *err = "trace_device needs the DAG graph (use_graph, dag_graph)";
        return false;
    }
    const int N = int(plan.ops.size());
    const size_t slots = 1 + size_t(N);
    TC_TRY(cudaMalloc(&d_trace_, slots * sizeof(unsigned long long)));
    TC_TRY(cudaMemset(d_trace_, 0, slots * sizeof(unsigned long long)));
    auto drop = [&] {
        if (gexec_) cudaGraphExecDestroy(gexec_);
        if (graph_) cudaGraphDestroy(graph_);
        gexec_ = nullptr;
        graph_ = nullptr;
    };
    drop();  // rebuild with stamp nodes
    const bool ok = enqueue(a_in, lda_in, l_out, lda_out, stream, err);
    std::vector<unsigned long long> h(slots, 0);
    const bool ok2 = ok && cudaStreamSynchronize(stream) == cudaSuccess &&
                     cudaMemcpy(h.data(), d_trace_, slots * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
                         cudaSuccess;
    drop();
    cudaFree(d_trace_);
    d_trace_ = nullptr;
    if (!ok2) {
        if (err && err->empty()) *err = "trace run failed";
        return false;
    }
    top.assign(size_t(N), 0.f);
    for (int i = 0; i < N; ++i)
        top[size_t(i)] = h[size_t(1 + i)] ? float(double((long long)(h[size_t(1 + i)] - h[0])) * 1e-6) : -1e9f;
    return true;
}

bool Engine::trace_host(double* host, long long lda, cudaStream_t stream, std::vector<float>& top,
                        std::vector<float>& th2d, std::vector<float>& td2h, std::string* err) {
    if (!prepare(err) || !ensure_stage(err)) return false;
    const int N = int(plan.ops.size());
    std::vector<Rect> hr, dr;  // the copy chunks run_host will issue
    for (int b : plan.block_order) chunk_rect(plan.blocks[size_t(b)].rect, hr);
    for (const Op& op : plan.ops)
        if (op.type == OP_EXPORT) chunk_rect(op.rect, dr);
    const int B = int(hr.size()), E = int(dr.size());
    const size_t slots = 1 + size_t(N) + size_t(B) + size_t(E);
    TC_TRY(cudaMalloc(&d_trace_, slots * sizeof(unsigned long long)));
    TC_TRY(cudaMemset(d_trace_, 0, slots * sizeof(unsigned long long)));
    auto drop = [&] {
        if (hexec_) cudaGraphExecDestroy(hexec_);
        if (hgraph_) cudaGraphDestroy(hgraph_);
        hexec_ = nullptr;
        hgraph_ = nullptr;
        hkey_ = nullptr;
        drop_host_phases();
    };
    drop();  // rebuild with stamp nodes
    const bool ok = enqueue_host(host, lda, stream, err);
    std::vector<unsigned long long> h(slots, 0);
    bool ok2 = ok && cudaStreamSynchronize(stream) == cudaSuccess &&
               cudaMemcpy(h.data(), d_trace_, slots * sizeof(unsigned long long), cudaMemcpyDeviceToHost) == cudaSuccess;
    drop();
    cudaFree(d_trace_);
    d_trace_ = nullptr;
    if (!ok2) {
        if (err && err->empty()) *err = "trace run failed";
        return false;
    }
    auto ms = [&](size_t k) { return h[k] ? float(double((long long)(h[k] - h[0])) * 1e-6) : -1e9f; };
    top.assign(N, 0.f);
    th2d.assign(B, 0.f);
    td2h.assign(E, 0.f);
    for (int i = 0; i < N; ++i) top[i] = ms(1 + i);
    for (int i = 0; i < B; ++i) th2d[i] = ms(1 + N + i);
    for (int i = 0; i < E; ++i) td2h[i] = ms(1 + N + B + i);
    return true;
}

bool Engine::profile(const double* a_in, long long lda_in, double* l_out, long long lda_out, cudaStream_t stream,
                     std::vector<float>& op_ms, std::string* err) {
    if (!prepare(err)) return false;
    RunArgs* slot = next_args(err);
    if (!slot) return false;
    // the caller's pointers refer to row plan.user_row0 (compact pieces)
    slot->a_in = a_in - plan.user_row0;
    slot->l_out = l_out - plan.user_row0;
    slot->lda_in = lda_in;
    slot->lda_out = lda_out;
    TC_TRY(cudaMemcpyAsync(d_ra_, slot, sizeof(RunArgs), cudaMemcpyHostToDevice, stream));
    const int N = int(plan.ops.size());
    std::vector<cudaEvent_t> ev(N + 1);
    for (auto& e : ev) TC_TRY(cudaEventCreate(&e));
    // gate the stream until everything is enqueued: the events then time the
    // device, not host launch gaps
    int* flag = nullptr;
    TC_TRY(cudaHostAlloc(&flag, sizeof(int), cudaHostAllocMapped));
    *reinterpret_cast<volatile int*>(flag) = 0;
    int* dflag = nullptr;
    TC_TRY(cudaHostGetDevicePointer(&dflag, flag, 0));
    launch_gate(dflag, stream);
    reset_words(stream);
    TC_TRY(cudaEventRecord(ev[0], stream));
    // release after a bounded backlog (the launch queue is finite); the host
    // then stays ahead of the serialized device work
    constexpr int kBacklog = 256;
    for (int i = 0; i < N; ++i) {
        launch_op(i, stream);
        TC_TRY(cudaEventRecord(ev[i + 1], stream));
        if (i + 1 == std::min(N, kBacklog)) {
            __sync_synchronize();
            *reinterpret_cast<volatile int*>(flag) = 1;
        }
    }
    TC_TRY(cudaStreamSynchronize(stream));
    cudaFreeHost(flag);
    TC_TRY(cudaGetLastError());
    op_ms.assign(N, 0.f);
    for (int i = 0; i < N; ++i) cudaEventElapsedTime(&op_ms[i], ev[i], ev[i + 1]);
    for (auto& e : ev) cudaEventDestroy(e);
    last_stream_ = stream;
    return true;
}

}  // namespace tcb
