// capi.cpp -- extern "C" entry points of libtreechol_b200.so (treechol_c.h).
// No exception crosses this boundary: every entry point returns a tc_status
// and leaves a thread-local message for tc_last_error().
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/treechol_c.h"
#include "engine.hpp"
#include "launch.hpp"
#include "plan.hpp"

using namespace tcb;

struct tc_plan {
    std::unique_ptr<Engine> eng;
    Failure last;
    bool have_result = false;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(TC_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

bool levels_ok(const int* levels, int nlevels) {
    if (!levels || nlevels < 1) return false;
    for (int i = 0; i < nlevels; ++i)
        if (levels[i] < 0 || levels[i] > 2) return false;
    return true;
}

void fill_info(const Failure& f, tc_info* info) {
    if (!info) return;
    std::memset(info, 0, sizeof(*info));
    info->status = f.status;
    info->index = f.index;
    info->row0 = f.block.r0;
    info->row1 = f.block.r0 + f.block.m - 1;
    info->col0 = f.block.c0;
    info->col1 = f.block.c0 + f.block.n - 1;
    info->elem_row = f.elem_row;
    info->elem_col = f.elem_col;
    info->diagonal = f.diagonal;
}

std::string message_of(const tc_info& info) {
    char buf[256];
    switch (info.status) {
        case TC_NOT_POSITIVE_DEFINITE:
            std::snprintf(buf, sizeof buf, "matrix is not positive definite: pivot %d is non-positive or non-finite",
                          info.index);
            return buf;
        case TC_SINGULAR_DIAGONAL:
            std::snprintf(buf, sizeof buf, "singular triangular factor: diagonal entry %d is zero or non-finite",
                          info.index);
            return buf;
        case TC_NUMERICAL_BREAKDOWN:
            std::snprintf(buf, sizeof buf,
                          "non-finite value in %s block (rows %d..%d, cols %d..%d) at element (%d, %d)",
                          info.diagonal ? "diagonal" : "off-diagonal", info.row0, info.row1, info.col0, info.col1,
                          info.elem_row, info.elem_col);
            return buf;
        default:
            return "";
    }
}

void flops_out(const uint64_t L[3], const uint64_t K[4], const uint64_t C[4], tc_flops* out) {
    for (int i = 0; i < 3; ++i) out->by_level[i] = L[i];
    for (int i = 0; i < 4; ++i) {
        out->by_kernel[i] = K[i];
        out->calls[i] = C[i];
    }
}

}  // namespace

namespace tcb {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace tcb

extern "C" {

const char* tc_last_error(void) { return g_err.c_str(); }

const char* tc_version(void) { return "treechol-b200 0.1 (sm_100a)"; }

int tc_device_available(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n > 0 ? 1 : 0;
}

int tc_config_parse(const char* text, int* levels, int* nlevels) {
    if (!text || !levels || !nlevels) return fail(TC_INVALID_ARGUMENT, "null argument");
    std::vector<int> lv;
    std::string err;
    const int r = parse_config(text, lv, err);
    if (r == 1) return fail(TC_SYNTAX_ERROR, err);
    if (r == 2) return fail(TC_VALIDATION_ERROR, err);
    if (lv.size() > 16) return fail(TC_INVALID_ARGUMENT, "more than 16 precision levels");
    for (size_t i = 0; i < lv.size(); ++i) levels[i] = lv[i];
    *nlevels = int(lv.size());
    return TC_OK;
}

int tc_config_to_string(const int* levels, int nlevels, char* buf, int buflen) {
    if (!levels_ok(levels, nlevels) || !buf || buflen < 1) return fail(TC_INVALID_ARGUMENT, "bad config");
    const std::string s = config_to_string(std::vector<int>(levels, levels + nlevels));
    std::snprintf(buf, size_t(buflen), "%s", s.c_str());
    return TC_OK;
}

int tc_flop_breakdown(int n, int b, const int* levels, int nlevels, tc_flops* out) {
    if (!out) return fail(TC_INVALID_ARGUMENT, "null output");
    if (n < 1 || b < 1) return fail(TC_INVALID_ARGUMENT, "flop_breakdown: n, b >= 1");
    if (!levels_ok(levels, nlevels)) return fail(TC_INVALID_ARGUMENT, "empty precision config");
    uint64_t L[3], K[4], C[4];
    static_flop_breakdown(n, b, std::vector<int>(levels, levels + nlevels), L, K, C);
    flops_out(L, K, C, out);
    return TC_OK;
}

int tc_plan_create(int n, int b, const int* levels, int nlevels, int quantize, int leaf_size, tc_plan** out) {
    if (!out) return fail(TC_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    if (b < 1) return fail(TC_INVALID_ARGUMENT, "leaf size must be >= 1");
    if (!levels || nlevels < 1) return fail(TC_INVALID_ARGUMENT, "empty precision config");
    if (!levels_ok(levels, nlevels)) return fail(TC_INVALID_ARGUMENT, "precision level out of range");
    if (n < 1) return fail(TC_INVALID_ARGUMENT, "tree requires a square matrix of order >= 1");
    if (n >= (1 << 20)) return fail(TC_INVALID_ARGUMENT, "order too large (n < 2^20)");
    try {
        PlanOptions po;
        Plan p = Plan::make(n, b, std::vector<int>(levels, levels + nlevels), quantize != 0, leaf_size, po);
        auto* h = new tc_plan;
        h->eng = std::make_unique<Engine>(std::move(p));
        *out = h;
        return TC_OK;
    } catch (const std::invalid_argument& e) {
        return fail(TC_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        return fail(TC_INVALID_ARGUMENT, e.what());
    }
}

void tc_plan_destroy(tc_plan* plan) { delete plan; }

int tc_plan_flops(const tc_plan* plan, tc_flops* out) {
    if (!plan || !out) return fail(TC_INVALID_ARGUMENT, "null argument");
    uint64_t L[3], K[4], C[4];
    plan->eng->plan.flop_totals(L, K, C);
    flops_out(L, K, C, out);
    return TC_OK;
}

// flops the reference would have added before stopping (partial on failure)
int tc_plan_run_flops(const tc_plan* plan, tc_flops* out) {
    if (!plan || !out) return fail(TC_INVALID_ARGUMENT, "null argument");
    uint64_t L[3], K[4], C[4];
    const uint32_t lim = (plan->have_result && plan->last.status) ? plan->last.seq : 0xffffffffu;
    plan->eng->plan.flop_totals(L, K, C, lim);
    flops_out(L, K, C, out);
    return TC_OK;
}

int tc_plan_stats(const tc_plan* plan, int* n_ops, int* n_launches, int* n_gemm_problems) {
    if (!plan) return fail(TC_INVALID_ARGUMENT, "null plan");
    if (n_ops) *n_ops = int(plan->eng->plan.ops.size());
    if (n_launches) *n_launches = plan->eng->launches_per_run();
    if (n_gemm_problems) *n_gemm_problems = int(plan->eng->plan.probs.size());
    return TC_OK;
}

}  // extern "C"

namespace tcb {
// plan-level options (they change the op list): rebuild the engine's plan
// with the option applied, keeping its run settings.  1 = applied, 0 = not a
// plan-level key, -1 = error (*err)
int apply_plan_option(std::unique_ptr<Engine>& eng, const std::string& k, int value, std::string* err) {
    static const char* keys[] = {"use_tc", "use_tc32", "inverse_trsm", "fuse_checks", "mma32_max_log2",
                                 "mma32w_max_log2", "syrk_split_min", "shadow_per_block", "sub32_max_rows",
                                 "trsm_row_split_min", "lookahead_prio", "fuse_inverse", "fuse_shadow"};
    bool known = false;
    for (const char* x : keys) known = known || k == x;
    if (!known) return 0;
    Engine& e = *eng;
    if (e.ready()) {
        *err = k + " must be set before the first run";
        return -1;
    }
    PlanOptions po = e.plan.opt;
    if (k == "use_tc") po.use_tc = value != 0;
    else if (k == "use_tc32") po.use_tc32 = value != 0;
    else if (k == "inverse_trsm") po.inverse_trsm = value != 0;
    else if (k == "fuse_checks") po.fuse_checks = value != 0;
    // FP32 GEMMs (in-place solves) with m*n*k <= 2^value run on mma.sync (negative: never)
    else if (k == "mma32_max_log2") po.mma32_max = value < 0 ? -1.0 : std::ldexp(1.0, value);
    else if (k == "mma32w_max_log2") po.mma32w_max = value < 0 ? -1.0 : std::ldexp(1.0, value);
    else if (k == "syrk_split_min") po.syrk_split_min = value < 1 ? (1 << 30) : value;
    else if (k == "sub32_max_rows") po.sub32_max_rows = value < 0 ? 0 : value;
    else if (k == "trsm_row_split_min") po.trsm_row_split_min = value < 0 ? 0 : value;
    else if (k == "lookahead_prio") po.lookahead_prio = value != 0;
    else if (k == "fuse_inverse") po.fuse_inverse = value != 0;
    else if (k == "fuse_shadow") po.fuse_shadow = value != 0;
    else po.shadow_per_block = value != 0;
    Plan p = Plan::make(e.plan.n, e.plan.b, e.plan.levels, e.plan.quantize, e.plan.leaf_size, po);
    const bool g = e.use_graph, dg = e.dag_graph, pdl = e.use_pdl;
    const int pmt = e.pair_min_tiles;
    const int s = e.n_streams, bt = e.bulk_tiles_per_cta, bm = e.bulk_max_ctas;
    const int ct = e.crit_tiles_per_cta, cm = e.crit_max_ctas, pl = e.prio_levels;
    const bool np = e.node_prio, il = e.import_low, ee = e.export_events, so = e.startup_order;
    const int ic = e.import_chain;
    eng = std::make_unique<Engine>(std::move(p));
    eng->use_graph = g;
    eng->dag_graph = dg;
    eng->use_pdl = pdl;
    eng->pair_min_tiles = pmt;
    eng->n_streams = s;
    eng->bulk_tiles_per_cta = bt;
    eng->bulk_max_ctas = bm;
    eng->crit_tiles_per_cta = ct;
    eng->crit_max_ctas = cm;
    eng->prio_levels = pl;
    eng->node_prio = np;
    eng->import_low = il;
    eng->export_events = ee;
    eng->startup_order = so;
    eng->import_chain = ic;
    return 1;
}
}  // namespace tcb

extern "C" {

int tc_plan_set_option(tc_plan* plan, const char* key, int value) {
    if (!plan || !key) return fail(TC_INVALID_ARGUMENT, "null argument");
    Engine& e = *plan->eng;
    const std::string k = key;
    if (k == "use_graph") {
        e.use_graph = value != 0;
        return TC_OK;
    }
    if (k == "dag_graph") {
        if (e.ready() && e.use_graph) return fail(TC_INVALID_ARGUMENT, k + " must be set before the first run");
        e.dag_graph = value != 0;
        return TC_OK;
    }
    if (k == "bulk_tiles_per_cta" || k == "bulk_max_ctas" || k == "crit_tiles_per_cta" || k == "crit_max_ctas" ||
        k == "prio_levels" || k == "node_prio" || k == "import_low" || k == "export_events" ||
        k == "startup_order") {
        if (e.ready() && e.use_graph) return fail(TC_INVALID_ARGUMENT, k + " must be set before the first run");
        if (k == "node_prio" || k == "import_low" || k == "export_events" || k == "startup_order") {
            (k == "node_prio"       ? e.node_prio
             : k == "import_low"    ? e.import_low
             : k == "export_events" ? e.export_events
                                    : e.startup_order) = value != 0;
            return TC_OK;
        }
        (k == "bulk_tiles_per_cta" ? e.bulk_tiles_per_cta
         : k == "bulk_max_ctas"    ? e.bulk_max_ctas
         : k == "crit_tiles_per_cta" ? e.crit_tiles_per_cta
         : k == "crit_max_ctas"    ? e.crit_max_ctas
                                   : e.prio_levels) = value < 0 ? 0 : value;
        return TC_OK;
    }
    if (k == "import_chain") {
        if (e.ready() && e.use_graph) return fail(TC_INVALID_ARGUMENT, k + " must be set before the first run");
        e.import_chain = value < 0 ? 0 : value;
        return TC_OK;
    }
    if (k == "use_pdl") {
        if (e.ready() && e.use_graph) return fail(TC_INVALID_ARGUMENT, k + " must be set before the first run");
        e.use_pdl = value != 0;
        return TC_OK;
    }
    if (k == "dev_skip") {  // development: see Engine::dev_skip
        if (e.ready() && e.use_graph) return fail(TC_INVALID_ARGUMENT, k + " must be set before the first run");
        e.dev_skip = value;
        return TC_OK;
    }
    if (k == "n_streams") {
        if (e.ready()) return fail(TC_INVALID_ARGUMENT, "n_streams must be set before the first run");
        e.n_streams = value < 1 ? 1 : value;
        return TC_OK;
    }
    std::string err;
    const int r = apply_plan_option(plan->eng, k, value, &err);
    if (r == 1) return TC_OK;
    if (r < 0) return fail(TC_INVALID_ARGUMENT, err);
    return fail(TC_INVALID_ARGUMENT, "unknown option '" + k + "'");
}

// per-op metadata for profiling: type, gemm class, level, flops, rect
int tc_plan_op_info(const tc_plan* plan, int i, int* type, int* gclass, int* level, double* flops, int* rect4) {
    if (!plan || i < 0 || i >= int(plan->eng->plan.ops.size())) return fail(TC_INVALID_ARGUMENT, "bad op index");
    const Op& op = plan->eng->plan.ops[i];
    if (type) *type = op.type;
    if (gclass) *gclass = op.type == OP_GEMM ? op.gclass : -1;
    if (level) *level = op.level;
    if (flops) *flops = op.flops;
    if (rect4) {
        rect4[0] = op.rect.r0;
        rect4[1] = op.rect.c0;
        rect4[2] = op.rect.m;
        rect4[3] = op.rect.n;
    }
    return TC_OK;
}

int tc_plan_op_probs(const tc_plan* plan, int i, int* out, int cap) {
    if (!plan || i < 0 || i >= int(plan->eng->plan.ops.size())) return fail(TC_INVALID_ARGUMENT, "bad op index");
    const Plan& P = plan->eng->plan;
    const Op& op = P.ops[size_t(i)];
    if (op.type != OP_GEMM) return 0;
    int k = 0;
    for (int q = op.prob_begin; q < op.prob_end; ++q, ++k) {
        if (!out || k >= cap) continue;
        const GemmProb& g = P.probs[size_t(q)];
        const int v[13] = {g.m, g.n, g.k, g.a_r0, g.a_c0, g.a_kwrap, g.b_buf, g.b_r0, g.b_c0, g.c_r0, g.c_c0,
                           g.exec_level, g.lower};
        for (int e = 0; e < 13; ++e) out[13 * k + e] = v[e];
    }
    return op.prob_end - op.prob_begin;
}

int tc_plan_create_trsm(int n1, int m, int b, const int* levels, int nlevels, int leaf_size, tc_plan** out) {
    if (!out || !levels_ok(levels, nlevels)) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    *out = nullptr;
    try {
        Plan p = Plan::make_trsm(n1, m, b, std::vector<int>(levels, levels + nlevels), leaf_size, PlanOptions{});
        auto* h = new tc_plan;
        h->eng = std::make_unique<Engine>(std::move(p));
        *out = h;
        return TC_OK;
    } catch (const std::exception& e) {
        return fail(TC_INVALID_ARGUMENT, e.what());
    }
}

int tc_plan_create_syrk_rows(int n2, int k, int b, const int* levels, int nlevels, int row_lo, int row_hi,
                             tc_plan** out) {
    if (!out || !levels_ok(levels, nlevels)) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    *out = nullptr;
    try {
        Plan p = Plan::make_syrk_rows(n2, k, b, std::vector<int>(levels, levels + nlevels), row_lo, row_hi,
                                      PlanOptions{});
        auto* h = new tc_plan;
        h->eng = std::make_unique<Engine>(std::move(p));
        *out = h;
        return TC_OK;
    } catch (const std::exception& e) {
        return fail(TC_INVALID_ARGUMENT, e.what());
    }
}

int tc_plan_create_trsm_ext(int n1, int m, int b, const int* levels, int nlevels, int leaf_size, tc_plan** out) {
    if (!out || !levels_ok(levels, nlevels)) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    *out = nullptr;
    try {
        Plan p = Plan::make_trsm(n1, m, b, std::vector<int>(levels, levels + nlevels), leaf_size, PlanOptions{},
                                 true);
        auto* h = new tc_plan;
        h->eng = std::make_unique<Engine>(std::move(p));
        *out = h;
        return TC_OK;
    } catch (const std::exception& e) {
        return fail(TC_INVALID_ARGUMENT, e.what());
    }
}

int tc_plan_create_syrk_rows_ext(int n2, int k, int b, const int* levels, int nlevels, int row_lo, int row_hi,
                                 tc_plan** out) {
    if (!out || !levels_ok(levels, nlevels)) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    *out = nullptr;
    try {
        Plan p = Plan::make_syrk_rows(n2, k, b, std::vector<int>(levels, levels + nlevels), row_lo, row_hi,
                                      PlanOptions{}, true);
        auto* h = new tc_plan;
        h->eng = std::make_unique<Engine>(std::move(p));
        *out = h;
        return TC_OK;
    } catch (const std::exception& e) {
        return fail(TC_INVALID_ARGUMENT, e.what());
    }
}

int tc_plan_input_rows(const tc_plan* plan, int* row0, int* rows) {
    if (!plan) return fail(TC_INVALID_ARGUMENT, "null plan");
    const Plan& P = plan->eng->plan;
    if (row0) *row0 = P.user_row0;
    if (rows) *rows = P.caller_rows();
    return TC_OK;
}

int tc_plan_device_bytes(const tc_plan* plan, unsigned long long* bytes) {
    if (!plan || !bytes) return fail(TC_INVALID_ARGUMENT, "null argument");
    *bytes = plan->eng->plan.device_bytes();
    return TC_OK;
}

int tc_plan_level_buffer(tc_plan* plan, int level, void** ptr, long long* ld, int* row_lo, int* row_hi) {
    if (!plan || !ptr || !ld || !row_lo || !row_hi) return fail(TC_INVALID_ARGUMENT, "null argument");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    std::string err;
    if (!plan->eng->level_buffer(level, ptr, ld, row_lo, row_hi, &err)) return fail(TC_INVALID_ARGUMENT, err);
    return TC_OK;
}

int tc_level_image_device(int m, int n, const double* src, int lds, int level, int lower, void* dst, long long ldd,
                          void* stream) {
    if (!src || !dst || m < 0 || n < 0 || lds < m || ldd < n || level < 0 || level > 2)
        return fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    if (m == 0 || n == 0) return TC_OK;
    launch_level_image(m, n, src, lds, level, lower, dst, ldd, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TC_OK : cuda_fail(e, "level image");
}

int tc_plan_set_external_absmax(tc_plan* plan, double absmax) {
    if (!plan) return fail(TC_INVALID_ARGUMENT, "null plan");
    std::string err;
    if (!plan->eng->set_external_absmax(absmax, &err)) return fail(TC_INVALID_ARGUMENT, err);
    return TC_OK;
}

int tc_plan_extent(const tc_plan* plan, int* rows, int* cols) {
    if (!plan) return fail(TC_INVALID_ARGUMENT, "null plan");
    if (rows) *rows = plan->eng->plan.rows;
    if (cols) *cols = plan->eng->plan.cols;
    return TC_OK;
}

int tc_absmax_device(int m, int n, const double* dA, int lda, double* out, void* stream) {
    if (!dA || !out || m < 0 || n < 0 || lda < m) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    *out = 0.0;
    if (m == 0 || n == 0) return TC_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_fail(e, "alloc");
    bo_absmax(dA, lda, m, n, d, s);
    unsigned long long bits = 0;
    e = cudaMemcpyAsync(&bits, d, sizeof bits, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "absmax");
    std::memcpy(out, &bits, sizeof bits);
    return TC_OK;
}

int tc_plan_op_deps(const tc_plan* plan, int i, int* deps, int cap) {
    if (!plan || i < 0 || i >= int(plan->eng->plan.ops.size())) return -1;
    const Op& op = plan->eng->plan.ops[i];
    const int k = int(op.deps.size());
    for (int j = 0; j < k && j < cap; ++j) deps[j] = op.deps[j];
    return k;
}

int tc_potrf_device(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out, int lda_out, void* stream,
                    tc_info* info) {
    if (!plan || !dA_in || !dL_out) return fail(TC_INVALID_ARGUMENT, "null argument");
    const Plan& P = plan->eng->plan;
    const int n = P.caller_rows();  // rows of the caller's operand
    if (lda_in < n || lda_out < n) return fail(TC_INVALID_ARGUMENT, "leading dimension < rows");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    std::string err;
    plan->have_result = false;
    if (!plan->eng->enqueue(dA_in, lda_in, dL_out, lda_out, static_cast<cudaStream_t>(stream), &err))
        return fail(TC_CUDA_ERROR, err);
    if (!info) return TC_OK;
    return tc_plan_status(plan, info);
}

int tc_plan_status(tc_plan* plan, tc_info* info) {
    if (!plan) return fail(TC_INVALID_ARGUMENT, "null plan");
    std::string err;
    Failure f;
    if (!plan->eng->result(&f, &err)) return fail(TC_CUDA_ERROR, err);
    plan->last = f;
    plan->have_result = true;
    fill_info(f, info);
    if (f.status) {
        tc_info tmp;
        fill_info(f, &tmp);
        g_err = message_of(tmp);
    }
    return f.status;
}

int tc_info_message(const tc_plan*, const tc_info* info, char* buf, int buflen) {
    if (!info || !buf || buflen < 1) return fail(TC_INVALID_ARGUMENT, "null argument");
    std::snprintf(buf, size_t(buflen), "%s", message_of(*info).c_str());
    return TC_OK;
}

int tc_potrf_host(tc_plan* plan, double* A, int lda, tc_info* info) {
    if (!plan || !A) return fail(TC_INVALID_ARGUMENT, "null argument");
    const int n = plan->eng->plan.n;
    if ((plan->eng->plan.rows > 0 && plan->eng->plan.rows != n) || plan->eng->plan.user_row0 != 0)
        return fail(TC_INVALID_ARGUMENT, "the host entry point takes whole-factorization plans only");
    if (lda < n) return fail(TC_INVALID_ARGUMENT, "leading dimension < n");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    std::string err;
    plan->have_result = false;
    // copies of the caller's lower triangle overlap the factorization
    // (Engine::enqueue_host); the strict upper triangle comes back bit-for-bit
    // unchanged (only the diagonal leaf squares carry upper elements along)
    if (!plan->eng->enqueue_host(A, lda, nullptr, &err)) return fail(TC_CUDA_ERROR, err);
    tc_info local;
    const int st = tc_plan_status(plan, &local);
    if (info) *info = local;
    return st;
}

int tc_plan_timeline(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out, int lda_out, void* stream,
                     float* t_start, float* t_end, int cap) {
    if (!plan || !dA_in || !dL_out || !t_start || !t_end) return fail(TC_INVALID_ARGUMENT, "null argument");
    std::vector<float> a, b;
    std::string err;
    if (!plan->eng->timeline(dA_in, lda_in, dL_out, lda_out, static_cast<cudaStream_t>(stream), a, b, &err))
        return fail(TC_CUDA_ERROR, err);
    for (int i = 0; i < cap && i < int(a.size()); ++i) {
        t_start[i] = a[i];
        t_end[i] = b[i];
    }
    return TC_OK;
}

int tc_plan_timeline_host(tc_plan* plan, double* host, int lda, void* stream, float* t_start, float* t_end,
                          int cap_ops, float* t_h2d, int cap_h2d, float* t_d2h, int cap_d2h) {
    if (!plan || !host || !t_start || !t_end || !t_h2d || !t_d2h) return fail(TC_INVALID_ARGUMENT, "null argument");
    std::vector<float> a, b, h, d;
    std::string err;
    if (!plan->eng->timeline_host(host, lda, static_cast<cudaStream_t>(stream), a, b, h, d, &err))
        return fail(TC_CUDA_ERROR, err);
    for (int i = 0; i < cap_ops && i < int(a.size()); ++i) {
        t_start[i] = a[i];
        t_end[i] = b[i];
    }
    for (int i = 0; i < cap_h2d && i < int(h.size()); ++i) t_h2d[i] = h[i];
    for (int i = 0; i < cap_d2h && i < int(d.size()); ++i) t_d2h[i] = d[i];
    return TC_OK;
}

int tc_plan_trace_device(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out, int lda_out, void* stream,
                         float* t_ops, int cap_ops) {
    if (!plan || !dA_in || !dL_out || !t_ops) return fail(TC_INVALID_ARGUMENT, "null argument");
    std::vector<float> a;
    std::string err;
    if (!plan->eng->trace_device(dA_in, lda_in, dL_out, lda_out, static_cast<cudaStream_t>(stream), a, &err))
        return fail(TC_CUDA_ERROR, err);
    for (int i = 0; i < cap_ops && i < int(a.size()); ++i) t_ops[i] = a[i];
    return TC_OK;
}

int tc_plan_trace_host(tc_plan* plan, double* host, int lda, void* stream, float* t_ops, int cap_ops, float* t_h2d,
                       int cap_h2d, float* t_d2h, int cap_d2h) {
    if (!plan || !host || !t_ops || !t_h2d || !t_d2h) return fail(TC_INVALID_ARGUMENT, "null argument");
    std::vector<float> a, h, d;
    std::string err;
    if (!plan->eng->trace_host(host, lda, static_cast<cudaStream_t>(stream), a, h, d, &err))
        return fail(TC_CUDA_ERROR, err);
    for (int i = 0; i < cap_ops && i < int(a.size()); ++i) t_ops[i] = a[i];
    for (int i = 0; i < cap_h2d && i < int(h.size()); ++i) t_h2d[i] = h[i];
    for (int i = 0; i < cap_d2h && i < int(d.size()); ++i) t_d2h[i] = d[i];
    return TC_OK;
}

int tc_plan_profile(tc_plan* plan, const double* dA_in, int lda_in, double* dL_out, int lda_out, void* stream,
                    float* op_ms, int cap) {
    if (!plan || !dA_in || !dL_out || !op_ms) return fail(TC_INVALID_ARGUMENT, "null argument");
    std::vector<float> ms;
    std::string err;
    if (!plan->eng->profile(dA_in, lda_in, dL_out, lda_out, static_cast<cudaStream_t>(stream), ms, &err))
        return fail(TC_CUDA_ERROR, err);
    for (int i = 0; i < cap && i < int(ms.size()); ++i) op_ms[i] = ms[i];
    return TC_OK;
}

// ---------------------------------------------------------------- analysis

int tc_spd_generate_host(int n, uint64_t seed, double* A, int lda) {
    if (!A || n < 1 || lda < n) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    // analysis.cpp:12-28 streamed in one pass: draw t = j*n + i is R(i,j);
    // the first-drawn partner of each pair is parked in the lower triangle
    std::mt19937_64 rng(seed);
    const double dn = double(n);
    for (int j = 0; j < n; ++j) {
        double* col = A + size_t(j) * lda;
        for (int i = 0; i < n; ++i) {
            const double r = double(rng() >> 11) * 0x1p-53;
            if (i < j) {
                double& lo = A[size_t(i) * lda + j];  // holds R(j, i)
                const double v = 0.5 * (r + lo);      // 0.5 * (R(i,j) + R(j,i))
                col[i] = v;
                lo = v;
            } else if (i == j) {
                col[i] = 0.5 * (r + r) + dn;
            } else {
                col[i] = r;
            }
        }
    }
    return TC_OK;
}

int tc_spd_generate_device(int n, uint64_t seed, double* dA, int lda, void* stream) {
    if (!dA || n < 1 || lda < n) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the draw stream is sequential (mt19937_64): the host produces whole
    // columns of raw R into two pinned buffers while the previous chunk is in
    // flight; the device then symmetrizes in place (bit-identical)
    const size_t ccols = std::max<size_t>(1, (size_t(64) << 20) / size_t(n));  // ~512 MB chunks
    double* hbuf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
        e = cudaMallocHost(&hbuf[k], sizeof(double) * ccols * size_t(n));
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
    }
    std::mt19937_64 rng(seed);
    int k = 0;
    for (size_t c0 = 0; c0 < size_t(n) && e == cudaSuccess; c0 += ccols, k ^= 1) {
        const size_t w = std::min(ccols, size_t(n) - c0);
        e = cudaEventSynchronize(ev[k]);
        if (e != cudaSuccess) break;
        double* h = hbuf[k];
        const size_t cnt = w * size_t(n);
        for (size_t t = 0; t < cnt; ++t) h[t] = double(rng() >> 11) * 0x1p-53;
        e = cudaMemcpy2DAsync(dA + c0 * size_t(lda), sizeof(double) * size_t(lda), h, sizeof(double) * size_t(n),
                              sizeof(double) * size_t(n), w, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(ev[k], s);
    }
    if (e == cudaSuccess) {
        launch_symmetrize(dA, lda, n, s);
        e = cudaStreamSynchronize(s);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    for (int j = 0; j < 2; ++j) {
        if (hbuf[j]) cudaFreeHost(hbuf[j]);
        if (ev[j]) cudaEventDestroy(ev[j]);
    }
    if (e != cudaSuccess) return cuda_fail(e, "spd_generate_device");
    return TC_OK;
}

int tc_factorization_error_device(int n, const double* dA, int lda, const double* dL, int ldl, double* out,
                                  void* stream) {
    if (!dA || !dL || !out || n < 1) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int T = 0;
    const int tiles = fact_error_partials(n, &T);
    double* d_part = nullptr;
    int* d_flag = nullptr;
    cudaError_t e = cudaMallocAsync(&d_part, sizeof(double) * (2 * size_t(tiles) + 1), s);
    if (e != cudaSuccess) return cuda_fail(e, "alloc");
    e = cudaMallocAsync(&d_flag, sizeof(int), s);
    if (e != cudaSuccess) return cuda_fail(e, "alloc");
    launch_fact_error(n, dA, lda, dL, ldl, d_part, d_flag, T, s);
    e = cudaMemcpyAsync(out, d_part + 2 * size_t(tiles), sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d_part, s);
    cudaFreeAsync(d_flag, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "factorization_error");
    return TC_OK;
}

int tc_factorization_error_host(int n, const double* A, int lda, const double* L, int ldl, double* out) {
    if (!A || !L || !out || n < 1 || lda < n || ldl < n) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    double* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(double) * 2 * size_t(n) * size_t(n));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    double* dL = d + size_t(n) * size_t(n);
    e = cudaMemcpy2D(d, sizeof(double) * size_t(n), A, sizeof(double) * size_t(lda), sizeof(double) * size_t(n),
                     size_t(n), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy2D(dL, sizeof(double) * size_t(n), L, sizeof(double) * size_t(ldl), sizeof(double) * size_t(n),
                         size_t(n), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(d);
        return cuda_fail(e, "H2D");
    }
    const int st = tc_factorization_error_device(n, d, n, dL, n, out, nullptr);
    cudaFree(d);
    return st;
}

int tc_potrs_device(int n, const double* dL, int ldl, double* dB, int ldb, int nrhs, void* stream) {
    if (!dL || !dB || n < 1 || nrhs < 1 || ldl < n || ldb < n) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nb = (n + 63) / 64;
    double* d_work = nullptr;
    cudaError_t e = cudaMallocAsync(&d_work, sizeof(double) * potrs_work_doubles(n, nrhs) +
                                                 sizeof(int) * size_t(nb + 1) * size_t(nrhs), s);
    if (e != cudaSuccess) return cuda_fail(e, "alloc");
    int* d_cnt = reinterpret_cast<int*>(d_work + potrs_work_doubles(n, nrhs));
    launch_potrs(n, dL, ldl, dB, ldb, nrhs, d_cnt, d_work, s);
    cudaFreeAsync(d_work, s);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "potrs");
    return TC_OK;
}

int tc_potrs_batch_device(int n, int nsys, const double* const* dL, int ldl, double* const* dB, int ldb, int nrhs,
                          void* stream) {
    if (!dL || !dB || n < 1 || nsys < 0 || nrhs < 1 || ldl < n || ldb < n)
        return fail(TC_INVALID_ARGUMENT, "bad arguments");
    for (int k = 0; k < nsys; ++k)
        if (!dL[k] || !dB[k]) return fail(TC_INVALID_ARGUMENT, "null system pointer");
    if (nsys == 0) return TC_OK;
    if (!tc_device_available()) return fail(TC_NO_DEVICE, "no CUDA device");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // pointer tables (L then B) right behind the workspace
    const size_t wbytes = (potrs_batch_work_bytes(n, nsys, nrhs) + 15) / 16 * 16;
    void* d_work = nullptr;
    cudaError_t e = cudaMallocAsync(&d_work, wbytes + 2 * sizeof(void*) * size_t(nsys), s);
    if (e != cudaSuccess) return cuda_fail(e, "alloc");
    std::vector<const void*> tab(2 * size_t(nsys));
    for (int k = 0; k < nsys; ++k) {
        tab[size_t(k)] = dL[k];
        tab[size_t(nsys + k)] = dB[k];
    }
    void** d_tab = reinterpret_cast<void**>(static_cast<char*>(d_work) + wbytes);
    e = cudaMemcpyAsync(d_tab, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        launch_potrs_batch(n, nsys, reinterpret_cast<const double* const*>(d_tab), ldl,
                           reinterpret_cast<double* const*>(d_tab + nsys), ldb, nrhs, d_work, 148 * 6, s);
        e = cudaStreamSynchronize(s);  // the host table must outlive the copy
    }
    cudaFreeAsync(d_work, s);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "potrs batch");
    return TC_OK;
}

int tc_solve_residual_device(int n, const double* dA, int lda, const double* dX, const double* dB, double* out,
                             void* stream) {
    if (!dA || !dX || !dB || !out || n < 1) return fail(TC_INVALID_ARGUMENT, "bad arguments");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nb = residual_partials(n);
    double* d_part = nullptr;
    cudaError_t e = cudaMallocAsync(&d_part, sizeof(double) * (4 * size_t(nb) + 1), s);
    if (e != cudaSuccess) return cuda_fail(e, "alloc");
    launch_residual(n, dA, lda, dX, dB, d_part, s);
    e = cudaMemcpyAsync(out, d_part + 4 * size_t(nb), sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d_part, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "residual");
    return TC_OK;
}

}  // extern "C"

namespace tcb {
void leaf_debug_clocks(long long* out, bool reset);
}
namespace tcb {
void potrf_debug_clocks(long long* out, bool reset);
}
extern "C" int tc_debug_potrf_clocks(long long* out8, int reset) {
    tcb::potrf_debug_clocks(out8, reset != 0);
    return TC_OK;
}
extern "C" int tc_debug_leaf_clocks(long long* out4, int reset) {
    tcb::leaf_debug_clocks(out4, reset != 0);
    return TC_OK;
}
namespace tcb {
void inv_debug_clocks(long long* out, bool reset);
}
extern "C" int tc_debug_inv_clocks(long long* out8, int reset) {
    tcb::inv_debug_clocks(out8, reset != 0);
    return TC_OK;
}
