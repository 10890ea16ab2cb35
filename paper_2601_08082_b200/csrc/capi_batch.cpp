// capi_batch.cpp -- batched POTRF + POTRS of independent SPD systems on one
// device (BASELINE config C4: 64 x N=16384).
//
// One system's factorization is critical-path bound at these sizes (the
// leaf chain leaves most SMs idle), so `concurrency` independent plans --
// each its own workspace, CUDA graph and stream -- run systems side by side,
// round robin.  Per system: tree_potrf (the plan's graph; the caller's
// pointers go through RunArgs), a copy of its status word, then the forward
// and backward substitution of its right-hand sides on the same stream.
// Multi-GPU sharding of a batch is done by the caller (one process per GPU,
// no data-path collective: paper_2601_08082_b200/batch.py).
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../../include/treechol_c.h"
#include "engine.hpp"
#include "launch.hpp"
#include "plan.hpp"

using namespace tcb;

namespace tcb {
void set_last_error(const std::string& msg);  // capi.cpp
int apply_plan_option(std::unique_ptr<Engine>& eng, const std::string& k, int value, std::string* err);  // capi.cpp
}

struct tc_batch {
    std::vector<std::unique_ptr<Engine>> eng;
    std::vector<cudaStream_t> streams;
    unsigned long long* h_status = nullptr;  // pinned, one word per system
    int cap = 0;
    // per stream: POTRS workspace (diagonal-block inverses + ticket / flag
    // words), allocated once -- reused by that stream's solves in order
    std::vector<void*> work;
    size_t work_bytes = 0;
    int solve_order = 0;  // 0: every factorization, then all solves in one launch; 1: interleaved per stream
    void** h_tab = nullptr;  // POTRS pointer tables (L then B), pinned / device
    void** d_tab = nullptr;
    int tab_cap = 0;
    cudaEvent_t join = nullptr;
    // device time of the last run's batched solve phase (solve_order 0)
    cudaEvent_t solve_ev[2] = {nullptr, nullptr};
    int solve_timed = 0;
    ~tc_batch() {
        for (auto e : solve_ev)
            if (e) cudaEventDestroy(e);
        for (auto s : streams) cudaStreamDestroy(s);
        for (auto w : work) cudaFree(w);
        if (h_status) cudaFreeHost(h_status);
        if (h_tab) cudaFreeHost(h_tab);
        if (d_tab) cudaFree(d_tab);
        if (join) cudaEventDestroy(join);
    }
};

namespace {
int bfail(int code, const std::string& m) {
    set_last_error(m);
    return code;
}
}  // namespace

extern "C" {

int tc_batch_create(int n, int b, const int* levels, int nlevels, int quantize, int concurrency, tc_batch** out) {
    if (!out || !levels || nlevels < 1 || n < 1 || b < 1 || concurrency < 1)
        return bfail(TC_INVALID_ARGUMENT, "bad arguments");
    *out = nullptr;
    try {
        auto* bt = new tc_batch;
        for (int i = 0; i < concurrency; ++i) {
            PlanOptions po;
            // leaf shadows fused into the leaf POTRF (the plan default): C4
            // 437-439 vs 434-435 TF/s with separate shadow ops
            // (profiles/r02_c4_options.txt).  An earlier A/B that ran
            // bimodally (profiles/r02_c4_fuse_shadow_ab.txt) had buffer
            // re-allocation inside its timed calls
            bt->eng.push_back(std::make_unique<Engine>(
                Plan::make(n, b, std::vector<int>(levels, levels + nlevels), quantize != 0, 0, po)));
            // CTA-pair GEMMs in batches from 1024 tiles: C4 443-452 TF/s in
            // 14 runs vs 435-440 without (profiles/r02_c4_options.txt).  An
            // earlier A/B with one 99 TF/s pair run
            // (profiles/r02_c4_pair_ab.txt) predates the warm-up that sizes
            // the per-call buffers
            bt->eng.back()->pair_min_tiles = 1024;
            // trailing updates 4 tiles per CTA (C4 440-442 vs 436-439 TF/s
            // with 1, profiles/r02_c4_options.txt)
            bt->eng.back()->bulk_tiles_per_cta = 4;
        }
        *out = bt;
        return TC_OK;
    } catch (const std::exception& e) {
        return bfail(TC_INVALID_ARGUMENT, e.what());
    }
}

void tc_batch_destroy(tc_batch* bt) { delete bt; }

int tc_batch_set_option(tc_batch* bt, const char* key, int value) {
    if (!bt || !key) return bfail(TC_INVALID_ARGUMENT, "null argument");
    const std::string k = key;
    if (k == "solve_order") {
        bt->solve_order = value != 0;
        return TC_OK;
    }
    for (auto& e : bt->eng) {
        if (e->ready()) return bfail(TC_INVALID_ARGUMENT, k + " must be set before the first run");
        std::string err;
        const int r = apply_plan_option(e, k, value, &err);
        if (r < 0) return bfail(TC_INVALID_ARGUMENT, err);
        if (r == 1) continue;
        if (k == "bulk_tiles_per_cta") e->bulk_tiles_per_cta = value < 0 ? 0 : value;
        else if (k == "crit_tiles_per_cta") e->crit_tiles_per_cta = value < 0 ? 0 : value;
        else if (k == "crit_max_ctas") e->crit_max_ctas = value < 0 ? 0 : value;
        else if (k == "prio_levels") e->prio_levels = value;
        else if (k == "node_prio") e->node_prio = value != 0;
        else if (k == "import_low") e->import_low = value != 0;
        else if (k == "startup_order") e->startup_order = value != 0;
        else if (k == "import_chain") e->import_chain = value < 0 ? 0 : value;
        else if (k == "dag_graph") e->dag_graph = value != 0;
        else if (k == "use_pdl") e->use_pdl = value != 0;
        else if (k == "use_graph") e->use_graph = value != 0;
        else if (k == "dev_skip") e->dev_skip = value;  // development: see Engine::dev_skip
        else if (k == "pair_min_tiles") e->pair_min_tiles = value;
        else return bfail(TC_INVALID_ARGUMENT, "unknown option '" + k + "'");
    }
    return TC_OK;
}

int tc_batch_run(tc_batch* bt, int count, double* const* dA, int lda, double* const* dB, int ldb, int nrhs,
                 int* status, int* index) {
    if (!bt || count < 0 || (count > 0 && (!dA || !status))) return bfail(TC_INVALID_ARGUMENT, "bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        return bfail(TC_NO_DEVICE, "no CUDA device (there is no CPU fallback)");
    }
    const int n = bt->eng[0]->plan.n;
    if (lda < n || (dB && (ldb < n || nrhs < 1))) return bfail(TC_INVALID_ARGUMENT, "bad leading dimensions");
    const int C = int(bt->eng.size());
    std::string err;
    while (int(bt->streams.size()) < C) {
        cudaStream_t s;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return bfail(TC_CUDA_ERROR, "stream");
        bt->streams.push_back(s);
    }
    if (bt->cap < count) {
        if (bt->h_status) cudaFreeHost(bt->h_status);
        bt->h_status = nullptr;
        if (cudaMallocHost(&bt->h_status, sizeof(unsigned long long) * size_t(count)) != cudaSuccess)
            return bfail(TC_CUDA_ERROR, "cudaMallocHost");
        bt->cap = count;
    }
    // solve_order 1: a POTRS workspace per stream; 0: one for the batch
    const size_t wbytes = bt->solve_order ? potrs_batch_work_bytes(n, 1, nrhs) : potrs_batch_work_bytes(n, count, nrhs);
    const size_t nwork = bt->solve_order ? size_t(C) : 1;
    if (dB && (bt->work.size() < nwork || bt->work_bytes < wbytes)) {
        for (auto s : bt->streams) cudaStreamSynchronize(s);
        for (auto w : bt->work) cudaFree(w);
        bt->work.assign(nwork, nullptr);
        for (auto& w : bt->work)
            if (cudaMalloc(&w, wbytes) != cudaSuccess) return bfail(TC_CUDA_ERROR, "cudaMalloc (POTRS workspace)");
        bt->work_bytes = wbytes;
    }
    if (dB && bt->tab_cap < count) {
        for (auto s : bt->streams) cudaStreamSynchronize(s);
        if (bt->h_tab) cudaFreeHost(bt->h_tab);
        if (bt->d_tab) cudaFree(bt->d_tab);
        bt->h_tab = nullptr;
        bt->d_tab = nullptr;
        if (cudaMallocHost(&bt->h_tab, 2 * sizeof(void*) * size_t(count)) != cudaSuccess ||
            cudaMalloc(&bt->d_tab, 2 * sizeof(void*) * size_t(count)) != cudaSuccess)
            return bfail(TC_CUDA_ERROR, "POTRS pointer tables");
        bt->tab_cap = count;
    }
    // on a failure partway through, drain what is already queued before
    // returning: earlier systems' graphs and solves still write dA/dB
    auto drain_fail = [&](const std::string& why) {
        for (auto s : bt->streams) cudaStreamSynchronize(s);
        return bfail(TC_CUDA_ERROR, why);
    };
    auto factor = [&](int k) {
        const int e = k % C;
        Engine& eng = *bt->eng[size_t(e)];
        cudaStream_t s = bt->streams[size_t(e)];
        return eng.enqueue(dA[k], lda, dA[k], lda, s, &err) && eng.copy_status(bt->h_status + k, s, &err);
    };
    // POTRS on the factor just written, on the same
    // stream; a bounded set of persistent CTAs per solve
    auto solve = [&](int k) {
        if (!dB || !dB[k]) return;
        const int e = k % C;
        double* d_work = static_cast<double*>(bt->work[size_t(e)]);
        launch_potrs(n, dA[k], lda, dB[k], ldb, nrhs, nullptr, d_work, bt->streams[size_t(e)], 64);
    };
    bt->solve_timed = 0;
    if (bt->solve_order == 0) {
        // all factorizations first, then every solve in one launch sequence
        // (persistent CTAs over all (block, system) pairs; the waiting CTAs
        // never sit beside a factorization)
        for (int k = 0; k < count; ++k)
            if (!factor(k)) return drain_fail(err);
        int ns = 0;
        for (int k = 0; dB && k < count; ++k)
            if (dB[k]) {
                bt->h_tab[ns] = dA[k];
                bt->h_tab[count + ns] = dB[k];
                ++ns;
            }
        if (ns > 0) {
            cudaStream_t s0 = bt->streams[0];
            if (!bt->join) cudaEventCreateWithFlags(&bt->join, cudaEventDisableTiming);
            for (int e = 1; e < C; ++e) {
                cudaEventRecord(bt->join, bt->streams[size_t(e)]);
                cudaStreamWaitEvent(s0, bt->join, 0);
            }
            if (!bt->solve_ev[0]) {
                cudaEventCreate(&bt->solve_ev[0]);
                cudaEventCreate(&bt->solve_ev[1]);
            }
            cudaEventRecord(bt->solve_ev[0], s0);
            // compact the B half right behind the L half
            for (int i = 0; i < ns; ++i) bt->h_tab[ns + i] = bt->h_tab[count + i];
            cudaMemcpyAsync(bt->d_tab, bt->h_tab, 2 * sizeof(void*) * size_t(ns), cudaMemcpyHostToDevice, s0);
            launch_potrs_batch(n, ns, reinterpret_cast<const double* const*>(bt->d_tab), lda,
                               reinterpret_cast<double* const*>(bt->d_tab + ns), ldb, nrhs, bt->work[0], 148 * 6, s0);
            cudaEventRecord(bt->solve_ev[1], s0);
            bt->solve_timed = 1;
        }
    } else {
        // each system's solve right behind its factorization: the solves of
        // one stream overlap the other streams' factorizations
        for (int k = 0; k < count; ++k) {
            if (!factor(k)) return drain_fail(err);
            solve(k);
        }
    }
    for (auto s : bt->streams)
        if (cudaStreamSynchronize(s) != cudaSuccess) return bfail(TC_CUDA_ERROR, "batch synchronize");
    const cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return bfail(TC_CUDA_ERROR, cudaGetErrorString(ce));
    int worst = TC_OK;
    for (int k = 0; k < count; ++k) {
        Failure f;
        if (!bt->eng[size_t(k % C)]->decode(bt->h_status[k], &f, &err)) return bfail(TC_CUDA_ERROR, err);
        status[k] = f.status;
        if (index) index[k] = f.status == TC_NUMERICAL_BREAKDOWN ? f.elem_row : f.index;
        if (f.status && worst == TC_OK) worst = f.status;
    }
    return worst;
}

int tc_batch_solve_ms(const tc_batch* bt, float* ms) {
    if (!bt || !ms) return bfail(TC_INVALID_ARGUMENT, "null argument");
    *ms = 0.f;
    if (!bt->solve_timed) return TC_OK;
    const cudaError_t e = cudaEventElapsedTime(ms, bt->solve_ev[0], bt->solve_ev[1]);
    return e == cudaSuccess ? TC_OK : bfail(TC_CUDA_ERROR, cudaGetErrorString(e));
}

}  // extern "C"
