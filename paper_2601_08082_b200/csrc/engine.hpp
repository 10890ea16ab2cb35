// engine.hpp -- executes a Plan on one device (internal).
//
// The op list is enqueued on a pool of CUDA streams, each op waiting on the
// events of the deps that live on other streams; the whole enqueue is
// captured once into a CUDA graph (cached per plan) and replayed per call.
// Device state per plan: the level buffers, the status word, the quantize
// alpha slots, the launch tables, and a RunArgs block the kernels read the
// caller's pointers from (so one graph serves every call).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "device.cuh"
#include "plan.hpp"

namespace tcb {

struct OpLaunch {
    int tiles = 0;
    int count = 0;
    int pair = 0;       // tcgen05 FP16 kind on CTA pairs (k_gemm_tc2)
    int kind = 0;       // tcgen05 kind (KIND_*)
    size_t offset = 0;  // into the table arena
};

struct Failure {
    int status = 0;  // tc_status
    int index = -1;
    Rect block;
    int elem_row = -1, elem_col = -1;
    int diagonal = 0;
    uint32_t seq = 0;
};

class Engine {
   public:
    explicit Engine(Plan p) : plan(std::move(p)) {}
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    Plan plan;
    bool use_graph = true;
    int n_streams = 6;
    // development (measurements only; results are garbage): ops whose type
    // bit (1 << OpType) or GEMM class bit (1 << (16 + GemmClass)) is set
    // launch an empty kernel instead
    int dev_skip = 0;
    // DAG graph: single-kernel ops as kernel nodes, with programmatic
    // dependent launch (PDL) on the edges into the chain's ops: the kernel
    // is launched while its producer finishes and waits in
    // griddepcontrol.wait (every factorization kernel starts with it)
    // CTA-pair GEMM threshold for this engine (-1: the process-wide
    // tc_pair_min_tiles; 0: never)
    int pair_min_tiles = -1;
    // narrow (128x128) FP16 tiles below this many 128x256 tiles (-1: the
    // process-wide tc_narrow_max_tiles)
    int narrow_max_tiles = -1;
    bool use_pdl = false;  // measured no faster (N=16384 12.62 -> 12.80 ms, C4 425 -> 420 TF/s): off
    bool pdl_src_ok(int i) const;
    int bulk_tiles_per_cta = 1;  // trailing-update GEMMs: 0 persistent, else tiles per CTA (1: SMs free up after every tile, so concurrent work -- other systems of a batch, the factorization chain -- gets them)
    int bulk_max_ctas = 0;       // persistent trailing-update GEMMs: CTA cap (0 = one per SM)
    int crit_tiles_per_cta = 0;  // the other (critical) tensor-core GEMMs: 0 persistent, else tiles per CTA
    int crit_max_ctas = 0;       // persistent critical GEMMs: CTA cap (0 = one per SM)
    // DAG-graph scheduling priorities: 2 = {chain + critical GEMMs, bulk};
    // 3 = {leaf chain, critical FP16 GEMMs, bulk}: the chain's small kernels
    // are dispatched before the queued CTAs of a big critical GEMM
    int prio_levels = 2;
    // DAG graphs instantiated with cudaGraphInstantiateFlagUseNodePriority:
    // without it a graph launch ignores the per-node priorities above and
    // runs every kernel at the launching stream's priority
    bool node_prio = false;
    bool import_low = false;  // imports at the bulk (lowest) priority
    // host path: an exported block's D2H starts when its export op has run
    // (an event-record node after it in the phase graph), not when its
    // whole phase has finished.  Measured neutral at C3 (0.533-0.536 s both
    // ways, profiles/r02_e2e_export_events.txt): the D2H tail is the L21
    // panel, which cannot be solved before all of A21 has landed
    bool export_events = false;
    bool startup_order = false;  // see build_dag_graph
    int import_chain = 0;        // device graph: at most this many imports in flight (0 = all at once)
    unsigned long long inst_flags() const { return node_prio ? cudaGraphInstantiateFlagUseNodePriority : 0; }
    bool dag_graph = true;       // explicit DAG graph (else: captured multi-stream enqueue)

    // enqueue one factorization (import .. export) on `stream`
    bool enqueue(const double* a_in, long long lda_in, double* l_out, long long lda_out, cudaStream_t stream,
                 std::string* err);
    // host buffers (the TileView contract): H2D of the lower triangle in
    // leaf-column strips, the factorization on a device staging copy, and a
    // D2H of every block as soon as it is exported -- copies overlap the
    // compute.  Captured into its own graph per (host pointer, lda) when the
    // buffer is pinned; eager otherwise.
    bool enqueue_host(double* host, long long lda, cudaStream_t stream, std::string* err);
    // wait for the last enqueue and decode the status word
    bool result(Failure* f, std::string* err);
    // enqueue a copy of the status word of the run just enqueued on `s`
    // into host memory (batched drivers), and decode such a copy
    bool copy_status(unsigned long long* host_slot, cudaStream_t s, std::string* err);
    bool decode(unsigned long long key, Failure* f, std::string* err) const;
    // serialized eager run with an event after every op (per-op timing)
    bool profile(const double* a_in, long long lda_in, double* l_out, long long lda_out, cudaStream_t stream,
                 std::vector<float>& op_ms, std::string* err);
    // partial flops of a failed run: calls with seq < failing seq
    int launches_per_run() const;

    bool ready() const { return ready_; }
    // distributed panel plans: the all-reduced max|B| of the panel rows
    bool set_external_absmax(double amax, std::string* err);
    // the real start (row row_lo) of a level buffer's allocated window, its
    // row stride in elements and the window rows (allocates if needed)
    bool level_buffer(int level, void** ptr, long long* ld, int* row_lo, int* row_hi, std::string* err);
    bool prepare(std::string* err);

   private:
    bool ready_ = false;
    int device_ = -1;
    DevCtx ctx_{};
    RunArgs* d_ra_ = nullptr;
    RunArgs* h_ra_ = nullptr;
    unsigned long long* h_status_ = nullptr;
    unsigned long long* h_ext_ = nullptr;     // pinned: external max|B| bits
    void* d_bufs_ = nullptr;
    size_t buf_off_[3] = {0, 0, 0};          // level windows inside d_bufs_
    unsigned long long* d_words_ = nullptr;  // status + alpha slots
    void* d_w16_ = nullptr;                  // leaf inverses + scales
    void* d_w32_ = nullptr;                  // FP32 leaf inverses
    unsigned char* d_arena_ = nullptr;
    std::vector<OpLaunch> launch_;
    std::vector<cudaStream_t> streams_;
    std::vector<cudaEvent_t> events_;
    cudaEvent_t fork_ = nullptr;
    cudaStream_t last_stream_ = nullptr;
    cudaGraph_t graph_ = nullptr;
    cudaGraphExec_t gexec_ = nullptr;
    std::vector<int> seq_op_;  // seq -> op index

    // host pipeline state
    struct HostIO {
        double* host;
        long long lda;
    };
    double* d_stage_ = nullptr;
    cudaStream_t cs_h2d_ = nullptr, cs_d2h_ = nullptr;
    std::vector<cudaEvent_t> ev_h2d_;     // per block: H2D done
    std::vector<cudaEvent_t> ev_d2h_;     // per export: D2H done (joined at the end)
    std::vector<cudaEvent_t>* tl_h2d_ = nullptr;  // timeline_host: timing events after each copy
    std::vector<cudaEvent_t>* tl_d2h_ = nullptr;
    bool ensure_stage(std::string* err);
    bool run_host(const HostIO& io, cudaStream_t stream, std::string* err);
    bool run_host_pipeline(const HostIO& io, cudaStream_t stream, std::string* err);
    std::vector<Rect> hc_rect_, dc_rect_;      // H2D chunks (block order), D2H chunks (by phase)
    std::vector<int> dc_phase_, ph_need_;      // phase of each D2H chunk; last H2D chunk a phase reads
    std::vector<int> dc_op_;                   // export op of each D2H chunk
    std::vector<cudaEvent_t> ev_ex_;           // per op: event recorded in its phase graph after an export
    std::vector<cudaEvent_t> ev_hc_, ev_dc_;   // per chunk: copy done
    unsigned long long* d_trace_ = nullptr;  // trace_host: stamp slots (null: no stamp nodes)
    cudaGraph_t hgraph_ = nullptr;
    cudaGraphExec_t hexec_ = nullptr;
    const double* hkey_ = nullptr;
    long long hkey_lda_ = 0;

    std::vector<cudaEvent_t> ra_ev_;  // per RunArgs slot: its H2D copy was issued
    int ra_next_ = 0;
    RunArgs* next_args(std::string* err);

    void launch_op(int i, cudaStream_t s);
    void reset_words(cudaStream_t s);
    bool enqueue_ops(cudaStream_t origin, std::string* err, const HostIO* io = nullptr,
                     std::vector<cudaEvent_t>* tl = nullptr);
    // the op DAG as an explicit CUDA graph: one child-graph node per op (its
    // launch captured alone), edges = the plan's dependencies only -- no
    // stream-order edges between independent ops
    bool build_dag_graph(cudaGraph_t* out, int phase, std::string* err);
    // host entry point: one DAG graph per phase of the H2D stream
    std::vector<cudaGraphExec_t> hph_exec_;
    std::vector<cudaEvent_t> ev_ph_;
    std::vector<int> ph_op_, ph_wait_;  // phase of each op; last block (H2D position) a phase reads (-1: none)
    bool build_host_phases(std::string* err);
    void drop_host_phases();

   public:
    // eager multi-stream run with a timing event before and after every op:
    // start/end (ms from the first op's start) -- the concurrency timeline
    bool timeline(const double* a_in, long long lda_in, double* l_out, long long lda_out, cudaStream_t stream,
                  std::vector<float>& t0, std::vector<float>& t1, std::string* err);
    // the same for the host entry point (eager): op start/end plus the
    // completion time of every H2D copy (block order) and D2H copy (export
    // order), ms from the first H2D's start
    bool timeline_host(double* host, long long lda, cudaStream_t stream, std::vector<float>& t0,
                       std::vector<float>& t1, std::vector<float>& th2d, std::vector<float>& td2h, std::string* err);
    // the host entry point's pipeline itself (DAG graph phases), with a
    // global-timer stamp after the root, every op and every H2D / D2H copy
    // chunk: completion times (ms from the root) -- ops in op order, H2D
    // chunks in issue order, D2H chunks in issue order
    // development: one run of the device-path DAG graph with a global-timer
    // stamp after every op; completion times in ms from the root
    bool trace_device(const double* a_in, long long lda_in, double* l_out, long long lda_out, cudaStream_t stream,
                      std::vector<float>& top, std::string* err);
    bool trace_host(double* host, long long lda, cudaStream_t stream, std::vector<float>& top,
                    std::vector<float>& th2d, std::vector<float>& td2h, std::string* err);
};

}  // namespace tcb
