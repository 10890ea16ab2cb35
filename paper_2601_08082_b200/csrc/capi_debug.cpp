// capi_debug.cpp -- development entry points (declared in treechol_c.h under
// "development"): one grouped-GEMM launch of a given operand class on scratch
// buffers, timed with CUDA events, for kernel tuning and single-kernel ncu
// captures.  Not used by the factorization path.
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/treechol_c.h"
#include "launch.hpp"
#include "plan.hpp"

using namespace tcb;

namespace tcb {
void set_last_error(const std::string& msg);  // capi.cpp
}

static unsigned long long g_last_stamps[15];

// %globaltimer stamps (ns) of CTA 0 of the last tc_debug_gemm launch:
// entry, after setup, first TMA issued, first stage landed, accumulator
// ready, epilogue done, exit (tcgen05 classes)
extern "C" int tc_debug_gemm_stamps(unsigned long long* out7) {
    if (!out7) return TC_INVALID_ARGUMENT;
    for (int i = 0; i < 15; ++i) out7[i] = g_last_stamps[i];
    return TC_OK;
}

extern "C" int tc_debug_gemm(int gclass, int m, int n, int k, int lower, double beta, int exec_level, int iters,
                             float* avg_us) {
    if (m < 1 || n < 1 || k < 1 || iters < 1 || !avg_us) return TC_INVALID_ARGUMENT;
    const long long rows = (long long)m + n + k;
    const long long ldw = ((k + n + 63) / 64) * 64;  // A at cols [0,k), C at cols [k, k+n)
    DevCtx c{};
    c.ldw = ldw;
    void* buf = nullptr;
    unsigned long long* words = nullptr;
    const size_t elems = size_t(rows) * size_t(ldw);
    if (cudaMalloc(&buf, elems * (2 + 4 + 8)) != cudaSuccess) return TC_CUDA_ERROR;
    cudaMalloc(&words, 256);
    cudaMemset(buf, 0, elems * 14);
    cudaMemset(words, 0xFF, 8);
    cudaMemset(words + 1, 0, 128);
    c.b16 = static_cast<__half*>(buf);
    c.b32 = reinterpret_cast<float*>(c.b16 + elems);
    c.b64 = reinterpret_cast<double*>(c.b32 + elems);
    c.status = words;
    c.stamps = words + 1;  // 15 stamps of the last launch's CTA 0 (words: 256 bytes)
    init_tc_attributes();
    init_mma32w_attributes();
    DevProb d{};
    d.m = m;
    d.n = n;
    d.k = k;
    d.a_r0 = n;  // A rows [n, n+m), B rows [0, n), both at cols [0, k)
    d.a_c0 = 0;
    d.b_r0 = 0;
    d.b_c0 = 0;
    d.c_r0 = n;
    d.c_c0 = k;
    if (lower) {  // syrk leaf: C square on the diagonal (rows and cols [k, k+m))
        d.b_r0 = n;
        d.c_r0 = k;
        d.c_c0 = k;
    }
    d.exec_level = exec_level;
    d.lower = lower;
    d.alpha = -1.0;
    d.beta = beta;
    d.b_buf = -1;
    std::vector<DevProb> v{d};
    std::vector<unsigned char> host;
    int tiles = 0;
    const bool tc = gclass == GC_TC16 || gclass == GC_TC32;
    std::string err;
    int pair = 0, kind = KIND_F16;
    if (tc) {
        tiles = tc_select_tables(c, gclass == GC_TC32, v, host, &err, tc_pair_min_tiles(), -1, &kind, &pair);
    } else {
        tiles = gclass == GC_MMA32W ? simt_tiles(v, M32W_ROWS, 256) : simt_tiles(v, gclass == GC_MMA32 ? M32_TILE : 0);
        host.assign(reinterpret_cast<unsigned char*>(v.data()), reinterpret_cast<unsigned char*>(v.data() + 1));
    }
    void* dprob = nullptr;
    cudaMalloc(&dprob, host.size());
    cudaMemcpy(dprob, host.data(), host.size(), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&] {
        if (pair) launch_gemm_tc_pair(c, kind, dprob, 1, tiles, nullptr);
        else if (tc) launch_gemm_tc(c, kind, dprob, 1, tiles, nullptr);
        else launch_gemm_simt(c, gclass, static_cast<DevProb*>(dprob), 1, tiles, nullptr);
    };
    launch();  // warm
    // back-to-back launches captured in a graph: device time per launch
    // without host launch gaps
    cudaStream_t cs;
    cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < iters; ++i) {
        if (pair) launch_gemm_tc_pair(c, kind, dprob, 1, tiles, cs);
        else if (tc) launch_gemm_tc(c, kind, dprob, 1, tiles, cs);
        else launch_gemm_simt(c, gclass, static_cast<DevProb*>(dprob), 1, tiles, cs);
    }
    cudaStreamEndCapture(cs, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, cs);
    cudaStreamSynchronize(cs);
    cudaEventRecord(e0, cs);
    cudaGraphLaunch(ge, cs);
    cudaEventRecord(e1, cs);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *avg_us = ms * 1000.f / float(iters);
    cudaMemcpy(g_last_stamps, words + 1, sizeof(g_last_stamps), cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(dprob);
    cudaFree(words);
    cudaFree(buf);
    if (e != cudaSuccess) {
        set_last_error(cudaGetErrorString(e));
        return TC_CUDA_ERROR;
    }
    return TC_OK;
}

// one problem of grouped-GEMM class gclass on CALLER level buffers (the
// engine's row-major layout, ld = ldw): the exact launch path the
// factorization graph uses, for kernel-level parity tests against
// gemm_mixed / syrk_leaf (kernels.cpp:94-132).  prob = {m, n, k, a_r0,
// a_c0, b_r0, b_c0, c_r0, c_c0, exec_level, lower}; A and B are read from
// the operand level's buffer (F16 for the FP16 classes, F32 for the FP32
// ones, F64 for GC_SIMT_F64), C from / to the exec level's buffer.
extern "C" int tc_gemm_problem_device(int gclass, void* b16, void* b32, void* b64, long long ldw, const int* prob,
                                      double alpha, double beta, void* stream) {
    if (!prob || ldw < 1 || gclass < 0 || gclass > GC_MMA32W) return TC_INVALID_ARGUMENT;
    DevProb d{};
    d.m = prob[0];
    d.n = prob[1];
    d.k = prob[2];
    d.a_r0 = prob[3];
    d.a_c0 = prob[4];
    d.b_r0 = prob[5];
    d.b_c0 = prob[6];
    d.c_r0 = prob[7];
    d.c_c0 = prob[8];
    d.exec_level = prob[9];
    d.lower = prob[10];
    d.alpha = alpha;
    d.beta = beta;
    d.b_buf = -1;
    if (d.m < 1 || d.n < 1 || d.k < 1) return TC_INVALID_ARGUMENT;
    if (!tc_device_available()) return TC_NO_DEVICE;
    DevCtx c{};
    c.ldw = ldw;
    c.b16 = static_cast<__half*>(b16);
    c.b32 = static_cast<float*>(b32);
    c.b64 = static_cast<double*>(b64);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long* words = nullptr;
    if (cudaMallocAsync(&words, 64, s) != cudaSuccess) return TC_CUDA_ERROR;
    cudaMemsetAsync(words, 0xFF, 64, s);
    c.status = words;
    init_tc_attributes();
    init_mma32w_attributes();
    std::vector<DevProb> v{d};
    std::vector<unsigned char> host;
    int tiles = 0;
    const bool tc = gclass == GC_TC16 || gclass == GC_TC32;
    std::string err;
    int pair = 0, kind = KIND_F16;
    if (tc) {
        tiles = tc_select_tables(c, gclass == GC_TC32, v, host, &err, tc_pair_min_tiles(), -1, &kind, &pair);
        if (tiles <= 0) {
            cudaFreeAsync(words, s);
            set_last_error("tc_build_probs: " + err);
            return TC_INVALID_ARGUMENT;
        }
    } else {
        tiles = gclass == GC_MMA32W ? simt_tiles(v, M32W_ROWS, 256) : simt_tiles(v, gclass == GC_MMA32 ? M32_TILE : 0);
        host.assign(reinterpret_cast<unsigned char*>(v.data()), reinterpret_cast<unsigned char*>(v.data() + 1));
    }
    void* dprob = nullptr;
    if (cudaMallocAsync(&dprob, host.size(), s) != cudaSuccess) return TC_CUDA_ERROR;
    cudaMemcpyAsync(dprob, host.data(), host.size(), cudaMemcpyHostToDevice, s);
    if (pair) launch_gemm_tc_pair(c, kind, dprob, 1, tiles, s);
    else if (tc) launch_gemm_tc(c, kind, dprob, 1, tiles, s);
    else launch_gemm_simt(c, gclass, static_cast<DevProb*>(dprob), 1, tiles, s);
    cudaFreeAsync(dprob, s);
    cudaFreeAsync(words, s);
    const cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        set_last_error(cudaGetErrorString(e));
        return TC_CUDA_ERROR;
    }
    return TC_OK;
}

// process-wide kernel settings (development / A-B measurements)
extern "C" int tc_set_global_option(const char* key, int value) {
    if (!key) return TC_INVALID_ARGUMENT;
    if (tc_set_option(key, value) || potrs_set_option(key, value) || elem_set_option(key, value)) return TC_OK;
    set_last_error(std::string("unknown global option '") + key + "'");
    return TC_INVALID_ARGUMENT;
}
