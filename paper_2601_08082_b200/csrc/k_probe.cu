// k_probe.cu -- development probe: throughput of the legacy warp-level
// tensor-core path (mma.sync) on one SM, to size leaf-kernel choices.
#include <cuda_runtime.h>

#include "device.cuh"
#include "launch.hpp"

namespace tcb {
namespace {
__global__ void k_mma_tf32(float* out, int iters) {
    float c[4][4] = {};
    uint32_t a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
    uint32_t b[2] = {threadIdx.x * 3, threadIdx.x * 5};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mma_f16(float* out, int iters) {
    float c[4][4] = {};
    uint32_t a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
    uint32_t b[2] = {threadIdx.x * 3, threadIdx.x * 5};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// the FP64 tensor pipe: mma.sync m8n8k4 f64 (DMMA), 4 independent chains
__global__ void k_mma_f64(double* out, int iters) {
    double c[4][2] = {};
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[q][0]), "+d"(c[q][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// plain FP64 FMA (DFMA) on the SIMT pipe, 8 independent chains per thread
__global__ void k_dfma(double* out, int iters) {
    double c[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = q;
    const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) c[q] = fma(c[q], a, b);
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

// FP64 FLOP/s of the whole GPU (ctas CTAs of 256 threads): kind 0 DMMA
// m8n8k4 (the FP64 tensor pipe), 1 DFMA (SIMT)
double probe_fp64(int kind, int iters, int ctas) {
    double* d = nullptr;
    cudaMalloc(&d, size_t(ctas) * 256 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&] {
        if (kind == 0) k_mma_f64<<<ctas, 256>>>(d, iters);
        else k_dfma<<<ctas, 256>>>(d, iters);
    };
    run();
    cudaEventRecord(e0);
    run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(d);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double warps = double(ctas) * 8;
    // DMMA m8n8k4: 256 FMAs per warp instruction; DFMA: 32 per warp instruction
    const double flop = kind == 0 ? warps * iters * 4 * 256 * 2 : warps * iters * 8 * 32 * 2;
    return flop / (ms * 1e-3);
}

// FMA/s of one SM (1 CTA of 512 threads) on mma.sync: kind 0 tf32 m16n8k8, 1 f16 m16n8k16
double probe_mma(int kind, int iters) {
    float* d = nullptr;
    cudaMalloc(&d, 512 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&] {
        if (kind == 0) k_mma_tf32<<<1, 512>>>(d, iters);
        else k_mma_f16<<<1, 512>>>(d, iters);
    };
    run();
    cudaEventRecord(e0);
    run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaFree(d);
    const double fma_per_mma = kind == 0 ? 16.0 * 8 * 8 : 16.0 * 8 * 16;
    return 16.0 * iters * 4 * fma_per_mma / (ms * 1e-3);  // 16 warps
}
}  // namespace tcb

extern "C" double tc_debug_mma_probe(int kind, int iters) { return tcb::probe_mma(kind, iters); }
extern "C" double tc_debug_fp64_probe(int kind, int iters, int ctas) { return tcb::probe_fp64(kind, iters, ctas); }

