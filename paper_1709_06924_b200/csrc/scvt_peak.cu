// scvt_peak.cu — FP64 FMA throughput microbenchmark (roofline denominator).
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the quadrature is FP64-bound, so the
// bench measures the DFMA pipe itself: every thread runs 8 independent FMA chains so the
// pipe, not latency, is the limit.  2 FLOPs per DFMA.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scvt_b200.h"

namespace {

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
    double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 1234.5) out[0] = s;   // defeat dead-code elimination
}

}  // namespace

extern "C" int scvt_fp64_peak(int device, double* tflops_out) {
    if (cudaSetDevice(device) != cudaSuccess) return SCVT_ERR_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return SCVT_ERR_CUDA;
    const int blocks = sms * 8, threads = 256, iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);   // warm-up
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8.0 * 16.0 * (double)iters * blocks * threads;
        double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return SCVT_ERR_CUDA;
    *tflops_out = best;
    return SCVT_OK;
}
