// Does the FP64 tensor-core path (mma.sync m8n8k4 f64, "DMMA") run beside the DFMA pipe on
// sm_100a, or on the same units?  Three kernels with independent chains: DFMA only, DMMA only,
// and both interleaved in the proportion that takes equal time on each alone.  If the mixed
// kernel takes ~max(a, b) the pipes are separate; if ~a + b they are one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define DMMA(c0, c1, a, b)                                                                   \
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" \
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b))

template <int NF, int NM>   // per inner step: NF x 8 DFMA, NM x 4 DMMA
__global__ void __launch_bounds__(256) k_mix(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-3, x2 = x0 + 2e-3, x3 = x0 + 3e-3;
    double x4 = x0 + 4e-3, x5 = x0 + 5e-3, x6 = x0 + 6e-3, x7 = x0 + 7e-3;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, c6 = 0, c7 = 0;
    const double ma = 1e-3 * (threadIdx.x & 7), mb = 1e-3;
    for (int k = 0; k < iters; ++k) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            }
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                DMMA(c0, c1, ma, mb); DMMA(c2, c3, ma, mb); DMMA(c4, c5, ma, mb); DMMA(c6, c7, ma, mb);
            }
        }
    }
    double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7)) + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
    if (s == 1234.5) out[0] = s;
}

template <int NF, int NM>
double run(double* out, int blocks, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_mix<NF, NM><<<blocks, 256>>>(out, 16, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_mix<NF, NM><<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    const int blocks = sms * 8, iters = 2048;
    const double warps = (double)blocks * 8;
    // per inner step (x4 per iteration): NF*8 DFMA warp-instructions (64 FLOP/lane-less: 2*32 each),
    // NM*4 DMMA (512 FLOP each)
    auto tf = [&](double ms, int nf, int nm) {
        return (nf * 8 * 64.0 + nm * 4 * 512.0) * 4 * iters * warps / (ms * 1e-3) / 1e12;
    };
    double a = run<2, 0>(out, blocks, iters);
    double b = run<0, 1>(out, blocks, iters);
    double b2 = run<0, 2>(out, blocks, iters);
    double m = run<2, 1>(out, blocks, iters);
    double m2 = run<2, 2>(out, blocks, iters);
    printf("DFMA only  (16 DFMA/step):          %.3f ms  %.2f TFLOP/s\n", a, tf(a, 2, 0));
    printf("DMMA only  (4 DMMA/step):           %.3f ms  %.2f TFLOP/s\n", b, tf(b, 0, 1));
    printf("DMMA only  (8 DMMA/step):           %.3f ms  %.2f TFLOP/s\n", b2, tf(b2, 0, 2));
    printf("mixed      (16 DFMA + 4 DMMA/step): %.3f ms  %.2f TFLOP/s   sum of parts %.3f ms, max %.3f ms\n",
           m, tf(m, 2, 1), a + b, a > b ? a : b);
    printf("mixed      (16 DFMA + 8 DMMA/step): %.3f ms  %.2f TFLOP/s   sum of parts %.3f ms, max %.3f ms\n",
           m2, tf(m2, 2, 2), a + b2, a > b2 ? a : b2);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
