// Arithmetic-pipe peak microbenchmarks (the roofline denominators the driver's
// MEASURED_PEAKS.json does not carry): non-FMA FP64 DADD/DMUL issue rate — the
// ops the exact predicate executes — and FP32 FFMA throughput.
#include <cuda_runtime.h>

#include "../../include/visrt.h"

namespace {

__global__ void k_fp64_peak(double* out, int iters, double m, double c) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
        a0 = __dadd_rn(__dmul_rn(a0, m), c);
        a1 = __dadd_rn(__dmul_rn(a1, m), c);
        a2 = __dadd_rn(__dmul_rn(a2, m), c);
        a3 = __dadd_rn(__dmul_rn(a3, m), c);
        a4 = __dadd_rn(__dmul_rn(a4, m), c);
        a5 = __dadd_rn(__dmul_rn(a5, m), c);
        a6 = __dadd_rn(__dmul_rn(a6, m), c);
        a7 = __dadd_rn(__dmul_rn(a7, m), c);
    }
    const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == 123.456) out[0] = r;
}

__global__ void k_fp32_peak(float* out, int iters, float m, float c) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __fmaf_rn(a[k], m, c);
    }
    float r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r += a[k];
    if (r == 123.456f) out[0] = r;
}

}  // namespace

extern "C" int visrt_measure_peaks(int device, double* fp64_ops, double* fp32_flops) {
    if (cudaSetDevice(device) != cudaSuccess) return VISRT_E_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    void* buf = nullptr;
    if (cudaMalloc(&buf, 64) != cudaSuccess) return VISRT_E_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    float best64 = 1e30f, best32 = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        float ms = 0;
        cudaEventRecord(e0);
        k_fp64_peak<<<blocks, threads>>>(static_cast<double*>(buf), iters, 0.999999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best64) best64 = ms;
        cudaEventRecord(e0);
        k_fp32_peak<<<blocks, threads>>>(static_cast<float*>(buf), iters * 4, 0.999999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best32) best32 = ms;
    }
    const double n = static_cast<double>(blocks) * threads;
    if (fp64_ops) *fp64_ops = n * iters * 16.0 / (best64 * 1e-3);
    if (fp32_flops) *fp32_flops = n * (iters * 4.0) * 16.0 / (best32 * 1e-3);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    return cudaGetLastError() == cudaSuccess ? VISRT_OK : VISRT_E_CUDA;
}
