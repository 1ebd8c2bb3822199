// K5: roofline probes (include/mfa_probe.h).
#include <cuda_runtime.h>

#include "../../include/mfa_probe.h"
#include "mfa_internal.cuh"

namespace mfa {

constexpr int kChains = 8;

template <int MODE>
__global__ void __launch_bounds__(256) fp32_probe_kernel(float* out, int iters, float b, float c) {
    float a[kChains];
    float2 a2[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
        a[i] = threadIdx.x * 1e-7f + i;
        a2[i] = make_float2(a[i], a[i] + 0.5f);
    }
    const float2 b2 = make_float2(b, b * 0.5f), c2 = make_float2(c, c * 0.5f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < kChains; ++i) {
                if constexpr (MODE == 0) a[i] = fmaf(a[i], b, c);
                else if constexpr (MODE == 1) a2[i] = __ffma2_rn(a2[i], b2, c2);
                else a[i] = fmaf(a[i], 0.999f, 1e-3f);
            }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += a[i] + a2[i].x + a2[i].y;
    if (s == 1.2345f) out[blockIdx.x] = s;   // keeps the chains live
}

__global__ void __launch_bounds__(256) read_probe_kernel(const int4* __restrict__ buf, int64_t n16, int reps,
                                                         int* out) {
    int acc = 0;
    for (int r = 0; r < reps; ++r)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
            const int4 v = __ldcg(buf + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678) out[0] = acc;
}

}  // namespace mfa

using namespace mfa;

extern "C" mfa_status mfa_probe_fp32(int32_t mode, double* tflops) {
    if (!tflops || mode < 0 || mode > 2) return fail(MFA_ERR_INVALID_ARG, "mode / tflops");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out = nullptr;
    cudaError_t e = cudaMalloc(&out, 65536 * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "probe alloc");
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&]() {
        if (mode == 0) fp32_probe_kernel<0><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        else if (mode == 1) fp32_probe_kernel<1><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        else fp32_probe_kernel<2><<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    };
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (e != cudaSuccess) return cuda_fail(e, "fp32 probe");
    const double fma_per_thread = (double)iters * 16 * kChains * (mode == 1 ? 2 : 1);
    const double flops = 5.0 * blocks * threads * fma_per_thread * 2.0;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return MFA_OK;
}

extern "C" mfa_status mfa_probe_read_bw(int64_t bytes, int32_t reps, double* gbps) {
    if (!gbps || bytes < 4096 || (bytes & 4095) || reps < 1) return fail(MFA_ERR_INVALID_ARG, "bytes / reps");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int4* buf = nullptr;
    int* out = nullptr;
    cudaError_t e = cudaMalloc(&buf, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "probe alloc");
    cudaMalloc(&out, sizeof(int));
    cudaMemset(buf, 1, bytes);
    const int64_t n16 = bytes / 16;
    const int blocks = sms * 8;
    read_probe_kernel<<<blocks, 256>>>(buf, n16, 1, out);   // warm (L2-resident if it fits)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    read_probe_kernel<<<blocks, 256>>>(buf, n16, reps, out);
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(out);
    if (e != cudaSuccess) return cuda_fail(e, "read probe");
    *gbps = (double)bytes * reps / (ms * 1e-3) / 1e9;
    return MFA_OK;
}
