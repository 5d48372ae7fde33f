// FP32 pipe peak microbenchmark (the lower bound t_min needs the MEASURED FP32 peak of
// the box, not the nominal 148 SMs x 128 lanes x 2 flop x clock).  Each thread runs 8 independent
// fused-multiply-add chains (paired FFMA2 = fma.rn.f32x2, or scalar FFMA) for `iters` rounds, so the
// FMA pipes never wait on a dependency; flops = 2 per FMA lane-op.  The result sinks into a store
// that the compiler cannot prove dead.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev.cuh"

namespace pty {

template <bool PAIRED>
__global__ void __launch_bounds__(512) k_fp32_peak(float* __restrict__ sink, int iters, float a, float b) {
    if constexpr (PAIRED) {
        float2 x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-6f + i, i * 0.5f);
        const float2 av = make_float2(a, a), bv = make_float2(b, b);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int r = 0; r < 16; ++r) {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = fma2(x[i], av, bv);
            }
        }
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
        if (s == 1234.5f) sink[threadIdx.x] = s;
    } else {
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-6f + i;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int r = 0; r < 16; ++r) {
#pragma unroll
                for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
            }
        }
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += x[i];
        if (s == 1234.5f) sink[threadIdx.x] = s;
    }
}

// returns TFLOP/s (best of 3 timed launches) or a negative value on failure
double measure_fp32_peak(int device, bool paired) {
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* sink = nullptr;
    if (cudaMalloc(&sink, 512 * sizeof(float)) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 512, iters = 2048;
    auto launch = [&]() {
        if (paired)
            k_fp32_peak<true><<<blocks, threads>>>(sink, iters, 0.999f, 1e-3f);
        else
            k_fp32_peak<false><<<blocks, threads>>>(sink, iters, 0.999f, 1e-3f);
    };
    launch();   // warm-up (clocks up, module loaded)
    double best = 0.0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        // FMA lane-ops: blocks x threads x iters x 16 rounds x 8 chains (x 2 lanes when paired)
        const double fmas = (double)blocks * threads * iters * 16.0 * 8.0 * (paired ? 2.0 : 1.0);
        const double tf = 2.0 * fmas / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    const bool ok = cudaGetLastError() == cudaSuccess;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    return ok ? best : -1.0;
}

}  // namespace pty
