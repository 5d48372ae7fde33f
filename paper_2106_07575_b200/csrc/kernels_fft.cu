// Batched unitary 2-D FFT kernel behind ptyger_fft2 (cross-check target of the FFT library).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "dev.cuh"

namespace pty {

// ----------------------------------------------------------------------------------------
// Batched 2-D FFT (API helper ptyger_fft2; also the unit-test target of the FFT library)
// ----------------------------------------------------------------------------------------
template <int N, bool INV>
__global__ void __launch_bounds__(512, 1) k_fft2(const float2* __restrict__ in, float2* __restrict__ out,
                                                 int64_t batch) {
    using C = FFTCfg<N>;
    constexpr int R = C::R, T = C::T, LD = C::LD;
    extern __shared__ float2 smem[];
    float2* sf = smem;
    float2* tw = smem + C::FPB * C::FRAME_ELEMS;
    build_twiddles<N>(tw);
    __syncthreads();
    const int64_t ngroups = (batch + C::FPB - 1) / C::FPB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float scale = 1.0f / (float)N;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int line = rd * C::LPR + tid / T, t = tid % T;
            const int f = line / N, row = line % N;
            const int64_t j = grp * C::FPB + f;
            float2 x[R];
            if (j < batch) {
                const float2* src = in + j * N * N + (int64_t)row * N + t;
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = ldg2(src + T * n1);
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = make_float2(0.f, 0.f);
            }
            row_fft<N, INV>(x, sf + f * C::FRAME_ELEMS + row * LD, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            const int f = line / N, c = line % N;
            col_fft_phase1<N, INV>(sf + f * C::FRAME_ELEMS + c, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            const int f = line / N, c = line % N;
            const int64_t j = grp * C::FPB + f;
            float2 X[R];
            col_fft_phase2<N, INV>(sf + f * C::FRAME_ELEMS + c, t, X);
            if (j < batch) {
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    const int k = col_out_row<N>(i, t);
                    out[j * N * N + (int64_t)k * N + c] = cscale(X[i], scale);
                }
            }
        }
        __syncthreads();
    }
}


// ----------------------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------------------
template <typename F>
static int set_smem(F* f, size_t bytes) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess ? 0 : -1;
}

template <int N, bool INV>
static int fft2_n(const float2* in, float2* out, int64_t batch, cudaStream_t s) {
    using C = FFTCfg<N>;
    if (set_smem(k_fft2<N, INV>, C::SMEM_BYTES)) return -1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ng = (batch + C::FPB - 1) / C::FPB;
    const int grid = (int)(ng < sms ? ng : sms);
    if (grid <= 0) return 0;
    k_fft2<N, INV><<<grid, C::NT, C::SMEM_BYTES, s>>>(in, out, batch);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_fft2(const float2* in, float2* out, int N, int64_t batch, bool inv, cudaStream_t s) {
    switch (N) {
        case 16: return inv ? fft2_n<16, true>(in, out, batch, s) : fft2_n<16, false>(in, out, batch, s);
        case 32: return inv ? fft2_n<32, true>(in, out, batch, s) : fft2_n<32, false>(in, out, batch, s);
        case 64: return inv ? fft2_n<64, true>(in, out, batch, s) : fft2_n<64, false>(in, out, batch, s);
        case 128: return inv ? fft2_n<128, true>(in, out, batch, s) : fft2_n<128, false>(in, out, batch, s);
        case 256: return launch_fft2_256(in, out, batch, inv, s);
    }
    return -2;
}

}  // namespace pty
