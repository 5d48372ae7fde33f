// sm_100a kernels of one ML-CG iteration (PAPER.md:462-471 four stages GRAD / DIR / LS /
// Update; Alg.1).  Design S: the far fields u = G psi and
// v = G eta stay resident in HBM and the line search uses linearity, G(psi + g eta) = u + g v.
//
//   k_fwd   u = G psi, F(psi) partials                      (init / set_state; Eq.1, Eq.2)
//   k_grad  u <- u + gamma_prev v; r = u - d u/|u|^2; y = conj(p) F^H r  (Eq.3 minus the scatter)
//   k_adj   g = sum_j scatter(y_j): tile-major, atomic-free, canonical frame order (Q^H of Eq.3)
//           + DY partials |g|^2, <eta, g - g_prev>                (Eq.6 / Eq.8 inner products)
//   k_dir   alpha (DY complex / real / FR, restart rules)          (Eq.6, Eq.8; R#6, R#9)
//   k_eta   eta = -g + alpha eta, ||eta||^2                        (Eq.6)
//   k_ls    v = F(p eta[window]) and K trial partials DeltaF_k     (Eq.7 with the Eq.2 objective)
//   k_lsx   further K-trial passes over (u, v, d) when no trial of the first pass was accepted
//   k_pick  first accepted trial, F update, trace                  (Eq.7, Alg.1 659-668)
//   k_upd   psi <- psi + gamma eta                                  (Eq.5, Alg.1 672)
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "fft.cuh"
#include "internal.h"

namespace pty {

#define FULLMASK 0xffffffffu

// ----------------------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(FULLMASK, v, m);
    return v;
}

// Block sum in fixed order (deterministic).  All threads must call; result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sred) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sred[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NT / 32; ++i) s += sred[i];
    }
    return s;
}

// Warp reduce-scatter of K (power of two <= 32) per-lane values: afterwards every lane holds
// the warp total of trial  lane >> (5 - log2 K).
template <int K>
__device__ __forceinline__ double warp_reduce_scatter(double (&v)[K], int lane) {
    constexpr int P = (K == 1) ? 0 : (K == 2) ? 1 : (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
#pragma unroll
    for (int s = 0; s < P; ++s) {
        const int h = K >> (s + 1);
        const int m = 16 >> s;
        const bool upper = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = upper ? v[i] : v[i + h];
            const double keep = upper ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(FULLMASK, send, m);
        }
    }
    double r = v[0];
#pragma unroll
    for (int m = (32 >> P) >> 1; m >= 1; m >>= 1) r += __shfl_xor_sync(FULLMASK, r, m);
    return r;
}

// Accurate, branch-free float log1p for z > -1 (max rel err 1.4e-7 measured in fp32 over the
// reduced range): w = 1 + z = m 2^e with m in [sqrt(1/2), sqrt(2)); when e = 0 the polynomial is
// evaluated on z itself (no rounding of 1 + z is ever used), otherwise on m - 1 (the rounding
// of 1 + z is then below 2e-7 of the result).  log1p(x) = x + x^2 P(x), P a degree-8 Chebyshev
// fit on [sqrt(1/2)-1, sqrt(2)-1] (fp64 fit, coefficients rounded to fp32).  No MUFU, no branch.
__device__ __forceinline__ float log1p_poly(float z) {
    const float w = 1.0f + z;
    const int iw = __float_as_int(w);
    const int e = (iw - 0x3f3504f3) >> 23;
    const float m = __int_as_float(iw - (e << 23));
    const float x = (e == 0) ? z : (m - 1.0f);
    float P = -0.07764425f;
    P = fmaf(P, x, 0.12656558f);
    P = fmaf(P, x, -0.13065042f);
    P = fmaf(P, x, 0.14209557f);
    P = fmaf(P, x, -0.1663307f);
    P = fmaf(P, x, 0.20001242f);
    P = fmaf(P, x, -0.25000605f);
    P = fmaf(P, x, 0.33333328f);
    P = fmaf(P, x, -0.49999997f);
    const float ef = __int_as_float(e + 0x4B400000) - 12582912.0f;   // (float)e on the FMA pipe
    return fmaf(ef, 0.693147182464599609375f, fmaf(x * x, P, x));
}

// Guarded definition of the per-pixel LS term (R#4): used only when |u| < eps or
// |u + gamma v| < eps or 1 + z underflows (warp-uniform slow path).
__device__ __noinline__ float ls_term_slow(float a, float b, float c, float dd, float gam, float eps2) {
    const float q = gam * fmaf(gam, b, a);
    const float cn = c + q;
    if (c >= eps2 && cn >= eps2) {
        const float z = q / c;
        if (z > -0.999f) return fmaf(-dd, log1p_poly(z), q);
    }
    return (cn - c) - dd * (logf(fmaxf(cn, eps2)) - logf(fmaxf(c, eps2)));
}

// Per-pixel difference-form LS terms for K trials (oracle ls_delta):  t_k = q_k - d log1p(q_k/c),
// q_k = gamma_k (a + gamma_k b), a = 2 Re(u* v), b = |v|^2, c = |u|^2.  Branch-free fast path;
// any lane needing the guarded definition sends its warp through ls_term_slow.
template <int K>
__device__ __forceinline__ void ls_terms(float2 uu, float2 vv, float dd, const float* sgam, float eps2,
                                         float (&acc)[K]) {
    const float a = 2.0f * fmaf(uu.x, vv.x, uu.y * vv.y);
    const float b = fmaf(vv.x, vv.x, vv.y * vv.y);
    const float c = fmaf(uu.x, uu.x, uu.y * uu.y);
    bool bad = !(c >= eps2);
    const float rc = bad ? 0.0f : 1.0f / c;
    float t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const float gam = sgam[k];
        const float q = gam * fmaf(gam, b, a);
        const float z = q * rc;
        bad |= (c + q < eps2) | (z <= -0.999f);
        t[k] = fmaf(-dd, log1p_poly(fmaxf(z, -0.5f)), q);
    }
    if (__any_sync(__activemask(), bad)) {
        if (bad) {
#pragma unroll 1
            for (int k = 0; k < K; ++k) t[k] = ls_term_slow(a, b, c, dd, sgam[k], eps2);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] += t[k];
}

__device__ __forceinline__ float2 ldg2(const float2* p) { return __ldg(p); }

// Residual of Eq.3: u - d/u^* = u - d u / |u|^2, quotient dropped where |u| < eps (R#4).
__device__ __forceinline__ float2 residual(float2 u, float dd, float eps2) {
    const float c = u.x * u.x + u.y * u.y;
    if (c >= eps2) {
        const float s = dd / c;
        return make_float2(u.x - s * u.x, u.y - s * u.y);
    }
    return u;
}

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
// k_fwd: u_j = F(p * psi[window s_j]) (Eq.1) and F partial sum (Eq.2) per CTA.
// ----------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(512, 1) k_fwd(Geometry g, const float2* __restrict__ psi,
                                                const float2* __restrict__ probe,
                                                const int2* __restrict__ pos, const int* __restrict__ order,
                                                const float* __restrict__ d, float2* __restrict__ u,
                                                double* __restrict__ part, float eps) {
    using C = FFTCfg<N>;
    constexpr int R = C::R, T = C::T, LD = C::LD;
    extern __shared__ float2 smem[];
    float2* sf = smem;
    float2* tw = smem + C::FPB * C::FRAME_ELEMS;
    __shared__ double sred[16];
    build_twiddles<N>(tw);
    __syncthreads();
    const int64_t nfr = g.n_local;
    const int64_t ngroups = (nfr + C::FPB - 1) / C::FPB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float scale = 1.0f / (float)N, eps2 = eps * eps;
    double facc = 0.0;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int line = rd * C::LPR + tid / T, t = tid % T;
            const int f = line / N, row = line % N;
            const int64_t i = grp * C::FPB + f;
            float2 x[R];
            if (i < nfr) {
                const int j = order[i];
                const int2 s = pos[j];
                const float2* src = psi + (int64_t)(s.x + row) * g.W + s.y + t;
                const float2* pp = probe + row * N + t;
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = cmul(ldg2(pp + T * n1), ldg2(src + T * n1));
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = make_float2(0.f, 0.f);
            }
            row_fft<N, false>(x, sf + f * C::FRAME_ELEMS + row * LD, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            col_fft_phase1<N, false>(sf + (line / N) * C::FRAME_ELEMS + line % N, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            const int f = line / N, c = line % N;
            const int64_t i = grp * C::FPB + f;
            float2 X[R];
            col_fft_phase2<N, false>(sf + f * C::FRAME_ELEMS + c, t, X);
            if (i < nfr) {
                const int64_t j = order[i];
                float fs = 0.f;
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int k = col_out_row<N>(q, t);
                    const int64_t o = j * N * N + (int64_t)k * N + c;
                    const float2 uu = cscale(X[q], scale);
                    u[o] = uu;
                    const float cc = uu.x * uu.x + uu.y * uu.y;
                    fs += cc - __ldg(d + o) * logf(fmaxf(cc, eps2));
                }
                facc += (double)fs;
            }
        }
        __syncthreads();
    }
    const double s = block_sum<512>(facc, sred);
    if (tid == 0) part[blockIdx.x] = s;
}

// ----------------------------------------------------------------------------------------
// k_grad: GRAD stage frame part (Alg.1 648-649): u <- u + gamma_prev v (lazy Eq.5 on the far
// field), r = u - d/u^*, y = conj(p) F^H r written into v's slot.
// ----------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(512, 1) k_grad(Geometry g, float2* __restrict__ u, float2* __restrict__ v,
                                                 const float* __restrict__ d, const float2* __restrict__ probe,
                                                 const DevState* __restrict__ st, float eps) {
    using C = FFTCfg<N>;
    constexpr int R = C::R, T = C::T, LD = C::LD;
    extern __shared__ float2 smem[];
    float2* sf = smem;
    float2* tw = smem + C::FPB * C::FRAME_ELEMS;
    if (st->numeric_error) return;
    build_twiddles<N>(tw);
    __syncthreads();
    const float gam = (float)st->gamma;
    const bool upd = gam != 0.0f;
    const int64_t nfr = g.n_local;
    const int64_t ngroups = (nfr + C::FPB - 1) / C::FPB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float scale = 1.0f / (float)N, eps2 = eps * eps;
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int line = rd * C::LPR + tid / T, t = tid % T;
            const int f = line / N, row = line % N;
            const int64_t j = grp * C::FPB + f;
            float2 x[R];
            if (j < nfr) {
                const int64_t base = j * N * N + (int64_t)row * N + t;
                float2 uu[R];
                float dd[R];
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) {
                    uu[n1] = u[base + T * n1];
                    dd[n1] = __ldg(d + base + T * n1);
                }
                if (upd) {
                    float2 vv[R];
#pragma unroll
                    for (int n1 = 0; n1 < R; ++n1) vv[n1] = v[base + T * n1];
#pragma unroll
                    for (int n1 = 0; n1 < R; ++n1) {
                        uu[n1] = make_float2(fmaf(gam, vv[n1].x, uu[n1].x), fmaf(gam, vv[n1].y, uu[n1].y));
                        u[base + T * n1] = uu[n1];
                    }
                }
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = residual(uu[n1], dd[n1], eps2);
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = make_float2(0.f, 0.f);
            }
            row_fft<N, true>(x, sf + f * C::FRAME_ELEMS + row * LD, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            col_fft_phase1<N, true>(sf + (line / N) * C::FRAME_ELEMS + line % N, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            const int f = line / N, c = line % N;
            const int64_t j = grp * C::FPB + f;
            float2 X[R];
            col_fft_phase2<N, true>(sf + f * C::FRAME_ELEMS + c, t, X);
            if (j < nfr) {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int k = col_out_row<N>(q, t);
                    const float2 pk = ldg2(probe + k * N + c);
                    v[j * N * N + (int64_t)k * N + c] = cscale(cconjmul(pk, X[q]), scale);
                }
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------------------
// k_adj: g[rho] = sum_j y_j[rho - s_j] over the frames whose window covers rho (Q^H of
// Eq.3), one 32x32 object tile per CTA, frames in canonical order from a CSR list
// (deterministic, no atomics).  Epilogue: DY partial sums over owned, non-band rows.
// ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_adj(Geometry g, const float2* __restrict__ y,
                                             const int4* __restrict__ ent, const int* __restrict__ tile_ptr,
                                             int ntx, float2* __restrict__ gcur,
                                             const float2* __restrict__ gprev, const float2* __restrict__ eta,
                                             double* __restrict__ part, const DevState* __restrict__ st) {
    __shared__ double sred[NDY][8];
    if (st->numeric_error) return;
    const int tile = blockIdx.x;
    const int tx = tile % ntx, ty = tile / ntx;
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    const int64_t col = (int64_t)tx * 32 + lane;
    const int64_t row0 = (int64_t)ty * 32 + wy;
    const int N = g.N;
    const int64_t NN = (int64_t)N * N;
    float2 acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
    const int beg = tile_ptr[tile], end = tile_ptr[tile + 1];
    int e = beg;
    for (; e + 2 <= end; e += 2) {
        float2 val[2][4];
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const int4 en = __ldg(ent + e + f);
            const int dc = (int)(col - en.z);
            const bool okc = (unsigned)dc < (unsigned)N;
            const float2* yb = y + (int64_t)en.x * NN + dc;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int dr = (int)(row0 + 8 * i - en.y);
                val[f][i] = (okc && (unsigned)dr < (unsigned)N) ? ldg2(yb + (int64_t)dr * N) : make_float2(0.f, 0.f);
            }
        }
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = cadd(acc[i], val[f][i]);
    }
    for (; e < end; ++e) {
        const int4 en = __ldg(ent + e);
        const int dc = (int)(col - en.z);
        const bool okc = (unsigned)dc < (unsigned)N;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int dr = (int)(row0 + 8 * i - en.y);
            if (okc && (unsigned)dr < (unsigned)N) acc[i] = cadd(acc[i], ldg2(y + (int64_t)en.x * NN + (int64_t)dr * N + dc));
        }
    }
    float s[NDY];
#pragma unroll
    for (int q = 0; q < NDY; ++q) s[q] = 0.f;
    if (col < g.W) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t r = row0 + 8 * i;
            if (r < g.SH) {
                const int64_t o = r * g.W + col;
                gcur[o] = acc[i];
                const bool own = r >= g.own_lo && r < g.own_hi && !(r >= g.band_lo0 && r < g.band_hi0) &&
                                 !(r >= g.band_lo1 && r < g.band_hi1);
                if (own) {
                    const float2 gp = gprev[o], et = eta[o];
                    const float2 dg = csub(acc[i], gp);
                    s[0] += acc[i].x * acc[i].x + acc[i].y * acc[i].y;
                    const float2 den = cconjmul(et, dg);
                    s[1] += den.x;
                    s[2] += den.y;
                    s[3] += gp.x * gp.x + gp.y * gp.y;
                    const float2 eg = cconjmul(et, acc[i]);
                    s[4] += eg.x;
                    s[5] += eg.y;
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NDY; ++q) {
        const double w = warp_sum((double)s[q]);
        if (lane == 0) sred[q][wy] = w;
    }
    __syncthreads();
    if (threadIdx.x < NDY) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += sred[threadIdx.x][k];
        part[(int64_t)tile * NDY + threadIdx.x] = t;
    }
}

// After the NCCL band exchange: g[band] += neighbour's partial; DY partials on band rows.
__global__ void __launch_bounds__(256) k_band_add(float2* __restrict__ gcur, const float2* __restrict__ recv,
                                                  int64_t row_lo, int64_t rows, int64_t W,
                                                  const float2* __restrict__ gprev, const float2* __restrict__ eta,
                                                  int64_t own_lo, int64_t own_hi, double* __restrict__ part) {
    __shared__ double sred[NDY][8];
    const int64_t total = rows * W;
    float s[NDY];
#pragma unroll
    for (int q = 0; q < NDY; ++q) s[q] = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = row_lo + i / W;
        const int64_t o = row_lo * W + i;
        const float2 gv = cadd(gcur[o], recv[i]);
        gcur[o] = gv;
        if (r >= own_lo && r < own_hi) {
            const float2 gp = gprev[o], et = eta[o];
            s[0] += gv.x * gv.x + gv.y * gv.y;
            const float2 den = cconjmul(et, csub(gv, gp));
            s[1] += den.x;
            s[2] += den.y;
            s[3] += gp.x * gp.x + gp.y * gp.y;
            const float2 eg = cconjmul(et, gv);
            s[4] += eg.x;
            s[5] += eg.y;
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NDY; ++q) {
        const double v = warp_sum((double)s[q]);
        if (lane == 0) sred[q][w] = v;
    }
    __syncthreads();
    if (threadIdx.x < NDY) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += sred[threadIdx.x][k];
        part[(int64_t)blockIdx.x * NDY + threadIdx.x] = t;
    }
}

// ----------------------------------------------------------------------------------------
// Deterministic reduction of per-block partials: dst[w] = sum_b part[b*width + w].
// ----------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_reduce(const double* __restrict__ part, int nblocks, int width,
                                                 double* __restrict__ dst) {
    __shared__ double sred[32];
    for (int w = 0; w < width; ++w) {
        double s = 0.0;
        for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += part[(int64_t)b * width + w];
        s = warp_sum(s);
        const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
        if (lane == 0) sred[wp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sred[i];
            dst[w] = t;
        }
        __syncthreads();
    }
}

__global__ void k_set_F(DevState* st, const double* src) {
    st->F = src[0];
    st->gamma = 0.0;
}

__global__ void k_begin_iter(DevState* st) {
    st->accepted = 0;
    st->kstar = -1;
    st->n_eval = 0;
    st->restarted = 0;
    st->stalled = 0;
    for (int k = 0; k < SMAX; ++k) st->ls_hist[k] = __longlong_as_double(0x7ff8000000000000LL);
}

// DIR stage (Alg.1 651-656): alpha from the reduced DY sums (Eq.8), restart rules (R#9).
__global__ void k_dir(DevState* st, SolverCfg c) {
    if (st->numeric_error) return;
    const double gg = st->dy[0];
    double are = 0.0, aim = 0.0;
    int restarted = 0;
    if (!isfinite(gg)) {
        st->numeric_error = 1;
        st->err_iter = st->m;
        st->gamma = 0.0;
        return;
    }
    if (st->m > 0) {
        double dre, dim;
        if (c.direction == PTYGER_DIR_FR) {
            dre = st->dy[3];
            dim = 0.0;
        } else {
            dre = st->dy[1];
            dim = st->dy[2];
        }
        const double den2 = dre * dre + dim * dim;
        if (sqrt(den2) < 1e-30) {
            restarted = 1;
        } else {
            // alpha = gg / den = gg conj(den) / |den|^2
            are = gg * dre / den2;
            aim = -gg * dim / den2;
            if (c.direction != PTYGER_DIR_DY) aim = 0.0;
            if (!isfinite(are) || !isfinite(aim)) {
                are = aim = 0.0;
                restarted = 1;
            }
        }
    }
    st->alpha_re = are;
    st->alpha_im = aim;
    st->restarted = restarted;
}

// eta = -g + alpha eta (Eq.6) over the storage rows; ||eta||^2 over owned rows.
__global__ void __launch_bounds__(256) k_eta(Geometry g, const float2* __restrict__ gcur, float2* __restrict__ eta,
                                             const DevState* __restrict__ st, double* __restrict__ part) {
    __shared__ double sred[8];
    const float2 al = make_float2((float)st->alpha_re, (float)st->alpha_im);
    const bool err = st->numeric_error != 0;
    const int64_t total = g.SH * g.W;
    const int64_t lo = g.own_lo * g.W, hi = g.own_hi * g.W;
    float s = 0.f;
    if (!err) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
            const float2 gv = gcur[i];
            const float2 ev = eta[i];
            const float2 ne = csub(cmul(al, ev), gv);
            eta[i] = ne;
            if (i >= lo && i < hi) s += ne.x * ne.x + ne.y * ne.y;
        }
    }
    const double t = block_sum<256>((double)s, sred);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// ----------------------------------------------------------------------------------------
// k_ls: LS stage first pass (Alg.1 659-668 with Eq.7): v_j = F(p * eta[window s_j]) written
// to HBM, then for K trials gamma_k = gamma0 tau^k the per-pixel difference-form terms
// against (u, d); per-CTA partial sums (fp64) of DeltaF_k.
// ----------------------------------------------------------------------------------------
template <int N, int K>
__global__ void __launch_bounds__(512, 1) k_ls(Geometry g, const float2* __restrict__ eta,
                                               const float2* __restrict__ probe, const int2* __restrict__ pos,
                                               const int* __restrict__ order, const float2* __restrict__ u,
                                               float2* __restrict__ v, const float* __restrict__ d,
                                               SolverCfg cfg, double* __restrict__ part,
                                               const DevState* __restrict__ st) {
    using C = FFTCfg<N>;
    constexpr int R = C::R, T = C::T, LD = C::LD;
    extern __shared__ float2 smem[];
    float2* sf = smem;
    float2* tw = smem + C::FPB * C::FRAME_ELEMS;
    __shared__ double sred[16][K];
    __shared__ float sgam[K];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool err = st->numeric_error != 0;
    build_twiddles<N>(tw);
    if (tid < K) sgam[tid] = (float)(cfg.gamma0 * pow(cfg.tau, (double)tid));
    __syncthreads();
    const int64_t nfr = err ? 0 : g.n_local;
    const int64_t ngroups = (nfr + C::FPB - 1) / C::FPB;
    const float scale = 1.0f / (float)N;
    const float eps2 = (float)(cfg.eps * cfg.eps);
    double tot = 0.0;  // running total of trial (lane >> (5 - log2 K))
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int line = rd * C::LPR + tid / T, t = tid % T;
            const int f = line / N, row = line % N;
            const int64_t i = grp * C::FPB + f;
            float2 x[R];
            if (i < nfr) {
                const int j = order[i];
                const int2 s = pos[j];
                const float2* src = eta + (int64_t)(s.x + row) * g.W + s.y + t;
                const float2* pp = probe + row * N + t;
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = cmul(ldg2(pp + T * n1), ldg2(src + T * n1));
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = make_float2(0.f, 0.f);
            }
            row_fft<N, false>(x, sf + f * C::FRAME_ELEMS + row * LD, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            col_fft_phase1<N, false>(sf + (line / N) * C::FRAME_ELEMS + line % N, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < C::ROUNDS; ++rd) {
            const int t = warp % T;
            const int line = rd * C::LPR + (warp / T) * 32 + lane;
            const int f = line / N, c = line % N;
            const int64_t i = grp * C::FPB + f;
            float2 X[R];
            col_fft_phase2<N, false>(sf + f * C::FRAME_ELEMS + c, t, X);
            float acc[K];
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = 0.f;
            if (i < nfr) {
                const int64_t j = order[i];
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int k = col_out_row<N>(q, t);
                    const int64_t o = j * N * N + (int64_t)k * N + c;
                    const float2 vv = cscale(X[q], scale);
                    v[o] = vv;
                    ls_terms<K>(u[o], vv, __ldg(d + o), sgam, eps2, acc);
                }
            }
            double dv[K];
#pragma unroll
            for (int k = 0; k < K; ++k) dv[k] = (double)acc[k];
            tot += warp_reduce_scatter<K>(dv, lane);
        }
        __syncthreads();
    }
    // block reduction: lane group leader of trial idx writes per warp, then fixed-order sum
    constexpr int P = (K == 1) ? 0 : (K == 2) ? 1 : (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    constexpr int G = 32 >> P;
    if ((lane & (G - 1)) == 0) sred[warp][lane >> (5 - P)] = tot;
    __syncthreads();
    if (tid < K) {
        double s = 0.0;
        for (int w = 0; w < 16; ++w) s += sred[w][tid];
        part[(int64_t)blockIdx.x * K + tid] = s;
    }
}

// Further LS passes (trials pass*K .. pass*K+K-1) over the cached (u, v, d): skipped on the
// device when an earlier pass already accepted a trial.
template <int K>
__global__ void __launch_bounds__(256) k_lsx(int64_t count, const float2* __restrict__ u,
                                             const float2* __restrict__ v, const float* __restrict__ d,
                                             SolverCfg cfg, int pass, double* __restrict__ part,
                                             const DevState* __restrict__ st) {
    __shared__ double sred[8][K];
    __shared__ float sgam[K];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool skip = st->accepted || st->numeric_error;
    if (tid < K) sgam[tid] = (float)(cfg.gamma0 * pow(cfg.tau, (double)(pass * K + tid)));
    __syncthreads();
    const float eps2 = (float)(cfg.eps * cfg.eps);
    float acc[K];
    double acc64[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { acc[k] = 0.f; acc64[k] = 0.0; }
    if (!skip) {
        int cnt = 0;
        for (int64_t o = (int64_t)blockIdx.x * blockDim.x + tid; o < count; o += (int64_t)gridDim.x * blockDim.x) {
            ls_terms<K>(u[o], v[o], __ldg(d + o), sgam, eps2, acc);
            if (++cnt == 16) {  // bounded fp32 run length, then fp64
#pragma unroll
                for (int k = 0; k < K; ++k) { acc64[k] += (double)acc[k]; acc[k] = 0.f; }
                cnt = 0;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc64[k] += (double)acc[k];
    const double tot = warp_reduce_scatter<K>(acc64, lane);
    constexpr int P = (K == 1) ? 0 : (K == 2) ? 1 : (K == 4) ? 2 : (K == 8) ? 3 : (K == 16) ? 4 : 5;
    constexpr int G = 32 >> P;
    __syncthreads();
    if ((lane & (G - 1)) == 0) sred[warp][lane >> (5 - P)] = tot;
    __syncthreads();
    if (tid < K) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sred[w][tid];
        part[(int64_t)blockIdx.x * K + tid] = s;
    }
}

// Line-search decision (Eq.7): first trial with DeltaF_k <= gamma_k t; F update (R#11);
// stall after max_shrinks trials (R#9); trace on the last pass.
__global__ void k_pick(DevState* st, SolverCfg c, int pass, int last_pass) {
    if (pass == 0) st->eta2 = st->ls_pass[KMAX];
    if (!st->numeric_error && !st->accepted) {
        for (int k = 0; k < c.K; ++k) {
            const int kk = pass * c.K + k;
            if (kk >= c.max_shrinks) break;
            const double dF = st->ls_pass[k];
            st->ls_hist[kk] = dF;
            st->n_eval = kk + 1;
            if (!isfinite(dF)) {
                st->numeric_error = 2;
                st->err_iter = st->m;
                st->gamma = 0.0;
                break;
            }
            const double gk = c.gamma0 * pow(c.tau, (double)kk);
            if (dF <= gk * c.t) {
                st->accepted = 1;
                st->kstar = kk;
                st->gamma = gk;
                st->F += dF;
                break;
            }
        }
    }
    if (!last_pass) return;
    if (st->numeric_error) return;
    if (!st->accepted) {
        st->stalled = 1;
        st->kstar = c.max_shrinks;
        st->gamma = 0.0;
    }
    if (!isfinite(st->F)) {
        st->numeric_error = 3;
        st->err_iter = st->m;
        st->gamma = 0.0;
        return;
    }
    ptyger_trace t;
    t.iter = st->m;
    t.shrinks = st->kstar;
    t.restarted = st->restarted;
    t.stalled = st->stalled;
    t.F = st->F;
    t.gamma = st->gamma;
    t.alpha_re = st->alpha_re;
    t.alpha_im = st->alpha_im;
    t.grad_norm = sqrt(st->dy[0]);
    t.step_norm = st->gamma * sqrt(st->eta2);
    if (st->trace_ptr && st->trace_idx < st->trace_cap) st->trace_ptr[st->trace_idx] = t;
    st->trace_idx += 1;
    st->m += 1;
}

// Update stage (Eq.5, Alg.1 672): psi <- psi + gamma eta over the storage rows.
__global__ void __launch_bounds__(256) k_upd(Geometry g, float2* __restrict__ psi, const float2* __restrict__ eta,
                                             const DevState* __restrict__ st) {
    if (st->numeric_error) return;
    const float gam = (float)st->gamma;
    if (gam == 0.0f) return;
    const int64_t total = g.SH * g.W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const float2 e = eta[i];
        float2 p = psi[i];
        p.x = fmaf(gam, e.x, p.x);
        p.y = fmaf(gam, e.y, p.y);
        psi[i] = p;
    }
}

// d must be finite and >= 0: records the smallest offending frame index.
__global__ void k_validate_d(const float* __restrict__ d, int64_t count, int64_t frame_elems,
                             unsigned long long* bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const float x = d[i];
        if (!(x >= 0.0f) || isinf(x)) atomicMin(bad, (unsigned long long)(i / frame_elems));
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
    }
    return -2;
}

template <int N>
static int fwd_n(const Geometry& g, const float2* psi, const float2* probe, const int2* pos,
                 const int* order, const float* d, float2* u, double* part, int grid, float eps,
                 cudaStream_t s) {
    using C = FFTCfg<N>;
    if (set_smem(k_fwd<N>, C::SMEM_BYTES)) return -1;
    k_fwd<N><<<grid, C::NT, C::SMEM_BYTES, s>>>(g, psi, probe, pos, order, d, u, part, eps);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_fwd(const Geometry& g, const float2* psi, const float2* probe, const int2* pos,
               const int* order, const float* d, float2* u, double* part, int grid, float eps,
               cudaStream_t s) {
    switch (g.N) {
        case 16: return fwd_n<16>(g, psi, probe, pos, order, d, u, part, grid, eps, s);
        case 32: return fwd_n<32>(g, psi, probe, pos, order, d, u, part, grid, eps, s);
        case 64: return fwd_n<64>(g, psi, probe, pos, order, d, u, part, grid, eps, s);
        case 128: return fwd_n<128>(g, psi, probe, pos, order, d, u, part, grid, eps, s);
    }
    return -2;
}

template <int N>
static int grad_n(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe,
                  const DevState* st, float eps, int grid, cudaStream_t s) {
    using C = FFTCfg<N>;
    if (set_smem(k_grad<N>, C::SMEM_BYTES)) return -1;
    k_grad<N><<<grid, C::NT, C::SMEM_BYTES, s>>>(g, u, v, d, probe, st, eps);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_grad(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe,
                const int* /*order*/, const DevState* st, float eps, int grid, cudaStream_t s) {
    switch (g.N) {
        case 16: return grad_n<16>(g, u, v, d, probe, st, eps, grid, s);
        case 32: return grad_n<32>(g, u, v, d, probe, st, eps, grid, s);
        case 64: return grad_n<64>(g, u, v, d, probe, st, eps, grid, s);
        case 128: return grad_n<128>(g, u, v, d, probe, st, eps, grid, s);
    }
    return -2;
}

int launch_adj(const Geometry& g, const float2* y, const int* tile_ptr, const int* tile_frames,
               int ntx, int nty, float2* gcur, const float2* gprev, const float2* eta, double* part,
               const DevState* st, cudaStream_t s) {
    // tile_frames holds int4 entries {frame, row, col, 0}
    k_adj<<<ntx * nty, 256, 0, s>>>(g, y, reinterpret_cast<const int4*>(tile_frames), tile_ptr, ntx, gcur,
                                    gprev, eta, part, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <int N, int K>
static int ls_nk(const Geometry& g, const float2* eta, const float2* probe, const int2* pos,
                 const int* order, const float2* u, float2* v, const float* d, const SolverCfg& c,
                 double* part, int grid, const DevState* st, cudaStream_t s) {
    using C = FFTCfg<N>;
    if (set_smem(k_ls<N, K>, C::SMEM_BYTES)) return -1;
    k_ls<N, K><<<grid, C::NT, C::SMEM_BYTES, s>>>(g, eta, probe, pos, order, u, v, d, c, part, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <int N>
static int ls_n(const Geometry& g, const float2* eta, const float2* probe, const int2* pos,
                const int* order, const float2* u, float2* v, const float* d, const SolverCfg& c,
                double* part, int grid, const DevState* st, cudaStream_t s) {
    switch (c.K) {
        case 8: return ls_nk<N, 8>(g, eta, probe, pos, order, u, v, d, c, part, grid, st, s);
        case 16: return ls_nk<N, 16>(g, eta, probe, pos, order, u, v, d, c, part, grid, st, s);
    }
    return -2;
}

int launch_ls(const Geometry& g, const float2* eta, const float2* probe, const int2* pos,
              const int* order, const float2* u, float2* v, const float* d, const SolverCfg& c,
              double* part, int grid, const DevState* st, cudaStream_t s) {
    switch (g.N) {
        case 16: return ls_n<16>(g, eta, probe, pos, order, u, v, d, c, part, grid, st, s);
        case 32: return ls_n<32>(g, eta, probe, pos, order, u, v, d, c, part, grid, st, s);
        case 64: return ls_n<64>(g, eta, probe, pos, order, u, v, d, c, part, grid, st, s);
        case 128: return ls_n<128>(g, eta, probe, pos, order, u, v, d, c, part, grid, st, s);
    }
    return -2;
}

int launch_lsx(const Geometry& g, const float2* u, const float2* v, const float* d,
               const SolverCfg& c, int pass, double* part, int grid, const DevState* st,
               cudaStream_t s) {
    const int64_t count = g.n_local * (int64_t)g.N * g.N;
    switch (c.K) {
        case 8: k_lsx<8><<<grid, 256, 0, s>>>(count, u, v, d, c, pass, part, st); break;
        case 16: k_lsx<16><<<grid, 256, 0, s>>>(count, u, v, d, c, pass, part, st); break;
        default: return -2;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_reduce(const double* part, int nblocks, int width, double* dst, cudaStream_t s) {
    k_reduce<<<1, 1024, 0, s>>>(part, nblocks, width, dst);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_dir(DevState* st, const SolverCfg& c, cudaStream_t s) {
    k_dir<<<1, 1, 0, s>>>(st, c);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_eta(const Geometry& g, const float2* gcur, float2* eta, const DevState* st, double* part,
               int grid, cudaStream_t s) {
    k_eta<<<grid, 256, 0, s>>>(g, gcur, eta, st, part);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_pick(DevState* st, const SolverCfg& c, int pass, int last_pass, cudaStream_t s) {
    k_pick<<<1, 1, 0, s>>>(st, c, pass, last_pass);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_upd(const Geometry& g, float2* psi, const float2* eta, const DevState* st, int grid,
               cudaStream_t s) {
    k_upd<<<grid, 256, 0, s>>>(g, psi, eta, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_begin_iter(DevState* st, cudaStream_t s) {
    k_begin_iter<<<1, 1, 0, s>>>(st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_validate_d(const float* d, int64_t count, int64_t frame_elems, unsigned long long* bad,
                      cudaStream_t s) {
    k_validate_d<<<1184, 256, 0, s>>>(d, count, frame_elems, bad);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_set_F(DevState* st, const double* src, cudaStream_t s) {
    k_set_F<<<1, 1, 0, s>>>(st, src);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_band_add(float2* gcur, const float2* recv, int64_t row_lo, int64_t rows, int64_t W,
                    const float2* gprev, const float2* eta, int64_t own_lo, int64_t own_hi,
                    double* part, int grid, cudaStream_t s) {
    k_band_add<<<grid, 256, 0, s>>>(gcur, recv, row_lo, rows, W, gprev, eta, own_lo, own_hi, part);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pty
