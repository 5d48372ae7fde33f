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
#include <stdlib.h>

#include "dev.cuh"
#include "tma.cuh"

namespace pty {

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
                window_row<R, T>(psi, g, pos[j], j, row, t, probe + row * N + t, x);
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
                    if (d) {  // d == nullptr: transform only (v = G eta for the split line search)
                        const float cc = uu.x * uu.x + uu.y * uu.y;
                        fs += objective_term(cc, __ldg(d + o), eps2, g.est);
                    }
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
                                                 const float* __restrict__ d, const float2* __restrict__ probe_s,
                                                 const DevState* __restrict__ st, float eps) {
    using C = FFTCfg<N>;
    constexpr int R = C::R, T = C::T, LD = C::LD;
    extern __shared__ float2 smem[];
    float2* sf = smem;
    float4* tw = reinterpret_cast<float4*>(smem + C::FPB * C::FRAME_ELEMS);
    if (st->numeric_error) return;
    ktime_start(st, 0);
    build_twiddles4<N, true>(tw);
    __syncthreads();
    const float gam = (float)st->gamma;
    const bool upd = gam != 0.0f;
    const int64_t nfr = g.n_local;
    const int64_t ngroups = (nfr + C::FPB - 1) / C::FPB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float eps2 = eps * eps;
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
                for (int n1 = 0; n1 < R; ++n1) x[n1] = residual(uu[n1], dd[n1], eps2, g.est);
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = make_float2(0.f, 0.f);
            }
            row_fft<N, true, true>(x, sf + f * C::FRAME_ELEMS + row * LD, t, tw, tw + N);
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
                    const float2 pk = ldg2(probe_s + k * N + c);   // conj(p / N): unitary scale folded in
                    v[j * N * N + (int64_t)k * N + c] = cconjmul(pk, X[q]);
                }
            }
        }
        __syncthreads();
    }
    __syncthreads();
    ktime_end(st, 0);
}


// ----------------------------------------------------------------------------------------
// k_ls: LS stage first pass (Alg.1 659-668 with Eq.7): v_j = F(p * eta[window s_j]) written
// to HBM, then the SCREENING terms (dev.cuh ls_push / ls_screen_nz) of the pass-0 trials gamma_k,
// k < keff (adaptive, read from the device state) against (u, d); per-CTA fp64 partials
// [S_0..S_{KC-1} | A, D, sum|a|, sum b].
// ----------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(512, 1) k_ls(Geometry g, const float2* __restrict__ eta,
                                               const float2* __restrict__ probe_s, const int2* __restrict__ pos,
                                               const int* __restrict__ order, const float2* __restrict__ u,
                                               float2* __restrict__ v, const float* __restrict__ d,
                                               SolverCfg cfg, double* __restrict__ part,
                                               const DevState* __restrict__ st, int pf) {
    using C = FFTCfg<N>;
    constexpr int R = C::R, T = C::T, LD = C::LD;
    extern __shared__ float2 smem[];
    float2* sf = smem;
    float4* tw = reinterpret_cast<float4*>(smem + C::FPB * C::FRAME_ELEMS);
    __shared__ double sred[16][KC];
    __shared__ double smom[16][4];
    __shared__ float sgam[KC];
    __shared__ LsWarpQ<2> wq[16];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool err = st->numeric_error != 0;
    int base, cnt;
    ls_pass_range(0, st->keff, cfg, base, cnt);
    ktime_start(st, 1);
    build_twiddles4<N, false>(tw);
    if (tid < KC) sgam[tid] = (float)trial_gamma(cfg.gamma0, cfg.tau, base + tid);
    __syncthreads();
    const int64_t nfr = err ? 0 : g.n_local;
    const int64_t ngroups = (nfr + C::FPB - 1) / C::FPB;
    const float eps2 = (float)(cfg.eps * cfg.eps);
    double tot = 0.0;  // running total of entry lane >> 1 of S
    double mom[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        if constexpr (C::FPB == 1) {
            // this frame's u, d into L2 now: the epilogue reads them after both transforms
            if (pf && grp < nfr) {
                const int64_t jp = order[grp];
                if (tid < 32) prefetch_l2_frame(u + jp * N * N, N * N * 8, tid);
                else if (tid < 64) prefetch_l2_frame(d + jp * N * N, N * N * 4, tid - 32);
            }
        }
        // row pass input of round rd: x[n1] = (p / N)[row, T n1 + t] * eta[s + (row, T n1 + t)]
        // (p / N: the unitary scale folded into the probe)
        auto load_row = [&](int rd, float2 (&x)[R]) {
            const int line = rd * C::LPR + tid / T, t = tid % T;
            const int f = line / N, row = line % N;
            const int64_t i = grp * C::FPB + f;
            if (i < nfr) {
                const int j = order[i];
                window_row<R, T>(eta, g, pos[j], j, row, t, probe_s + row * N + t, x);
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) x[n1] = make_float2(0.f, 0.f);
            }
        };
        auto fft_row = [&](int rd, float2 (&x)[R]) {
            const int line = rd * C::LPR + tid / T, t = tid % T;
            row_fft<N, false, true>(x, sf + (line / N) * C::FRAME_ELEMS + (line % N) * LD, t, tw, tw + N);
        };
        if constexpr (C::ROUNDS == 2) {
            // both rounds' gathers in flight before the first transform (hides the L2 latency of
            // the eta window once per frame instead of twice)
            float2 xa[R], xb[R];
            load_row(0, xa);
            load_row(1, xb);
            fft_row(0, xa);
            fft_row(1, xb);
        } else {
#pragma unroll 1
            for (int rd = 0; rd < C::ROUNDS; ++rd) {
                float2 x[R];
                load_row(rd, x);
                fft_row(rd, x);
            }
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
            float2* scol = sf + f * C::FRAME_ELEMS + c;
            {
                // phase 2 with the outputs parked in the thread's own input rows (T k1 + k2,
                // thread-private: no barrier), so the LS epilogue below can run as a ROLLED loop
                // (a fully unrolled 16-element x KC-trial epilogue overflows the instruction cache)
                float2 X[R];
                col_fft_phase2<N, false>(scol, t, X);
#pragma unroll
                for (int q = 0; q < R; ++q) scol[(T * ((q / T) * T + t) + q % T) * LD] = X[q];
            }
            float S[KC];
            LsMom m;
#pragma unroll
            for (int k = 0; k < KC; ++k) S[k] = 0.f;
            // all lanes run the epilogue (lanes of a frame past the end push zeros) because the
            // d > 0 compaction ring is warp-collective
            const bool valid = i < nfr;
            const int64_t j = valid ? order[i] : 0;
            // this thread's column c of frame j at row t: element q of its column sits at row
            // (q / T) T + t + R (q % T); 32-bit in-frame offsets off a 64-bit frame base
            const int64_t fb = j * (int64_t)(N * N) + (int64_t)t * N + c;
            const float2* __restrict__ ub = u + fb;
            const float* __restrict__ db = d + fb;
            float2* __restrict__ vb = v + fb;
            if (cnt > 0) trial_dispatch(cnt, cfg, [&]<int KT, bool LSE, bool QG>() {
                float gk[KT];   // trial gammas in registers for the whole run
#pragma unroll
                for (int k = 0; k < KT; ++k) gk[k] = sgam[k];
                LsQState qs;
                if constexpr (T >= 4) {
                    // groups of 4 consecutive elements q = 4 gi + e share j = q / T, so inside a
                    // group the global offsets step by R N and the parked rows by one (immediates)
                    float2 un[4];
                    float dn[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        un[e] = valid ? ldg2_na(ub + e * R * N) : make_float2(0.f, 0.f);
                        dn[e] = valid ? ldg1_na(db + e * R * N) : 0.f;
                    }
#pragma unroll 1
                    for (int gi = 0; gi < R / 4; ++gi) {
                        const int q0 = 4 * gi;
                        const int go = ((q0 / T) * T + R * (q0 % T)) * N;
                        const float2* sp = scol + (T * ((q0 / T) * T + t) + q0 % T) * LD;
                        float2 uc[4];
                        float dc[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            uc[e] = un[e];
                            dc[e] = dn[e];
                        }
                        if (gi + 1 < R / 4 && valid) {  // prefetch the next group's u, d
                            const int q1 = q0 + 4;
                            const int gn = ((q1 / T) * T + R * (q1 % T)) * N;
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                un[e] = ldg2_na(ub + gn + e * R * N);
                                dn[e] = ldg1_na(db + gn + e * R * N);
                            }
                        }
                        float2 vc[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            vc[e] = sp[e * LD];
                            if (valid) vb[go + e * R * N] = vc[e];
                            else vc[e] = make_float2(0.f, 0.f);
                        }
                        ls_push<KT, LSE, QG>(wq[warp], qs, slice<0, 2>(uc), slice<0, 2>(vc), slice<0, 2>(dc), gk, eps2,
                                         S, m, lane);
                        ls_push<KT, LSE, QG>(wq[warp], qs, slice<2, 2>(uc), slice<2, 2>(vc), slice<2, 2>(dc), gk, eps2,
                                         S, m, lane);
                    }
                } else {
                    auto off = [&](int q) -> int { return ((q / T) * T + R * (q % T)) * N; };
#pragma unroll 1
                    for (int q = 0; q < R; ++q) {
                        float2 vv[1] = {scol[(T * ((q / T) * T + t) + q % T) * LD]};
                        float2 uu[1] = {make_float2(0.f, 0.f)};
                        float dd[1] = {0.f};
                        if (valid) {
                            uu[0] = ub[off(q)];
                            dd[0] = __ldg(db + off(q));
                            vb[off(q)] = vv[0];
                        } else {
                            vv[0] = make_float2(0.f, 0.f);
                        }
                        ls_push<KT, LSE, QG>(wq[warp], qs, uu, vv, dd, gk, eps2, S, m, lane);
                    }
                }
                ls_flush<KT, LSE, QG>(wq[warp], qs, gk, eps2, S, m, lane);
            });
            ls_run_out<KC>(S, m, tot, mom, lane);
        }
        __syncthreads();
    }
    ktime_end(st, 1);
    ls_block_out<KC, 16>(tot, mom, sred, smom, part);
}


// ----------------------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------------------
template <typename F>
static int set_smem(F* f, size_t bytes) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess ? 0 : -1;
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
        case 256: return launch_fwd256(g, psi, probe, pos, order, d, u, part, grid, eps, s);
    }
    return -2;
}

template <int N>
static int grad_n(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe,
                  const DevState* st, float eps, int grid, cudaStream_t s) {
    using C = FFTCfg<N>;
    if (set_smem(k_grad<N>, C::SMEM_BYTES4)) return -1;
    k_grad<N><<<grid, C::NT, C::SMEM_BYTES4, s>>>(g, u, v, d, probe, st, eps);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_grad(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe,
                const float2* probe_s, const DevState* st, float eps, int grid, cudaStream_t s) {
    switch (g.N) {
        case 16: return grad_n<16>(g, u, v, d, probe_s, st, eps, grid, s);
        case 32: return grad_n<32>(g, u, v, d, probe_s, st, eps, grid, s);
        case 64: return grad_n<64>(g, u, v, d, probe_s, st, eps, grid, s);
        case 128:
            // direct-load k_grad<128> (2.57 ms, 88 % of HBM at paper scale); a TMA-ring variant
            // (cp.async.bulk rows into a 2 x 43 KB ring) measured 3.13 ms and was removed
            return grad_n<128>(g, u, v, d, probe_s, st, eps, grid, s);
        case 256: return launch_grad256(g, u, v, d, probe, st, eps, grid, s);
    }
    return -2;
}

template <int N>
static int ls_n(const Geometry& g, const float2* eta, const float2* probe, const int2* pos,
                const int* order, const float2* u, float2* v, const float* d, const SolverCfg& c,
                double* part, int grid, const DevState* st, cudaStream_t s) {
    using C = FFTCfg<N>;
    if (set_smem(k_ls<N>, C::SMEM_BYTES4)) return -1;
    // L2 prefetch of each frame's u, d at its start (measured: k_ls 3.29 -> 3.23 ms at paper scale)
    static const int pf = getenv("PTYGER_PF") ? atoi(getenv("PTYGER_PF")) : 1;
    k_ls<N><<<grid, C::NT, C::SMEM_BYTES4, s>>>(g, eta, probe, pos, order, u, v, d, c, part, st, pf != 0);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_ls(const Geometry& g, const float2* eta, const float2* probe, const float2* probe_s, const int2* pos,
              const int* order, const float2* u, float2* v, const float* d, const SolverCfg& c,
              double* part, int grid, const DevState* st, cudaStream_t s) {
    switch (g.N) {
        case 16: return ls_n<16>(g, eta, probe_s, pos, order, u, v, d, c, part, grid, st, s);
        case 32: return ls_n<32>(g, eta, probe_s, pos, order, u, v, d, c, part, grid, st, s);
        case 64: return ls_n<64>(g, eta, probe_s, pos, order, u, v, d, c, part, grid, st, s);
        case 128: {
            static const bool ws = !(getenv("PTYGER_LS_WS") && atoi(getenv("PTYGER_LS_WS")) == 0);
            if (ws) return launch_ls_ws(g, eta, probe_s, pos, order, u, v, d, c, part, grid, st, s);
            return ls_n<128>(g, eta, probe_s, pos, order, u, v, d, c, part, grid, st, s);
        }
        case 256: return launch_ls_c256(g, eta, probe_s, pos, order, u, v, d, c, part, st, s);
    }
    return -2;
}

}  // namespace pty
