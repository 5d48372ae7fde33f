// Frame kernels for N = 256 (BASELINE "large" view: 8192^2 object, 256^2 detector).
//
// A 256x256 complex64 frame is 512 KB: it does not fit one SM (228 KB shared memory), so each
// 2-D FFT runs as TWO passes of one CTA over the frame, with the frame's OWN far-field slot in
// HBM (v, which is dead at that point in both kernels) as the transpose buffer:
//   pass 1: 32-row batches; a row is 16 threads x 16 elements (N = 16 x 16: radix-16 in
//           registers, W_256 twiddle, XOR-swizzled exchange, radix-16 across the 16 lanes);
//           results go from registers to the slot's rows (coalesced 128-B segments);
//   pass 2: 32-column batches; lanes = 32 consecutive columns, the 16 sub-threads of a column in
//           16 warps; phase 1 reads the slot (L2-resident: written microseconds earlier by this
//           CTA), phase 2 produces whole columns and runs the epilogue (y = conj(p) X / N for
//           k_grad; v = X/N plus the LS screening terms against u, d for k_ls).
// The intermediate lines are overwritten by the final values while still in L2, so HBM traffic
// stays at the design-S bytes (36 B/px k_grad, 20 B/px k_ls); L2 carries +16 B/px.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev.cuh"

namespace pty {

namespace n256 {
constexpr int N = 256, R = 16, T = 16, LD = N + 8;
constexpr int NT = 512;
constexpr int ROWB = NT / T;      // 32 rows per pass-1 batch
constexpr int COLB = 32;          // 32 columns per pass-2 batch
constexpr int BUF = ROWB * LD;    // complex elements of the batch buffer (>= N * COLB)
static_assert(BUF >= N * COLB, "buffer too small for a column batch");
constexpr size_t SMEM = (size_t)(BUF + N + R * T) * sizeof(float2);   // + twiddle tables (tw, twr [k1][t])
}  // namespace n256

// pass 2 of a 2-D transform: column batch cb (columns cb*32 .. +31) of slot (frame base `src`,
// row-major N x N); returns X[k2] = output row t + 16 k2 of column c (unnormalised).
template <bool INV>
__device__ __forceinline__ void n256_column(const float2* __restrict__ src, int cb, float2* buf, const float2* tw,
                                            float2 (&X)[16], int& c) {
    using namespace n256;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = warp;  // 16 warps = 16 sub-threads of every column
    c = cb * COLB + lane;
    float2 x[R];
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) x[n1] = __ldcg(src + (int64_t)(T * n1 + t) * N + c);
    DFT<R, INV>::run(x);
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) x[k1] = twmul<INV>(x[k1], tw[t * k1]);
    __syncthreads();  // previous batch's readers are done with buf
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) buf[(T * k1 + t) * COLB + lane] = x[k1];
    __syncthreads();
    // phase 2: k1 = t (R / T = 1), inputs rows T*t + n2
#pragma unroll
    for (int n2 = 0; n2 < T; ++n2) X[n2] = buf[(T * t + n2) * COLB + lane];
    DFT<T, INV>::run(X);
}

// ---------------------------------------------------------------------------------------------
// k_grad (N = 256): u <- u + gamma v, r = u - d/u^*, y = conj(p) F^H r into v's slot.
// A CLUSTER PAIR of CTAs shares each frame: CTA r transforms rows [128 r, 128 r + 128) in pass 1 and
// columns [128 r, 128 r + 128) in pass 2, with one cluster barrier (release / acquire: the slot rows
// the peer wrote are visible) in between.  Against one CTA per frame this halves the slot
// intermediates in flight (74 x 512 KB instead of 148 x 512 KB), which otherwise overflowed L2
// (ncu r2b: 39.4 B/px DRAM against 36 algorithmic).
// ---------------------------------------------------------------------------------------------
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    k_grad256(Geometry g, float2* __restrict__ u, float2* __restrict__ v, const float* __restrict__ d,
              const float2* __restrict__ probe, const DevState* __restrict__ st, float eps) {
    using namespace n256;
    extern __shared__ float2 smem[];
    float2* buf = smem;
    float2* tw = smem + BUF;
    if (st->numeric_error) return;   // uniform over the grid: both CTAs of a pair leave together
    ktime_start(st, 0);
    build_twiddles<N>(tw);
    build_row_twiddles<N>(tw + N);
    __syncthreads();
    uint32_t rank, cid, ncl;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(ncl));
    const float gam = (float)st->gamma;
    const bool upd = gam != 0.0f;
    const float eps2 = eps * eps, scale = 1.0f / (float)N;
    const int tid = threadIdx.x;
    constexpr int HB = N / ROWB / 2;   // row batches (and column batches) per CTA
    // streamed once: u, v, d reads and the u / y writes; reused within microseconds: the slot rows
    const uint64_t pol_s = l2_evict_first(), pol_k = l2_evict_last();
    for (int64_t j = cid; j < g.n_local; j += ncl) {
        float2* vj = v + j * N * N;
        // pass 1: this CTA's rows
#pragma unroll 1
        for (int rb = rank * HB; rb < (int)(rank + 1) * HB; ++rb) {
            const int row = rb * ROWB + tid / T, t = tid % T;
            const int64_t base = j * N * N + (int64_t)row * N + t;
            float2 uu[R];
            float dd[R];
#pragma unroll
            for (int n1 = 0; n1 < R; ++n1) {
                uu[n1] = ld2_hint(u + base + T * n1, pol_s);
                dd[n1] = ld1_hint(d + base + T * n1, pol_s);
            }
            if (upd) {
                float2 vv[R];
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) vv[n1] = ld2_hint(v + base + T * n1, pol_s);
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) {
                    uu[n1] = make_float2(fmaf(gam, vv[n1].x, uu[n1].x), fmaf(gam, vv[n1].y, uu[n1].y));
                    st2_hint(u + base + T * n1, uu[n1], pol_s);
                }
            }
            float2 x[R];
#pragma unroll
            for (int n1 = 0; n1 < R; ++n1) x[n1] = residual(uu[n1], dd[n1], eps2, g.est);
            float2* srow = buf + (tid / T) * LD;
            __syncwarp();
            row_fft_regs<N, true, true>(x, srow, t, tw, tw + N);
            // x[k2] is column t + 16 k2; v of this row was consumed above, so the slot row is free
            float2* dst = vj + (int64_t)row * N + t;
#pragma unroll
            for (int k2 = 0; k2 < T; ++k2) st2_hint(dst + R * k2, x[k2], pol_k);
        }
        // both halves of the row pass are in the slot (cluster-scope release / acquire)
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        // pass 2: this CTA's columns, epilogue y = conj(p) X / N
#pragma unroll 1
        for (int cb = rank * (N / COLB / 2); cb < (int)(rank + 1) * (N / COLB / 2); ++cb) {
            float2 X[16];
            int c;
            n256_column<true>(vj, cb, buf, tw, X, c);
            const int t = tid >> 5;
#pragma unroll
            for (int k2 = 0; k2 < T; ++k2) {
                const int k = t + R * k2;
                st2_hint(vj + (int64_t)k * N + c, cscale(cconjmul(ldg2(probe + k * N + c), X[k2]), scale), pol_s);
            }
        }
        __syncthreads();
    }
    __syncthreads();
    ktime_end(st, 0);
}

// ---------------------------------------------------------------------------------------------
// k_ls256_side: LS pass 0 for N = 256 on the SMs the four-CTA clusters of k_ls_c256ws leave idle (a GPC
// whose SM count is not a multiple of four keeps 2 SMs free: 16 of 148 on B200).  It runs CONCURRENTLY
// with the cluster kernel on a static tail of the canonical frame order [i0, n): the cluster kernel
// releases it with a programmatic-dependent-launch trigger once all its CTAs are resident (so these
// CTAs land on the free SMs and never delay a cluster), and it waits for the cluster grid's completion
// (griddepcontrol.wait) before it exits, so the reduction launched after it sees both kernels' partials.
// One CTA per frame, the frame's own v slot in HBM as the transpose buffer (pass 1: window rows x p/N ->
// row DFTs -> slot rows; pass 2: 32-column batches back from L2 -> column DFTs = v), then the screening
// epilogue of every LS kernel (dev.cuh ls_push / ls_flush) on (u, v, d).  Its per-CTA partial rows follow
// the cluster kernel's in `part` (reduced in one fixed order: bitwise reproducible).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1)
    k_ls256_side(Geometry g, const float2* __restrict__ eta, const float2* __restrict__ probe_s,
                 const int2* __restrict__ pos, const int* __restrict__ order, const float2* __restrict__ u,
                 float2* __restrict__ v, const float* __restrict__ d, SolverCfg cfg, double* __restrict__ part,
                 const DevState* __restrict__ st, int64_t i0) {
    using namespace n256;
    extern __shared__ float2 smem[];
    float2* buf = smem;
    float2* tw = smem + BUF;
    __shared__ double sred[16][KC];
    __shared__ double smom[16][4];
    __shared__ float sgam[KC];
    __shared__ LsWarpQ<2> wq[16];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool err = st->numeric_error != 0;
    int base, cnt;
    ls_pass_range(0, st->keff, cfg, base, cnt);
    ktime_start(st, 1);
    build_twiddles<N>(tw);
    build_row_twiddles<N>(tw + N);
    if (tid < KC) sgam[tid] = (float)trial_gamma(cfg.gamma0, cfg.tau, base + tid);
    __syncthreads();
    const int64_t nfr = err ? 0 : g.n_local;
    const float eps2 = (float)(cfg.eps * cfg.eps);
    const uint64_t pol_s = l2_evict_first(), pol_k = l2_evict_last();
    double tot = 0.0;
    double mom[4] = {0.0, 0.0, 0.0, 0.0};
    trial_dispatch(cnt, cfg, [&]<int KT, bool LSE, bool QG>() {
        float gk[KT];
#pragma unroll
        for (int k = 0; k < KT; ++k) gk[k] = sgam[k];
        for (int64_t i = i0 + blockIdx.x; i < nfr; i += gridDim.x) {
            const int64_t j = order[i];
            const int2 s = pos[j];
            float2* vj = v + j * N * N;
            // ---- pass 1: 8 batches of 32 rows, row DFTs -> slot rows (kept in L2)
#pragma unroll 1
            for (int rb = 0; rb < N / ROWB; ++rb) {
                const int row = rb * ROWB + tid / T, t = tid % T;
                float2 x[R];
                window_row<R, T>(eta, g, s, j, row, t, probe_s + row * N + t, x);
                __syncwarp();
                row_fft_regs<N, false, true>(x, buf + (tid / T) * LD, t, tw, tw + N);
                float2* dst = vj + (int64_t)row * N + t;
#pragma unroll
                for (int k2 = 0; k2 < T; ++k2) st2_hint(dst + R * k2, x[k2], pol_k);
            }
            __syncthreads();   // every slot row written (CTA-scope order of the global stores)
            // ---- pass 2: 8 batches of 32 columns; X[k2] = v at row warp + 16 k2, column c
#pragma unroll 1
            for (int cb = 0; cb < N / COLB; ++cb) {
                float2 X[R];
                int c;
                n256_column<false>(vj, cb, buf, tw, X, c);
                // park X in this thread's own phase-2 slots of buf (read only by this thread) so the
                // epilogue is a rolled loop over groups of four
                float2* mine = buf + (T * warp) * COLB + lane;
#pragma unroll
                for (int k2 = 0; k2 < T; ++k2) mine[k2 * COLB] = X[k2];
                const int64_t ob = j * N * N + (int64_t)warp * N + c;
                float S[KC];
                LsMom m;
#pragma unroll
                for (int k = 0; k < KC; ++k) S[k] = 0.f;
                LsQState qs;
#pragma unroll 1
                for (int gi = 0; gi < T / 4; ++gi) {
                    float2 uc[4], vc[4];
                    float dc[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int64_t o = ob + (int64_t)(4 * gi + e) * R * N;
                        uc[e] = ld2_hint_na(u + o, pol_s);
                        dc[e] = ld1_hint_na(d + o, pol_s);
                        vc[e] = mine[(4 * gi + e) * COLB];
                        st2_hint(v + o, vc[e], pol_s);
                    }
                    ls_push<KT, LSE, QG>(wq[warp], qs, slice<0, 2>(uc), slice<0, 2>(vc), slice<0, 2>(dc), gk, eps2, S,
                                         m, lane);
                    ls_push<KT, LSE, QG>(wq[warp], qs, slice<2, 2>(uc), slice<2, 2>(vc), slice<2, 2>(dc), gk, eps2, S,
                                         m, lane);
                }
                ls_flush<KT, LSE, QG>(wq[warp], qs, gk, eps2, S, m, lane);
                ls_run_out_r<(KT <= 8 ? 8 : KC)>(S, m, tot, mom, lane);
            }
            __syncthreads();   // buf free before the next frame's row exchanges
        }
    });
    ktime_end(st, 1);
    if (cnt <= 8)   // = KT <= 8 (trial_dispatch_k)
        ls_block_out_r<8, 16>(tot, mom, sred, smom, part);
    else
        ls_block_out_r<KC, 16>(tot, mom, sred, smom, part);
    // the kernels after this one in the stream must see the cluster kernel's partials as well
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

int launch_ls256_side(const Geometry& g, const float2* eta, const float2* probe_s, const int2* pos, const int* order,
                      const float2* u, float2* v, const float* d, const SolverCfg& c, double* part, const DevState* st,
                      int64_t i0, int grid, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(k_ls256_side, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)n256::SMEM) !=
            cudaSuccess)
            return -1;
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(512, 1, 1);
    cfg.dynamicSmemBytes = n256::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, k_ls256_side, g, eta, probe_s, pos, order, u, v, d, c, part, st, i0) != cudaSuccess)
        return -1;
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------------------------------------
// k_fwd (N = 256): u = F(p * psi[window]) (pass 1 rows -> u slot, pass 2 columns) and the Eq.2
// objective partials (init / set_state; the LS pass runs on clusters of four, kernels_c256.cu).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(512, 1) k_fwd256(Geometry g, const float2* __restrict__ obj,
                                                   const float2* __restrict__ probe, const int2* __restrict__ pos,
                                                   const int* __restrict__ order, float2* __restrict__ u,
                                                   const float* __restrict__ d, double* __restrict__ part, float eps) {
    using namespace n256;
    extern __shared__ float2 smem[];
    float2* buf = smem;
    float2* tw = smem + BUF;
    __shared__ double sred[16];
    const int tid = threadIdx.x;
    build_twiddles<N>(tw);
    __syncthreads();
    const int64_t nfr = g.n_local;
    const float eps2 = eps * eps, scale = 1.0f / (float)N;
    double facc = 0.0;
    for (int64_t i = blockIdx.x; i < nfr; i += gridDim.x) {
        const int64_t j = order[i];
        const int2 s = pos[j];
        float2* oj = u + j * N * N;
#pragma unroll 1
        for (int rb = 0; rb < N / ROWB; ++rb) {
            const int row = rb * ROWB + tid / T, t = tid % T;
            float2 x[R];
            window_row<R, T>(obj, g, s, j, row, t, probe + row * N + t, x);
            float2* srow = buf + (tid / T) * LD;
            __syncwarp();
            row_fft_regs<N, false>(x, srow, t, tw);
            float2* dst = oj + (int64_t)row * N + t;
#pragma unroll
            for (int k2 = 0; k2 < T; ++k2) dst[R * k2] = x[k2];
        }
        __syncthreads();
#pragma unroll 1
        for (int cb = 0; cb < N / COLB; ++cb) {
            float2 X[16];
            int c;
            n256_column<false>(oj, cb, buf, tw, X, c);
            const int t = tid >> 5;
            float fs = 0.f;
#pragma unroll
            for (int k2 = 0; k2 < T; ++k2) {
                const int64_t o = j * N * N + (int64_t)(t + R * k2) * N + c;
                const float2 uu = cscale(X[k2], scale);
                u[o] = uu;
                const float cc = uu.x * uu.x + uu.y * uu.y;
                if (d) fs += objective_term(cc, __ldg(d + o), eps2, g.est);
            }
            facc += (double)fs;
        }
        __syncthreads();
    }
    const double s2 = block_sum<512>(facc, sred);
    if (tid == 0) part[blockIdx.x] = s2;
}

// Batched 2-D FFT (ptyger_fft2, N = 256): pass 1 writes row transforms into `out`, pass 2 reads
// them back column-wise and writes the final values in place.
template <bool INV>
__global__ void __launch_bounds__(512, 1) k_fft2_256(const float2* __restrict__ in, float2* __restrict__ out,
                                                     int64_t batch) {
    using namespace n256;
    extern __shared__ float2 smem[];
    float2* buf = smem;
    float2* tw = smem + BUF;
    build_twiddles<N>(tw);
    __syncthreads();
    const int tid = threadIdx.x;
    const float scale = 1.0f / (float)N;
    for (int64_t j = blockIdx.x; j < batch; j += gridDim.x) {
        float2* oj = out + j * N * N;
#pragma unroll 1
        for (int rb = 0; rb < N / ROWB; ++rb) {
            const int row = rb * ROWB + tid / T, t = tid % T;
            const float2* src = in + j * N * N + (int64_t)row * N + t;
            float2 x[R];
#pragma unroll
            for (int n1 = 0; n1 < R; ++n1) x[n1] = ldg2(src + T * n1);
            float2* srow = buf + (tid / T) * LD;
            __syncwarp();
            row_fft_regs<N, INV>(x, srow, t, tw);
            float2* dst = oj + (int64_t)row * N + t;
#pragma unroll
            for (int k2 = 0; k2 < T; ++k2) dst[R * k2] = x[k2];
        }
        __syncthreads();
#pragma unroll 1
        for (int cb = 0; cb < N / COLB; ++cb) {
            float2 X[16];
            int c;
            n256_column<INV>(oj, cb, buf, tw, X, c);
            const int t = tid >> 5;
#pragma unroll
            for (int k2 = 0; k2 < T; ++k2) oj[(int64_t)(t + R * k2) * N + c] = cscale(X[k2], scale);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ launchers
template <typename F>
static int n256_smem(F* f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)n256::SMEM) == cudaSuccess ? 0
                                                                                                              : -1;
}

int launch_grad256(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe, const DevState* st,
                   float eps, int grid, cudaStream_t s) {
    (void)grid;
    static int pairs = 0;   // resident cluster pairs (one CTA per SM)
    if (n256_smem(k_grad256)) return -1;
    if (pairs == 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * 74, 1, 1);
        cfg.blockDim = dim3(512, 1, 1);
        cfg.dynamicSmemBytes = n256::SMEM;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_grad256, &cfg) != cudaSuccess || ncl <= 0) {
            cudaGetLastError();
            ncl = 148 / 2;
        }
        pairs = ncl;
    }
    const int64_t np = g.n_local < pairs ? (g.n_local > 0 ? g.n_local : 1) : pairs;
    k_grad256<<<(int)(2 * np), 512, n256::SMEM, s>>>(g, u, v, d, probe, st, eps);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_fwd256(const Geometry& g, const float2* psi, const float2* probe, const int2* pos, const int* order,
                  const float* d, float2* u, double* part, int grid, float eps, cudaStream_t s) {
    if (n256_smem(k_fwd256)) return -1;
    k_fwd256<<<grid, 512, n256::SMEM, s>>>(g, psi, probe, pos, order, u, d, part, eps);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_fft2_256(const float2* in, float2* out, int64_t batch, bool inv, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)(batch < sms ? batch : sms);
    if (grid <= 0) return 0;
    if (inv) {
        if (n256_smem(k_fft2_256<true>)) return -1;
        k_fft2_256<true><<<grid, 512, n256::SMEM, s>>>(in, out, batch);
    } else {
        if (n256_smem(k_fft2_256<false>)) return -1;
        k_fft2_256<false><<<grid, 512, n256::SMEM, s>>>(in, out, batch);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pty
