// LS pass 0 for N = 128 frames, WARP-SPECIALISED (Alg.1 659-668, Eq.7 on the Eq.2 objective; the
// screening contract of k_ls<N> in kernels_frame.cu is unchanged).
//
// r2 measurement of the single-group k_ls<128> (profiles/r2_history.md): its three phases --
// window gathers (0.61 ms), the two FFT passes + v store (1.39 ms) and the screening epilogue
// (1.24 ms at 10 trials) -- ADD UP (3.17 ms): all 16 warps run the same phase at the same time, so
// the gather latency, the shared-memory FFT and the MUFU / u,d-streaming epilogue never overlap.
// Here one persistent 512-thread CTA per SM splits into two groups that work on different frames:
//
//   FFT group (warps 0-7):  frame j's eta window -> shared memory by the TMA engine (one 1-D bulk
//       copy per row, cp.async.bulk, issued as soon as the frame buffer is free, so the copy flies
//       while the group finishes the previous frame), x = (p / N) eta, row pass, column pass; the
//       column-pass outputs v_j go to TENSOR MEMORY (tcgen05.st), not back to shared memory;
//   epilogue group (warps 8-15): frame j-1's v from tensor memory (tcgen05.ld), v store to HBM,
//       u / d streamed from HBM (bulk L2 prefetch one frame ahead), the screening terms of the
//       pass-0 trials (dev.cuh ls_push / ls_flush).
//
// Tensor memory (256 KB per SM, otherwise unused here: nothing in the path is a dense contraction)
// is the hand-off buffer: 2 slots x 128 KB = one frame of v each, double-buffered.  Lane quarter
// rule: warp w may only touch TMEM lanes 32 (w % 4) .. +31, so FFT warp w and epilogue warp w + 8 share
// a quarter; w / 4 picks the 128-column half.  Per thread and frame: 4 column rounds x 16 complex =
// 128 32-bit columns.  Hand-off with named barriers (bar.arrive / bar.sync, 512 threads): FULL[b]
// (FFT -> epilogue, slot b written) and EMPTY[b] (epilogue -> FFT, slot b read), plus the
// tcgen05.fence::before/after_thread_sync pair around each.
//
// Everything else is the arithmetic of the other frame kernels (fft.cuh radix-16 x radix-8 lines,
// fp64-built twiddles, paired FP32); the trial sums, moments and partial layout are those of k_ls,
// so k_reduce / k_pick consume them unchanged.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "dev.cuh"
#include "tma.cuh"

namespace pty {

namespace ws {
constexpr int N = 128, R = 16, T = 8, LD = N + 8;
constexpr int NT = 512, NF = 256;             // FFT group = threads [0, 256), epilogue group = [256, 512)
constexpr int RROWS = NF / T;                 // 32 rows per row-pass round
constexpr int ROUNDS = N / RROWS;             // 4 row rounds
constexpr int CROUNDS = N * T / NF;           // 4 column rounds of 32 columns
constexpr size_t FRAME_BYTES = (size_t)N * LD * 8;                  // 139 264
constexpr size_t TW_OFF = FRAME_BYTES;                              // float4 tw[N], twr[R*T]
constexpr int SROWS = N / 2;                  // window rows staged ahead of the frame buffer
constexpr int SLD = N + 8;                    // staged row stride (complex), same bank offset as LD
constexpr size_t STG_OFF = TW_OFF + (size_t)(N + R * T) * 16;
constexpr size_t DYN_BYTES = STG_OFF + (size_t)SROWS * SLD * 8;
constexpr int TMEM_COLS = 512;
// named barrier ids (0 is __syncthreads)
constexpr int BAR_FFT = 1, BAR_FULL = 2, BAR_EMPTY = 4;
}  // namespace ws

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 complex (32 words) of this thread into TMEM columns [col, col + 32) of the warp's lane quarter
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float2 (&x)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(x[0].x), "f"(x[0].y), "f"(x[1].x), "f"(x[1].y), "f"(x[2].x), "f"(x[2].y), "f"(x[3].x), "f"(x[3].y),
        "f"(x[4].x), "f"(x[4].y), "f"(x[5].x), "f"(x[5].y), "f"(x[6].x), "f"(x[6].y), "f"(x[7].x), "f"(x[7].y),
        "f"(x[8].x), "f"(x[8].y), "f"(x[9].x), "f"(x[9].y), "f"(x[10].x), "f"(x[10].y), "f"(x[11].x), "f"(x[11].y),
        "f"(x[12].x), "f"(x[12].y), "f"(x[13].x), "f"(x[13].y), "f"(x[14].x), "f"(x[14].y), "f"(x[15].x),
        "f"(x[15].y)
        : "memory");
}
// 4 complex (8 words) from TMEM columns [col, col + 8)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float2 (&x)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(x[0].x), "=f"(x[0].y), "=f"(x[1].x), "=f"(x[1].y), "=f"(x[2].x), "=f"(x[2].y), "=f"(x[3].x),
                   "=f"(x[3].y)
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <bool DMA>
__global__ void __launch_bounds__(512, 1) k_ls_ws(Geometry g, const float2* __restrict__ eta,
                                                  const float2* __restrict__ probe_s, const int2* __restrict__ pos,
                                                  const int* __restrict__ order, const float2* __restrict__ u,
                                                  float2* __restrict__ v, const float* __restrict__ d, SolverCfg cfg,
                                                  double* __restrict__ part, const DevState* __restrict__ st,
                                                  int pf) {
    using namespace ws;
    extern __shared__ __align__(16) unsigned char smraw[];
    float2* sf = reinterpret_cast<float2*>(smraw);
    float4* tw = reinterpret_cast<float4*>(smraw + TW_OFF);
    __shared__ double sred[16][KC];
    __shared__ double smom[16][4];
    __shared__ float sgam[KC];
    __shared__ LsWarpQ<2> wq[8];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_mbar[2];   // [0] staged rows 0..63, [1] rows 64..127 in sf
    __shared__ int s_done[2];                      // FFT warps done reading [0] the staging, [1] the frame buffer
    float2* stg = reinterpret_cast<float2*>(smraw + STG_OFF);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool err = st->numeric_error != 0;
    int base, cnt;
    ls_pass_range(0, st->keff, cfg, base, cnt);
    ktime_start(st, 1);
    build_twiddles4<N, false>(tw);
    if (tid < KC) sgam[tid] = (float)trial_gamma(cfg.gamma0, cfg.tau, base + tid);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&s_mbar[0], 1);
        mbar_init(&s_mbar[1], 1);
        fence_mbar_init();
        s_done[0] = s_done[1] = 0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = s_tmem;
    const int64_t nfr = err ? 0 : g.n_local;
    const int64_t W = g.W;
    // quarter / half of this warp's TMEM region (FFT warp w and epilogue warp w + 8 share it)
    const int wq4 = warp & 3, whalf = (warp & 7) >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * wq4) << 16) + (uint32_t)(128 * whalf);

    // TMA bulk copies of frame i's eta window rows [h 64, h 64 + 64) (warp 0 of the FFT group, one
    // row per lane and step): h = 0 into the staging buffer, issued as soon as the previous frame's
    // row pass has read it (so it flies during that frame's column pass and epilogue hand-off);
    // h = 1 into rows 64..127 of the frame buffer, issued once the previous frame's column pass
    // has released it (it flies during this frame's first two row rounds).  A window starting at an
    // odd column is copied from the column before it (16-B alignment, 130 elements) and read at
    // offset 1.
    auto issue_dma = [&](int64_t i, int h) {
        const int j = order[i];
        const int2 s = pos[j];
        const int off = s.y & 1;
        const uint32_t bytes = (uint32_t)(N + 2 * off) * 8u;
        if (lane == 0) mbar_arrive_expect_tx(&s_mbar[h], bytes * SROWS);
        __syncwarp();
        const float2* src = eta + (int64_t)(s.x + h * SROWS) * W + (s.y - off);
        float2* dst = h ? sf + SROWS * LD : stg;
        const int ld = h ? LD : SLD;
#pragma unroll
        for (int q = 0; q < SROWS / 32; ++q) {
            const int r = q * 32 + lane;
            bulk_g2s(dst + r * ld, src + (int64_t)r * W, bytes, &s_mbar[h]);
        }
    };
    // Staged half (h = 0) of the next frame, per warp: the 8 rows this warp reads in rounds 0 and 1 (a
    // row's 8 sub-threads sit in one warp), so no other warp's reads are overwritten and no counter is
    // needed; warp 0 posts the transaction count of all 64 rows (the phase cannot complete before it).
    auto issue_own_staged = [&](int64_t inext) {
        const int jn = order[inext];
        const int2 sn = pos[jn];
        const int off = sn.y & 1;
        const uint32_t bytes = (uint32_t)(N + 2 * off) * 8u;
        __syncwarp();
        if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&s_mbar[0], bytes * SROWS);
        if (lane < 8) {
            fence_proxy_async();
            const int r = (lane < 4 ? 0 : RROWS) + 4 * warp + (lane & 3);
            bulk_g2s(stg + r * SLD, eta + (int64_t)(sn.x + r) * W + (sn.y - off), bytes, &s_mbar[0]);
        }
    };
    // An FFT warp is done reading buffer h (0 staging, 1 frame buffer) of this frame: the LAST of the 8
    // to get there issues the next frame's copy into it, so no warp waits for the others.  Generic reads
    // -> release / acquire on the counter -> proxy fence -> async-proxy writes.
    auto done_reading = [&](int64_t i, int h) {
        __syncwarp();
        int last = 0;
        if (lane == 0) {
            fence_proxy_async();
            const int old = atomicAdd_block(&s_done[h], 1);
            __threadfence_block();
            last = old == NF / 32 - 1;
            if (last) s_done[h] = 0;   // re-armed before any warp can reach this point again (bar B2)
        }
        last = __shfl_sync(FULLMASK, last, 0);
        if (last) {
            fence_proxy_async();
            if (i + gridDim.x < nfr) issue_dma(i + gridDim.x, h);
        }
    };

    double tot = 0.0;
    double mom[4] = {0.0, 0.0, 0.0, 0.0};
    if (tid < NF) {
        // ============================ FFT group ============================
        const int ft = tid;
        if (DMA && warp == 0 && blockIdx.x < nfr) {
            issue_dma(blockIdx.x, 0);
            issue_dma(blockIdx.x, 1);
        }
        int it = 0;
        for (int64_t i = blockIdx.x; i < nfr; i += gridDim.x, ++it) {
            const int b = it & 1;
            const int j = order[i];
            const int2 s = pos[j];
            // ---- row pass: 4 rounds of 32 rows, two rounds' inputs in flight at a time
            const int t = ft % T, rrow = ft / T;
            auto load_row = [&](int rd, float2 (&x)[R]) {
                const int row = rd * RROWS + rrow;
                const float2* pp = probe_s + row * N + t;
                if constexpr (DMA) {
                    const float2* se = (row < SROWS ? stg + row * SLD : sf + row * LD) + (s.y & 1) + t;
#pragma unroll
                    for (int n1 = 0; n1 < R; ++n1) x[n1] = cmul(ldg2(pp + T * n1), se[T * n1]);
                } else {
                    window_row<R, T>(eta, g, s, j, row, t, pp, x);
                }
            };
#pragma unroll 1
            for (int rp = 0; rp < ROUNDS; rp += 2) {
                if (DMA) mbar_wait(&s_mbar[rp / 2], (uint32_t)(it & 1));
                float2 xa[R], xb[R];
                load_row(rp, xa);
                load_row(rp + 1, xb);
                // this warp's staged rows (4w..4w+3, 32+4w..32+4w+3: exactly the rows it read) are
                // consumed: the next frame's copies of them are issued right away by the warp itself
                if (DMA && rp == 0 && i + gridDim.x < nfr) issue_own_staged(i + gridDim.x);
                row_fft_a<N, false, true>(xa, t, tw, tw + N);
                row_fft_a<N, false, true>(xb, t, tw, tw + N);
                // every FFT warp has finished the previous frame's column pass (its reads of the frame
                // buffer) before this frame's first row writes land in it
                if (rp == 0) bar_sync_n(BAR_FFT, NF);
                __syncwarp();   // every lane of the warp has read its rows before any exchange write
                row_fft_b<N, false>(xa, sf + (rp * RROWS + rrow) * LD, t);
                row_fft_b<N, false>(xb, sf + ((rp + 1) * RROWS + rrow) * LD, t);
            }
            bar_sync_n(BAR_FFT, NF);
            // ---- column pass phase 1: 4 rounds of 32 columns, sub-thread t = warp
#pragma unroll 1
            for (int rd = 0; rd < CROUNDS; ++rd) col_fft_phase1<N, false>(sf + rd * 32 + lane, warp, tw);
            bar_sync_n(BAR_FFT, NF);
            // ---- slot b must have been read by the epilogue (frame it - 2)
            if (it >= 2) {
                bar_sync_n(BAR_EMPTY + b, NT);
                tc_fence_after();
            }
            // ---- column pass phase 2 -> tensor memory slot b, 32 columns per round
#pragma unroll 1
            for (int rd = 0; rd < CROUNDS; ++rd) {
                float2 X[R];
                col_fft_phase2<N, false>(sf + rd * 32 + lane, warp, X);
                tmem_st32(tq + (uint32_t)(256 * b + 32 * rd), X);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            bar_arrive_n(BAR_FULL + b, NT);
            // ---- this warp's reads of the frame buffer are done: the next frame's second window half
            // may land in it once all eight are (the barrier before the next row writes orders the rest)
            if (DMA) done_reading(i, 1);
        }
    } else {
        // ============================ epilogue group ============================
        const int ew = warp - 8;                  // = the FFT warp whose outputs this warp reads
        const float eps2 = (float)(cfg.eps * cfg.eps);
        int nmine = 0;
        for (int64_t i = blockIdx.x; i < nfr; i += gridDim.x) ++nmine;
        trial_dispatch(cnt, cfg, [&]<int KT, bool LSE, bool QG>() {
            float gk[KT];   // trial gammas in registers for the whole run
#pragma unroll
            for (int k = 0; k < KT; ++k) gk[k] = sgam[k];
            // u, d of one group of 4 elements: frame jf, round rd (column c = 32 rd + lane), elements
            // q = 4 gi .. 4 gi + 3 at rows (q / T) T + ew + R (q % T).  The loads run one group ahead
            // ACROSS rounds and frames, so no round starts on an exposed L2 latency.
            auto elem_base = [&](int64_t jf, int rd) -> int64_t {
                return jf * (int64_t)(N * N) + (int64_t)ew * N + rd * 32 + lane;
            };
            auto goff = [](int gi) -> int {
                const int q0 = 4 * gi;
                return ((q0 / T) * T + R * (q0 % T)) * N;
            };
            float2 un[4];
            float dn[4];
            auto load_group = [&](int64_t jf, int rd, int gi) {
                const int64_t o = elem_base(jf, rd) + goff(gi);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    un[e] = ldg2_na(u + o + e * R * N);
                    dn[e] = ldg1_na(d + o + e * R * N);
                }
            };
            if (nmine > 0) load_group(order[blockIdx.x], 0, 0);
            int it = 0;
            for (int64_t i = blockIdx.x; i < nfr; i += gridDim.x, ++it) {
                const int b = it & 1;
                const int64_t jf = order[i];
                const int64_t jnext = i + gridDim.x < nfr ? (int64_t)order[i + gridDim.x] : -1;
                // this frame's u, d into L2 while its transform is still running
                // (issued by the FFT group half a frame earlier, or one frame ahead: measured no better
                // than no prefetch at all, 3.12 / 2.98 ms against 2.72 ms)
                if (pf) {
                    if (ew == 0) prefetch_l2_frame(u + jf * N * N, N * N * 8, lane);
                    else if (ew == 1) prefetch_l2_frame(d + jf * N * N, N * N * 4, lane);
                }
                bar_sync_n(BAR_FULL + b, NT);
                tc_fence_after();
#pragma unroll 1
                for (int rd = 0; rd < CROUNDS; ++rd) {
                    float2* __restrict__ vb = v + elem_base(jf, rd);
                    float S[KC];
                    LsMom m;
#pragma unroll
                    for (int k = 0; k < KC; ++k) S[k] = 0.f;
                    LsQState qs;
#pragma unroll 1
                    for (int gi = 0; gi < R / 4; ++gi) {
                        const int go = goff(gi);
                        float2 uc[4];
                        float dc[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            uc[e] = un[e];
                            dc[e] = dn[e];
                        }
                        if (gi + 1 < R / 4)
                            load_group(jf, rd, gi + 1);
                        else if (rd + 1 < CROUNDS)
                            load_group(jf, rd + 1, 0);
                        else if (jnext >= 0)
                            load_group(jnext, 0, 0);
                        float2 X[4];
                        tmem_ld8(tq + (uint32_t)(256 * b + 32 * rd + 8 * gi), X);
#pragma unroll
                        for (int e = 0; e < 4; ++e) vb[go + e * R * N] = X[e];
                        ls_push<KT, LSE, QG>(wq[ew], qs, slice<0, 2>(uc), slice<0, 2>(X), slice<0, 2>(dc), gk, eps2, S,
                                         m, lane);
                        ls_push<KT, LSE, QG>(wq[ew], qs, slice<2, 2>(uc), slice<2, 2>(X), slice<2, 2>(dc), gk, eps2, S,
                                         m, lane);
                    }
                    ls_flush<KT, LSE, QG>(wq[ew], qs, gk, eps2, S, m, lane);
                    ls_run_out_r<(KT <= 8 ? 8 : KC)>(S, m, tot, mom, lane);
                }
                // slot b read: the FFT group may overwrite it (frame it + 2) -- no arrival without a waiter
                tc_fence_before();
                if (it + 2 < nmine) bar_arrive_n(BAR_EMPTY + b, NT);
            }
        });
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TMEM_COLS));
    ktime_end(st, 1);
    if (cnt <= 8)   // = KT <= 8 (trial_dispatch_k)
        ls_block_out_r<8, 16>(tot, mom, sred, smom, part);
    else
        ls_block_out_r<KC, 16>(tot, mom, sred, smom, part);
}

int launch_ls_ws(const Geometry& g, const float2* eta, const float2* probe_s, const int2* pos, const int* order,
                 const float2* u, float2* v, const float* d, const SolverCfg& c, double* part, int grid,
                 const DevState* st, cudaStream_t s) {
    // the row DMA needs 16-B aligned window rows: even object width, integer positions
    const bool dma = (g.W % 2 == 0) && g.frac == nullptr;
    static const int pf = getenv("PTYGER_PF") ? atoi(getenv("PTYGER_PF")) : 1;   // L2 prefetch of u, d
    if (dma) {
        if (cudaFuncSetAttribute(k_ls_ws<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws::DYN_BYTES) !=
            cudaSuccess)
            return -1;
        k_ls_ws<true><<<grid, ws::NT, ws::DYN_BYTES, s>>>(g, eta, probe_s, pos, order, u, v, d, c, part, st, pf);
    } else {
        if (cudaFuncSetAttribute(k_ls_ws<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws::DYN_BYTES) !=
            cudaSuccess)
            return -1;
        k_ls_ws<false><<<grid, ws::NT, ws::DYN_BYTES, s>>>(g, eta, probe_s, pos, order, u, v, d, c, part, st, pf);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pty
