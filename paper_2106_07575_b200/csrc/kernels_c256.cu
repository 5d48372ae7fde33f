// Frame kernels for N = 256 on a CLUSTER OF FOUR CTAs per frame (distributed shared memory).
//
// A 256 x 256 complex64 frame is 512 KB, more than one SM's shared memory.  The slot kernels
// (kernels_n256.cu) transpose through the frame's own v slot in HBM, which at the large config
// costs +34 % DRAM traffic in k_grad (the 76 MB of in-flight intermediates overflow L2) and leaves
// both passes latency-bound.  Here the four CTAs of a cluster (4 SMs, 4 x 218 KB of shared memory)
// hold the frame between the two passes:
//   * CTA r transforms rows [64 r, 64 r + 64) (row pass, inputs straight from global memory);
//   * output column k of a row belongs to CTA k / 64: each row's 256 outputs are stored straight
//     into the owning CTA's 256 x 64 column block (st.shared::cluster, 3/4 of them remote), so the
//     2-D transpose is the DSMEM exchange (96 KB out of every CTA per frame);
//   * CTA r runs the column pass and the fused epilogue on its 64 columns locally.
// The arithmetic is that of the other FFT paths (fft.cuh: radix-16 in registers x radix-16
// across 16 threads per dimension, fp64-built twiddles, paired-FP32 complex arithmetic); the
// unitary 1/N rides on the prescaled probe (probe_s = p / N).
//
//   k_ls_c256    LS pass 0 (Alg.1 659-668, Eq.7 on the Eq.2 objective): v = F(p eta[window]) and
//                the screening partials of the pass-0 trials against (u, d)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "dev.cuh"
#include "tma.cuh"

namespace pty {

namespace c256 {
constexpr int N = 256, R = 16, T = 16, NT = 512, NW = NT / 32, CL = 4;
constexpr int QC = N / CL;                  // 64 columns owned per CTA
constexpr int QR = N / CL;                  // 64 rows transformed per CTA
constexpr int SROWS = NT / T;               // 32 rows per row-pass round
constexpr int SLD = N + 8;                  // row-scratch stride (complex)
constexpr size_t BLK_BYTES = (size_t)N * QC * 8;           // 131072
constexpr size_t SCR_OFF = BLK_BYTES;
constexpr size_t TW_OFF = SCR_OFF + (size_t)SROWS * SLD * 8; // + 67584
constexpr size_t DYN_BYTES = TW_OFF + (size_t)(N + R * T) * 16;   // float4 tw[N] + row-pass table twr [k1][t]
}  // namespace c256

__device__ __forceinline__ uint32_t c4_mapa(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void c4_st2(uint32_t caddr, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(caddr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ uint32_t c4_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t c4_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t c4_count() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void c4_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void c4_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void c4_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// The GRAD pass keeps the v-slot kernel of kernels_n256.cu: a cluster version of it measured
// 63.7 ms against 46.6 ms at the large config (phase-locked CTAs, one per SM) and was removed.

// Row pass of one row (16 sub-threads t of one row, consecutive lanes): x[n1] = input at column
// 16 n1 + t.  After the transform x[k2] is output column t + 16 k2, owned by CTA k2 / 4 at local
// column t + 16 (k2 % 4).  `first` (round 0): wait until every peer has released its block.
template <bool INV, typename TW>
__device__ __forceinline__ void c4_row(float2 (&x)[16], float2* srow, int t, const TW* tw, int row,
                                       const uint32_t (&cb)[4], bool first) {
    using namespace c256;
    row_fft_regs<N, INV, true>(x, srow, t, tw, tw + N);   // twr [k1][t] follows tw
    if (first) c4_wait();
#pragma unroll
    for (int k2 = 0; k2 < T; ++k2)
        c4_st2(cb[k2 >> 2] + (uint32_t)(row * QC + t + R * (k2 & 3)) * 8u, x[k2]);
}

// Column pass on the local 256 x 64 block: phase 1 for local column cl, sub-thread t (= warp).
template <bool INV, typename TW>
__device__ __forceinline__ void c4_col1(float2* blk, int cl, int t, const TW* tw) {
    using namespace c256;
    float2 x[R];
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) x[n1] = blk[(T * n1 + t) * QC + cl];
    DFT<R, INV>::run(x);
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) x[k1] = twm<INV>(x[k1], tw, t * k1);
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) blk[(T * k1 + t) * QC + cl] = x[k1];
}

// phase 2: X[k2] = output row t + 16 k2 of local column cl (k1 = t, inputs rows 16 t + n2)
template <bool INV>
__device__ __forceinline__ void c4_col2(const float2* blk, int cl, int t, float2 (&X)[16]) {
    using namespace c256;
#pragma unroll
    for (int n2 = 0; n2 < T; ++n2) X[n2] = blk[(T * t + n2) * QC + cl];
    DFT<T, INV>::run(X);
}

// ----------------------------------------------------------------------------------------
// k_ls_c256 (screening contract: k_ls<N> in kernels_frame.cu)
// ----------------------------------------------------------------------------------------
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(512, 1)
    k_ls_c256(Geometry g, const float2* __restrict__ eta, const float2* __restrict__ probe_s,
              const int2* __restrict__ pos, const int* __restrict__ order, const float2* __restrict__ u,
              float2* __restrict__ v, const float* __restrict__ d, SolverCfg cfg, double* __restrict__ part,
              const DevState* __restrict__ st) {
    using namespace c256;
    extern __shared__ __align__(16) unsigned char smraw[];
    float2* blk = reinterpret_cast<float2*>(smraw);
    float2* scr = reinterpret_cast<float2*>(smraw + SCR_OFF);
    float4* tw = reinterpret_cast<float4*>(smraw + TW_OFF);
    // the d > 0 queues of the epilogue live in the row-pass scratch (free between the cluster
    // barrier after the row pass and the next frame's row pass)
    LsWarpQ<4>* wq = reinterpret_cast<LsWarpQ<4>*>(scr);
    static_assert(sizeof(LsWarpQ<4>) * NW <= (size_t)SROWS * SLD * 8, "queues exceed the row scratch");
    __shared__ double sred[NW][KC];
    __shared__ double smom[NW][4];
    __shared__ float sgam[KC];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = c4_rank();
    const int64_t cid = c4_id(), ncl = c4_count();
    const bool err = st->numeric_error != 0;
    int base, cnt;
    ls_pass_range(0, st->keff, cfg, base, cnt);
    ktime_start(st, 1);
    build_twiddles4<N, false>(tw);
    if (tid < KC) sgam[tid] = (float)trial_gamma(cfg.gamma0, cfg.tau, base + tid);
    uint32_t cb[4];
    {
        const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(blk));
#pragma unroll
        for (int q = 0; q < 4; ++q) cb[q] = c4_mapa(sb, q);
    }
    __syncthreads();
    c4_arrive_relaxed();
    const int64_t nfr = err ? 0 : g.n_local;
    const float eps2 = (float)(cfg.eps * cfg.eps);
    double tot = 0.0;
    double mom[4] = {0.0, 0.0, 0.0, 0.0};
    const int rt = tid & 15, rrow = tid >> 4;
    for (int64_t i = cid; i < nfr; i += ncl) {
        const int j = order[i];
        const int2 s = pos[j];
        // ---- row pass: rows 64 rank + 32 rd + rrow of (p / N) * eta[window]
        {
            float2 xa[R], xb[R];
            const int row0 = (int)rank * QR + rrow, row1 = row0 + SROWS;
            window_row<R, T>(eta, g, s, j, row0, rt, probe_s + row0 * N + rt, xa);
            window_row<R, T>(eta, g, s, j, row1, rt, probe_s + row1 * N + rt, xb);
            c4_row<false>(xa, scr + rrow * SLD, rt, tw, row0, cb, true);
            c4_row<false>(xb, scr + rrow * SLD, rt, tw, row1, cb, false);
        }
        c4_arrive();
        c4_wait();
#pragma unroll 1
        for (int rd = 0; rd < QC / 32; ++rd) c4_col1<false>(blk, rd * 32 + lane, warp, tw);
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < QC / 32; ++rd) {
            const int cl = rd * 32 + lane;
            float2* mine = blk + (T * warp) * QC + cl;   // the thread's own phase-2 rows 16 t + k2
            {
                float2 X[R];
                c4_col2<false>(blk, cl, warp, X);
#pragma unroll
                for (int k2 = 0; k2 < T; ++k2) mine[k2 * QC] = X[k2];
            }
            float S[KC];
            LsMom m;
#pragma unroll
            for (int k = 0; k < KC; ++k) S[k] = 0.f;
            // element k2 of column c sits at frame row t + 16 k2: offset (t + 16 k2) N + c
            const int64_t fb = (int64_t)j * (N * N) + (int64_t)warp * N + (int64_t)rank * QC + cl;
            const float2* __restrict__ ub = u + fb;
            const float* __restrict__ db = d + fb;
            float2* __restrict__ vb = v + fb;
            if (cnt > 0) trial_dispatch(cnt, cfg, [&]<int KT, bool LSE, bool QG>() {
                float gk[KT];
#pragma unroll
                for (int k = 0; k < KT; ++k) gk[k] = sgam[k];
                LsQState qs;
                const uint64_t pol = l2_evict_first();   // u, d read once, v written once per pass
                float2 un[4];
                float dn[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    un[e] = ld2_hint_na(ub + e * R * N, pol);
                    dn[e] = ld1_hint_na(db + e * R * N, pol);
                }
#pragma unroll 1
                for (int gi = 0; gi < T / 4; ++gi) {
                    const int go = gi * 4 * R * N;
                    float2 uc[4];
                    float dc[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        uc[e] = un[e];
                        dc[e] = dn[e];
                    }
                    if (gi + 1 < T / 4) {
                        const int gn = go + 4 * R * N;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            un[e] = ld2_hint_na(ub + gn + e * R * N, pol);
                            dn[e] = ld1_hint_na(db + gn + e * R * N, pol);
                        }
                    }
                    float2 vv[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        vv[e] = mine[(gi * 4 + e) * QC];
                        st2_hint(vb + go + e * R * N, vv[e], pol);
                    }
                    ls_push<KT, LSE, QG>(wq[warp], qs, uc, vv, dc, gk, eps2, S, m, lane);
                }
                ls_flush<KT, LSE, QG>(wq[warp], qs, gk, eps2, S, m, lane);
            });
            ls_run_out<KC>(S, m, tot, mom, lane);
        }
        __syncthreads();
        c4_arrive_relaxed();
    }
    c4_wait();
    ktime_end(st, 1);
    ls_block_out<KC, NW>(tot, mom, sred, smom, part);
}

// ----------------------------------------------------------------------------------------
// k_ls_c256ws: the same cluster-of-four frame, WARP-SPECIALISED like k_ls_ws (kernels_ls128.cu):
// in every CTA an FFT group (warps 0-7) runs the row pass (remote stores into the owners' column
// blocks) and the column pass of its block, whose outputs go to TENSOR MEMORY (2 slots x 128 KB =
// the CTA's 256 x 64 block of v, double-buffered); an epilogue group (warps 8-15) stores v and
// screens the trials against u, d for the previous frame meanwhile.  The four FFT groups synchronise
// through mbarriers with remote (shared::cluster) arrivals instead of cluster barriers, so the
// epilogue warps are never held by the exchange:
//   rows_in[q]  (count 4 CTAs x 8 warps): every warp of every CTA has stored its rows of frame f
//               into the block of CTA q  -> CTA q may run its column pass of frame f;
//   peer_free[q] (count 32): every warp of every CTA has finished reading its own block for frame
//               f (column pass done)  -> CTA q may store frame f + 1 rows into the other blocks.
// Release / acquire at cluster scope (per warp: __syncwarp, then lane 0 arrives).
// ----------------------------------------------------------------------------------------
namespace c4w {
constexpr int N = 256, R = 16, T = 16, NT = 512, NF = 256, QC = 64;
constexpr int RROWS = NF / T;              // 16 rows per row-pass round
constexpr int SLD = N + 8;
constexpr size_t BLK_BYTES = (size_t)N * QC * 8;                    // 131072
constexpr size_t SCR_OFF = BLK_BYTES;                               // 2 x 16 exchange rows
constexpr size_t TW_OFF = SCR_OFF + (size_t)2 * RROWS * SLD * 8;    // + 67584
constexpr size_t DYN_BYTES = TW_OFF + (size_t)(N + R * T) * 16;     // float4 tw[N] + twr[R*T]
constexpr int TMEM_COLS = 512;
constexpr int BAR_FFT = 1, BAR_FULL = 2, BAR_EMPTY = 4;
}  // namespace c4w

__device__ __forceinline__ void c4_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void c4_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void c4_tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void c4_tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// arrive on the mbarriers of the four CTAs (shared::cluster addresses): one release fence at cluster
// scope, then relaxed arrivals (a .release arrival each costs its own fence)
__device__ __forceinline__ void c4_remote_arrive4(const uint32_t (&caddr)[4]) {
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
#pragma unroll
    for (int q = 0; q < 4; ++q)
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr[q]) : "memory");
}
// bounded wait (acquire, cluster scope) for the phase of parity `ph` of a local mbarrier
__device__ __forceinline__ void c4_wait_parity(uint64_t* bar, uint32_t ph) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    uint32_t ok = 0, spins = 0;
    while (true) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(a), "r"(ph)
            : "memory");
        if (ok) break;
        if (++spins == (1u << 26)) __trap();
    }
}
__device__ __forceinline__ void c4_tmem_st32(uint32_t taddr, const float2 (&x)[16]) {
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
__device__ __forceinline__ void c4_tmem_ld8(uint32_t taddr, float2 (&x)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(x[0].x), "=f"(x[0].y), "=f"(x[1].x), "=f"(x[1].y), "=f"(x[2].x), "=f"(x[2].y), "=f"(x[3].x),
                   "=f"(x[3].y)
                 : "r"(taddr)
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(512, 1)
    k_ls_c256ws(Geometry g, const float2* __restrict__ eta, const float2* __restrict__ probe_s,
                const int2* __restrict__ pos, const int* __restrict__ order, const float2* __restrict__ u,
                float2* __restrict__ v, const float* __restrict__ d, SolverCfg cfg, double* __restrict__ part,
                const DevState* __restrict__ st, int pf) {
    using namespace c4w;
    extern __shared__ __align__(16) unsigned char smraw[];
    float2* blk = reinterpret_cast<float2*>(smraw);
    float2* scr = reinterpret_cast<float2*>(smraw + SCR_OFF);
    float4* tw = reinterpret_cast<float4*>(smraw + TW_OFF);
    __shared__ double sred[16][KC];
    __shared__ double smom[16][4];
    __shared__ float sgam[KC];
    __shared__ LsWarpQ<2> wq[8];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_rows_in, s_peer_free;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = c4_rank();
    const int64_t cid = c4_id(), ncl = c4_count();
    const bool err = st->numeric_error != 0;
    int base, cnt;
    ls_pass_range(0, st->keff, cfg, base, cnt);
    ktime_start(st, 1);
    build_twiddles4<N, false>(tw);
    if (tid < KC) sgam[tid] = (float)trial_gamma(cfg.gamma0, cfg.tau, base + tid);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&s_tmem))),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&s_rows_in))),
                     "r"(4 * (NF / 32)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(&s_peer_free))),
                     "r"(4 * (NF / 32)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    uint32_t cb[4], rin[4], pfr[4];
    {
        const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(blk));
        const uint32_t a0 = static_cast<uint32_t>(__cvta_generic_to_shared(&s_rows_in));
        const uint32_t a1 = static_cast<uint32_t>(__cvta_generic_to_shared(&s_peer_free));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            cb[q] = c4_mapa(sb, q);
            rin[q] = c4_mapa(a0, q);
            pfr[q] = c4_mapa(a1, q);
        }
    }
    c4_tc_before();
    __syncthreads();
    c4_tc_after();
    // every CTA's barriers are initialised before any remote arrival
    c4_arrive();
    c4_wait();
    const uint32_t tbase = s_tmem;
    // every CTA of the grid is resident: release the side kernel (k_ls256_side, launched after this one
    // with programmatic stream serialization) onto the SMs the clusters leave idle
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t nfr = err ? 0 : g.n_local;
    const int wq4 = warp & 3, whalf = (warp & 7) >> 2;
    const uint32_t tq = tbase + ((uint32_t)(32 * wq4) << 16) + (uint32_t)(128 * whalf);
    double tot = 0.0;
    double mom[4] = {0.0, 0.0, 0.0, 0.0};
    if (tid < NF) {
        // ============================ FFT group ============================
        const int rt = tid & 15, rrow = tid >> 4;   // 16 sub-threads of a row, 16 rows per round
        int it = 0;
        for (int64_t i = cid; i < nfr; i += ncl, ++it) {
            const int b = it & 1;
            const int j = order[i];
            const int2 s = pos[j];
            // ---- row pass: rows 64 rank + 16 rd + rrow, two rounds in flight
#pragma unroll 1
            for (int rp = 0; rp < 4; rp += 2) {
                float2 xa[R], xb[R];
                const int row0 = (int)rank * QC + rp * RROWS + rrow, row1 = row0 + RROWS;
                window_row<R, T>(eta, g, s, j, row0, rt, probe_s + row0 * N + rt, xa);
                window_row<R, T>(eta, g, s, j, row1, rt, probe_s + row1 * N + rt, xb);
                row_fft_a<N, false, true>(xa, rt, tw, tw + N);
                row_fft_a<N, false, true>(xb, rt, tw, tw + N);
                // exchange through the warp-private scratch rows, outputs stay in registers
                float2* sa = scr + rrow * SLD;
                float2* sb2 = scr + (RROWS + rrow) * SLD;
                __syncwarp();
#pragma unroll
                for (int k1 = 0; k1 < R; ++k1) {
                    sa[T * k1 + (rt ^ (k1 & (T - 1)))] = xa[k1];
                    sb2[T * k1 + (rt ^ (k1 & (T - 1)))] = xb[k1];
                }
                __syncwarp();
#pragma unroll
                for (int n2 = 0; n2 < T; ++n2) {
                    xa[n2] = sa[T * rt + (n2 ^ rt)];
                    xb[n2] = sb2[T * rt + (n2 ^ rt)];
                }
                DFT<T, false>::run(xa);
                DFT<T, false>::run(xb);
                // the owners' blocks are free once every warp of every CTA has read its block of the
                // previous frame
                if (rp == 0 && it > 0) c4_wait_parity(&s_peer_free, (uint32_t)((it - 1) & 1));
                // x[k2] is output column rt + 16 k2: CTA k2 / 4 owns it, local column rt + 16 (k2 % 4)
#pragma unroll
                for (int k2 = 0; k2 < T; ++k2) {
                    const uint32_t o = (uint32_t)(rt + R * (k2 & 3)) * 8u;
                    c4_st2(cb[k2 >> 2] + (uint32_t)(row0 * QC) * 8u + o, xa[k2]);
                    c4_st2(cb[k2 >> 2] + (uint32_t)(row1 * QC) * 8u + o, xb[k2]);
                }
            }
            // this warp's rows are in every owner's block
            __syncwarp();
            if (lane == 0) c4_remote_arrive4(rin);
            // ... and every warp's rows are in mine
            c4_wait_parity(&s_rows_in, (uint32_t)(it & 1));
            // ---- column pass phase 1 on the local 256 x 64 block: 4 rounds, sub-thread t = warp + 8 h
#pragma unroll 1
            for (int rd = 0; rd < 4; ++rd) c4_col1<false>(blk, (rd >> 1) * 32 + lane, warp + 8 * (rd & 1), tw);
            c4_bar_sync(BAR_FFT, NF);
            // ---- slot b must have been read by the epilogue (frame it - 2)
            if (it >= 2) {
                c4_bar_sync(BAR_EMPTY + b, NT);
                c4_tc_after();
            }
            // ---- phase 2 -> tensor memory slot b
#pragma unroll 1
            for (int rd = 0; rd < 4; ++rd) {
                float2 X[R];
                c4_col2<false>(blk, (rd >> 1) * 32 + lane, warp + 8 * (rd & 1), X);
                c4_tmem_st32(tq + (uint32_t)(256 * b + 32 * rd), X);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            c4_tc_before();
            c4_bar_arrive(BAR_FULL + b, NT);
            // this warp is done reading my block: the peers may overwrite it with the next frame
            __syncwarp();
            if (lane == 0) c4_remote_arrive4(pfr);
        }
    } else {
        // ============================ epilogue group ============================
        const int ew = warp - 8;   // = the FFT warp whose outputs this warp reads
        const float eps2 = (float)(cfg.eps * cfg.eps);
        int nmine = 0;
        for (int64_t i = cid; i < nfr; i += ncl) ++nmine;
        // (no cnt guard: the FFT group's hand-off needs the epilogue's arrivals on every frame)
        trial_dispatch(cnt, cfg, [&]<int KT, bool LSE, bool QG>() {
            float gk[KT];
#pragma unroll
            for (int k = 0; k < KT; ++k) gk[k] = sgam[k];
            const uint64_t pol = l2_evict_first();   // u, d read once, v written once per pass
            // u, d of one group of 4 elements: frame jf, round rd (column 64 rank + 32 (rd / 2) + lane,
            // rows t + 16 k2 with t = ew + 8 (rd % 2)), elements k2 = 4 gi .. 4 gi + 3.  The loads run
            // one group ahead ACROSS rounds and frames (the next round's / frame's first group is issued
            // during the last group of the current one), so no round starts on an exposed L2 latency.
            auto elem_base = [&](int64_t jf, int rd) -> int64_t {
                return jf * (int64_t)(N * N) + (int64_t)(ew + 8 * (rd & 1)) * N + (int64_t)rank * QC + (rd >> 1) * 32 +
                       lane;
            };
            float2 un[4];
            float dn[4];
            auto load_group = [&](int64_t jf, int rd, int gi) {
                const int64_t o = elem_base(jf, rd) + (int64_t)gi * 4 * R * N;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    un[e] = ld2_hint_na(u + o + e * R * N, pol);
                    dn[e] = ld1_hint_na(d + o + e * R * N, pol);
                }
            };
            if (nmine > 0) load_group(order[cid], 0, 0);
            int it = 0;
            for (int64_t i = cid; i < nfr; i += ncl, ++it) {
                const int b = it & 1;
                const int64_t jf = order[i];
                const int64_t jnext = i + ncl < nfr ? (int64_t)order[i + ncl] : -1;
                // this frame's u, d into L2: CTA r prefetches full rows [64 r, 64 r + 64) (contiguous
                // 128 + 64 KB), so the cluster covers the frame once and every CTA finds its column
                // quarter in L2 (per-CTA strided quarters, 256 small prefetches, measured slower)
                if (pf) {
                    const int64_t ro = jf * (int64_t)(N * N) + (int64_t)rank * QC * N;
                    if (ew == 0) prefetch_l2_frame(u + ro, QC * N * 8, lane);
                    else if (ew == 1) prefetch_l2_frame(d + ro, QC * N * 4, lane);
                }
                c4_bar_sync(BAR_FULL + b, NT);
                c4_tc_after();
#pragma unroll 1
                for (int rd = 0; rd < 4; ++rd) {
                    float2* __restrict__ vb = v + elem_base(jf, rd);
                    float S[KC];
                    LsMom m;
#pragma unroll
                    for (int k = 0; k < KC; ++k) S[k] = 0.f;
                    LsQState qs;
#pragma unroll 1
                    for (int gi = 0; gi < T / 4; ++gi) {
                        const int go = gi * 4 * R * N;
                        float2 uc[4];
                        float dc[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            uc[e] = un[e];
                            dc[e] = dn[e];
                        }
                        if (gi + 1 < T / 4)
                            load_group(jf, rd, gi + 1);
                        else if (rd + 1 < 4)
                            load_group(jf, rd + 1, 0);
                        else if (jnext >= 0)
                            load_group(jnext, 0, 0);
                        float2 X[4];
                        c4_tmem_ld8(tq + (uint32_t)(256 * b + 32 * rd + 8 * gi), X);
#pragma unroll
                        for (int e = 0; e < 4; ++e) st2_hint(vb + go + e * R * N, X[e], pol);
                        ls_push<KT, LSE, QG>(wq[ew], qs, slice<0, 2>(uc), slice<0, 2>(X), slice<0, 2>(dc), gk, eps2,
                                             S, m, lane);
                        ls_push<KT, LSE, QG>(wq[ew], qs, slice<2, 2>(uc), slice<2, 2>(X), slice<2, 2>(dc), gk, eps2,
                                             S, m, lane);
                    }
                    ls_flush<KT, LSE, QG>(wq[ew], qs, gk, eps2, S, m, lane);
                    ls_run_out_r<(KT <= 8 ? 8 : KC)>(S, m, tot, mom, lane);
                }
                // slot b read: the FFT group may overwrite it (frame it + 2) -- no arrival without a waiter
                c4_tc_before();
                if (it + 2 < nmine) c4_bar_arrive(BAR_EMPTY + b, NT);
            }
        });
    }
    // no CTA leaves while a peer may still arrive on its barriers or store into its block
    c4_tc_before();
    __syncthreads();
    c4_tc_after();
    c4_arrive();
    c4_wait();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TMEM_COLS));
    ktime_end(st, 1);
    if (cnt <= 8)   // = KT <= 8 (trial_dispatch_k)
        ls_block_out_r<8, 16>(tot, mom, sred, smom, part);
    else
        ls_block_out_r<KC, 16>(tot, mom, sred, smom, part);
}

// ----------------------------------------------------------------------------------------
// launchers: grid = 4 x (resident clusters, capped by the frame count)
// ----------------------------------------------------------------------------------------
template <typename K>
static int c256_grid(K* kern, int64_t nfr) {
    static int cached = 0;
    if (cached == 0) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c256::DYN_BYTES) !=
            cudaSuccess)
            return -1;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(4 * 148, 1, 1);
        cfg.blockDim = dim3(c256::NT, 1, 1);
        cfg.dynamicSmemBytes = c256::DYN_BYTES;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 4;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl <= 0) {
            cudaGetLastError();
            ncl = 148 / 4;
        }
        cached = ncl;
    }
    const int64_t ncl = nfr < cached ? (nfr > 0 ? nfr : 1) : cached;
    return (int)(4 * ncl);
}

static int c256ws_grid(int64_t nfr) {
    static int cached = 0;
    if (cached == 0) {
        if (cudaFuncSetAttribute(k_ls_c256ws, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c4w::DYN_BYTES) !=
            cudaSuccess)
            return -1;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(4 * 148, 1, 1);
        cfg.blockDim = dim3(c4w::NT, 1, 1);
        cfg.dynamicSmemBytes = c4w::DYN_BYTES;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 4;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_ls_c256ws, &cfg) != cudaSuccess || ncl <= 0) {
            cudaGetLastError();
            ncl = 148 / 4;
        }
        cached = ncl;
    }
    const int64_t ncl = nfr < cached ? (nfr > 0 ? nfr : 1) : cached;
    return (int)(4 * ncl);
}

static bool c256_ws() {
    static const bool ws = !(getenv("PTYGER_C256_WS") && atoi(getenv("PTYGER_C256_WS")) == 0);
    return ws;
}

// Side kernel on the SMs the clusters leave idle (kernels_n256.cu k_ls256_side): it takes the last
// n2 = nfr * share / 1000 frames of the canonical order (SolverCfg::side, PTYGER_C256_SIDE at init,
// default 110), one CTA per idle SM; off when fewer
// frames than side CTAs.  Measured at the large view (profiles/r2_history.md, session 3): the side
// kernel needs ~71 us per frame and SM against ~75-80 SM-us in the clusters, but the clusters slow by
// ~7 % while it runs (the board is at its power cap), so the pass gains ~2.5 %: 55.9 ms without, 54.6 /
// 54.4 ms at 100 / 120 per mille, 61.9 ms at 140 (the side kernel becomes the tail).
static void c256_side_split(int64_t nfr, int cgrid, int share, int64_t& n1, int& sgrid) {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = -1;
    }
    n1 = nfr;
    sgrid = 0;
    const int idle = sms - cgrid;
    if (!c256_ws() || idle <= 0 || share <= 0) return;
    const int64_t n2 = nfr * share / 1000;
    if (n2 < idle) return;
    n1 = nfr - n2;
    sgrid = idle;
}

int c256_ls_side(int64_t nfr, int side) {
    if (!c256_ws()) return 0;
    const int cg = c256ws_grid(nfr);
    if (cg < 0) return 0;
    int64_t n1;
    int sg;
    c256_side_split(nfr, cg, side, n1, sg);
    return sg;
}

int c256_ls_parts(int64_t nfr, int side) {
    if (!c256_ws()) return c256_grid(k_ls_c256, nfr);
    const int cg = c256ws_grid(nfr);
    if (cg < 0) return cg;
    int64_t n1;
    int sg;
    c256_side_split(nfr, cg, side, n1, sg);
    return cg + sg;
}

int launch_ls_c256(const Geometry& g, const float2* eta, const float2* probe_s, const int2* pos, const int* order,
                   const float2* u, float2* v, const float* d, const SolverCfg& c, double* part, const DevState* st,
                   cudaStream_t s) {
    if (c256_ws()) {
        const int grid = c256ws_grid(g.n_local);
        if (grid < 0) return -1;
        static const int pf = getenv("PTYGER_C256_PF") ? atoi(getenv("PTYGER_C256_PF")) : 1;
        int64_t n1;
        int sg;
        c256_side_split(g.n_local, grid, c.side, n1, sg);
        Geometry g1 = g;
        g1.n_local = n1;
        k_ls_c256ws<<<grid, c4w::NT, c4w::DYN_BYTES, s>>>(g1, eta, probe_s, pos, order, u, v, d, c, part, st, pf);
        if (cudaGetLastError() != cudaSuccess) return -1;
        if (sg > 0)
            return launch_ls256_side(g, eta, probe_s, pos, order, u, v, d, c, part + (size_t)grid * LSP, st, n1, sg, s);
        return 0;
    }
    const int grid = c256_grid(k_ls_c256, g.n_local);
    if (grid < 0) return -1;
    k_ls_c256<<<grid, c256::NT, c256::DYN_BYTES, s>>>(g, eta, probe_s, pos, order, u, v, d, c, part, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pty
