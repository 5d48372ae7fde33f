// k_ls for N = 128: the LS-stage frame kernel (Alg.1 659-668, Eq.7) with the forward 2-D FFT
// ordered COLUMNS FIRST so that its last pass produces whole rows, and a TMA ring that streams
// the u and d rows those rows need.
//
//   column pass   x = p * eta[window s_j] read straight from global (L2-resident object, lanes =
//                 32 consecutive columns: coalesced), radix-16 x radix-8 over the rows; phase 2
//                 writes its 8 outputs back into the 8 rows it read (thread-private, no barrier),
//                 which stores logical row k in storage row sigma(k) = 8 (k mod 16) + floor(k/16).
//   row pass      storage row s (logical row k(s)) -> row DFT with the results kept in registers.
//   epilogue      v = X/N to HBM; u, d of the same pixels from the ring; LS screening terms
//                 (dev.cuh ls_screen) for K trials; fp64 partials as in the generic k_ls.
// The ring holds 3 chunks of 16 storage rows (u rows 1088-B stride, d rows 544-B stride,
// 26 KB per chunk); the group that empties a slot issues the chunk three ahead, so the u/d
// stream runs during the column pass of the frame that needs it.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev.cuh"
#include "tma.cuh"

namespace pty {

namespace l128 {
constexpr int N = 128, R = 16, T = 8, LD = 136;
constexpr int ROWS = 16, CHUNKS = N / ROWS;
constexpr int UST = 1024 + 64, DST = 512 + 32;
constexpr int SLOT_U = 0, SLOT_D = ROWS * UST;
constexpr int SLOT_BYTES = ROWS * UST + ROWS * DST;  // 26112
constexpr int NSLOT = 3;
constexpr int FRAME_BYTES = N * LD * 8;
constexpr int RING_OFF = FRAME_BYTES + N * 8;
constexpr int BAR_OFF = RING_OFF + NSLOT * SLOT_BYTES;
// Chunk c waits on barrier c % NBAR.  NBAR = lcm(issue distance NSLOT = 3, 4 consumer groups):
// the barrier's previous use, chunk c - 12, was consumed by the waiting group itself (so a parity
// wait cannot match a stale phase), and it landed before chunk c - 9, c - 6, c - 3 were issued in
// turn (so the issuer of c, which consumed c - 3, never arms a barrier whose phase is still open).
constexpr int NBAR = 12;
constexpr size_t SMEM = BAR_OFF + NBAR * 8;
static_assert(SMEM <= 232448, "exceeds the 227 KB per-CTA shared memory");
__device__ __forceinline__ int logical_row(int s) { return (s >> 3) + 16 * (s & 7); }
}  // namespace l128

template <int K>
__global__ void __launch_bounds__(512, 1) k_ls128(Geometry g, const float2* __restrict__ eta,
                                                  const float2* __restrict__ probe, const int2* __restrict__ pos,
                                                  const int* __restrict__ order, const float2* __restrict__ u,
                                                  float2* __restrict__ v, const float* __restrict__ d, SolverCfg cfg,
                                                  double* __restrict__ part, const DevState* __restrict__ st) {
    using namespace l128;
    extern __shared__ __align__(128) unsigned char sm[];
    float2* sf = reinterpret_cast<float2*>(sm);
    float2* tw = reinterpret_cast<float2*>(sm + FRAME_BYTES);
    unsigned char* ring = sm + RING_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BAR_OFF);
    __shared__ double sred[16][2 * K];
    __shared__ double smom[16][3];
    __shared__ float sgam[K];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp = tid >> 7, gtid = tid & 127;
    const bool err = st->numeric_error != 0;
    const int64_t nfr = err ? 0 : g.n_local;
    const int64_t nmine = nfr > (int64_t)blockIdx.x ? (nfr - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nchunks = nmine * CHUNKS;
    const float scale = 1.0f / (float)N;
    const float eps2 = (float)(cfg.eps * cfg.eps);

    // chunk c: frame fi = c / 8 (processing order), storage rows 16 q .. 16 q + 15 (q = c % 8)
    auto issue = [&](int64_t c) {
        const int64_t fi = c / CHUNKS;
        const int q = (int)(c % CHUNKS);
        const int64_t j = order[(int64_t)blockIdx.x + fi * gridDim.x];
        const int sid = (int)(c % NSLOT);
        unsigned char* slot = ring + sid * SLOT_BYTES;
        uint64_t* b = bar + (c % NBAR);
        mbar_arrive_expect_tx(b, ROWS * (1024u + 512u));
        for (int r = 0; r < ROWS; ++r) {
            const int64_t off = j * N * N + (int64_t)logical_row(q * ROWS + r) * N;
            bulk_g2s(slot + SLOT_U + r * UST, u + off, 1024, b);
            bulk_g2s(slot + SLOT_D + r * DST, d + off, 512, b);
        }
    };

    build_twiddles<N>(tw);
    if (tid < K) sgam[tid] = (float)trial_gamma(cfg.gamma0, cfg.tau, tid);
    if (tid == 0) {
        for (int i = 0; i < NBAR; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0)
        for (int64_t c = 0; c < NSLOT && c < nchunks; ++c) issue(c);

    double tot = 0.0, md = 0.0, ma = 0.0, mb = 0.0;
    for (int64_t fi = 0; fi < nmine; ++fi) {
        const int64_t j = order[(int64_t)blockIdx.x + fi * gridDim.x];
        const int2 s = pos[j];
        // ---- column pass, phase 1 from global: x = p * eta[window]
#pragma unroll 1
        for (int rd = 0; rd < 2; ++rd) {
            const int t = warp % T;
            const int c = rd * 64 + (warp / T) * 32 + lane;
            const float2* src = eta + (int64_t)(s.x + t) * g.W + s.y + c;
            const float2* pp = probe + t * N + c;
            float2 x[R];
#pragma unroll
            for (int n1 = 0; n1 < R; ++n1) x[n1] = cmul(ldg2(pp + T * n1 * N), ldg2(src + (int64_t)T * n1 * g.W));
            DFT<R, false>::run(x);
#pragma unroll
            for (int k1 = 1; k1 < R; ++k1) x[k1] = twmul<false>(x[k1], tw[t * k1]);
#pragma unroll
            for (int k1 = 0; k1 < R; ++k1) sf[(T * k1 + t) * LD + c] = x[k1];
        }
        __syncthreads();
        // ---- column pass, phase 2: results back into the rows just read (storage row sigma(k))
#pragma unroll 1
        for (int rd = 0; rd < 2; ++rd) {
            const int t = warp % T;
            const int c = rd * 64 + (warp / T) * 32 + lane;
#pragma unroll
            for (int jj = 0; jj < R / T; ++jj) {
                float2* base = sf + (64 * jj + 8 * t) * LD + c;
                float2 b[T];
#pragma unroll
                for (int n2 = 0; n2 < T; ++n2) b[n2] = base[n2 * LD];
                DFT<T, false>::run(b);
#pragma unroll
                for (int k2 = 0; k2 < T; ++k2) base[k2 * LD] = b[k2];
            }
        }
        __syncthreads();
        // ---- row pass (registers) + epilogue fed by the ring
#pragma unroll 1
        for (int rd = 0; rd < 2; ++rd) {
            const int q = rd * 4 + grp;
            const int srow = q * ROWS + (gtid >> 3), t = gtid & 7;
            const int k = logical_row(srow);
            float2 X[R];
            float2* sr = sf + srow * LD;
#pragma unroll
            for (int n1 = 0; n1 < R; ++n1) X[n1] = sr[T * n1 + t];
            row_fft_regs<N, false>(X, sr, t, tw);
            const int64_t cc = fi * CHUNKS + q;
            const int sid = (int)(cc % NSLOT);
            mbar_wait(&bar[cc % NBAR], (uint32_t)((cc / NBAR) & 1));
            const unsigned char* slot = ring + sid * SLOT_BYTES;
            const float2* su = reinterpret_cast<const float2*>(slot + SLOT_U + (srow & 15) * UST);
            const float* sd = reinterpret_cast<const float*>(slot + SLOT_D + (srow & 15) * DST);
            float2 uu[R];
            float dd[R];
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int col = (i / T) * T + t + R * (i % T);
                uu[i] = su[col];
                dd[i] = sd[col];
            }
            named_bar_sync(1 + grp, 128);
            if (gtid == 0 && cc + NSLOT < nchunks) {
                fence_proxy_async();
                issue(cc + NSLOT);
            }
            float S[K], A[K];
            float sd_ = 0.f, sa_ = 0.f, sb_ = 0.f;
#pragma unroll
            for (int kk = 0; kk < K; ++kk) S[kk] = A[kk] = 0.f;
            float2* vrow = v + j * N * N + (int64_t)k * N;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int col = (i / T) * T + t + R * (i % T);
                const float2 vv = cscale(X[i], scale);
                vrow[col] = vv;
                ls_screen<K>(uu[i], vv, dd[i], sgam, eps2, S, A, sd_, sa_, sb_);
            }
            double dv[2 * K];
#pragma unroll
            for (int kk = 0; kk < K; ++kk) {
                dv[kk] = (double)S[kk];
                dv[K + kk] = (double)A[kk];
            }
            tot += warp_reduce_scatter<2 * K>(dv, lane);
            md += (double)sd_;
            ma += (double)sa_;
            mb += (double)sb_;
        }
        __syncthreads();
    }
    constexpr int P = Log2<2 * K>::value;
    constexpr int G = 32 >> P;
    if ((lane & (G - 1)) == 0) sred[warp][lane >> (5 - P)] = tot;
    md = warp_sum(md);
    ma = warp_sum(ma);
    mb = warp_sum(mb);
    if (lane == 0) {
        smom[warp][0] = md;
        smom[warp][1] = ma;
        smom[warp][2] = mb;
    }
    __syncthreads();
    constexpr int WID = 2 * K + 3;
    if (tid < 2 * K) {
        double a = 0.0;
        for (int w = 0; w < 16; ++w) a += sred[w][tid];
        part[(int64_t)blockIdx.x * WID + tid] = a;
    } else if (tid < WID) {
        double a = 0.0;
        for (int w = 0; w < 16; ++w) a += smom[w][tid - 2 * K];
        part[(int64_t)blockIdx.x * WID + tid] = a;
    }
}

int launch_ls128(const Geometry& g, const float2* eta, const float2* probe, const int2* pos, const int* order,
                 const float2* u, float2* v, const float* d, const SolverCfg& c, double* part, int grid,
                 const DevState* st, cudaStream_t s) {
    if (c.K == 8) {
        if (cudaFuncSetAttribute(k_ls128<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l128::SMEM) !=
            cudaSuccess)
            return -1;
        k_ls128<8><<<grid, 512, l128::SMEM, s>>>(g, eta, probe, pos, order, u, v, d, c, part, st);
    } else if (c.K == 16) {
        if (cudaFuncSetAttribute(k_ls128<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l128::SMEM) !=
            cudaSuccess)
            return -1;
        k_ls128<16><<<grid, 512, l128::SMEM, s>>>(g, eta, probe, pos, order, u, v, d, c, part, st);
    } else {
        return -2;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pty
