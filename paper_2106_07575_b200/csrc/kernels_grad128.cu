// k_grad for N = 128 with a TMA (bulk-copy) input ring: the GRAD-stage frame kernel
// (Alg.1 648-649: u <- u + gamma_prev v, r = u - d/u^*, y = conj(p) F^H r; Eq.3 minus the scatter).
//
// Why a ring: one 128x128 complex64 frame (139 KB with padding) fills a CTA's shared memory,
// so only one frame is in flight per SM.  Loading u, v, d straight into registers leaves HBM idle
// while the frame is transformed.  Here the u/v/d rows of a frame are streamed by the TMA engine
// (cp.async.bulk, 16-row chunks of 40 KB) into a 2-slot ring (85 KB) that sits next to the frame
// buffer.  Four groups of 128 threads consume the chunks in order; the group that empties a slot
// immediately issues the chunk two ahead into it, so the copies run continuously, including the
// first chunks of the NEXT frame while this frame's column pass runs.  Rows are copied one by one
// into padded slot rows (u/v stride 1088 B, d stride 544 B) so the ring reads are bank-conflict
// free.  Everything else (FFT, residual, epilogue) is the generic k_grad path.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "dev.cuh"
#include "tma.cuh"

namespace pty {

namespace g128 {
constexpr int N = 128, R = 16, T = 8, LD = 136;
constexpr int ROWS = 16;                       // rows per chunk = rows of one 128-thread group
constexpr int CHUNKS = N / ROWS;               // 8 chunks per frame, 2 rounds x 4 groups
constexpr int UST = 1024 + 64;                 // u / v slot row stride (bytes)
constexpr int DST = 512 + 32;                  // d slot row stride (bytes)
constexpr int SLOT_U = 0, SLOT_V = ROWS * UST, SLOT_D = 2 * ROWS * UST;
constexpr int SLOT_BYTES = 2 * ROWS * UST + ROWS * DST;  // 43520
constexpr int NSLOT = 2;
constexpr int FRAME_BYTES = N * LD * 8;        // 139264
constexpr int RING_OFF = FRAME_BYTES + N * 8;  // after the twiddle table
constexpr int BAR_OFF = RING_OFF + NSLOT * SLOT_BYTES;
constexpr size_t SMEM = BAR_OFF + 64;          // 227392 B
static_assert(SMEM <= 232448, "exceeds the 227 KB per-CTA shared memory");
}  // namespace g128

__global__ void __launch_bounds__(512, 1) k_grad128(Geometry g, float2* __restrict__ u, float2* __restrict__ v,
                                                    const float* __restrict__ d, const float2* __restrict__ probe_s,
                                                    const DevState* __restrict__ st, float eps) {
    using namespace g128;
    extern __shared__ __align__(128) unsigned char sm[];
    float2* sf = reinterpret_cast<float2*>(sm);
    float2* tw = reinterpret_cast<float2*>(sm + FRAME_BYTES);
    unsigned char* ring = sm + RING_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + BAR_OFF);
    if (st->numeric_error) return;
    const float gam = (float)st->gamma;
    const bool upd = gam != 0.0f;
    const int64_t nfr = g.n_local;
    const int64_t nmine = nfr > (int64_t)blockIdx.x ? (nfr - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t nchunks = nmine * CHUNKS;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp = tid >> 7, gtid = tid & 127;
    const uint32_t chunk_bytes = ROWS * ((upd ? 2048u : 1024u) + 512u);
    const float eps2 = eps * eps;

    auto issue = [&](int64_t c) {
        const int64_t fi = c / CHUNKS;
        const int q = (int)(c % CHUNKS);
        const int64_t j = (int64_t)blockIdx.x + fi * gridDim.x;
        unsigned char* slot = ring + (c & 1) * SLOT_BYTES;
        uint64_t* b = bar + (c & 3);
        mbar_arrive_expect_tx(b, chunk_bytes);
        const int64_t off = j * N * N + (int64_t)q * ROWS * N;
        for (int r = 0; r < ROWS; ++r) {
            bulk_g2s(slot + SLOT_U + r * UST, u + off + r * N, 1024, b);
            if (upd) bulk_g2s(slot + SLOT_V + r * UST, v + off + r * N, 1024, b);
            bulk_g2s(slot + SLOT_D + r * DST, d + off + r * N, 512, b);
        }
    };

    ktime_start(st, 0);
    build_twiddles<N>(tw);
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        if (nchunks > 0) issue(0);
        if (nchunks > 1) issue(1);
    }
    for (int64_t fi = 0; fi < nmine; ++fi) {
        const int64_t j = (int64_t)blockIdx.x + fi * gridDim.x;
        // ---- row pass (inverse FFT along rows), fed from the ring
#pragma unroll 1
        for (int rd = 0; rd < 2; ++rd) {
            const int q = rd * 4 + grp;
            const int64_t cc = fi * CHUNKS + q;
            const int sid = (int)(cc & 1);
            // barrier cc % 4 = lcm(issue distance 2, 4 groups): its previous use, chunk cc - 4, was
            // consumed by this same group (no stale-parity match), and it landed before chunk
            // cc - 2 was issued (so the issuer of cc, which consumed cc - 2, arms a closed phase)
            mbar_wait(&bar[cc & 3], (uint32_t)((cc >> 2) & 1));
            const unsigned char* slot = ring + sid * SLOT_BYTES;
            const int rloc = gtid >> 3, t = gtid & 7;
            const int row = q * ROWS + rloc;
            float2 uu[R];
            float dd[R];
            const float2* su = reinterpret_cast<const float2*>(slot + SLOT_U + rloc * UST) + t;
            const float* sd = reinterpret_cast<const float*>(slot + SLOT_D + rloc * DST) + t;
#pragma unroll
            for (int n1 = 0; n1 < R; ++n1) {
                uu[n1] = su[T * n1];
                dd[n1] = sd[T * n1];
            }
            const int64_t base = j * N * N + (int64_t)row * N + t;
            if (upd) {
                const float2* sv = reinterpret_cast<const float2*>(slot + SLOT_V + rloc * UST) + t;
                float2 vv[R];
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) vv[n1] = sv[T * n1];
                named_bar_sync(1 + grp, 128);   // slot consumed by the whole group
                if (gtid == 0 && cc + 2 < nchunks) {
                    fence_proxy_async();
                    issue(cc + 2);
                }
#pragma unroll
                for (int n1 = 0; n1 < R; ++n1) {
                    uu[n1] = make_float2(fmaf(gam, vv[n1].x, uu[n1].x), fmaf(gam, vv[n1].y, uu[n1].y));
                    u[base + T * n1] = uu[n1];
                }
            } else {
                named_bar_sync(1 + grp, 128);
                if (gtid == 0 && cc + 2 < nchunks) {
                    fence_proxy_async();
                    issue(cc + 2);
                }
            }
            float2 x[R];
#pragma unroll
            for (int n1 = 0; n1 < R; ++n1) x[n1] = residual(uu[n1], dd[n1], eps2, g.est);
            row_fft<N, true>(x, sf + row * LD, t, tw);
        }
        __syncthreads();
        // ---- column pass (inverse FFT along columns), epilogue y = conj(p) X / N into v's slot
#pragma unroll 1
        for (int rd = 0; rd < 2; ++rd) {
            const int t = warp % T;
            const int c = rd * 64 + (warp / T) * 32 + lane;
            col_fft_phase1<N, true>(sf + c, t, tw);
        }
        __syncthreads();
#pragma unroll 1
        for (int rd = 0; rd < 2; ++rd) {
            const int t = warp % T;
            const int c = rd * 64 + (warp / T) * 32 + lane;
            float2 X[R];
            col_fft_phase2<N, true>(sf + c, t, X);
#pragma unroll
            for (int qq = 0; qq < R; ++qq) {
                const int k = col_out_row<N>(qq, t);
                const float2 pk = ldg2(probe_s + k * N + c);   // conj(p / N): unitary scale folded in
                v[j * N * N + (int64_t)k * N + c] = cconjmul(pk, X[qq]);
            }
        }
        __syncthreads();
    }
    ktime_end(st, 0);
}

int launch_grad128(const Geometry& g, float2* u, float2* v, const float* d, const float2* probe_s,
                   const DevState* st, float eps, int grid, cudaStream_t s) {
    if (cudaFuncSetAttribute(k_grad128, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g128::SMEM) !=
        cudaSuccess)
        return -1;
    k_grad128<<<grid, 512, g128::SMEM, s>>>(g, u, v, d, probe_s, st, eps);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pty
