// Peer-memory transport for world > 1 (PTYGER_TRANSPORT_P2P): the iteration's exchanges are done by
// kernels that store straight into the other ranks' CUDA-IPC-mapped exchange windows and signal with
// epoch flags (system-scope release / acquire), instead of NCCL calls:
//   * band exchange (R#15): k_adj itself stores the partial gradient of the rows a rank shares with
//     a neighbour into that neighbour's receive buffer and its last tile raises the flag (compute and
//     exchange in one kernel); k_p2p_wait then waits for the neighbours' flags before k_band_add;
//   * scalar allreduce (DY sums, LS partials, F0): every rank writes its vector into slot [rank] of
//     every window's mailbox, waits for all flags and sums the slots in rank order, so all ranks get
//     bitwise identical results (k_p2p_allreduce);
//   * object gather (get_object / get_gradient): owned rows into every window's full-object buffer.
// Mailboxes are double-buffered by epoch parity: a rank can only start epoch e + 2 after it has seen
// every peer's epoch e + 1, i.e. after every peer finished reading epoch e.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev.cuh"
#include "p2p.h"

namespace pty {

// ---- band exchange: the stores are fused into k_adj (kernels_misc.cu) -----------------------
// wait for the neighbours' band data (channel ch, from ranks with a band), then advance the epoch
__global__ void k_p2p_wait(P2PView v, DevState* st, int ch, int from_left, int from_right) {
    if (st->numeric_error) return;   // the producing k_adj skipped too (the flag is rank-consistent)
    const unsigned long long e = st->p2p_epoch[ch];
    if (from_left) flag_wait(win_flag(v, v.rank, v.rank - 1, ch), e);
    if (from_right) flag_wait(win_flag(v, v.rank, v.rank + 1, ch), e);
    st->p2p_epoch[ch] = e + 1;
}

// ---- scalar allreduce (fixed rank order) ----------------------------------------------------
__global__ void k_p2p_allreduce(double* buf, int count, P2PView v, DevState* st) {
    p2p_allreduce_block(buf, count, v, st);
}

// ---- object gather: owned rows [lo, hi) of src (storage-local row 0 = global row st_lo) ----------
__global__ void k_p2p_gather_put(const float2* __restrict__ src, int64_t st_lo, int64_t lo, int64_t hi, int64_t W,
                                 P2PView v, DevState* st) {
    const unsigned long long e = st->p2p_epoch[P2P_CH_GATHER];
    const int64_t n = (hi - lo) * W;
    const int64_t par = (int64_t)(e & 1);   // double-buffered: see the file header
    for (int r = 0; r < v.world; ++r) {
        float2* dst = reinterpret_cast<float2*>(v.win[r] + v.off_full) + par * v.full_elems + lo * W;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            dst[i] = src[(lo - st_lo) * W + i];
    }
    int to[P2P_MAX_RANKS];
    for (int r = 0; r < v.world; ++r) to[r] = r;
    grid_signal(st, P2P_CH_GATHER, v, to, v.world, e);
}

__global__ void k_p2p_wait_all(P2PView v, DevState* st, int ch) {
    const unsigned long long e = st->p2p_epoch[ch];
    for (int r = 0; r < v.world; ++r) flag_wait(win_flag(v, v.rank, r, ch), e);
    st->p2p_epoch[ch] = e + 1;
}

// ---- launchers -------------------------------------------------------------------------------
int launch_p2p_wait_band(const P2PView& v, DevState* st, int from_left, int from_right, cudaStream_t s) {
    k_p2p_wait<<<1, 1, 0, s>>>(v, st, P2P_CH_BAND, from_left, from_right);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_p2p_allreduce(double* buf, int count, const P2PView& v, DevState* st, cudaStream_t s) {
    k_p2p_allreduce<<<1, 32, 0, s>>>(buf, count, v, st);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

int launch_p2p_gather(const float2* src, int64_t st_lo, int64_t lo, int64_t hi, int64_t W, const P2PView& v,
                      DevState* st, int grid, cudaStream_t s) {
    k_p2p_gather_put<<<grid, 256, 0, s>>>(src, st_lo, lo, hi, W, v, st);
    k_p2p_wait_all<<<1, 1, 0, s>>>(v, st, P2P_CH_GATHER);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace pty
