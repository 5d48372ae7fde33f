// Peer-memory transport (kernels_p2p.cu): exchange-window layout shared by the host runtime and the
// kernels.  Every rank's window is one cudaMalloc allocation exported with CUDA IPC:
//   [flags u64 [P2P_MAX_RANKS][P2P_CHANNELS] | mailbox f64 [2][P2P_MAX_RANKS][P2P_MBW] |
//    full object c64 [2][H*W] | recv0 c64 [band rows from the left neighbour * W] | recv1 (right)]
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace pty {

constexpr int P2P_MAX_RANKS = 8;
constexpr int P2P_CHANNELS = 4;
constexpr int P2P_CH_BAND = 0, P2P_CH_SCALAR = 1, P2P_CH_GATHER = 2;
constexpr int P2P_MBW = 32;   // doubles per mailbox slot (>= LSW)
static_assert(P2P_MBW >= LSW, "mailbox slot too small");

struct P2PView {
    unsigned char* win[P2P_MAX_RANKS];   // every rank's window mapped into this process (own included)
    int world, rank;
    int64_t off_flags, off_mail, off_full, full_elems;
    int64_t off_recv0[P2P_MAX_RANKS], off_recv1[P2P_MAX_RANKS];
};

#ifdef __CUDACC__
__device__ __forceinline__ void flag_release(unsigned long long* f, unsigned long long e) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
}
__device__ __forceinline__ unsigned long long* win_flag(const P2PView& v, int owner, int src, int ch) {
    return reinterpret_cast<unsigned long long*>(v.win[owner] + v.off_flags) + src * P2P_CHANNELS + ch;
}
__device__ __forceinline__ unsigned long long flag_acquire(const unsigned long long* f) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
    return v;
}
// bounded spin: a lost peer becomes a launch failure (trap) after ~tens of seconds, not a hang
__device__ __forceinline__ void flag_wait(const unsigned long long* f, unsigned long long e) {
    unsigned long long spins = 0;
    while (flag_acquire(f) < e) {
        if (++spins == (1ull << 36)) __trap();
    }
}

__device__ __forceinline__ double* win_mail(const P2PView& v, int owner, int par, int src) {
    return reinterpret_cast<double*>(v.win[owner] + v.off_mail) + ((int64_t)par * v.world + src) * P2P_MBW;
}

// In-place fp64 sum over ranks of buf[0..count) by ONE block: own values into slot [rank] of every
// window's mailbox (epoch parity), flags, wait for all ranks, sum the slots in rank order.
__device__ __forceinline__ void p2p_allreduce_block(double* buf, int count, const P2PView& v, DevState* st) {
    const unsigned long long e = st->p2p_epoch[P2P_CH_SCALAR];
    const int par = (int)(e & 1);
    __syncthreads();
    for (int r = 0; r < v.world; ++r) {
        double* m = win_mail(v, r, par, v.rank);
        for (int i = threadIdx.x; i < count; i += blockDim.x) m[i] = buf[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int r = 0; r < v.world; ++r) flag_release(win_flag(v, r, v.rank, P2P_CH_SCALAR), e);
        for (int r = 0; r < v.world; ++r) flag_wait(win_flag(v, v.rank, r, P2P_CH_SCALAR), e);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        double sum = 0.0;
        for (int r = 0; r < v.world; ++r) sum += win_mail(v, v.rank, par, r)[i];
        buf[i] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) st->p2p_epoch[P2P_CH_SCALAR] = e + 1;
}

// Grid-wide "all blocks stored" -> the last block raises the flags of channel ch (epoch e) in the
// windows of the ranks to[0..nto).  st->p2p_done[ch] counts the blocks.
__device__ __forceinline__ void grid_signal(DevState* st, int ch, const P2PView& v, const int* to, int nto,
                                            unsigned long long e) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned int prev = atomicAdd(&st->p2p_done[ch], 1u);
        if (prev == gridDim.x - 1) {
            st->p2p_done[ch] = 0;
            __threadfence_system();
            for (int i = 0; i < nto; ++i) flag_release(win_flag(v, to[i], v.rank, ch), e);
        }
    }
}
#endif

// band receive: wait for the neighbours' flags of the current band epoch, then advance it
int launch_p2p_wait_band(const P2PView& v, DevState* st, int from_left, int from_right, cudaStream_t s);
int launch_p2p_allreduce(double* buf, int count, const P2PView& v, DevState* st, cudaStream_t s);
// gathers owned rows [lo, hi) (global) of src into every window's full buffer of the current epoch
// parity; returns that parity through *par_out (host-known: the gather epoch counter is mirrored)
int launch_p2p_gather(const float2* src, int64_t st_lo, int64_t lo, int64_t hi, int64_t W, const P2PView& v,
                      DevState* st, int grid, cudaStream_t s);

}  // namespace pty
