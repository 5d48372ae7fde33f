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
